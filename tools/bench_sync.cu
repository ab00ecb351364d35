// Latency of block-level primitives in ONE CTA (the fused select's tail runs in one CTA).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ int block_excl_scan(int x, int *tmp, int *total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, incl, o); if (lane >= o) incl += y; }
  if (lane == 31) tmp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int wt = lane < nw ? tmp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, wt, o); if (lane >= o) wt += y; }
    if (lane < nw) tmp[lane] = wt;
  }
  __syncthreads();
  const int ex = (warp ? tmp[warp - 1] : 0) + incl - x;
  *total = tmp[nw - 1];
  __syncthreads();
  return ex;
}
__global__ void k(long long *out, int iters) {
  __shared__ int tmp[40];
  int acc = threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { int tot; acc = block_excl_scan(acc & 7, tmp, &tot) + tot; }
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t2 = clock64();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / iters; out[1] = (t2 - t1) / iters; out[2] = acc; }
}
int main() {
  long long *d, h[3];
  cudaMalloc(&d, 24);
  for (int threads : {128, 256, 512, 1024}) {
    k<<<1, threads>>>(d, 100); cudaDeviceSynchronize();
    k<<<1, threads>>>(d, 1000); cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("threads %4d: block_excl_scan %lld cycles, __syncthreads %lld cycles\n", threads, h[0], h[1]);
  }
  return 0;
}
