// Cycle counts of the select building blocks in ONE CTA (the fused select's tail).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include -o tools/bench_blocks tools/bench_blocks.cu
#include <cstdio>
#include <vector>
#include "../paper_2604_10898_b200/csrc/select_common.cuh"
using namespace zoomr;

__global__ void k_topc(const int *vg, const long long *ag, int nt, int c, int iters, long long *out) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  SmemCarve sm{sm_raw};
  long long *A = sm.take<long long>(nt);
  int *v = sm.take<int>(nt);
  int *grp = sm.take<int>(2 * nt);
  int *hist = sm.take<int>(kHistBins);
  int *scratch = sm.take<int>(40);
  uint8_t *fl = sm.take<uint8_t>(nt);
  for (int i = threadIdx.x; i < nt; i += blockDim.x) { v[i] = vg[i]; A[i] = ag[i]; }
  __shared__ float agv;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) block_topc(v, A, nt, c, fl, hist, grp, scratch, &agv);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}

__global__ void k_index(const int *bdg, const uint8_t *flg, int nt, int T, int iters, int *outidx, int *cnt, long long *out, int cap) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  SmemCarve sm{sm_raw};
  int4 *bds = sm.take<int4>(nt);
  uint8_t *fl = sm.take<uint8_t>(nt);
  int *piece = sm.take<int>(2 * nt);
  int *scratch = sm.take<int>(40);
  for (int i = threadIdx.x; i < nt; i += blockDim.x) { bds[i] = reinterpret_cast<const int4 *>(bdg)[i]; fl[i] = flg[i]; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    block_build_index(reinterpret_cast<const int *>(bds), nt, T, fl, 4, 512, outidx, cap, cnt, piece, scratch, nullptr);
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}

int main() {
  for (int nt : {120, 240}) {
  const int T = 16384 * (nt / 120);
  std::vector<int> v(nt, 0), bd(nt * 4);
  std::vector<long long> a(nt, 0);
  std::vector<uint8_t> fl(nt, 1);
  for (int i = 0; i < nt; ++i) { v[i] = (i * 7) % 5 == 0 ? 0 : 1 + (i % 3); a[i] = (long long)(i * 977 % 1000) << 32; }
  v[5] = 700; v[37] = 650; v[71] = 600; v[100] = 550;
  for (int i = 0; i < nt; ++i) { int s = 4 + 132 * i; bd[4*i] = s; bd[4*i+1] = s + 116; bd[4*i+2] = s + 116; bd[4*i+3] = s + 132; }
  fl[5] = fl[37] = fl[71] = fl[100] = 2;
  int *dv, *dbd, *didx, *dcnt; long long *da, *dout; uint8_t *dfl;
  cudaMalloc(&dv, nt * 4); cudaMalloc(&da, nt * 8); cudaMalloc(&dbd, nt * 16); cudaMalloc(&dfl, nt);
  cudaMalloc(&didx, 65536 * 4); cudaMalloc(&dcnt, 4); cudaMalloc(&dout, 8);
  cudaMemcpy(dv, v.data(), nt * 4, cudaMemcpyHostToDevice); cudaMemcpy(da, a.data(), nt * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dbd, bd.data(), nt * 16, cudaMemcpyHostToDevice); cudaMemcpy(dfl, fl.data(), nt, cudaMemcpyHostToDevice);
  long long h;
  for (int threads : {256, 512}) {
    for (int c : {4, 9}) {
      k_topc<<<1, threads, 32 * 1024>>>(dv, da, nt, c, 50, dout); cudaDeviceSynchronize();
      cudaMemcpy(&h, dout, 8, cudaMemcpyDeviceToHost);
      printf("threads %d: block_topc(nt=%d, c=%d%s) %lld cycles\n", threads, nt, c, c <= kTopcRounds ? ", rounds" : "", h);
    }
    for (int cap : {1 << 16, 1}) {
      k_index<<<1, threads, 32 * 1024>>>(dbd, dfl, nt, T, 50, didx, dcnt, dout, cap); cudaDeviceSynchronize();
      cudaMemcpy(&h, dout, 8, cudaMemcpyDeviceToHost);
      int c; cudaMemcpy(&c, dcnt, 4, cudaMemcpyDeviceToHost);
      printf("threads %d: block_build_index(nt=%d, cap %d) %lld cycles (count %d) %s\n", threads, nt, cap, h, c, cudaGetErrorString(cudaGetLastError()));
    }
  }
  }
  return 0;
}
