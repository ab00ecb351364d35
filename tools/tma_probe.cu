// Probe: TMA 2D tensor loads with SWIZZLE_128B into shared memory at a
// destination that is 128-byte but not 1024-byte aligned -- does it work, and
// which swizzle phase do the rows get?  Also times random 16-row boxes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tools/tma_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <vector>
#include <random>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap tm, int dst_row, int src_row, int box_rows, uint16_t *out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  unsigned char *buf = sm;  // 32 rows x 128 B region, 1024-aligned
  for (int i = threadIdx.x; i < 32 * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(buf)[i] = 0xffffffffu;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(box_rows * 128));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(buf + dst_row * 128)),
        "l"(&tm), "r"(0), "r"(src_row), "r"(smem_u32(&bar))
        : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0,1,0,p;\n}\n"
                 : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
  for (int i = threadIdx.x; i < 32 * 64; i += blockDim.x) out[i] = reinterpret_cast<uint16_t *>(buf)[i];
}

// throughput: every warp loads random 16-row boxes (both 64-col halves) into its own ring
__global__ void __launch_bounds__(256) stream_boxes(const __grid_constant__ CUtensorMap tm, const int *rows, int nbox,
                                                    int stages, unsigned long long *sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int stage_bytes = 2 * 16 * 128;
  unsigned char *ring = sm + warp * stages * stage_bytes;
  __shared__ __align__(8) uint64_t bars[8][8];
  if (lane == 0)
    for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[warp][s])));
  __syncwarp();
  const int gw = blockIdx.x * nw + warp, NW = gridDim.x * nw;
  const int b0 = (int)((long long)nbox * gw / NW), b1 = (int)((long long)nbox * (gw + 1) / NW);
  for (int k = 0; k < b1 - b0; ++k) {
    const int s = k % stages;
    if (k >= stages) {
      uint32_t done = 0, par = ((k / stages) - 1) & 1;
      while (!done)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}\n"
                     : "=r"(done) : "r"(smem_u32(&bars[warp][s])), "r"(par) : "memory");
    }
    if (lane == 0) {
      const int r = rows[b0 + k];
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[warp][s])), "r"(stage_bytes));
      for (int h = 0; h < 2; ++h)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                smem_u32(ring + s * stage_bytes + h * 2048)),
            "l"(&tm), "r"(64 * h), "r"(r), "r"(smem_u32(&bars[warp][s]))
            : "memory");
    }
    __syncwarp();
  }
  const int n = b1 - b0;
  for (int k = (n > stages ? n - stages : 0); k < n; ++k) {
    uint32_t done = 0, par = (k / stages) & 1;
    while (!done)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}\n"
                   : "=r"(done) : "r"(smem_u32(&bars[warp][k % stages])), "r"(par) : "memory");
  }
  if (ring[lane] == 0x7f) sink[0] = 1;
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                             const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  EncodeFn encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&encode, cudaEnableDefault, &q);
  if (!encode) { printf("no encode\n"); return 1; }
  const int64_t nrows = 1 << 22;  // 4M rows x 256 B = 1 GB
  uint16_t *g;
  cudaMalloc(&g, nrows * 256);
  {
    std::vector<uint16_t> h(256 * 128);
    for (int r = 0; r < 256; ++r)
      for (int c = 0; c < 128; ++c) h[r * 128 + c] = (uint16_t)(r * 128 + c);
    cudaMemcpy(g, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  }
  CUtensorMap tm16, tm8;
  cuuint64_t dims[2] = {128, (cuuint64_t)nrows};
  cuuint64_t strides[1] = {256};
  cuuint32_t box16[2] = {64, 16}, box8[2] = {64, 8}, es[2] = {1, 1};
  CUresult r1 = encode(&tm16, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g, dims, strides, box16, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = encode(&tm8, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g, dims, strides, box8, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d %d\n", (int)r1, (int)r2);
  uint16_t *out;
  cudaMalloc(&out, 32 * 64 * 2);
  for (int dst : {0, 3, 8, 5}) {
    probe<<<1, 128, 32 * 128 + 1024>>>(tm8, dst, 10, 8, out);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<uint16_t> h(32 * 64);
    cudaMemcpy(h.data(), out, h.size() * 2, cudaMemcpyDeviceToHost);
    printf("dst_row %d: %s\n", dst, cudaGetErrorString(e));
    if (e != cudaSuccess) return 0;
    for (int r = 0; r < 16; ++r) {
      printf("  slot %2d:", r);
      for (int ch = 0; ch < 8; ++ch) {
        uint16_t v = h[r * 64 + ch * 8];
        if (v == 0xffff) printf("   .  "); else printf(" %2d/%d", v / 128, (v % 128) / 8);
      }
      printf("\n");
    }
  }
  // throughput of random 16-row boxes
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int nbox = 1 << 16;
  std::vector<int> rows(nbox);
  std::mt19937 rng(3);
  for (int i = 0; i < nbox; ++i) rows[i] = (int)(rng() % (nrows / 16)) * 16;
  int *drows;
  cudaMalloc(&drows, nbox * 4);
  cudaMemcpy(drows, rows.data(), nbox * 4, cudaMemcpyHostToDevice);
  unsigned long long *sink;
  cudaMalloc(&sink, 8);
  for (int warps : {4, 8}) for (int stages : {3, 6}) {
    const int smem = warps * stages * 4096 + 1024;
    cudaFuncSetAttribute(stream_boxes, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    stream_boxes<<<nsm, warps * 32, smem>>>(tm16, drows, nbox, stages, sink);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) stream_boxes<<<nsm, warps * 32, smem>>>(tm16, drows, nbox, stages, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("random 16-row boxes (2 x 2KB ops): warps %d stages %d: %.1f GB/s %s\n", warps, stages,
           10.0 * nbox * 4096 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
