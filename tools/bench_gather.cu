// Microbenchmark of the B200 data-movement paths a5 can use for a row gather
// (DESIGN.md section 6 evidence).  Each CTA streams rows of `row_bytes` from a
// large buffer into a shared-memory ring and discards them; rows are either
// contiguous or a random permutation of row-sized slots.
//   mode 0: cp.async.cg 16 B per lane (LDGSTS), warp copies whole rows
//   mode 1: cp.async.bulk (TMA, UBLKCP) one op per run of `run_rows` rows, issued by one lane
//   mode 2: ld.global.nc.v4 into registers (LDG.128), no shared memory
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bench_gather tools/bench_gather.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>
#include <algorithm>
#include <random>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t par) {
  uint32_t done;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}\n"
                 : "=r"(done) : "r"(smem_u32(bar)), "r"(par) : "memory");
  } while (!done);
}

// every warp streams its share of `nrows_total` rows; stage = rows_per_stage rows
template <int MODE>
__global__ void __launch_bounds__(1024) stream_kernel(const char *__restrict__ src, const int *__restrict__ perm,
                                                      int64_t nrows, int row_bytes, int rows_per_stage, int stages,
                                                      int run_rows, unsigned long long *sink) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int stage_bytes = rows_per_stage * row_bytes;
  unsigned char *ring = smem + (size_t)warp * stages * stage_bytes;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + (size_t)nw * stages * stage_bytes) + warp * stages;
  const int64_t gw = (int64_t)blockIdx.x * nw + warp, NW = (int64_t)gridDim.x * nw;
  const int64_t ntiles = nrows / rows_per_stage;
  const int64_t t0 = ntiles * gw / NW, t1 = ntiles * (gw + 1) / NW;
  unsigned long long acc = 0;
  if (MODE == 1 && lane == 0)
    for (int s = 0; s < stages; ++s) mbar_init(&bars[s], 1);
  __syncwarp();
  for (int64_t t = t0; t < t1; ++t) {
    const int64_t k = t - t0;
    const int s = (int)(k % stages);
    unsigned char *st = ring + s * stage_bytes;
    if (MODE == 0) {
      if (k >= stages - 1) asm volatile("cp.async.wait_group %0;" ::"n"(2) : "memory");
      const int cpr = row_bytes / 16;
      for (int x = lane; x < rows_per_stage * cpr; x += 32) {
        const int r = x / cpr, c = x % cpr;
        const int64_t row = perm ? perm[t * rows_per_stage + r] : t * rows_per_stage + r;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(st + r * row_bytes + c * 16)),
                     "l"(src + row * row_bytes + c * 16) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      if (lane == 0) acc += st[0];
    } else if (MODE == 1) {
      if (k >= stages) mbar_wait(&bars[s], (uint32_t)(((k / stages) - 1) & 1));
      if (lane == 0) {
        mbar_expect(&bars[s], (uint32_t)stage_bytes);
        for (int r = 0; r < rows_per_stage; r += run_rows) {
          const int64_t row = perm ? perm[(t * rows_per_stage + r) / run_rows] * (int64_t)run_rows : t * rows_per_stage + r;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           smem_u32(st + r * row_bytes)),
                       "l"(src + row * row_bytes), "r"(run_rows * row_bytes), "r"(smem_u32(&bars[s]))
                       : "memory");
        }
      }
      __syncwarp();
    } else {
      const int cpr = row_bytes / 16;
      uint4 v = make_uint4(0, 0, 0, 0);
      for (int x = lane; x < rows_per_stage * cpr; x += 32) {
        const int r = x / cpr, c = x % cpr;
        const int64_t row = perm ? perm[t * rows_per_stage + r] : t * rows_per_stage + r;
        uint4 w;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w) : "l"(src + row * row_bytes + c * 16));
        v.x ^= w.x;
      }
      acc += v.x;
    }
  }
  if (MODE == 0) asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (MODE == 1) {
    const int64_t n = t1 - t0;
    for (int64_t k = (n > stages ? n - stages : 0); k < n; ++k) mbar_wait(&bars[k % stages], (uint32_t)((k / stages) & 1));
  }
  if (acc == 0x12345) sink[0] = acc;
}

int main(int argc, char **argv) {
  const int64_t bytes = 4ll << 30;
  char *buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  unsigned long long *sink;
  cudaMalloc(&sink, 8);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  struct Cfg { int mode, row_bytes, rows_per_stage, stages, warps, run_rows, random; };
  std::vector<Cfg> cfgs = {
      {0, 256, 32, 3, 4, 1, 0}, {0, 256, 32, 3, 8, 1, 0}, {0, 256, 16, 6, 8, 1, 0}, {0, 256, 32, 3, 8, 1, 1},
      {0, 256, 16, 4, 12, 1, 1}, {0, 256, 16, 3, 16, 1, 1},
      {1, 256, 32, 3, 4, 32, 0}, {1, 256, 32, 3, 8, 32, 0}, {1, 256, 32, 3, 8, 16, 1}, {1, 256, 32, 3, 8, 8, 1},
      {1, 256, 32, 3, 8, 4, 1}, {1, 256, 32, 3, 8, 1, 1}, {1, 256, 32, 3, 16, 1, 1}, {1, 256, 16, 4, 12, 16, 1},
      {2, 256, 32, 1, 8, 1, 0}, {2, 256, 32, 1, 16, 1, 1}, {2, 256, 32, 1, 32, 1, 1},
  };
  const int row_bytes = 256;
  const int64_t nrows = bytes / row_bytes / 2;  // read 2 GB per launch
  int *perm_rows = nullptr, *perm_runs[5] = {};
  {
    std::vector<int> h(nrows);
    for (int64_t i = 0; i < nrows; ++i) h[i] = (int)i;
    std::mt19937 rng(1);
    std::shuffle(h.begin(), h.end(), rng);
    cudaMalloc(&perm_rows, nrows * 4);
    cudaMemcpy(perm_rows, h.data(), nrows * 4, cudaMemcpyHostToDevice);
    for (int rr : {4, 8, 16}) {
      const int64_t nr = nrows / rr;
      std::vector<int> g(nr);
      for (int64_t i = 0; i < nr; ++i) g[i] = (int)i;
      std::shuffle(g.begin(), g.end(), rng);
      int *d;
      cudaMalloc(&d, nr * 4);
      cudaMemcpy(d, g.data(), nr * 4, cudaMemcpyHostToDevice);
      perm_runs[rr == 4 ? 0 : rr == 8 ? 1 : 2] = d;
    }
  }
  for (auto c : cfgs) {
    const size_t smem = (size_t)c.warps * c.stages * c.rows_per_stage * c.row_bytes + c.warps * c.stages * 8;
    if (smem > 227 * 1024) { printf("skip smem %zu\n", smem); continue; }
    const int *perm = nullptr;
    if (c.random) {
      if (c.mode == 1 && c.run_rows > 1) perm = perm_runs[c.run_rows == 4 ? 0 : c.run_rows == 8 ? 1 : 2];
      else perm = perm_rows;
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto launch = [&]() {
      if (c.mode == 0) {
        cudaFuncSetAttribute(stream_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        stream_kernel<0><<<nsm, c.warps * 32, smem>>>(buf, perm, nrows, row_bytes, c.rows_per_stage, c.stages, 1, sink);
      } else if (c.mode == 1) {
        cudaFuncSetAttribute(stream_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        stream_kernel<1><<<nsm, c.warps * 32, smem>>>(buf, perm, nrows, row_bytes, c.rows_per_stage, c.stages, c.run_rows, sink);
      } else {
        stream_kernel<2><<<nsm, c.warps * 32, 0>>>(buf, perm, nrows, row_bytes, c.rows_per_stage, c.stages, 1, sink);
      }
    };
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    printf("mode %d rows/stage %2d stages %d warps %2d run %2d random %d : %7.1f GB/s %s\n", c.mode, c.rows_per_stage,
           c.stages, c.warps, c.run_rows, c.random, 5.0 * nrows * row_bytes / (ms * 1e-3) / 1e9,
           err == cudaSuccess ? "" : cudaGetErrorString(err));
  }
  return 0;
}
