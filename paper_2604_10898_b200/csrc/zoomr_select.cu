// a3 -- global consensus top-c (Alg.1 @P:418-419).
//
// I_all = {i : v_i > 0}, I_c = the c summaries with the most votes
// (P:64), ties broken by the aggregated score A_i, then by the smaller (older)
// index (readings Q2, Q3); I_s = I_all \ I_c.
//
// One CTA per sequence.  The N_t (v, A, i) keys are sorted in shared memory by
// a block-wide bitonic network in the total order (v desc, A desc, i asc) --
// integer comparisons only, so the result is exact and deterministic -- and the
// first min(c, |I_all|) voted entries are flagged 2, the rest of I_all 1.
// N_t <= 4096: at most 78 compare-exchange rounds of 1024 threads.
#include "common.cuh"

namespace zoomr {

struct VKey {
  int32_t v;
  int32_t i;
  long long a;
};

// "x comes before y" in (v desc, A desc, i asc)
__device__ __forceinline__ bool before(const VKey &x, const VKey &y) {
  if (x.v != y.v) return x.v > y.v;
  if (x.a != y.a) return x.a > y.a;
  return x.i < y.i;
}

__global__ void __launch_bounds__(1024) select_topc_kernel(
    const int64_t *__restrict__ partial, const int32_t *__restrict__ num_summaries,
    int32_t max_summaries, int32_t n2, int32_t c, uint8_t *__restrict__ flags,
    float *__restrict__ agreeability, int32_t *status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  VKey *key = reinterpret_cast<VKey *>(smem_raw);  // [n2]
  __shared__ long long red_c[32], red_all[32];
  const int b = blockIdx.x;
  int nt = num_summaries[b];
  if (nt > max_summaries || nt < 0) {
    if (threadIdx.x == 0) set_status(status, ZOOMR_ERR_INDEX_RANGE);
    nt = nt < 0 ? 0 : max_summaries;
  }
  const int64_t *votes = partial + (int64_t)b * 2 * max_summaries;
  const int64_t *A = votes + max_summaries;
  uint8_t *fl = flags + (int64_t)b * max_summaries;
  for (int x = threadIdx.x; x < n2; x += blockDim.x) {
    VKey k;
    if (x < nt) {
      k.v = (int32_t)votes[x];
      k.a = A[x];
      k.i = x;
    } else {
      k.v = -1;  // padding sorts last
      k.a = 0;
      k.i = x;
    }
    key[x] = k;
  }
  for (int x = threadIdx.x; x < max_summaries; x += blockDim.x) fl[x] = 0;
  __syncthreads();
  // bitonic sort of n2 (power of two) keys into "before" order
  for (int kk = 2; kk <= n2; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int x = threadIdx.x; x < n2; x += blockDim.x) {
        const int y = x ^ j;
        if (y > x) {
          const VKey kx = key[x], ky = key[y];
          const bool up = (x & kk) == 0;
          if (up ? before(ky, kx) : before(kx, ky)) {
            key[x] = ky;
            key[y] = kx;
          }
        }
      }
      __syncthreads();
    }
  }
  long long vc = 0, vall = 0;
  for (int r = threadIdx.x; r < nt; r += blockDim.x) {
    const VKey k = key[r];
    if (k.v > 0) {  // voted entries come first in the order
      fl[k.i] = (uint8_t)(r < c ? 2 : 1);
      vall += k.v;
      if (r < c) vc += k.v;
    }
  }
  if (agreeability) {
    for (int off = 16; off; off >>= 1) {
      vc += __shfl_xor_sync(0xffffffffu, vc, off);
      vall += __shfl_xor_sync(0xffffffffu, vall, off);
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
      red_c[warp] = vc;
      red_all[warp] = vall;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      long long tc = 0, ta = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        tc += red_c[w];
        ta += red_all[w];
      }
      agreeability[b] = ta > 0 ? (float)((double)tc / (double)ta) : 0.f;
    }
  }
}

}  // namespace zoomr

using namespace zoomr;

extern "C" int zoomr_select_topc(int32_t batch, const int64_t *partial,
                                 const int32_t *num_summaries, int32_t max_summaries, int32_t c,
                                 uint8_t *flags, float *agreeability, int32_t *dev_status,
                                 void *stream) {
  if (batch < 1 || !partial || !num_summaries || !flags || max_summaries < 1 || c < 0)
    return ZOOMR_ERR_INVALID_ARG;
  if (max_summaries > kMaxSummaries) return ZOOMR_ERR_UNSUPPORTED;
  int n2 = 1;
  while (n2 < max_summaries) n2 <<= 1;
  const size_t smem = (size_t)n2 * sizeof(VKey);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(select_topc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int threads = n2 >= 1024 ? 1024 : (n2 < 32 ? 32 : n2);
  select_topc_kernel<<<batch, threads, smem, (cudaStream_t)stream>>>(
      partial, num_summaries, max_summaries, n2, c, flags, agreeability, dev_status);
  return launch_status();
}
