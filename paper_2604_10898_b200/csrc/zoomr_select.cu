// a3 -- global consensus top-c (Alg.1 @P:418-419).
//
// I_all = {i : v_i > 0}, I_c = the c summaries with the most votes
// (P:64), ties broken by the aggregated score A_i, then by the smaller (older)
// index (readings Q2, Q3); I_s = I_all \ I_c.
//
// One CTA per sequence: the N_t (v, A) pairs are loaded into shared memory and
// block_topc (select_common.cuh) finds the consensus set exactly with integer
// work only: a vote histogram locates the threshold vote count, and only the
// tie group at the threshold is ranked by the full key (v desc, A desc, i asc).
#include "select_common.cuh"

namespace zoomr {

__global__ void __launch_bounds__(512) select_topc_kernel(
    const int64_t *__restrict__ partial, const int32_t *__restrict__ num_summaries,
    int32_t max_summaries, int32_t c, uint8_t *__restrict__ flags, float *__restrict__ agreeability,
    int32_t *status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SmemCarve sm{smem_raw};
  long long *A = sm.take<long long>(max_summaries);
  int *v = sm.take<int>(max_summaries);
  int *grp = sm.take<int>(max_summaries);
  int *hist = sm.take<int>(kHistBins);
  int *scratch = sm.take<int>(40);
  uint8_t *fl = sm.take<uint8_t>(max_summaries);
  const int b = blockIdx.x;
  int nt = num_summaries[b];
  if (nt > max_summaries || nt < 0) {
    if (threadIdx.x == 0) set_status(status, ZOOMR_ERR_INDEX_RANGE);
    nt = nt < 0 ? 0 : max_summaries;
  }
  const int64_t *pv = partial + (int64_t)b * 2 * max_summaries;
  for (int i = threadIdx.x; i < nt; i += blockDim.x) {
    v[i] = (int)pv[i];
    A[i] = pv[max_summaries + i];
  }
  __syncthreads();
  block_topc(v, A, nt, c, fl, hist, grp, scratch, agreeability ? agreeability + b : nullptr);
  uint8_t *out = flags + (int64_t)b * max_summaries;
  for (int i = threadIdx.x; i < max_summaries; i += blockDim.x) out[i] = i < nt ? fl[i] : 0;
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
  const size_t smem = (size_t)max_summaries * (8 + 4 + 4 + 1) + (kHistBins + 40) * 4 + 6 * 16;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(select_topc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  prefer_max_smem(select_topc_kernel);
  select_topc_kernel<<<batch, 512, smem, (cudaStream_t)stream>>>(partial, num_summaries, max_summaries, c,
                                                                 flags, agreeability, dev_status);
  return launch_status((cudaStream_t)stream);
}
