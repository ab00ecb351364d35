// a4 -- the multi-granularity index set (Alg.1 @P:421-422):
//
//   I_f = I_p  u  I_w  u  (u_{i in I_c} R_i)  u  (u_{i in I_s} S_i)
//
// with I_p = [0, s') (s' = min(sink, T), reading Q12) and
// I_w = [max(0, T - w), T) (reading Q13).  Because the segment table is ordered
// and disjoint (r0 <= r1 <= s0 < s1 <= next r0), clipping every selected R_i /
// S_i to the middle zone [s', w0), w0 = max(T - w, s'), makes all pieces
// disjoint and already sorted: the union is the concatenation
//   [0, s') ++ clipped pieces in i order ++ [w0, T)
// and each piece's write offset is an exclusive prefix sum of the clipped
// lengths.  One CTA per sequence: a block scan over <= 4096 pieces, then one
// warp per piece writes its positions with coalesced stores.  Integer work,
// bit-exact by construction; the segment-table invariants are checked here.
#include "select_common.cuh"

namespace zoomr {

__global__ void __launch_bounds__(512) build_index_kernel(
    const int32_t *__restrict__ bounds, const int32_t *__restrict__ num_summaries,
    const int32_t *__restrict__ seq_len, int32_t max_summaries, const uint8_t *__restrict__ flags,
    int32_t sink, int32_t window, int32_t *__restrict__ index, int32_t cap,
    int32_t *__restrict__ index_count, int32_t *status) {
  extern __shared__ int32_t off[];  // [2*max_summaries] clipped pieces: start, offset
  __shared__ int32_t scratch[40];
  allow_dependents();
  const int b = blockIdx.x;
  const int T = seq_len[b];
  int nt = num_summaries[b];
  if (nt > max_summaries || nt < 0) {
    if (threadIdx.x == 0) set_status(status, ZOOMR_ERR_INDEX_RANGE);
    nt = nt < 0 ? 0 : max_summaries;
  }
  if (T < 1) {
    if (threadIdx.x == 0) {
      set_status(status, ZOOMR_ERR_INVALID_ARG);
      index_count[b] = 0;
    }
    return;
  }
  block_build_index(bounds + (int64_t)b * max_summaries * 4, nt, T,
                    flags ? flags + (int64_t)b * max_summaries : nullptr, sink, window,
                    index + (int64_t)b * cap, cap, index_count + b, off, scratch, status);
}

}  // namespace zoomr

using namespace zoomr;

extern "C" int zoomr_build_index(int32_t batch, const zoomr_segments *seg, const uint8_t *flags,
                                 int32_t sink, int32_t window, int32_t *index,
                                 int32_t index_capacity, int32_t *index_count, int32_t *dev_status,
                                 void *stream) {
  if (batch < 1 || !seg || !seg->bounds || !seg->num_summaries || !seg->seq_len || !index ||
      !index_count || index_capacity < 1 || sink < 0 || window < 1 || seg->max_summaries < 1)
    return ZOOMR_ERR_INVALID_ARG;
  if (seg->max_summaries > kMaxSummaries) return ZOOMR_ERR_UNSUPPORTED;
  const size_t smem = (size_t)(2 * seg->max_summaries + 1) * sizeof(int32_t);
  prefer_max_smem(build_index_kernel);
  build_index_kernel<<<batch, 512, smem, (cudaStream_t)stream>>>(
      seg->bounds, seg->num_summaries, seg->seq_len, seg->max_summaries, flags, sink, window,
      index, index_capacity, index_count, dev_status);
  return launch_status((cudaStream_t)stream);
}
