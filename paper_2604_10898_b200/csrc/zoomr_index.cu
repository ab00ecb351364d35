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
#include "common.cuh"

namespace zoomr {

__global__ void __launch_bounds__(1024) build_index_kernel(
    const int32_t *__restrict__ bounds, const int32_t *__restrict__ num_summaries,
    const int32_t *__restrict__ seq_len, int32_t max_summaries, const uint8_t *__restrict__ flags,
    int32_t sink, int32_t window, int32_t *__restrict__ index, int32_t cap,
    int32_t *__restrict__ index_count, int32_t *status) {
  extern __shared__ int32_t off[];  // [max_summaries + 1] exclusive offsets of clipped pieces
  __shared__ int32_t warp_tot[32];
  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int T = seq_len[b];
  int nt = num_summaries[b];
  if (nt > max_summaries || nt < 0) {
    if (tid == 0) set_status(status, ZOOMR_ERR_INDEX_RANGE);
    nt = nt < 0 ? 0 : max_summaries;
  }
  if (T < 1) {
    if (tid == 0) {
      set_status(status, ZOOMR_ERR_INVALID_ARG);
      index_count[b] = 0;
    }
    return;
  }
  const int sp = sink < T ? sink : T;                 // s'
  const int w0 = (T - window > sp) ? T - window : sp;  // start of the window piece
  const int32_t *bd = bounds + (int64_t)b * max_summaries * 4;
  const uint8_t *fl = flags ? flags + (int64_t)b * max_summaries : nullptr;

  // each thread owns a contiguous run of pieces [i0, i1)
  const int per = (nt + (int)blockDim.x - 1) / (int)blockDim.x;
  const int i0 = tid * per, i1 = min(nt, i0 + per);
  int local = 0;
  for (int i = i0; i < i1; ++i) {
    const int r0 = bd[4 * i], r1 = bd[4 * i + 1], s0 = bd[4 * i + 2], s1 = bd[4 * i + 3];
    if (s1 <= s0) set_status(status, ZOOMR_ERR_EMPTY_SEGMENT);
    else if (r0 < 0 || r1 < r0 || s0 < r1 || (i + 1 < nt && bd[4 * (i + 1)] < s1))
      set_status(status, ZOOMR_ERR_SEGMENT_ORDER);
    else if (s1 > T) set_status(status, ZOOMR_ERR_INDEX_RANGE);
    const int f = fl ? fl[i] : 0;
    int a = 0, e = 0;
    if (f == 2) { a = r0; e = r1; }        // zoom: R_i
    else if (f == 1) { a = s0; e = s1; }   // keep: S_i
    a = max(a, sp);
    e = min(e, w0);
    local += max(0, e - a);
  }
  // block exclusive scan of the per-thread totals
  int incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int wt = lane < nwarps ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, wt, o);
      if (lane >= o) wt += y;
    }
    if (lane < nwarps) warp_tot[lane] = wt;  // inclusive warp prefix
  }
  __syncthreads();
  int run = (warp ? warp_tot[warp - 1] : 0) + incl - local;  // exclusive offset of piece i0
  for (int i = i0; i < i1; ++i) {
    off[i] = run;
    const int f = fl ? fl[i] : 0;
    int a = 0, e = 0;
    if (f == 2) { a = bd[4 * i]; e = bd[4 * i + 1]; }
    else if (f == 1) { a = bd[4 * i + 2]; e = bd[4 * i + 3]; }
    run += max(0, min(e, w0) - max(a, sp));
  }
  const int total = warp_tot[nwarps - 1];
  __syncthreads();
  const int count = sp + total + (T - w0);
  int32_t *out = index + (int64_t)b * cap;
  if (tid == 0) {
    if (count > cap) set_status(status, ZOOMR_ERR_CAPACITY);
    index_count[b] = count < cap ? count : cap;
  }
  // sink [0, s') and window [w0, T)
  for (int j = tid; j < sp && j < cap; j += blockDim.x) out[j] = j;
  const int wbase = sp + total;
  for (int j = tid; j < T - w0; j += blockDim.x)
    if (wbase + j < cap) out[wbase + j] = w0 + j;
  // one warp per selected piece
  for (int i = warp; i < nt; i += nwarps) {
    const int f = fl ? fl[i] : 0;
    if (f != 1 && f != 2) continue;
    int a = f == 2 ? bd[4 * i] : bd[4 * i + 2];
    int e = f == 2 ? bd[4 * i + 1] : bd[4 * i + 3];
    a = max(a, sp);
    e = min(e, w0);
    const int base = sp + off[i];
    for (int j = lane; j < e - a; j += 32)
      if (base + j < cap) out[base + j] = a + j;
  }
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
  const size_t smem = (size_t)(seg->max_summaries + 1) * sizeof(int32_t);
  build_index_kernel<<<batch, 1024, smem, (cudaStream_t)stream>>>(
      seg->bounds, seg->num_summaries, seg->seq_len, seg->max_summaries, flags, sink, window,
      index, index_capacity, index_count, dev_status);
  return launch_status();
}
