// a1 -- mean summary keys (Alg.1 @P:408-409).
//
//   kbar_i^{(l,g)} = (1/|S_i|) * sum_{j in S_i} k_j^{(l,g)}
//
// One CTA per (item, layer); one warp per KV head; each lane owns D/32 (or one)
// elements of the head dimension and walks the summary's tokens in ascending
// order, gathering each token row (2*D bytes, coalesced across the warp) from
// its page.  The sum is kept in fp64 and divided once, then rounded to fp32:
// the result is the correctly-rounded fp32 of the exact mean for any |S_i| the
// caches hold, so the stored key carries no accumulation error into a2.
// Bytes per summary: |S_i| * L * H_kv * D * 2 read + L * H_kv * D * 4 written.
#include "common.cuh"

namespace zoomr {

template <int D>
__global__ void __launch_bounds__(256) mean_keys_kernel(
    const __nv_bfloat16 *__restrict__ kpool, int64_t num_pages, const int32_t *__restrict__ page_table,
    int32_t max_pages, const int32_t *__restrict__ bounds, const int32_t *__restrict__ num_summaries,
    const int32_t *__restrict__ seq_len, int32_t max_summaries, const int32_t *__restrict__ items,
    int32_t L, int32_t Hkv, int32_t P, float *__restrict__ mean_keys, int32_t *status) {
  constexpr int EPL = D >= 32 ? D / 32 : 1;       // elements per lane
  constexpr int LANES = D >= 32 ? 32 : D;          // active lanes
  const int item = blockIdx.x, l = blockIdx.y;
  const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (g >= Hkv) return;
  const int b = items[2 * item], i = items[2 * item + 1];
  if (i < 0 || i >= max_summaries || i >= num_summaries[b]) {
    if (threadIdx.x == 0) set_status(status, ZOOMR_ERR_INDEX_RANGE);
    return;
  }
  const int32_t *bd = bounds + ((int64_t)b * max_summaries + i) * 4;
  const int s0 = bd[2], s1 = bd[3], T = seq_len[b];
  if (s1 <= s0) {
    if (threadIdx.x == 0) set_status(status, ZOOMR_ERR_EMPTY_SEGMENT);
    return;
  }
  if (s0 < 0 || s1 > T || (s1 - 1) / P >= max_pages) {
    if (threadIdx.x == 0) set_status(status, ZOOMR_ERR_INDEX_RANGE);
    return;
  }
  if (lane >= LANES) return;
  const int32_t *pt = page_table + (int64_t)b * max_pages;
  double acc[EPL];
#pragma unroll
  for (int e = 0; e < EPL; ++e) acc[e] = 0.0;
  // ascending j, exactly the order of the definition
  for (int j = s0; j < s1; ++j) {
    const int page = pt[j / P];
    if (page < 0 || page >= num_pages) {
      set_status(status, ZOOMR_ERR_INDEX_RANGE);
      return;
    }
    const __nv_bfloat16 *row = kpool + ((((int64_t)l * num_pages + page) * Hkv + g) * P + (j % P)) * D;
    if constexpr (EPL == 4) {
      const uint2 w = *reinterpret_cast<const uint2 *>(row + lane * 4);
      acc[0] += (double)bf16lo_to_float(w.x);
      acc[1] += (double)bf16hi_to_float(w.x);
      acc[2] += (double)bf16lo_to_float(w.y);
      acc[3] += (double)bf16hi_to_float(w.y);
    } else if constexpr (EPL == 2) {
      const uint32_t w = *reinterpret_cast<const uint32_t *>(row + lane * 2);
      acc[0] += (double)bf16lo_to_float(w);
      acc[1] += (double)bf16hi_to_float(w);
    } else {
      acc[0] += (double)__bfloat162float(row[lane]);
    }
  }
  const double n = (double)(s1 - s0);
  float *out = mean_keys + ((((int64_t)b * L + l) * Hkv + g) * max_summaries + i) * D + lane * EPL;
#pragma unroll
  for (int e = 0; e < EPL; ++e) out[e] = (float)(acc[e] / n);
}

}  // namespace zoomr

using namespace zoomr;

extern "C" int zoomr_update_mean_keys(const zoomr_geom *geom, int32_t batch, const zoomr_kv *kv,
                                      const zoomr_segments *seg, const int32_t *items,
                                      int32_t n_items, float *mean_keys, int32_t *dev_status,
                                      void *stream) {
  int rc = check_geom(geom);
  if (rc) return rc;
  if (batch < 1 || n_items < 0 || !kv || !seg || !kv->k || !kv->page_table || !seg->bounds ||
      !seg->num_summaries || !seg->seq_len || !mean_keys || (n_items > 0 && !items) ||
      seg->max_summaries < 1 || kv->num_pages < 1 || kv->max_pages < 1)
    return ZOOMR_ERR_INVALID_ARG;
  if (geom->num_kv_heads > 8) return ZOOMR_ERR_UNSUPPORTED;  // one warp per KV head per CTA
  if (n_items == 0) return ZOOMR_OK;
  dim3 grid(n_items, geom->num_layers), block(32 * geom->num_kv_heads);
  cudaStream_t s = (cudaStream_t)stream;
  auto *k = (const __nv_bfloat16 *)kv->k;
#define ZOOMR_MK(D)                                                                                  \
  mean_keys_kernel<D><<<grid, block, 0, s>>>(k, kv->num_pages, kv->page_table, kv->max_pages,       \
                                             seg->bounds, seg->num_summaries, seg->seq_len,         \
                                             seg->max_summaries, items, geom->num_layers,           \
                                             geom->num_kv_heads, geom->page_size, mean_keys,        \
                                             dev_status)
  switch (geom->head_dim) {
    case 16: ZOOMR_MK(16); break;
    case 32: ZOOMR_MK(32); break;
    case 64: ZOOMR_MK(64); break;
    default: ZOOMR_MK(128); break;
  }
#undef ZOOMR_MK
  return launch_status();
}
