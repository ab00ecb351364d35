// a1 -- mean summary keys (Alg.1 @P:408-409).
//
//   kbar_i^{(l,g)} = (1/|S_i|) * sum_{j in S_i} k_j^{(l,g)}
//
// One CTA per (item, layer, KV head): block_mean_key (select_common.cuh) lets
// the warps take the summary's tokens round-robin (independent loads in flight)
// and the lanes the head dimension (coalesced 2*D-byte rows from the pages);
// fp64 partial sums meet in shared memory and are divided once, then rounded to
// fp32.  The fp64 sum of bf16 values is exact, so the stored key is the
// correctly-rounded fp32 of the exact mean (bit-identical to the oracle's).
// Bytes per summary: |S_i| * L * H_kv * D * 2 read + L * H_kv * D * 4 written.
#include "select_common.cuh"

namespace zoomr {

template <int D>
__global__ void __launch_bounds__(128) mean_keys_kernel(
    const __nv_bfloat16 *__restrict__ kpool, int64_t num_pages, const int32_t *__restrict__ page_table,
    int32_t max_pages, const int32_t *__restrict__ bounds, const int32_t *__restrict__ num_summaries,
    const int32_t *__restrict__ seq_len, int32_t max_summaries, const int32_t *__restrict__ items,
    int32_t L, int32_t Hkv, int32_t P, float *__restrict__ mean_keys, int32_t *status) {
  __shared__ double red[4 * D];
  const int item = blockIdx.x, lg = blockIdx.y;
  const int l = lg / Hkv, g = lg - l * Hkv;
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
  if (s0 < 0 || s1 > T) {
    if (threadIdx.x == 0) set_status(status, ZOOMR_ERR_INDEX_RANGE);
    return;
  }
  block_mean_key<D>(kpool, num_pages, page_table + (int64_t)b * max_pages, max_pages, P, Hkv, l, g, s0, s1,
                    red, mean_keys + ((((int64_t)b * L + l) * Hkv + g) * max_summaries + i) * D, status);
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
  if (n_items == 0) return ZOOMR_OK;
  dim3 grid(n_items, geom->num_layers * geom->num_kv_heads), block(128);
  cudaStream_t s = (cudaStream_t)stream;
  auto *k = (const __nv_bfloat16 *)kv->k;
#define ZOOMR_MK(D)                                                                                  \
  prefer_max_smem(mean_keys_kernel<D>);                                                            \
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
  return launch_status((cudaStream_t)stream);
}
