// Algorithm 1's per-token bookkeeping around the hot path,
// on device so that a whole decode step -- append, segment tracking, selection
// update at semantic boundaries, attention -- is one CUDA-graph replay:
//
//  * zoomr_append_kv     a0: "Append k_t and v_t to KV cache" (Alg.1 @P:407);
//  * zoomr_track_segments: the summary delimiters (<|begin_of_summary|>,
//    <|end_of_summary|>, SPEC ingest_token S:36-45) maintain the
//    segment table, a closed summary is reported for a1 ("if a new summary S_Nt
//    is complete", Alg.1 @P:408), and a semantic-boundary token (the preset
//    punctuation list, P:109 / Appendix) requests the selection update
//    ("if at a semantic boundary", Alg.1 @P:417).
#include "common.cuh"

namespace zoomr {

// one CTA per (b, layer); threads over (KV head, d/8 chunks): 16-byte copies
__global__ void append_kv_kernel(const uint4 *__restrict__ k_new, const uint4 *__restrict__ v_new,
                                 __nv_bfloat16 *kpool, __nv_bfloat16 *vpool, int64_t num_pages,
                                 const int32_t *__restrict__ page_table, int32_t max_pages, int32_t L, int32_t Hkv,
                                 int32_t P, int32_t d, const int32_t *__restrict__ seq_len_in, int32_t back,
                                 int32_t *status) {
  const int b = blockIdx.y, l = blockIdx.x;
  const int T = seq_len_in[b] - back;  // back = 1: the newest token, already counted in seq_len
  const int lp = T / P;
  int page = (T >= 0 && lp < max_pages) ? page_table[(int64_t)b * max_pages + lp] : -1;
  if (back && page == -1 && T >= 0 && lp < max_pages) return;  // newest row, page not resident: nothing to update
  if (page < 0 || page >= num_pages) {
    if (threadIdx.x == 0) set_status(status, ZOOMR_ERR_INDEX_RANGE);
    return;
  }
  const int cpr = d / 8;  // 16-byte chunks per row
  for (int x = threadIdx.x; x < Hkv * cpr; x += blockDim.x) {
    const int g = x / cpr, c = x - g * cpr;
    const int64_t src = (((int64_t)b * L + l) * Hkv + g) * cpr + c;
    const int64_t dst = (((((int64_t)l * num_pages + page) * Hkv + g) * P + (T - lp * P)) * d) / 8 + c;
    reinterpret_cast<uint4 *>(kpool)[dst] = k_new[src];
    reinterpret_cast<uint4 *>(vpool)[dst] = v_new[src];
  }
}

__global__ void advance_kernel(int32_t *seq_len, int32_t batch) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < batch) seq_len[b] += 1;
}

// segment tracking of sequence b for the token at position pos (one thread)
__device__ void track_one(int b, int tok, int pos, int32_t begin_id, int32_t end_id,
                          const int32_t *__restrict__ boundary_ids, int32_t n_boundary, int32_t *bounds,
                          int32_t *num_summaries, int32_t max_summaries, int4 *state, int32_t *close_items,
                          uint8_t *update, int32_t *status) {
  int4 st = state[b];              // (open summary start or -1, open-tail start, pending R start, pending R end)
  int closed = -1;
  if (tok == begin_id) {
    if (st.x >= 0) set_status(status, ZOOMR_ERR_SEGMENT_ORDER);  // begin inside an open summary
    else {
      st.z = st.y;  // the open tail before the delimiter becomes the pending R
      st.w = pos;
      st.x = pos;
    }
  } else if (tok == end_id) {
    if (st.x < 0) set_status(status, ZOOMR_ERR_SEGMENT_ORDER);  // end without an open summary
    else {
      const int i = num_summaries[b];
      if (i >= max_summaries) set_status(status, ZOOMR_ERR_CAPACITY);
      else {
        int32_t *bd = bounds + ((int64_t)b * max_summaries + i) * 4;
        bd[0] = st.z;
        bd[1] = st.w;
        bd[2] = st.x;
        bd[3] = pos + 1;  // delimiters included
        num_summaries[b] = i + 1;
        closed = i;
      }
      st.x = -1;
      st.y = pos + 1;
    }
  }
  state[b] = st;
  close_items[2 * b] = b;
  close_items[2 * b + 1] = closed;
  bool bnd = false;
  for (int j = 0; j < n_boundary; ++j) bnd |= tok == boundary_ids[j];
  update[b] = bnd ? 1 : 0;
}

// one thread per sequence
__global__ void track_kernel(int32_t batch, const int32_t *__restrict__ token_ids, int32_t begin_id, int32_t end_id,
                             const int32_t *__restrict__ boundary_ids, int32_t n_boundary,
                             const int32_t *__restrict__ seq_len, int32_t *bounds, int32_t *num_summaries,
                             int32_t max_summaries, int4 *state, int32_t *close_items, uint8_t *update,
                             int32_t *status) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  track_one(b, token_ids[b], seq_len[b] - 1 /* the token just appended */, begin_id, end_id, boundary_ids,
            n_boundary, bounds, num_summaries, max_summaries, state, close_items, update, status);
}

// a0 + segment tracking as two launches that chain without a host round trip:
//  * append_rows_kernel, one CTA per (layer, b) as append_kv: the token's rows at
//    position T = seq_len[b]; each CTA triggers its dependents once it has used T;
//  * track_advance_kernel (PDL behind it), one thread per sequence: the tracking of
//    position T, then seq_len[b] = T + 1 -- launched only when every row CTA has
//    read T, so no CTA can see the advanced T.
// Right behind a chained a5 the row copy is launched with PDL and runs while that
// a5 finishes (a5 read seq_len in its prologue, before its trigger, and reads no
// row at position T).  Both kernels end with griddepcontrol.wait, so each
// completes only after its predecessor: the next launch on the stream (the
// selection, which rewrites I_f) is ordered after the a5 as well.
// a pool the row copy writes to: (K, V, pages, page table) with its own page size
struct RowDst {
  __nv_bfloat16 *k, *v;
  int64_t num_pages;
  const int32_t *page_table;
  int32_t max_pages, P;
};

__global__ void append_rows_kernel(const uint4 *__restrict__ k_new, const uint4 *__restrict__ v_new, RowDst dst0,
                                   RowDst mirror, int32_t L, int32_t Hkv, int32_t d,
                                   const int32_t *__restrict__ seq_len, int32_t *status) {
  const int b = blockIdx.y, l = blockIdx.x;
  const int T = seq_len[b];
  // row of (l, g = 0, position T) in a pool, or -1; `optional`: a page that is
  // not resident (-1) is skipped instead of being an error (the host tier's HBM
  // hot pool: zoomr_write_newest_kv's rule)
  auto row_of = [&](const RowDst &q, bool optional, bool &err) -> int64_t {
    const int lp = T / q.P;
    const int page = (T >= 0 && lp < q.max_pages) ? q.page_table[(int64_t)b * q.max_pages + lp] : -2;
    if (optional && page == -1) return -1;
    if (page < 0 || page >= q.num_pages) {
      err = true;
      return -1;
    }
    return ((int64_t)l * q.num_pages + page) * Hkv * q.P + (T - lp * q.P);
  };
  bool err = false;
  const int64_t row0 = row_of(dst0, false, err);
  const int64_t row1 = mirror.k ? row_of(mirror, true, err) : -1;
  __syncthreads();            // every thread of the CTA has used T
  allow_dependents();         // (the tracking may now advance seq_len)
  if (err && threadIdx.x == 0) set_status(status, ZOOMR_ERR_INDEX_RANGE);
  const int cpr = d / 8;  // 16-byte chunks per row
  for (int x = threadIdx.x; x < Hkv * cpr; x += blockDim.x) {
    const int g = x / cpr, c = x - g * cpr;
    const int64_t src = (((int64_t)b * L + l) * Hkv + g) * cpr + c;
    const uint4 kx = k_new[src], vx = v_new[src];
    if (row0 >= 0) {
      const int64_t o = ((row0 + (int64_t)g * dst0.P) * d) / 8 + c;
      reinterpret_cast<uint4 *>(dst0.k)[o] = kx;
      reinterpret_cast<uint4 *>(dst0.v)[o] = vx;
    }
    if (row1 >= 0) {
      const int64_t o = ((row1 + (int64_t)g * mirror.P) * d) / 8 + c;
      reinterpret_cast<uint4 *>(mirror.k)[o] = kx;
      reinterpret_cast<uint4 *>(mirror.v)[o] = vx;
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");  // complete only after the preceding kernel
}

__global__ void track_advance_kernel(int32_t batch, const int32_t *__restrict__ token_ids, int32_t begin_id,
                                     int32_t end_id, const int32_t *__restrict__ boundary_ids, int32_t n_boundary,
                                     int32_t *seq_len, int32_t *bounds, int32_t *num_summaries,
                                     int32_t max_summaries, int4 *state, int32_t *close_items, uint8_t *update,
                                     int32_t *status) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < batch) {
    const int T = seq_len[b];
    seq_len[b] = T + 1;
    track_one(b, token_ids[b], T, begin_id, end_id, boundary_ids, n_boundary, bounds, num_summaries, max_summaries,
              state, close_items, update, status);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");  // complete only after the row copy
}

}  // namespace zoomr

using namespace zoomr;

extern "C" int zoomr_append_kv(const zoomr_geom *geom, int32_t batch, const zoomr_kv *kv, const void *k_new,
                               const void *v_new, int32_t *seq_len, int32_t *dev_status, void *stream) {
  int rc = check_geom(geom);
  if (rc) return rc;
  if (batch < 1 || !kv || !kv->k || !kv->v || !kv->page_table || !k_new || !v_new || !seq_len ||
      kv->num_pages < 1 || kv->max_pages < 1)
    return ZOOMR_ERR_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  append_kv_kernel<<<dim3(geom->num_layers, batch), 128, 0, s>>>(
      (const uint4 *)k_new, (const uint4 *)v_new, (__nv_bfloat16 *)kv->k, (__nv_bfloat16 *)kv->v, kv->num_pages,
      kv->page_table, kv->max_pages, geom->num_layers, geom->num_kv_heads, geom->page_size, geom->head_dim, seq_len,
      0, dev_status);
  advance_kernel<<<(batch + 127) / 128, 128, 0, s>>>(seq_len, batch);
  return launch_status((cudaStream_t)stream);
}

extern "C" int zoomr_write_newest_kv(const zoomr_geom *geom, int32_t batch, const zoomr_kv *kv, const void *k_new,
                                     const void *v_new, const int32_t *seq_len, int32_t *dev_status, void *stream) {
  int rc = check_geom(geom);
  if (rc) return rc;
  if (batch < 1 || !kv || !kv->k || !kv->v || !kv->page_table || !k_new || !v_new || !seq_len ||
      kv->num_pages < 1 || kv->max_pages < 1)
    return ZOOMR_ERR_INVALID_ARG;
  append_kv_kernel<<<dim3(geom->num_layers, batch), 128, 0, (cudaStream_t)stream>>>(
      (const uint4 *)k_new, (const uint4 *)v_new, (__nv_bfloat16 *)kv->k, (__nv_bfloat16 *)kv->v, kv->num_pages,
      kv->page_table, kv->max_pages, geom->num_layers, geom->num_kv_heads, geom->page_size, geom->head_dim, seq_len,
      1, dev_status);
  return launch_status((cudaStream_t)stream);
}

extern "C" int zoomr_track_segments(int32_t batch, const int32_t *token_ids, int32_t begin_id, int32_t end_id,
                                    const int32_t *boundary_ids, int32_t n_boundary, const int32_t *seq_len,
                                    int32_t *bounds, int32_t *num_summaries, int32_t max_summaries, int32_t *state,
                                    int32_t *close_items, uint8_t *update, int32_t *dev_status, void *stream) {
  if (batch < 1 || !token_ids || (n_boundary > 0 && !boundary_ids) || n_boundary < 0 || !seq_len || !bounds ||
      !num_summaries || max_summaries < 1 || !state || !close_items || !update)
    return ZOOMR_ERR_INVALID_ARG;
  track_kernel<<<(batch + 127) / 128, 128, 0, (cudaStream_t)stream>>>(
      batch, token_ids, begin_id, end_id, boundary_ids, n_boundary, seq_len, bounds, num_summaries, max_summaries,
      reinterpret_cast<int4 *>(state), close_items, update, dev_status);
  return launch_status((cudaStream_t)stream);
}

extern "C" int zoomr_append_track(const zoomr_geom *geom, int32_t batch, const zoomr_kv *kv, const zoomr_kv *mirror,
                                  int32_t mirror_page_size, const void *k_new, const void *v_new,
                                  const int32_t *token_ids, int32_t begin_id, int32_t end_id,
                                  const int32_t *boundary_ids, int32_t n_boundary, int32_t *seq_len, int32_t *bounds,
                                  int32_t *num_summaries, int32_t max_summaries, int32_t *state, int32_t *close_items,
                                  uint8_t *update, int32_t *dev_status, void *stream) {
  int rc = check_geom(geom);
  if (rc) return rc;
  if (batch < 1 || !kv || !kv->k || !kv->v || !kv->page_table || !k_new || !v_new || !seq_len ||
      kv->num_pages < 1 || kv->max_pages < 1 || !token_ids || (n_boundary > 0 && !boundary_ids) || n_boundary < 0 ||
      !bounds || !num_summaries || max_summaries < 1 || !state || !close_items || !update)
    return ZOOMR_ERR_INVALID_ARG;
  if (mirror && (!mirror->k || !mirror->v || !mirror->page_table || mirror->num_pages < 1 || mirror->max_pages < 1 ||
                 mirror_page_size < 1))
    return ZOOMR_ERR_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const dim3 grid(geom->num_layers, batch);
  const RowDst d0{(__nv_bfloat16 *)kv->k, (__nv_bfloat16 *)kv->v, kv->num_pages, kv->page_table, kv->max_pages,
                  geom->page_size};
  const RowDst d1 = mirror ? RowDst{(__nv_bfloat16 *)mirror->k, (__nv_bfloat16 *)mirror->v, mirror->num_pages,
                                    mirror->page_table, mirror->max_pages, mirror_page_size}
                           : RowDst{nullptr, nullptr, 0, nullptr, 0, 1};
  // the row copy with PDL only right behind the library's chained a5 (see the kernels' comment)
  if (prev_launch_is(s, kLaunchA5Chained, nullptr))
    launch_pdl(append_rows_kernel, grid, 128, 0, s, (const uint4 *)k_new, (const uint4 *)v_new, d0, d1,
               geom->num_layers, geom->num_kv_heads, geom->head_dim, (const int32_t *)seq_len, dev_status);
  else
    append_rows_kernel<<<grid, 128, 0, s>>>((const uint4 *)k_new, (const uint4 *)v_new, d0, d1, geom->num_layers,
                                            geom->num_kv_heads, geom->head_dim, (const int32_t *)seq_len,
                                            dev_status);
  launch_pdl(track_advance_kernel, dim3((batch + 127) / 128), 128, 0, s, batch, token_ids, begin_id, end_id,
             boundary_ids, n_boundary, seq_len, bounds, num_summaries, max_summaries, reinterpret_cast<int4 *>(state),
             close_items, update, dev_status);
  return launch_status(s);
}
