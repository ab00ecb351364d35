/*
 * zoomr.h -- C-ABI of the B200-native ZoomR select + sparse-decode hot path
 * (arXiv 2604.10898, "ZoomR").  Implemented by libzoomr.so (hand-written
 * sm_100a CUDA kernels in paper_2604_10898_b200/csrc/).
 *
 * Citations: "P:n" = PAPER.md line n (section / equation / Algorithm 1 line),
 * "S:n" = SPEC.md line n.  The readings of the paper that the kernels follow
 * are listed in DESIGN.md section 3 (Q1..Q25).
 *
 * The five entry points are the five steps of the path, in order:
 *   zoomr_update_mean_keys    a1  mean summary keys             P:36-41, Alg.1 @P:408-409
 *   zoomr_score               a2  alpha = q.kbar, per-head top-k,
 *                                 votes + sum-alpha aggregation  P:43-63, Alg.1 @P:411-417
 *   zoomr_select_topc         a3  global top-c consensus         P:64-67, Alg.1 @P:418-419
 *   zoomr_build_index         a4  multi-granularity index I_f    P:69-72, Alg.1 @P:421-422
 *   zoomr_sparse_decode_attn  a5  paged gather + GQA decode
 *                                 attention over I_f
 * plus the fused select (a1..a4 in one launch), Algorithm 1's per-token
 * bookkeeping (KV append, segment tracking), the token-sharded split-K
 * pieces (index restriction, a5 with log-sum-exp, the merge) and the H2O
 * comparison policy (a5 with logits, score accumulation, eviction) and the
 * host-memory tier (HBM hot pool caching a pinned host cache).
 *
 * Conventions shared by every call
 *  - Ownership: every array argument is DEVICE memory allocated and owned by
 *    the caller.  The library never allocates device memory and never frees or
 *    retains a pointer past the call.  Its only host state is, per stream, the
 *    kind of its own most recent launch (a small mutex-protected table): it is
 *    what lets a chained call detect an unsafe predecessor and fall back to
 *    the serialised launch (see "Chained launches").  Host structs
 *    (zoomr_geom, zoomr_kv, zoomr_segments) are read during the call only.
 *  - Streams: `stream` is a cudaStream_t (passed as void*); all work is
 *    enqueued on it asynchronously; no call synchronizes the host.  Every call
 *    is CUDA-graph capturable.  Concurrent calls on different streams are safe
 *    when their output and workspace buffers are distinct.
 *  - Tokens: 0-based absolute positions.  Summary index i: 0-based; a smaller
 *    index is an older summary (the tie-break, readings Q3/Q20).
 *  - GQA: query head h reads KV head h / (H_q / H_kv) (reading Q6).  In the
 *    KV-head-sharded mode the geometry holds the rank's LOCAL heads.
 *  - Errors: the int return value is ZOOMR_OK or a host-detectable error
 *    (NULL pointer, bad size, unsupported head_dim, launch failure); nothing is
 *    enqueued when it is not ZOOMR_OK.  Data-dependent errors are detected on
 *    the device and recorded, first one wins (atomicCAS from 0), into the
 *    optional `dev_status` int32 (device memory, caller zeroes it); after a
 *    device-detected error that sequence's outputs are defined but unspecified.
 */
#ifndef ZOOMR_H
#define ZOOMR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ZOOMR_ABI_VERSION 9

typedef enum {
  ZOOMR_OK = 0,
  ZOOMR_ERR_INVALID_ARG = 1,   /* NULL pointer, negative size, top_k < 1, c < 0, ...     */
  ZOOMR_ERR_DIM_MISMATCH = 2,  /* H_q % H_kv != 0, G = H_q/H_kv not in {1, 2, 4, 7, 8}    */
  ZOOMR_ERR_EMPTY_SEGMENT = 3, /* device: s1 <= s0 (SPEC EmptySegment)             */
  ZOOMR_ERR_SEGMENT_ORDER = 4, /* device: r0<=r1<=s0<s1<=next r0 violated        */
  ZOOMR_ERR_INDEX_RANGE = 5,   /* device: s1 > T, N_t > max_summaries, page beyond table  */
  ZOOMR_ERR_CAPACITY = 6,      /* device: |I_f| > index_capacity (count is clamped)        */
  ZOOMR_ERR_UNSUPPORTED = 7,   /* head_dim not in {16, 32, 64, 128}, N_t > 4096, k > 32   */
  ZOOMR_ERR_CUDA = 8,          /* a CUDA launch failed                                     */
  ZOOMR_ERR_WORKSPACE = 9      /* workspace smaller than zoomr_attn_workspace_bytes()      */
} zoomr_status;

/* Fixed-point scale of the aggregated score A_i in `partial` (reading Q2 +
 * DESIGN.md "deterministic aggregation"): A_i is stored as the int64
 * sum over voters of round(alpha * 2^32).  Integer addition is associative, so
 * the value does not depend on accumulation order, on the number of ranks in
 * the head-sharded all-reduce, or on the run. */
#define ZOOMR_A_FRAC_BITS 32

/* Model geometry.  heads are rank-local in the KV-head-sharded mode. */
typedef struct {
  int32_t num_layers;   /* N_L                                    */
  int32_t num_q_heads;  /* H_q                                            */
  int32_t num_kv_heads; /* H_kv; G = H_q / H_kv in {1, 2, 4, 7, 8}         */
  int32_t head_dim;     /* d in {16, 32, 64, 128}                         */
  int32_t page_size;    /* P >= 1 tokens per KV page                      */
} zoomr_geom;

/* Paged KV cache (the paper's full cache K_t, V_t, held in HBM).
 * k, v: bf16 [L][num_pages][H_kv][P][d] (element (l, p, g, j, e) at
 *       (((l*num_pages + p)*H_kv + g)*P + j)*d + e).  16-byte aligned.
 * page_table: int32 [B][max_pages]; token t of sequence b lives at physical
 *       page page_table[b*max_pages + t/P], slot t%P.  Pages may alias across
 *       sequences (read-only). */
typedef struct {
  const void *k;
  const void *v;
  int64_t num_pages;
  const int32_t *page_table;
  int32_t max_pages;
} zoomr_kv;

/* Segment table (the paper's R_i / S_i; SPEC SegmentMap S:22-28).
 * bounds: int32 [B][max_summaries][4] = (r0, r1, s0, s1), half-open absolute
 *         token ranges of R_i and S_i; only the first num_summaries[b] rows
 *         (the CLOSED summaries, N_t) are read.  Must satisfy
 *         r0 <= r1 <= s0 < s1 <= r0_{i+1} and s1 <= T (checked on device).
 * num_summaries: int32 [B] = N_t.   seq_len: int32 [B] = T, tokens in the
 *         cache counting the current one (T >= 1). */
typedef struct {
  const int32_t *bounds;
  const int32_t *num_summaries;
  const int32_t *seq_len;
  int32_t max_summaries;
} zoomr_segments;

/* a1 -- mean summary keys, P:36-41 (eq. kbar_i = (1/|S_i|) sum_{j in S_i} k_j),
 * Alg.1 @P:408-409.  For each item (b, i) in `items` (device int32 [n_items][2]),
 * for every layer and KV head, writes
 *   mean_keys[((b*L + l)*H_kv + g)*max_summaries + i][0..d)   (fp32)
 * accumulated in fp64 from the bf16 keys of S_i = [s0_i, s1_i).  Entries not
 * listed are untouched (the cache is written once per closed summary).
 * Device errors: EMPTY_SEGMENT, INDEX_RANGE (i >= max_summaries or s1 > T or a
 * page index beyond the page table). */
int zoomr_update_mean_keys(const zoomr_geom *geom, int32_t batch, const zoomr_kv *kv,
                           const zoomr_segments *seg, const int32_t *items, int32_t n_items,
                           float *mean_keys, int32_t *dev_status, void *stream);

/* a2 -- scoring, per-head voting and aggregation, Alg.1 @P:411-417.
 *   alpha[b,l,h,i] = q[b,l,h] . kbar[b,l,h/G,i]         (fp32, no 1/sqrt(d): P:45, reading Q7)
 *   per voter (l,h): top-min(k, N_t) summaries by (alpha desc, i asc)  (reading Q3/Q5)
 *   partial[b][0][i] = v_i = number of voters that chose i
 *   partial[b][1][i] = A_i = sum over those voters of round(alpha*2^32) (reading Q2)
 * q: bf16 [B][L][H_q][d].  mean_keys: fp32 as written by a1.  partial: int64
 * [B][2][max_summaries], fully overwritten (entries i >= N_t are 0).  In the
 * KV-head-sharded mode each rank passes its local heads and the caller sums
 * `partial` across ranks (one all-reduce) before a3.
 * alpha_out (nullable): fp32 [B][L][H_q][max_summaries].  topk_out (nullable):
 * int32 [B][L*H_q][top_k], -1 past min(k, N_t).  1 <= top_k <= 32.
 * Device errors: INDEX_RANGE (N_t > max_summaries), UNSUPPORTED (N_t > 4096). */
int zoomr_score(const zoomr_geom *geom, int32_t batch, const void *q, const float *mean_keys,
                const int32_t *num_summaries, int32_t max_summaries, int32_t top_k,
                int64_t *partial, float *alpha_out, int32_t *topk_out, int32_t *dev_status,
                void *stream);

/* a3 -- global consensus top-c, Alg.1 @P:418-419.
 * I_all = {i < N_t : v_i > 0}; I_c = the first min(c, |I_all|) of I_all in the
 * order (v desc, A desc, i asc) (readings Q2/Q5); I_s = I_all \ I_c.
 * flags: uint8 [B][max_summaries], 2 for I_c (zoom into R_i), 1 for I_s (keep
 * S_i), 0 otherwise (entries i >= N_t are 0).  agreeability (nullable): fp32
 * [B], AG = sum_{I_c} v / sum_{I_all} v (0 when I_all is empty). */
int zoomr_select_topc(int32_t batch, const int64_t *partial, const int32_t *num_summaries,
                      int32_t max_summaries, int32_t c, uint8_t *flags, float *agreeability,
                      int32_t *dev_status, void *stream);

/* a4 -- the multi-granularity index set, P:69-72 (eq. I_f = I_p u I_w u R(I_c) u S(I_s)),
 * Alg.1 @P:421-422.  I_p = [0, min(sink, T)) (reading Q12), I_w = [max(0, T-window), T)
 * (reading Q13: the window holds the current token), R_i for flag 2, S_i for flag 1.
 * Writes the sorted set union to index[b*index_capacity + 0 .. count) and
 * index_count[b] = |I_f|.  If |I_f| > index_capacity the list is truncated to
 * the capacity and CAPACITY is recorded.  window >= 1, sink >= 0.  flags may be
 * NULL when every N_t is 0. */
int zoomr_build_index(int32_t batch, const zoomr_segments *seg, const uint8_t *flags,
                      int32_t sink, int32_t window, int32_t *index, int32_t index_capacity,
                      int32_t *index_count, int32_t *dev_status, void *stream);

/* Workspace for a5: split-K partial results and per-(b,l,g) arrival counters.
 * Must be zero-filled once before the first call; every call leaves it zeroed.
 * Independent of layer_begin / layer_count: one workspace serves every layer range. */
size_t zoomr_attn_workspace_bytes(const zoomr_geom *geom, int32_t batch);

/* a5 -- sparse GQA decode attention over I_f, P:74 and P:145-149:
 *   out[b,l,h] = sum_{j in I_f,b} softmax_j(q[b,l,h] . k_j * softmax_scale) v_j
 * with k_j, v_j of KV head h/G gathered from the paged pool.  fp32 logits,
 * online softmax and accumulation; out fp32 [B][L][H_q][d].  index / index_count
 * as written by a4 (count >= 1).  index_phys (nullable, [B][index_capacity]):
 * the page-resolved rows zoomr_select_fused can write alongside I_f
 * (page_table[t/P]*H_kv*P + t%P); when given, the page table is not read.
 * softmax_scale is normally 1/sqrt(d).
 *
 * layer_begin, layer_count: attend layers [layer_begin,
 * layer_begin + layer_count) only -- a model calls a5 once per layer, and the
 * host-memory tier pipelines the per-layer fetch against it.  q, out
 * and the pools keep their full [.][L][..] layout; out rows of other layers
 * are not written.  layer_count = 0 means "through the last layer"; a range
 * outside [0, L) is INVALID_ARG.
 *
 * seq_len (nullable, int32 [B], device) + sink + window: when given, I_f MUST
 * be a4's output for the same T = seq_len[b], sink and window, i.e. start with
 * I_p = [0, min(sink, T)) and end with I_w = [max(min(sink, T), T - window), T)
 * (readings Q12, Q13, Q17).  The kernel then attends over those rows -- known
 * from T alone -- before it waits for the producer of I_f (it is launched with
 * programmatic dependent launch), so that part of the gather overlaps the
 * selection; the rest of I_f is read from `index` afterwards.  Only this
 * kernel's workspace is written before the wait.  If the library's previous
 * launch on this stream was a chained a5 on the same workspace (which may still
 * be merging from it), the call detects it and attends index-only instead (as
 * if seq_len were NULL): no caller rule to keep.  NULL: every row comes from
 * `index` (any sorted or unsorted list of positions is then accepted). */
int zoomr_sparse_decode_attn(const zoomr_geom *geom, int32_t batch, const void *q,
                             const zoomr_kv *kv, const int32_t *index, const int32_t *index_phys,
                             const int32_t *index_count, int32_t index_capacity,
                             const int32_t *seq_len, int32_t sink, int32_t window,
                             float softmax_scale, int32_t layer_begin, int32_t layer_count,
                             float *out, void *workspace, size_t workspace_bytes,
                             int32_t *dev_status, void *stream);

/* a1 + a2 + a3 + a4 fused into ONE launch for the single-rank / batch-sharded
 * step (Algorithm 1's selection).  Same semantics and bit-identical
 * outputs as calling, in order,
 *   zoomr_update_mean_keys(close_items) ; zoomr_score ; zoomr_select_topc ;
 *   zoomr_build_index
 * with the same arguments (plus, if index_phys is non-NULL, the page-resolved
 * row of every I_f entry for zoomr_sparse_decode_attn): each (layer, KV head) CTA recomputes the mean keys
 * of the summaries in close_items (device int32 [n_close][2] of (b, i); may be
 * empty) for its own (l, g), scores, and publishes its voters' top-k; the last
 * CTA of each sequence aggregates (exact integer votes and fixed-point A),
 * selects the consensus and writes the index set.  partial, agreeability,
 * alpha_out and topk_out are optional outputs (nullable).  Not for the
 * KV-head-sharded mode (no all-reduce point): use the separate calls there.
 * workspace: >= zoomr_select_workspace_bytes(geom, batch, max_summaries) bytes of
 * device memory, zero-filled once before the first call; every call leaves it
 * ready for the next (its per-sequence tickets are reset).
 *
 * close_items entries (b, i) with i < 0 mean "nothing closed" and are skipped
 * (zoomr_track_segments writes one entry per sequence).  update (nullable,
 * uint8 [B]): update[b] == 0 keeps sequence b's flags from the last update --
 * no a2/a3 for it, partial / agreeability untouched -- while a1 and a4 still
 * run (the selection is refreshed only at semantic boundaries, Alg.1 @P:417;
 * I_f is rebuilt every step from the held flags, reading Q14). */
size_t zoomr_select_workspace_bytes(const zoomr_geom *geom, int32_t batch, int32_t max_summaries);

int zoomr_select_fused(const zoomr_geom *geom, int32_t batch, const void *q, const zoomr_kv *kv,
                       const zoomr_segments *seg, const int32_t *close_items, int32_t n_close,
                       const uint8_t *update,
                       float *mean_keys, int32_t top_k, int32_t c, int32_t sink, int32_t window,
                       int64_t *partial, uint8_t *flags, float *agreeability, int32_t *index,
                       int32_t *index_phys, int32_t index_capacity, int32_t *index_count, float *alpha_out,
                       int32_t *topk_out, void *workspace, size_t workspace_bytes,
                       int32_t *dev_status, void *stream);

/* Chained launches across decode steps (ABI 8; ABI 9 made the ordering
 * self-checking).  Same arguments, semantics and bit-identical outputs as
 * zoomr_sparse_decode_attn / zoomr_select_fused; only the launch overlap differs:
 *   zoomr_sparse_decode_attn_chained lets a successor launched with
 *   programmatic dependent launch start as soon as every CTA has passed its
 *   griddepcontrol.wait -- so after this launch's own predecessor (the select
 *   that wrote I_f) has completed -- i.e. during this launch's streaming and
 *   end spread;
 *   zoomr_select_fused_chained, when the library's previous launch on the
 *   stream is a chained a5, is launched with PDL and runs a1 + a2 (mean keys,
 *   scoring, the per-voter top-k and the vote atomics) before
 *   griddepcontrol.wait, and a3 + a4 (writing partial / flags / index / count)
 *   after it, when that a5 has completed and its writes are visible.  After
 *   any other launch it runs exactly like zoomr_select_fused.
 * So two selects on the same workspace never overlap (select(t+1) starts after
 * a5(t) passed its wait, which is after select(t) completed), and an a5 never
 * writes its workspace while a chained a5 on it may still run (detected above).
 * Remaining caller rule: a FOREIGN kernel enqueued between a chained a5 and
 * zoomr_select_fused_chained must not write a1/a2's inputs (q, the pools, page
 * table, segment table, seq_len, close_items, update, mean keys) after
 * triggering its own dependents early -- the library cannot see foreign
 * launches.  Launched without PDL (the common case) such a kernel is safe. */
int zoomr_sparse_decode_attn_chained(const zoomr_geom *geom, int32_t batch, const void *q,
                                     const zoomr_kv *kv, const int32_t *index, const int32_t *index_phys,
                                     const int32_t *index_count, int32_t index_capacity,
                                     const int32_t *seq_len, int32_t sink, int32_t window,
                                     float softmax_scale, int32_t layer_begin, int32_t layer_count,
                                     float *out, void *workspace, size_t workspace_bytes,
                                     int32_t *dev_status, void *stream);

int zoomr_select_fused_chained(const zoomr_geom *geom, int32_t batch, const void *q, const zoomr_kv *kv,
                               const zoomr_segments *seg, const int32_t *close_items, int32_t n_close,
                               const uint8_t *update,
                               float *mean_keys, int32_t top_k, int32_t c, int32_t sink, int32_t window,
                               int64_t *partial, uint8_t *flags, float *agreeability, int32_t *index,
                               int32_t *index_phys, int32_t index_capacity, int32_t *index_count, float *alpha_out,
                               int32_t *topk_out, void *workspace, size_t workspace_bytes,
                               int32_t *dev_status, void *stream);

/* The fused select split around the KV-head-sharded exchange (SURVEY 8(e).2,
 * ABI 9): the caller all-reduces `partial` (SUM over ranks) between the two.
 *   zoomr_select_front = a1 + a2 of zoomr_select_fused (mean keys of close_items,
 *     alpha, per-voter top-k) for the rank's local heads, with the
 *     cross-head / cross-layer aggregation: writes partial int64 [B][2][max_summaries]
 *     = (votes, fixed-point A; entries >= N_t zero) -- the same values as
 *     zoomr_score.  Sequences with update[b] == 0 are skipped (partial row
 *     untouched).  workspace as for zoomr_select_fused (the same buffer may serve both).
 *   zoomr_select_tail = a3 + a4 from a given partial: flags,
 *     agreeability (nullable), I_f, count; one CTA per sequence.  kv may be NULL
 *     unless index_phys is given (it supplies the page table).  Launched so that a
 *     following a5 with early rows overlaps it.
 * front + all-reduce + tail is bit-identical to zoomr_score + all-reduce +
 * zoomr_select_topc + zoomr_build_index (and, on one rank, to zoomr_select_fused). */
int zoomr_select_front(const zoomr_geom *geom, int32_t batch, const void *q, const zoomr_kv *kv,
                       const zoomr_segments *seg, const int32_t *close_items, int32_t n_close,
                       const uint8_t *update, float *mean_keys, int32_t top_k, int64_t *partial,
                       float *alpha_out, int32_t *topk_out, void *workspace, size_t workspace_bytes,
                       int32_t *dev_status, void *stream);

int zoomr_select_tail(const zoomr_geom *geom, int32_t batch, const zoomr_kv *kv, const zoomr_segments *seg,
                      const int64_t *partial, const uint8_t *update, int32_t c, int32_t sink, int32_t window,
                      uint8_t *flags, float *agreeability, int32_t *index, int32_t *index_phys,
                      int32_t index_capacity, int32_t *index_count, int32_t *dev_status, void *stream);

/* ---- Algorithm 1's per-token bookkeeping, on device ----------
 *
 * a0 -- KV append, Alg.1 @P:407 ("Append k_t and v_t to KV cache"): writes the
 * current token's rows k_new / v_new (bf16 [B][L][H_kv][d]) at position
 * T = seq_len[b] of sequence b (page page_table[b][T / P], slot T % P), then sets
 * seq_len[b] = T + 1.  The pools may be pinned host memory (the host tier's
 * write-through copy).  Device errors: INDEX_RANGE (no page for T). */
int zoomr_append_kv(const zoomr_geom *geom, int32_t batch, const zoomr_kv *kv, const void *k_new,
                    const void *v_new, int32_t *seq_len, int32_t *dev_status, void *stream);

/* The rows of the newest token (position seq_len[b] - 1, already counted) into
 * another copy of the cache -- the host tier's hot pool after zoomr_tier_fetch
 * made the page resident (the host copy took it through zoomr_append_kv).
 * seq_len is not changed.  A position whose page entry is -1 (not resident, e.g.
 * in the host tier's hot pool) is skipped: the tier's fetch brings the page with
 * the row from the host cache.  Device errors: INDEX_RANGE (an entry out of range). */
int zoomr_write_newest_kv(const zoomr_geom *geom, int32_t batch, const zoomr_kv *kv, const void *k_new,
                          const void *v_new, const int32_t *seq_len, int32_t *dev_status, void *stream);

/* Segment tracking from the token just appended (P:19-21 summary delimiters,
 * SPEC ingest_token S:36-45; P:109 semantic boundaries).  token_ids[b] is the id
 * of the token at position pos = seq_len[b] - 1 of sequence b:
 *   begin_id: a summary opens at pos; the open tail before it becomes the pending R;
 *   end_id:   the open summary closes: S_i = [open, pos + 1) (both delimiters
 *             included), R_i = the pending R; bounds[b][i] = (r0, r1, s0, s1),
 *             num_summaries[b] = i + 1, close_items[b] = (b, i) -- else (b, -1);
 *   any id in boundary_ids[0..n_boundary): update[b] = 1 (selection update this
 *             step, for zoomr_select_fused), else 0.
 * state: int32 [B][4], 16-byte aligned, = (open summary start or -1, open-tail
 * start, pending R start, pending R end), initialised by the caller to
 * (-1, N_p, N_p, N_p) after a prompt of N_p tokens.  Device errors:
 * SEGMENT_ORDER (begin inside an open summary, end without one), CAPACITY
 * (more than max_summaries summaries). */
int zoomr_track_segments(int32_t batch, const int32_t *token_ids, int32_t begin_id, int32_t end_id,
                         const int32_t *boundary_ids, int32_t n_boundary, const int32_t *seq_len,
                         int32_t *bounds, int32_t *num_summaries, int32_t max_summaries, int32_t *state,
                         int32_t *close_items, uint8_t *update, int32_t *dev_status, void *stream);

/* The paper's transfer unit, layer by layer ("For each layer of the
 * model, the required KV cache slices are transferred to the GPU ... while the
 * KVs for the next layer are prefetched"): copies the rows
 * of I_f (index / index_count as a4 writes them) of layers [layer_begin,
 * layer_begin + layer_count), every KV head, K and V, from the host cache
 * (host_kv: pinned host pools read through their unified address, bf16
 * [L][num_pages][H_kv][P][d], device page table) into the slice buffers
 * slice_k / slice_v, device bf16 [layer_count][B * slice_pages_per_seq][H_kv]
 * [slice_page_size][d]: row j of sequence b lands in slice page
 * b * slice_pages_per_seq + j / slice_page_size, slot j % slice_page_size.  The
 * slice is then a pool that a5 attends with the identity page table and the
 * index 0 .. count-1 (positions are irrelevant to attention).
 * slice_page_size * slice_pages_per_seq >= index_capacity.  Launched with PDL:
 * the index is read after the preceding kernel completed.  Device errors:
 * INDEX_RANGE (a position without a host page). */
int zoomr_tier_gather_slice(const zoomr_geom *geom, int32_t batch, const zoomr_kv *host_kv, const int32_t *index,
                            const int32_t *index_count, int32_t index_capacity, int32_t layer_begin,
                            int32_t layer_count, void *slice_k, void *slice_v, int32_t slice_page_size,
                            int32_t slice_pages_per_seq, int32_t *dev_status, void *stream);

/* zoomr_append_kv + zoomr_track_segments without a host round trip (ABI 9): the
 * token's rows at position T = seq_len[b] (one CTA per (layer, sequence)), then a
 * tracking kernel launched with PDL behind the row copy -- it starts once every
 * row CTA has used T -- that tracks position T and sets seq_len[b] = T + 1.  The
 * same results as the two calls.  Right behind the library's chained a5 the row
 * copy is itself launched with PDL and overlaps that a5's end (a5 has read
 * seq_len in its prologue and reads no row at position T); both kernels end with
 * griddepcontrol.wait, so the call completes only after that a5 and the next
 * launch (the selection, which rewrites I_f) does not overlap it.  The pools may
 * be pinned host memory (the host tier's write-through).  mirror (nullable,
 * page size mirror_page_size, its own page table): a second pool that also gets
 * the rows where their page is resident (entry -1: skipped, as
 * zoomr_write_newest_kv) -- the host tier's HBM hot pool, in the same launch.
 * Other arguments as the two calls. */
int zoomr_append_track(const zoomr_geom *geom, int32_t batch, const zoomr_kv *kv, const zoomr_kv *mirror,
                       int32_t mirror_page_size, const void *k_new, const void *v_new, const int32_t *token_ids,
                       int32_t begin_id, int32_t end_id,
                       const int32_t *boundary_ids, int32_t n_boundary, int32_t *seq_len, int32_t *bounds,
                       int32_t *num_summaries, int32_t max_summaries, int32_t *state, int32_t *close_items,
                       uint8_t *update, int32_t *dev_status, void *stream);

/* ---- Token-sharded split-K across GPUs (H_kv < #GPUs) --------
 *
 * The KV cache of a sequence is spread over R ranks by token (owner[b][t] = the
 * rank holding token t; a rank's page table maps the pages of its tokens).  The
 * selection (a1..a4) is replicated -- every rank holds the mean keys of every
 * closed summary -- so every rank derives the same I_f.  Each rank attends over
 * the part of I_f it owns and the R partial results are combined by their
 * partition functions: for disjoint I_1 .. I_R with union I_f,
 *   softmax-attention over I_f = sum_r e^{lse_r} o_r / sum_r e^{lse_r},
 *   lse_r = ln sum_{j in I_r} exp(s_j),  s_j = q . k_j * softmax_scale.
 *
 * zoomr_shard_index: local_index[b*cap + 0 .. local_count[b]) = the entries t of
 * index[b*cap + 0 .. min(index_count[b], cap)) with owner[b*owner_stride + t] ==
 * rank, order kept.  owner: uint8 [B][owner_stride] (device).  Device errors:
 * INDEX_RANGE (t < 0 or t >= owner_stride; the entry is dropped). */
int zoomr_shard_index(int32_t batch, const int32_t *index, const int32_t *index_count,
                      int32_t index_capacity, const uint8_t *owner, int32_t owner_stride, int32_t rank,
                      int32_t *local_index, int32_t *local_count, int32_t *dev_status, void *stream);

/* a5 over an arbitrary (e.g. rank-local) index list, also writing the natural-log
 * partition function lse: fp32 [B][L][H_q], lse[b,l,h] = ln sum_{j in I_b}
 * exp(q[b,l,h] . k_j * softmax_scale).  Arguments as zoomr_sparse_decode_attn
 * without the phase-A rows (seq_len = NULL); lse must be non-NULL.  A sequence
 * with index_count 0 is skipped: its out and lse rows are left untouched (the
 * merge below excludes it through part_count).  Nothing is read before the
 * preceding kernel on the stream has completed -- the page table included, so
 * it may be that kernel's output (zoomr_tier_fetch's residency table).
 * layer_begin / layer_count as for zoomr_sparse_decode_attn (lse rows of other
 * layers untouched): the host tier attends layer by layer behind its fetch.
 * seq_len / sink / window (nullable seq_len, ABI 9): the early rows of
 * zoomr_sparse_decode_attn -- I_p and I_w attended before the wait, their
 * page-table entries read from global memory then -- for a page table that the
 * preceding kernels may still be changing elsewhere: the caller guarantees that
 * the entries of the sink and window pages do not change during this call (the
 * host tier: zoomr_tier_fetch with seq_len keeps the next token's page resident
 * one step ahead, so after one warm step they never do). */
int zoomr_sparse_decode_attn_lse(const zoomr_geom *geom, int32_t batch, const void *q,
                                 const zoomr_kv *kv, const int32_t *index, const int32_t *index_phys,
                                 const int32_t *index_count, int32_t index_capacity,
                                 const int32_t *seq_len, int32_t sink, int32_t window, float softmax_scale,
                                 int32_t layer_begin, int32_t layer_count, float *out, float *lse,
                                 void *workspace, size_t workspace_bytes, int32_t *dev_status, void *stream);

/* zoomr_sparse_decode_attn_lse with the chained trigger of
 * zoomr_sparse_decode_attn_chained (ABI 9): a PDL-launched successor -- the host
 * tier's next zoomr_append_track -- may start once every CTA has passed its
 * wait.  Same arguments and results. */
int zoomr_sparse_decode_attn_lse_chained(const zoomr_geom *geom, int32_t batch, const void *q,
                                         const zoomr_kv *kv, const int32_t *index, const int32_t *index_phys,
                                         const int32_t *index_count, int32_t index_capacity,
                                         const int32_t *seq_len, int32_t sink, int32_t window, float softmax_scale,
                                         int32_t layer_begin, int32_t layer_count, float *out, float *lse,
                                         void *workspace, size_t workspace_bytes, int32_t *dev_status, void *stream);

/* Combine n_parts partial attention results (normally the all-gathered outputs
 * of zoomr_sparse_decode_attn_lse on each rank, over disjoint index sets):
 *   part_out fp32 [n_parts][B][L][H_q][d], part_lse fp32 [n_parts][B][L][H_q],
 *   part_count int32 [n_parts][B] (nullable): part r of sequence b is skipped
 *   when part_count[r*B + b] == 0 (its rows are not read).
 *   out[b,l,h] = sum_r w_r part_out[r,b,l,h] / sum_r w_r,  w_r = exp(lse_r - max_r lse_r),
 * parts in order r = 0 .. n_parts-1 (deterministic, identical on every rank);
 * lse (nullable) = the combined partition function.  A sequence with no part
 * gets out = 0, lse = -inf. */
int zoomr_merge_attn(const zoomr_geom *geom, int32_t batch, int32_t n_parts, const float *part_out,
                     const float *part_lse, const int32_t *part_count, float *out, float *lse,
                     void *stream);

/* ---- H2O, the paper's heavy-hitter comparison policy ----
 * The paper only cites H2O; the rule is SPEC h2o_step, readings H1-H2
 * in DESIGN.md 8c.  One H2O step = zoomr_h2o_select (the retained set I for the
 * current T) -> zoomr_sparse_decode_attn_logits over I -> zoomr_h2o_accumulate.
 *
 * a5 over any index list (as zoomr_sparse_decode_attn_lse), also writing the
 * logits: logits fp32 [B][L][H_q][index_capacity], logits[b,l,h,i] =
 * q[b,l,h] . k_{index[b,i]} * softmax_scale for i < index_count[b] (other
 * entries untouched).  lse and logits must be non-NULL. */
int zoomr_sparse_decode_attn_logits(const zoomr_geom *geom, int32_t batch, const void *q,
                                    const zoomr_kv *kv, const int32_t *index, const int32_t *index_count,
                                    int32_t index_capacity, float softmax_scale, float *out, float *lse,
                                    float *logits, void *workspace, size_t workspace_bytes,
                                    int32_t *dev_status, void *stream);

/* The attention each retained token received this step, averaged over layers
 * and query heads ("per-retained-token softmax weights averaged over
 * heads/layers"), added to its cumulative score:
 *   score[b*score_stride + index[b,i]] += (1/(L*H_q)) sum_{l,h} exp(logits[b,l,h,i] - lse[b,l,h])
 * (fixed summation order: deterministic).  score: fp32 [B][score_stride],
 * score_stride > every position.  index entries must be distinct within a
 * sequence.  index_copy / count_copy (nullable, [B][index_capacity] / [B]):
 * receive a copy of the index set -- the prev_index of the next
 * zoomr_h2o_select.  Device errors: INDEX_RANGE (position >= score_stride). */
int zoomr_h2o_accumulate(const zoomr_geom *geom, int32_t batch, const int32_t *index,
                         const int32_t *index_count, int32_t index_capacity, const float *logits,
                         const float *lse, float *score, int32_t score_stride, int32_t *index_copy,
                         int32_t *count_copy, int32_t *dev_status, void *stream);

/* The retained set for T = seq_len[b]: with s' = min(sink, T) and
 * w0 = max(s', T - window),
 *   index[b] = [0, s') u top-K(prev_index[b] n [s', w0)) u [w0, T),  K = max(0, budget - s' - (T - w0)),
 * top-K by cumulative score desc, ties -> smaller position; written sorted
 * ascending (prev_index must be sorted ascending, as this function writes it).
 * prev_index and index: int32 [B][index_capacity], distinct buffers.  Evicted
 * positions never return (they are not in prev_index).  Device errors:
 * CAPACITY (count clamped), INDEX_RANGE, UNSUPPORTED (more than 16384
 * previously retained positions in [s', w0)). */
int zoomr_h2o_select(int32_t batch, const int32_t *prev_index, const int32_t *prev_count,
                     int32_t index_capacity, const float *score, int32_t score_stride,
                     const int32_t *seq_len, int32_t sink, int32_t window, int32_t budget, int32_t *index,
                     int32_t *index_count, int32_t *dev_status, void *stream);

/* ---- Host-memory tier (the paper's system) -------------
 * The full cache lives in pinned host memory (host_kv: same layout and page
 * table as zoomr_kv; k and v must be device-accessible, i.e. pinned with
 * cudaHostAlloc / cudaHostRegister, read through their unified addresses).
 * HBM holds a hot pool of hot_pages pages of hot_page_size tokens (Ph, a
 * divisor of the host page size P; R = P / Ph) caching it:
 *   hot_k, hot_v   bf16 [L][hot_pages][H_kv][Ph][d],
 *   hot_page_table int32 [B][max_pages * R]: hot logical page (tokens
 *                  [j*Ph, (j+1)*Ph) of sequence b) -> hot page or -1,
 *   hot_owner      int32 [hot_pages]: b*max_pages*R + hot logical page, or -1 (free),
 *   hot_stamp      int32 [hot_pages]: last step the page was used, -1 if never;
 * initialised by the caller to -1 / -1 / -1; workspace zero-filled once
 * (zoomr_tier_workspace_bytes(batch, max_pages * R, hot_pages)).
 * zoomr_tier_fetch makes every hot logical page that I_f (index / index_count,
 * as a4 writes it) touches resident: pages already resident are stamped with
 * the step; each missing page takes, in page order, the least recently used
 * hot page (smallest (stamp, page)) among those this step does not touch, and
 * its rows are copied from the host (all layers, K and V).  Afterwards a5 runs
 * on the hot pool (geometry page_size = Ph, zoomr_kv {hot_k, hot_v, hot_pages,
 * hot_page_table, max_pages * R}) through zoomr_sparse_decode_attn_lse, which
 * reads nothing before this call's kernels have completed.  Device errors:
 * CAPACITY (the hot pool cannot hold the pages of this step's I_f; the rest
 * stay missing), INDEX_RANGE. */
size_t zoomr_tier_workspace_bytes(int32_t batch, int32_t hot_max_pages, int32_t hot_pages);
/* seq_len (nullable, device int32 [B], ABI 9): also make the hot page of
 * position seq_len[b] -- the NEXT token's -- resident now (look-ahead), so that
 * at the next step every sink and window page is resident before that step's
 * plan runs (its a5 may then read their entries early, see
 * zoomr_sparse_decode_attn_lse, and zoomr_append_track's mirror /
 * zoomr_write_newest_kv find the newest token's page resident).  When
 * seq_len[b] is a multiple of hot_page_size the page holds no row yet: it is
 * allocated without copying anything from the host. */
int zoomr_tier_fetch(const zoomr_geom *geom, int32_t batch, const zoomr_kv *host_kv, void *hot_k, void *hot_v,
                     int32_t hot_pages, int32_t hot_page_size, int32_t *hot_page_table, int32_t *hot_owner,
                     int32_t *hot_stamp, const int32_t *index, const int32_t *index_count,
                     int32_t index_capacity, const int32_t *seq_len, void *workspace, size_t workspace_bytes,
                     int32_t *dev_status, void *stream);

/* Human-readable status name; never NULL. */
const char *zoomr_status_str(int status);

/* ZOOMR_ABI_VERSION of the loaded library. */
int zoomr_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ZOOMR_H */
