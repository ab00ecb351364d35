// zoomr_select_fused -- a1 + a2 + a3 + a4 of one decode step in ONE launch.
//
// Algorithm 1's per-step selection has a natural all-to-one shape:
// every (layer, KV head) scores independently (a1, a2), then one consensus per
// sequence (a3) decides the index set (a4).  The standalone kernels express that
// with four launches and a global reduction through memory; on B200 at batch 1
// each launch boundary and each dependent round trip costs microseconds against
// a ~60 us step, so this kernel keeps the same building blocks
// (select_common.cuh) but chains them with a last-CTA-arrives handoff:
//   * CTA (l, g, b): recompute the mean key of every summary of b that closed
//     this step (a1, block_mean_key), score all N_t mean keys against the G
//     queries and take each voter's top-k (a2, block_score_topk), and add its
//     G*k votes to per-sequence accumulators in the workspace with integer
//     atomics at L2 -- votes and A = sum round(alpha*2^32), exact and
//     order-independent (reading Q2);
//   * the last CTA of sequence b to arrive (atomic ticket) reads the
//     aggregate (and zeroes the accumulators for the next call), runs the
//     consensus top-c (a3, block_topc) and builds I_f (a4, block_build_index),
//     writing partial / flags / index / count, and resets its ticket.
// (A first version published the picks and aggregated them in the last CTA
// with shared-memory atomics: the consensus votes concentrate on a few
// summaries, and the 64-bit shared atomic is a CAS loop -- 17 us of
// serialisation; L2 integer atomics spread over the CTAs' lifetimes cost ~0.)
// Results are bit-identical to the standalone chain (same arithmetic, integer
// aggregation).  Single-rank only: the KV-head-sharded mode needs the
// all-reduce between a2 and a3 and uses the standalone entry points.
#include "common.cuh"

ZOOMR_TL_STORAGE(fused)
#ifdef ZOOMR_TIMELINE  // timeline builds: marks inside the scoring loop of the fused select
#define ZOOMR_SCORE_MARK(i)                             \
  do {                                                  \
    const bool tl_on_ = *(volatile int *)&zoomr::g_tl_on; \
    TL(i);                                              \
  } while (0)
#endif
#include "select_common.cuh"

namespace zoomr {


struct FusedParams {
  const __nv_bfloat16 *q;
  const __nv_bfloat16 *kpool;
  int64_t num_pages;
  const int32_t *page_table;
  int32_t max_pages;
  const int32_t *bounds;
  const int32_t *num_summaries;
  const int32_t *seq_len;
  int32_t max_summaries;
  const int32_t *items;
  int32_t n_items;
  float *mean_keys;
  int32_t top_k, c, sink, window;
  int64_t *partial;       // nullable
  uint8_t *flags;
  float *agreeability;    // nullable
  int32_t *index;
  int32_t *index_phys;    // nullable: page-resolved rows for a5
  int32_t cap;
  int32_t *count;
  float *alpha_out;       // nullable
  int32_t *topk_out;      // nullable
  int32_t *ws_votes;      // [B][MS]  accumulators, zero between calls
  long long *ws_a;        // [B][MS]
  int32_t *ws_ticket;     // [B]
  int32_t L, Hkv, P;
  int32_t *status;
  int32_t stop_after;  // debug A/B only: 0 full; 1 after the ticket; 2 after collect; 3 after a3
  int32_t pdl_front;  // chained: launched with PDL after a5; a1/a2 run before griddepcontrol.wait, a3/a4 after
  int32_t designated_tail;  // cooperative launch (grid co-resident): the last-launched CTA of b runs a3/a4
  const uint8_t *update;    // nullable: update[b] == 0 keeps b's flags (no a2/a3; a1 and a4 still run)
  int32_t mode;             // kFull a1..a4 | kFront a1 + a2 -> partial | kTail partial -> a3 + a4
};

// The KV-head-sharded step splits the fused select around its all-reduce
// (SURVEY 8(e).2): the front (every (l, g) CTA: a1, a2, top-k, vote atomics;
// the last CTA of b writes the rank's partial) and the tail (one CTA per
// sequence: a3 + a4 from the all-reduced partial) -- two launches instead of
// the five separate ones, and a5's early rows still overlap the tail.
enum FusedMode : int { kFull = 0, kFront = 1, kTail = 2 };

// kT threads per CTA: 256 (two CTAs per SM) when the grid fits in about one wave;
// 64 (eight per SM) for large batches, where the (l, g, b) CTAs come in many
// waves and each one's front end is a chain of dependent round trips -- four
// times the CTAs in flight hide that latency (configs[2]: 64 x 257 CTAs).
template <int D, int G, int kT = 256>
__global__ void __launch_bounds__(kT, 512 / kT) fused_select_kernel(const FusedParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int ticket_last;
  if (!p.pdl_front) allow_dependents();  // a5 may launch and run its prologue; it waits for our completion
  TL_INIT();
  TL(0);
  const int lg = blockIdx.x, b = blockIdx.y;
  const int l = lg / p.Hkv, g = lg - l * p.Hkv;
  const int Hq = p.Hkv * G, V = p.L * Hq, MS = p.max_summaries;
  int nt = p.num_summaries[b];
  if (nt > MS || nt < 0) {
    if (threadIdx.x == 0) set_status(p.status, ZOOMR_ERR_INDEX_RANGE);
    nt = nt < 0 ? 0 : MS;
  }
  const int T = p.seq_len[b];
  const int32_t *bd = p.bounds + (int64_t)b * MS * 4;
  float *mk = p.mean_keys + (((int64_t)b * p.L + l) * p.Hkv + g) * (int64_t)MS * D;

  const bool tail_only = p.mode == kTail;  // grid (1, B): straight to the collect of the given partial
  const int nlg = p.L * p.Hkv;
  // designated tail: CTA nlg of sequence b does no (l, g) work; it runs the tail's
  // code once on dummy shared-memory data while the others score (so a3/a4 then
  // run from a warm instruction cache instead of fetching each new block of code
  // through an L2 that a5's gather keeps flushing), then waits for their count
  const bool tail_cta = p.designated_tail && lg == nlg;
  // a selection update for b this step (else a2 / a3 are skipped and the flags held)
  const bool upd = !p.update || p.update[b];
  // Nothing for the (l, g) CTAs of b to do (no update, no summary closing: a decode
  // loop's typical token): they exit without counting and the tail CTA goes
  // straight to a4 instead of waiting for their arrivals.  Every CTA of b
  // evaluates the same condition from the same inputs.
  bool idle = false;
  if (p.designated_tail && p.mode == kFull && !upd) {
    idle = true;
    for (int it = 0; it < p.n_items; ++it)
      if (p.items[2 * it] == b && p.items[2 * it + 1] >= 0) idle = false;
  }
  if (idle && !tail_cta) return;
#ifndef ZOOMR_AB_NO_WARM  // A/B builds only: the tail CTA without the warm-up pass
  // (only when a3 will run: without an update the tail is collect + a4, and the
  // warm-up pass would sit on its critical path)
  if (tail_cta && upd) {
    SmemCarve sm{smem_raw};
    long long *A = sm.take<long long>(MS);
    int *v = sm.take<int>(MS);
    int *grp = sm.take<int>(2 * MS);
    int *hist = sm.take<int>(kHistBins);
    int *scratch = sm.take<int>(40);
    int4 *bds = sm.take<int4>(MS);
    sm.take<int>(p.max_pages);
    uint8_t *fl = sm.take<uint8_t>(MS);
    __shared__ float warm_ag;
    __shared__ int warm_count;
    for (int i = threadIdx.x; i < MS; i += blockDim.x) {
      // distinct votes at the top, the rest 1: every top-c path runs, with a tie group of one
      // (dummy data with a large tie group made the warm-up outlast the front end: +24 us at c = 32)
      v[i] = i < 40 ? 2000 - i : 1;
      A[i] = (long long)(i * 7919 % 1000) << 20;
      bds[i] = make_int4(8 * i + 4, 8 * i + 8, 8 * i + 8, 8 * i + 12);
    }
    __syncthreads();
    block_topc(v, A, nt, p.c > 0 ? p.c : 1, fl, hist, grp, scratch, &warm_ag);
    __syncthreads();
    block_build_index(reinterpret_cast<const int32_t *>(bds), nt, 8 * nt + 16, fl, 4, 8,
                      reinterpret_cast<int32_t *>(A), 2 * MS, &warm_count, grp, scratch, nullptr);
    __syncthreads();
  }
#endif
  // the G queries of this (l, g): loaded now, so that the load overlaps a1's chain
  // instead of adding a round trip between a1 and the scoring
  constexpr int kQPT = (G * D + kT - 1) / kT;  // per thread
  float qreg[kQPT];
  const __nv_bfloat16 *qb = p.q + (((int64_t)b * p.L + l) * Hq + (int64_t)g * G) * D;
  if (upd && !tail_only && !tail_cta) {
#pragma unroll
    for (int j = 0; j < kQPT; ++j) {
      const int x = threadIdx.x + j * kT;
      qreg[j] = x < G * D ? __bfloat162float(qb[x]) : 0.f;
    }
  }
  // ---- a1: mean keys of the summaries of b that closed this step -----------
  if (!tail_only && !tail_cta) {
    double *red = reinterpret_cast<double *>(smem_raw);  // [nwarps][D]
    for (int it = 0; it < p.n_items; ++it) {
      if (p.items[2 * it] != b) continue;
      const int i = p.items[2 * it + 1];
      if (i < 0) continue;  // "nothing closed" entry
      if (i >= nt) {
        if (threadIdx.x == 0) set_status(p.status, ZOOMR_ERR_INDEX_RANGE);
        continue;
      }
      const int s0 = bd[4 * i + 2], s1 = bd[4 * i + 3];
      if (s1 <= s0 || s0 < 0 || s1 > T) {
        if (threadIdx.x == 0) set_status(p.status, s1 <= s0 ? ZOOMR_ERR_EMPTY_SEGMENT : ZOOMR_ERR_INDEX_RANGE);
        continue;
      }
      block_mean_key<D>(p.kpool, p.num_pages, p.page_table + (int64_t)b * p.max_pages, p.max_pages, p.P, p.Hkv,
                        l, g, s0, s1, red, mk + (int64_t)i * D, p.status);
    }
    __syncthreads();  // this CTA's own global writes are visible to it after the barrier
    if (threadIdx.x == 0) TL(6);
  }

  // ---- a2: alpha + per-voter top-k (only at a selection update) ---------------------
  if (upd && !tail_only && !tail_cta) {
    float *qs = reinterpret_cast<float *>(smem_raw);                 // [G][D]
    float *al = qs + G * D;                                          // [G][MS]
    int *sel_i = reinterpret_cast<int *>(al + G * MS);               // [G][k]
    float *sel_a = reinterpret_cast<float *>(sel_i + G * p.top_k);   // [G][k]
    float *ao = p.alpha_out ? p.alpha_out + (((int64_t)b * p.L + l) * Hq + (int64_t)g * G) * MS : nullptr;
#pragma unroll
    for (int j = 0; j < kQPT; ++j) {
      const int x = threadIdx.x + j * kT;
      if (x < G * D) qs[x] = qreg[j];
    }
    __syncthreads();
    block_score_topk<D, G>(nullptr, mk, nt, p.top_k, qs, al, MS, ao, MS, sel_i, sel_a);
    if (threadIdx.x == 0) TL(8);
    const int kk = p.top_k < nt ? p.top_k : nt;
    for (int x = threadIdx.x; x < G * p.top_k; x += blockDim.x) {
      const int hh = x / p.top_k, r = x - hh * p.top_k;
      const int64_t voter = (int64_t)l * Hq + g * G + hh;
      if (r < kk) {  // votes and fixed-point A: integer atomics at L2, order-independent
        atomicAdd(&p.ws_votes[(int64_t)b * MS + sel_i[x]], 1);
        atomicAdd(reinterpret_cast<unsigned long long *>(&p.ws_a[(int64_t)b * MS + sel_i[x]]),
                  (unsigned long long)alpha_fixed(sel_a[x]));
      }
      if (p.topk_out) p.topk_out[((int64_t)b * V + voter) * p.top_k + r] = r < kk ? sel_i[x] : -1;
    }
  }
  // ---- ticket: the last CTA of sequence b carries on --------------------------
  // bar.sync orders the CTA's writes before thread 0's acq_rel ticket (release,
  // cumulative at gpu scope); the winner's acquire + bar.sync order its reads after.
  __syncthreads();
  if (threadIdx.x == 0) TL(1);
  if (tail_only) {
  } else if (p.designated_tail) {
  // The (l, g) CTAs count themselves with a fire-and-forget release add and exit
  // at once (their SMs go to a5 a round trip earlier); the tail CTA waits
  // (acquire) until all have counted.  Used only under a cooperative launch
  // (the whole grid is resident at once), so the CTAs it waits for are running.
  if (!tail_cta) {
    if (threadIdx.x == 0)
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.ws_ticket + b) : "memory");
    return;
  }
  if (threadIdx.x == 0 && !idle) {
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.ws_ticket + b) : "memory");
    } while (v != (unsigned)nlg);
  }
  __syncthreads();
  } else {
  if (threadIdx.x == 0) {
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(p.ws_ticket + b) : "memory");
    ticket_last = (old == (unsigned)(p.L * p.Hkv - 1));
  }
  __syncthreads();
  if (!ticket_last) return;
  }
  if (p.pdl_front) {  // the predecessor (a5) reads index / count: wait for it before a3/a4 write them
    asm volatile("griddepcontrol.wait;" ::: "memory");
    allow_dependents();
  }
  if (threadIdx.x == 0) TL(2);
  if (p.stop_after == 1 || (p.mode == kFront && !upd)) {  // (front without an update: only a1 had work)
    if (threadIdx.x == 0) p.ws_ticket[b] = 0;
    return;
  }

  // ---- aggregation (a2, cross-head / cross-layer), exact integer atomics --------
  SmemCarve sm{smem_raw};
  long long *A = sm.take<long long>(MS);
  int *v = sm.take<int>(MS);
  int *grp = sm.take<int>(2 * MS);      // a3 tie group, then a4 pieces
  int *hist = sm.take<int>(kHistBins);
  int *scratch = sm.take<int>(40);
  int4 *bds = sm.take<int4>(MS);        // segment table of b
  int *pts = sm.take<int>(p.max_pages); // page table of b (for index_phys)
  uint8_t *fl = sm.take<uint8_t>(MS);
  if (p.index_phys)
    for (int x = threadIdx.x; x < p.max_pages; x += blockDim.x) pts[x] = p.page_table[(int64_t)b * p.max_pages + x];
  // collect the aggregate (leaving the accumulators zeroed for the next call)
  // and stage the segment table for a4; without an update, the held flags
  // (kCU entries per thread per round, every load issued before the stores:
  // one round trip per round instead of one per entry)
  constexpr int kCU = 4;
  for (int i0 = threadIdx.x; i0 < nt; i0 += kCU * blockDim.x) {
    int4 bq[kCU];
    int vq[kCU];
    long long aq[kCU];
#pragma unroll
    for (int u = 0; u < kCU; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < nt) {
        bq[u] = reinterpret_cast<const int4 *>(bd)[i];
        if (upd && tail_only) {  // the (all-reduced) partial: votes, fixed-point A
          vq[u] = (int)p.partial[(int64_t)b * 2 * MS + i];
          aq[u] = p.partial[(int64_t)b * 2 * MS + MS + i];
        } else if (upd) {
          vq[u] = __ldcg(&p.ws_votes[(int64_t)b * MS + i]);
          aq[u] = __ldcg(&p.ws_a[(int64_t)b * MS + i]);
        } else {
          vq[u] = p.flags[(int64_t)b * MS + i];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kCU; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < nt) {
        bds[i] = bq[u];
        if (upd) {
          v[i] = vq[u];
          A[i] = aq[u];
          if (!tail_only) {
            p.ws_votes[(int64_t)b * MS + i] = 0;
            p.ws_a[(int64_t)b * MS + i] = 0;
          }
        } else {
          fl[i] = (uint8_t)vq[u];
        }
      }
    }
  }
  __syncthreads();
  if (upd) {
  if (p.partial && !tail_only) {
    int64_t *pv = p.partial + (int64_t)b * 2 * MS;
    for (int i = threadIdx.x; i < MS; i += blockDim.x) {
      pv[i] = i < nt ? v[i] : 0;
      pv[MS + i] = i < nt ? A[i] : 0;
    }
  }
  if (p.stop_after == 2 || p.mode == kFront) { if (threadIdx.x == 0) p.ws_ticket[b] = 0; return; }
  if (threadIdx.x == 0) TL(3);
  // ---- a3: consensus top-c ----------------------------------------------------------
  block_topc(v, A, nt, p.c, fl, hist, grp, scratch, p.agreeability ? p.agreeability + b : nullptr);

  uint8_t *fo = p.flags + (int64_t)b * MS;
  for (int i = threadIdx.x; i < MS; i += blockDim.x) fo[i] = i < nt ? fl[i] : 0;
  __syncthreads();
  }  // upd
  if (p.stop_after == 3) { if (threadIdx.x == 0) p.ws_ticket[b] = 0; return; }
  if (threadIdx.x == 0) TL(4);
  // ---- a4: the index set --------------------------------------------------------------
  if (T < 1) {
    if (threadIdx.x == 0) {
      set_status(p.status, ZOOMR_ERR_INVALID_ARG);
      p.count[b] = 0;
    }
  } else {
    block_build_index(reinterpret_cast<const int32_t *>(bds), nt, T, fl, p.sink, p.window, p.index + (int64_t)b * p.cap,
                      p.cap, p.count + b, grp, scratch, p.status,
                      p.index_phys ? p.index_phys + (int64_t)b * p.cap : nullptr, pts, p.P, p.Hkv * p.P);
  }
  if (threadIdx.x == 0 && !tail_only) p.ws_ticket[b] = 0;  // ready for the next step
  __syncthreads();
  if (threadIdx.x == 0) TL(5);
}

template <int D, int G>
size_t fused_smem_bytes(int MS, int top_k, int max_pages, int threads = 256) {
  const size_t a1 = 8 * (size_t)(threads / 32) * D;
  const size_t a2 = (size_t)G * D * 4 + (size_t)G * MS * 4 + (size_t)G * top_k * 8;
  const size_t a3 = (size_t)MS * (8 + 4 + 8 + 16 + 1) + (kHistBins + 40) * 4 + (size_t)max_pages * 4 + 9 * 16;
  return a1 > a2 ? (a1 > a3 ? a1 : a3) : (a2 > a3 ? a2 : a3);
}

}  // namespace zoomr

using namespace zoomr;

extern "C" size_t zoomr_select_workspace_bytes(const zoomr_geom *geom, int32_t batch, int32_t max_summaries) {
  if (check_geom(geom) || batch < 1 || max_summaries < 1) return 0;
  return (size_t)batch * max_summaries * (8 + 4) + (size_t)batch * 4 + 256;
}

#ifdef ZOOMR_AB_NO_COOP  // A/B builds only: the last-arriving CTA runs a3/a4 (no cooperative launch)
constexpr bool kDesignatedTail = false;
#else
constexpr bool kDesignatedTail = true;
#endif

static int select_fused(const zoomr_geom *geom, int32_t batch, const void *q, const zoomr_kv *kv,
                        const zoomr_segments *seg, const int32_t *close_items, int32_t n_close,
                        const uint8_t *update,
                        float *mean_keys, int32_t top_k, int32_t c, int32_t sink, int32_t window,
                        int64_t *partial, uint8_t *flags, float *agreeability, int32_t *index,
                        int32_t *index_phys, int32_t index_capacity, int32_t *index_count, float *alpha_out,
                        int32_t *topk_out, void *workspace, size_t workspace_bytes,
                        int32_t *dev_status, void *stream, bool chained, int mode = kFull) {
  int rc = check_geom(geom);
  if (rc) return rc;
  if (batch < 1 || !seg || !seg->bounds || !seg->num_summaries || !seg->seq_len || seg->max_summaries < 1)
    return ZOOMR_ERR_INVALID_ARG;
  const bool front = mode != kTail, back = mode != kFront;  // runs a1 + a2 / runs a3 + a4
  if (front && (!q || !kv || !kv->k || !kv->page_table || kv->num_pages < 1 || kv->max_pages < 1 || !mean_keys ||
                top_k < 1 || n_close < 0 || (n_close > 0 && !close_items) || !workspace))
    return ZOOMR_ERR_INVALID_ARG;
  if (back && (!flags || !index || !index_count || index_capacity < 1 || c < 0 || sink < 0 || window < 1))
    return ZOOMR_ERR_INVALID_ARG;
  if (mode != kFull && !partial) return ZOOMR_ERR_INVALID_ARG;  // the front's output / the tail's input
  if (index_phys && (!kv || !kv->page_table || kv->max_pages < 1)) return ZOOMR_ERR_INVALID_ARG;
  if ((front && top_k > kMaxTopK) || seg->max_summaries > kMaxSummaries) return ZOOMR_ERR_UNSUPPORTED;
  if (front && workspace_bytes < zoomr_select_workspace_bytes(geom, batch, seg->max_summaries))
    return ZOOMR_ERR_WORKSPACE;
  if (!front) {
    top_k = 1;  // unused by the tail; keeps the shared-memory sizing valid
    n_close = 0;
  }
  FusedParams p;
  p.mode = mode;
  p.q = (const __nv_bfloat16 *)q;
  p.kpool = kv ? (const __nv_bfloat16 *)kv->k : nullptr;
  p.num_pages = kv ? kv->num_pages : 0;
  p.page_table = kv ? kv->page_table : nullptr;
  p.max_pages = kv ? kv->max_pages : 1;
  p.bounds = seg->bounds;
  p.num_summaries = seg->num_summaries;
  p.seq_len = seg->seq_len;
  p.max_summaries = seg->max_summaries;
  p.items = close_items;
  p.n_items = n_close;
  p.update = update;
  p.mean_keys = mean_keys;
  p.top_k = top_k;
  p.c = c;
  p.sink = sink;
  p.window = window;
  p.partial = partial;
  p.flags = flags;
  p.agreeability = agreeability;
  p.index = index;
  p.index_phys = index_phys;
  p.cap = index_capacity;
  p.count = index_count;
  p.alpha_out = alpha_out;
  p.topk_out = topk_out;
  const size_t nacc = (size_t)batch * seg->max_summaries;
  p.ws_a = (long long *)workspace;
  p.ws_votes = (int32_t *)((char *)workspace + nacc * 8);
  p.ws_ticket = (int32_t *)((char *)workspace + nacc * 12);
  p.L = geom->num_layers;
  p.Hkv = geom->num_kv_heads;
  p.P = geom->page_size;
  p.status = dev_status;
  cudaStream_t s = (cudaStream_t)stream;
  // The chained variant overlaps a1/a2 with its predecessor only when that
  // predecessor is the library's chained a5 (which writes none of a1/a2's
  // inputs); after anything else it is launched like the plain one.
  p.pdl_front = chained && prev_launch_is(s, kLaunchA5Chained, nullptr) ? 1 : 0;
  p.stop_after = 0;
#ifdef ZOOMR_EXPERIMENTS
  {
    const char *e = getenv("ZOOMR_FUSED_STOP");  // experiment builds only: cut the kernel short for A/B timing
    p.stop_after = e ? atoi(e) : 0;
  }
#endif
  const int G = geom->num_q_heads / geom->num_kv_heads;
  dim3 grid(mode == kTail ? 1 : geom->num_layers * geom->num_kv_heads, batch);
  const int max_pages = p.max_pages;
  /* more than one wave of 256-thread CTAs (two per SM): 64-thread CTAs, eight per SM */
  const bool many = mode == kFull && (int64_t)(grid.x + 1) * grid.y > (int64_t)2 * num_sms();
#ifndef ZOOMR_MANY_THREADS  // (A/B builds: 128 or 32)
#define ZOOMR_MANY_THREADS 64
#endif
  /* a grid of at most one CTA per SM (e.g. one KV head's 80 layers): 512-thread CTAs */
#ifndef ZOOMR_FEW_MODES
#define ZOOMR_FEW_MODES 1  // 1: kFull only; 2: kFull and kFront
#endif
  const bool few = (mode == kFull || (ZOOMR_FEW_MODES == 2 && mode == kFront)) &&
                   (int64_t)(grid.x + 1) * grid.y <= (int64_t)num_sms();
  const int nthr = many ? ZOOMR_MANY_THREADS : few ? 512 : 256;
#define ZOOMR_FS(DD, GG)                                                                         \
  do {                                                                                           \
    auto kfn = many  ? fused_select_kernel<DD, GG, ZOOMR_MANY_THREADS>                           \
               : few ? fused_select_kernel<DD, GG, 512>                                          \
                     : fused_select_kernel<DD, GG, 256>;                                         \
    const size_t smem = fused_smem_bytes<DD, GG>(seg->max_summaries, top_k, max_pages, nthr);   \
    if (smem > 200 * 1024) return ZOOMR_ERR_UNSUPPORTED;                                         \
    if (smem > 48 * 1024) cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    prefer_max_smem(kfn);                                                                        \
    int per_sm = 0;                                                                              \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, nthr, smem);                     \
    /* the designated tail CTA spins until the (l, g) CTAs of its sequence have counted;    \
       those never wait on anything, so they progress whenever any slot is free -- the B    \
       tail CTAs never fill the GPU, since the whole grid fits at once (checked here).  The \
       plain launch is cooperative, which makes the driver guarantee it; the chained one is \
       launched with PDL behind a5, whose CTAs leave as they finish, and the tail CTAs -- the \
       last of the grid -- start last (advisor note: no spin on CTAs that cannot run). */    \
    p.designated_tail = kDesignatedTail && mode != kTail &&                                      \
                        (int64_t)(grid.x + 1) * grid.y <= (int64_t)per_sm * num_sms();           \
    if (p.designated_tail) grid.x += 1; /* + the tail CTA of each sequence */                   \
    if (p.pdl_front) launch_pdl(kfn, grid, nthr, smem, s, p);                                    \
    else if (p.designated_tail) launch_cooperative(kfn, grid, nthr, smem, s, p);                 \
    else kfn<<<grid, nthr, smem, s>>>(p);                                                        \
  } while (0)
#define ZOOMR_FS_G(DD)               \
  switch (G) {                       \
    case 1: ZOOMR_FS(DD, 1); break;  \
    case 2: ZOOMR_FS(DD, 2); break;  \
    case 4: ZOOMR_FS(DD, 4); break;  \
    case 7: ZOOMR_FS(DD, 7); break;  \
    default: ZOOMR_FS(DD, 8); break; \
  }
  switch (geom->head_dim) {
    case 16: ZOOMR_FS_G(16); break;
    case 32: ZOOMR_FS_G(32); break;
    case 64: ZOOMR_FS_G(64); break;
    default: ZOOMR_FS_G(128); break;
  }
#undef ZOOMR_FS_G
#undef ZOOMR_FS
  return launch_status(s);
}

#define ZOOMR_SELECT_FUSED_ARGS                                                                                 \
  const zoomr_geom *geom, int32_t batch, const void *q, const zoomr_kv *kv, const zoomr_segments *seg,          \
      const int32_t *close_items, int32_t n_close, const uint8_t *update, float *mean_keys, int32_t top_k,      \
      int32_t c, int32_t sink, int32_t window, int64_t *partial, uint8_t *flags, float *agreeability,           \
      int32_t *index, int32_t *index_phys, int32_t index_capacity, int32_t *index_count, float *alpha_out,     \
      int32_t *topk_out, void *workspace, size_t workspace_bytes, int32_t *dev_status, void *stream
#define ZOOMR_SELECT_FUSED_CALL(CH)                                                                            \
  select_fused(geom, batch, q, kv, seg, close_items, n_close, update, mean_keys, top_k, c, sink, window,        \
               partial, flags, agreeability, index, index_phys, index_capacity, index_count, alpha_out,        \
               topk_out, workspace, workspace_bytes, dev_status, stream, CH)

extern "C" int zoomr_select_fused(ZOOMR_SELECT_FUSED_ARGS) { return ZOOMR_SELECT_FUSED_CALL(false); }

extern "C" int zoomr_select_fused_chained(ZOOMR_SELECT_FUSED_ARGS) { return ZOOMR_SELECT_FUSED_CALL(true); }

extern "C" int zoomr_select_front(const zoomr_geom *geom, int32_t batch, const void *q, const zoomr_kv *kv,
                                  const zoomr_segments *seg, const int32_t *close_items, int32_t n_close,
                                  const uint8_t *update, float *mean_keys, int32_t top_k, int64_t *partial,
                                  float *alpha_out, int32_t *topk_out, void *workspace, size_t workspace_bytes,
                                  int32_t *dev_status, void *stream) {
  return select_fused(geom, batch, q, kv, seg, close_items, n_close, update, mean_keys, top_k, 0, 0, 1, partial,
                      nullptr, nullptr, nullptr, nullptr, 0, nullptr, alpha_out, topk_out, workspace, workspace_bytes,
                      dev_status, stream, false, kFront);
}

extern "C" int zoomr_select_tail(const zoomr_geom *geom, int32_t batch, const zoomr_kv *kv, const zoomr_segments *seg,
                                 const int64_t *partial, const uint8_t *update, int32_t c, int32_t sink,
                                 int32_t window, uint8_t *flags, float *agreeability, int32_t *index,
                                 int32_t *index_phys, int32_t index_capacity, int32_t *index_count,
                                 int32_t *dev_status, void *stream) {
  return select_fused(geom, batch, nullptr, kv, seg, nullptr, 0, update, nullptr, 1, c, sink, window,
                      const_cast<int64_t *>(partial), flags, agreeability, index, index_phys, index_capacity,
                      index_count, nullptr, nullptr, nullptr, 0, dev_status, stream, false, kTail);
}
