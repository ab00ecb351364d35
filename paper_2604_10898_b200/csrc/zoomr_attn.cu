// a5 -- sparse GQA decode attention over the selected index set
// ("the attention mechanism will compute over the keys and values
// corresponding only to the indices in I_f"; attention equation):
//
//   o^{(l,h)} = sum_{j in I_f} softmax_j( q^{(l,h)} . k_j^{(l,h/G)} * scale ) v_j^{(l,h/G)}
//
// B200 design:
//  * Work = the flattened sequence of 32-token tiles of every (b, l, g)
//    segment.  A persistent grid (one CTA per SM) gives each math warp a
//    contiguous, equal share of that sequence ("stream-K" split): perfect load
//    balance whatever |I_f| turns out to be on the device, and at most two
//    partial results per warp.  Segments split across warps are merged by the
//    last-arriving warp (arrival counter per segment, self-resetting).
//  * Warp specialisation in producer/consumer PAIRS.  The producer warp runs a
//    5-deep address pipeline (I_f position 4 tiles ahead, page-table entry 2
//    tiles ahead) and gathers each 32-token K/V tile with TMA: the tile's
//    tokens are cut into runs of consecutive tokens in one page, each run into
//    16- and 8-row boxes loaded by cp.async.bulk.tensor (2D tensor map over the
//    whole pool, 128-byte swizzle: rows land bank-conflict-free for ldmatrix),
//    and the < 8-row leftovers (plus zero-filled rows past the end of a
//    segment) by 16-byte cp.async with the same swizzle applied by hand.  TMA
//    bytes complete on the stage's mbarrier (expect_tx), the cp.async part via
//    cp.async.mbarrier.arrive.noinc on the same barrier; the math warp frees the
//    stage with a plain arrive.  History (profiles/): v0 one TMA bulk copy per
//    256-byte row (issue-bound, 12 % of peak); v1 gather + math in one warp
//    (latency-bound, 27 %); v2/v3 LDGSTS producer (72 %, capped by the LDGSTS
//    path: tools/bench_gather.cu measures <= 5.3 TB/s); v4 this TMA gather.
//  * Math on tensor cores (mma.sync m16n8k16, bf16 in, fp32 accumulate):
//      S^T-tile = K_tile (32 tok x d) . Q^T (d x 8 padded heads)
//      O^T     += V_tile^T (d x 32 tok) . P (32 tok x 8)
//    The G query heads of the KV head share every gathered K/V tile (GQA).
//    The 8 MMA columns hold the G heads twice: P is split p = hi + lo into two
//    bf16 values (hi = bf16(p), lo = bf16(p - hi)) in the two copies, so the PV
//    product carries ~16 bits of P (bf16 alone would cost up to ~8e-3 abs,
//    SURVEY 7.3-1) at no extra MMA for G <= 4.  The S accumulator fragment is
//    transposed into the PV B-operand with movmatrix.
//  * fp32 online softmax (exp2 with scale*log2e folded in), fp32 output.
#include <cuda.h>  // CUtensorMap (the encode entry point is fetched through the runtime)
#include <mutex>
#include <unordered_map>

#include "common.cuh"

ZOOMR_TL_STORAGE(attn)

namespace zoomr {

constexpr int kTile = 32;   // tokens per tile (one per lane when resolving addresses)
constexpr int kPairs = 4;   // producer/consumer warp pairs per CTA
constexpr int kStages = 3;  // ring depth per pair
constexpr int kPtSmem = 4096; // page-table entries staged in shared memory when they fit
#ifndef ZOOMR_MERGE_STAGE
#define ZOOMR_MERGE_STAGE 1  // last-flush merges read the parts through the idle ring (A/B: -DZOOMR_MERGE_STAGE=0)
#endif

template <int D>
struct AttnShape {
  static constexpr int RB = 2 * D;                      // bytes of one K or V row (bf16)
  static constexpr bool SWZ = D >= 64;                  // 128-byte swizzled 64-column regions
  static constexpr int NREG = SWZ ? D / 64 : 1;         // regions per tile (column halves)
  static constexpr int RBR = SWZ ? 128 : RB;            // bytes of a row inside one region
  static constexpr int BX = SWZ ? 64 : D;               // TMA box inner extent (elements)
  static constexpr int REG_BYTES = kTile * RBR;         // one region of one tile
  static constexpr int TILE_BYTES = NREG * REG_BYTES;   // K (or V) part of a stage
  static constexpr int STAGE_BYTES = 2 * TILE_BYTES;
  static constexpr int RING_BYTES = kPairs * kStages * STAGE_BYTES;
  static constexpr int BAR_BYTES = (2 * kPairs * kStages + kPairs) * 8;  // full, empty, and one merge barrier per pair
  static constexpr int CPR = RB / 16;                   // 16-byte chunks per row
  static constexpr int RPI = 32 / CPR;                  // rows per warp-wide cp.async
  // shared address of (row r, 16-byte chunk c) inside a K or V tile starting at `base`
  __device__ static __forceinline__ uint32_t at(uint32_t base, int r, int c) {
    if constexpr (SWZ)
      return base + (uint32_t)((c >> 3) * REG_BYTES + r * 128 + (((c & 7) ^ (r & 7)) << 4));
    else
      return base + (uint32_t)(r * RB + (c << 4));
  }
};

struct TmaMaps {
  CUtensorMap k32, k16, k8, v32, v16, v8;  // 2D [total rows][D] views of the pools, boxes of 32 / 16 / 8 rows
};

struct AttnParams {
  const __nv_bfloat16 *q;
  const __nv_bfloat16 *kpool;
  const __nv_bfloat16 *vpool;
  int64_t num_pages;
  const int32_t *page_table;
  int32_t max_pages;
  const int32_t *index;
  const int32_t *index_phys;  // nullable: page-resolved rows written by the fused select
  const int32_t *count;
  int32_t cap;
  float *out;
  float *lse;      // nullable: natural-log partition function per (b, l, h) (token-sharded split-K)
  float *logits;   // kLogits only: s_j = q . k_j * scale per (b, l, h, index position) (H2O)
  float *ws_part;  // [2][NW + B*L*Hkv][SLOT]: partial of (phase, warp w, segment s) at [phase][w + s]
  int32_t *ws_cnt; // [B*L*Hkv]
  int32_t B, L, Hkv, P, Pshift;  // L: layers of q / out / the pools; Pshift = log2(P) when P is a power of two, else -1
  int32_t l0, Lc;                // this launch attends layers [l0, l0 + Lc) (a model's per-layer call)
  int32_t pt_smem;               // page table staged in shared memory (B*max_pages <= kPtSmem)
  int32_t early_trigger;         // chained: a PDL-launched successor may start once this CTA passed its wait
  float scale_log2;
  const int32_t *seq_len;  // nullable: with it, I_p and I_w are attended before the wait (phase A)
  int32_t sink, window;
  int32_t *status;
};

// ------------------------------------------------------------ PTX helpers --
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t *bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, int x, int64_t y, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(map), "r"(x), "r"((int)y), "r"(smem_u32(bar))
      : "memory");
}
// 1D bulk copy global -> shared (TMA), completion as tx bytes on an mbarrier
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
#ifdef ZOOMR_WATCHDOG
// experiment builds only: a spin lasting > 0.5 s writes (site, a, b) for its
// (block, warp) into host-mapped memory (zoomr_watchdog_set), readable while hung
__device__ unsigned long long *g_wd_host;  // [1024 blocks][8 warps][4]
__device__ __noinline__ void wd_fire(int site, int a, int b) {
  if (g_wd_host && blockIdx.x < 1024) {
    volatile unsigned long long *r = g_wd_host + ((size_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * 4;
    r[0] = (unsigned)site;
    r[1] = (unsigned)a;
    r[2] = (unsigned)b;
    r[3] = 1;
    __threadfence_system();
  }
}
__device__ __forceinline__ unsigned long long wd_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define WD_DECL unsigned long long wd_t0_ = 0
#define WD_TICK(site, a, b)                                                                  \
  do {                                                                                       \
    const unsigned long long wd_t_ = wd_now();                                               \
    if (!wd_t0_) wd_t0_ = wd_t_;                                                             \
    else if (wd_t_ - wd_t0_ > 500000000ull) { wd_fire(site, (int)(a), (int)(b)); wd_t0_ = wd_t_; } \
  } while (0)
#else
#define WD_DECL do { } while (0)
#define WD_TICK(site, a, b) do { } while (0)
#endif
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity, int site = 0) {
  uint32_t done;
  WD_DECL;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (!done) WD_TICK(site, parity, 0);
  } while (!done);
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t &a0, uint32_t &a1, uint32_t &a2, uint32_t &a3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t &a0, uint32_t &a1, uint32_t &a2, uint32_t &a3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
               : "r"(addr));
}
__device__ __forceinline__ uint32_t movm_t(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo_elem, float hi_elem) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo_elem, hi_elem);
  return *reinterpret_cast<uint32_t *>(&v);
}

// ----------------------------------------------------------- tile geometry --
struct Sched {
  const int32_t *prefix;  // smem [B+1]: first global tile of sequence b
  int64_t T_tot;
  int64_t NWe;  // effective number of math warps (<= T_tot)
  int32_t B, LH;  // LH = L * Hkv segments per sequence
  __device__ __forceinline__ int64_t range_start(int64_t w) const { return T_tot * w / NWe; }
  double inv_T;   // 1 / T_tot (warp_of without a 64-bit division)
  __device__ __forceinline__ int64_t warp_of(int64_t t) const {  // floor(((t + 1) * NWe - 1) / T_tot)
    const int64_t x = (t + 1) * NWe - 1;
    int64_t q = (int64_t)((double)x * inv_T);  // x < 2^53: off by at most one
    if (q * T_tot > x) --q;
    else if ((q + 1) * T_tot <= x) ++q;
    return q;
  }
  // global tile -> (b, segment within b, tile within segment, tiles per segment of b)
  __device__ __forceinline__ void locate(int64_t t, int &b, int &seg, int &tis, int &nts) const {
    int lo = 0, hi = B - 1;
    while (lo < hi) {  // last b with prefix[b] <= t
      const int mid = (lo + hi + 1) >> 1;
      if (prefix[mid] <= t) lo = mid; else hi = mid - 1;
    }
    b = lo;
    nts = (prefix[b + 1] - prefix[b]) / LH;
    const int r = (int)(t - prefix[b]);
    seg = r / nts;
    tis = r - seg * nts;
  }
};

// Two phases of work per launch.  Phase A: the rows of I_f that are known from
// T alone -- I_p = [0, s') and I_w = [w0, T), which a4 puts first and last in
// I_f (readings Q12, Q13, Q17) -- are attended BEFORE griddepcontrol.wait, so
// that part of the gather overlaps the tail of the kernel that builds I_f.
// Phase B: the middle of I_f (zoomed segments and kept summaries), positions
// [s', s' + n_B) of `index`, after the wait.  Each phase is its own stream-K
// split over all math warps; a segment's softmax partials from both phases are
// merged by the last-arriving warp.  Phase-A partials are published before the
// wait but counted (arrival atomics) only after it, when the phase-B split --
// and so the number of parts of every segment -- is known.
template <int D, int G, bool kLogits = false>
__global__ void __launch_bounds__(64 * kPairs, 1)
    sparse_attn_kernel(const AttnParams p, const __grid_constant__ TmaMaps maps) {
  using S = AttnShape<D>;
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  // the 128-byte swizzle pattern follows address bits [7:9]: keep the ring 1024-aligned
  unsigned char *smem = smem_dyn + ((1024 - (smem_u32(smem_dyn) & 1023)) & 1023);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + S::RING_BYTES);  // [kPairs][kStages]
  uint64_t *empty = full + kPairs * kStages;                             // [kPairs][kStages]
  uint64_t *bready = reinterpret_cast<uint64_t *>(smem + S::RING_BYTES + S::BAR_BYTES);  // phase-B schedule published
  int4 *info = reinterpret_cast<int4 *>(bready + 2);  // [B]: a1, T - a2, n_A, n_B
  int32_t *pts = reinterpret_cast<int32_t *>(info + p.B);  // [kPtSmem] page tables
  int32_t *prefA = pts + (p.pt_smem ? kPtSmem : 0);        // [B+1] first phase-A tile of sequence b
  int32_t *prefB = prefA + p.B + 1;                        // [B+1] first phase-B tile
  int32_t *bstate = prefB + p.B + 1;                       // phase-B schedule: 0 unclaimed, 1 claimed
  // warp index through a shuffle: ptxas then treats it (and the pair's ring and
  // barriers) as warp-uniform, which keeps the TMA issue's operands in uniform registers
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int Hq = p.Hkv * G;
  const int LH = p.Lc * p.Hkv;  // segments (b, layer in [l0, l0 + Lc), KV head) per sequence
  TL_INIT();
  if (threadIdx.x == 0) {
    TL(0);
    TL_CTA(1);
  }

  if (S::SWZ && threadIdx.x < 6) {  // the tensor maps' descriptors, fetched while the prologue runs
    const CUtensorMap *m = &maps.k32 + threadIdx.x;
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
  }
  if (threadIdx.x == 0) {
    for (int x = 0; x < kPairs * kStages; ++x) {
      mbar_init(&full[x], 33);  // producer lane 0's expect_tx arrive + one cp.async (noinc) arrive per lane
      mbar_init(&empty[x], 1);  // the math warp's lane 0
    }
    for (int x = 0; x < kPairs; ++x) mbar_init(&empty[kPairs * kStages + x], 1);  // merge staging (lane 0's expect_tx)
    *bstate = 0;
    mbar_init(bready, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // Page tables, T, q and the pools are inputs, not outputs of the preceding
  // kernel (a4 / the fused select): read them while that kernel is finishing.
  if (p.pt_smem)
    for (int x = threadIdx.x; x < p.B * p.max_pages; x += blockDim.x) pts[x] = p.page_table[x];
  if (warp == 0) {  // phase-A tiles per sequence -> prefix (chunks of 32 sequences)
    int carry = 0;
    for (int b0 = 0; b0 < p.B; b0 += 32) {
      const int b = b0 + lane;
      int n = 0;
      if (b < p.B) {
        // phase A = the first a1 and the last a2 entries of I_f: the sink and the
        // newest window rows, n_A = a1 + a2 rounded DOWN to whole tiles (the
        // window rows left over join phase B, whose index positions stay
        // contiguous: [a1, |I_f| - a2)), so neither phase adds a ragged tile
        int a1 = 0, a2 = 0;
        if (p.seq_len) {
          const int T = max(p.seq_len[b], 0);
          const int sp = min(p.sink, T);
          const int w0 = max(sp, T - p.window);
          const int na = (sp + (T - w0)) / kTile * kTile;
          a1 = min(sp, na);
          a2 = na - a1;
          info[b] = make_int4(a1, T - a2, na, 0);
        } else {
          info[b] = make_int4(0, 0, 0, 0);
        }
        const int na = a1 + a2;
        n = na > 0 ? (na + kTile - 1) / kTile * LH : 0;
      }
      int incl = n;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (b < p.B) prefA[b] = carry + incl - n;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) prefA[p.B] = carry;
  }
  __syncthreads();

  if (threadIdx.x == 0) TL(1);
  const int64_t NW = (int64_t)gridDim.x * kPairs;
  const int pair = warp % kPairs;
  const bool producer = warp >= kPairs;
  const int64_t gw = (int64_t)blockIdx.x * kPairs + pair;  // global math-warp id of the pair
  Sched sA, sB;
  sA.prefix = prefA;
  sA.T_tot = prefA[p.B];
  sA.NWe = NW < sA.T_tot ? NW : sA.T_tot;
  sA.inv_T = sA.T_tot > 0 ? 1.0 / (double)sA.T_tot : 0.0;
  sA.B = sB.B = p.B;
  sA.LH = sB.LH = LH;
  sB.prefix = prefB;
  sB.T_tot = 0;
  sB.NWe = 0;
  int64_t a0 = 0, nAk = 0, b0r = 0, nBk = 0;  // this warp's tiles: [a0, a0+nAk) of A, [b0r, b0r+nBk) of B
  if (gw < sA.NWe) {
    a0 = sA.range_start(gw);
    nAk = sA.range_start(gw + 1) - a0;
  }
  bool bres = false;  // phase-B schedule known (implies griddepcontrol.wait done)
  // Programmatic dependent launch: after the wait the producer of I_f has
  // completed and its writes are visible.  The first warp to get here derives
  // n_B and the phase-B prefix for the CTA; the others wait for it.
  auto resolve_b = [&]() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    int st = 0;
    if (lane == 0) st = atomicCAS(bstate, 0, 1);
    st = __shfl_sync(0xffffffffu, st, 0);
    if (st == 0) {
      int carry = 0;
      for (int c0 = 0; c0 < p.B; c0 += 32) {
        const int b = c0 + lane;
        int n = 0;
        if (b < p.B) {
          int c = p.count[b];
          c = c < p.cap ? c : p.cap;
          const int nb = max(0, c - info[b].z);
          info[b].w = nb;
          n = nb > 0 ? (nb + kTile - 1) / kTile * LH : 0;
        }
        int incl = n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        if (b < p.B) prefB[b] = carry + incl - n;
        carry += __shfl_sync(0xffffffffu, incl, 31);
      }
      if (lane == 0) prefB[p.B] = carry;
      __syncwarp();
      if (lane == 0) mbar_arrive(bready);  // release: the schedule above is visible to the waiters
      // Chained: the successor (normally the next step's fused select) may launch
      // once every CTA got here, i.e. after griddepcontrol.wait -- so after this
      // launch's own predecessor (the select writing I_f, and the select's
      // workspace) has completed.  Triggering any earlier would let select(t+1)
      // touch the shared selection workspace while select(t) still runs.
      if (p.early_trigger) allow_dependents();
    } else {
      mbar_wait(bready, 0, 7);  // acquire (suspends instead of hammering shared memory)
    }
    __syncwarp();
    sB.T_tot = prefB[p.B];
    sB.NWe = NW < sB.T_tot ? NW : sB.T_tot;
    sB.inv_T = sB.T_tot > 0 ? 1.0 / (double)sB.T_tot : 0.0;
    if (gw < sB.NWe) {
      b0r = sB.range_start(gw);
      nBk = sB.range_start(gw + 1) - b0r;
    }
    bres = true;
    TL(2);
  };
  // k-th tile of this warp's list (A tiles, then B tiles) -> (phase, b, segment,
  // tile in segment).  Tiles are visited in order, so the walk advances
  // incrementally; it searches the prefix only at its start and at the phase switch.
  struct Walk {
    int ph = -1, b = 0, seg = 0, tis = 0, nts = 0;
    int64_t k = -2;
  };
  auto where = [&](Walk &w, int64_t k) {
    const int ph = k < nAk ? 0 : 1;
    if (ph == w.ph && k == w.k + 1) {
      w.k = k;
      if (++w.tis < w.nts) return;
      w.tis = 0;
      if (++w.seg < LH) return;
      w.seg = 0;
      const int32_t *pf = ph ? prefB : prefA;
      do {
        ++w.b;
      } while (w.b < p.B - 1 && pf[w.b + 1] == pf[w.b]);  // sequences without tiles in this phase
      w.nts = (pf[w.b + 1] - pf[w.b]) / LH;
      return;
    }
    w.ph = ph;
    w.k = k;
    if (ph == 0) sA.locate(a0 + k, w.b, w.seg, w.tis, w.nts);
    else sB.locate(b0r + (k - nAk), w.b, w.seg, w.tis, w.nts);
  };
  const uint32_t ring = smem_u32(smem) + (uint32_t)(pair * kStages * S::STAGE_BYTES);
  uint64_t *fullp = full + pair * kStages;
  uint64_t *emptyp = empty + pair * kStages;

  if (producer) {
    // ================= producer: address pipeline + TMA / cp.async copies =====
    TL(8);
#ifdef ZOOMR_TL_RAMP
    TLW_SET(gw, 4, clock64());
#endif
    // A(k+4): I_f position   B(k+2): page-table entry   C(k): row copies.
    // Each dependent load is consumed two iterations after it is issued, so the
    // index -> page -> row chain never stalls the copy issue in steady state.
    struct Addr {
      int ph, b, l, g, ok, tok, slot, page;
    };
    Walk wk;
    auto stage_a = [&](int64_t k, Addr &a) {
      where(wk, k);
      a.ph = wk.ph;
      a.b = wk.b;
      const int seg = wk.seg, tis = wk.tis;
      const int4 in = info[a.b];
      const int sl = seg / p.Hkv;
      a.l = p.l0 + sl;
      a.g = seg - sl * p.Hkv;
      const int pos = tis * kTile + lane;
      if (a.ph == 0) {  // [0, s') ++ [w0, T)
        a.ok = pos < in.z;
        a.tok = pos < in.x ? pos : in.y + (pos - in.x);
      } else {
        a.ok = pos < in.w;
        // with index_phys, `tok` carries the page-resolved row and stage B is a no-op;
        // the load is guarded by the capacity, not the count, so it does not wait for it
        const int ip = in.x + pos;
        const int32_t *src = p.index_phys ? p.index_phys : p.index;
        a.tok = ip < p.cap ? src[(int64_t)a.b * p.cap + ip] : 0;
      }
    };
    auto stage_b = [&](Addr &a) {
      a.page = 0;
      a.slot = 0;
      if (a.ok && !(a.ph && p.index_phys)) {
        const int lp = p.Pshift >= 0 ? (a.tok >> p.Pshift) : a.tok / p.P;
        a.slot = a.tok - lp * p.P;
        if (a.tok >= 0 && lp < p.max_pages)
          a.page = p.pt_smem ? pts[a.b * p.max_pages + lp] : p.page_table[(int64_t)a.b * p.max_pages + lp];
        else a.page = -1;
      }
    };
    // pipeline depth: the I_f load runs kAheadA tiles ahead, the page-table load
    // kAheadB tiles ahead of the copies
    constexpr int kAheadA = 4, kAheadB = 2;
    Addr q0{}, q1{}, q2{}, q3{}, q4{};  // tiles k .. k+4
    int64_t ntiles = nAk;
    int64_t kfill = 0;  // first tile of the current pass: stage C is skipped below it (pipeline fill)
    // one loop, one call site per stage (the pipeline fill is its first kAheadA
    // iterations): the kernel's code stays small enough for the instruction cache.
    // Phase A's tiles are all issued BEFORE griddepcontrol.wait: the address
    // pipeline stops at the phase boundary, and only when every phase-A copy is
    // in flight does the producer wait for I_f (the ring still holds up to
    // kStages phase-A tiles for its math warp, which cover the refill of the
    // pipeline for phase B).  Waiting as soon as the first phase-B tile entered
    // the pipeline (kAheadA tiles early) stalled the phase-A stream for the
    // whole select tail.
    for (int64_t k = -kAheadA;; ++k) {
#ifdef ZOOMR_AB_OLD_WAIT  // A/B builds only: wait as soon as the first phase-B tile enters the pipeline
      if (!bres && k + kAheadA >= nAk) {
        resolve_b();
        ntiles = nAk + nBk;
      }
#endif
      if (!bres && k >= nAk) {  // every phase-A tile issued: wait for I_f, then refill for phase B
        resolve_b();
        ntiles = nAk + nBk;
        if (k >= ntiles) break;
        k = nAk - kAheadA;
        kfill = nAk;
      }
      if (k >= ntiles) break;
      if (k + kAheadA < ntiles) stage_a(k + kAheadA, q4);
      if (k == -kAheadA) {
        TL(9);
#ifdef ZOOMR_TL_RAMP
        TLW_SET(gw, 5, clock64());
#endif
      }
      if (k + kAheadB >= kfill && k + kAheadB < ntiles) stage_b(q2);
      if (k < kfill) {
        q0 = q1;
        q1 = q2;
        q2 = q3;
        q3 = q4;
        continue;
      }
      Addr &ac = q0;
      // stage C: global row of every token of tile k
      const int cok = ac.ok;
      const bool usephys = ac.ph && p.index_phys;
      int64_t grow = 0;
      int page = ac.page;
      if (usephys) {
        // row(l, g, t) = (l*num_pages*H_kv + g)*P + phys(t); consecutive phys = contiguous rows
        int phys = ac.tok;
        if (cok && (phys < 0 || (int64_t)phys >= p.num_pages * p.Hkv * p.P)) {
          set_status(p.status, ZOOMR_ERR_INDEX_RANGE);
          phys = 0;
        }
        if (cok) grow = ((int64_t)ac.l * p.num_pages * p.Hkv + ac.g) * p.P + phys;
      } else {
        if (cok && (page < 0 || page >= p.num_pages)) {
          set_status(p.status, ZOOMR_ERR_INDEX_RANGE);
          page = 0;
        }
        if (cok) grow = (((int64_t)ac.l * p.num_pages + page) * p.Hkv + ac.g) * p.P + ac.slot;
      }
      // runs of consecutive tokens in one page -> boxes of 16 / 8 rows; the rest by cp.async.
      // (A table of 16/8/4/2/1-row boxes without cp.async measured 1-2 us slower per launch.)
      const int ptok = __shfl_up_sync(0xffffffffu, ac.tok, 1);
      const int ppage = __shfl_up_sync(0xffffffffu, page, 1);
      const int pok = __shfl_up_sync(0xffffffffu, cok, 1);
      const bool cont = cok && lane > 0 && pok && ptok + 1 == ac.tok && (usephys || ppage == page);
      const unsigned validm = __ballot_sync(0xffffffffu, cok);
      const unsigned startm = __ballot_sync(0xffffffffu, cok && !cont);
      const unsigned upto = lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
      const int rs = 31 - __clz(startm & upto | 1u);               // my run's first slot
      const unsigned after = (startm | ~validm) & ~upto;
      const int re = after ? __ffs(after) - 1 : 32;                // one past my run's last slot
      const int pos = lane - rs, len = re - rs;
      const int n16 = (len >> 4) << 4, n8 = ((len & 15) >> 3) << 3;
      // TMA boxes need 128-byte aligned destinations: d >= 64 only (d < 64 configs are toy-sized)
      // a whole tile that is one run (a window or zoomed stretch inside one page): one 32-row box
      const bool whole = S::SWZ && len == 32;
      const bool lead32 = whole && cok && pos == 0;
      const bool lead16 = S::SWZ && !whole && cok && pos < n16 && (pos & 15) == 0;
      const bool lead8 = S::SWZ && !whole && cok && n8 && pos == n16;
      // the last len % 8 rows of a run of >= 8: one more 8-row box ending at the run's
      // end, overlapping the previous box (the overlapped rows are written twice with
      // the same bytes); only runs shorter than 8 rows go through cp.async
#ifdef ZOOMR_AB_TAILBOX  // A/B builds only: one more 8-row box ending at the run's end, overlapping the
      // previous box, instead of len % 8 rows by cp.async (index-only a5 -0.6 us at 8B-16K, but the step
      // +0.5 us there and +8..23 us at configs[4] L_R = 1024, c = 32: kept out)
      const bool leadT = S::SWZ && !whole && cok && len >= 8 && (len & 7) && pos == len - 8;
      const bool byhand = !cok || !S::SWZ || (len < 8 && pos >= n16 + n8);
#else
      const bool leadT = false;
      const bool byhand = !cok || !S::SWZ || pos >= n16 + n8;
#endif
      const unsigned m16 = __ballot_sync(0xffffffffu, lead16), m8 = __ballot_sync(0xffffffffu, lead8 || leadT);
      const uint32_t tx = (uint32_t)((__ballot_sync(0xffffffffu, lead32) ? 32 : 0) * S::RB * 2 +
                                     (__popc(m16) * 16 + __popc(m8) * 8) * S::RB * 2);
      const int s = (int)(k % kStages);
      mbar_wait(&emptyp[s], (uint32_t)(((k / kStages) & 1) ^ 1), 6000000 + (int)k);
      const uint32_t stK = ring + (uint32_t)(s * S::STAGE_BYTES);
      const uint32_t stV = stK + S::TILE_BYTES;
      if (k == 0) {
        TL(7);
#ifdef ZOOMR_TL_RAMP
        TLW_SET(gw, 3, clock64());
#endif
      }
      if (lane == 0) mbar_arrive_expect_tx(&fullp[s], tx);
      __syncwarp();
      // one issue block per box height: the tensor map (like the barrier and the
      // stage) is warp-uniform, so only the row and the destination vary per lane
      if (lead32) {
#pragma unroll
        for (int rg = 0; rg < S::NREG; ++rg) {
          const uint32_t off = (uint32_t)(rg * S::REG_BYTES);
          tma_load_2d(stK + off, &maps.k32, rg * S::BX, grow, &fullp[s]);
          tma_load_2d(stV + off, &maps.v32, rg * S::BX, grow, &fullp[s]);
        }
      }
      if (lead16) {
#pragma unroll
        for (int rg = 0; rg < S::NREG; ++rg) {
          // destination = the row's unswizzled start; the TMA unit applies the 128-byte swizzle
          const uint32_t off = (uint32_t)(rg * S::REG_BYTES + lane * S::RBR);
          tma_load_2d(stK + off, &maps.k16, rg * S::BX, grow, &fullp[s]);
          tma_load_2d(stV + off, &maps.v16, rg * S::BX, grow, &fullp[s]);
        }
      }
      if (lead8 || leadT) {
#pragma unroll
        for (int rg = 0; rg < S::NREG; ++rg) {
          const uint32_t off = (uint32_t)(rg * S::REG_BYTES + lane * S::RBR);
          tma_load_2d(stK + off, &maps.k8, rg * S::BX, grow, &fullp[s]);
          tma_load_2d(stV + off, &maps.v8, rg * S::BX, grow, &fullp[s]);
        }
      }
      // leftover rows (and zero rows past the end): 16-byte cp.async, swizzle by hand
      unsigned mh = __ballot_sync(0xffffffffu, byhand);
      const __nv_bfloat16 *krow = p.kpool + grow * D, *vrow = p.vpool + grow * D;
      const int rsub = lane / S::CPR, ch = lane % S::CPR;
      while (mh) {
        int r = -1;
        unsigned take = mh;
#pragma unroll
        for (int u = 0; u < S::RPI; ++u) {  // the u-th pending row goes to lanes [u*CPR, (u+1)*CPR)
          const int rr = take ? __ffs(take) - 1 : -1;
          if (u == rsub) r = rr;
          if (take) take &= take - 1;
        }
        mh = take;
        const int rsrc = r < 0 ? 0 : r;
        const __nv_bfloat16 *kr = (const __nv_bfloat16 *)__shfl_sync(0xffffffffu, (unsigned long long)krow, rsrc);
        const __nv_bfloat16 *vr = (const __nv_bfloat16 *)__shfl_sync(0xffffffffu, (unsigned long long)vrow, rsrc);
        const int rok = __shfl_sync(0xffffffffu, cok, rsrc);
        if (r >= 0) {
          const uint32_t n = rok ? 16u : 0u;  // 0: zero-fill
          cp_async16(S::at(stK, r, ch), kr + ch * 8, n);
          cp_async16(S::at(stV, r, ch), vr + ch * 8, n);
        }
      }
      cp_async_arrive_noinc(&fullp[s]);
#ifdef ZOOMR_AB_PROD_DELAY  // A/B builds only: does the producer pace the stream? (it does not)
      __nanosleep(ZOOMR_AB_PROD_DELAY);
#endif
      if (k == ntiles - 1) {
        TL(6);
        TLW_SET(gw, 6, TL_NOW());
      }
#if defined(ZOOMR_TIMELINE) && !defined(ZOOMR_TL_RAMP)
      const unsigned tl_cp = __ballot_sync(0xffffffffu, byhand && cok);
      TLW_ADD(gw, 4, __popc(tl_cp));
      TLW_ADD(gw, 5, __popc(m16) + __popc(m8));
#endif
      q0 = q1;
      q1 = q2;
      q2 = q3;
      q3 = q4;
    }
    return;
  }

  // ====================== math warp: tensor-core flash-decode ==============
  const int gq = lane >> 2, tq = lane & 3;  // mma fragment row group / thread-in-group
  const int n0 = 2 * tq;                    // the two MMA columns this thread holds: n0, n0+1
  constexpr int NKS = D / 16;               // k-steps of QK^T and m-tiles of O^T
  constexpr bool kTwoN = (G > 4);           // hi and lo in separate n-tiles (G = 7: column 7 is padding)
  // column -> (head, part) for G <= 4: head = n % G, part = n / G (0 hi, 1 lo, >=2 none)
  const int part0 = kTwoN ? 0 : n0 / G, part1 = kTwoN ? 0 : (n0 + 1) / G;
  constexpr int HDR = (2 * G + 3) / 4 * 4;  // m[G], l[G] padded to a 16-byte boundary
  constexpr int SLOT = HDR + G * D;         // partial result: header, then O[G][D]

  int cur_ph = -2, cur_b = -1, cur_seg = -1;  // -2: no segment yet (never equal to a past-the-end k)
  uint64_t *mrgbar = empty + kPairs * kStages + pair;  // this pair's merge-staging barrier
  uint32_t mrgphase = 0;
  int npend = 0;  // phase-A partials published before the wait, not yet counted: the first npend segments of the A range
  uint32_t qf[NKS][2];
  float o[NKS][4], o2[kTwoN ? NKS : 1][4];
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  // parts of segment (b, seg): A warps [wf0, wf0 + n0w), B warps [wf1, wf1 + n1w) (needs bres)
  auto seg_parts = [&](int b, int seg, int64_t &wf0, int &n0w, int64_t &wf1, int &n1w) {
    n0w = n1w = 0;
    wf0 = wf1 = 0;
    const int na = (prefA[b + 1] - prefA[b]) / LH;
    if (na > 0) {
      const int64_t st0 = prefA[b] + (int64_t)seg * na;
      wf0 = sA.warp_of(st0);
      n0w = (int)(sA.warp_of(st0 + na - 1) - wf0 + 1);
    }
    const int nb = (prefB[b + 1] - prefB[b]) / LH;
    if (nb > 0) {
      const int64_t st0 = prefB[b] + (int64_t)seg * nb;
      wf1 = sB.warp_of(st0);
      n1w = (int)(sB.warp_of(st0 + nb - 1) - wf1 + 1);
    }
  };
  // Partial-result slot of (phase, warp w, segment s): the (w, s) pairs a
  // stream-K split produces form a staircase on which w + s strictly increases,
  // so w + s (< NW + #segments) is a unique slot per phase.
  const int64_t nslots = NW + (int64_t)p.B * LH;
  auto part_slot = [&](int ph, int64_t w, int b, int seg) -> int64_t {
    return ph * nslots + w + (int64_t)b * LH + seg;
  };
  // where part j of segment (b, seg) lives
  auto part_ptr = [&](int b, int seg, int j, int64_t wf0, int n0w, int64_t wf1) -> const float * {
    const int ph = j < n0w ? 0 : 1;
    const int64_t w = ph ? wf1 + (j - n0w) : wf0 + j;
    return p.ws_part + part_slot(ph, w, b, seg) * SLOT;
  };

  auto flush = [&](int ph, int b, int seg, bool at_end) {
#ifndef ZOOMR_TL_RAMP
    TLW_ADD(gw, 7, 1);
#endif
    // At the warp's last flush: if every other part of the segment has already
    // arrived, this part is the last one -- merge right away, with this part
    // taken from shared memory, instead of publishing it, fencing and counting
    // (the counter is read now; its latency hides behind the reductions below).
    unsigned cnt_seen = 0xffffffffu;
    if (at_end && bres && npend == 0 && lane == 0)
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cnt_seen)
                   : "l"(p.ws_cnt + (int64_t)b * LH + seg) : "memory");
    // finish the segment's softmax state and publish it (final or partial)
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      l0 += __shfl_xor_sync(0xffffffffu, l0, off);
      l1 += __shfl_xor_sync(0xffffffffu, l1, off);
    }
    float ov[NKS][4];
#pragma unroll
    for (int me = 0; me < NKS; ++me)
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        float v = o[me][x];
        if constexpr (kTwoN) v += o2[me][x];
        else if constexpr (G == 4) v += __shfl_xor_sync(0xffffffffu, v, 2);
        else if constexpr (G == 2) v += __shfl_xor_sync(0xffffffffu, v, 1);
        ov[me][x] = v;
      }
    if constexpr (G == 1) {
#pragma unroll
      for (int me = 0; me < NKS; ++me) {
        ov[me][0] += ov[me][1];
        ov[me][2] += ov[me][3];
      }
    }
    // owners: threads whose columns are the hi copies of real heads
    const bool owner = kTwoN || (G == 4 && tq < 2) || (G <= 2 && tq == 0);
    // heads held by an owner thread: n0 (and n0 + 1 when it is a real head)
    const int nh = (G == 1) ? 1 : (kTwoN && n0 + 1 >= G) ? 1 : 2;
    int64_t wf0, wf1;
    int n0w, n1w;
    bool final_out = false;
    if (bres) {
      seg_parts(b, seg, wf0, n0w, wf1, n1w);
      final_out = n0w + n1w == 1;
      if (final_out) {  // this warp is the segment's only part: final output
        const int sl = seg / p.Hkv, g = seg - sl * p.Hkv, l = p.l0 + sl;
        float *ob = p.out + (((int64_t)b * p.L + l) * Hq + (int64_t)g * G) * D;
        if (owner) {
          const float inv0 = 1.f / l0, inv1 = 1.f / l1;
#pragma unroll
          for (int me = 0; me < NKS; ++me) {
            const int e = me * 16 + gq;
            ob[(int64_t)n0 * D + e] = ov[me][0] * inv0;
            ob[(int64_t)n0 * D + e + 8] = ov[me][2] * inv0;
            if (nh == 2) {
              ob[(int64_t)(n0 + 1) * D + e] = ov[me][1] * inv1;
              ob[(int64_t)(n0 + 1) * D + e + 8] = ov[me][3] * inv1;
            }
          }
          if (p.lse && gq == 0) {  // ln sum_j exp(s_j) = (m + log2 l) * ln 2 (scores are in the log2 domain)
            float *lb = p.lse + ((int64_t)b * p.L + l) * Hq + (int64_t)g * G;
            lb[n0] = (m0 + log2f(l0)) * 0.6931471805599453f;
            if (nh == 2) lb[n0 + 1] = (m1 + log2f(l1)) * 0.6931471805599453f;
          }
        }
        if (npend == 0) return;  // else: still count the pending phase-A partials below
      }
    }
    cnt_seen = __shfl_sync(0xffffffffu, cnt_seen, 0);
    const bool shortcut = !final_out && bres && cnt_seen == (unsigned)(n0w + n1w - 1);
    // the pair's ring is idle at its last flush: stage 0 holds this part for the merge
    float *own = reinterpret_cast<float *>(smem + pair * kStages * S::STAGE_BYTES);
    if (!final_out) {  // partial (published, or kept in shared memory for the shortcut)
      float *ps = shortcut ? own : p.ws_part + part_slot(ph, gw, b, seg) * SLOT;
      if (owner) {
        if (gq == 0) {
          ps[n0] = m0;
          ps[G + n0] = l0;
          if (nh == 2) {
            ps[n0 + 1] = m1;
            ps[G + n0 + 1] = l1;
          }
        }
#pragma unroll
        for (int me = 0; me < NKS; ++me) {
          const int e = me * 16 + gq;
          ps[HDR + n0 * D + e] = ov[me][0];
          ps[HDR + n0 * D + e + 8] = ov[me][2];
          if (nh == 2) {
            ps[HDR + (n0 + 1) * D + e] = ov[me][1];
            ps[HDR + (n0 + 1) * D + e + 8] = ov[me][3];
          }
        }
      }
      __syncwarp();  // orders the lanes' partial stores before lane 0's release
      if (ZOOMR_MERGE_STAGE && lane == 0) asm volatile("fence.proxy.async.global;" ::: "memory");  // read by TMA later
    }
    if (!bres) {  // phase A before the wait: count it later
      ++npend;
      return;
    }
    // count the pending phase-A partials (segments of the A range in order), then
    // this one; the last arriving part of a segment merges all of its parts
    int64_t t = a0;
    const int npa = npend, narr = npend + (final_out ? 0 : 1);  // pending phase-A partials first, then this one
    npend = 0;
    for (int it = 0; it < narr; ++it) {
      int xb = b, xs = seg;
      if (it < npa) {
        int xt, xn;
        sA.locate(t, xb, xs, xt, xn);
        t += xn - xt;  // first tile of the next segment
      }
      seg_parts(xb, xs, wf0, n0w, wf1, n1w);
      const int nparts = n0w + n1w;
      int32_t *cnt = p.ws_cnt + (int64_t)xb * LH + xs;
      int own_j = -1;  // index of this warp's part when it is merged from shared memory
      if (shortcut && it == narr - 1) {
        own_j = ph ? n0w + (int)(gw - wf1) : (int)(gw - wf0);
      } else {
        int old = 0;
        if (lane == 0)
          asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
        old = __shfl_sync(0xffffffffu, old, 0);
        if (old != nparts - 1) continue;  // not the last arriving part
      }
      const unsigned long long tl_m0 = TL_NOW();
      __syncwarp();  // the other lanes' partial loads below are ordered after lane 0's acquire
      // last arriver: online merge of the parts in a fixed order (deterministic),
      // NPF parts per round with all their loads in flight
      const int xsl = xs / p.Hkv, xg = xs - xsl * p.Hkv, xl = p.l0 + xsl;
      float *ob = p.out + (((int64_t)xb * p.L + xl) * Hq + (int64_t)xg * G) * D;
      constexpr int NV4 = G * D / 4;
      constexpr int PER = (NV4 + 31) / 32;
      constexpr int NPF = G > 4 ? 2 : 4;
      float Mh[G], Lh[G];
      float4 acc[PER];
#pragma unroll
      for (int h = 0; h < G; ++h) {
        Mh[h] = -INFINITY;
        Lh[h] = 0.f;
      }
#pragma unroll
      for (int u = 0; u < PER; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      // At the warp's last flush the pair's ring is idle: stage every other part
      // into it (after this warp's own part) with all copies in flight at once --
      // one L2 round trip for the whole merge instead of one per NPF parts.
      float *stg = own + SLOT;
      const bool staged = ZOOMR_MERGE_STAGE && at_end && (nparts + 1) * SLOT * 4 <= kStages * S::STAGE_BYTES;
      if (staged) {
        // one 1D TMA bulk copy per part (lane j copies part j): a few instructions
        // instead of SLOT/4 16-byte cp.async per part (for G = 8, 8 parts were
        // ~2300 issues from one warp, ~7 us at the end of the kernel)
        __syncwarp();  // a previous merge's shared-memory reads are done
        const uint32_t nbytes = (uint32_t)((nparts - (own_j >= 0 ? 1 : 0)) * SLOT * 4);
        if (lane == 0) {
          asm volatile("fence.proxy.async.global;" ::: "memory");      // the parts were written by generic stores
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the staging area was read generically
          mbar_arrive_expect_tx(mrgbar, nbytes);
        }
        __syncwarp();
        for (int j = lane; j < nparts; j += 32) {
          if (j == own_j) continue;
          bulk_g2s(smem_u32(stg + j * SLOT), part_ptr(xb, xs, j, wf0, n0w, wf1), (uint32_t)(SLOT * 4), mrgbar);
        }
        mbar_wait(mrgbar, mrgphase, 8);
        mrgphase ^= 1u;
      }
      for (int j0 = 0; j0 < nparts; j0 += NPF) {
        float mh[NPF][G], lh[NPF][G];
        float4 ov4[NPF][PER];
#pragma unroll
        for (int j = 0; j < NPF; ++j) {
          if (j0 + j == own_j) {  // this warp's part, in shared memory
#pragma unroll
            for (int h = 0; h < G; ++h) {
              mh[j][h] = own[h];
              lh[j][h] = own[G + h];
            }
#pragma unroll
            for (int u = 0; u < PER; ++u) {
              const int f = lane + 32 * u;
              ov4[j][u] = f < NV4 ? reinterpret_cast<const float4 *>(own + HDR)[f] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
          } else if (j0 + j < nparts && staged) {  // staged in shared memory
            const float *qp = stg + (j0 + j) * SLOT;
#pragma unroll
            for (int h = 0; h < G; ++h) {
              mh[j][h] = qp[h];
              lh[j][h] = qp[G + h];
            }
#pragma unroll
            for (int u = 0; u < PER; ++u) {
              const int f = lane + 32 * u;
              ov4[j][u] = f < NV4 ? reinterpret_cast<const float4 *>(qp + HDR)[f] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
          } else if (j0 + j < nparts) {
            const float *qp = part_ptr(xb, xs, j0 + j, wf0, n0w, wf1);
#pragma unroll
            for (int h = 0; h < G; ++h) {
              mh[j][h] = __ldcg(qp + h);
              lh[j][h] = __ldcg(qp + G + h);
            }
#pragma unroll
            for (int u = 0; u < PER; ++u) {
              const int f = lane + 32 * u;
              ov4[j][u] = f < NV4 ? __ldcg(reinterpret_cast<const float4 *>(qp + HDR) + f)
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
            }
          } else {
#pragma unroll
            for (int h = 0; h < G; ++h) {
              mh[j][h] = -INFINITY;
              lh[j][h] = 0.f;
            }
#pragma unroll
            for (int u = 0; u < PER; ++u) ov4[j][u] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
        float w[NPF][G], so[G];
#pragma unroll
        for (int h = 0; h < G; ++h) {
          float mn = Mh[h];
#pragma unroll
          for (int j = 0; j < NPF; ++j) mn = fmaxf(mn, mh[j][h]);
          so[h] = ex2(Mh[h] - mn);  // -inf -> 0 on the first round
          Lh[h] *= so[h];
#pragma unroll
          for (int j = 0; j < NPF; ++j) {
            w[j][h] = ex2(mh[j][h] - mn);
            Lh[h] += lh[j][h] * w[j][h];
          }
          Mh[h] = mn;
        }
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int h = (4 * (lane + 32 * u)) / D < G ? (4 * (lane + 32 * u)) / D : G - 1;
          float4 a = acc[u];
          a.x *= so[h];
          a.y *= so[h];
          a.z *= so[h];
          a.w *= so[h];
#pragma unroll
          for (int j = 0; j < NPF; ++j) {
            a.x += ov4[j][u].x * w[j][h];
            a.y += ov4[j][u].y * w[j][h];
            a.z += ov4[j][u].z * w[j][h];
            a.w += ov4[j][u].w * w[j][h];
          }
          acc[u] = a;
        }
      }
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const int f = lane + 32 * u;
        if (f < NV4) {
          const float inv = 1.f / Lh[(4 * f) / D];
          reinterpret_cast<float4 *>(ob)[f] =
              make_float4(acc[u].x * inv, acc[u].y * inv, acc[u].z * inv, acc[u].w * inv);
        }
      }
      if (p.lse && lane == 0) {
        float *lb = p.lse + ((int64_t)xb * p.L + xl) * Hq + (int64_t)xg * G;
#pragma unroll
        for (int h = 0; h < G; ++h) lb[h] = (Mh[h] + log2f(Lh[h])) * 0.6931471805599453f;
      }
      if (lane == 0) *cnt = 0;  // leave the workspace zeroed for the next call
      TLW_ADD(gw, 2, 1);
#ifndef ZOOMR_TL_RAMP
      TLW_ADD(gw, 3, TL_NOW() - tl_m0);
#endif
    }
  };

  Walk wk;
  int64_t ntot = nAk;
  for (int64_t k = 0;; ++k) {  // the iteration past the last tile only flushes
    if (!bres && k >= nAk) {
      resolve_b();
      ntot = nAk + nBk;
    }
    int ph = -1, b = -1, seg = -1, tis = 0;
    if (k < ntot) {
      where(wk, k);
      ph = wk.ph;
      b = wk.b;
      seg = wk.seg;
      tis = wk.tis;
    }
    if (ph != cur_ph || b != cur_b || seg != cur_seg) {
      if (cur_b >= 0) flush(cur_ph, cur_b, cur_seg, k >= ntot);
      if (k >= ntot) {
        TL(5);
        TL_CTA(2);
        TLW_SET(gw, 0, TL_NOW());
        TLW_SET(gw, 1, ntot);
        break;
      }
      cur_ph = ph;
      cur_b = b;
      cur_seg = seg;
      // Q fragments (B operand of QK^T): Q[head n % G][k-chunk], this thread's column n = gq
      const int sl = seg / p.Hkv, g = seg - sl * p.Hkv, l = p.l0 + sl;
      const __nv_bfloat16 *qh = p.q + (((int64_t)b * p.L + l) * Hq + (int64_t)g * G + (gq % G)) * D;
#pragma unroll
      for (int ks = 0; ks < NKS; ++ks) {
        qf[ks][0] = *reinterpret_cast<const uint32_t *>(qh + ks * 16 + 2 * tq);
        qf[ks][1] = *reinterpret_cast<const uint32_t *>(qh + ks * 16 + 8 + 2 * tq);
      }
#pragma unroll
      for (int me = 0; me < NKS; ++me)
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          o[me][x] = 0.f;
          if constexpr (kTwoN) o2[me][x] = 0.f;
        }
      m0 = m1 = -INFINITY;
      l0 = l1 = 0.f;
    }
    const int4 in = info[b];
    const int cnt = ph ? in.w : in.z;
    const int nvalid = min(kTile, cnt - tis * kTile);
    const int s = (int)(k % kStages);
    mbar_wait(&fullp[s], (uint32_t)((k / kStages) & 1), 5000000 + (int)k);
#ifdef ZOOMR_AB_CONS_DELAY  // A/B builds only: does the math warp pace the stream? (it does not)
    __nanosleep(ZOOMR_AB_CONS_DELAY);
#endif
    if (k == 0) {
      TL(3);
#ifdef ZOOMR_TL_RAMP
      TLW_SET(gw, 7, clock64());
#endif
    }
    if (k == nAk) TL(4);
    const uint32_t stK = ring + (uint32_t)(s * S::STAGE_BYTES);
    const uint32_t stV = stK + S::TILE_BYTES;

    // ---- S = K . Q^T  (2 m-tiles of 16 tokens) ----
    float sacc[2][4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
      for (int x = 0; x < 4; ++x) sacc[mt][x] = 0.f;
#pragma unroll
      for (int ks = 0; ks < NKS; ++ks) {
        uint32_t a0r, a1r, a2r, a3r;
        const int row = mt * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        ldsm_x4(S::at(stK, row, ks * 2 + (lane >> 4)), a0r, a1r, a2r, a3r);
        mma_bf16(sacc[mt], a0r, a1r, a2r, a3r, qf[ks][0], qf[ks][1]);
      }
    }
    // ---- online softmax over the tile's tokens, per column ----
    float cm0 = -INFINITY, cm1 = -INFINITY;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int t0 = mt * 16 + gq, t1 = t0 + 8;
      sacc[mt][0] = t0 < nvalid ? sacc[mt][0] * p.scale_log2 : -INFINITY;
      sacc[mt][1] = t0 < nvalid ? sacc[mt][1] * p.scale_log2 : -INFINITY;
      sacc[mt][2] = t1 < nvalid ? sacc[mt][2] * p.scale_log2 : -INFINITY;
      sacc[mt][3] = t1 < nvalid ? sacc[mt][3] * p.scale_log2 : -INFINITY;
      cm0 = fmaxf(cm0, fmaxf(sacc[mt][0], sacc[mt][2]));
      cm1 = fmaxf(cm1, fmaxf(sacc[mt][1], sacc[mt][3]));
    }
    if constexpr (kLogits) {  // H2O: the logits of the tile's rows (index positions, no early rows)
      const int sl = seg / p.Hkv, g = seg - sl * p.Hkv, l = p.l0 + sl;
      float *lg = p.logits + (((int64_t)b * p.L + l) * Hq + (int64_t)g * G) * p.cap + (int64_t)tis * kTile;
      const bool c0 = kTwoN ? n0 < G : part0 == 0, c1 = kTwoN ? n0 + 1 < G : part1 == 0;
      const int h0 = kTwoN ? n0 : n0 % G, h1 = kTwoN ? n0 + 1 : (n0 + 1) % G;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int t0 = mt * 16 + gq, t1 = t0 + 8;
        if (t0 < nvalid) {
          if (c0) lg[(int64_t)h0 * p.cap + t0] = sacc[mt][0] * 0.6931471805599453f;
          if (c1) lg[(int64_t)h1 * p.cap + t0] = sacc[mt][1] * 0.6931471805599453f;
        }
        if (t1 < nvalid) {
          if (c0) lg[(int64_t)h0 * p.cap + t1] = sacc[mt][2] * 0.6931471805599453f;
          if (c1) lg[(int64_t)h1 * p.cap + t1] = sacc[mt][3] * 0.6931471805599453f;
        }
      }
    }
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      cm0 = fmaxf(cm0, __shfl_xor_sync(0xffffffffu, cm0, off));
      cm1 = fmaxf(cm1, __shfl_xor_sync(0xffffffffu, cm1, off));
    }
    const float mn0 = fmaxf(m0, cm0), mn1 = fmaxf(m1, cm1);
    const float al0 = ex2(m0 - mn0), al1 = ex2(m1 - mn1);  // m = -inf -> 0
    m0 = mn0;
    m1 = mn1;
    float ps0 = 0.f, ps1 = 0.f;
    uint32_t bh[2][2], bl[2][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const float p00 = ex2(sacc[mt][0] - mn0), p01 = ex2(sacc[mt][1] - mn1);
      const float p10 = ex2(sacc[mt][2] - mn0), p11 = ex2(sacc[mt][3] - mn1);
      ps0 += p00 + p10;
      ps1 += p01 + p11;
      // hi = bf16(p), lo = bf16(p - hi)
      const float h00 = __bfloat162float(__float2bfloat16_rn(p00));
      const float h01 = __bfloat162float(__float2bfloat16_rn(p01));
      const float h10 = __bfloat162float(__float2bfloat16_rn(p10));
      const float h11 = __bfloat162float(__float2bfloat16_rn(p11));
      if constexpr (kTwoN) {
        bh[mt][0] = movm_t(pack_bf16(h00, h01));
        bh[mt][1] = movm_t(pack_bf16(h10, h11));
        bl[mt][0] = movm_t(pack_bf16(p00 - h00, p01 - h01));
        bl[mt][1] = movm_t(pack_bf16(p10 - h10, p11 - h11));
      } else {
        const float v00 = part0 == 0 ? h00 : (part0 == 1 ? p00 - h00 : 0.f);
        const float v01 = part1 == 0 ? h01 : (part1 == 1 ? p01 - h01 : 0.f);
        const float v10 = part0 == 0 ? h10 : (part0 == 1 ? p10 - h10 : 0.f);
        const float v11 = part1 == 0 ? h11 : (part1 == 1 ? p11 - h11 : 0.f);
        bh[mt][0] = movm_t(pack_bf16(v00, v01));
        bh[mt][1] = movm_t(pack_bf16(v10, v11));
      }
    }
    l0 = l0 * al0 + ps0;
    l1 = l1 * al1 + ps1;
    // ---- O^T = alpha * O^T + V^T . P ----
#pragma unroll
    for (int me = 0; me < NKS; ++me) {
      o[me][0] *= al0;
      o[me][1] *= al1;
      o[me][2] *= al0;
      o[me][3] *= al1;
      if constexpr (kTwoN) {
        o2[me][0] *= al0;
        o2[me][1] *= al1;
        o2[me][2] *= al0;
        o2[me][3] *= al1;
      }
#pragma unroll
      for (int kt = 0; kt < 2; ++kt) {
        uint32_t a0, a1, a2, a3;
        const int row = kt * 16 + (lane & 7) + ((lane >> 4) & 1) * 8;
        ldsm_x4_t(S::at(stV, row, me * 2 + ((lane >> 3) & 1)), a0, a1, a2, a3);
        mma_bf16(o[me], a0, a1, a2, a3, bh[kt][0], bh[kt][1]);
        if constexpr (kTwoN) mma_bf16(o2[me], a0, a1, a2, a3, bl[kt][0], bl[kt][1]);
      }
    }
    __syncwarp();  // every lane is done reading the stage
    if (lane == 0) mbar_arrive(&emptyp[s]);
  }
}

template <int D, int G>
size_t attn_smem_bytes(int B) {
  return 1024 + (size_t)AttnShape<D>::RING_BYTES + AttnShape<D>::BAR_BYTES + 16 + (size_t)B * sizeof(int4) +
         (size_t)kPtSmem * sizeof(int32_t) + (size_t)(2 * B + 3) * sizeof(int32_t);
}

// SMs left out of a5's persistent grid.  With the early-known rows (seq_len
// given) one SM is left free by default: the producer of I_f ends with one
// CTA per sequence building I_f, and an a5 CTA that had to wait for that SM
// would start its equal share of the work late and finish last.
inline int attn_spare_env() {
  static int spare = -2;
  if (spare == -2) {
    const char *e = getenv("ZOOMR_ATTN_SPARE_SMS");  // A/B experiments only
    spare = e ? atoi(e) : -1;
  }
  return spare;
}
inline int attn_grid(bool early = false) {
  const int env = attn_spare_env();
  const int spare = env >= 0 ? env : (early ? 1 : 0);
  const int g = num_sms() - spare;
  return g > 0 ? g : 1;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// 2D tensor map over a whole pool viewed as [rows][d] bf16, boxes of `box_rows`
// rows x (64 or d) columns, 128-byte swizzle for d >= 64.
inline int encode_pool_map(CUtensorMap *m, const void *base, int d, uint64_t rows, int box_rows) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return 1;
  }
  const bool swz = d >= 64;
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)d * 2};
  cuuint32_t box[2] = {(cuuint32_t)(swz ? 64 : d), (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : 1;
}

inline size_t attn_ws_part_floats(const zoomr_geom *g, int32_t batch) {
  const int G = g->num_q_heads / g->num_kv_heads;
  const size_t slots = 2 * ((size_t)attn_grid() * kPairs + (size_t)batch * g->num_layers * g->num_kv_heads);
  return slots * ((2 * G + 3) / 4 * 4 + G * g->head_dim);
}

}  // namespace zoomr

using namespace zoomr;

extern "C" size_t zoomr_attn_workspace_bytes(const zoomr_geom *geom, int32_t batch) {
  if (check_geom(geom) || batch < 1) return 0;
  const size_t part = attn_ws_part_floats(geom, batch) * sizeof(float);
  const size_t cnt = (size_t)batch * geom->num_layers * geom->num_kv_heads * sizeof(int32_t);
  return ((part + 255) / 256) * 256 + cnt;
}

static int sparse_decode_attn(const zoomr_geom *geom, int32_t batch, const void *q, const zoomr_kv *kv,
                              const int32_t *index, const int32_t *index_phys, const int32_t *index_count,
                              int32_t index_capacity, const int32_t *seq_len, int32_t sink, int32_t window,
                              float softmax_scale, int32_t layer_begin, int32_t layer_count, float *out, float *lse,
                              void *workspace, size_t workspace_bytes, int32_t *dev_status, void *stream,
                              float *logits = nullptr, bool chained = false) {
  int rc = check_geom(geom);
  if (rc) return rc;
  if (batch < 1 || !q || !kv || !kv->k || !kv->v || !kv->page_table || !index || !index_count ||
      index_capacity < 1 || !out || !workspace || kv->num_pages < 1 || kv->max_pages < 1)
    return ZOOMR_ERR_INVALID_ARG;
  if (layer_count == 0) layer_count = geom->num_layers - layer_begin;  // 0: every layer from layer_begin on
  if (layer_begin < 0 || layer_count < 1 || layer_begin + layer_count > geom->num_layers) return ZOOMR_ERR_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  // Right behind a chained a5 on the same workspace (on this stream), the early
  // rows would write the workspace while that launch may still be merging from
  // it: attend index-only (nothing written before the wait) instead.
  if (seq_len && prev_launch_is(s, kLaunchA5Chained, workspace)) seq_len = nullptr;
  if (batch > 65536) return ZOOMR_ERR_UNSUPPORTED;
  if (seq_len && (sink < 0 || window < 0)) return ZOOMR_ERR_INVALID_ARG;
  const size_t need = zoomr_attn_workspace_bytes(geom, batch);
  if (workspace_bytes < need) return ZOOMR_ERR_WORKSPACE;
  AttnParams prm;
  prm.q = (const __nv_bfloat16 *)q;
  prm.kpool = (const __nv_bfloat16 *)kv->k;
  prm.vpool = (const __nv_bfloat16 *)kv->v;
  prm.num_pages = kv->num_pages;
  prm.page_table = kv->page_table;
  prm.max_pages = kv->max_pages;
  prm.index = index;
  prm.index_phys = index_phys;
  prm.count = index_count;
  prm.cap = index_capacity;
  prm.out = out;
  prm.lse = lse;
  prm.logits = logits;
  if (logits && seq_len) return ZOOMR_ERR_INVALID_ARG;
  const size_t part = attn_ws_part_floats(geom, batch) * sizeof(float);
  prm.ws_part = (float *)workspace;
  prm.ws_cnt = (int32_t *)((char *)workspace + ((part + 255) / 256) * 256);
  prm.B = batch;
  prm.L = geom->num_layers;
  prm.l0 = layer_begin;
  prm.Lc = layer_count;
  prm.Hkv = geom->num_kv_heads;
  prm.P = geom->page_size;
  // the page table is staged in shared memory before the wait, except in the
  // lse / logits variants, where it may be the preceding kernel's output (the
  // host tier's residency table): read from global memory after the wait
  prm.pt_smem = !lse && (int64_t)batch * kv->max_pages <= kPtSmem;
  prm.Pshift = -1;
  for (int sft = 0; sft < 31; ++sft)
    if ((1 << sft) == geom->page_size) prm.Pshift = sft;
  prm.scale_log2 = softmax_scale * 1.4426950408889634f;
  prm.early_trigger = chained ? 1 : 0;
  prm.seq_len = seq_len;
  prm.sink = sink;
  prm.window = window;
  prm.status = dev_status;
  const int G = geom->num_q_heads / geom->num_kv_heads;
  const int grid = attn_grid(seq_len != nullptr);
  TmaMaps maps;
  {
    const uint64_t rows = (uint64_t)geom->num_layers * kv->num_pages * geom->num_kv_heads * geom->page_size;
    if (rows >= (1ull << 31)) return ZOOMR_ERR_UNSUPPORTED;  // TMA row coordinate is int32
    const int d = geom->head_dim;
    if (encode_pool_map(&maps.k32, kv->k, d, rows, 32) || encode_pool_map(&maps.v32, kv->v, d, rows, 32) ||
        encode_pool_map(&maps.k16, kv->k, d, rows, 16) || encode_pool_map(&maps.k8, kv->k, d, rows, 8) ||
        encode_pool_map(&maps.v16, kv->v, d, rows, 16) || encode_pool_map(&maps.v8, kv->v, d, rows, 8))
      return ZOOMR_ERR_CUDA;
  }
#define ZOOMR_AT(DD, GG)                                                                 \
  do {                                                                                   \
    auto kfn = logits ? sparse_attn_kernel<DD, GG, true> : sparse_attn_kernel<DD, GG>;   \
    const size_t smem = attn_smem_bytes<DD, GG>(batch);                                  \
    if (smem > 227 * 1024) return ZOOMR_ERR_UNSUPPORTED;                                 \
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);   \
    prefer_max_smem(kfn);                                                                \
    launch_pdl(kfn, grid, 64 * kPairs, smem, s, prm, maps);                              \
  } while (0)
#define ZOOMR_AT_G(DD)               \
  switch (G) {                       \
    case 1: ZOOMR_AT(DD, 1); break;  \
    case 2: ZOOMR_AT(DD, 2); break;  \
    case 4: ZOOMR_AT(DD, 4); break;  \
    case 7: ZOOMR_AT(DD, 7); break;  \
    default: ZOOMR_AT(DD, 8); break; \
  }
  switch (geom->head_dim) {
    case 16: ZOOMR_AT_G(16); break;
    case 32: ZOOMR_AT_G(32); break;
    case 64: ZOOMR_AT_G(64); break;
    default: ZOOMR_AT_G(128); break;
  }
#undef ZOOMR_AT_G
#undef ZOOMR_AT
  return launch_status(s, chained ? kLaunchA5Chained : kLaunchOther, workspace);
}

extern "C" int zoomr_sparse_decode_attn(const zoomr_geom *geom, int32_t batch, const void *q,
                                        const zoomr_kv *kv, const int32_t *index, const int32_t *index_phys,
                                        const int32_t *index_count, int32_t index_capacity,
                                        const int32_t *seq_len, int32_t sink, int32_t window,
                                        float softmax_scale, int32_t layer_begin, int32_t layer_count, float *out,
                                        void *workspace, size_t workspace_bytes, int32_t *dev_status, void *stream) {
  return sparse_decode_attn(geom, batch, q, kv, index, index_phys, index_count, index_capacity, seq_len, sink, window,
                            softmax_scale, layer_begin, layer_count, out, nullptr, workspace, workspace_bytes,
                            dev_status, stream);
}

extern "C" int zoomr_sparse_decode_attn_chained(const zoomr_geom *geom, int32_t batch, const void *q,
                                                const zoomr_kv *kv, const int32_t *index, const int32_t *index_phys,
                                                const int32_t *index_count, int32_t index_capacity,
                                                const int32_t *seq_len, int32_t sink, int32_t window,
                                                float softmax_scale, int32_t layer_begin, int32_t layer_count,
                                                float *out, void *workspace, size_t workspace_bytes,
                                                int32_t *dev_status, void *stream) {
  return sparse_decode_attn(geom, batch, q, kv, index, index_phys, index_count, index_capacity, seq_len, sink, window,
                            softmax_scale, layer_begin, layer_count, out, nullptr, workspace, workspace_bytes,
                            dev_status, stream, nullptr, true);
}

extern "C" int zoomr_sparse_decode_attn_lse(const zoomr_geom *geom, int32_t batch, const void *q,
                                            const zoomr_kv *kv, const int32_t *index, const int32_t *index_phys,
                                            const int32_t *index_count, int32_t index_capacity,
                                            const int32_t *seq_len, int32_t sink, int32_t window,
                                            float softmax_scale, int32_t layer_begin, int32_t layer_count, float *out,
                                            float *lse, void *workspace, size_t workspace_bytes, int32_t *dev_status,
                                            void *stream) {
  if (!lse) return ZOOMR_ERR_INVALID_ARG;
  return sparse_decode_attn(geom, batch, q, kv, index, index_phys, index_count, index_capacity, seq_len, sink, window,
                            softmax_scale, layer_begin, layer_count, out, lse, workspace, workspace_bytes, dev_status,
                            stream);
}

extern "C" int zoomr_sparse_decode_attn_lse_chained(const zoomr_geom *geom, int32_t batch, const void *q,
                                                    const zoomr_kv *kv, const int32_t *index,
                                                    const int32_t *index_phys, const int32_t *index_count,
                                                    int32_t index_capacity, const int32_t *seq_len, int32_t sink,
                                                    int32_t window, float softmax_scale, int32_t layer_begin,
                                                    int32_t layer_count, float *out, float *lse, void *workspace,
                                                    size_t workspace_bytes, int32_t *dev_status, void *stream) {
  if (!lse) return ZOOMR_ERR_INVALID_ARG;
  return sparse_decode_attn(geom, batch, q, kv, index, index_phys, index_count, index_capacity, seq_len, sink, window,
                            softmax_scale, layer_begin, layer_count, out, lse, workspace, workspace_bytes, dev_status,
                            stream, nullptr, true);
}

extern "C" int zoomr_sparse_decode_attn_logits(const zoomr_geom *geom, int32_t batch, const void *q,
                                               const zoomr_kv *kv, const int32_t *index, const int32_t *index_count,
                                               int32_t index_capacity, float softmax_scale, float *out, float *lse,
                                               float *logits, void *workspace, size_t workspace_bytes,
                                               int32_t *dev_status, void *stream) {
  if (!lse || !logits) return ZOOMR_ERR_INVALID_ARG;
  return sparse_decode_attn(geom, batch, q, kv, index, nullptr, index_count, index_capacity, nullptr, 0, 0,
                            softmax_scale, 0, 0, out, lse, workspace, workspace_bytes, dev_status, stream, logits);
}

// ---- the per-stream record of the library's last launch (common.cuh) ----------
namespace {
struct LaunchRec {
  int kind;
  const void *ws;
};
std::mutex g_launch_mu;
std::unordered_map<cudaStream_t, LaunchRec> g_launch;
}  // namespace

void zoomr::note_launch(cudaStream_t s, int kind, const void *ws) {
  std::lock_guard<std::mutex> lk(g_launch_mu);
  if (kind == kLaunchOther) {
    auto it = g_launch.find(s);
    if (it != g_launch.end()) g_launch.erase(it);  // the common case keeps the table empty
  } else {
    g_launch[s] = LaunchRec{kind, ws};
  }
}

bool zoomr::prev_launch_is(cudaStream_t s, int kind, const void *ws) {
  std::lock_guard<std::mutex> lk(g_launch_mu);
  auto it = g_launch.find(s);
  if (it == g_launch.end()) return kind == kLaunchOther;
  return it->second.kind == kind && (!ws || it->second.ws == ws);
}

extern "C" const char *zoomr_status_str(int status) {
  switch (status) {
    case ZOOMR_OK: return "ZOOMR_OK";
    case ZOOMR_ERR_INVALID_ARG: return "ZOOMR_ERR_INVALID_ARG";
    case ZOOMR_ERR_DIM_MISMATCH: return "ZOOMR_ERR_DIM_MISMATCH";
    case ZOOMR_ERR_EMPTY_SEGMENT: return "ZOOMR_ERR_EMPTY_SEGMENT";
    case ZOOMR_ERR_SEGMENT_ORDER: return "ZOOMR_ERR_SEGMENT_ORDER";
    case ZOOMR_ERR_INDEX_RANGE: return "ZOOMR_ERR_INDEX_RANGE";
    case ZOOMR_ERR_CAPACITY: return "ZOOMR_ERR_CAPACITY";
    case ZOOMR_ERR_UNSUPPORTED: return "ZOOMR_ERR_UNSUPPORTED";
    case ZOOMR_ERR_CUDA: return "ZOOMR_ERR_CUDA";
    case ZOOMR_ERR_WORKSPACE: return "ZOOMR_ERR_WORKSPACE";
    default: return "ZOOMR_ERR_UNKNOWN";
  }
}

extern "C" int zoomr_abi_version(void) { return ZOOMR_ABI_VERSION; }

#ifdef ZOOMR_WATCHDOG
extern "C" int zoomr_watchdog_set(void *host_mapped_dev_ptr) {
  return cudaMemcpyToSymbol(zoomr::g_wd_host, &host_mapped_dev_ptr, sizeof(void *)) == cudaSuccess ? 0 : 8;
}
#endif
