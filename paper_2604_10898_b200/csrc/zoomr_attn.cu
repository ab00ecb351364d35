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

#include "common.cuh"

namespace zoomr {

constexpr int kTile = 32;   // tokens per tile (one per lane when resolving addresses)
constexpr int kPairs = 4;   // producer/consumer warp pairs per CTA
constexpr int kStages = 3;  // ring depth per pair
constexpr int kPtSmem = 4096; // page-table entries staged in shared memory when they fit

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
  static constexpr int BAR_BYTES = 2 * kPairs * kStages * 8;
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
  CUtensorMap k16, k8, v16, v8;  // 2D [total rows][D] views of the pools, boxes of 16 / 8 rows
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
  float *ws_part;  // [NW][2][G*(D+2)]
  int32_t *ws_cnt; // [B*L*Hkv]
  int32_t B, L, Hkv, P, Pshift;  // Pshift = log2(P) when P is a power of two, else -1
  int32_t pt_smem;               // page table staged in shared memory (B*max_pages <= kPtSmem)
  float scale_log2;
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
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
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
  __device__ __forceinline__ int64_t warp_of(int64_t t) const { return ((t + 1) * NWe - 1) / T_tot; }
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

template <int D, int G>
__global__ void __launch_bounds__(64 * kPairs, 1)
    sparse_attn_kernel(const AttnParams p, const __grid_constant__ TmaMaps maps) {
  using S = AttnShape<D>;
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  // the 128-byte swizzle pattern follows address bits [7:9]: keep the ring 1024-aligned
  unsigned char *smem = smem_dyn + ((1024 - (smem_u32(smem_dyn) & 1023)) & 1023);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + S::RING_BYTES);  // [kPairs][kStages]
  uint64_t *empty = full + kPairs * kStages;                             // [kPairs][kStages]
  int32_t *pts = reinterpret_cast<int32_t *>(smem + S::RING_BYTES + S::BAR_BYTES);  // [kPtSmem] page tables
  int32_t *prefix = pts + (p.pt_smem ? kPtSmem : 0);                                  // [B+1]
  int32_t *cnts = prefix + p.B + 1;                                                   // [B] clamped |I_f|
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Hq = p.Hkv * G;

  if (threadIdx.x == 0) {
    for (int x = 0; x < kPairs * kStages; ++x) {
      mbar_init(&full[x], 33);  // producer lane 0's expect_tx arrive + one cp.async (noinc) arrive per lane
      mbar_init(&empty[x], 1);  // the math warp's lane 0
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // The page tables are inputs, not outputs of the preceding kernel (a4 / the
  // fused select): stage them while that kernel is still finishing.
  if (p.pt_smem)
    for (int x = threadIdx.x; x < p.B * p.max_pages; x += blockDim.x) pts[x] = p.page_table[x];
  // Programmatic dependent launch: everything above overlaps the producer of
  // I_f (a4 / the fused select); from here on its results are visible.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // tiles per sequence -> prefix (warp 0 scans in chunks of 32 sequences)
  if (warp == 0) {
    int carry = 0;
    for (int b0 = 0; b0 < p.B; b0 += 32) {
      const int b = b0 + lane;
      int n = 0;
      if (b < p.B) {
        int c = p.count[b];
        c = c < p.cap ? c : p.cap;
        cnts[b] = c;
        n = c > 0 ? (c + kTile - 1) / kTile * p.L * p.Hkv : 0;
      }
      int incl = n;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (b < p.B) prefix[b] = carry + incl - n;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) prefix[p.B] = carry;
  }
  __syncthreads();

  Sched sc;
  sc.prefix = prefix;
  sc.T_tot = prefix[p.B];
  sc.B = p.B;
  sc.LH = p.L * p.Hkv;
  if (sc.T_tot == 0) return;
  const int64_t NW = (int64_t)gridDim.x * kPairs;
  sc.NWe = NW < sc.T_tot ? NW : sc.T_tot;

  const int pair = warp % kPairs;
  const bool producer = warp >= kPairs;
  const int64_t gw = (int64_t)blockIdx.x * kPairs + pair;  // global math-warp id of the pair
  if (gw >= sc.NWe) return;
  const int64_t r0 = sc.range_start(gw), r1 = sc.range_start(gw + 1);
  const int64_t ntiles = r1 - r0;
  const uint32_t ring = smem_u32(smem) + (uint32_t)(pair * kStages * S::STAGE_BYTES);
  uint64_t *fullp = full + pair * kStages;
  uint64_t *emptyp = empty + pair * kStages;

  if (producer) {
    // ================= producer: 3-stage address pipeline, LDGSTS copies =====
    // A(k+2): I_f position load   B(k+1): page-table load   C(k): row copies.
    // Each dependent load is consumed one iteration after it is issued, so the
    // index -> page -> row chain never stalls the copy issue in steady state.
    struct Addr {
      int b, l, g, ok, tok, slot, page;
    };
    auto stage_a = [&](int64_t k, Addr &a) {
      int seg, tis, nts;
      sc.locate(r0 + k, a.b, seg, tis, nts);
      const int cnt = cnts[a.b];
      a.l = seg / p.Hkv;
      a.g = seg - a.l * p.Hkv;
      const int pos = tis * kTile + lane;
      a.ok = pos < cnt;
      // with index_phys, `tok` carries the page-resolved row and stage B is a no-op;
      // the load is guarded by the capacity, not the count, so it does not wait for it
      const int32_t *src = p.index_phys ? p.index_phys : p.index;
      a.tok = pos < p.cap ? src[(int64_t)a.b * p.cap + pos] : 0;
    };
    auto stage_b = [&](Addr &a) {
      a.page = 0;
      a.slot = 0;
      if (a.ok && !p.index_phys) {
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
    const int rsub = lane / S::CPR, ch = lane % S::CPR;
    // one loop, one call site per stage (the pipeline fill is its first kAheadA
    // iterations): the kernel's code stays small enough for the instruction cache
    for (int64_t k = -kAheadA; k < ntiles; ++k) {
      if (k + kAheadA < ntiles) stage_a(k + kAheadA, q4);
      if (k + kAheadB >= 0 && k + kAheadB < ntiles) stage_b(q2);
      if (k < 0) {
        q0 = q1;
        q1 = q2;
        q2 = q3;
        q3 = q4;
        continue;
      }
      Addr &ac = q0;
      // stage C: global row of every token of tile k
      const int cok = ac.ok;
      int64_t grow = 0;
      int page = ac.page;
      if (p.index_phys) {
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
      // runs of consecutive tokens in one page -> boxes of 16 / 8 rows; the rest by cp.async
      const int ptok = __shfl_up_sync(0xffffffffu, ac.tok, 1);
      const int ppage = __shfl_up_sync(0xffffffffu, page, 1);
      const int pok = __shfl_up_sync(0xffffffffu, cok, 1);
      const bool cont = cok && lane > 0 && pok && ptok + 1 == ac.tok && (p.index_phys || ppage == page);
      const unsigned validm = __ballot_sync(0xffffffffu, cok);
      const unsigned startm = __ballot_sync(0xffffffffu, cok && !cont);
      const unsigned upto = lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
      const int rs = 31 - __clz(startm & upto | 1u);               // my run's first slot
      const unsigned after = (startm | ~validm) & ~upto;
      const int re = after ? __ffs(after) - 1 : 32;                // one past my run's last slot
      const int pos = lane - rs, len = re - rs;
      const int n16 = (len >> 4) << 4, n8 = ((len & 15) >> 3) << 3;
      // TMA boxes need 128-byte aligned destinations: d >= 64 only (d < 64 configs are toy-sized)
      const bool lead16 = S::SWZ && cok && pos < n16 && (pos & 15) == 0;
      const bool lead8 = S::SWZ && cok && n8 && pos == n16;
      const bool byhand = !cok || !S::SWZ || pos >= n16 + n8;
      const unsigned m16 = __ballot_sync(0xffffffffu, lead16), m8 = __ballot_sync(0xffffffffu, lead8);
      const uint32_t tx = (uint32_t)((__popc(m16) * 16 + __popc(m8) * 8) * S::RB * 2);
      const int s = (int)(k % kStages);
      mbar_wait(&emptyp[s], (uint32_t)(((k / kStages) & 1) ^ 1));
      const uint32_t stK = ring + (uint32_t)(s * S::STAGE_BYTES);
      const uint32_t stV = stK + S::TILE_BYTES;
      if (lane == 0) mbar_arrive_expect_tx(&fullp[s], tx);
      __syncwarp();
      if (lead16 || lead8) {
        const CUtensorMap *mk = lead16 ? &maps.k16 : &maps.k8;
        const CUtensorMap *mv = lead16 ? &maps.v16 : &maps.v8;
#pragma unroll
        for (int rg = 0; rg < S::NREG; ++rg) {
          // destination = the row's unswizzled start; the TMA unit applies the 128-byte swizzle
          const uint32_t off = (uint32_t)(rg * S::REG_BYTES + lane * S::RBR);
          tma_load_2d(stK + off, mk, rg * S::BX, grow, &fullp[s]);
          tma_load_2d(stV + off, mv, rg * S::BX, grow, &fullp[s]);
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
  constexpr bool kTwoN = (G == 8);          // hi and lo in separate n-tiles
  // column -> (head, part) for G <= 4: head = n % G, part = n / G (0 hi, 1 lo, >=2 none)
  const int part0 = kTwoN ? 0 : n0 / G, part1 = kTwoN ? 0 : (n0 + 1) / G;
  constexpr int HDR = (2 * G + 3) / 4 * 4;  // m[G], l[G] padded to a 16-byte boundary
  constexpr int SLOT = HDR + G * D;         // partial result: header, then O[G][D]

  int first_b = -1, first_seg = -1;  // the first segment of this warp's range (slot rule)
  int cur_b = -1, cur_seg = -1;
  uint32_t qf[NKS][2];
  float o[NKS][4], o2[kTwoN ? NKS : 1][4];
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  auto flush = [&](int b, int seg) {
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
        if constexpr (G == 8) v += o2[me][x];
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
    const bool owner = (G == 8) || (G == 4 && tq < 2) || (G <= 2 && tq == 0);
    const int nh = (G == 1) ? 1 : 2;  // heads held by an owner thread: n0 (and n0+1)
    const int l = seg / p.Hkv, g = seg - l * p.Hkv;
    const int nts = (sc.prefix[b + 1] - sc.prefix[b]) / sc.LH;
    const int64_t st0 = sc.prefix[b] + (int64_t)seg * nts, st1 = st0 + nts;
    const int64_t wf = sc.warp_of(st0), wl = sc.warp_of(st1 - 1);
    float *ob = p.out + (((int64_t)b * p.L + l) * Hq + (int64_t)g * G) * D;
    if (wf == wl) {  // this warp owns the whole segment: final output
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
      }
      return;
    }
    // partial: slot 0 if this is the warp's first segment, else slot 1
    const int slot = (b == first_b && seg == first_seg) ? 0 : 1;
    float *ps = p.ws_part + ((int64_t)gw * 2 + slot) * SLOT;
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
    int32_t *cnt = p.ws_cnt + (int64_t)b * sc.LH + seg;
    int old = 0;
    if (lane == 0)
      asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
    old = __shfl_sync(0xffffffffu, old, 0);
    if (old != (int)(wl - wf)) return;  // not the last arriving warp
    __syncwarp();  // the other lanes' partial loads below are ordered after lane 0's acquire
    // last arriver: merge the partials of warps wf..wl (fixed order -> deterministic).
    const int nparts = (int)(wl - wf + 1);
    constexpr int NV4 = G * D / 4;
    constexpr int PER = (NV4 + 31) / 32;
    constexpr int NPF = G >= 8 ? 2 : 4;  // fast path: every load of up to NPF parts in flight at once
    if (nparts <= NPF) {
      const float *qp[NPF];
      float mh[NPF][G], lh[NPF][G];
      float4 ov4[NPF][PER];
#pragma unroll
      for (int j = 0; j < NPF; ++j) {
        if (j < nparts) {
          int fb, fs, ft, fn;
          sc.locate(sc.range_start(wf + j), fb, fs, ft, fn);
          qp[j] = p.ws_part + ((wf + j) * 2 + ((fb == b && fs == seg) ? 0 : 1)) * SLOT;
#pragma unroll
          for (int h = 0; h < G; ++h) {
            mh[j][h] = __ldcg(qp[j] + h);
            lh[j][h] = __ldcg(qp[j] + G + h);
          }
#pragma unroll
          for (int u = 0; u < PER; ++u) {
            const int f = lane + 32 * u;
            ov4[j][u] = f < NV4 ? __ldcg(reinterpret_cast<const float4 *>(qp[j] + HDR) + f) : make_float4(0, 0, 0, 0);
          }
        }
      }
      float Mh[G], Lh[G];
#pragma unroll
      for (int h = 0; h < G; ++h) {
        Mh[h] = -INFINITY;
        Lh[h] = 0.f;
#pragma unroll
        for (int j = 0; j < NPF; ++j)
          if (j < nparts) Mh[h] = fmaxf(Mh[h], mh[j][h]);
      }
      float w[NPF][G];
#pragma unroll
      for (int j = 0; j < NPF; ++j)
#pragma unroll
        for (int h = 0; h < G; ++h) {
          w[j][h] = j < nparts ? ex2(mh[j][h] - Mh[h]) : 0.f;
          Lh[h] += j < nparts ? lh[j][h] * w[j][h] : 0.f;
        }
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const int f = lane + 32 * u;
        if (f < NV4) {
          const int h = (4 * f) / D;
          float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int j = 0; j < NPF; ++j)
            if (j < nparts) {
              a.x += ov4[j][u].x * w[j][h];
              a.y += ov4[j][u].y * w[j][h];
              a.z += ov4[j][u].z * w[j][h];
              a.w += ov4[j][u].w * w[j][h];
            }
          const float inv = 1.f / Lh[h];
          reinterpret_cast<float4 *>(ob)[f] = make_float4(a.x * inv, a.y * inv, a.z * inv, a.w * inv);
        }
      }
      if (lane == 0) *cnt = 0;  // leave the workspace zeroed for the next call
      return;
    }
    // (general path) lane j fetches part j's header (slot pointer, m[G], l[G])
    // so that all the round trips of a chunk of 32 parts are in flight together.
    float Mh[G], Lh[G];
    float4 acc[PER];
#pragma unroll
    for (int h = 0; h < G; ++h) {
      Mh[h] = -INFINITY;
      Lh[h] = 0.f;
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int pass = 0; pass < 2; ++pass) {
      for (int j0 = 0; j0 < nparts; j0 += 32) {
        const int j = j0 + lane;
        const float *q2 = nullptr;
        float mj[G], lj[G];
        if (j < nparts) {
          int fb, fs, ft, fn;
          sc.locate(sc.range_start(wf + j), fb, fs, ft, fn);
          q2 = p.ws_part + ((wf + j) * 2 + ((fb == b && fs == seg) ? 0 : 1)) * SLOT;
#pragma unroll
          for (int h = 0; h < G; ++h) {
            mj[h] = __ldcg(q2 + h);
            lj[h] = __ldcg(q2 + G + h);
          }
        }
        if (pass == 0) {  // per-head max over all parts
          if (j < nparts)
#pragma unroll
            for (int h = 0; h < G; ++h) Mh[h] = fmaxf(Mh[h], mj[h]);
          continue;
        }
        float wj[G];
#pragma unroll
        for (int h = 0; h < G; ++h) {
          wj[h] = j < nparts ? ex2(mj[h] - Mh[h]) : 0.f;
          Lh[h] += j < nparts ? lj[h] * wj[h] : 0.f;
        }
        const int nj = min(32, nparts - j0);
        for (int u0 = 0; u0 < nj; ++u0) {
          const float *qq = (const float *)__shfl_sync(0xffffffffu, (unsigned long long)q2, u0);
          float w[G];
#pragma unroll
          for (int h = 0; h < G; ++h) w[h] = __shfl_sync(0xffffffffu, wj[h], u0);
          const float4 *O4 = reinterpret_cast<const float4 *>(qq + HDR);
#pragma unroll
          for (int u = 0; u < PER; ++u) {
            const int f = lane + 32 * u;
            if (f < NV4) {
              const float4 v = __ldcg(O4 + f);
              const float ww = w[(4 * f) / D];
              acc[u].x += v.x * ww;
              acc[u].y += v.y * ww;
              acc[u].z += v.z * ww;
              acc[u].w += v.w * ww;
            }
          }
        }
      }
      if (pass == 0) {
#pragma unroll
        for (int h = 0; h < G; ++h)
#pragma unroll
          for (int off = 16; off; off >>= 1) Mh[h] = fmaxf(Mh[h], __shfl_xor_sync(0xffffffffu, Mh[h], off));
      }
    }
#pragma unroll
    for (int h = 0; h < G; ++h)
#pragma unroll
      for (int off = 16; off; off >>= 1) Lh[h] += __shfl_xor_sync(0xffffffffu, Lh[h], off);
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int f = lane + 32 * u;
      if (f < NV4) {
        const float inv = 1.f / Lh[(4 * f) / D];
        reinterpret_cast<float4 *>(ob)[f] =
            make_float4(acc[u].x * inv, acc[u].y * inv, acc[u].z * inv, acc[u].w * inv);
      }
    }
    if (lane == 0) *cnt = 0;  // leave the workspace zeroed for the next call
  };

  for (int64_t k = 0; k <= ntiles; ++k) {  // k == ntiles: only the final flush
    int b = -1, seg = -1, tis = 0, nts = 0;
    if (k < ntiles) sc.locate(r0 + k, b, seg, tis, nts);
    if (k == 0) {
      first_b = b;
      first_seg = seg;
    }
    if (b != cur_b || seg != cur_seg) {
      if (cur_b >= 0) flush(cur_b, cur_seg);
      if (k == ntiles) break;
      cur_b = b;
      cur_seg = seg;
      // Q fragments (B operand of QK^T): Q[head n % G][k-chunk], this thread's column n = gq
      const int l = seg / p.Hkv, g = seg - l * p.Hkv;
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
    const int cnt = cnts[b];
    const int nvalid = min(kTile, cnt - tis * kTile);
    const int s = (int)(k % kStages);
    mbar_wait(&fullp[s], (uint32_t)((k / kStages) & 1));
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
        uint32_t a0, a1, a2, a3;
        const int row = mt * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        ldsm_x4(S::at(stK, row, ks * 2 + (lane >> 4)), a0, a1, a2, a3);
        mma_bf16(sacc[mt], a0, a1, a2, a3, qf[ks][0], qf[ks][1]);
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
  return 1024 + (size_t)AttnShape<D>::RING_BYTES + AttnShape<D>::BAR_BYTES + (size_t)kPtSmem * sizeof(int32_t) +
         (size_t)(2 * B + 1) * sizeof(int32_t);
}

inline int attn_grid() {
  static int spare = -1;
  if (spare < 0) {
    const char *e = getenv("ZOOMR_ATTN_SPARE_SMS");  // A/B experiments only
    spare = e ? atoi(e) : 0;
  }
  return num_sms() - spare;
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

inline size_t attn_ws_part_floats(const zoomr_geom *g) {
  const int G = g->num_q_heads / g->num_kv_heads;
  return (size_t)attn_grid() * kPairs * 2 * ((2 * G + 3) / 4 * 4 + G * g->head_dim);
}

}  // namespace zoomr

using namespace zoomr;

extern "C" size_t zoomr_attn_workspace_bytes(const zoomr_geom *geom, int32_t batch) {
  if (check_geom(geom) || batch < 1) return 0;
  const size_t part = attn_ws_part_floats(geom) * sizeof(float);
  const size_t cnt = (size_t)batch * geom->num_layers * geom->num_kv_heads * sizeof(int32_t);
  return ((part + 255) / 256) * 256 + cnt;
}

extern "C" int zoomr_sparse_decode_attn(const zoomr_geom *geom, int32_t batch, const void *q,
                                        const zoomr_kv *kv, const int32_t *index, const int32_t *index_phys,
                                        const int32_t *index_count, int32_t index_capacity,
                                        float softmax_scale, float *out, void *workspace,
                                        size_t workspace_bytes, int32_t *dev_status, void *stream) {
  int rc = check_geom(geom);
  if (rc) return rc;
  if (batch < 1 || !q || !kv || !kv->k || !kv->v || !kv->page_table || !index || !index_count ||
      index_capacity < 1 || !out || !workspace || kv->num_pages < 1 || kv->max_pages < 1)
    return ZOOMR_ERR_INVALID_ARG;
  if (batch > 65536) return ZOOMR_ERR_UNSUPPORTED;
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
  const size_t part = attn_ws_part_floats(geom) * sizeof(float);
  prm.ws_part = (float *)workspace;
  prm.ws_cnt = (int32_t *)((char *)workspace + ((part + 255) / 256) * 256);
  prm.B = batch;
  prm.L = geom->num_layers;
  prm.Hkv = geom->num_kv_heads;
  prm.P = geom->page_size;
  prm.pt_smem = (int64_t)batch * kv->max_pages <= kPtSmem;
  prm.Pshift = -1;
  for (int sft = 0; sft < 31; ++sft)
    if ((1 << sft) == geom->page_size) prm.Pshift = sft;
  prm.scale_log2 = softmax_scale * 1.4426950408889634f;
  prm.status = dev_status;
  const int G = geom->num_q_heads / geom->num_kv_heads;
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = attn_grid();
  TmaMaps maps;
  {
    const uint64_t rows = (uint64_t)geom->num_layers * kv->num_pages * geom->num_kv_heads * geom->page_size;
    if (rows >= (1ull << 31)) return ZOOMR_ERR_UNSUPPORTED;  // TMA row coordinate is int32
    const int d = geom->head_dim;
    if (encode_pool_map(&maps.k16, kv->k, d, rows, 16) || encode_pool_map(&maps.k8, kv->k, d, rows, 8) ||
        encode_pool_map(&maps.v16, kv->v, d, rows, 16) || encode_pool_map(&maps.v8, kv->v, d, rows, 8))
      return ZOOMR_ERR_CUDA;
  }
#define ZOOMR_AT(DD, GG)                                                                 \
  do {                                                                                   \
    auto kfn = sparse_attn_kernel<DD, GG>;                                               \
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
  return launch_status();
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
