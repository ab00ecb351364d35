// select_common.cuh -- block-level building blocks of the selection stages a1-a4,
// shared by the standalone entry points (zoomr_update_mean_keys, zoomr_score,
// zoomr_select_topc, zoomr_build_index) and the fused one (zoomr_select_fused).
#pragma once

#include "common.cuh"

namespace zoomr {

#ifndef ZOOMR_SCORE_MARK
#define ZOOMR_SCORE_MARK(i) do { } while (0)
#endif
constexpr int kHistBins = 2048;  // vote histogram bins of the top-c threshold search
constexpr int kTopcRounds = 8;   // c <= this: the c largest votes by c block-max rounds, then the tie group
constexpr int kTopcRoundsMinN = 192;  // ... when N_t is above this (below, direct ranking is cheaper:
                                      // tools/bench_blocks.cu, 4.3 K vs 5.0 K cycles at N_t = 120, 9.7 K vs
                                      // 5.2 K at N_t = 240 -- a barrier costs ~220 cycles, redux ~200)

// Carves 16-byte-aligned sub-arrays out of dynamic shared memory.
struct SmemCarve {
  unsigned char *p;
  template <typename T>
  __device__ __forceinline__ T *take(size_t n) {
    T *r = reinterpret_cast<T *>(((uintptr_t)p + 15) & ~(uintptr_t)15);
    p = reinterpret_cast<unsigned char *>(r + n);
    return r;
  }
};

__device__ __forceinline__ bool better_alpha(float a, int i, float b, int j) {
  return a > b || (a == b && i < j);  // (alpha desc, index asc): reading Q3
}

// "x before y" in the consensus order (v desc, A desc, i asc): readings Q2, Q3
__device__ __forceinline__ bool before_key(int vx, long long ax, int ix, int vy, long long ay, int iy) {
  if (vx != vy) return vx > vy;
  if (ax != ay) return ax > ay;
  return ix < iy;
}

// round(alpha * 2^ZOOMR_A_FRAC_BITS) -- the fixed-point A contribution of one vote
__device__ __forceinline__ long long alpha_fixed(float a) { return __double2ll_rn((double)a * 4294967296.0); }

// Block exclusive scan of one int per thread (blockDim.x <= 1024, multiple of 32).
// `tmp` is >= 33 ints of shared memory.  Returns the exclusive prefix; *total gets the sum.
__device__ __forceinline__ int block_excl_scan(int x, int *tmp, int *total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) tmp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int wt = lane < nw ? tmp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, wt, o);
      if (lane >= o) wt += y;
    }
    if (lane < nw) tmp[lane] = wt;
  }
  __syncthreads();
  const int ex = (warp ? tmp[warp - 1] : 0) + incl - x;
  *total = tmp[nw - 1];
  __syncthreads();
  return ex;
}

// ---------------------------------------------------------------- a1 -----
// Mean key of summary i for one (l, g) by the whole block: warps take the
// summary's tokens round-robin, lanes take the head dimension, fp64 partial
// sums meet in shared memory.  The fp64 sum of bf16 values (8 significant bits)
// is exact for any realistic exponent spread, so the warp order does not change
// the result: it equals the sequential sum of the definition.
template <int D>
__device__ void block_mean_key(const __nv_bfloat16 *__restrict__ kpool, int64_t num_pages,
                               const int32_t *__restrict__ pt, int32_t max_pages, int P, int Hkv, int l,
                               int g, int s0, int s1, double *red /* smem [nwarps][D] */,
                               float *__restrict__ out, int32_t *status, float *fresh = nullptr) {
  constexpr int EPL = D >= 32 ? D / 32 : 1;
  constexpr int LANES = D >= 32 ? 32 : D;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double acc[EPL];
#pragma unroll
  for (int e = 0; e < EPL; ++e) acc[e] = 0.0;
  if (lane < LANES) {
    for (int j = s0 + warp; j < s1; j += nw) {
      const int lp = j / P;
      int page = lp < max_pages ? pt[lp] : -1;
      if (page < 0 || page >= num_pages) {
        set_status(status, ZOOMR_ERR_INDEX_RANGE);
        page = 0;
      }
      const __nv_bfloat16 *row = kpool + ((((int64_t)l * num_pages + page) * Hkv + g) * P + (j - lp * P)) * D;
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
#pragma unroll
    for (int e = 0; e < EPL; ++e) red[warp * D + lane * EPL + e] = acc[e];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < D; e += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += red[w * D + e];
    out[e] = (float)(s / (double)(s1 - s0));  // (1/|S_i|) * sum
    if (fresh) fresh[e] = out[e];
  }
  __syncthreads();
}

// ---------------------------------------------------------------- a2 -----
// alpha[hh][i] = q_hh . kbar_i for the G query heads of one KV head, into shared
// memory (and alpha_out), then every warp hh < G selects voter hh's top-k:
// sel_i[hh*top_k + r], sel_a[...] (alpha of the pick) for r < min(k, nt).
template <int D, int G>
__device__ void block_score_topk(const __nv_bfloat16 *__restrict__ qb /* [G][D] */,
                                 const float *__restrict__ mk /* [nt][D] fp32 */, int nt, int top_k,
                                 float *qs /* smem [G][D] */, float *al /* smem [G][ald] */, int ald,
                                 float *__restrict__ alpha_out /* [G][ald_out] or null */, int64_t ald_out,
                                 int *sel_i /* smem [G][top_k] */, float *sel_a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (qb) {  // (null: the caller has staged qs already)
    for (int x = threadIdx.x; x < G * D; x += blockDim.x) qs[x] = __bfloat162float(qb[x]);
    __syncthreads();
  }
  constexpr int FPL = D / 8;  // floats per octet lane
  constexpr int NV = FPL >= 4 ? FPL / 4 : 1;
  const int oct = lane >> 3, l8 = lane & 7;
  // each warp takes 8 rows per step (2 per octet); the next step's rows are
  // loaded before this step's math (double buffering), so at large N_t the
  // loop streams instead of paying one round trip per step
  float4 kv[2][NV], kn[2][NV];
  float2 kv2[2], kn2[2];
  auto load = [&](int base, float4 (&dst)[2][NV], float2 (&dst2)[2]) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = base + u * 4 + oct;
      const float *row = mk + (int64_t)(i < nt ? i : 0) * D;
      if constexpr (FPL >= 4) {
#pragma unroll
        for (int m = 0; m < NV; ++m) dst[u][m] = *reinterpret_cast<const float4 *>(row + m * 32 + l8 * 4);
      } else {
        dst2[u] = *reinterpret_cast<const float2 *>(row + l8 * 2);
      }
    }
  };
  const int step = nw * 8;
  if (threadIdx.x == 0) ZOOMR_SCORE_MARK(10);
  if (warp * 8 < nt) load(warp * 8, kv, kv2);
  for (int base = warp * 8; base < nt; base += step) {
    if (base + step < nt) load(base + step, kn, kn2);
    float acc[2][G];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int hh = 0; hh < G; ++hh) {
        float a = 0.f;
        if constexpr (FPL >= 4) {
#pragma unroll
          for (int m = 0; m < NV; ++m) {
            const float4 qv = *reinterpret_cast<const float4 *>(qs + hh * D + m * 32 + l8 * 4);
            a = fmaf(kv[u][m].x, qv.x, a);
            a = fmaf(kv[u][m].y, qv.y, a);
            a = fmaf(kv[u][m].z, qv.z, a);
            a = fmaf(kv[u][m].w, qv.w, a);
          }
        } else {
          const float2 qv = *reinterpret_cast<const float2 *>(qs + hh * D + l8 * 2);
          a = fmaf(kv2[u].x, qv.x, a);
          a = fmaf(kv2[u].y, qv.y, a);
        }
        a += __shfl_xor_sync(0xffffffffu, a, 4);
        a += __shfl_xor_sync(0xffffffffu, a, 2);
        a += __shfl_xor_sync(0xffffffffu, a, 1);
        acc[u][hh] = a;
      }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = base + u * 4 + oct;
      if (i < nt) {
#pragma unroll
        for (int hh = 0; hh < G; ++hh)
          if (l8 == hh) {
            al[hh * ald + i] = acc[u][hh];
            if (alpha_out) alpha_out[hh * ald_out + i] = acc[u][hh];
          }
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
#pragma unroll
      for (int m = 0; m < NV; ++m) kv[u][m] = kn[u][m];
      kv2[u] = kn2[u];
    }
  }
  if (lane == 0) ZOOMR_SCORE_MARK(9);
  __syncthreads();
  const int kk = top_k < nt ? top_k : nt;
  for (int hh = warp; hh < G; hh += nw) {
    float *a = al + hh * ald;
    for (int r = 0; r < kk; ++r) {
      float ba = -INFINITY;
      int bi = 0x7fffffff;
      for (int i = lane; i < nt; i += 32) {
        const float x = a[i];
        if (better_alpha(x, i, ba, bi)) { ba = x; bi = i; }
      }
#pragma unroll
      for (int off = 16; off; off >>= 1) {
        const float oa = __shfl_xor_sync(0xffffffffu, ba, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (better_alpha(oa, oi, ba, bi)) { ba = oa; bi = oi; }
      }
      if (lane == 0) {
        sel_i[hh * top_k + r] = bi;
        sel_a[hh * top_k + r] = ba;
        a[bi] = -INFINITY;  // exclude from the next round
      }
      __syncwarp();
    }
  }
  __syncthreads();
}

// per-voter top-k over al (smem) for the G voters of the block: warp hh < G
__device__ __forceinline__ void block_topk_voters(int G, float *al, int ald, int nt, int top_k, int *sel_i,
                                                  float *sel_a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int kk = top_k < nt ? top_k : nt;
  for (int hh = warp; hh < G; hh += nw) {
    float *a = al + hh * ald;
    for (int r = 0; r < kk; ++r) {
      float ba = -INFINITY;
      int bi = 0x7fffffff;
      for (int i = lane; i < nt; i += 32) {
        const float x = a[i];
        if (better_alpha(x, i, ba, bi)) { ba = x; bi = i; }
      }
#pragma unroll
      for (int off = 16; off; off >>= 1) {
        const float oa = __shfl_xor_sync(0xffffffffu, ba, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (better_alpha(oa, oi, ba, bi)) { ba = oa; bi = oi; }
      }
      if (lane == 0) {
        sel_i[hh * top_k + r] = bi;
        sel_a[hh * top_k + r] = ba;
        a[bi] = -INFINITY;  // exclude from the next round
      }
      __syncwarp();
    }
  }
}


// ---------------------------------------------------------------- a3 -----
// Global consensus over one sequence's (v, A), all in shared memory:
// flags fl[i] = 2 (I_c), 1 (I_s = I_all \ I_c), 0 (unvoted).  Exact integer work:
//  1. histogram of votes (bin = min(v, kHistBins-1), monotone in v);
//  2. the threshold bin b* where the count of voted entries at or above it
//     first reaches c (suffix scan); entries above b* are in I_c;
//  3. the tie group at b* is ranked by the full key (v desc, A desc, i asc) and
//     its first c - n_above members join I_c.
// Returns nothing; *ag (if non-null, thread 0) = sum_{I_c} v / sum_{I_all} v.
// small c (every BASELINE config but the stress sweep's c = 32), large N_t:
//  1. the c largest VOTE COUNTS, one occurrence per round: c rounds of a
//     block max over 32-bit votes (redux.sync per warp, one barrier per
//     round) -> the threshold v* = the c-th largest vote, n_above = #{v > v*};
//  2. the tie group {v == v*} is ranked by the rest of the key (A desc, i asc)
//     and its first c - n_above members join I_c.
// O(c + m^2 / T) per thread (m = tie-group size, usually small) instead of the
// O(N_t) compares per entry of direct ranking (~5 us at N_t = 240 on one CTA).
// A function of its own, so that block_topc's common path stays compact.
static __device__ __noinline__ void block_topc_rounds(const int *v, const long long *A, int nt, int c, uint8_t *fl,
                                                      int *hist, int *grp, int *scratch, float *ag) {
  const int T = blockDim.x, tid = threadIdx.x;
  int *wm = hist;  // [2][32] warp maxima (double-buffered: one barrier per round)
  const int lane = tid & 31, warp = tid >> 5, nw = (T + 31) >> 5;
  unsigned removed = 0;
  int sv = 0, vstar = 0, got = 0;
  for (int j = 0, i = tid; i < nt; ++j, i += T) {
    const int vi = v[i];
    fl[i] = vi > 0 ? 1 : 0;
    sv += vi > 0 ? vi : 0;
  }
  for (int r = 0; r < c; ++r) {
    int lm = 0, lj = -1;
    for (int j = 0, i = tid; i < nt; ++j, i += T) {
      const int vi = v[i];
      if (vi > lm && !(removed >> j & 1u)) {
        lm = vi;
        lj = j;
      }
    }
    const int wmax = __reduce_max_sync(0xffffffffu, lm);
    int *buf = wm + (r & 1) * 32;
    if (lane == 0) buf[warp] = wmax;
    __syncthreads();
    int gmax = 0, ow = 0;
    for (int w = 0; w < nw; ++w) {
      const int x = buf[w];
      if (x > gmax) {
        gmax = x;
        ow = w;
      }
    }
    if (gmax == 0) break;  // fewer than c voted summaries: all of them are in I_c (uniform)
    if (warp == ow) {      // one occurrence of gmax leaves: the lowest lane of the first warp holding it
      const unsigned m = __ballot_sync(0xffffffffu, lm == gmax);
      if (lane == __ffs(m) - 1) removed |= 1u << lj;
    }
    vstar = gmax;
    ++got;
  }
  // I_c = {v > v*} + the first (c - n_above) of {v == v*} by (A desc, i asc);
  // got < c means every voted entry fits (v* = smallest voted vote, all join)
  if (tid == 0) {
    scratch[34] = 0;  // tie-group size
    scratch[35] = 0;  // sum v over I_c
    scratch[36] = 0;  // sum v over I_all
    scratch[37] = 0;  // n_above
  }
  __syncthreads();
  int above = 0;
  for (int i = tid; i < nt; i += T) {
    const int vi = v[i];
    if (vi <= 0 || got == 0) continue;
    if (got < c || vi > vstar) {
      fl[i] = 2;
      ++above;
    } else if (vi == vstar) {
      grp[atomicAdd(&scratch[34], 1)] = i;
    }
  }
  if (above) atomicAdd(&scratch[37], above);
  __syncthreads();
  const int m = scratch[34], need = c - scratch[37];
  for (int x = tid; x < m && need > 0; x += T) {
    const int i = grp[x];
    const long long ai = A[i];
    int rk = 0;
    for (int y = 0; y < m; ++y) {
      const int jj = grp[y];
      const long long aj = A[jj];
      rk += (aj > ai) | ((aj == ai) & (jj < i));
    }
    if (rk < need) fl[i] = 2;
  }
  __syncthreads();
  if (ag) {
    int sc_ = 0;
    for (int i = tid; i < nt; i += T)
      if (fl[i] == 2) sc_ += v[i];
    if (sc_) atomicAdd(&scratch[35], sc_);
    if (sv) atomicAdd(&scratch[36], sv);
    __syncthreads();
    if (tid == 0) *ag = scratch[36] > 0 ? (float)((double)scratch[35] / (double)scratch[36]) : 0.f;
    __syncthreads();
  }
}

// __noinline__: the fused select's tail CTA runs it once on dummy data first, and the
// real call must then execute the very same (now cached) instructions
static __device__ __noinline__ void block_topc(const int *v, const long long *A, int nt, int c, uint8_t *fl,
                           int *hist /* smem [kHistBins] */, int *grp /* smem [nt] */,
                           int *scratch /* smem >= 40 ints */, float *ag) {
  const int T = blockDim.x, tid = threadIdx.x;
  if (c <= kTopcRounds && nt > kTopcRoundsMinN && nt <= 32 * T) {
    block_topc_rounds(v, A, nt, c, fl, hist, grp, scratch, ag);
    return;
  }
  if (nt <= T) {
    // small N_t: every voted entry's rank in the full order by direct counting
    // over a packed 128-bit key: hi = v<<44 | (A+2^63)>>20, lo = low 20 bits of
    // (A+2^63) <<44 | (2^20-1-i): one branch-free compare chain per pair.
    unsigned long long *kh = reinterpret_cast<unsigned long long *>(hist);  // 16 B/entry, nt <= 512
    if (tid == 0) {
      scratch[35] = 0;
      scratch[36] = 0;
    }
    if (tid < nt) {
      const unsigned long long ab = (unsigned long long)A[tid] ^ 0x8000000000000000ull;  // order-preserving
      kh[2 * tid] = ((unsigned long long)(unsigned)max(v[tid], 0) << 44) | (ab >> 20);
      kh[2 * tid + 1] = ((ab & 0xfffffull) << 44) | (unsigned long long)(0xfffff - tid);
    }
    __syncthreads();
    if (tid < nt) {
      const int vi = v[tid];
      uint8_t f = 0;
      if (vi > 0) {
        const unsigned long long hi = kh[2 * tid], lo = kh[2 * tid + 1];
        int r = 0;
#pragma unroll 8
        for (int j = 0; j < nt; ++j) {
          const ulonglong2 kj = reinterpret_cast<const ulonglong2 *>(kh)[j];
          r += (kj.x > hi) | ((kj.x == hi) & (kj.y > lo));
        }
        f = r < c ? 2 : 1;
        if (ag) {
          atomicAdd(&scratch[36], vi);
          if (f == 2) atomicAdd(&scratch[35], vi);
        }
      }
      fl[tid] = f;
    }
    __syncthreads();
    if (ag && tid == 0) *ag = scratch[36] > 0 ? (float)((double)scratch[35] / (double)scratch[36]) : 0.f;
    return;
  }
  for (int x = tid; x < kHistBins; x += T) hist[x] = 0;
  if (tid == 0) {
    scratch[34] = 0;  // group size
    scratch[35] = 0;  // sum v over I_c
    scratch[36] = 0;  // sum v over I_all
  }
  __syncthreads();
  for (int i = tid; i < nt; i += T)
    if (v[i] > 0) atomicAdd(&hist[min(v[i], kHistBins - 1)], 1);
  __syncthreads();
  // suffix scan: thread t owns bins [kHistBins - (t+1)*per, kHistBins - t*per), highest first
  const int per = (kHistBins + T - 1) / T;
  const int hi = kHistBins - tid * per, lo = max(0, hi - per);
  int mine = 0;
  for (int x = lo; x < hi; ++x) mine += hist[x];
  int total;
  const int above = block_excl_scan(mine, scratch, &total);  // voted entries in bins >= hi
  if (tid == 0) {
    scratch[32] = (c == 0) ? kHistBins : 0;  // b*: c = 0 -> nothing zoomed; c >= |I_all| -> all
    scratch[33] = (c == 0) ? 0 : total;      // n_above
  }
  __syncthreads();
  if (c > 0 && total > c) {
    int run = above;
    for (int x = hi - 1; x >= lo; --x) {
      const int h = hist[x];
      if (run < c && run + h >= c) {  // unique crossing bin
        scratch[32] = x;
        scratch[33] = run;
      }
      run += h;
    }
  }
  __syncthreads();
  const int bstar = scratch[32], need = c - scratch[33];
  for (int i = tid; i < nt; i += T) {
    const int vi = v[i];
    const int bin = min(vi, kHistBins - 1);
    uint8_t f = 0;
    if (vi > 0) {
      f = 1;
      if (bin > bstar || (bstar == 0)) f = 2;  // bstar 0: every voted entry fits in I_c
      else if (bin == bstar) grp[atomicAdd(&scratch[34], 1)] = i;
    }
    fl[i] = f;
  }
  __syncthreads();
  const int m = scratch[34];
  for (int x = tid; x < m; x += T) {
    const int i = grp[x];
    int r = 0;
    for (int y = 0; y < m; ++y) {
      const int j = grp[y];
      r += before_key(v[j], A[j], j, v[i], A[i], i) ? 1 : 0;
    }
    if (r < need) fl[i] = 2;
  }
  __syncthreads();
  if (ag) {
    int sc_ = 0, sa = 0;
    for (int i = tid; i < nt; i += T) {
      if (fl[i] == 2) sc_ += v[i];
      if (v[i] > 0) sa += v[i];
    }
    atomicAdd(&scratch[35], sc_);
    atomicAdd(&scratch[36], sa);
    __syncthreads();
    if (tid == 0) *ag = scratch[36] > 0 ? (float)((double)scratch[35] / (double)scratch[36]) : 0.f;
  }
}

// ---------------------------------------------------------------- a4 -----
// I_f = [0, s') ++ clipped selected pieces in i order ++ [w0, T) for one sequence
// (see zoomr_index.cu).  fl may live in shared or global memory.
// One pass reads the segment table (validation + clipped piece extents into
// shared memory), a block scan turns lengths into offsets, and the fill reads
// only shared memory: coalesced stores (a shuffle search over 32 pieces per warp).
// With `phys` non-null, also writes the page-resolved row of every entry,
// phys[j] = pt[t/P] * HkvP + t%P (HkvP = H_kv*P), so that a5 needs no page-table
// lookup: row(l, g, t) = (l*num_pages*H_kv + g)*P + phys.  `pt` is the sequence's
// page table (shared or global memory).
static __device__ __noinline__ void block_build_index(const int32_t *__restrict__ bd /* [nt][4] */, int nt, int T,
                                         const uint8_t *fl, int sink, int window, int32_t *__restrict__ out,
                                         int cap, int32_t *__restrict__ count_out,
                                         int *piece /* smem [2*nt]: start, then offset */,
                                         int *scratch /* smem >= 33 ints */, int32_t *status,
                                         int32_t *__restrict__ phys = nullptr, const int32_t *pt = nullptr,
                                         int P = 1, int HkvP = 1) {
  auto emit = [&](int j, int t) {
    out[j] = t;
    if (phys) {
      const int lp = t / P;
      phys[j] = pt[lp] * HkvP + (t - lp * P);
    }
  };
  const int tid = threadIdx.x;
  const int sp = sink < T ? sink : T;                  // s'
  const int w0 = (T - window > sp) ? T - window : sp;  // start of the window piece
  const int per = (nt + (int)blockDim.x - 1) / (int)blockDim.x;
  const int i0 = tid * per, i1 = min(nt, i0 + per);
  int local = 0;
  for (int i = i0; i < i1; ++i) {
    const int4 r = *reinterpret_cast<const int4 *>(bd + 4 * i);  // (r0, r1, s0, s1)
    const int nr0 = (i + 1 < nt) ? bd[4 * (i + 1)] : 0x7fffffff;
    if (r.w <= r.z) set_status(status, ZOOMR_ERR_EMPTY_SEGMENT);
    else if (r.x < 0 || r.y < r.x || r.z < r.y || nr0 < r.w) set_status(status, ZOOMR_ERR_SEGMENT_ORDER);
    else if (r.w > T) set_status(status, ZOOMR_ERR_INDEX_RANGE);
    const int f = fl ? fl[i] : 0;
    int a = 0, e = 0;
    if (f == 2) { a = r.x; e = r.y; }        // zoom: R_i
    else if (f == 1) { a = r.z; e = r.w; }   // keep: S_i
    a = max(a, sp);
    const int len = max(0, min(e, w0) - a);
    piece[i] = len > 0 ? a : -1;
    piece[nt + i] = len;  // length for now, offset after the scan
    local += len;
  }
  int total;
  int run = block_excl_scan(local, scratch, &total);
  for (int i = i0; i < i1; ++i) {
    const int len = piece[nt + i];
    piece[nt + i] = run;
    run += len;
  }
  __syncthreads();
  const int count = sp + total + (T - w0);
  if (tid == 0) {
    if (count > cap) set_status(status, ZOOMR_ERR_CAPACITY);
    *count_out = count < cap ? count : cap;
  }
  // Fill, every store coalesced.  Output layout: [0, s') ++ pieces ++ [w0, T).
  // Sink and window: positions strided over the block.  Pieces: warp w takes
  // groups of 32 consecutive pieces (lane l holds piece g0 + l's start and
  // offset); the group's output positions go 32 at a time, one per lane, and a
  // 5-step shuffle search over the lanes' offsets finds the piece of each.
  const int lim = count < cap ? count : cap;
  const int wbase = sp + total;
  for (int j = tid; j < sp && j < lim; j += blockDim.x) emit(j, j);                   // sink
  for (int j = wbase + tid; j < lim; j += blockDim.x) emit(j, w0 + (j - wbase));      // window
  const int lane = tid & 31, warp = tid >> 5, nwarp = ((int)blockDim.x + 31) >> 5;
  const int *off = piece + nt;  // exclusive offsets of the clipped pieces (relative to s')
  const int pend = min(total, lim - sp);  // piece positions [0, pend) are written
  const int Ew = ((pend + nwarp - 1) / nwarp + 127) & ~127;
  const int c1 = min(pend, (warp + 1) * Ew);
  int cur = warp * Ew;
  if (nt > 0 && cur < c1) {
    int bi = 0, hi = nt - 1;  // the window's first piece: last piece with offset <= cur
    while (bi < hi) {
      const int mid = (bi + hi + 1) >> 1;
      if (off[mid] <= cur) bi = mid; else hi = mid - 1;
    }
    while (cur < c1) {
      const int i = bi + lane;
      const int my_off = i < nt ? off[i] : total;
      const int my_start = i < nt ? piece[i] : 0;
      const int wend = min(c1, bi + 32 < nt ? off[bi + 32] : total);
      for (; cur < wend; cur += 128) {  // warp-uniform: 4 positions per lane in flight
        int L[4] = {0, 0, 0, 0};
#pragma unroll
        for (int st = 16; st; st >>= 1) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int o = __shfl_sync(0xffffffffu, my_off, L[u] + st);
            if (o <= cur + 32 * u + lane) L[u] += st;
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int r = cur + 32 * u + lane;
          const int ps = __shfl_sync(0xffffffffu, my_start, L[u]), po = __shfl_sync(0xffffffffu, my_off, L[u]);
          if (r < wend) emit(sp + r, ps + (r - po));
        }
      }
      cur = wend;
      bi += 32;
    }
  }
}

}  // namespace zoomr
