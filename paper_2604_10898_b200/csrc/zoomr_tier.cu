// Host-memory tier (the paper's own system, P:103-109:
// "we offload these initial KVs to CPU memory ... only the subset of the KV
// cache specified by the index set" is loaded per step).
//
// B200 design: the full cache lives in pinned host memory (mapped, so kernels
// read it over PCIe / C2C through its unified address); HBM holds a HOT POOL
// of pages that caches it.  Per step, after I_f is known:
//   zoomr_tier_fetch = plan (one CTA: which logical pages I_f touches, which
//   of them are not resident, least-recently-used victims among the pages
//   this step does not touch) + copy (all SMs: the missing pages, every layer,
//   K and V, host -> hot pool), then a5 runs on the hot pool.
// Because I_f changes little from step to step (the window advances one token,
// zoomed segments change at semantic boundaries), the steady-state transfer is
// the pages that ENTERED I_f, not I_f itself (the paper reloads I_f per layer).
#include "common.cuh"

namespace zoomr {

constexpr int kPlanThreads = 1024;
constexpr int kPlanSmemNP = 4096;  // hot-page-table entries (B * max_pages * R) kept in shared memory

__device__ __forceinline__ int tier_block_scan(int x, int *wsum, int *total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int v = wsum[lane];
    int vi = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, vi, o);
      if (lane >= o) vi += y;
    }
    wsum[lane] = vi - v;
    if (lane == 31) wsum[32] = vi;
  }
  __syncthreads();
  const int r = wsum[warp] + incl - x;
  *total = wsum[32];
  __syncthreads();
  return r;
}

// Hot pages may be smaller than host pages: Ph = P / R tokens.  Hot logical page
// x = b*hmp + lph (hmp = max_pages * R) holds tokens [lph*Ph, (lph+1)*Ph) of
// sequence b: sub-page lph % R of host page host_pt[b][lph / R].
// ws layout (int32): [0] step counter, [1] n_fetch, then need[B*hmp] (as int32),
// missing[hot_pages], fetch_hot[hot_pages], fetch_host[hot_pages] (= host page * R + sub-page)
__global__ void __launch_bounds__(kPlanThreads) tier_plan_kernel(
    int32_t B, const int32_t *__restrict__ index, const int32_t *__restrict__ count, int32_t cap, int32_t Ph,
    int32_t R, int32_t max_pages, const int32_t *__restrict__ host_pt, int32_t *__restrict__ hot_pt,
    int32_t *__restrict__ owner, int32_t *__restrict__ stamp, int32_t hot_pages, int32_t *__restrict__ ws,
    int32_t *status, const int32_t *__restrict__ seq_len) {
  __shared__ int wsum[33];
  __shared__ int hist[256];
  __shared__ unsigned long long s_prefix;
  __shared__ int s_need;
  extern __shared__ int plan_smem[];  // [NP] need, [NP] hot page table (when NP <= kPlanSmemNP)
  // launched with PDL behind the select: the copy kernel may launch now (it waits
  // for this plan), and I_f / its count are read only after the select completed
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int tid = threadIdx.x;
  const int hmp = max_pages * R;
  const int NP = B * hmp;
  int32_t *missing = ws + 2 + NP, *fetch_hot = missing + hot_pages, *fetch_host = fetch_hot + hot_pages;
  // The page marks and a snapshot of the hot page table live in shared memory when
  // they fit; both are set up before the wait (the select writes neither, and the
  // previous step's plan / copy have completed), so after the wait the plan costs
  // the I_f load and nothing else until the block scan.
  const bool in_smem = NP <= kPlanSmemNP;
  int32_t *need = in_smem ? plan_smem : ws + 2;
  const int32_t *hpt = in_smem ? plan_smem + NP : hot_pt;
  for (int x = tid; x < NP; x += kPlanThreads) {
    need[x] = 0;
    if (in_smem) plan_smem[NP + x] = hot_pt[x];
  }
  const int step = ws[0] + 1;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // 1. pages touched by I_f
  __syncthreads();
  for (int b = 0; b < B; ++b) {
    int n = count[b];
    n = n < cap ? n : cap;
    for (int i = tid; i < n; i += kPlanThreads) {
      const int t = index[(int64_t)b * cap + i];
      const int lp = t / Ph;
      if (t < 0 || lp >= hmp) set_status(status, ZOOMR_ERR_INDEX_RANGE);
      else need[b * hmp + lp] = 1;
    }
  }
  __syncthreads();
  // look-ahead: the page of position T (the next token's) is made resident now, so
  // that in the next step every sink / window page is resident before that step's
  // plan runs -- its a5 may then read their page entries before its wait.  When T
  // starts the page, none of its rows exists yet: it is allocated without a copy
  // (mark 2; the appends write its rows one by one) -- else it would be a page of
  // rows from the host copied every Ph tokens for nothing
  if (seq_len)
    for (int b = tid; b < B; b += kPlanThreads) {
      const int T = seq_len[b], lp = T / Ph;
      if (T >= 0 && lp < hmp) {
        if (T % Ph == 0) atomicCAS(&need[b * hmp + lp], 0, 2);
        else need[b * hmp + lp] = 1;
      }
    }
  __syncthreads();
  // 2. resident ones are stamped with this step; the others are missing (in page order)
  int nmiss = 0;
  for (int x0 = 0; x0 < NP; x0 += kPlanThreads) {
    const int x = x0 + tid;
    bool miss = false;
    if (x < NP && need[x]) {
      const int h = hpt[x];
      if (h >= 0 && h < hot_pages) stamp[h] = step;
      else miss = true;
    }
    int tot;
    const int off = tier_block_scan(miss ? 1 : 0, wsum, &tot);
    if (miss && nmiss + off < hot_pages) missing[nmiss + off] = x;
    nmiss += tot;
  }
  __syncthreads();  // the stamps above are visible to the victim search
  // 3. victims: the nmiss least recently used hot pages this step does not touch
  //    (free pages have stamp -1); key (stamp + 1, page) -- unique
  int ncand = 0;
  for (int h0 = 0; h0 < hot_pages && nmiss > 0; h0 += kPlanThreads) {  // (warm step: nothing missing, no search)
    const int h = h0 + tid;
    int tot;
    tier_block_scan((h < hot_pages && stamp[h] < step) ? 1 : 0, wsum, &tot);
    ncand += tot;
  }
  if (nmiss > ncand) {  // the hot pool cannot hold this step's I_f
    if (tid == 0) set_status(status, ZOOMR_ERR_CAPACITY);
    nmiss = ncand;
  }
  unsigned long long thr = ~0ull;  // victims: candidate keys <= thr
  if (nmiss > 0 && nmiss < ncand) {  // radix select of the nmiss-th smallest key, MSB first
    if (tid == 0) {
      s_prefix = 0ull;
      s_need = nmiss;
    }
    unsigned long long mask = 0ull;
    for (int pass = 0; pass < 8; ++pass) {
      const int shift = 56 - 8 * pass;
      if (tid < 256) hist[tid] = 0;
      __syncthreads();
      const unsigned long long prefix = s_prefix;
      for (int h = tid; h < hot_pages; h += kPlanThreads) {
        if (stamp[h] >= step) continue;
        const unsigned long long k = ((unsigned long long)(uint32_t)(stamp[h] + 1) << 32) | (uint32_t)h;
        if ((k & mask) == prefix) atomicAdd(&hist[(k >> shift) & 255], 1);
      }
      __syncthreads();
      if (tid < 32) {  // digit d with below(d) < need <= below(d) + hist[d] (ascending)
        const int lane = tid;
        int hh[8], sum = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          hh[j] = hist[8 * lane + j];
          sum += hh[j];
        }
        int incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        const int need_ = s_need;
        int below = incl - sum, found = -1, nbelow = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (found < 0 && below < need_ && need_ <= below + hh[j]) {
            found = 8 * lane + j;
            nbelow = below;
          }
          below += hh[j];
        }
        const unsigned bal = __ballot_sync(0xffffffffu, found >= 0);
        const int src = __ffs(bal) - 1;
        found = __shfl_sync(0xffffffffu, found, src);
        nbelow = __shfl_sync(0xffffffffu, nbelow, src);
        if (lane == 0) {
          s_prefix = prefix | ((unsigned long long)found << shift);
          s_need = need_ - nbelow;
        }
      }
      mask |= 0xffull << shift;
      __syncthreads();
    }
    thr = s_prefix;
  }
  // 4. victims in page order take the missing pages in page order
  int nv = 0;
  for (int h0 = 0; h0 < hot_pages && nmiss > 0; h0 += kPlanThreads) {
    const int h = h0 + tid;
    bool v = false;
    if (h < hot_pages && stamp[h] < step) {
      const unsigned long long k = ((unsigned long long)(uint32_t)(stamp[h] + 1) << 32) | (uint32_t)h;
      v = k <= thr;
    }
    int tot;
    const int j = nv + tier_block_scan(v ? 1 : 0, wsum, &tot);
    if (v && j < nmiss) {
      const int x = missing[j];
      const int old = owner[h];
      if (old >= 0 && old < NP) hot_pt[old] = -1;  // evicted (not needed this step)
      owner[h] = x;
      hot_pt[x] = h;
      stamp[h] = step;
      const int xb = x / hmp, lph = x - xb * hmp;
      const int hp = host_pt[xb * max_pages + lph / R];
      fetch_hot[j] = h;
      fetch_host[j] = hp < 0 ? -1 : need[x] == 2 ? -2 : hp * R + lph % R;  // -2: allocate only (no copy)
      if (hp < 0) set_status(status, ZOOMR_ERR_INDEX_RANGE);
    }
    nv += tot;
  }
  if (tid == 0) {
    ws[0] = step;
    ws[1] = nmiss;
  }
}

// all SMs: work item w = (fetch j, layer l, K or V) copies, for every KV head g,
// the Ph*d block of sub-page (fetch_host[j] % R) of host page fetch_host[j] / R
// to hot page fetch_hot[j]
__global__ void __launch_bounds__(256) tier_copy_kernel(const uint4 *__restrict__ host_k,
                                                         const uint4 *__restrict__ host_v, int64_t host_pages,
                                                         uint4 *__restrict__ hot_k, uint4 *__restrict__ hot_v,
                                                         int64_t hot_pages, int32_t L, int32_t Hkv, int32_t R,
                                                         int32_t row16, const int32_t *__restrict__ ws, int32_t NP) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // a5 may launch (it waits for this copy)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int nf = ws[1];
  const int32_t *fetch_hot = ws + 2 + NP + hot_pages, *fetch_host = fetch_hot + hot_pages;
  const int64_t items = (int64_t)nf * L * 2;
  for (int64_t w = blockIdx.x; w < items; w += gridDim.x) {
    const int kv = (int)(w & 1);
    const int64_t jl = w >> 1;
    const int j = (int)(jl / L), l = (int)(jl - (int64_t)j * L);
    const int hs = fetch_host[j], hh = fetch_hot[j];
    const int hp = hs < 0 ? -1 : hs / R, sub = hs < 0 ? 0 : hs - hp * R;
    if (hp < 0 || hp >= host_pages) continue;
    // host block of (l, hp, g): R*row16 uint4; this sub-page: row16 of them at sub*row16
    const uint4 *src = (kv ? host_v : host_k) + ((int64_t)l * host_pages + hp) * Hkv * R * row16 + sub * row16;
    uint4 *dst = (kv ? hot_v : hot_k) + ((int64_t)l * hot_pages + hh) * Hkv * row16;
    const int n16 = Hkv * row16;
    int e = threadIdx.x;
    for (; e + 3 * 256 < n16; e += 4 * 256) {  // four 16-byte host reads in flight per thread
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int x = e + u * 256, g = x / row16;
        v[u] = __ldcs(src + (int64_t)g * R * row16 + (x - g * row16));
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) dst[e + u * 256] = v[u];
    }
    for (; e < n16; e += 256) {
      const int g = e / row16;
      dst[e] = __ldcs(src + (int64_t)g * R * row16 + (e - g * row16));
    }
  }
}

// The paper's own transfer unit: the rows of I_f of one group of
// layers, gathered from the host cache into an HBM slice laid out as a small
// pool [layer_count][B * spp][H_kv][Ps][d]: row j of sequence b sits in slice
// page b * spp + j / Ps, slot j % Ps (spp = slice pages per sequence).  Work
// item = (layer, sequence, 8 consecutive rows of I_f, K or V); a warp moves one
// (row, head) run of 2*d bytes per 16-byte lane group, four host reads in
// flight per thread.  Launched with PDL: the index is read after the wait.
constexpr int kSliceRows = 8;
__global__ void __launch_bounds__(256) tier_gather_slice_kernel(
    const __nv_bfloat16 *__restrict__ host_k, const __nv_bfloat16 *__restrict__ host_v, int64_t host_pages,
    const int32_t *__restrict__ page_table, int32_t max_pages, const int32_t *__restrict__ index,
    const int32_t *__restrict__ count, int32_t cap, int32_t B, int32_t L, int32_t Hkv, int32_t P, int32_t D,
    int32_t l0, int32_t Lc, __nv_bfloat16 *__restrict__ slice_k, __nv_bfloat16 *__restrict__ slice_v, int32_t Ps,
    int32_t spp, int32_t *status) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int c16 = D / 8;                  // 16-byte chunks of one (row, head)
  const int per_item = kSliceRows * Hkv * c16;
  const int64_t blocks_per_seq = (cap + kSliceRows - 1) / kSliceRows;
  const int64_t items = (int64_t)Lc * B * blocks_per_seq * 2;
  for (int64_t w = blockIdx.x; w < items; w += gridDim.x) {
    const int kv = (int)(w & 1);
    int64_t r = w >> 1;
    const int64_t blk = r % blocks_per_seq;
    r /= blocks_per_seq;
    const int b = (int)(r % B), ll = (int)(r / B), l = l0 + ll;
    int n = count[b];
    n = n < cap ? n : cap;
    const int j0 = (int)blk * kSliceRows;
    if (j0 >= n) continue;
    const __nv_bfloat16 *src = kv ? host_v : host_k;
    __nv_bfloat16 *dst = kv ? slice_v : slice_k;
    for (int e0 = threadIdx.x; e0 < per_item; e0 += 4 * 256) {
      uint4 val[4];
      int64_t dsto[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + u * 256;
        dsto[u] = -1;
        if (e >= per_item) continue;
        const int c = e % c16, gh = (e / c16) % Hkv, jr = e / (c16 * Hkv);
        const int j = j0 + jr;
        if (j >= n) continue;
        const int t = index[(int64_t)b * cap + j];
        const int lp = t / P;
        const int page = (t >= 0 && lp < max_pages) ? page_table[(int64_t)b * max_pages + lp] : -1;
        if (page < 0 || page >= host_pages) {
          set_status(status, ZOOMR_ERR_INDEX_RANGE);
          continue;
        }
        const int64_t so = ((((int64_t)l * host_pages + page) * Hkv + gh) * P + (t - lp * P)) * D + c * 8;
        val[u] = __ldcs(reinterpret_cast<const uint4 *>(src + so));
        const int sp = b * spp + j / Ps;
        dsto[u] = ((((int64_t)ll * B * spp + sp) * Hkv + gh) * Ps + (j % Ps)) * D + c * 8;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (dsto[u] >= 0) *reinterpret_cast<uint4 *>(dst + dsto[u]) = val[u];
    }
  }
}

}  // namespace zoomr

using namespace zoomr;

extern "C" int zoomr_tier_gather_slice(const zoomr_geom *geom, int32_t batch, const zoomr_kv *host_kv,
                                       const int32_t *index, const int32_t *index_count, int32_t index_capacity,
                                       int32_t layer_begin, int32_t layer_count, void *slice_k, void *slice_v,
                                       int32_t slice_page_size, int32_t slice_pages_per_seq, int32_t *dev_status,
                                       void *stream) {
  int rc = check_geom(geom);
  if (rc) return rc;
  if (batch < 1 || !host_kv || !host_kv->k || !host_kv->v || !host_kv->page_table || host_kv->num_pages < 1 ||
      host_kv->max_pages < 1 || !index || !index_count || index_capacity < 1 || !slice_k || !slice_v ||
      slice_page_size < 1 || layer_begin < 0 || layer_count < 1 || layer_begin + layer_count > geom->num_layers)
    return ZOOMR_ERR_INVALID_ARG;
  if ((int64_t)slice_page_size * slice_pages_per_seq < index_capacity) return ZOOMR_ERR_INVALID_ARG;
  if (geom->head_dim % 8) return ZOOMR_ERR_UNSUPPORTED;
  cudaStream_t s = (cudaStream_t)stream;
  launch_pdl(tier_gather_slice_kernel, 4 * num_sms(), 256, 0, s, (const __nv_bfloat16 *)host_kv->k,
             (const __nv_bfloat16 *)host_kv->v, (int64_t)host_kv->num_pages, host_kv->page_table, host_kv->max_pages,
             index, index_count, index_capacity, batch, geom->num_layers, geom->num_kv_heads, geom->page_size,
             geom->head_dim, layer_begin, layer_count, (__nv_bfloat16 *)slice_k, (__nv_bfloat16 *)slice_v,
             slice_page_size, slice_pages_per_seq, dev_status);
  return launch_status(s);
}

extern "C" size_t zoomr_tier_workspace_bytes(int32_t batch, int32_t hot_max_pages, int32_t hot_pages) {
  if (batch < 1 || hot_max_pages < 1 || hot_pages < 1) return 0;
  return sizeof(int32_t) * (2 + (size_t)batch * hot_max_pages + 3 * (size_t)hot_pages);
}

extern "C" int zoomr_tier_fetch(const zoomr_geom *geom, int32_t batch, const zoomr_kv *host_kv, void *hot_k,
                                void *hot_v, int32_t hot_pages, int32_t hot_page_size, int32_t *hot_page_table,
                                int32_t *hot_owner,
                                int32_t *hot_stamp, const int32_t *index, const int32_t *index_count,
                                int32_t index_capacity, const int32_t *seq_len, void *workspace,
                                size_t workspace_bytes, int32_t *dev_status, void *stream) {
  int rc = check_geom(geom);
  if (rc) return rc;
  if (batch < 1 || !host_kv || !host_kv->k || !host_kv->v || !host_kv->page_table || host_kv->num_pages < 1 ||
      host_kv->max_pages < 1 || !hot_k || !hot_v || hot_pages < 1 || !hot_page_table || !hot_owner || !hot_stamp ||
      !index || !index_count || index_capacity < 1 || !workspace)
    return ZOOMR_ERR_INVALID_ARG;
  const int P = geom->page_size, Ph = hot_page_size;
  if (Ph < 1 || P % Ph) return ZOOMR_ERR_INVALID_ARG;
  const int R = P / Ph;
  const int64_t hmp = (int64_t)host_kv->max_pages * R;
  if (hmp * batch > 0x7fffffff || (int64_t)host_kv->num_pages * R > 0x7fffffff) return ZOOMR_ERR_UNSUPPORTED;
  if (workspace_bytes < zoomr_tier_workspace_bytes(batch, (int32_t)hmp, hot_pages)) return ZOOMR_ERR_WORKSPACE;
  const int64_t row = (int64_t)Ph * geom->head_dim * 2;  // bytes of one (page, layer, head) block of the hot pool
  if (row % 16) return ZOOMR_ERR_UNSUPPORTED;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t plan_smem = batch * hmp <= kPlanSmemNP ? (size_t)2 * batch * hmp * sizeof(int32_t) : 0;
  launch_pdl(tier_plan_kernel, 1, kPlanThreads, plan_smem, s, batch, index, index_count, index_capacity, Ph, R,
             host_kv->max_pages, host_kv->page_table, hot_page_table, hot_owner, hot_stamp, hot_pages,
             (int32_t *)workspace, dev_status, seq_len);
  rc = launch_status(s);
  if (rc) return rc;
  launch_pdl(tier_copy_kernel, 2 * num_sms(), 256, 0, s, (const uint4 *)host_kv->k, (const uint4 *)host_kv->v,
             (int64_t)host_kv->num_pages, (uint4 *)hot_k, (uint4 *)hot_v, (int64_t)hot_pages, geom->num_layers,
             geom->num_kv_heads, R, (int32_t)(row / 16), (const int32_t *)workspace, (int32_t)(batch * hmp));
  return launch_status((cudaStream_t)stream);
}
