// H2O, the paper's heavy-hitter comparison policy (P:186 / P:240, SURVEY 8(f)
// NEXT-3; the scoring rule is SPEC h2o_step S:349-357 -- the paper only cites
// the method), on the same kernels as ZoomR:
//
//  * a5 with its logits (zoomr_sparse_decode_attn_logits) attends over the
//    retained set and writes s_j = q . k_j * scale for every (l, h, j);
//  * zoomr_h2o_accumulate: the attention each retained token received this
//    step, averaged over layers and heads, w_j = mean_{l,h} exp(s_j - lse),
//    is added to its cumulative score;
//  * zoomr_h2o_select: the next retained set = sink u window u the
//    budget - |sink u window| previously retained tokens outside them with the
//    largest cumulative score (ties -> smaller position).
#include "common.cuh"

namespace zoomr {

// one CTA per (16 index positions, b): thread (i = tid % 16, grp = tid / 16)
// sums the (l, h) pairs grp, grp + 64, ... (4 loads in flight); the 64 group
// sums are added in group order (deterministic).  16 positions per CTA: enough
// CTAs to cover the SMs at a budget of a few thousand tokens, 64-byte rows.
constexpr int kAccTok = 16, kAccGrp = 64;
__global__ void __launch_bounds__(kAccTok * kAccGrp) h2o_accumulate_kernel(
    const int32_t *__restrict__ index, const int32_t *__restrict__ count, int32_t cap, int32_t LH,
    const float *__restrict__ logits, const float *__restrict__ lse, float *__restrict__ score, int32_t stride,
    int32_t *__restrict__ index_copy, int32_t *__restrict__ count_copy, int32_t *status) {
  __shared__ float red[kAccGrp][kAccTok + 1];
  const int b = blockIdx.y, ti = threadIdx.x % kAccTok, grp = threadIdx.x / kAccTok;
  int n = count[b];
  n = n < cap ? n : cap;
  const int i = blockIdx.x * kAccTok + ti;
  float acc = 0.f;
  if (i < n) {
    const float *lg = logits + (int64_t)b * LH * cap + i;
    const float *ls = lse + (int64_t)b * LH;
    int lh = grp;
    for (; lh + 3 * kAccGrp < LH; lh += 4 * kAccGrp) {
      const float x0 = lg[(int64_t)lh * cap], x1 = lg[(int64_t)(lh + kAccGrp) * cap];
      const float x2 = lg[(int64_t)(lh + 2 * kAccGrp) * cap], x3 = lg[(int64_t)(lh + 3 * kAccGrp) * cap];
      const float y0 = ls[lh], y1 = ls[lh + kAccGrp], y2 = ls[lh + 2 * kAccGrp], y3 = ls[lh + 3 * kAccGrp];
      acc += expf(x0 - y0);
      acc += expf(x1 - y1);
      acc += expf(x2 - y2);
      acc += expf(x3 - y3);
    }
    for (; lh < LH; lh += kAccGrp) acc += expf(lg[(int64_t)lh * cap] - ls[lh]);
  }
  red[grp][ti] = acc;
  __syncthreads();
  if (grp == 0 && i < n) {
    float w = 0.f;
    for (int g2 = 0; g2 < kAccGrp; ++g2) w += red[g2][ti];
    const int t = index[(int64_t)b * cap + i];
    if (t < 0 || t >= stride) set_status(status, ZOOMR_ERR_INDEX_RANGE);
    else score[(int64_t)b * stride + t] += w / (float)LH;
    if (index_copy) index_copy[(int64_t)b * cap + i] = t;
  }
  if (count_copy && blockIdx.x == 0 && threadIdx.x == 0) count_copy[b] = n;
}

// order-preserving key: larger = kept first; cumulative score desc, then position asc
__device__ __forceinline__ uint64_t h2o_key(float sc, int t) {
  uint32_t u = __float_as_uint(sc);
  u ^= (u >> 31) ? 0xffffffffu : 0x80000000u;
  return ((uint64_t)u << 32) | (uint64_t)(0xffffffffu - (uint32_t)t);
}

constexpr int kSelThreads = 1024;
constexpr int kPer = 16;
constexpr int kMaxCand = kSelThreads * kPer;  // previously retained tokens per sequence held in shared memory

// block-wide exclusive scan of one int per thread; returns this thread's offset,
// *total = the block sum.  wsum: 32 ints of shared memory.
__device__ __forceinline__ int block_excl_scan(int x, int *wsum, int *total) {
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
  __syncthreads();  // wsum reusable
  return r;
}

__global__ void __launch_bounds__(kSelThreads) h2o_select_kernel(
    const int32_t *__restrict__ prev_index, const int32_t *__restrict__ prev_count, int32_t cap,
    const float *__restrict__ score, int32_t stride, const int32_t *__restrict__ seq_len, int32_t sink,
    int32_t window, int32_t budget, int32_t *__restrict__ index, int32_t *__restrict__ index_count,
    int32_t *status) {
  extern __shared__ __align__(16) unsigned char sm[];
  uint64_t *key = reinterpret_cast<uint64_t *>(sm);              // [kMaxCand]
  int32_t *cand = reinterpret_cast<int32_t *>(key + kMaxCand);   // [kMaxCand]
  __shared__ int wsum[33];
  __shared__ int hist[256];
  __shared__ unsigned long long s_prefix;
  __shared__ int s_need;
  allow_dependents();  // a5 (PDL) may start its prologue; it waits for our completion before reading I
  const int b = blockIdx.x, tid = threadIdx.x;
  const int T = seq_len[b];
  const int sp = min(sink, T), w0 = max(sp, T - window);
  const int nfixed = sp + (T - w0);
  const int K = max(0, budget - nfixed);
  int np = prev_count[b];
  np = np < cap ? np : cap;
  // 1. candidates: previously retained positions in [s', w0), order kept; thread
  // tid takes the contiguous run [tid*per, (tid+1)*per) (all loads in flight)
  if (np > kSelThreads * kPer) {
    if (tid == 0) set_status(status, ZOOMR_ERR_UNSUPPORTED);
    np = kSelThreads * kPer;
  }
  const int per = (np + kSelThreads - 1) / kSelThreads;
  int tv[kPer];
  float sv[kPer];
  unsigned cm = 0;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int i = tid * per + j;
    tv[j] = (j < per && i < np) ? prev_index[(int64_t)b * cap + i] : -1;
  }
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const bool c = tv[j] >= sp && tv[j] < w0;
    sv[j] = 0.f;
    if (c) {
      if (tv[j] >= stride) set_status(status, ZOOMR_ERR_INDEX_RANGE);
      else {
        sv[j] = score[(int64_t)b * stride + tv[j]];
        cm |= 1u << j;
      }
    }
  }
  int nc;
  {
    int off = block_excl_scan(__popc(cm), wsum, &nc);
#pragma unroll
    for (int j = 0; j < kPer; ++j)
      if (cm >> j & 1u) {
        cand[off] = tv[j];
        key[off] = h2o_key(sv[j], tv[j]);
        ++off;
      }
  }
  __syncthreads();
  // 2. threshold = the K-th largest key (keys are unique): MSB-first radix select
  unsigned long long thr = 0;
  if (nc > K) {
    if (tid == 0) {
      s_prefix = 0ull;
      s_need = K;
    }
    unsigned long long mask = 0ull;
    for (int pass = 0; pass < 8 && K > 0; ++pass) {
      const int shift = 56 - 8 * pass;
      if (tid < 256) hist[tid] = 0;
      __syncthreads();
      const unsigned long long prefix = s_prefix;
      for (int i = tid; i < nc; i += kSelThreads)
        if ((key[i] & mask) == prefix) atomicAdd(&hist[(key[i] >> shift) & 255], 1);
      __syncthreads();
      if (tid < 32) {  // digit d with above(d) < need <= above(d) + hist[d], above = keys with a larger digit
        const int lane = tid;
        int h[8], sum = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {  // lane holds digits 255 - 8 lane - j (descending)
          h[j] = hist[255 - 8 * lane - j];
          sum += h[j];
        }
        int incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        const int need = s_need;
        int above = incl - sum;
        int found = -1, nabove = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (found < 0 && above < need && need <= above + h[j]) {
            found = 255 - 8 * lane - j;
            nabove = above;
          }
          above += h[j];
        }
        const unsigned bal = __ballot_sync(0xffffffffu, found >= 0);
        const int src = __ffs(bal) - 1;
        found = __shfl_sync(0xffffffffu, found, src);
        nabove = __shfl_sync(0xffffffffu, nabove, src);
        if (lane == 0) {
          s_prefix = prefix | ((unsigned long long)found << shift);
          s_need = need - nabove;
        }
      }
      mask |= 0xffull << shift;
      __syncthreads();
    }
    thr = K > 0 ? s_prefix : ~0ull;  // K = 0: nothing is kept
  }
  // 3. I = [0, s') ++ kept candidates (position order) ++ [w0, T)
  const int64_t base = (int64_t)b * cap;
  const int cper = (nc + kSelThreads - 1) / kSelThreads;
  unsigned km = 0;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int i = tid * cper + j;
    if (j < cper && i < nc && (nc <= K || (K > 0 && key[i] >= thr))) km |= 1u << j;
  }
  int nk;
  {
    int pos = sp + block_excl_scan(__popc(km), wsum, &nk);
#pragma unroll
    for (int j = 0; j < kPer; ++j)
      if (km >> j & 1u) {
        if (pos < cap) index[base + pos] = cand[tid * cper + j];
        ++pos;
      }
  }
  for (int t = tid; t < sp; t += kSelThreads)
    if (t < cap) index[base + t] = t;
  const int wb = sp + nk;
  for (int t = w0 + tid; t < T; t += kSelThreads)
    if (wb + t - w0 < cap) index[base + wb + t - w0] = t;
  if (tid == 0) {
    const int total = wb + (T - w0);
    if (total > cap) set_status(status, ZOOMR_ERR_CAPACITY);
    index_count[b] = total < cap ? total : cap;
  }
}

}  // namespace zoomr

using namespace zoomr;

extern "C" int zoomr_h2o_accumulate(const zoomr_geom *geom, int32_t batch, const int32_t *index,
                                    const int32_t *index_count, int32_t index_capacity, const float *logits,
                                    const float *lse, float *score, int32_t score_stride, int32_t *index_copy,
                                    int32_t *count_copy, int32_t *dev_status, void *stream) {
  int rc = check_geom(geom);
  if (rc) return rc;
  if (batch < 1 || batch > 65535 || !index || !index_count || index_capacity < 1 || !logits || !lse || !score ||
      score_stride < 1 || (index_copy && index_copy == index))
    return ZOOMR_ERR_INVALID_ARG;
  const dim3 grid((index_capacity + kAccTok - 1) / kAccTok, batch);
  h2o_accumulate_kernel<<<grid, kAccTok * kAccGrp, 0, (cudaStream_t)stream>>>(
      index, index_count, index_capacity, geom->num_layers * geom->num_q_heads, logits, lse, score, score_stride,
      index_copy, count_copy, dev_status);
  return launch_status((cudaStream_t)stream);
}

extern "C" int zoomr_h2o_select(int32_t batch, const int32_t *prev_index, const int32_t *prev_count,
                                int32_t index_capacity, const float *score, int32_t score_stride,
                                const int32_t *seq_len, int32_t sink, int32_t window, int32_t budget,
                                int32_t *index, int32_t *index_count, int32_t *dev_status, void *stream) {
  if (batch < 1 || !prev_index || !prev_count || index_capacity < 1 || !score || score_stride < 1 || !seq_len ||
      sink < 0 || window < 1 || budget < 0 || !index || !index_count || index == prev_index)
    return ZOOMR_ERR_INVALID_ARG;
  const size_t smem = (size_t)kMaxCand * (sizeof(uint64_t) + sizeof(int32_t));
  cudaFuncSetAttribute(h2o_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  h2o_select_kernel<<<batch, kSelThreads, smem, (cudaStream_t)stream>>>(prev_index, prev_count, index_capacity,
                                                                       score, score_stride, seq_len, sink, window,
                                                                       budget, index, index_count, dev_status);
  return launch_status((cudaStream_t)stream);
}
