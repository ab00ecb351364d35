// a2 -- per-head importance scoring, voting and the cross-head / cross-layer
// aggregation (Alg.1 @P:411-417).
//
//   alpha_i^{(l,h)} = q_t^{(l,h)} . kbar_i^{(l, h/G)}          (no 1/sqrt(d))
//   I_topk^{(l,h)}  = arg top-k_i alpha_i^{(l,h)}               (ties -> smaller i)
//   v_i = sum_{l,h} 1(i in I_topk^{(l,h)}),  A_i = sum of alpha over those voters
//
// One CTA per (layer, KV head, sequence).  The G query heads of a KV head share
// every mean-key row: an octet of lanes reads one fp32 row (coalesced 128-byte
// float4 loads) and forms the G dot products against the queries staged in
// shared memory; a 3-step butterfly inside the octet finishes each sum.  This is
// a batched GEMV (G <= 8 rows against fp32 keys, ~G/2 flop/byte) on CUDA cores:
// it is HBM-bound and there is no dense contraction for the tensor cores.
// All alphas of the CTA stay in shared memory; warp hh then runs voter
// (l, g*G+hh)'s top-k by k rounds of a warp arg-max with the (alpha desc,
// index asc) order, and adds its votes to `partial` with integer atomics:
// votes as int64 counts, A as the int64 sum of round(alpha * 2^32).  Integer
// addition is associative, so the aggregate is bit-identical for any launch
// order, any number of head shards, and any run.
#include "select_common.cuh"

namespace zoomr {

__global__ void zero_i64_kernel(int64_t *__restrict__ p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 0;
}

template <int D, int G>
__global__ void __launch_bounds__(256) score_kernel(
    const __nv_bfloat16 *__restrict__ q, const float *__restrict__ mean_keys,
    const int32_t *__restrict__ num_summaries, int32_t max_summaries, int32_t top_k, int32_t L,
    int32_t Hkv, int64_t *__restrict__ partial, float *__restrict__ alpha_out,
    int32_t *__restrict__ topk_out, int32_t *status) {
  extern __shared__ __align__(16) float smem[];
  float *qs = smem;                                    // [G][D]
  float *al = smem + G * D;                            // [G][max_summaries]
  int *sel_i = reinterpret_cast<int *>(al + G * max_summaries);  // [G][top_k]
  float *sel_a = reinterpret_cast<float *>(sel_i + G * top_k);  // [G][top_k]
  const int lg = blockIdx.x, b = blockIdx.y;
  const int l = lg / Hkv, g = lg % Hkv;
  const int Hq = Hkv * G;
  int nt = num_summaries[b];
  if (nt > max_summaries || nt < 0) {
    if (threadIdx.x == 0) set_status(status, ZOOMR_ERR_INDEX_RANGE);
    nt = nt < 0 ? 0 : max_summaries;
  }
  const __nv_bfloat16 *qb = q + (((int64_t)b * L + l) * Hq + (int64_t)g * G) * D;
  const float *mk = mean_keys + (((int64_t)b * L + l) * Hkv + g) * (int64_t)max_summaries * D;
  float *ao = alpha_out ? alpha_out + (((int64_t)b * L + l) * Hq + (int64_t)g * G) * max_summaries : nullptr;
  block_score_topk<D, G>(qb, mk, nt, top_k, qs, al, max_summaries, ao, max_summaries, sel_i, sel_a);
  // votes and fixed-point A into `partial` with integer atomics (order-independent)
  const int kk = top_k < nt ? top_k : nt;
  int64_t *pv = partial + (int64_t)b * 2 * max_summaries;
  for (int x = threadIdx.x; x < G * top_k; x += blockDim.x) {
    const int hh = x / top_k, r = x - hh * top_k;
    const int64_t voter = (int64_t)l * Hq + g * G + hh;
    if (r < kk) {
      const int i = sel_i[x];
      atomicAdd(reinterpret_cast<unsigned long long *>(pv + i), 1ull);
      atomicAdd(reinterpret_cast<unsigned long long *>(pv + max_summaries + i),
                (unsigned long long)alpha_fixed(sel_a[x]));
    }
    if (topk_out) topk_out[((int64_t)b * L * Hq + voter) * top_k + r] = r < kk ? sel_i[x] : -1;
  }
}

}  // namespace zoomr

using namespace zoomr;

extern "C" int zoomr_score(const zoomr_geom *geom, int32_t batch, const void *q,
                           const float *mean_keys, const int32_t *num_summaries,
                           int32_t max_summaries, int32_t top_k, int64_t *partial,
                           float *alpha_out, int32_t *topk_out, int32_t *dev_status, void *stream) {
  int rc = check_geom(geom);
  if (rc) return rc;
  if (batch < 1 || !q || !mean_keys || !num_summaries || !partial || max_summaries < 1 || top_k < 1)
    return ZOOMR_ERR_INVALID_ARG;
  if (top_k > kMaxTopK || top_k > 32 || max_summaries > kMaxSummaries) return ZOOMR_ERR_UNSUPPORTED;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = (int64_t)batch * 2 * max_summaries;
  prefer_max_smem(zero_i64_kernel);
  zero_i64_kernel<<<(int)((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024), 256, 0, s>>>(partial, n);
  const int G = geom->num_q_heads / geom->num_kv_heads, D = geom->head_dim;
  const size_t smem = (size_t)G * D * 4 + (size_t)G * max_summaries * 4 + (size_t)G * top_k * 8;
  dim3 grid(geom->num_layers * geom->num_kv_heads, batch);
#define ZOOMR_SC(DD, GG)                                                                           \
  do {                                                                                             \
    auto kfn = score_kernel<DD, GG>;                                                               \
    prefer_max_smem(kfn);                                                                          \
    if (smem > 48 * 1024) cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    kfn<<<grid, 256, smem, s>>>((const __nv_bfloat16 *)q, mean_keys, num_summaries, max_summaries, \
                                top_k, geom->num_layers, geom->num_kv_heads, partial, alpha_out,  \
                                topk_out, dev_status);                                            \
  } while (0)
#define ZOOMR_SC_G(DD)                     \
  switch (G) {                             \
    case 1: ZOOMR_SC(DD, 1); break;        \
    case 2: ZOOMR_SC(DD, 2); break;        \
    case 4: ZOOMR_SC(DD, 4); break;        \
    case 7: ZOOMR_SC(DD, 7); break;        \
    default: ZOOMR_SC(DD, 8); break;       \
  }
  switch (D) {
    case 16: ZOOMR_SC_G(16); break;
    case 32: ZOOMR_SC_G(32); break;
    case 64: ZOOMR_SC_G(64); break;
    default: ZOOMR_SC_G(128); break;
  }
#undef ZOOMR_SC_G
#undef ZOOMR_SC
  return launch_status((cudaStream_t)stream);
}
