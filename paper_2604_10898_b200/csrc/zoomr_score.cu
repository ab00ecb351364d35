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
#include "common.cuh"

namespace zoomr {

__global__ void zero_i64_kernel(int64_t *__restrict__ p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 0;
}

__device__ __forceinline__ bool better(float a, int i, float b, int j) {
  return a > b || (a == b && i < j);
}

template <int D, int G>
__global__ void __launch_bounds__(256) score_kernel(
    const __nv_bfloat16 *__restrict__ q, const float *__restrict__ mean_keys,
    const int32_t *__restrict__ num_summaries, int32_t max_summaries, int32_t top_k, int32_t L,
    int32_t Hkv, int64_t *__restrict__ partial, float *__restrict__ alpha_out,
    int32_t *__restrict__ topk_out, int32_t *status) {
  extern __shared__ __align__(16) float smem[];
  float *qs = smem;              // [G][D]
  float *al = smem + G * D;      // [G][max_summaries]
  const int lg = blockIdx.x, b = blockIdx.y;
  const int l = lg / Hkv, g = lg % Hkv;
  const int Hq = Hkv * G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  int nt = num_summaries[b];
  if (nt > max_summaries || nt < 0) {
    if (threadIdx.x == 0) set_status(status, ZOOMR_ERR_INDEX_RANGE);
    nt = nt < 0 ? 0 : max_summaries;
  }
  // stage the G queries of this KV head as fp32
  const __nv_bfloat16 *qb = q + (((int64_t)b * L + l) * Hq + (int64_t)g * G) * D;
  for (int x = threadIdx.x; x < G * D; x += blockDim.x) qs[x] = __bfloat162float(qb[x]);
  __syncthreads();

  // ---- alpha for every (head, summary): octet per summary --------------------
  constexpr int FPL = D / 8;  // floats per octet lane (D=16 -> 2, D=128 -> 16)
  const int oct = lane >> 3, l8 = lane & 7;
  const float *mk = mean_keys + (((int64_t)b * L + l) * Hkv + g) * (int64_t)max_summaries * D;
  for (int base = warp * 8; base < nt; base += 8 * 8) {
    // two summaries per octet per iteration: base + oct and base + 4 + oct
    float acc[2][G];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int hh = 0; hh < G; ++hh) acc[u][hh] = 0.f;
    float4 kv[2][FPL >= 4 ? FPL / 4 : 1];
    float2 kv2[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = base + u * 4 + oct;
      const int ic = i < nt ? i : 0;
      const float *row = mk + (int64_t)ic * D;
      if constexpr (FPL >= 4) {
#pragma unroll
        for (int m = 0; m < FPL / 4; ++m) kv[u][m] = *reinterpret_cast<const float4 *>(row + m * 32 + l8 * 4);
      } else {
        kv2[u] = *reinterpret_cast<const float2 *>(row + l8 * 2);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
#pragma unroll
      for (int hh = 0; hh < G; ++hh) {
        float a = 0.f;
        if constexpr (FPL >= 4) {
#pragma unroll
          for (int m = 0; m < FPL / 4; ++m) {
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
        acc[u][hh] = a;
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int hh = 0; hh < G; ++hh) {
        float a = acc[u][hh];
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
            al[hh * max_summaries + i] = acc[u][hh];
            if (alpha_out)
              alpha_out[(((int64_t)b * L + l) * Hq + g * G + hh) * (int64_t)max_summaries + i] = acc[u][hh];
          }
      }
    }
  }
  __syncthreads();

  // ---- per-voter top-k and the vote aggregation --------------------------------
  if (warp >= G) return;
  const int hh = warp;
  const int kk = top_k < nt ? top_k : nt;
  float *a = al + hh * max_summaries;
  const int64_t voter = (int64_t)l * Hq + g * G + hh;
  int my_i = -1;
  float my_a = 0.f;
  for (int r = 0; r < kk; ++r) {
    float ba = -INFINITY;
    int bi = 0x7fffffff;
    for (int i = lane; i < nt; i += 32) {
      const float x = a[i];
      if (better(x, i, ba, bi)) { ba = x; bi = i; }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      const float oa = __shfl_xor_sync(0xffffffffu, ba, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (better(oa, oi, ba, bi)) { ba = oa; bi = oi; }
    }
    if (lane == r) { my_i = bi; my_a = ba; }
    __syncwarp();
    if (lane == 0) a[bi] = -INFINITY;  // exclude from the next round
    __syncwarp();
  }
  if (lane < kk) {
    int64_t *pv = partial + (int64_t)b * 2 * max_summaries;
    atomicAdd(reinterpret_cast<unsigned long long *>(pv + my_i), 1ull);
    const long long fx = __double2ll_rn((double)my_a * 4294967296.0);  // 2^ZOOMR_A_FRAC_BITS
    atomicAdd(reinterpret_cast<unsigned long long *>(pv + max_summaries + my_i), (unsigned long long)fx);
  }
  if (topk_out && lane < top_k)
    topk_out[((int64_t)b * L * Hq + voter) * top_k + lane] = lane < kk ? my_i : -1;
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
  zero_i64_kernel<<<(int)((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024), 256, 0, s>>>(partial, n);
  const int G = geom->num_q_heads / geom->num_kv_heads, D = geom->head_dim;
  const size_t smem = (size_t)G * D * 4 + (size_t)G * max_summaries * 4;
  dim3 grid(geom->num_layers * geom->num_kv_heads, batch);
#define ZOOMR_SC(DD, GG)                                                                           \
  do {                                                                                             \
    auto kfn = score_kernel<DD, GG>;                                                               \
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
  return launch_status();
}
