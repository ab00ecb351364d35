// Token-sharded split-K across GPUs (for H_kv < #GPUs):
// the KV cache of one sequence is spread over R ranks by token, every rank
// runs the (replicated, tiny) selection and obtains the same I_f, attends over
// the part of I_f it holds, and the R partial results are combined with their
// log-sum-exp weights.  The exchange of (out, lse) between ranks is the
// caller's collective (an all-gather); these are the kernels either side of it.
//
//  * zoomr_shard_index: I_f restricted to the tokens this rank owns (order kept);
//  * zoomr_merge_attn:  softmax over a union of disjoint index sets from the
//    per-set softmax outputs and their partition functions (the split-K identity
//    of P:148's softmax: sum_j e^{s_j} v_j / sum_j e^{s_j} over the union =
//    sum_r e^{lse_r} o_r / sum_r e^{lse_r}).
#include "common.cuh"

namespace zoomr {

// one CTA of 1024 threads per sequence; thread i handles a contiguous run of
// up to kPer entries (all its index and owner loads in flight at once), one
// block-wide exclusive scan of the per-thread keep counts, then the writes.
// Launched with PDL: it waits for the producer of I_f, and lets a5 start its
// prologue right away.
constexpr int kShardThreads = 1024, kPer = 16;
__global__ void __launch_bounds__(kShardThreads) shard_index_kernel(
    const int32_t *__restrict__ index, const int32_t *__restrict__ count, int32_t cap,
    const uint8_t *__restrict__ owner, int32_t owner_stride, int32_t rank, int32_t *__restrict__ local_index,
    int32_t *__restrict__ local_count, int32_t *status) {
  __shared__ int wsum[32];
  __shared__ int carry;
  allow_dependents();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int n = count[b];
  n = n < cap ? n : cap;
  if (tid == 0) carry = 0;
  const int32_t *ib = index + (int64_t)b * cap;
  const uint8_t *ob = owner + (int64_t)b * owner_stride;
  for (int c0 = 0; c0 < n; c0 += kShardThreads * kPer) {
    const int m = min(n - c0, kShardThreads * kPer);
    const int per = (m + kShardThreads - 1) / kShardThreads;  // entries per thread this round
    const int i0 = c0 + tid * per;
    int t[kPer];
    unsigned keep = 0;
#pragma unroll
    for (int j = 0; j < kPer; ++j) t[j] = (j < per && i0 + j < c0 + m) ? ib[i0 + j] : -2;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      if (t[j] == -2) continue;
      if (t[j] < 0 || t[j] >= owner_stride) set_status(status, ZOOMR_ERR_INDEX_RANGE);
      else if (ob[t[j]] == (uint8_t)rank) keep |= 1u << j;
    }
    // exclusive scan of the keep counts over the block
    const int k = __popc(keep);
    int incl = k;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int x = wsum[lane], xi = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, xi, o);
        if (lane >= o) xi += y;
      }
      wsum[lane] = xi - x;  // exclusive warp offsets
    }
    __syncthreads();
    int pos = carry + wsum[warp] + incl - k;
#pragma unroll
    for (int j = 0; j < kPer; ++j)
      if (keep >> j & 1u) local_index[(int64_t)b * cap + pos++] = t[j];
    __syncthreads();  // everyone has read carry / wsum
    if (tid == kShardThreads - 1) carry += wsum[warp] + incl;
    __syncthreads();
  }
  if (tid == 0) local_count[b] = carry;
}

// one warp per (b, l, h) row; parts merged in rank order (deterministic, the
// same on every rank).  Lane r < n_parts loads part r's lse, so the weights of
// up to 32 parts take one round trip; the part outputs are then read NU at a
// time with all their loads in flight.
__global__ void merge_attn_kernel(int64_t rows, int32_t rows_per_seq, int32_t B, int32_t d, int32_t n_parts,
                                  const float *__restrict__ part_out, const float *__restrict__ part_lse,
                                  const int32_t *__restrict__ part_count, float *__restrict__ out,
                                  float *__restrict__ lse_out) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int b = (int)(row / rows_per_seq);
  float M = -INFINITY;
  for (int r0 = 0; r0 < n_parts; r0 += 32) {
    const int r = r0 + lane;
    float x = -INFINITY;
    if (r < n_parts && !(part_count && part_count[(int64_t)r * B + b] == 0)) x = part_lse[(int64_t)r * rows + row];
#pragma unroll
    for (int o = 16; o; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
    M = fmaxf(M, x);
  }
  float acc[4] = {0.f, 0.f, 0.f, 0.f};  // d <= 128: element lane + 32 * k
  float den = 0.f;
  if (M > -INFINITY) {
    for (int r0 = 0; r0 < n_parts; r0 += 32) {
      const int r = r0 + lane;
      float wl = 0.f;  // lane r's weight (0 for an empty part)
      if (r < n_parts && !(part_count && part_count[(int64_t)r * B + b] == 0))
        wl = expf(part_lse[(int64_t)r * rows + row] - M);
      const int nr = min(32, n_parts - r0);
      constexpr int NU = 4;
      for (int j0 = 0; j0 < nr; j0 += NU) {
        float w[NU], v[NU][4];
#pragma unroll
        for (int j = 0; j < NU; ++j) {
          w[j] = __shfl_sync(0xffffffffu, wl, (j0 + j) & 31);
          const float *o = part_out + ((int64_t)(r0 + j0 + j) * rows + row) * d;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            v[j][k] = (j0 + j < nr && w[j] != 0.f && lane + 32 * k < d) ? o[lane + 32 * k] : 0.f;
        }
#pragma unroll
        for (int j = 0; j < NU; ++j) {
          if (j0 + j >= nr) w[j] = 0.f;
          den += w[j];
#pragma unroll
          for (int k = 0; k < 4; ++k) acc[k] += w[j] * v[j][k];
        }
      }
    }
  }
  const float inv = den > 0.f ? 1.f / den : 0.f;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (lane + 32 * k < d) out[row * d + lane + 32 * k] = acc[k] * inv;
  if (lse_out && lane == 0) lse_out[row] = den > 0.f ? M + logf(den) : -INFINITY;
}

}  // namespace zoomr

using namespace zoomr;

extern "C" int zoomr_shard_index(int32_t batch, const int32_t *index, const int32_t *index_count,
                                 int32_t index_capacity, const uint8_t *owner, int32_t owner_stride, int32_t rank,
                                 int32_t *local_index, int32_t *local_count, int32_t *dev_status, void *stream) {
  if (batch < 1 || !index || !index_count || index_capacity < 1 || !owner || owner_stride < 1 || rank < 0 ||
      rank > 255 || !local_index || !local_count || local_index == index)
    return ZOOMR_ERR_INVALID_ARG;
  launch_pdl(shard_index_kernel, batch, kShardThreads, 0, (cudaStream_t)stream, index, index_count, index_capacity,
             owner, owner_stride, rank, local_index, local_count, dev_status);
  return launch_status((cudaStream_t)stream);
}

extern "C" int zoomr_merge_attn(const zoomr_geom *geom, int32_t batch, int32_t n_parts, const float *part_out,
                                const float *part_lse, const int32_t *part_count, float *out, float *lse,
                                void *stream) {
  int rc = check_geom(geom);
  if (rc) return rc;
  if (batch < 1 || n_parts < 1 || !part_out || !part_lse || !out) return ZOOMR_ERR_INVALID_ARG;
  const int32_t rps = geom->num_layers * geom->num_q_heads;
  const int64_t rows = (int64_t)batch * rps;
  const int wpb = 8;
  const int64_t grid = (rows + wpb - 1) / wpb;
  if (grid > 0x7fffffff) return ZOOMR_ERR_UNSUPPORTED;
  merge_attn_kernel<<<(unsigned)grid, 32 * wpb, 0, (cudaStream_t)stream>>>(
      rows, rps, batch, geom->head_dim, n_parts, part_out, part_lse, part_count, out, lse);
  return launch_status((cudaStream_t)stream);
}
