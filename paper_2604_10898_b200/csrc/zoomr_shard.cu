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

// one CTA per sequence; block-wide stream compaction in chunks of blockDim.x
__global__ void __launch_bounds__(256) shard_index_kernel(const int32_t *__restrict__ index,
                                                          const int32_t *__restrict__ count, int32_t cap,
                                                          const uint8_t *__restrict__ owner, int32_t owner_stride,
                                                          int32_t rank, int32_t *__restrict__ local_index,
                                                          int32_t *__restrict__ local_count, int32_t *status) {
  __shared__ int wsum[8];
  __shared__ int base;
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int n = count[b];
  n = n < cap ? n : cap;
  if (tid == 0) base = 0;
  __syncthreads();
  for (int c0 = 0; c0 < n; c0 += 256) {
    const int i = c0 + tid;
    int t = -1;
    bool keep = false;
    if (i < n) {
      t = index[(int64_t)b * cap + i];
      if (t < 0 || t >= owner_stride) set_status(status, ZOOMR_ERR_INDEX_RANGE);
      else keep = owner[(int64_t)b * owner_stride + t] == (uint8_t)rank;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    int off = base;
    for (int w = 0; w < warp; ++w) off += wsum[w];
    if (keep) local_index[(int64_t)b * cap + off + __popc(bal & ((1u << lane) - 1))] = t;
    __syncthreads();
    if (tid == 0)
      for (int w = 0; w < 8; ++w) base += wsum[w];
    __syncthreads();
  }
  if (tid == 0) local_count[b] = base;
}

// one warp per (b, l, h) row; parts merged in rank order (deterministic, the
// same on every rank)
__global__ void merge_attn_kernel(int64_t rows, int32_t rows_per_seq, int32_t B, int32_t d, int32_t n_parts,
                                  const float *__restrict__ part_out, const float *__restrict__ part_lse,
                                  const int32_t *__restrict__ part_count, float *__restrict__ out,
                                  float *__restrict__ lse_out) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int b = (int)(row / rows_per_seq);
  float M = -INFINITY;
  for (int r = 0; r < n_parts; ++r) {
    if (part_count && part_count[(int64_t)r * B + b] == 0) continue;  // nothing of I_f on rank r
    M = fmaxf(M, part_lse[(int64_t)r * rows + row]);
  }
  float acc[4] = {0.f, 0.f, 0.f, 0.f};  // d <= 128: element lane + 32 * k
  float den = 0.f;
  if (M > -INFINITY) {
    for (int r = 0; r < n_parts; ++r) {
      if (part_count && part_count[(int64_t)r * B + b] == 0) continue;
      const float w = expf(part_lse[(int64_t)r * rows + row] - M);
      den += w;
      const float *o = part_out + ((int64_t)r * rows + row) * d;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (lane + 32 * k < d) acc[k] += w * o[lane + 32 * k];
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
  shard_index_kernel<<<batch, 256, 0, (cudaStream_t)stream>>>(index, index_count, index_capacity, owner, owner_stride,
                                                               rank, local_index, local_count, dev_status);
  return launch_status();
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
  return launch_status();
}
