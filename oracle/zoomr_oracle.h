/*
 * zoomr_oracle.h -- plain, slow, obviously-correct CPU oracle for the ZoomR
 * select + sparse-decode hot path (arXiv 2604.10898).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2604_10898_b200/) never links, imports or calls it,
 * and it shares no code, header, table or helper with the CUDA path.
 *
 * Everything is one sequence at a time, in fp64, on the exact decoded values
 * of the bf16 inputs, in LOGICAL token order (no paging -- paging is a layout
 * choice of the GPU path, not part of the method).
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n.
 * The readings of the paper that these functions implement are listed in
 * DESIGN.md section 3 ("Readings"), numbered Q1..Q25 as in SURVEY.md 8(c).
 *
 * Layouts (all row-major, C order):
 *   keys / values : uint16 bf16 bit patterns [T][L][H_kv][d]
 *   q             : uint16 bf16 bit patterns [L][H_q][d]
 *   seg           : int32 [n_sum][4] = (r0, r1, s0, s1), half-open, 0-based
 *   mean keys     : double [L][H_kv][n_sum][d]
 *   alpha         : double [L][H_q][n_sum]           (voter v = l*H_q + h)
 *   topk          : int32  [L*H_q][kk], kk = min(top_k, n_sum)
 *   votes, A      : int64 [n_sum], double [n_sum]
 *   flags         : uint8 [n_sum] in {0 dropped, 1 kept as summary (I_s), 2 zoomed (I_c)}
 *   index         : int32 [count] ascending token positions (I_f)
 *   out           : double [L][H_q][d]
 * Query head h reads KV head h / (H_q / H_kv)  (reading Q6).
 */
#ifndef ZOOMR_ORACLE_H
#define ZOOMR_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ZO_OK = 0,
  ZO_ERR_INVALID_ARG = 1,
  ZO_ERR_EMPTY_SEGMENT = 2,   /* S_i with s1 <= s0 (SPEC EmptySegment)          */
  ZO_ERR_SEGMENT_ORDER = 3,   /* r0<=r1<=s0<s1<=next r0 violated              */
  ZO_ERR_INDEX_RANGE = 4,     /* segment beyond T (S:200 UnknownSegment)        */
  ZO_ERR_CAPACITY = 5         /* |I_f| larger than the caller's buffer                   */
};

typedef struct {
  int32_t num_layers;   /* N_L                  */
  int32_t num_q_heads;  /* H (query heads)              */
  int32_t num_kv_heads; /* KV heads (GQA, reading Q6)   */
  int32_t head_dim;     /* d                    */
} zo_geom;

/* Decode one bf16 bit pattern exactly (bf16 is the top half of an IEEE fp32). */
double zo_bf16_to_double(uint16_t bits);

/* Segment-table validation (SPEC S:24-27 invariants; reading Q13/Q18). */
int zo_validate_segments(const int32_t *seg, int32_t n_sum, int32_t T);

/* O1  mean summary key  k_i = (1/|S_i|) sum_{j in S_i} k_j          (Alg.1 @P:408-409) */
int zo_update_mean_keys(const zo_geom *g, const uint16_t *keys, int32_t T,
                        const int32_t *seg, int32_t n_sum, double *mean_keys);

/* O2  alpha_i^{(l,h)} = q^T kbar_i  (no 1/sqrt(d); reading Q7)
 * O3  per-voter top-k by (alpha desc, i asc)            (Alg.1 @P:412; reading Q3, Q5)
 * O4  votes v_i and A_i = sum of alpha over voters that chose i, (l,h) lexicographic
 *                                                        (Alg.1 @P:416-417; reading Q1, Q2)
 * voter_near_tie[v] = 1 when the last kept and first dropped alpha are within 1e-6 relative
 * without being equal (reading Q23).  Any output pointer except alpha/topk/votes/A may be NULL. */
int zo_score(const zo_geom *g, const uint16_t *q, const double *mean_keys, int32_t n_sum,
             int32_t top_k, double *alpha, int32_t *topk, int64_t *votes, double *A,
             uint8_t *voter_near_tie);

/* O4 alone, from given per-voter sets (used by the parity checker to re-run the
 * downstream stages with the GPU's choice inside a certified near-tie). */
int zo_aggregate(const zo_geom *g, const double *alpha, int32_t n_sum, int32_t kk,
                 const int32_t *topk, int64_t *votes, double *A);

/* O5  I_c = first min(c, #I_all) of I_all ordered by (v desc, A desc, i asc);
 *     I_s = I_all \ I_c                                  (Alg.1 @P:418-419; reading Q2, Q5)
 * agreeability AG = sum_{I_c} v / sum_{I_all} v; 0 when I_all empty.
 * cut_near_tie = 1 when the last kept and first dropped have equal votes and A within 1e-6. */
int zo_select_topc(const int64_t *votes, const double *A, int32_t n_sum, int32_t c,
                   uint8_t *flags, double *agreeability, uint8_t *cut_near_tie);

/* O6  I_f = [0,min(s,T)) u [max(0,T-w),T) u R_i (flag 2) u S_i (flag 1), as a sorted set
 *                                                        (Alg.1 @P:421-422; reading Q12-Q19) */
int zo_build_index(const int32_t *seg, int32_t n_sum, const uint8_t *flags, int32_t T,
                   int32_t sink, int32_t window, int32_t *index, int32_t capacity,
                   int32_t *count);

/* O7  one head: o = sum_j softmax_j(q.k_j * scale) v_j over j in I_f
 * k_rows/v_rows point at token 0 of this (l, kv-head); row j is at +j*row_stride elements. */
int zo_attend_one(const uint16_t *q_vec, const uint16_t *k_rows, const uint16_t *v_rows,
                  int64_t row_stride, int32_t d, const int32_t *index, int32_t count,
                  double scale, double *out);

/* O7 for every (l, h) of one sequence. keys/values [T][L][H_kv][d]. num_threads<=0: all cores. */
int zo_sparse_decode_attn(const zo_geom *g, const uint16_t *q, const uint16_t *keys,
                          const uint16_t *values, int32_t T, const int32_t *index,
                          int32_t count, double scale, double *out, int32_t num_threads);

/* O8  (token-sharded split-K) the softmax normaliser of O7 in log form:
 *     lse[l][h] = ln sum_{j in index} exp(q.k_j * scale)          (P:148's denominator)
 * for every (l, h) of one sequence.  Not a step of the paper: it is the quantity by
 * which attention over disjoint index sets combines into attention over their union. */
int zo_log_partition(const zo_geom *g, const uint16_t *q, const uint16_t *keys, int32_t T,
                     const int32_t *index, int32_t count, double scale, double *lse);

/* O9  H2O, the paper's heavy-hitter baseline (the paper only cites it, the rule is
 *     SPEC h2o_step S:349-357):
 *  zo_h2o_weights: w[j] = (1/(L*H_q)) sum_{l,h} softmax_j(q_{l,h}.k_j * scale) over j in index
 *                  ("per-retained-token softmax weights averaged over heads/layers");
 *  zo_h2o_select:  the next retained set = [0, min(sink,T)) u [max(that, T-window), T) u the
 *                  top-(budget - |sink u window|) entries of prev outside them by score desc,
 *                  ties -> smaller position; sorted ascending into out[0..*count). */
int zo_h2o_weights(const zo_geom *g, const uint16_t *q, const uint16_t *keys, int32_t T,
                   const int32_t *index, int32_t count, double scale, double *w);
int zo_h2o_select(const int32_t *prev, int32_t n_prev, const double *score, int32_t T, int32_t sink,
                  int32_t window, int32_t budget, int32_t *out, int32_t capacity, int32_t *count);

/* The whole step O1..O7 for one sequence, as Algorithm 1 orders it. */
typedef struct {
  int32_t top_k, c, sink, window;
} zo_params;

int zo_step(const zo_geom *g, const zo_params *p, const uint16_t *q, const uint16_t *keys,
            const uint16_t *values, int32_t T, const int32_t *seg, int32_t n_sum,
            double *mean_keys, double *alpha, int32_t *topk, int64_t *votes, double *A,
            uint8_t *flags, int32_t *index, int32_t capacity, int32_t *count,
            double *out, int32_t num_threads);

/* Number of OpenMP threads the oracle would use for num_threads (for reporting). */
int zo_num_threads(int32_t num_threads);

#ifdef __cplusplus
}
#endif
#endif
