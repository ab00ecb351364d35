/*
 * zoomr_oracle.c -- plain fp64 CPU oracle for ZoomR's select + sparse decode
 * (arXiv 2604.10898).  See zoomr_oracle.h for layouts.
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py; never by the product path.
 *
 * Each function follows the paper's statement step by step, in the paper's
 * order, with no blocking, fusion or reordering.  The only parallelism is an
 * OpenMP loop over independent (layer, head) attention outputs in O7; every
 * reduction runs in a fixed sequential order.
 *
 * Parity pins: every function here is pinned by tests/test_oracle_*.py against
 * the SPEC worked examples, the paper's printed |I_f| denominators,
 * closed forms, brute force and torch's fp64 SDPA.
 */
#include "zoomr_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

double zo_bf16_to_double(uint16_t bits) {
  /* bf16 is the high 16 bits of an IEEE-754 binary32: exact widening. */
  uint32_t w = ((uint32_t)bits) << 16;
  float f;
  memcpy(&f, &w, sizeof f);
  return (double)f;
}

int zo_num_threads(int32_t num_threads) {
#ifdef _OPENMP
  return num_threads > 0 ? num_threads : omp_get_max_threads();
#else
  (void)num_threads;
  return 1;
#endif
}

/* reading Q23: a != b and |a - b| <= 1e-6 * max(|a|, |b|) */
static int near_tie(double a, double b) {
  if (a == b) return 0;
  double m = fabs(a) > fabs(b) ? fabs(a) : fabs(b);
  return fabs(a - b) <= 1e-6 * m;
}

int zo_validate_segments(const int32_t *seg, int32_t n_sum, int32_t T) {
  /* segments partition the generated tokens in order:
   * r0 <= r1 <= s0 < s1 <= next r0, and nothing beyond the cache (s1 <= T). */
  if (n_sum < 0 || T < 1) return ZO_ERR_INVALID_ARG;
  if (n_sum > 0 && !seg) return ZO_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n_sum; ++i) {
    int32_t r0 = seg[4 * i + 0], r1 = seg[4 * i + 1], s0 = seg[4 * i + 2], s1 = seg[4 * i + 3];
    if (s1 <= s0) return ZO_ERR_EMPTY_SEGMENT;
    if (r0 < 0 || r1 < r0 || s0 < r1) return ZO_ERR_SEGMENT_ORDER;
    if (i + 1 < n_sum && seg[4 * (i + 1) + 0] < s1) return ZO_ERR_SEGMENT_ORDER;
    if (s1 > T) return ZO_ERR_INDEX_RANGE;
  }
  return ZO_OK;
}

/* ---------------------------------------------------------------- O1 ---- */
int zo_update_mean_keys(const zo_geom *g, const uint16_t *keys, int32_t T,
                        const int32_t *seg, int32_t n_sum, double *mean_keys) {
  if (!g || !keys || !mean_keys) return ZO_ERR_INVALID_ARG;
  int rc = zo_validate_segments(seg, n_sum, T);
  if (rc) return rc;
  const int32_t L = g->num_layers, Hk = g->num_kv_heads, d = g->head_dim;
  for (int32_t l = 0; l < L; ++l)
    for (int32_t h = 0; h < Hk; ++h)
      for (int32_t i = 0; i < n_sum; ++i) {
        const int32_t s0 = seg[4 * i + 2], s1 = seg[4 * i + 3];
        double *out = mean_keys + (((int64_t)l * Hk + h) * n_sum + i) * d;
        for (int32_t e = 0; e < d; ++e) {
          double sum = 0.0;
          for (int32_t j = s0; j < s1; ++j) /* ascending j */
            sum += zo_bf16_to_double(keys[(((int64_t)j * L + l) * Hk + h) * d + e]);
          out[e] = sum / (double)(s1 - s0); /* (1/|S_i|) * sum */
        }
      }
  return ZO_OK;
}

/* ---------------------------------------------------------- O2..O4 ---- */
typedef struct {
  double a;
  int32_t i;
} zo_ai;

static int cmp_alpha_desc_index_asc(const void *x, const void *y) {
  const zo_ai *p = (const zo_ai *)x, *q = (const zo_ai *)y;
  if (p->a > q->a) return -1;
  if (p->a < q->a) return 1;
  return (p->i > q->i) - (p->i < q->i);
}

int zo_aggregate(const zo_geom *g, const double *alpha, int32_t n_sum, int32_t kk,
                 const int32_t *topk, int64_t *votes, double *A) {
  if (!g || !votes || !A || (n_sum > 0 && (!alpha || !topk))) return ZO_ERR_INVALID_ARG;
  const int32_t V = g->num_layers * g->num_q_heads;
  for (int32_t i = 0; i < n_sum; ++i) {
    votes[i] = 0;
    A[i] = 0.0;
  }
  /* v_i = sum_{l,h} 1(i in I_topk^{(l,h)}); A_i in (l,h) lexicographic order */
  for (int32_t v = 0; v < V; ++v)
    for (int32_t r = 0; r < kk; ++r) {
      int32_t i = topk[(int64_t)v * kk + r];
      if (i < 0 || i >= n_sum) return ZO_ERR_INDEX_RANGE;
      votes[i] += 1;
      A[i] += alpha[(int64_t)v * n_sum + i];
    }
  return ZO_OK;
}

int zo_score(const zo_geom *g, const uint16_t *q, const double *mean_keys, int32_t n_sum,
             int32_t top_k, double *alpha, int32_t *topk, int64_t *votes, double *A,
             uint8_t *voter_near_tie) {
  if (!g || !q || top_k < 1 || n_sum < 0) return ZO_ERR_INVALID_ARG;
  if (n_sum > 0 && (!mean_keys || !alpha || !topk || !votes || !A)) return ZO_ERR_INVALID_ARG;
  const int32_t L = g->num_layers, Hq = g->num_q_heads, Hk = g->num_kv_heads, d = g->head_dim;
  if (Hk < 1 || Hq % Hk) return ZO_ERR_INVALID_ARG;
  const int32_t G = Hq / Hk;
  const int32_t kk = top_k < n_sum ? top_k : n_sum; /* reading Q5: clamp to min(k, N_t) */
  if (n_sum == 0) return ZO_OK;                     /* reading Q19: nothing to score */
  zo_ai *order = (zo_ai *)malloc(sizeof(zo_ai) * (size_t)n_sum);
  if (!order) return ZO_ERR_INVALID_ARG;
  for (int32_t l = 0; l < L; ++l)
    for (int32_t h = 0; h < Hq; ++h) {
      const int32_t v = l * Hq + h, hk = h / G;
      const uint16_t *qv = q + ((int64_t)l * Hq + h) * d;
      /* O2: alpha_i = q^T kbar_i, no 1/sqrt(d) */
      for (int32_t i = 0; i < n_sum; ++i) {
        const double *kb = mean_keys + (((int64_t)l * Hk + hk) * n_sum + i) * d;
        double s = 0.0;
        for (int32_t e = 0; e < d; ++e) s += zo_bf16_to_double(qv[e]) * kb[e];
        alpha[(int64_t)v * n_sum + i] = s;
        order[i].a = s;
        order[i].i = i;
      }
      /* O3: arg top-k, ties -> smaller index  (reading Q3) */
      qsort(order, (size_t)n_sum, sizeof(zo_ai), cmp_alpha_desc_index_asc);
      for (int32_t r = 0; r < kk; ++r) topk[(int64_t)v * kk + r] = order[r].i;
      if (voter_near_tie)
        voter_near_tie[v] = (uint8_t)(kk < n_sum && near_tie(order[kk - 1].a, order[kk].a));
    }
  free(order);
  /* O4 */
  return zo_aggregate(g, alpha, n_sum, kk, topk, votes, A);
}

/* --------------------------------------------------------------- O5 ---- */
typedef struct {
  int64_t v;
  double a;
  int32_t i;
} zo_vai;

static int cmp_votes_desc_a_desc_index_asc(const void *x, const void *y) {
  const zo_vai *p = (const zo_vai *)x, *q = (const zo_vai *)y;
  if (p->v != q->v) return p->v > q->v ? -1 : 1;
  if (p->a > q->a) return -1;
  if (p->a < q->a) return 1;
  return (p->i > q->i) - (p->i < q->i);
}

int zo_select_topc(const int64_t *votes, const double *A, int32_t n_sum, int32_t c,
                   uint8_t *flags, double *agreeability, uint8_t *cut_near_tie) {
  if (c < 0 || n_sum < 0 || (n_sum > 0 && (!votes || !A || !flags))) return ZO_ERR_INVALID_ARG;
  zo_vai *all = (zo_vai *)malloc(sizeof(zo_vai) * (size_t)(n_sum > 0 ? n_sum : 1));
  if (!all) return ZO_ERR_INVALID_ARG;
  int32_t n_all = 0;
  for (int32_t i = 0; i < n_sum; ++i) {
    flags[i] = 0;
    if (votes[i] > 0) { /* I_all = union of the per-head sets = {i : v_i > 0} */
      all[n_all].v = votes[i];
      all[n_all].a = A[i];
      all[n_all].i = i;
      ++n_all;
    }
  }
  qsort(all, (size_t)n_all, sizeof(zo_vai), cmp_votes_desc_a_desc_index_asc);
  const int32_t nc = c < n_all ? c : n_all; /* |I_c| = min(c, |I_all|)  (reading Q5) */
  int64_t vc = 0, vall = 0;
  for (int32_t r = 0; r < n_all; ++r) {
    flags[all[r].i] = (uint8_t)(r < nc ? 2 : 1); /* I_c zoomed, I_s = I_all \ I_c kept */
    if (r < nc) vc += all[r].v;
    vall += all[r].v;
  }
  if (agreeability) *agreeability = vall > 0 ? (double)vc / (double)vall : 0.0;
  if (cut_near_tie)
    *cut_near_tie = (uint8_t)(nc > 0 && nc < n_all && all[nc - 1].v == all[nc].v &&
                              near_tie(all[nc - 1].a, all[nc].a));
  free(all);
  return ZO_OK;
}

/* --------------------------------------------------------------- O6 ---- */
int zo_build_index(const int32_t *seg, int32_t n_sum, const uint8_t *flags, int32_t T,
                   int32_t sink, int32_t window, int32_t *index, int32_t capacity,
                   int32_t *count) {
  if (sink < 0 || window < 1 || !count || (n_sum > 0 && !flags)) return ZO_ERR_INVALID_ARG;
  int rc = zo_validate_segments(seg, n_sum, T);
  if (rc) return rc;
  /* The definition is a set union; mark membership, then list ascending. */
  uint8_t *in = (uint8_t *)calloc((size_t)T, 1);
  if (!in) return ZO_ERR_INVALID_ARG;
  for (int32_t j = 0; j < T && j < sink; ++j) in[j] = 1;                 /* I_p (reading Q12) */
  for (int32_t j = (T - window > 0 ? T - window : 0); j < T; ++j) in[j] = 1; /* I_w (Q13) */
  for (int32_t i = 0; i < n_sum; ++i) {
    int32_t a = 0, b = 0;
    if (flags[i] == 2) { a = seg[4 * i + 0]; b = seg[4 * i + 1]; }      /* R_i, i in I_c */
    else if (flags[i] == 1) { a = seg[4 * i + 2]; b = seg[4 * i + 3]; } /* S_i, i in I_s */
    for (int32_t j = a; j < b; ++j) in[j] = 1;
  }
  int32_t n = 0;
  for (int32_t j = 0; j < T; ++j)
    if (in[j]) {
      if (index && n < capacity) index[n] = j;
      ++n;
    }
  free(in);
  *count = n;
  return n > capacity ? ZO_ERR_CAPACITY : ZO_OK;
}

/* --------------------------------------------------------------- O7 ---- */
int zo_attend_one(const uint16_t *q_vec, const uint16_t *k_rows, const uint16_t *v_rows,
                  int64_t row_stride, int32_t d, const int32_t *index, int32_t count,
                  double scale, double *out) {
  if (!q_vec || !k_rows || !v_rows || !index || !out || count < 1 || d < 1)
    return ZO_ERR_INVALID_ARG;
  double *z = (double *)malloc(sizeof(double) * (size_t)count);
  if (!z) return ZO_ERR_INVALID_ARG;
  /* z_j = q . k_j / sqrt(d) */
  double m = -INFINITY;
  for (int32_t t = 0; t < count; ++t) {
    const uint16_t *k = k_rows + (int64_t)index[t] * row_stride;
    double s = 0.0;
    for (int32_t e = 0; e < d; ++e) s += zo_bf16_to_double(q_vec[e]) * zo_bf16_to_double(k[e]);
    z[t] = s * scale;
    if (z[t] > m) m = z[t];
  }
  /* softmax with the max subtracted (mathematically identical) */
  double denom = 0.0;
  for (int32_t t = 0; t < count; ++t) {
    z[t] = exp(z[t] - m);
    denom += z[t];
  }
  for (int32_t e = 0; e < d; ++e) {
    double acc = 0.0;
    for (int32_t t = 0; t < count; ++t)
      acc += z[t] * zo_bf16_to_double(v_rows[(int64_t)index[t] * row_stride + e]);
    out[e] = acc / denom;
  }
  free(z);
  return ZO_OK;
}

int zo_sparse_decode_attn(const zo_geom *g, const uint16_t *q, const uint16_t *keys,
                          const uint16_t *values, int32_t T, const int32_t *index,
                          int32_t count, double scale, double *out, int32_t num_threads) {
  if (!g || !q || !keys || !values || !index || !out || count < 1) return ZO_ERR_INVALID_ARG;
  const int32_t L = g->num_layers, Hq = g->num_q_heads, Hk = g->num_kv_heads, d = g->head_dim;
  if (Hk < 1 || Hq % Hk) return ZO_ERR_INVALID_ARG;
  for (int32_t t = 0; t < count; ++t)
    if (index[t] < 0 || index[t] >= T) return ZO_ERR_INDEX_RANGE;
  const int32_t G = Hq / Hk;
  const int64_t stride = (int64_t)L * Hk * d; /* one token row across (l, kv-head) */
  int rc = ZO_OK;
  (void)num_threads;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic) num_threads(zo_num_threads(num_threads)) reduction(| : rc)
#endif
  for (int32_t lh = 0; lh < L * Hq; ++lh) {
    const int32_t l = lh / Hq, h = lh % Hq, hk = h / G;
    const int64_t base = ((int64_t)l * Hk + hk) * d;
    rc |= zo_attend_one(q + (int64_t)lh * d, keys + base, values + base, stride, d, index, count,
                        scale, out + (int64_t)lh * d);
  }
  return rc;
}

/* ---------------------------------------------- O8 log partition ---- */
int zo_log_partition(const zo_geom *g, const uint16_t *q, const uint16_t *keys, int32_t T,
                     const int32_t *index, int32_t count, double scale, double *lse) {
  if (!g || !q || !keys || !index || !lse || count < 1) return ZO_ERR_INVALID_ARG;
  const int32_t L = g->num_layers, Hq = g->num_q_heads, Hk = g->num_kv_heads, d = g->head_dim;
  if (Hk < 1 || Hq % Hk) return ZO_ERR_INVALID_ARG;
  for (int32_t t = 0; t < count; ++t)
    if (index[t] < 0 || index[t] >= T) return ZO_ERR_INDEX_RANGE;
  const int32_t G = Hq / Hk;
  const int64_t stride = (int64_t)L * Hk * d;
  for (int32_t lh = 0; lh < L * Hq; ++lh) {
    const int32_t l = lh / Hq, h = lh % Hq;
    const uint16_t *qv = q + (int64_t)lh * d;
    const uint16_t *k0 = keys + ((int64_t)l * Hk + h / G) * d;
    /* ln sum_j exp(z_j) = m + ln sum_j exp(z_j - m), m = max_j z_j (identical) */
    double m = -INFINITY;
    for (int32_t t = 0; t < count; ++t) {
      double s = 0.0;
      for (int32_t e = 0; e < d; ++e) s += zo_bf16_to_double(qv[e]) * zo_bf16_to_double(k0[(int64_t)index[t] * stride + e]);
      if (s * scale > m) m = s * scale;
    }
    double sum = 0.0;
    for (int32_t t = 0; t < count; ++t) {
      double s = 0.0;
      for (int32_t e = 0; e < d; ++e) s += zo_bf16_to_double(qv[e]) * zo_bf16_to_double(k0[(int64_t)index[t] * stride + e]);
      sum += exp(s * scale - m);
    }
    lse[lh] = m + log(sum);
  }
  return ZO_OK;
}

/* --------------------------------------------------------- O9 H2O ---- */
int zo_h2o_weights(const zo_geom *g, const uint16_t *q, const uint16_t *keys, int32_t T,
                   const int32_t *index, int32_t count, double scale, double *w) {
  if (!g || !q || !keys || !index || !w || count < 1) return ZO_ERR_INVALID_ARG;
  const int32_t L = g->num_layers, Hq = g->num_q_heads, Hk = g->num_kv_heads, d = g->head_dim;
  if (Hk < 1 || Hq % Hk) return ZO_ERR_INVALID_ARG;
  for (int32_t t = 0; t < count; ++t)
    if (index[t] < 0 || index[t] >= T) return ZO_ERR_INDEX_RANGE;
  const int32_t G = Hq / Hk;
  const int64_t stride = (int64_t)L * Hk * d;
  double *z = (double *)malloc(sizeof(double) * (size_t)count);
  if (!z) return ZO_ERR_INVALID_ARG;
  for (int32_t t = 0; t < count; ++t) w[t] = 0.0;
  for (int32_t lh = 0; lh < L * Hq; ++lh) {
    const int32_t l = lh / Hq, h = lh % Hq;
    const uint16_t *qv = q + (int64_t)lh * d;
    const uint16_t *k0 = keys + ((int64_t)l * Hk + h / G) * d;
    double m = -INFINITY, den = 0.0;
    for (int32_t t = 0; t < count; ++t) {
      double s = 0.0;
      for (int32_t e = 0; e < d; ++e) s += zo_bf16_to_double(qv[e]) * zo_bf16_to_double(k0[(int64_t)index[t] * stride + e]);
      z[t] = s * scale;
      if (z[t] > m) m = z[t];
    }
    for (int32_t t = 0; t < count; ++t) den += exp(z[t] - m);
    for (int32_t t = 0; t < count; ++t) w[t] += exp(z[t] - m) / den; /* softmax weight of row t for (l, h) */
  }
  for (int32_t t = 0; t < count; ++t) w[t] /= (double)(L * Hq);
  free(z);
  return ZO_OK;
}

typedef struct {
  double score;
  int32_t t;
} zo_st;

static int cmp_score_desc_pos_asc(const void *x, const void *y) {
  const zo_st *a = (const zo_st *)x, *b = (const zo_st *)y;
  if (a->score > b->score) return -1;
  if (a->score < b->score) return 1;
  return (a->t > b->t) - (a->t < b->t);
}

int zo_h2o_select(const int32_t *prev, int32_t n_prev, const double *score, int32_t T, int32_t sink,
                  int32_t window, int32_t budget, int32_t *out, int32_t capacity, int32_t *count) {
  if ((!prev && n_prev) || !score || !out || !count || T < 1 || sink < 0 || window < 1 || budget < 0)
    return ZO_ERR_INVALID_ARG;
  const int32_t sp = sink < T ? sink : T;
  const int32_t w0 = T - window > sp ? T - window : sp;
  const int32_t K = budget - (sp + (T - w0)) > 0 ? budget - (sp + (T - w0)) : 0;
  zo_st *cand = (zo_st *)malloc(sizeof(zo_st) * (size_t)(n_prev > 0 ? n_prev : 1));
  uint8_t *in = (uint8_t *)calloc((size_t)T, 1);
  if (!cand || !in) return ZO_ERR_INVALID_ARG;
  int32_t nc = 0;
  for (int32_t i = 0; i < n_prev; ++i) {
    if (prev[i] < 0 || prev[i] >= T) { free(cand); free(in); return ZO_ERR_INDEX_RANGE; }
    if (prev[i] >= sp && prev[i] < w0) {
      cand[nc].score = score[prev[i]];
      cand[nc].t = prev[i];
      ++nc;
    }
  }
  qsort(cand, (size_t)nc, sizeof(zo_st), cmp_score_desc_pos_asc);
  for (int32_t t = 0; t < sp; ++t) in[t] = 1;
  for (int32_t t = w0; t < T; ++t) in[t] = 1;
  for (int32_t i = 0; i < nc && i < K; ++i) in[cand[i].t] = 1;
  int32_t n = 0;
  for (int32_t t = 0; t < T; ++t)
    if (in[t]) {
      if (n >= capacity) { free(cand); free(in); return ZO_ERR_CAPACITY; }
      out[n++] = t;
    }
  *count = n;
  free(cand);
  free(in);
  return ZO_OK;
}

/* ------------------------------------------------- the whole step ---- */
int zo_step(const zo_geom *g, const zo_params *p, const uint16_t *q, const uint16_t *keys,
            const uint16_t *values, int32_t T, const int32_t *seg, int32_t n_sum,
            double *mean_keys, double *alpha, int32_t *topk, int64_t *votes, double *A,
            uint8_t *flags, int32_t *index, int32_t capacity, int32_t *count, double *out,
            int32_t num_threads) {
  if (!g || !p) return ZO_ERR_INVALID_ARG;
  int rc;
  if (n_sum > 0) {
    /* Alg.1: mean keys (@P:408-409), scoring + per-head top-k (@P:411-412),
     * aggregation and consensus (@P:416-419). */
    if ((rc = zo_update_mean_keys(g, keys, T, seg, n_sum, mean_keys))) return rc;
    if ((rc = zo_score(g, q, mean_keys, n_sum, p->top_k, alpha, topk, votes, A, NULL))) return rc;
    if ((rc = zo_select_topc(votes, A, n_sum, p->c, flags, NULL, NULL))) return rc;
  }
  /* I_w and I_f (@P:421-422); N_t = 0 gives sink u window (reading Q19). */
  if ((rc = zo_build_index(seg, n_sum, flags, T, p->sink, p->window, index, capacity, count)))
    return rc;
  return zo_sparse_decode_attn(g, q, keys, values, T, index, *count,
                               1.0 / sqrt((double)g->head_dim), out, num_threads);
}
