/*
 * moe_oracle.c — TEST INFRASTRUCTURE ONLY (see moe_oracle.h).
 *
 * Plain-C fp64 restatement of the reference hot path.  Every function cites
 * the reference file:line it restates.  Compiled with -O2 -ffp-contract=off
 * and no -march so the arithmetic order (and hence every fp64 bit) matches
 * the reference's Release build (proj/CMakeLists.txt:7-9, x86-64 baseline,
 * no FMA contraction).
 *
 * Parity pinned: tests/test_oracle.py compares this file bit-for-bit with
 * the reference compiled from /root/reference (oracle/_ref) and with the
 * golden vectors under tests/golden/.
 */
#include "moe_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- geometry: ModelShape::validate, shape.cpp:7-16 ---- */
int oracle_shape_validate(const oracle_shape* s) {
  if (s->num_layers < 0) return ORACLE_SHAPE_ERROR;
  if (s->experts_per_layer <= 0 || s->top_k <= 0 || s->hidden_dim <= 0 ||
      s->ffn_dim <= 0 || s->bytes_per_param <= 0)
    return ORACLE_SHAPE_ERROR;
  if (s->top_k > s->experts_per_layer) return ORACLE_SHAPE_ERROR;
  return ORACLE_OK;
}

/* ---- std::mt19937_64 (the engine model.cpp:36 seeds) ---- */
#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x000000007FFFFFFFULL

void oracle_rng_seed(oracle_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) +
               (uint64_t)i;
  r->idx = MT_N;
}

static void mt_twist(oracle_rng* r) {
  for (int i = 0; i < MT_N; ++i) {
    uint64_t x = (r->mt[i] & MT_UPPER) | (r->mt[(i + 1) % MT_N] & MT_LOWER);
    uint64_t xa = x >> 1;
    if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
    r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
  }
  r->idx = 0;
}

uint64_t oracle_rng_next(oracle_rng* r) {
  if (r->idx >= MT_N) mt_twist(r);
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

/* generate_canonical<double, 53>(mt19937_64): one 64-bit draw / 2^64,
 * clamped below 1. */
static double canonical(oracle_rng* r) {
  double v = (double)oracle_rng_next(r) / 18446744073709551616.0;
  if (v >= 1.0) v = nextafter(1.0, 0.0);
  return v;
}

/* libstdc++ normal_distribution<double>::operator() (Marsaglia polar), with
 * the cached second variate.  One distribution object == one call here,
 * matching random_matrix's fresh `dist` (model.cpp:15). */
void oracle_normal_fill(oracle_rng* r, double stddev, double* out, int64_t n) {
  int have_saved = 0;
  double saved = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double ret;
    if (have_saved) {
      have_saved = 0;
      ret = saved;
    } else {
      double x, y, r2;
      do {
        x = 2.0 * canonical(r) - 1.0;
        y = 2.0 * canonical(r) - 1.0;
        r2 = x * x + y * y;
      } while (r2 > 1.0 || r2 == 0.0);
      const double mult = sqrt(-2.0 * log(r2) / r2);
      saved = x * mult;
      have_saved = 1;
      ret = y * mult;
    }
    const double v = ret * stddev + 0.0;
    if (out) out[i] = v;
  }
}

/* random_model, model.cpp:34-53 (random_matrix :13-18). */
int oracle_random_model(const oracle_shape* s, uint64_t seed, double* const* w_in,
                        double* const* w_gate, double* const* w_out,
                        double* const* router) {
  if (oracle_shape_validate(s)) return ORACLE_SHAPE_ERROR;
  oracle_rng rng;
  oracle_rng_seed(&rng, seed);
  const double scale = 1.0 / sqrt((double)s->hidden_dim);
  const int64_t fd = (int64_t)s->ffn_dim * s->hidden_dim;
  const int E = s->experts_per_layer;
  for (int l = 0; l < s->num_layers; ++l) {
    for (int e = 0; e < E; ++e) {
      oracle_normal_fill(&rng, scale, w_in ? w_in[l * E + e] : NULL, fd);
      oracle_normal_fill(&rng, scale, w_gate ? w_gate[l * E + e] : NULL, fd);
      oracle_normal_fill(&rng, scale, w_out ? w_out[l * E + e] : NULL, fd);
    }
    oracle_normal_fill(&rng, scale, router ? router[l] : NULL,
                       (int64_t)E * s->hidden_dim);
  }
  return ORACLE_OK;
}

/* matvec, model.cpp:20-30. */
void oracle_matvec(int rows, int cols, const double* m, const double* x, double* y) {
  for (int r = 0; r < rows; ++r) {
    double acc = 0.0;
    const double* row = m + (size_t)r * cols;
    for (int c = 0; c < cols; ++c) acc += row[c] * x[c];
    y[r] = acc;
  }
}

/* silu, model.hpp:51. */
double oracle_silu(double x) { return x / (1.0 + exp(-x)); }

/* expert_ffn, model.cpp:55-67. */
void oracle_expert_ffn(int d, int f, const double* w_in, const double* w_gate,
                       const double* w_out, const double* x, double* y) {
  double* up = (double*)malloc(sizeof(double) * (size_t)f);
  double* gate = (double*)malloc(sizeof(double) * (size_t)f);
  oracle_matvec(f, d, w_in, x, up);
  oracle_matvec(f, d, w_gate, x, gate);
  for (int i = 0; i < f; ++i) up[i] = oracle_silu(up[i]) * gate[i];
  oracle_matvec(d, f, w_out, up, y);
  free(up);
  free(gate);
}

/* expert_ffn (model.cpp:55-67) for n tokens against ONE expert: the same
 * per-token arithmetic and summation order as oracle_expert_ffn (each output
 * y_t bit-identical to it), with the weight rows visited once for the whole
 * batch (large-shape parity checks stream 1.4 GB of fp64 weights per
 * expert).  X, Y: [n x d] row-major. */
void oracle_expert_ffn_batch(int d, int f, const double* w_in, const double* w_gate,
                             const double* w_out, int n, const double* X, double* Y) {
  double* up = (double*)malloc(sizeof(double) * (size_t)f * (size_t)(n > 0 ? n : 1));
  for (int r = 0; r < f; ++r) {
    const double* a = w_in + (size_t)r * d;
    const double* b = w_gate + (size_t)r * d;
    for (int t = 0; t < n; ++t) {
      const double* x = X + (size_t)t * d;
      double sa = 0.0, sb = 0.0;
      for (int c = 0; c < d; ++c) sa += a[c] * x[c];
      for (int c = 0; c < d; ++c) sb += b[c] * x[c];
      up[(size_t)t * f + r] = oracle_silu(sa) * sb;
    }
  }
  for (int i = 0; i < d; ++i) {
    const double* o = w_out + (size_t)i * f;
    for (int t = 0; t < n; ++t) {
      const double* u = up + (size_t)t * f;
      double s = 0.0;
      for (int r = 0; r < f; ++r) s += o[r] * u[r];
      Y[(size_t)t * d + i] = s;
    }
  }
  free(up);
}

/* gate_topk, model.cpp:69-101.  The stable_sort on (logit desc, id asc) is a
 * total order, so a selection of the k best under that order is the same
 * set; ids are then re-sorted ascending (:86) and the softmax is taken over
 * the selected logits in ascending-id order (:89-99). */
int oracle_gate_topk(int E, int d, const double* router_l, const double* x, int k,
                     int32_t* ids, double* weights, double* logits_out) {
  double* logits = (double*)malloc(sizeof(double) * (size_t)E);
  oracle_matvec(E, d, router_l, x, logits);
  if (logits_out) memcpy(logits_out, logits, sizeof(double) * (size_t)E);
  if (k < 1 || k > E) {
    free(logits);
    return ORACLE_SHAPE_ERROR;
  }
  uint8_t* taken = (uint8_t*)calloc((size_t)E, 1);
  for (int j = 0; j < k; ++j) {
    int best = -1;
    for (int e = 0; e < E; ++e) {
      if (taken[e]) continue;
      if (best < 0 || logits[e] > logits[best]) best = e; /* ties keep lower id */
    }
    taken[best] = 1;
  }
  int n = 0;
  for (int e = 0; e < E; ++e)
    if (taken[e]) ids[n++] = e;
  double max_logit = logits[ids[0]];
  for (int j = 0; j < k; ++j)
    if (logits[ids[j]] > max_logit) max_logit = logits[ids[j]];
  double denom = 0.0;
  for (int j = 0; j < k; ++j) {
    const double w = exp(logits[ids[j]] - max_logit);
    denom += w;
    weights[j] = w;
  }
  for (int j = 0; j < k; ++j) weights[j] /= denom;
  free(taken);
  free(logits);
  return ORACLE_OK;
}

/* model_forward, model.cpp:103-161 (token-major; layers in order; experts
 * in ascending id; combined starts at 0 and is added to x after all k). */
int oracle_model_forward(const oracle_shape* s, const double* const* w_in,
                         const double* const* w_gate, const double* const* w_out,
                         const double* const* router, int n_tok, double* tokens,
                         int32_t* tally, double* gate_sum, int32_t* ids_out,
                         double* gates_out, oracle_sink sink, void* sink_ctx) {
  if (oracle_shape_validate(s)) return ORACLE_SHAPE_ERROR;
  const int L = s->num_layers, E = s->experts_per_layer, k = s->top_k;
  const int d = s->hidden_dim, f = s->ffn_dim;
  if (tally) memset(tally, 0, sizeof(int32_t) * (size_t)L * E);
  if (gate_sum) memset(gate_sum, 0, sizeof(double) * (size_t)L * E);
  if (L == 0 || n_tok == 0) return ORACLE_OK;

  int32_t* ids = (int32_t*)malloc(sizeof(int32_t) * (size_t)k);
  double* g = (double*)malloc(sizeof(double) * (size_t)k);
  double* combined = (double*)malloc(sizeof(double) * (size_t)d);
  double* y = (double*)malloc(sizeof(double) * (size_t)d);
  double* up = (double*)malloc(sizeof(double) * (size_t)f);
  double* gate = (double*)malloc(sizeof(double) * (size_t)f);
  for (int t = 0; t < n_tok; ++t) {
    double* x = tokens + (size_t)t * d;
    for (int l = 0; l < L; ++l) {
      oracle_gate_topk(E, d, router[l], x, k, ids, g, NULL);
      for (int i = 0; i < d; ++i) combined[i] = 0.0;
      for (int j = 0; j < k; ++j) {
        const int e = ids[j];
        const int we = l * E + e;
        if (sink) {
          /* model.cpp:131-139: post-SiLU values, before the gate multiply. */
          oracle_matvec(f, d, w_in[we], x, up);
          for (int i = 0; i < f; ++i) up[i] = oracle_silu(up[i]);
          sink(l, up, f, sink_ctx);
          oracle_matvec(f, d, w_gate[we], x, gate);
          for (int i = 0; i < f; ++i) up[i] *= gate[i];
          oracle_matvec(d, f, w_out[we], up, y);
        } else {
          oracle_expert_ffn(d, f, w_in[we], w_gate[we], w_out[we], x, y);
        }
        for (int i = 0; i < d; ++i) combined[i] += g[j] * y[i];
        if (tally) tally[l * E + e] += 1;
        if (gate_sum) gate_sum[l * E + e] += g[j];
        if (ids_out) ids_out[((size_t)t * L + l) * k + j] = e;
        if (gates_out) gates_out[((size_t)t * L + l) * k + j] = g[j];
      }
      for (int i = 0; i < d; ++i) x[i] += combined[i];
    }
  }
  free(ids);
  free(g);
  free(combined);
  free(y);
  free(up);
  free(gate);
  return ORACLE_OK;
}

/* ---- placement.cpp ---- */

/* profile_from_trace, placement.cpp:30-43 (one step's per-layer tallies). */
int64_t oracle_profile_add(int L, int E, const int32_t* tally, int64_t* counts) {
  int64_t total = 0;
  for (int i = 0; i < L * E; ++i) {
    counts[i] += tally[i];
    total += tally[i];
  }
  return total;
}

static const int64_t* g_rank_counts;
static int rank_cmp(const void* a, const void* b) {
  const int32_t ia = *(const int32_t*)a, ib = *(const int32_t*)b;
  const int64_t ca = g_rank_counts[ia], cb = g_rank_counts[ib];
  if (ca != cb) return ca > cb ? -1 : 1;
  return ia < ib ? -1 : (ia > ib); /* flat l*E+e order == (layer, expert) lex */
}

/* ranked_by_popularity, placement.cpp:53-64. */
void oracle_ranked(int L, int E, const int64_t* counts, int32_t* order) {
  for (int i = 0; i < L * E; ++i) order[i] = i;
  g_rank_counts = counts;
  qsort(order, (size_t)L * E, sizeof(int32_t), rank_cmp);
}

/* greedy_place, placement.cpp:68-95. */
int oracle_greedy_place(int L, int E, const int64_t* counts, int capacity,
                        int per_layer_quota, uint8_t* resident) {
  if (capacity < 0) return ORACLE_VALIDATION_ERROR;
  memset(resident, 0, (size_t)L * E);
  if (!per_layer_quota) {
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(L * E + 1));
    oracle_ranked(L, E, counts, order);
    const int take = capacity < L * E ? capacity : L * E;
    for (int i = 0; i < take; ++i) resident[order[i]] = 1;
    free(order);
    return ORACLE_OK;
  }
  if (L == 0) return ORACLE_OK;
  const int quota = capacity / L;
  for (int l = 0; l < L; ++l) {
    /* per-layer sort: count desc, expert asc (placement.cpp:83-89). */
    for (int q = 0; q < quota && q < E; ++q) {
      int best = -1;
      for (int e = 0; e < E; ++e) {
        if (resident[l * E + e]) continue;
        if (best < 0 || counts[l * E + e] > counts[l * E + best]) best = e;
      }
      resident[l * E + best] = 1;
    }
  }
  return ORACLE_OK;
}

/* expected_hit_rate, placement.cpp:97-105. */
int oracle_expected_hit_rate(int L, int E, const int64_t* counts, int64_t total,
                             const uint8_t* resident, double* out) {
  if (total <= 0) return ORACLE_VALIDATION_ERROR;
  int64_t hits = 0;
  for (int i = 0; i < L * E; ++i)
    if (resident[i]) hits += counts[i];
  *out = (double)hits / (double)total;
  return ORACLE_OK;
}

/* hit_rate_bounds, placement.cpp:107-124. */
int oracle_hit_rate_bounds(int L, int E, const int64_t* counts, int64_t total,
                           int capacity, double* out3) {
  if (total <= 0) return ORACLE_VALIDATION_ERROR;
  const int n = L * E;
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  oracle_ranked(L, E, counts, order);
  const int take = capacity < n ? capacity : n;
  int64_t best = 0, worst = 0;
  for (int i = 0; i < take; ++i) {
    best += counts[order[i]];
    worst += counts[order[n - 1 - i]];
  }
  out3[0] = (double)best / (double)total;
  out3[1] = (double)worst / (double)total;
  out3[2] = (double)take / (double)n;
  free(order);
  return ORACLE_OK;
}

/* sparsity_histogram, placement.cpp:126-142. */
int oracle_sparsity_histogram(const double* acts, int64_t n, const double* thr,
                              int nthr, double* out) {
  if (n <= 0) return ORACLE_VALIDATION_ERROR;
  for (int i = 1; i < nthr; ++i)
    if (thr[i] <= thr[i - 1]) return ORACLE_VALIDATION_ERROR;
  for (int i = 0; i < nthr; ++i) out[i] = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    const double a = fabs(acts[j]);
    for (int i = 0; i < nthr; ++i)
      if (a < thr[i]) out[i] += 1.0;
  }
  for (int i = 0; i < nthr; ++i) out[i] /= (double)n;
  return ORACLE_OK;
}
