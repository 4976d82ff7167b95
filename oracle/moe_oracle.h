/*
 * moe_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, CPU, fp64 restatement of the reference's MoE functional core
 * (/root/reference/proj/src/model.cpp) and placement policy
 * (/root/reference/proj/src/placement.cpp).  It is the *checker* for the
 * CUDA product path: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  Nothing under
 * paper_2402_07033_b200/ links or calls it.
 *
 * Parity of this restatement is pinned against the reference itself:
 * oracle/Makefile compiles the reference's own shape.cpp/model.cpp/
 * placement.cpp/trace.cpp into oracle/_ref/libmoe_ref.so, and
 * tests/golden/make_golden.py writes the golden vectors in tests/golden/
 * from it.  tests/test_oracle.py checks this file bit-exactly against both.
 */
#ifndef MOE_ORACLE_H
#define MOE_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors ModelShape (reference include/moe_orch/shape.hpp:9-35). */
typedef struct oracle_shape {
  int32_t num_layers;
  int32_t experts_per_layer;
  int32_t top_k;
  int32_t hidden_dim;
  int32_t ffn_dim;
  int32_t bytes_per_param;
} oracle_shape;

enum { ORACLE_OK = 0, ORACLE_SHAPE_ERROR = 1, ORACLE_VALIDATION_ERROR = 2 };

/* ModelShape::validate, shape.cpp:7-16. */
int oracle_shape_validate(const oracle_shape* s);

/* std::mt19937_64 + libstdc++ std::normal_distribution<double> (Marsaglia
 * polar, generate_canonical<double,53>) — the generator random_model uses
 * (model.cpp:13-18).  A fresh distribution per call (the saved second
 * variate is dropped), exactly like random_matrix. */
typedef struct oracle_rng {
  uint64_t mt[312];
  int idx;
} oracle_rng;
void oracle_rng_seed(oracle_rng* r, uint64_t seed);
uint64_t oracle_rng_next(oracle_rng* r);
/* Fills n values of N(0, stddev) with one distribution object. */
void oracle_normal_fill(oracle_rng* r, double stddev, double* out, int64_t n);

/* random_model, model.cpp:34-53.  Draw order per layer: for each expert
 * w_in[f*d], w_gate[f*d], w_out[d*f]; then router[E*d].
 * w_in/w_gate/w_out are arrays of L*E pointers (index l*E+e), router is an
 * array of L pointers.  A NULL expert pointer skips storing (the draws still
 * happen, so later matrices are unchanged). */
int oracle_random_model(const oracle_shape* s, uint64_t seed, double* const* w_in,
                        double* const* w_gate, double* const* w_out,
                        double* const* router);

/* matvec, model.cpp:20-30: y[r] = sum_c m[r*cols+c]*x[c], left to right. */
void oracle_matvec(int rows, int cols, const double* m, const double* x, double* y);

/* silu, model.hpp:51. */
double oracle_silu(double x);

/* expert_ffn for n tokens of one expert (bit-identical per token). */
void oracle_expert_ffn_batch(int d, int f, const double* w_in, const double* w_gate,
                             const double* w_out, int n, const double* X, double* Y);
/* expert_ffn, model.cpp:55-67.  w_in,w_gate [f x d], w_out [d x f]. */
void oracle_expert_ffn(int d, int f, const double* w_in, const double* w_gate,
                       const double* w_out, const double* x, double* y);

/* gate_topk, model.cpp:69-101.  ids ascending, weights = softmax over the
 * selected logits.  Returns ORACLE_SHAPE_ERROR if k not in [1,E].
 * If logits_out != NULL the E raw logits are written too. */
int oracle_gate_topk(int E, int d, const double* router_l, const double* x, int k,
                     int32_t* ids, double* weights, double* logits_out);

/* ActivationSink, model.hpp:73-74. */
typedef void (*oracle_sink)(int layer, const double* values, int n, void* ctx);

/* model_forward, model.cpp:103-161.  tokens is [n_tok x d] row-major and is
 * updated in place (outputs).  tally[L*E] (int32) and gate_sum[L*E] receive
 * the per-(layer,expert) routing tallies; ids_out/gates_out (optional,
 * [n_tok][L][k]) receive every routing decision. */
int oracle_model_forward(const oracle_shape* s, const double* const* w_in,
                         const double* const* w_gate, const double* const* w_out,
                         const double* const* router, int n_tok, double* tokens,
                         int32_t* tally, double* gate_sum, int32_t* ids_out,
                         double* gates_out, oracle_sink sink, void* sink_ctx);

/* ---- placement (placement.cpp) ---- */

/* profile_from_trace for a single step (placement.cpp:30-43): counts[L*E]
 * += tally.  Returns total selections. */
int64_t oracle_profile_add(int L, int E, const int32_t* tally, int64_t* counts);

/* ranked_by_popularity (placement.cpp:53-64): order[L*E] of flat (l*E+e)
 * indices, count desc, ties by (layer, expert) ascending. */
void oracle_ranked(int L, int E, const int64_t* counts, int32_t* order);

/* greedy_place (placement.cpp:68-95).  resident[L*E] set to 0/1.
 * Returns ORACLE_VALIDATION_ERROR for capacity < 0. */
int oracle_greedy_place(int L, int E, const int64_t* counts, int capacity,
                        int per_layer_quota, uint8_t* resident);

/* expected_hit_rate (placement.cpp:97-105). */
int oracle_expected_hit_rate(int L, int E, const int64_t* counts, int64_t total,
                             const uint8_t* resident, double* out);

/* hit_rate_bounds (placement.cpp:107-124): out = {best, worst, random}. */
int oracle_hit_rate_bounds(int L, int E, const int64_t* counts, int64_t total,
                           int capacity, double* out3);

/* sparsity_histogram (placement.cpp:126-142). */
int oracle_sparsity_histogram(const double* acts, int64_t n, const double* thr,
                              int nthr, double* out);

#ifdef __cplusplus
}
#endif

#endif
