// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" wrapper around the REFERENCE's own C++ implementation
// (compiled unmodified from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libmoe_ref.so).  It exists so the Python tests, the golden
// generator and bench.py's reference arm can drive the reference through flat
// buffers.  No reference source is copied here: this file only includes the
// reference headers and calls the reference functions.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "moe_orch/cost_model.hpp"
#include "moe_orch/error.hpp"
#include "moe_orch/model.hpp"
#include "moe_orch/placement.hpp"
#include "moe_orch/shape.hpp"
#include "moe_orch/trace.hpp"
#include "moe_orch/trace.hpp"

using namespace moe_orch;

namespace {

thread_local std::string g_err;

int map_exc() {
  try {
    throw;
  } catch (const ShapeError& e) {
    g_err = e.what();
    return 1;
  } catch (const ValidationError& e) {
    g_err = e.what();
    return 2;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

ModelShape to_shape(const int32_t* s) {
  ModelShape m;
  m.num_layers = s[0];
  m.experts_per_layer = s[1];
  m.top_k = s[2];
  m.hidden_dim = s[3];
  m.ffn_dim = s[4];
  m.bytes_per_param = s[5];
  return m;
}

Matrix to_matrix(int rows, int cols, const double* p) {
  Matrix m(rows, cols);
  if (p) std::memcpy(m.data.data(), p, sizeof(double) * m.data.size());
  return m;
}

// Builds ModelWeights from flat per-(layer,expert) pointers.  A NULL expert
// pointer leaves that expert as empty matrices (never touched unless routed).
ModelWeights to_weights(const ModelShape& s, const double* const* w_in,
                        const double* const* w_gate, const double* const* w_out,
                        const double* const* router) {
  ModelWeights w;
  const int L = s.num_layers, E = s.experts_per_layer, d = s.hidden_dim, f = s.ffn_dim;
  w.experts.resize(L);
  for (int l = 0; l < L; ++l) {
    for (int e = 0; e < E; ++e) {
      ExpertWeights ew;
      if (w_in[l * E + e]) {
        ew.w_in = to_matrix(f, d, w_in[l * E + e]);
        ew.w_gate = to_matrix(f, d, w_gate[l * E + e]);
        ew.w_out = to_matrix(d, f, w_out[l * E + e]);
      }
      w.experts[l].push_back(std::move(ew));
    }
    w.router.layers.push_back(to_matrix(E, d, router[l]));
  }
  return w;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_shape_validate(const int32_t* shape) {
  try {
    to_shape(shape).validate();
    return 0;
  } catch (...) {
    return map_exc();
  }
}

int ref_shape_preset(const char* name, int32_t* out) {
  try {
    ModelShape s = ModelShape::preset(name);
    const int32_t v[6] = {s.num_layers, s.experts_per_layer, s.top_k,
                          s.hidden_dim, s.ffn_dim, s.bytes_per_param};
    std::memcpy(out, v, sizeof(v));
    return 0;
  } catch (...) {
    return map_exc();
  }
}

// random_model (model.cpp:34-53) flattened into caller buffers.
int ref_random_model(const int32_t* shape, uint64_t seed, double* const* w_in,
                     double* const* w_gate, double* const* w_out, double* const* router) {
  try {
    const ModelShape s = to_shape(shape);
    const ModelWeights w = random_model(s, seed);
    const int E = s.experts_per_layer;
    for (int l = 0; l < s.num_layers; ++l) {
      for (int e = 0; e < E; ++e) {
        const auto& ew = w.experts[l][e];
        if (w_in && w_in[l * E + e])
          std::memcpy(w_in[l * E + e], ew.w_in.data.data(), ew.w_in.data.size() * 8);
        if (w_gate && w_gate[l * E + e])
          std::memcpy(w_gate[l * E + e], ew.w_gate.data.data(), ew.w_gate.data.size() * 8);
        if (w_out && w_out[l * E + e])
          std::memcpy(w_out[l * E + e], ew.w_out.data.data(), ew.w_out.data.size() * 8);
      }
      if (router && router[l])
        std::memcpy(router[l], w.router.layers[l].data.data(),
                    w.router.layers[l].data.size() * 8);
    }
    return 0;
  } catch (...) {
    return map_exc();
  }
}

int ref_expert_ffn(int d, int f, const double* w_in, const double* w_gate,
                   const double* w_out, const double* x, int x_len, double* y) {
  try {
    ExpertWeights w;
    w.w_in = to_matrix(f, d, w_in);
    w.w_gate = to_matrix(f, d, w_gate);
    w.w_out = to_matrix(d, f, w_out);
    const auto out = expert_ffn(w, std::vector<double>(x, x + x_len));
    std::memcpy(y, out.data(), out.size() * 8);
    return 0;
  } catch (...) {
    return map_exc();
  }
}

int ref_gate_topk(int E, int d, const double* router_l, const double* x, int k,
                  int32_t* ids, double* weights) {
  try {
    RouterWeights r;
    r.layers.push_back(to_matrix(E, d, router_l));
    const auto sel = gate_topk(r, 0, std::vector<double>(x, x + d), k);
    for (size_t j = 0; j < sel.size(); ++j) {
      ids[j] = sel[j].first;
      weights[j] = sel[j].second;
    }
    return 0;
  } catch (...) {
    return map_exc();
  }
}

struct SinkBuf {
  std::vector<int32_t> layers;
  std::vector<double> values;
};

static void collect(int layer, const std::vector<double>& v, void* ctx) {
  auto* b = static_cast<SinkBuf*>(ctx);
  b->layers.push_back(layer);
  b->values.insert(b->values.end(), v.begin(), v.end());
}

// model_forward (model.cpp:103-161).  tokens [n_tok*d] in, outputs out.
// sel_* receive the trace (per layer up to E selections: expert, count, gate)
// as dense [L*E] arrays (count 0 = not selected).  If sink_vals != NULL the
// ActivationSink path runs and post-SiLU values are copied out in call order
// (capacity sink_cap doubles); *sink_n receives the count.
int ref_model_forward(const int32_t* shape, const double* const* w_in,
                      const double* const* w_gate, const double* const* w_out,
                      const double* const* router, int n_tok, int tok_width,
                      const double* tokens, double* outputs, int32_t* sel_count,
                      double* sel_gate, int32_t* step_kind, double* sink_vals,
                      int64_t sink_cap, int64_t* sink_n) {
  try {
    const ModelShape s = to_shape(shape);
    const ModelWeights w = to_weights(s, w_in, w_gate, w_out, router);
    std::vector<std::vector<double>> toks(n_tok);
    for (int t = 0; t < n_tok; ++t)
      toks[t].assign(tokens + (size_t)t * tok_width, tokens + (size_t)(t + 1) * tok_width);
    SinkBuf buf;
    const ForwardResult r = sink_vals ? model_forward(s, w, toks, &collect, &buf)
                                      : model_forward(s, w, toks);
    for (int t = 0; t < n_tok; ++t)
      std::memcpy(outputs + (size_t)t * tok_width, r.outputs[t].data(), tok_width * 8);
    const int E = s.experts_per_layer;
    std::memset(sel_count, 0, sizeof(int32_t) * (size_t)s.num_layers * E);
    std::memset(sel_gate, 0, sizeof(double) * (size_t)s.num_layers * E);
    *step_kind = -1;
    if (!r.trace.steps.empty()) {
      r.trace.validate(s);
      const auto& st = r.trace.steps[0];
      *step_kind = st.kind == StepKind::Decode ? 1 : 0;
      for (size_t l = 0; l < st.layers.size(); ++l)
        for (const auto& sel : st.layers[l]) {
          sel_count[l * E + sel.expert] = sel.token_count;
          sel_gate[l * E + sel.expert] = sel.gate_weight;
        }
    }
    if (sink_vals) {
      *sink_n = (int64_t)buf.values.size();
      const size_t n = std::min<size_t>(buf.values.size(), (size_t)sink_cap);
      std::memcpy(sink_vals, buf.values.data(), n * 8);
    }
    return 0;
  } catch (...) {
    return map_exc();
  }
}

// Times the reference model_forward on n_tok tokens (each token is an
// independent call, as the reference is token-major anyway).  Weights are
// built before the clock starts.  Returns wall seconds in *seconds.
int ref_time_forward(const int32_t* shape, const double* const* w_in,
                     const double* const* w_gate, const double* const* w_out,
                     const double* const* router, int n_tok, const double* tokens,
                     double* outputs, double* seconds) {
  try {
    const ModelShape s = to_shape(shape);
    const ModelWeights w = to_weights(s, w_in, w_gate, w_out, router);
    const int d = s.hidden_dim;
    std::vector<std::vector<double>> toks(n_tok);
    for (int t = 0; t < n_tok; ++t) toks[t].assign(tokens + (size_t)t * d, tokens + (size_t)(t + 1) * d);
    const auto t0 = std::chrono::steady_clock::now();
    const ForwardResult r = model_forward(s, w, toks);
    const auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    for (int t = 0; t < n_tok; ++t) std::memcpy(outputs + (size_t)t * d, r.outputs[t].data(), d * 8);
    return 0;
  } catch (...) {
    return map_exc();
  }
}

// Persistent reference model for the CPU baseline: the weights are built
// once and shared (const) by concurrent model_forward calls — the reference
// is reentrant, so N host threads each push their own tokens.
struct RefModel {
  ModelShape shape;
  ModelWeights weights;
};

void* ref_model_create(const int32_t* shape, const double* const* w_in,
                       const double* const* w_gate, const double* const* w_out,
                       const double* const* router) {
  try {
    auto* m = new RefModel();
    m->shape = to_shape(shape);
    m->weights = to_weights(m->shape, w_in, w_gate, w_out, router);
    return m;
  } catch (...) {
    map_exc();
    return nullptr;
  }
}

void ref_model_destroy(void* h) { delete static_cast<RefModel*>(h); }

// model_forward on n_tok tokens of the shared model; wall seconds in *seconds.
int ref_model_forward_timed(void* h, int n_tok, const double* tokens, double* outputs,
                            double* seconds) {
  try {
    const RefModel* m = static_cast<const RefModel*>(h);
    const int d = m->shape.hidden_dim;
    std::vector<std::vector<double>> toks(n_tok);
    for (int t = 0; t < n_tok; ++t) toks[t].assign(tokens + (size_t)t * d, tokens + (size_t)(t + 1) * d);
    const auto t0 = std::chrono::steady_clock::now();
    const ForwardResult r = model_forward(m->shape, m->weights, toks);
    const auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    if (outputs)
      for (int t = 0; t < n_tok; ++t) std::memcpy(outputs + (size_t)t * d, r.outputs[t].data(), d * 8);
    return 0;
  } catch (...) {
    return map_exc();
  }
}

// ---- placement (placement.cpp) ----
static PopularityProfile to_profile(int L, int E, const int64_t* counts, int64_t total) {
  PopularityProfile p;
  p.counts.assign(L, std::vector<std::int64_t>(E, 0));
  for (int l = 0; l < L; ++l)
    for (int e = 0; e < E; ++e) p.counts[l][e] = counts[l * E + e];
  p.total_selections = total;
  return p;
}

int ref_greedy_place(int L, int E, const int64_t* counts, int64_t total, int capacity,
                     int per_layer_quota, uint8_t* resident) {
  try {
    const Placement pl = greedy_place(to_profile(L, E, counts, total), capacity,
                                      per_layer_quota != 0);
    std::memset(resident, 0, (size_t)L * E);
    for (const auto& [l, e] : pl.resident) resident[l * E + e] = 1;
    return 0;
  } catch (...) {
    return map_exc();
  }
}

int ref_expected_hit_rate(int L, int E, const int64_t* counts, int64_t total,
                          const uint8_t* resident, double* out) {
  try {
    Placement pl;
    for (int l = 0; l < L; ++l)
      for (int e = 0; e < E; ++e)
        if (resident[l * E + e]) pl.resident.insert({l, e});
    *out = expected_hit_rate(pl, to_profile(L, E, counts, total));
    return 0;
  } catch (...) {
    return map_exc();
  }
}

int ref_hit_rate_bounds(int L, int E, const int64_t* counts, int64_t total, int capacity,
                        double* out3) {
  try {
    const HitRateBounds b = hit_rate_bounds(to_profile(L, E, counts, total), capacity);
    out3[0] = b.best;
    out3[1] = b.worst;
    out3[2] = b.random;
    return 0;
  } catch (...) {
    return map_exc();
  }
}

int ref_sparsity_histogram(const double* acts, int64_t n, const double* thr, int nthr,
                           double* out) {
  try {
    const auto f = sparsity_histogram(std::vector<double>(acts, acts + n),
                                      std::vector<double>(thr, thr + nthr));
    std::memcpy(out, f.data(), f.size() * 8);
    return 0;
  } catch (...) {
    return map_exc();
  }
}

// load_records_csv + fit (cost_model.cpp:57-156): out[6] = weight_copy_ms,
// activation_copy_ms, fast_exec_ms, slow_ms_per_token, slow_intercept_ms,
// nonexpert_ms_per_step.
int ref_fit_records(const char* path, double nonexpert_ms, double* out) {
  try {
    const CostModel m = fit(load_records_csv(std::string(path)), nonexpert_ms);
    out[0] = m.weight_copy_ms;
    out[1] = m.activation_copy_ms;
    out[2] = m.fast_exec_ms;
    out[3] = m.slow_ms_per_token;
    out[4] = m.slow_intercept_ms;
    out[5] = m.nonexpert_ms_per_step;
    return m.decode_assumption_check() ? 0 : 100;  // 100: ok, but the paper's decode premise fails
  } catch (...) {
    return map_exc();
  }
}

// load_trace_jsonl (trace.cpp:110-141): parses AND validates a JSONL trace
// against the shape; returns the number of steps in *n_steps.
int ref_load_trace_jsonl(const char* path, const int32_t* shape, int* n_steps) {
  try {
    const RoutingTrace t = load_trace_jsonl(std::string(path), to_shape(shape));
    *n_steps = (int)t.steps.size();
    return 0;
  } catch (...) {
    return map_exc();
  }
}

}  // extern "C"
