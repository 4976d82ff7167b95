// moe_orch_host.cpp — host-side half of the drop-in moe_orch API (B200 build):
// geometry, routing-trace types and I/O, placement policy (+ the expert-
// parallel shard map), seeded weight init.  The math entry points live in
// moe_orch_device.cpp and go through the C-ABI to the GPU.
//
// Behavioural references (file:line in /root/reference/proj):
//   ModelShape           src/shape.cpp:7-40
//   trace validation     src/trace.cpp:25-88, JSONL format include/moe_orch/trace.hpp:49-56
//   placement            src/placement.cpp:13-296
//   random_model         src/model.cpp:34-53   synth_trace src/model.cpp:163-255
#include <algorithm>
#include <cmath>
#include <fstream>
#include <map>
#include <numeric>
#include <random>
#include <set>
#include <sstream>
#include <tuple>

#include "moe_orch/b200.hpp"
#include "shard_plan.h"
#include "moe_orch/error.hpp"
#include "moe_orch/model.hpp"
#include "moe_orch/placement.hpp"
#include "moe_orch/shape.hpp"
#include "moe_orch/trace.hpp"

namespace moe_orch {

// ---- geometry -------------------------------------------------------------
void ModelShape::validate() const {
  if (num_layers < 0) throw ShapeError("num_layers must be non-negative");
  const bool positive = experts_per_layer > 0 && top_k > 0 && hidden_dim > 0 && ffn_dim > 0 &&
                        bytes_per_param > 0;
  if (!positive) throw ShapeError("all shape counts must be strictly positive");
  if (top_k > experts_per_layer) throw ShapeError("top_k must not exceed experts_per_layer");
}

ModelShape ModelShape::toy() {
  ModelShape s;
  s.num_layers = 4;
  s.experts_per_layer = 8;
  s.top_k = 2;
  s.hidden_dim = 32;
  s.ffn_dim = 64;
  s.bytes_per_param = 2;
  return s;
}

ModelShape ModelShape::mixtral_8x7b() {
  ModelShape s = toy();
  s.num_layers = 32;
  s.hidden_dim = 4096;
  s.ffn_dim = 14336;
  return s;
}

ModelShape ModelShape::preset(const std::string& name) {
  if (name == "toy") return toy();
  if (name == "mixtral") return mixtral_8x7b();
  throw ConfigError("unknown shape preset: " + name);
}

// ---- routing trace ----------------------------------------------------------
std::string to_string(StepKind kind) { return kind == StepKind::Decode ? "decode" : "prefill"; }

StepKind step_kind_from_string(const std::string& s) {
  if (s == "decode") return StepKind::Decode;
  if (s == "prefill") return StepKind::Prefill;
  throw ValidationError("unknown step kind: " + s);
}

int TraceStep::token_count(int top_k) const {
  if (kind == StepKind::Decode) return 1;
  if (layers.empty()) return 0;
  std::int64_t n = 0;
  for (const Selection& s : layers.front()) n += s.token_count;
  return static_cast<int>(n / top_k);
}

namespace {

[[noreturn]] void step_error(size_t idx, const char* what) {
  throw ValidationError("trace step " + std::to_string(idx) + ": " + what);
}

void check_step(const TraceStep& st, const ModelShape& shape, size_t idx) {
  if (static_cast<int>(st.layers.size()) != shape.num_layers)
    step_error(idx, "layer count does not match shape");
  std::int64_t first_total = -1;
  for (const auto& sels : st.layers) {
    std::vector<char> seen(shape.experts_per_layer, 0);
    std::int64_t total = 0;
    for (const Selection& s : sels) {
      if (s.expert < 0 || s.expert >= shape.experts_per_layer)
        step_error(idx, "expert id out of range");
      if (seen[s.expert]) step_error(idx, "duplicate expert in layer selection");
      seen[s.expert] = 1;
      if (s.token_count < 1) step_error(idx, "token_count must be >= 1");
      if (!(s.gate_weight > 0.0)) step_error(idx, "gate_weight must be positive");
      total += s.token_count;
    }
    if (st.kind == StepKind::Decode) {
      if (static_cast<int>(sels.size()) != shape.top_k)
        step_error(idx, "decode step must select exactly top_k experts per layer");
      for (const Selection& s : sels)
        if (s.token_count != 1) step_error(idx, "decode selections must carry exactly one token");
      continue;
    }
    if (total % shape.top_k != 0) step_error(idx, "prefill token total must be a multiple of top_k");
    if (first_total < 0) first_total = total;
    if (total != first_total) step_error(idx, "prefill token totals differ across layers");
    const std::int64_t n_tok = total / shape.top_k;
    if (n_tok < 1) step_error(idx, "prefill step must carry tokens");
    if (static_cast<std::int64_t>(sels.size()) <
        std::min<std::int64_t>(shape.top_k, shape.experts_per_layer))
      step_error(idx, "prefill layer selects fewer than top_k experts");
    for (const Selection& s : sels)
      if (s.token_count > n_tok) step_error(idx, "expert receives more tokens than the step carries");
  }
}

// Minimal JSON reader for the trace line format (objects, arrays, numbers,
// strings) — enough for {"kind":...,"layers":[[[e,n,g],...],...]}.
struct Json {
  const std::string& s;
  size_t i = 0;
  explicit Json(const std::string& str) : s(str) {}
  void ws() {
    while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
  }
  bool eat(char c) {
    ws();
    if (i < s.size() && s[i] == c) {
      ++i;
      return true;
    }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) throw ValidationError(std::string("expected '") + c + "'");
  }
  std::string str() {
    expect('"');
    std::string out;
    while (i < s.size() && s[i] != '"') out += s[i++];
    expect('"');
    return out;
  }
  // JSON number grammar only (RFC 8259 §6): -?(0|[1-9][0-9]*)(.[0-9]+)?([eE][+-]?[0-9]+)?
  // — no inf/nan, hex floats, leading '+' or bare '.5' (std::stod accepts them)
  double num() {
    ws();
    const size_t b = i;
    size_t p = i;
    auto digits = [&] {
      const size_t q = p;
      while (p < s.size() && s[p] >= '0' && s[p] <= '9') ++p;
      return p > q;
    };
    if (p < s.size() && s[p] == '-') ++p;
    if (p < s.size() && s[p] == '0') ++p;
    else if (!digits()) throw ValidationError("malformed number");
    if (p < s.size() && s[p] == '.') {
      ++p;
      if (!digits()) throw ValidationError("malformed number");
    }
    if (p < s.size() && (s[p] == 'e' || s[p] == 'E')) {
      ++p;
      if (p < s.size() && (s[p] == '+' || s[p] == '-')) ++p;
      if (!digits()) throw ValidationError("malformed number");
    }
    i = p;
    return std::strtod(s.substr(b, p - b).c_str(), nullptr);
  }
  void end() {
    ws();
    if (i != s.size()) throw ValidationError("unexpected text after the JSON object");
  }
};

}  // namespace

void RoutingTrace::validate(const ModelShape& shape) const {
  shape.validate();
  for (size_t i = 0; i < steps.size(); ++i) check_step(steps[i], shape, i);
}

void save_trace_jsonl(const RoutingTrace& trace, std::ostream& out) {
  out.precision(17);
  for (const TraceStep& st : trace.steps) {
    out << "{\"kind\":\"" << to_string(st.kind) << "\",\"layers\":[";
    for (size_t l = 0; l < st.layers.size(); ++l) {
      out << (l ? ",[" : "[");
      for (size_t j = 0; j < st.layers[l].size(); ++j) {
        const Selection& s = st.layers[l][j];
        out << (j ? "," : "") << '[' << s.expert << ',' << s.token_count << ',' << s.gate_weight
            << ']';
      }
      out << ']';
    }
    out << "]}\n";
  }
}

void save_trace_jsonl(const RoutingTrace& trace, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw ValidationError("cannot open trace file for writing: " + path);
  save_trace_jsonl(trace, out);
}

RoutingTrace load_trace_jsonl(std::istream& in, const ModelShape& shape) {
  RoutingTrace trace;
  std::string line;
  size_t lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
    TraceStep st;
    // parse errors name the line, as the reference loader does (trace.cpp:116-124)
    try {
      Json j(line);
      bool have_kind = false, have_layers = false;
      j.expect('{');
      do {
        const std::string key = j.str();
        j.expect(':');
        if (key == "kind") {
          st.kind = step_kind_from_string(j.str());
          have_kind = true;
        } else if (key == "layers") {
          j.expect('[');
          if (!j.eat(']')) {
            do {
              std::vector<Selection> sels;
              j.expect('[');
              if (!j.eat(']')) {
                do {
                  j.expect('[');
                  Selection s;
                  s.expert = static_cast<int>(j.num());
                  j.expect(',');
                  s.token_count = static_cast<int>(j.num());
                  j.expect(',');
                  s.gate_weight = j.num();
                  j.expect(']');
                  sels.push_back(s);
                } while (j.eat(','));
                j.expect(']');
              }
              st.layers.push_back(std::move(sels));
            } while (j.eat(','));
            j.expect(']');
          }
          have_layers = true;
        } else {
          throw ValidationError("unknown key " + key);
        }
      } while (j.eat(','));
      j.expect('}');
      j.end();
      if (!have_kind || !have_layers) throw ValidationError("missing kind or layers");
    } catch (const ValidationError& e) {
      throw ValidationError("trace line " + std::to_string(lineno) + ": " + e.what());
    }
    trace.steps.push_back(std::move(st));
  }
  trace.validate(shape);
  return trace;
}

RoutingTrace load_trace_jsonl(const std::string& path, const ModelShape& shape) {
  std::ifstream in(path);
  if (!in) throw ValidationError("cannot open trace file: " + path);
  return load_trace_jsonl(in, shape);
}

// ---- seeded init (host; bit-identical to the reference's stream) ------------
namespace {
Matrix gaussian(int rows, int cols, std::mt19937_64& rng, double stddev) {
  Matrix m(rows, cols);
  std::normal_distribution<double> normal(0.0, stddev);  // one object per matrix
  std::generate(m.data.begin(), m.data.end(), [&] { return normal(rng); });
  return m;
}
}  // namespace

ModelWeights random_model(const ModelShape& shape, std::uint64_t seed) {
  shape.validate();
  std::mt19937_64 rng(seed);
  const double stddev = 1.0 / std::sqrt(static_cast<double>(shape.hidden_dim));
  const int d = shape.hidden_dim, f = shape.ffn_dim, E = shape.experts_per_layer;
  ModelWeights w;
  w.experts.assign(shape.num_layers, {});
  for (int l = 0; l < shape.num_layers; ++l) {
    auto& layer = w.experts[l];
    layer.resize(E);
    for (int e = 0; e < E; ++e) {
      layer[e].w_in = gaussian(f, d, rng, stddev);
      layer[e].w_gate = gaussian(f, d, rng, stddev);
      layer[e].w_out = gaussian(d, f, rng, stddev);
    }
    w.router.layers.push_back(gaussian(E, d, rng, stddev));
  }
  return w;
}

RoutingTrace synth_trace(const ModelShape& shape, double popularity_skew, int input_len,
                         int output_len, std::uint64_t seed) {
  shape.validate();
  if (input_len < 1) throw ValidationError("input_len must be >= 1");
  if (output_len < 0) throw ValidationError("output_len must be >= 0");
  const int L = shape.num_layers, E = shape.experts_per_layer, k = shape.top_k;
  // per-layer log popularity: rank weights (r+1)^-skew, shuffled per layer
  std::vector<std::vector<double>> logw(L, std::vector<double>(E));
  for (int l = 0; l < L; ++l) {
    std::vector<double> wts(E);
    for (int e = 0; e < E; ++e) wts[e] = std::pow(static_cast<double>(e + 1), -popularity_skew);
    std::mt19937_64 perm(seed ^ (0x9e3779b97f4a7c15ULL * static_cast<std::uint64_t>(l + 1)));
    std::shuffle(wts.begin(), wts.end(), perm);
    for (int e = 0; e < E; ++e) logw[l][e] = std::log(wts[e]);
  }
  std::mt19937_64 rng(seed);
  // Gumbel-top-k draw of k distinct experts, ascending ids
  auto draw = [&](int l) {
    std::uniform_real_distribution<double> u(1e-12, 1.0);
    std::vector<std::pair<double, int>> keyed(E);
    for (int e = 0; e < E; ++e) keyed[e] = {logw[l][e] - std::log(-std::log(u(rng))), e};
    std::partial_sort(keyed.begin(), keyed.begin() + k, keyed.end(),
                      [](const auto& a, const auto& b) { return a.first > b.first; });
    std::vector<int> ids(k);
    for (int i = 0; i < k; ++i) ids[i] = keyed[i].second;
    std::sort(ids.begin(), ids.end());
    return ids;
  };
  auto gates = [&] {
    std::uniform_real_distribution<double> u(0.05, 1.0);
    std::vector<double> g(k);
    double sum = 0.0;
    for (double& v : g) sum += (v = u(rng));
    for (double& v : g) v /= sum;
    return g;
  };
  RoutingTrace trace;
  TraceStep pre;
  pre.kind = StepKind::Prefill;
  pre.layers.resize(L);
  for (int l = 0; l < L; ++l) {
    std::vector<int> cnt(E, 0);
    std::vector<double> gs(E, 0.0);
    for (int t = 0; t < input_len; ++t) {
      const auto ids = draw(l);
      const auto g = gates();
      for (int i = 0; i < k; ++i) {
        ++cnt[ids[i]];
        gs[ids[i]] += g[i];
      }
    }
    for (int e = 0; e < E; ++e)
      if (cnt[e]) pre.layers[l].push_back({e, cnt[e], gs[e] / cnt[e]});
  }
  trace.steps.push_back(std::move(pre));
  for (int t = 0; t < output_len; ++t) {
    TraceStep dec;
    dec.kind = StepKind::Decode;
    dec.layers.resize(L);
    for (int l = 0; l < L; ++l) {
      const auto ids = draw(l);
      const auto g = gates();
      for (int i = 0; i < k; ++i) dec.layers[l].push_back({ids[i], 1, g[i]});
    }
    trace.steps.push_back(std::move(dec));
  }
  return trace;
}

// ---- placement ----------------------------------------------------------------
PopularityProfile PopularityProfile::zeros(const ModelShape& shape) {
  PopularityProfile p;
  p.counts.assign(shape.num_layers, std::vector<std::int64_t>(shape.experts_per_layer, 0));
  return p;
}

PopularityProfile PopularityProfile::uniform(int num_layers, int experts_per_layer,
                                             std::int64_t count_per_expert) {
  PopularityProfile p;
  p.counts.assign(num_layers, std::vector<std::int64_t>(experts_per_layer, count_per_expert));
  p.total_selections = static_cast<std::int64_t>(num_layers) * experts_per_layer * count_per_expert;
  return p;
}

PopularityProfile profile_from_trace(const RoutingTrace& trace, const ModelShape& shape) {
  trace.validate(shape);
  PopularityProfile p = PopularityProfile::zeros(shape);
  for (const TraceStep& st : trace.steps)
    for (size_t l = 0; l < st.layers.size(); ++l)
      for (const Selection& s : st.layers[l]) {
        p.counts[l][s.expert] += s.token_count;
        p.total_selections += s.token_count;
      }
  return p;
}

namespace {
// (layer, expert) flat indices by count desc, then (layer, expert) asc.
std::vector<std::pair<int, int>> popularity_order(const PopularityProfile& p) {
  std::vector<std::pair<int, int>> order;
  for (int l = 0; l < p.num_layers(); ++l)
    for (int e = 0; e < p.experts_per_layer(); ++e) order.emplace_back(l, e);
  std::stable_sort(order.begin(), order.end(), [&](const auto& a, const auto& b) {
    return p.counts[a.first][a.second] > p.counts[b.first][b.second];
  });
  return order;
}
}  // namespace

Placement greedy_place(const PopularityProfile& profile, int capacity, bool per_layer_quota) {
  if (capacity < 0) throw ValidationError("capacity must be >= 0");
  Placement pl;
  pl.capacity = capacity;
  if (!per_layer_quota) {
    const auto order = popularity_order(profile);
    const size_t take = std::min<size_t>(capacity, order.size());
    pl.resident.insert(order.begin(), order.begin() + take);
    return pl;
  }
  const int L = profile.num_layers();
  if (L == 0) return pl;
  const int quota = capacity / L;
  for (int l = 0; l < L; ++l) {
    std::vector<int> ex(profile.experts_per_layer());
    std::iota(ex.begin(), ex.end(), 0);
    std::stable_sort(ex.begin(), ex.end(), [&](int a, int b) {
      return profile.counts[l][a] > profile.counts[l][b];
    });
    for (int i = 0; i < std::min<int>(quota, static_cast<int>(ex.size())); ++i)
      pl.resident.insert({l, ex[i]});
  }
  return pl;
}

double expected_hit_rate(const Placement& placement, const PopularityProfile& profile) {
  if (profile.total_selections <= 0)
    throw ValidationError("hit rate undefined: profile has no selections");
  std::int64_t hits = 0;
  for (const auto& [l, e] : placement.resident) hits += profile.counts[l][e];
  return static_cast<double>(hits) / static_cast<double>(profile.total_selections);
}

HitRateBounds hit_rate_bounds(const PopularityProfile& profile, int capacity) {
  if (profile.total_selections <= 0)
    throw ValidationError("hit rate undefined: profile has no selections");
  const auto order = popularity_order(profile);
  const int n = static_cast<int>(order.size());
  const int take = std::min(capacity, n);
  std::int64_t best = 0, worst = 0;
  for (int i = 0; i < take; ++i) {
    best += profile.counts[order[i].first][order[i].second];
    worst += profile.counts[order[n - 1 - i].first][order[n - 1 - i].second];
  }
  HitRateBounds b;
  b.best = static_cast<double>(best) / profile.total_selections;
  b.worst = static_cast<double>(worst) / profile.total_selections;
  b.random = static_cast<double>(take) / static_cast<double>(profile.total_experts());
  return b;
}

std::vector<double> sparsity_histogram(const std::vector<double>& activations,
                                       const std::vector<double>& thresholds) {
  if (activations.empty())
    throw ValidationError("sparsity histogram undefined on empty activations");
  if (std::adjacent_find(thresholds.begin(), thresholds.end(), std::greater_equal<double>()) !=
      thresholds.end())
    throw ValidationError("thresholds must be strictly increasing");
  std::vector<double> frac(thresholds.size(), 0.0);
  for (double a : activations) {
    const double m = std::fabs(a);
    for (size_t i = 0; i < thresholds.size(); ++i)
      if (m < thresholds[i]) frac[i] += 1.0;
  }
  for (double& f : frac) f /= static_cast<double>(activations.size());
  return frac;
}

ProfileStats profile_stats(const PopularityProfile& profile) {
  std::int64_t mx = 0;
  for (const auto& row : profile.counts)
    for (std::int64_t c : row) mx = std::max(mx, c);
  if (mx == 0) throw ValidationError("profile stats undefined: all counts zero");
  std::vector<double> v;
  for (const auto& row : profile.counts)
    for (std::int64_t c : row) v.push_back(static_cast<double>(c) / static_cast<double>(mx));
  std::sort(v.begin(), v.end());
  const double n = static_cast<double>(v.size());
  const double mean = std::accumulate(v.begin(), v.end(), 0.0) / n;
  double var = 0.0;
  for (double x : v) var += (x - mean) * (x - mean);
  auto quantile = [&](double q) {  // linear interpolation between order stats
    const double pos = q * (n - 1.0);
    const size_t lo = static_cast<size_t>(std::floor(pos));
    const size_t hi = std::min(lo + 1, v.size() - 1);
    const double t = pos - static_cast<double>(lo);
    return v[lo] * (1.0 - t) + v[hi] * t;
  };
  ProfileStats st;
  st.mean = mean;
  st.stddev = std::sqrt(var / n);
  st.p25 = quantile(0.25);
  st.p75 = quantile(0.75);
  st.min = v.front();
  st.max = v.back();
  return st;
}

namespace {
std::vector<std::string> split_csv(const std::string& line) {
  std::vector<std::string> out;
  std::stringstream ss(line);
  std::string f;
  while (std::getline(ss, f, ',')) out.push_back(f);
  return out;
}
long long parse_int(const std::string& s, const std::string& where) {
  size_t used = 0;
  long long v = 0;
  try {
    v = std::stoll(s, &used);
  } catch (const std::exception&) {
    throw ValidationError(where + ": malformed numeric field");
  }
  if (used != s.size()) throw ValidationError(where + ": malformed numeric field");
  return v;
}
}  // namespace

void save_profile_csv(const PopularityProfile& profile, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw ValidationError("cannot open profile CSV for writing: " + path);
  out << "layer,expert,count\n";
  for (int l = 0; l < profile.num_layers(); ++l)
    for (int e = 0; e < profile.experts_per_layer(); ++e)
      out << l << ',' << e << ',' << profile.counts[l][e] << '\n';
}

PopularityProfile load_profile_csv(std::istream& in) {
  std::map<std::pair<int, int>, std::int64_t> cells;
  int L = 0, E = 0;
  std::string line;
  size_t lineno = 0;
  bool header = false;
  while (std::getline(in, line)) {
    ++lineno;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty()) continue;
    if (!header) {
      if (line != "layer,expert,count") throw ValidationError("profile CSV: bad header");
      header = true;
      continue;
    }
    const std::string where = "profile CSV line " + std::to_string(lineno);
    const auto f = split_csv(line);
    if (f.size() != 3) throw ValidationError(where + ": expected 3 fields");
    const int l = static_cast<int>(parse_int(f[0], where));
    const int e = static_cast<int>(parse_int(f[1], where));
    const std::int64_t c = parse_int(f[2], where);
    if (l < 0 || e < 0 || c < 0) throw ValidationError(where + ": negative field");
    cells[{l, e}] = c;
    L = std::max(L, l + 1);
    E = std::max(E, e + 1);
  }
  if (cells.empty()) throw ValidationError("profile CSV has no data rows");
  PopularityProfile p;
  p.counts.assign(L, std::vector<std::int64_t>(E, 0));
  for (const auto& [le, c] : cells) {
    p.counts[le.first][le.second] = c;
    p.total_selections += c;
  }
  return p;
}

PopularityProfile load_profile_csv(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ValidationError("cannot open profile CSV: " + path);
  return load_profile_csv(in);
}

void save_placement_csv(const Placement& placement, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw ValidationError("cannot open placement CSV for writing: " + path);
  out << "# capacity=" << placement.capacity << "\nlayer,expert\n";
  for (const auto& [l, e] : placement.resident) out << l << ',' << e << '\n';
}

Placement load_placement_csv(std::istream& in) {
  Placement pl;
  std::string line;
  size_t lineno = 0;
  bool header = false;
  while (std::getline(in, line)) {
    ++lineno;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty()) continue;
    const std::string cap = "# capacity=";
    if (line.compare(0, cap.size(), cap) == 0) {
      pl.capacity = static_cast<int>(parse_int(line.substr(cap.size()), "placement CSV"));
      continue;
    }
    if (!header) {
      if (line != "layer,expert") throw ValidationError("placement CSV: expected header layer,expert");
      header = true;
      continue;
    }
    const std::string where = "placement CSV line " + std::to_string(lineno);
    const auto f = split_csv(line);
    if (f.size() < 2) throw ValidationError(where + ": expected 2 fields");
    pl.resident.insert({static_cast<int>(parse_int(f[0], where)),
                        static_cast<int>(parse_int(f[1], where))});
  }
  if (static_cast<int>(pl.resident.size()) > pl.capacity)
    throw ValidationError("placement CSV: resident set exceeds capacity");
  return pl;
}

Placement load_placement_csv(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ValidationError("cannot open placement CSV: " + path);
  return load_placement_csv(in);
}

// ---- expert-parallel shard map ------------------------------------------------
namespace b200 {

std::vector<std::vector<int>> ep_shard_map(const PopularityProfile& profile, int world) {
  if (world < 1) throw ValidationError("world must be >= 1");
  const int L = profile.num_layers(), E = profile.experts_per_layer();
  const int cap = (E + world - 1) / world;
  std::vector<std::vector<int>> owner(L, std::vector<int>(E, 0));
  for (int l = 0; l < L; ++l) {
    std::vector<int> order(E);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      return profile.counts[l][a] > profile.counts[l][b];
    });
    std::vector<std::int64_t> load(world, 0);
    std::vector<int> held(world, 0);
    for (int e : order) {
      int best = -1;
      for (int r = 0; r < world; ++r)
        if (held[r] < cap && (best < 0 || load[r] < load[best])) best = r;
      owner[l][e] = best;
      load[best] += profile.counts[l][e];
      ++held[best];
    }
  }
  return owner;
}

std::vector<std::vector<int>> ep_shard_map_coselect(
    const PopularityProfile& profile,
    const std::vector<std::vector<std::vector<std::int64_t>>>& pair_counts, int world) {
  if (world < 1) throw ValidationError("world must be >= 1");
  const int L = profile.num_layers(), E = profile.experts_per_layer();
  if (static_cast<int>(pair_counts.size()) != L) throw ValidationError("pair counts: one matrix per layer");
  std::vector<std::vector<int>> owner(L, std::vector<int>(E, 0));
  std::vector<std::int64_t> pair(static_cast<size_t>(E) * E), pop(E);
  for (int l = 0; l < L; ++l) {
    if (static_cast<int>(pair_counts[l].size()) != E) throw ValidationError("pair counts: E x E per layer");
    for (int a = 0; a < E; ++a) {
      if (static_cast<int>(pair_counts[l][a].size()) != E) throw ValidationError("pair counts: E x E per layer");
      for (int b = 0; b < E; ++b) {
        if (pair_counts[l][a][b] < 0) throw ValidationError("negative co-selection count");
        pair[static_cast<size_t>(a) * E + b] = pair_counts[l][a][b];
      }
      pop[a] = profile.counts[l][a];
    }
    moe::coselect_layer(pair.data(), pop.data(), E, world, owner[l].data());
  }
  return owner;
}

std::vector<std::vector<std::uint32_t>> ep_replica_masks(const PopularityProfile& profile,
                                                         int world, int hot) {
  if (world < 1 || world > 8) throw ValidationError("replicas need 1 <= world <= 8");
  if (hot < 0) throw ValidationError("hot must be >= 0");
  const int L = profile.num_layers(), E = profile.experts_per_layer();
  std::vector<std::vector<std::uint32_t>> mask(L, std::vector<std::uint32_t>(E, 0u));
  for (int l = 0; l < L; ++l) {
    std::vector<int> order(E);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      return profile.counts[l][a] > profile.counts[l][b];
    });
    for (int i = 0; i < std::min(hot, E); ++i) mask[l][order[i]] = (1u << world) - 1u;
  }
  return mask;
}

PopularityProfile profile_from_counts(const std::vector<std::vector<std::int64_t>>& counts) {
  PopularityProfile p;
  p.counts = counts;
  for (const auto& row : counts) {
    if (row.size() != counts.front().size()) throw ValidationError("ragged routing counts");
    for (std::int64_t c : row) {
      if (c < 0) throw ValidationError("negative routing count");
      p.total_selections += c;
    }
  }
  return p;
}

Placement rank_placement(const std::vector<std::vector<int>>& owner, int rank) {
  Placement pl;
  for (size_t l = 0; l < owner.size(); ++l)
    for (size_t e = 0; e < owner[l].size(); ++e)
      if (owner[l][e] == rank) pl.resident.insert({static_cast<int>(l), static_cast<int>(e)});
  pl.capacity = static_cast<int>(pl.resident.size());
  return pl;
}

}  // namespace b200
}  // namespace moe_orch
