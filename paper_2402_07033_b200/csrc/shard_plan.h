// shard_plan.h — co-selection-aware expert-parallel shard map (SURVEY §8e:
// "a shard map that separates frequently co-selected pairs (a
// co-occurrence-aware extension of greedy_place) lowers the G=2 and G=4
// figures").  Host code shared by the C-ABI (moe_ep_shard_map_coselect,
// capi_weights.cu) and the drop-in (b200::ep_shard_map_coselect,
// moe_orch_host.cpp).
//
// At batch 1 under expert parallelism a layer costs the largest number of the
// token's k experts held by one rank (each streams its experts' weights; the
// others wait at the combine): with top-2, 1 expert-stream when the two land
// on different ranks, 2 when they share one.  Summed over a calibration
// trace, sum_t (1 + [rank(e1_t) == rank(e2_t)]) = T + sum over co-located
// pairs of pair[e1][e2], so the map minimises the co-located co-selection
// count (for k > 2 this pair count is the proxy), subject to the memory
// balance of the popularity map: every rank holds floor(E/G) or ceil(E/G)
// experts.  Ties go to the smaller largest per-rank popularity load (the
// prefill balance greedy_place/LPT aims at); the search is deterministic, so
// every rank computes the same map.
//
// First a pairwise-swap local search from the popularity LPT map
// (ep_shard_map's; first improvement in (e1, e2) order until no swap
// improves (cost, load)), then an exact branch and bound over the set
// partitions (ranks labelled by first appearance) seeded with it, under a
// node budget (E <= 24): exact when it finishes, else the best map found.
#pragma once

#include <stdint.h>

#include <algorithm>
#include <numeric>
#include <vector>

namespace moe {

struct CoselectCost {
  int64_t pair = 0, load = 0;  // co-located co-selections, largest rank load
  bool operator<(const CoselectCost& o) const { return pair != o.pair ? pair < o.pair : load < o.load; }
};

// pair: [E x E] (entries e1 < e2 used: pair[e1*E+e2] + pair[e2*E+e1]),
// pop: [E] selections per expert, owner: [E] rank per expert
inline CoselectCost coselect_cost(const int64_t* pair, const int64_t* pop, const int* owner, int E,
                                  int world) {
  CoselectCost c;
  for (int a = 0; a < E; ++a)
    for (int b = a + 1; b < E; ++b)
      if (owner[a] == owner[b]) c.pair += pair[a * E + b] + pair[b * E + a];
  std::vector<int64_t> load(world, 0);
  for (int e = 0; e < E; ++e) load[owner[e]] += pop[e];
  c.load = world > 0 ? *std::max_element(load.begin(), load.end()) : 0;
  return c;
}

// the popularity LPT map of one layer (ep_shard_map): experts by selections
// desc (stable), each to the least-loaded rank with room (ties: lower rank)
inline void lpt_layer(const int64_t* pop, int E, int world, int* owner) {
  const int cap = (E + world - 1) / world;
  std::vector<int> order(E);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return pop[a] > pop[b]; });
  std::vector<int64_t> load(world, 0);
  std::vector<int> held(world, 0);
  for (int e : order) {
    int best = -1;
    for (int r = 0; r < world; ++r)
      if (held[r] < cap && (best < 0 || load[r] < load[best])) best = r;
    owner[e] = best;
    load[best] += pop[e];
    ++held[best];
  }
}

namespace detail {
struct CoselectSearch {
  const int64_t* pair;
  const int64_t* pop;
  int E, world, hi, n_hi;  // block sizes: n_hi blocks of hi, the rest hi - 1 (or all hi)
  long long nodes = 0, budget;
  std::vector<int> cur, best;
  CoselectCost best_cost;
  bool have = false;
  std::vector<int> size;

  // blocks of size hi used so far must not exceed n_hi
  bool sizes_ok(bool final) const {
    int n_full = 0;
    for (int r = 0; r < world; ++r) {
      if (size[r] > hi) return false;
      n_full += size[r] == hi;
    }
    if (hi * world != E && n_full > n_hi) return false;
    if (final)
      for (int r = 0; r < world; ++r)
        if (size[r] < (hi * world == E ? hi : hi - 1)) return false;
    return true;
  }
  // pc: co-located co-selections of experts [0, e) — only grows as experts
  // are added (counts >= 0), so a branch already above the best is cut
  void rec(int e, int used, int64_t pc) {
    if (++nodes > budget || (have && pc > best_cost.pair)) return;
    if (e == E) {
      if (used != world || !sizes_ok(true)) return;
      const CoselectCost c = coselect_cost(pair, pop, cur.data(), E, world);
      if (!have || c < best_cost) {
        best_cost = c;
        best = cur;
        have = true;
      }
      return;
    }
    // room check: the experts left must fill the blocks not yet opened
    if (E - e < world - used) return;
    for (int r = 0; r <= std::min(used, world - 1); ++r) {
      int64_t add = 0;
      for (int q = 0; q < e; ++q)
        if (cur[q] == r) add += pair[q * E + e] + pair[e * E + q];
      cur[e] = r;
      ++size[r];
      if (sizes_ok(false)) rec(e + 1, used + (r == used), pc + add);
      --size[r];
    }
  }
};
}  // namespace detail

// One layer's map: owner[E] in [0, world).  Returns true when the search was
// exact (finished within the node budget).
inline bool coselect_layer(const int64_t* pair, const int64_t* pop, int E, int world, int* owner,
                           long long node_budget = 2000000) {
  if (world <= 1 || world >= E) {
    for (int e = 0; e < E; ++e) owner[e] = world <= 1 ? 0 : e % world;
    if (world > 1 && world >= E) lpt_layer(pop, E, world, owner);
    return true;
  }
  // local search from the popularity map: the seed (and the fallback).
  // A swap's change is evaluated in O(E + world); passes repeat until one
  // applies no swap ((pair, load) falls strictly at every swap: it ends)
  lpt_layer(pop, E, world, owner);
  CoselectCost c = coselect_cost(pair, pop, owner, E, world);
  std::vector<int64_t> load(world, 0);
  for (int e = 0; e < E; ++e) load[owner[e]] += pop[e];
  auto P = [&](int a, int b) { return pair[a * E + b] + pair[b * E + a]; };
  for (bool improved = true; improved;) {
    improved = false;
    for (int a = 0; a < E; ++a)
      for (int b = a + 1; b < E; ++b) {
        const int ra = owner[a], rb = owner[b];
        if (ra == rb) continue;
        int64_t dp = 0;
        for (int q = 0; q < E; ++q) {
          if (q == a || q == b) continue;
          if (owner[q] == rb) dp += P(a, q) - P(b, q);
          else if (owner[q] == ra) dp += P(b, q) - P(a, q);
        }
        const int64_t la = load[ra] - pop[a] + pop[b], lb = load[rb] - pop[b] + pop[a];
        int64_t mx = std::max(la, lb);
        for (int r = 0; r < world; ++r)
          if (r != ra && r != rb) mx = std::max(mx, load[r]);
        if (dp < 0 || (dp == 0 && mx < c.load)) {
          owner[a] = rb;
          owner[b] = ra;
          load[ra] = la;
          load[rb] = lb;
          c.pair += dp;
          c.load = mx;
          improved = true;
        }
      }
  }
  if (E > 24) return false;  // the exact search cannot finish: keep the local optimum
  detail::CoselectSearch s;
  s.pair = pair;
  s.pop = pop;
  s.E = E;
  s.world = world;
  s.hi = (E + world - 1) / world;
  s.n_hi = E % world == 0 ? world : E % world;
  s.budget = node_budget;
  s.cur.assign(E, 0);
  s.size.assign(world, 0);
  s.best.assign(owner, owner + E);
  s.best_cost = c;
  s.have = true;
  s.rec(0, 0, 0);
  std::copy(s.best.begin(), s.best.end(), owner);
  return s.nodes <= node_budget;
}

}  // namespace moe
