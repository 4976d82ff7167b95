// replica_plan.h — per-step token split of replicated experts over the ranks
// that hold them.  Shared by the device planner kernel
// (prefill.cu), the host entry point moe_replica_plan (capi_weights.cu) and tests.
//
// The reference's scheduler (scheduler.cpp:97-204) splits one layer's active
// experts between two devices so that max(slow_sum, fast_sum) is minimal, ties
// to the smaller fast-device cost (scheduler.cpp:128-140); its greedy variant
// takes experts by token count desc, id asc (scheduler.cpp:154-188).  Under
// expert parallelism the "devices" are the G ranks and the choice is, for a
// hot expert held by several ranks, how many of its holders run a share of
// its tokens.  Cost of running m rows of one expert on one rank (the B200
// roofline of the grouped GEMM plus a fixed ramp): part_ps + max(weight_ps,
// m * row_ps) — streaming the expert's weights once vs the tensor-core time
// of its rows.  Splitting over
// q holders costs the weight stream q times, so it only wins when the expert
// is compute-bound (large prefill batches); decode never splits.
//
// Experts held by one rank are fixed load, placed first.  The greedy
// objective of one choice for a replicated expert is max(largest rank load
// after it, the mean load after it plus the unsplit cost of the replicated
// experts still to place): the bare max would split even a barely
// compute-bound expert onto idle ranks and pay its weight stream twice for
// nothing (LPT's lower bound).  Ties go to the smaller largest load (a
// compute-bound expert splits at no extra cost while the mean bound binds),
// then to fewer holders.
//
// Rows are split at `chunk`-row boundaries (the grouped kernel's token tile)
// and every rank evaluates the same integer arithmetic on the same counts, so
// the plan is identical on all ranks without any exchange.
#pragma once

#include <stdint.h>

#if defined(__CUDACC__)
#define MOE_HD __host__ __device__ __forceinline__
#else
#define MOE_HD inline
#endif

namespace moe {

constexpr int kReplicaMaxRanks = 8;

struct ReplicaCost {
  long long weight_ps;  // time to stream one expert's weights (this rank's share), ps
  long long row_ps;     // tensor-core time per (token, slot) row, ps
  long long part_ps;    // fixed cost of running any rows of one expert (pipeline ramp), ps
  int chunk;            // split granularity in rows
};

MOE_HD long long replica_run_cost(int rows, const ReplicaCost& c) {
  const long long flops = (long long)rows * c.row_ps;
  return c.part_ps + (flops > c.weight_ps ? flops : c.weight_ps);
}

MOE_HD int replica_popcount(uint32_t v) {
  int n = 0;
  for (; v; v &= v - 1u) ++n;
  return n;
}

// order: experts sorted by (counts desc, id asc).  holders[e]: bit r set when
// rank r holds expert e (0 = nobody: its rows are not computed).  Experts with
// one holder are fixed load and placed first; then each replicated expert, in
// order, tries q = 1.. of its least-loaded holders, dealing its chunks one at
// a time to the holder whose load grows least (water-filling), and keeps the
// q with the best objective.  Writes, for rank `rank`, [lo[e], hi[e]) of
// expert e's rows (lo == hi: not on this rank; parts are laid out in holder
// order) and returns the plan's makespan (max rank load, ps).
MOE_HD long long replica_split_plan(const int32_t* counts, const int32_t* order, int E,
                                    const uint32_t* holders, int world, const ReplicaCost& c,
                                    int rank, int32_t* lo, int32_t* hi) {
  const int nw = world < kReplicaMaxRanks ? world : kReplicaMaxRanks;
  long long load[kReplicaMaxRanks];
  for (int r = 0; r < kReplicaMaxRanks; ++r) load[r] = 0;
  long long rem = 0;  // unsplit cost of the replicated experts not yet placed
  for (int e = 0; e < E; ++e) {
    lo[e] = hi[e] = 0;
    const uint32_t h = holders[e] & ((1u << nw) - 1u);
    if (counts[e] <= 0 || h == 0u) continue;
    if (replica_popcount(h) == 1) {
      int r = 0;
      while (!((h >> r) & 1u)) ++r;
      load[r] += replica_run_cost(counts[e], c);
      if (r == rank) hi[e] = counts[e];
    } else {
      rem += replica_run_cost(counts[e], c);
    }
  }
  for (int i = 0; i < E; ++i) {
    const int e = order[i];
    const int m = counts[e];
    const uint32_t h = holders[e] & ((1u << nw) - 1u);
    if (m <= 0 || replica_popcount(h) < 2) continue;
    // holders by (load, rank) ascending
    int cand[kReplicaMaxRanks];
    int nc = 0;
    for (int r = 0; r < nw; ++r)
      if ((h >> r) & 1u) {
        int j = nc++;
        while (j > 0 && (load[cand[j - 1]] > load[r] ||
                         (load[cand[j - 1]] == load[r] && cand[j - 1] > r))) {
          cand[j] = cand[j - 1];
          --j;
        }
        cand[j] = r;
      }
    rem -= replica_run_cost(m, c);
    const int nch = (m + c.chunk - 1) / c.chunk;
    int best_cnt[kReplicaMaxRanks];
    long long best = -1, best_max = -1;
    for (int q = 1; q <= nc && q <= nch; ++q) {
      int cnt[kReplicaMaxRanks];
      for (int p = 0; p < q; ++p) cnt[p] = 0;
      for (int j = 0; j < nch; ++j) {
        int bp = 0;
        long long bv = -1;
        for (int p = 0; p < q; ++p) {
          const long long v = load[cand[p]] + replica_run_cost((cnt[p] + 1) * c.chunk, c);
          if (bv < 0 || v < bv) {
            bv = v;
            bp = p;
          }
        }
        ++cnt[bp];
      }
      long long mx = 0, sum = rem;
      for (int r = 0; r < nw; ++r) {
        long long v = load[r];
        for (int p = 0; p < q; ++p)
          if (cand[p] == r) {
            int r0 = 0;
            for (int pp = 0; pp < p; ++pp) r0 += cnt[pp] * c.chunk;
            const int a = r0 < m ? r0 : m;
            const int b = r0 + cnt[p] * c.chunk < m ? r0 + cnt[p] * c.chunk : m;
            if (b > a) v += replica_run_cost(b - a, c);
          }
        mx = v > mx ? v : mx;
        sum += v;
      }
      const long long mean = (sum + nw - 1) / nw;
      const long long obj = mean > mx ? mean : mx;
      // ties: smaller largest load, then fewer holders (less weight traffic)
      if (best < 0 || obj < best || (obj == best && mx < best_max)) {
        best = obj;
        best_max = mx;
        for (int p = 0; p < kReplicaMaxRanks; ++p) best_cnt[p] = p < q ? cnt[p] : 0;
      }
    }
    int r0 = 0;
    for (int p = 0; p < nc; ++p) {
      const int a = r0 < m ? r0 : m;
      const int b = r0 + best_cnt[p] * c.chunk < m ? r0 + best_cnt[p] * c.chunk : m;
      r0 += best_cnt[p] * c.chunk;
      if (b <= a) continue;
      load[cand[p]] += replica_run_cost(b - a, c);
      if (cand[p] == rank) {
        lo[e] = a;
        hi[e] = b;
      }
    }
  }
  long long mk = 0;
  for (int r = 0; r < nw; ++r) mk = load[r] > mk ? load[r] : mk;
  return mk;
}

// Position of expert e in the (counts desc, id asc) order.
MOE_HD int replica_order_pos(const int32_t* counts, int E, int e) {
  int pos = 0;
  for (int j = 0; j < E; ++j)
    if (counts[j] > counts[e] || (counts[j] == counts[e] && j < e)) ++pos;
  return pos;
}

}  // namespace moe
