// moe_orch/b200.hpp — B200-specific additions to the drop-in API.
#pragma once

#include <cstdint>
#include <vector>

#include "moe_orch/placement.hpp"

namespace moe_orch::b200 {

enum class Dtype { BF16 = 0, F32 = 1 };

// Device-side storage type of the expert weights used by expert_ffn /
// model_forward (default F32: closest to the fp64 reference; BF16 is the
// serving configuration).  The residual stream and accumulation are fp32.
void set_dtype(Dtype dtype);
Dtype dtype();
// CUDA device used by the drop-in entry points (default 0 / $MOE_B200_DEVICE).
void set_device(int device);
// Device copies of ModelWeights are cached by a digest of their full
// contents (an in-place edit anywhere is seen); this drops the cache.
void invalidate_weights_cache();

// The paper's popularity placement re-expressed as expert parallelism:
// owner[l][e] in [0, world).  Per layer, experts are taken in the reference
// ranking (count desc, expert asc — placement.cpp:53-64) and assigned to the
// least-loaded rank with spare slots (LPT; ties to the lower rank), each rank
// holding ceil(E / world) experts at most.
std::vector<std::vector<int>> ep_shard_map(const PopularityProfile& profile, int world);
// Co-selection-aware variant: per layer, the balanced map
// (floor/ceil(E / world) experts per rank) that minimises the co-selections
// of experts sharing a rank — pair_counts[l][a][b] tokens chose both a and b
// (moe_routing_pair_histogram, read back) — since a batch-1 token whose
// top-2 share a rank streams both there; ties to the smaller largest
// popularity load; deterministic.  Pairwise-swap local search from
// ep_shard_map's map, then an exact branch and bound seeded with it under a
// node budget (shard_plan.h).  ValidationError on shape mismatch or negative counts.
std::vector<std::vector<int>> ep_shard_map_coselect(
    const PopularityProfile& profile,
    const std::vector<std::vector<std::vector<std::int64_t>>>& pair_counts, int world);
// profile_from_trace (placement.cpp:30-43) from per-(layer, expert) selection
// counts, e.g. a device routing histogram (moe_routing_histogram) read back
// after a calibration run; ValidationError on ragged rows or negative counts.
PopularityProfile profile_from_counts(const std::vector<std::vector<std::int64_t>>& counts);
// Replicated hot experts (moe_weights_create_ep's replica_mask): per layer
// the `hot` most popular experts (same ranking) are held by every rank; the
// prefill path then splits their tokens over the holders per step by the
// scheduler's min-max objective (scheduler.cpp:97-204).  world <= 8.
std::vector<std::vector<std::uint32_t>> ep_replica_masks(const PopularityProfile& profile,
                                                         int world, int hot);
// Rank r's share as a Placement (capacity = its expert count).
Placement rank_placement(const std::vector<std::vector<int>>& owner, int rank);

}  // namespace moe_orch::b200
