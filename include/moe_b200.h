/*
 * moe_b200.h — C-ABI of the B200-native MoE-layer hot path.
 *
 * Plain pointers and sizes only (no torch / no CUDA types in signatures; a
 * stream is passed as `void*` = cudaStream_t, NULL = the context's stream).
 * Every entry point returns an int status (MOE_OK = 0); moe_last_error()
 * gives the message of the last failure on this thread.
 *
 * Each function replaces a reference interface of the `moe_orch` C++ API
 * (/root/reference/proj/include/moe_orch/...).  The drop-in C++ shim
 * (paper_2402_07033_b200/csrc/moe_orch_device.cpp for the math and
 * moe_orch_host.cpp for placement / trace / shape, headers include/moe_orch/)
 * implements the reference signatures on top of these calls; INTEGRATION.md
 * shows the bindings.
 *
 * Threading: a moe_weights may be used from several threads and streams;
 * calls on one moe_weights are serialized (a per-weights lock on the host,
 * and every call's device work is ordered after the previous call's on
 * whatever stream that ran, because the calls share the weights' scratch).
 * Calls on different moe_weights run concurrently (each has its own stream
 * for the host-buffer entry points).
 */
#ifndef MOE_B200_H
#define MOE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: error.hpp:8-27 taxonomy + device failures ---------- */
enum {
  MOE_OK = 0,
  MOE_ERR_SHAPE = 1,       /* moe_orch::ShapeError       (error.hpp:19-22)  */
  MOE_ERR_VALIDATION = 2,  /* moe_orch::ValidationError  (error.hpp:14-17)  */
  MOE_ERR_CUDA = 3,        /* CUDA runtime / launch failure                  */
  MOE_ERR_NCCL = 4,        /* NCCL failure (expert-parallel exchange)        */
  MOE_ERR_OOM = 5,         /* device allocation failed                       */
  MOE_ERR_ARG = 6,         /* NULL pointer, bad enum, out-of-range id        */
  MOE_ERR_UNSUPPORTED = 7, /* valid request this build cannot serve          */
  MOE_ERR_NO_DEVICE = 8    /* no sm_100 device visible: there is NO CPU path */
};

/* Weight storage type on the device.  The residual stream, router and all
 * accumulation are fp32 in both modes. */
enum { MOE_DTYPE_BF16 = 0, MOE_DTYPE_F32 = 1 };

/* Mirrors moe_orch::ModelShape (shape.hpp:9-35), field for field. */
typedef struct moe_shape {
  int32_t num_layers;
  int32_t experts_per_layer;
  int32_t top_k;
  int32_t hidden_dim;
  int32_t ffn_dim;
  int32_t bytes_per_param;
} moe_shape;

typedef struct moe_ctx moe_ctx;         /* device, stream, scratch, graphs, EP comm */
typedef struct moe_weights moe_weights; /* device-resident experts + fp32 router   */

/* ---- library / context ------------------------------------------------ */
int moe_version(void);
const char* moe_last_error(void);
/* ModelShape::validate (shape.cpp:7-16): MOE_ERR_SHAPE on violation. */
int moe_shape_validate(const moe_shape* shape);
int moe_ctx_create(int device, moe_ctx** out);
/* Destroy every moe_weights created on the context first. */
int moe_ctx_destroy(moe_ctx* ctx);
/* The context's stream (cudaStream_t) used when a call passes stream=NULL. */
void* moe_ctx_stream(moe_ctx* ctx);
int moe_ctx_synchronize(moe_ctx* ctx);
int moe_ctx_sm_count(moe_ctx* ctx);

/* ---- expert parallelism ------------------------------------
 * The paper's popularity placement (placement.cpp:68-95) re-expressed as an
 * expert -> rank shard map.  moe_ep_unique_id fills 128 bytes on rank 0
 * (ncclGetUniqueId); every rank passes the same bytes to moe_ctx_init_ep.
 * NCCL is dlopen'ed: without libnccl the call fails with MOE_ERR_NCCL. */
int moe_ep_unique_id(void* uid128);
int moe_ctx_init_ep(moe_ctx* ctx, int world, int rank, const void* uid128);
int moe_ctx_world(moe_ctx* ctx, int* world, int* rank);
/* Peer-memory combine (SURVEY §8e "native path"): the batch-1 per-layer
 * exchange runs as ONE kernel that pushes this rank's reduced delta into
 * every peer's HBM window over NVLink (P2P stores), releases per-block flags
 * and sums all ranks' deltas in rank order (bit-identical on every rank), in
 * place of ncclAllReduce.  Multi-process: every rank calls
 * moe_ctx_peer_window (exports a 64-byte CUDA IPC handle), the host
 * all-gathers the handles, then moe_ctx_open_peers.  In one process (several
 * contexts, e.g. on one GPU for testing): moe_ctx_link_peers.  Waits are
 * bounded; moe_ctx_peer_check reports a rank that never arrived. */
int moe_ctx_peer_window(moe_ctx* ctx, int world, int max_hidden, void* ipc_handle64);
int moe_ctx_open_peers(moe_ctx* ctx, int world, int rank, const void* handles64);
int moe_ctx_link_peers(moe_ctx* const* ctxs, int world, int max_hidden);
int moe_ctx_peer_check(moe_ctx* ctx);
/* Same, with a multi-token area for up to max_tokens tokens: multi-token
 * (prefill) layers then combine across the ranks with a reduce-scatter +
 * all-gather kernel over the windows (rank-ordered, bit-identical on every
 * rank) instead of ncclAllReduce.  The decode path does not need it. */
int moe_ctx_peer_window_tokens(moe_ctx* ctx, int world, int max_hidden, int max_tokens,
                               void* ipc_handle64);
int moe_ctx_link_peers_tokens(moe_ctx* const* ctxs, int world, int max_hidden, int max_tokens);
/* Testing hook: give this context an expert-parallel (world, rank) with NO
 * communicator.  Weights created on it hold only rank `rank`'s experts and
 * the per-layer exchange is skipped, so x_out = x + (this rank's partial
 * delta); a test sums the ranks' partials itself (e.g. W contexts on one GPU). */
int moe_ctx_set_virtual_rank(moe_ctx* ctx, int world, int rank);

/* ---- weights (ModelWeights, model.hpp:29-49) ---------------------------
 * owner_rank: optional [L*E] shard map (NULL = every expert local).  Only
 * experts owned by the context's rank are allocated.  The router is
 * replicated (fp32). */
int moe_weights_create(moe_ctx* ctx, const moe_shape* shape, int dtype,
                       const int32_t* owner_rank, moe_weights** out);
/* Tensor parallelism: every rank of the context's (world,
 * rank) holds ffn rows [rank*f/world, (rank+1)*f/world) of EVERY expert (W1 /
 * W3 rows, W2 columns), so at batch 1 all ranks stream 1/world of each routed
 * expert and the per-layer exchange sums their partial deltas — the split
 * that uses every GPU's HBM bandwidth, where expert parallelism streams on at
 * most top_k owner GPUs.  upload/download/random take and give the reference
 * layout; download fills only this rank's slice of the full-size buffers. */
int moe_weights_create_tp(moe_ctx* ctx, const moe_shape* shape, int dtype, moe_weights** out);
int moe_weights_tp(const moe_weights* w, int* tp_world, int* tp_rank, int* ffn_local);
/* Expert parallelism with replicated hot experts (the
 * reference scheduler's min-max split, scheduler.cpp:97-204, re-expressed
 * for expert-parallel load balance).  replica_mask: optional [L*E] rank
 * bitmasks; bit r set = rank r also holds expert (l, e) besides its owner
 * (world <= 8).  Decode and the generic kernels run every expert on its
 * owner only; the tcgen05 prefill path splits each expert's sorted rows over
 * its holders per step, on the device, with the plan of moe_replica_plan
 * (identical on all ranks; no host sync, no exchange). */
int moe_weights_create_ep(moe_ctx* ctx, const moe_shape* shape, int dtype,
                          const int32_t* owner_rank, const uint32_t* replica_mask,
                          moe_weights** out);
/* The split's cost model, picoseconds: m rows of one expert on one rank cost
 * part_ps + max(weight_ps, m * row_ps) — a fixed ramp, streaming the
 * expert's weights, tensor-core time per (token, slot) row.  Defaults from
 * the grouped kernel on B200: 6.54 TB/s (3*d*f*esize B), 1.25 PFLOP/s
 * (6*d*f flop per row), part_ps = 2/3 weight_ps. */
/* Measurement: enable = 1 starts recording CUDA events on the launching
 * stream right around every tcgen05 grouped prefill kernel launch of these
 * weights; enable = 0 stops, waits for them and returns the summed kernel
 * time (us) and the number of launches timed.  (The events break the PDL
 * edge into the kernel, so time a separate loop, not the headline one.) */
int moe_debug_kernel_timing(moe_weights* w, int enable, double* total_us, int64_t* launches);
int moe_weights_set_replica_cost(moe_weights* w, int64_t weight_ps, int64_t row_ps,
                                 int64_t part_ps);
int moe_weights_replica_cost(const moe_weights* w, int64_t* weight_ps, int64_t* row_ps,
                             int64_t* part_ps);
/* Host mirror of the device planner (same code, replica_plan.h): experts by
 * (count desc, id asc); each takes the number q of its least-loaded holders
 * that minimises the max rank load, where m rows on a rank cost
 * max(weight_ps, m * row_ps) and rows are dealt in `chunk`-row pieces (ties:
 * fewer holders).  Writes rank `rank`'s rows [lo[e], hi[e]) of every expert
 * and the plan's makespan (ps).  Needs no device. */
int moe_replica_plan(const int32_t* counts, int E, const uint32_t* holders, int world,
                     int64_t weight_ps, int64_t row_ps, int64_t part_ps, int chunk, int rank,
                     int32_t* lo, int32_t* hi, int64_t* makespan);
/* Co-selection-aware expert-parallel shard map (an extension of
 * the popularity placement, placement.cpp:68-95, re-expressed for EP): per
 * layer, owner[l][e] in [0, world) minimising the co-selections
 * pairs[l][a][b] + pairs[l][b][a] of experts on the same rank (at batch 1 a
 * token whose top-2 share a rank streams both there: 2 expert-streams
 * instead of 1), with floor/ceil(E/world) experts per rank; ties to the
 * smaller largest per-rank popularity load counts[l][e]; deterministic.
 * Pairwise-swap local search from the popularity LPT map, then a branch and
 * bound seeded with it: exact[l] = 1 when that finished within its node
 * budget (the map is optimal), else 0 (the best map found).  counts [L x E], pairs
 * [L x E x E] (moe_routing_pair_histogram's, read back), host memory; exact
 * may be NULL.  Needs no device. */
int moe_ep_shard_map_coselect(const int64_t* counts, const int64_t* pairs, int n_layers, int n_experts,
                              int world, int32_t* owner, int32_t* exact);
/* Device co-selection histogram: pairs[l][a][b] (int64, device,
 * [n_layers x n_experts x n_experts], a < b) += the number of tokens of
 * layer l whose top-k holds both a and b, from an ids record
 * [n_layers x n_tok x top_k].  Accumulates across calls, like
 * moe_routing_histogram; feeds moe_ep_shard_map_coselect. */
int moe_routing_pair_histogram(moe_ctx* ctx, const int32_t* ids, int n_layers, int n_tok, int top_k,
                               int n_experts, int64_t* pairs, void* stream);
/* Allocate every scratch buffer for calls of up to max_tokens tokens (and the
 * batch-1 router projections) now, so no later call allocates or frees
 * device memory (cudaFree synchronizes the device).  Serving loops and
 * peer-linked ranks call it once before the first forward. */
int moe_weights_reserve(moe_weights* w, int max_tokens);
int moe_weights_destroy(moe_weights* w);
int64_t moe_weights_device_bytes(const moe_weights* w);
/* Upload one expert from the reference's host layout (Matrix::data, row
 * major): w_in/w_gate [ffn x hidden], w_out [hidden x ffn]; rounded RNE to
 * the storage dtype on the device.  No-op for experts this rank does not own. */
int moe_weights_upload_expert(moe_weights* w, int layer, int expert, const double* w_in,
                              const double* w_gate, const double* w_out);
int moe_weights_upload_router(moe_weights* w, int layer, const double* router);
/* Device counter-based N(0, 1/sqrt(hidden)) init (Philox4x32-10, Box-Muller);
 * the value of a weight depends only on (seed, layer, expert, matrix, index),
 * so sharded and unsharded models hold identical weights.  Not the
 * reference's mt19937_64 stream (random_model, model.cpp:34-53): at the
 * 32/56-layer configs that init is 361 GB of fp64 on the host. */
int moe_weights_random(moe_weights* w, uint64_t seed);
/* Read back the device-rounded values in the reference layout (fp64). */
int moe_weights_download_expert(moe_weights* w, int layer, int expert, double* w_in,
                                double* w_gate, double* w_out);
int moe_weights_download_router(moe_weights* w, int layer, double* router);

/* ---- device-pointer hot path ------------------------------------------
 * x, x_out: fp32 [n_tok x hidden]; ids int32 / gates fp32 [n_tok x top_k]
 * (expert ids ascending per token, gates = softmax over the selected).
 * All calls are asynchronous on `stream`. */

/* gate_topk (model.cpp:69-101): fp32 router GEMV, top-k by (logit desc,
 * id asc), softmax over the selected logits. */
int moe_router_topk(moe_weights* w, int layer, const float* x, int n_tok, int32_t* ids,
                    float* gates, void* stream);
/* Deterministic permutation of (token, slot) pairs by expert (stable:
 * tokens ascending inside an expert).  counts/offsets [E], perm and
 * inv_perm [n_tok*top_k]: perm[offsets[e]+i] = t*top_k+j. */
int moe_permute(moe_ctx* ctx, const int32_t* ids, int n_tok, int top_k, int n_experts,
                int32_t* counts, int32_t* offsets, int32_t* perm, int32_t* inv_perm,
                void* stream);
/* Device routing histogram (profile_from_trace, placement.cpp:30-43):
 * counts[l][e] (int64, device, [n_layers x n_experts]) += the number of
 * (token, slot) pairs of layer l routed to expert e, from an ids record
 * [n_layers x n_tok x top_k] (moe_forward's).  Accumulates across calls, so
 * a serving loop profiles popularity on the device and reads it back only to
 * recompute the placement / expert-parallel shard map. */
int moe_routing_histogram(moe_ctx* ctx, const int32_t* ids, int n_layers, int n_tok, int top_k,
                          int n_experts, int64_t* counts, void* stream);
/* One RoutingTrace step (model.cpp:120-158, trace.hpp:18-47) from a device
 * routing record ids/gates [n_layers x n_tok x top_k] (on the context's
 * stream; synchronous): host token_count / gate_weight [n_layers x n_experts]
 * = per (layer, expert) the number of routed (token, slot) pairs and their
 * mean gate (fp64 sum in token order / count; 0 where count is 0).  The
 * Selection rows of the step are the entries with count > 0, ascending
 * expert; the step is a decode step iff n_tok == 1 (model.cpp:116).  See
 * paper_2402_07033_b200.trace for the JSONL emitter (trace.cpp:90-108). */
int moe_routing_trace_step(moe_ctx* ctx, const int32_t* ids, const float* gates, int n_layers,
                           int n_tok, int top_k, int n_experts, int32_t* token_count,
                           double* gate_weight);
/* The expert half of one model_forward layer (model.cpp:128-147): SwiGLU
 * experts of the routed tokens, gate-weighted combine, residual add:
 * x_out = x + sum_j gates[j] * expert_ffn(ids[j], x).  post_silu (optional,
 * [n_tok x top_k x ffn]) receives silu(w_in x) for the ActivationSink. */
int moe_experts_forward(moe_weights* w, int layer, const float* x, int n_tok,
                        const int32_t* ids, const float* gates, float* x_out,
                        float* post_silu, void* stream);
/* The streaming batch-1 expert kernel alone (TMA ring, one CTA per SM):
 * ypart [moe_ctx_sm_count() x hidden] receives per-CTA partial sums of
 * sum_j gates[j] * W2_j (silu(W1_j x) * (W3_j x)) over this rank's experts.
 * MOE_ERR_UNSUPPORTED if the shape has no streaming plan. */
int moe_decode_experts_partial(moe_weights* w, int layer, const float* x, const int32_t* ids,
                               const float* gates, float* ypart, void* stream);
/* One full MoE layer: router + experts + combine + residual. */
int moe_layer_forward(moe_weights* w, int layer, const float* x, float* x_out, int n_tok,
                      int32_t* ids, float* gates, void* stream);
/* model_forward's math (model.cpp:103-161), layer-major: all num_layers
 * layers in place on x.  ids/gates: [L x n_tok x top_k] routing record
 * (the RoutingTrace source).  Batch-1 decode runs as one CUDA graph. */
int moe_forward(moe_weights* w, float* x, int n_tok, int32_t* ids, float* gates,
                void* stream);

/* model_forward (as moe_forward, no graph) that also counts activation
 * sparsity in the up-projection epilogues: counts (int64,
 * device, [num_layers x n_thresholds], accumulated) += per layer the number
 * of post-SiLU values silu(w_in x) — the ActivationSink values of
 * model.cpp:131-139, over every (token, selected expert, ffn row) — with
 * |v| < thresholds[i], compared in fp32.  Dividing by n_tok*top_k*ffn gives
 * sparsity_histogram (placement.cpp:126-142) with no D2H of the values.
 * thresholds strictly increasing (else MOE_ERR_VALIDATION), at most 8.
 * Counted by the tcgen05 grouped-GEMM epilogue (prefill) or the generic up
 * kernel (other shapes / batch 1).  Under tensor or expert parallelism each
 * rank counts its resident rows / experts: sum the ranks' counts. */
int moe_forward_sparsity(moe_weights* w, float* x, int n_tok, int32_t* ids, float* gates,
                         const double* thresholds, int n_thresholds, int64_t* counts,
                         void* stream);

/* ---- host-buffer entry points (what the drop-in shim calls) ------------
 * Copies in, runs on the device, copies out, synchronizes.  tokens/out are
 * fp64 [n_tok x hidden] (the reference's vector<vector<double>>); ids [L x
 * n_tok x k]; gates fp64 [L x n_tok x k]; post_silu optional fp64
 * [n_tok x L x k x ffn] in the reference's sink call order. */
int moe_forward_host(moe_weights* w, const double* tokens, int n_tok, double* out,
                     int32_t* ids, double* gates, double* post_silu);
/* Pipelined host-buffer steps (no synchronize): enqueue the H2D of x_host
 * (fp32 [n_tok x hidden], pinned for overlap), one layer (layer >= 0:
 * moe_layer_forward; ids/gates [n_tok x k]) or the whole stack (layer == -1:
 * moe_forward; ids/gates [L x n_tok x k]) and the D2H of the result and the
 * routing, and return.  Multi-token copies run on their own streams, so
 * the copies of consecutive calls overlap the previous / next call's compute
 * (two device staging slots); a batch-1 step's copies ride the compute
 * stream (a decode step has nothing to overlap).  Results land in ticket
 * order.  *ticket identifies the call; moe_host_wait(w, ticket) blocks until
 * its outputs (and every earlier call's) are in host memory (ticket < 0:
 * every call).  The
 * host buffers must stay valid until then. */
int moe_forward_host_async(moe_weights* w, int layer, const float* x_host, int n_tok,
                           float* out_host, int32_t* ids_host, float* gates_host,
                           int64_t* ticket);
int moe_host_wait(moe_weights* w, int64_t ticket);
/* expert_ffn (model.cpp:55-67) on one host expert (uploaded per call). */
int moe_expert_ffn_host(moe_ctx* ctx, int dtype, int hidden, int ffn, const double* w_in,
                        const double* w_gate, const double* w_out, const double* x,
                        double* y);
/* gate_topk on a host router matrix [E x hidden]. */
int moe_gate_topk_host(moe_ctx* ctx, int n_experts, int hidden, const double* router,
                       const double* x, int top_k, int32_t* ids, double* gates);

/* ---- introspection for tests / bench ---------------------------------- */
/* Which expert kernel moe_experts_forward uses for (n_tok): 1 = streaming
 * decode (TMA ring), 2 = generic CUDA, 3 = tcgen05 grouped GEMM prefill. */
int moe_expert_path(moe_weights* w, int n_tok);
/* Number of kernels one moe_forward(n_tok) launches. */
int moe_forward_launches(moe_weights* w, int n_tok);
/* Number of kernels one moe_layer_forward(n_tok) launches (1 at batch 1 on
 * one GPU: the persistent kernel as a 1-layer stack). */
int moe_layer_launches(moe_weights* w, int n_tok);
/* Diagnostics: one batch-1 moe_forward through the persistent stack kernel
 * with per-CTA clock64 stamps (tools/trace_stack.py).  trace receives
 * [L][sm_count][16] u64 (slot meanings in tools/trace_stack.py).  Synchronous. */
int moe_debug_trace_forward(moe_weights* w, float* x, int32_t* ids, float* gates,
                            uint64_t* trace, int64_t cap);
/* One batch-1 moe_forward through the persistent stack kernel that also
 * records every layer's fp32 router logits (logits: device [L x E]) — the
 * values its top-k ranked, for the routing-margin report (SURVEY §8c:
 * tokens whose 2nd-3rd logit margin is below 1e-5 max|logit|).  Asynchronous
 * on `stream`.  MOE_ERR_UNSUPPORTED without a persistent-kernel plan. */
int moe_forward_logits(moe_weights* w, float* x, int32_t* ids, float* gates, float* logits,
                       void* stream);

/* ---- debug / A-B switches (tests and tools/ only) ----------------------
 * The library never reads the environment; these set process-wide options
 * (read when a moe_weights is created, or at launch):
 *   stack (1), stack_kernel (2), rw (1), prefill (1), prefill_splits (2),
 *   stack_grid (0), virtual_stack (0), noncoop (0), force_ep (0), no_pdl (0),
 *   combine4 (0), pf_debug, pf_evict, pf_lag, pf_late8, pf_slo, pf_persist.
 * Unknown names return MOE_ERR_ARG.  See DESIGN.md §6b. */
int moe_debug_set_option(const char* name, int64_t value);
int moe_debug_get_option(const char* name, int64_t* value);
/* Per-tile timeline file of the grouped prefill kernel (NULL / "" = off). */
int moe_debug_set_trace_path(const char* path);

#ifdef __cplusplus
}
#endif

#endif /* MOE_B200_H */
