// kernels.h — host-side launchers for the sm_100a kernels (internal).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace moe {

constexpr int kMaxExperts = 256;

// Debug / A-B switches (moe_debug_set_option, include/moe_b200.h).  The
// product never reads the environment: its code path changes only through
// this explicit API, which tests and tools/ call.  Values are read when a
// moe_weights is created (stack, rw, prefill, prefill_splits) or at launch.
struct DebugOptions {
  int stack = 1;           // batch-1 decode: persistent stack kernel (0: per-layer kernels)
  int stack_kernel = 2;    // 3: routing-ahead single-barrier kernel, 2: fixed-point single-barrier, 1: two-barrier
  int rw = 1;              // precomputed R_{l+1} W2 router projections
  int prefill = 1;         // tcgen05 grouped prefill (0: generic kernels)
  int prefill_splits = 2;  // max down K splits of the grouped kernel (0: two-kernel path)
  int stack_grid = 0;      // >0: persistent-kernel grid (several linked ranks on one GPU)
  int virtual_stack = 0;   // a virtual rank runs its shard through the persistent kernel
  int noncoop = 0;         // launch the stack kernel without the cooperative attribute
  int force_ep = 0;        // world 1 + NCCL communicator: the EP code path on one GPU
  int no_pdl = 0;          // no programmatic dependent launch anywhere
  int combine4 = 0;        // looped combine instead of combine_k2_kernel
  int prefill_fused = 1;   // prefill layer as router(+dispatch) -> grouped kernel (+combine)
  int pf_debug = 0, pf_evict = 0, pf_lag = kMaxExperts, pf_late8 = 3, pf_slo = 0, pf_persist = 1,
      pf_cut16 = 0;
};
DebugOptions& debug_options();
// per-tile timeline file of the grouped prefill kernel (tools/trace_prefill.py); empty = off
const char* debug_trace_path();

// Expert weights of one layer on this rank: slot s (local expert) holds
// [W1 f x d][W3 f x d][W2T f x d] contiguously (W2T = w_out transposed so the
// decode kernel streams whole d-rows for every ffn index r).
struct LayerWeights {
  const void* experts;        // base of slot 0
  long long expert_stride;    // elements between slots (= 3*f*d)
  long long mat_stride;       // elements between W1/W3/W2T (= f*d)
  const float* router;        // fp32 [E x d] (replicated)
  int16_t slot_of[kMaxExperts];  // expert id -> local slot, -1 = remote
};

struct Dims {
  int d, f, E, k;
  int dtype;  // MOE_DTYPE_*
};

// Fused activation-sparsity counters (sparsity_histogram, placement.cpp:126-142,
// over the ActivationSink values of model.cpp:131-139): the up-projection
// epilogues add |{v : |silu(w_in x)| < thr[i]}| into counts[i] (one layer).
constexpr int kMaxThresholds = 8;
struct SparsityCounters {
  unsigned long long* counts = nullptr;  // [n] device, accumulated; nullptr = off
  float thr[kMaxThresholds] = {};
  int n = 0;
};

// ---- router -------------------------------------------------------------
cudaError_t launch_router_topk(const float* router, const float* x, int n_tok, const Dims& dm,
                               int32_t* ids, float* gates, cudaStream_t s, bool pdl);
// The router of the fused prefill path: the same routing (bit for bit) plus
// each router block's (route_block_tokens() tokens) per-expert pair counts
// blk_count[route_blocks(n)][E], and the zeroing of n_zero words for the
// grouped kernel that follows.
struct RouteDispatch {
  int32_t* blk_count = nullptr;  // [nblk][E] out
  int* zero = nullptr;
  int n_zero = 0;
};
bool route_dispatch_supported(const Dims& dm);
int route_blocks(int n_tok);
int route_block_tokens();
cudaError_t launch_route_dispatch(const float* router, const float* x, int n_tok, const Dims& dm,
                                  int32_t* ids, float* gates, const RouteDispatch& rd,
                                  cudaStream_t s, bool pdl);

// ---- streaming batch-1 decode (TMA bulk ring) -----------------------------
struct DecodePlan {
  bool ok = false;
  int nv = 0;          // 16-byte vectors per consumer thread per row
  int ncons = 0;       // consumer threads
  int rps = 0;         // rows per ring stage
  int stages = 0;
  int smem = 0;        // dynamic smem bytes
  int grid = 0;        // CTAs (= SM count)
};
DecodePlan plan_decode(const Dims& dm, int sm_count);
// ypart[grid][d] <- per-CTA partial sums of sum_j g_j W2_j (silu(W1_j x) * (W3_j x))
cudaError_t launch_decode_experts(const DecodePlan& p, const LayerWeights& lw, const Dims& dm,
                                  const int32_t* ids, const float* gates, const float* x,
                                  float* ypart, cudaStream_t s, bool pdl);
// The whole L-layer batch-1 forward in one persistent cooperative launch.
struct StackDesc {
  const void* const* layer_experts;  // device array [L]
  const int16_t* slot_of;            // device array [L][E]
  long long expert_stride, mat_stride;
  const float* router;               // [L][E][d]
  int L;
  unsigned long long* trace = nullptr;  // optional [L][G][16] clock64 stamps
  const float* const* rw = nullptr;     // device [L]: R_{l+1} W2 per local expert, [f][E]
};
// rw[slot][r][e] = sum_i R_next[e][i] * W2T[slot][r][i]   (fp32; E <= 8)
cudaError_t launch_router_projection(const void* layer_experts, int n_local, const Dims& dm,
                                     const float* router_next, float* rw, cudaStream_t s);
struct PeerArgs;
// pa (optional): expert/tensor-parallel ranks linked by peer windows; each
// layer's x_{l+1} and next-layer router logits are then summed over the ranks
// inside the kernel (one launch per token on every GPU).
cudaError_t launch_decode_stack(const DecodePlan& p, const StackDesc& sd, const Dims& dm,
                                float* x, float* xbuf, float* ypart, float* rpart,
                                int32_t* ids_out, float* gates_out, unsigned* gbar,
                                cudaStream_t s, const PeerArgs* pa = nullptr);
// The same forward with ONE grid barrier per layer: partials summed in 64-bit
// fixed point with L2 integer atomics (order-independent, bit-reproducible).
// Single GPU only (no peers), E <= 8, router projections (sd.rw) required.
// accbuf: stack2_acc_bytes(dm) bytes, zeroed once at allocation (the kernel
// leaves it reusable: counters and buffer rotation carry across launches).
bool stack2_supported(const DecodePlan& p, const Dims& dm);
size_t stack2_acc_bytes(const Dims& dm);
cudaError_t launch_decode_stack2(const DecodePlan& p, const StackDesc& sd, const Dims& dm, float* x,
                                 void* accbuf, int32_t* ids_out, float* gates_out,
                                 float* logits_out, cudaStream_t s, float* x_out = nullptr);
// x_out = x + sum_p ypart[p]; optionally the next layer's router + top-k
// (deterministic fixed-order partial sums, last-block-done).
cudaError_t launch_reduce_residual(const float* ypart, int nparts, const float* x, float* x_out,
                                   const Dims& dm, const float* next_router, float* rpart,
                                   unsigned* counter, int32_t* next_ids, float* next_gates,
                                   cudaStream_t s, bool pdl);
int reduce_blocks(const Dims& dm);

// ---- expert-parallel combine over peer memory (NVLink P2P / IPC) -----------
// Every rank owns one "exchange window" in its HBM:
//   inbox [2 parity][world][d] fp32 | flags [world][kPeerSlots] u32 |
//   zbox [2 parity][world][kMaxExperts] fp32 | zflags [world] u32 |
//   seq [kPeerSlots] u32 | zseq u32 | err u32
// and holds device pointers to every peer's window (its own included).  A
// "slot" is one exchanging block: a 32-column block of reduce_exchange_kernel
// or one CTA of the persistent stack kernel; its sequence counter advances by
// one per exchange on every rank alike, and selects the inbox parity.
constexpr int kMaxRanks = 8;
constexpr int kPeerSlots = 512;
// Multi-token area (optional, max_tokens > 0): a reduce-scatter + all-gather
// of [n x d] deltas over kMtBlocks element blocks; block b is summed by rank
// b % world.  recv [2 parity][world][cap] | gath [2][cap] fp32 |
// pflag [world][kMtBlocks] | gflag [kMtBlocks] | seq [kMtBlocks] u32.
// 32 blocks: plenty for NVLink-rate pushes, and small enough that several
// ranks' spinning exchange kernels stay co-resident when ranks share one GPU
// (tests): with 128 blocks only two ranks' kernels were resident at once.
constexpr int kMtBlocks = 32;
struct PeerArgs {
  float* inbox[kMaxRanks];     // rank r's inbox base
  unsigned* flags[kMaxRanks];  // rank r's flags base
  float* zbox[kMaxRanks];      // rank r's router-partial inbox (stack kernel)
  unsigned* zflags[kMaxRanks];
  unsigned* seq;               // own per-slot exchange counters
  unsigned* zseq;              // own router-partial exchange counter
  unsigned* err;               // own: set when a peer never arrives (bounded wait)
  float* mt_recv[kMaxRanks];
  float* mt_gath[kMaxRanks];
  unsigned* mt_pflag[kMaxRanks];
  unsigned* mt_gflag[kMaxRanks];
  unsigned* mt_seq;            // own: [0] blocks of multi-token exchanges finished (monotonic)
  unsigned* mt_done[kMaxRanks];   // rank r's [world] words: the last multi-token exchange each rank completed
  unsigned* mt_cflag[kMaxRanks];  // rank r's per-(source, home token) contribution flags [world][max_tokens]
  unsigned* mt_tflag[kMaxRanks];  // rank r's per-token gathered-row flags [max_tokens]
  long long mt_cap;            // elements per copy (max_tokens x max_hidden; 0 = none)
  int mt_tokens;               // max_tokens of the windows
  int world, rank;
};
struct PeerParts {
  float* inbox;
  unsigned* flags;
  float* zbox;
  unsigned* zflags;
  unsigned *seq, *zseq, *err;
  float *mt_recv, *mt_gath;
  unsigned *mt_pflag, *mt_gflag, *mt_seq;
  unsigned *mt_cflag, *mt_tflag;
};
size_t peer_window_bytes(int world, int max_hidden, int max_tokens = 0);
// Carve a window allocation into its parts (same layout on every rank).
PeerParts peer_window_parts(void* base, int world, int max_hidden, int max_tokens = 0);
// Multi-token combine over peer memory (prefill under EP/TP): x_out = x + the
// rank-ordered sum of every rank's delta [n], as a reduce-scatter (block b
// summed by rank b % world) + all-gather through the windows; bit-identical
// on every rank, no NCCL.  n <= pa.mt_cap.
// The fused prefill path's combine under expert parallelism with peer
// windows: streamed beside the grouped kernel from its completion queue,
// every token reduced by its home rank t % world over the peer windows and
// gathered to every rank (decode.cu, ep_combine_kernel).  n_tok <= the
// windows' max_tokens; seq = the per-context call counter (same on every rank).
cudaError_t launch_ep_combine(const float* x, const float* y, int n_tok, const Dims& dm, float* x_out,
                              const int32_t* ids, const int32_t* split_of, const int16_t* slot_of,
                              const uint32_t* holders, int* queue, const PeerArgs& pa, unsigned seq,
                              cudaStream_t s, bool pdl);
cudaError_t launch_peer_allreduce(const float* delta, const float* x, float* x_out, long long n,
                                  const PeerArgs& pa, unsigned seq, cudaStream_t s);
// x_out = x + sum_{r in rank order} delta_r, where delta_r = this layer's
// fixed-order sum of rank r's per-CTA partials.  Each block reduces 32 hidden
// columns, stores them into every peer's inbox (P2P stores), releases a
// per-(rank, block) flag, waits for all ranks' flags and sums the inbox in
// rank order — so every rank computes bit-identical x_out (consistent
// routing) with no NCCL call.  Fused with the next layer's router + top-k.
cudaError_t launch_reduce_exchange(const float* ypart, int nparts, const float* x, float* x_out,
                                   const Dims& dm, const float* next_router, float* rpart,
                                   unsigned* counter, int32_t* next_ids, float* next_gates,
                                   const PeerArgs& pa, cudaStream_t s, bool pdl);

// ---- generic (any shape, any token count) ---------------------------------
// h[t][j][r] = silu(W1 x_t) * (W3 x_t) for expert ids[t][j]; post_silu optional.
cudaError_t launch_generic_up(const LayerWeights& lw, const Dims& dm, const float* x, int n_tok,
                              const int32_t* ids, float* h, float* post_silu, cudaStream_t s,
                              bool pdl, const SparsityCounters& sp = SparsityCounters());
// y[t][j][i] = sum_r W2T[r][i] h[t][j][r]
cudaError_t launch_generic_down(const LayerWeights& lw, const Dims& dm, const float* h,
                                int n_tok, const int32_t* ids, float* y, cudaStream_t s,
                                bool pdl);
// x_out[t][i] = x[t][i] + (0 + sum_j g[t][j] * y[t][j][i])   (model.cpp:128-147)
cudaError_t launch_combine(const float* x, const float* y, const float* gates, int n_tok,
                           const Dims& dm, float* x_out, cudaStream_t s, bool pdl, int nsplit = 1,
                           const int32_t* ids = nullptr, const int32_t* split_of = nullptr);
// Token chunk of the grouped prefill kernel (tokens per tile, UMMA N).
#ifndef MOE_PREFILL_CHUNK
#define MOE_PREFILL_CHUNK 256
#endif
constexpr int kPrefillChunk = MOE_PREFILL_CHUNK;
// The grouped prefill kernel's per-expert K-split record inside its sync
// buffer (sync = [tile counter][E x chunks done flags][E splits]).
inline int32_t* prefill_split_of(int* sync, int E, int n_tok) {
  return sync + 1 + E * ((n_tok + kPrefillChunk - 1) / kPrefillChunk);
}

// out = a + b (elementwise; expert-parallel residual after the all-reduce)
cudaError_t launch_add(const float* a, const float* b, float* out, long long n, cudaStream_t s,
                       bool pdl);

// ---- tcgen05 prefill (prefill.cu) ---------------------------------------------
bool prefill_supported(const Dims& dm);
// counts/offsets/perm from launch_permute; writes y[pair][d] = g * expert(x_t)
// for this rank's experts (rows of remote experts are left untouched).
cudaError_t launch_prefill_experts(const LayerWeights& lw, int n_local, const Dims& dm,
                                   int n_tok, const float* x, const int32_t* counts,
                                   const int32_t* offsets, const int32_t* perm,
                                   const float* gates, const int16_t* slot_of_dev,
                                   __nv_bfloat16* xg, __nv_bfloat16* h, float* y, int* sync,
                                   int sm_count, int splits, cudaStream_t s,
                                   const SparsityCounters& sp = SparsityCounters(),
                                   cudaEvent_t t0 = nullptr, cudaEvent_t t1 = nullptr,
                                   const struct PrefillFuse* fz = nullptr);
// The fused single-GPU prefill layer (splits > 0, every expert local): two
// launches — the router (launch_route_dispatch: ids, gates, counts, offsets,
// per-block bases) and the grouped kernel, which scatters perm + Xg itself and
// writes x_out = x + the combined expert outputs (no permute, gather or
// combine launch).  counts/offsets/perm passed to launch_prefill_experts are
// then outputs.  sync needs prefill_sync_words(E, n_tok, d) ints.
struct PrefillFuse {
  const float* router = nullptr;  // this layer's [E][d]
  int32_t* ids = nullptr;         // [n_tok][k] out
  float* gates = nullptr;         // [n_tok][k] out
  int32_t* route = nullptr;       // [route_blocks(n_tok) * E] per-block expert counts
  float* x_out = nullptr;         // [n_tok][d] out; may alias x (token t's row is
                                  // combined only after its own dispatch read it)
  // expert parallelism over peer windows (nullptr: single GPU)
  const PeerArgs* pa = nullptr;
  const uint32_t* holders = nullptr;  // [E] rank bitmask holding each expert (nullptr: all, TP)
  unsigned seq = 0;                   // per-context call counter, same on every rank
};
inline size_t prefill_sync_words(int E, int n_tok, int d) {
  const size_t chunks = (n_tok + kPrefillChunk - 1) / kPrefillChunk;
  return 1 + (size_t)E * chunks + E /*splits*/ + 1 /*dispatch*/ + E /*x_ready*/ +
         (size_t)n_tok * (d / 256) /*partials landed*/ + n_tok /*blocks landed*/ +
         4 + (size_t)n_tok /*combine queue*/;
}
// The fused path's combine: launched right behind the grouped kernel (PDL; it
// starts once every grouped CTA is resident), each block claims queue slots
// in completion order, waits for the slot's token (published by the down
// epilogue that landed its last partial) and writes
// x_out[t] = x[t] + sum over slots (asc) and K splits (asc) of y — combine_k2's
// adds.  It waits for the grouped grid before exiting, so later launches see
// both complete.
cudaError_t launch_combine_ready(const float* x, const float* y, int n_tok, const Dims& dm,
                                 float* x_out, int nsplit, const int32_t* ids, const int32_t* split_of,
                                 int* queue, int blocks, cudaStream_t s, bool pdl);

// Replicated experts under expert parallelism (replica_plan.h):
// one block computes this rank's share [lo, hi) of every expert's sorted rows
// from the step's counts and writes the grouped kernel's inputs
// counts_out[e] = hi - lo, offsets_out[e] = offsets[e] + lo.
// holders: [E] rank bitmasks of this layer.
cudaError_t launch_replica_plan(const int32_t* counts, const int32_t* offsets, int E,
                                const uint32_t* holders, int world, int rank, long long weight_ps,
                                long long row_ps, long long part_ps, int32_t* counts_out,
                                int32_t* offsets_out, cudaStream_t s);
// splits > 0: persistent grouped kernel, y is [splits][n*k][d] (sum the splits);
// splits == 0: two-kernel path, y is [n*k][d].  sync: 1 + E*ceil(n_tok/256) ints.

// ---- routing histogram: counts[l][e] += selections (int64, device) ----------
cudaError_t launch_routing_pair_histogram(const int32_t* ids, int L, int n_tok, int k, int E,
                                          int64_t* pairs, cudaStream_t s);
cudaError_t launch_routing_histogram(const int32_t* ids, int L, int n_tok, int k, int E,
                                     int64_t* counts, cudaStream_t s);

// count[l][e] / gsum[l][e] of one trace step from ids/gates [L x n_tok x k]
cudaError_t launch_trace_step(const int32_t* ids, const float* gates, int L, int n_tok, int k,
                              int E, int32_t* count, double* gsum, cudaStream_t s);

// ---- permutation ------------------------------------------------------------
cudaError_t launch_permute(const int32_t* ids, int n_tok, int k, int E, int32_t* counts,
                           int32_t* offsets, int32_t* perm, int32_t* inv_perm, cudaStream_t s,
                           bool pdl = false);

// ---- weights ----------------------------------------------------------------
// dst (dtype) = src (fp64) with optional transpose of a [rows x cols] matrix.
cudaError_t launch_convert(const double* src, void* dst, int dtype, long long rows,
                           long long cols, bool transpose, cudaStream_t s);
cudaError_t launch_to_double(const void* src, int dtype, double* dst, long long rows,
                             long long cols, bool transpose, cudaStream_t s);
cudaError_t launch_convert_f32(const double* src, float* dst, long long n, cudaStream_t s);
// Counter-based normal init of one logical matrix (reference layout rows x
// cols), stored transposed when `transpose`.  tag identifies (layer, expert, m).
// Element (r, c) takes variate #(r * ld + c + off) of the stream, so a
// [rows x cols] slice of a larger matrix (ld = its row length, off = the
// slice origin) holds exactly the values of the full matrix (ld <= 0: cols).
cudaError_t launch_random(void* dst, int dtype, long long rows, long long cols, bool transpose,
                          uint64_t seed, uint64_t tag, float scale, cudaStream_t s,
                          long long ld = 0, long long off = 0);

}  // namespace moe
