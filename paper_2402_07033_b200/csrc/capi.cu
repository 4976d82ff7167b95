// capi.cu — the extern "C" boundary (include/moe_b200.h): context, device
// weights, expert-parallel exchange and the layer-major orchestration of the
// reference's model_forward (model.cpp:103-161).
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "../../include/moe_b200.h"
#include "kernels.h"
#include "replica_plan.h"
#include "host_io.h"

using moe::Dims;
using moe::LayerWeights;

namespace moe {
DebugOptions& debug_options() {
  static DebugOptions o;
  return o;
}
static std::string& trace_path_store() {
  static std::string p;
  return p;
}
const char* debug_trace_path() { return trace_path_store().c_str(); }
}  // namespace moe

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CU(expr)                                                                      \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess) {                                                          \
      return fail(_e == cudaErrorMemoryAllocation ? MOE_ERR_OOM : MOE_ERR_CUDA,       \
                  std::string(#expr) + ": " + cudaGetErrorString(_e));                \
    }                                                                                 \
  } while (0)

#define TRY(expr)                \
  do {                           \
    int _rc = (expr);            \
    if (_rc != MOE_OK) return _rc; \
  } while (0)

// ---- NCCL, dlopen'ed (only needed for expert parallelism) ------------------
struct NcclApi {
  void* h = nullptr;
  int (*getUniqueId)(void*) = nullptr;
  void* commInitRankSym = nullptr;  // takes ncclUniqueId by value, see CommInitRankFn
  int (*allReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*commDestroy)(void*) = nullptr;
  const char* (*errStr)(int) = nullptr;
};
struct NcclUid {
  char internal[128];
};
typedef int (*CommInitRankFn)(void**, int, NcclUid, int);

NcclApi* nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (!api.h) return;
    api.getUniqueId = (int (*)(void*))dlsym(api.h, "ncclGetUniqueId");
    api.commInitRankSym = dlsym(api.h, "ncclCommInitRank");
    api.allReduce = (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))dlsym(
        api.h, "ncclAllReduce");
    api.commDestroy = (int (*)(void*))dlsym(api.h, "ncclCommDestroy");
    api.errStr = (const char* (*)(int))dlsym(api.h, "ncclGetErrorString");
  });
  if (!api.h || !api.getUniqueId || !api.commInitRankSym || !api.allReduce) return nullptr;
  return &api;
}

constexpr int kNcclFloat32 = 7;
constexpr int kNcclSum = 0;

}  // namespace

// ---------------------------------------------------------------------------
struct moe_ctx {
  int device = 0;
  int sm_count = 0;
  cudaStream_t stream = nullptr;
  int world = 1, rank = 0;
  void* comm = nullptr;  // ncclComm_t
  bool virtual_ep = false;  // sharded math without a communicator (testing hook)
  bool ep_forced = false;   // world == 1 but the EP path + NCCL exchange (MOE_B200_FORCE_EP)
  bool ep() const { return world > 1 || ep_forced; }
  // peer-memory exchange window (NVLink P2P / CUDA IPC; kernels.h PeerArgs)
  void* win = nullptr;
  int win_world = 0, win_hidden = 0, win_tokens = 0;
  bool peers = false;
  moe::PeerArgs pa{};
  std::vector<void*> ipc_opened;
  std::mutex mu;
};

constexpr int kIoChunks = 4;  // moe_forward_host transfer chunks

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int ensure(size_t n) {
    if (n <= bytes) return MOE_OK;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, n);
    if (e != cudaSuccess) return fail(MOE_ERR_OOM, "cudaMalloc scratch failed");
    // legacy-stream memset, waited for on that stream only (the kernels run on
    // non-blocking streams; a device-wide sync would also wait for a peer-linked
    // rank's exchange kernel that is spinning on this process's other ranks)
    if (cudaMemset(p, 0, n) != cudaSuccess || cudaStreamSynchronize(cudaStreamLegacy) != cudaSuccess)
      return fail(MOE_ERR_CUDA, "scratch memset failed");
    bytes = n;
    return MOE_OK;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct GraphEntry {
  cudaGraphExec_t exec = nullptr;
};

struct moe_weights {
  moe_ctx* ctx = nullptr;
  moe_shape shape{};
  int dtype = MOE_DTYPE_BF16;
  int esize = 2;
  std::vector<int32_t> owner;      // [L*E]
  std::vector<int16_t> slot_of;    // [L*E] resident slot (owned or replica), -1 = not here
  std::vector<int16_t> exec_slot;  // [L*E] slot if this rank OWNS the expert, else -1
  std::vector<uint32_t> holders;   // [L*E] rank bitmask: owner | replicas
  bool replicas = false;           // some expert is held by more than one rank
  long long rep_weight_ps = 0, rep_row_ps = 0, rep_part_ps = 0;  // replica split cost model
  DevBuf dev_holders, dev_res_slots, pf_counts2, pf_offsets2;
  std::vector<int> n_local;        // [L]
  std::vector<void*> layer_mem;    // [L] device, n_local[l] * 3*f*d elements
  float* router = nullptr;         // [L][E][d]
  int64_t device_bytes = 0;
  moe::DecodePlan plan;
  // scratch
  DevBuf ypart, rpart, counter, xa, xb, xin, h, y, delta, ids, gates, post;
  DevBuf xbuf2, gbar, dev_layers, dev_slots;  // persistent stack kernel
  DevBuf stack_acc;  // decode_stack2_kernel: fixed-point accumulators + barrier state
  DevBuf pf_counts, pf_offsets, pf_perm, pf_xg, pf_h, pf_sync;  // tcgen05 prefill
  DevBuf pf_route;  // fused prefill: router last-block counter + per-block dispatch bases
  DevBuf io;  // host-buffer API, batch 1: [x][ids][gates] (one D2H)
  // moe_debug_kernel_timing: event pairs around each grouped prefill launch
  bool ktime_on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> kev;
  size_t kev_used = 0;
  bool prefill_enabled = true;
  int prefill_splits = 2;  // max K splits of the down GEMM in the grouped kernel (0: 2-kernel path)
  // router projections R_{l+1} W2 for the stack kernel's z partials
  std::vector<DevBuf> rw_mem;  // [L-1]
  DevBuf dev_rw;               // device [L] pointers
  bool rw_enabled = false, rw_dirty = true;
  bool stack_enabled = true;
  // fused sparsity counters of the call in flight (moe_forward_sparsity):
  // counts [L][sp.n]; layer l adds into sp.counts + l * sp.n
  moe::SparsityCounters sp;
  DevBuf stage_d;  // fp64 staging for uploads / downloads
  void* host_pin = nullptr;
  size_t host_pin_bytes = 0;
  // key: (x, ids, gates, host buffer, stack kernel option)
  std::map<std::tuple<float*, int32_t*, float*, cudaStream_t, int>, GraphEntry> graphs;
  cudaStream_t cap_stream = nullptr;  // private stream for graph capture
  cudaStream_t io_stream = nullptr;   // host-buffer entry points (moe_forward_host)
  cudaEvent_t io_ev[kIoChunks] = {};  // host-buffer API: per-chunk D2H completion
  // Cross-stream ordering of the scratch above: a call on stream s waits for
  // the last call's work (on another stream) through order_ev, then records
  // it (StreamOrder).  w->mu only serialises the enqueueing.
  cudaStream_t last_stream = nullptr;
  cudaEvent_t order_ev = nullptr;
  // moe_forward_host_async: two staging slots, copy streams in / out
  struct MoeHostAsyncT {
    cudaStream_t cin = nullptr, cout = nullptr;
    DevBuf x[2], y[2], ids[2], gates[2];
    cudaEvent_t in_done[2] = {}, comp_done[2] = {}, out_done[2] = {};
    int64_t next = 0;
  } ha;
  using MoeHostAsync = MoeHostAsyncT;
  std::mutex mu;

  int L() const { return shape.num_layers; }
  int E() const { return shape.experts_per_layer; }
  int k() const { return shape.top_k; }
  int d() const { return shape.hidden_dim; }
  // tensor parallelism: this rank holds ffn rows [tp_rank*f_local, +f_local)
  // of every expert (W1/W3 rows, W2 columns); tp == 1 otherwise
  int tp = 1, tp_rank = 0, f_local = 0;
  int f() const { return f_local; }      // ffn rows resident on this rank
  int f_glob() const { return shape.ffn_dim; }
  long long r0() const { return (long long)tp_rank * f_local; }
  Dims dims() const { return Dims{d(), f(), E(), k(), dtype}; }
  long long mat_elems() const { return (long long)f() * d(); }
  LayerWeights layer(int l) const {
    LayerWeights lw{};
    lw.experts = layer_mem[l];
    lw.expert_stride = 3 * mat_elems();
    lw.mat_stride = mat_elems();
    lw.router = router + (size_t)l * E() * d();
    for (int e = 0; e < moe::kMaxExperts; ++e)
      lw.slot_of[e] = e < E() ? exec_slot[(size_t)l * E() + e] : (int16_t)-1;
    return lw;
  }
  void* expert_ptr(int l, int e, int m) const {
    const int s = slot_of[(size_t)l * E() + e];
    if (s < 0) return nullptr;
    return static_cast<char*>(layer_mem[l]) + ((size_t)s * 3 + m) * mat_elems() * esize;
  }
};

namespace {

cudaStream_t pick(moe_ctx* c, void* s) { return s ? static_cast<cudaStream_t>(s) : c->stream; }

// Orders one call's work on stream s after the previous call on these weights
// (whatever stream that was) and records it for the next: the scratch, the
// persistent kernels' barrier words and the captured graphs are per-weights,
// so calls on different streams must not overlap on the device.  Held under
// w->mu.  A stream the caller is capturing into a graph is not ordered
// against work outside the capture (CUDA forbids that wait); it follows the
// caller's own graph order.
struct StreamOrder {
  moe_weights* w;
  cudaStream_t s;
  bool capturing = false;
  StreamOrder(moe_weights* w_, cudaStream_t s_) : w(w_), s(s_) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &st) != cudaSuccess) cudaGetLastError();
    capturing = st != cudaStreamCaptureStatusNone;
    if (capturing) return;
    if (!w->order_ev && cudaEventCreateWithFlags(&w->order_ev, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      w->order_ev = nullptr;
    }
    if (w->order_ev && w->last_stream && w->last_stream != s) cudaStreamWaitEvent(s, w->order_ev, 0);
  }
  ~StreamOrder() {
    if (capturing || !w->order_ev) return;
    if (cudaEventRecord(w->order_ev, s) == cudaSuccess) w->last_stream = s;
  }
};

int check_shape(const moe_shape* s) {
  if (!s) return fail(MOE_ERR_ARG, "null shape");
  if (s->num_layers < 0) return fail(MOE_ERR_SHAPE, "num_layers must be non-negative");
  if (s->experts_per_layer <= 0 || s->top_k <= 0 || s->hidden_dim <= 0 || s->ffn_dim <= 0 ||
      s->bytes_per_param <= 0)
    return fail(MOE_ERR_SHAPE, "all shape counts must be strictly positive");
  if (s->top_k > s->experts_per_layer)
    return fail(MOE_ERR_SHAPE, "top_k must not exceed experts_per_layer");
  return MOE_OK;
}

int set_device(moe_ctx* c) {
  CU(cudaSetDevice(c->device));
  cudaGetLastError();  // launches below report their own errors, not a stale one
  return MOE_OK;
}

void drop_graphs(moe_weights* w) {
  for (auto& kv : w->graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  w->graphs.clear();
}

int ensure_scratch_impl(moe_weights* w, int n_tok);
bool use_prefill(const moe_weights* w, int n_tok, const float* post);

// Per-call scratch sized for n_tok tokens; captured graphs hold scratch
// pointers, so any reallocation invalidates them.
int ensure_scratch(moe_weights* w, int n_tok) {
  const void* before[] = {w->xa.p, w->xb.p, w->delta.p, w->ypart.p, w->rpart.p, w->counter.p};
  TRY(ensure_scratch_impl(w, n_tok));
  const void* after[] = {w->xa.p, w->xb.p, w->delta.p, w->ypart.p, w->rpart.p, w->counter.p};
  for (int i = 0; i < 6; ++i)
    if (before[i] != after[i]) {
      drop_graphs(w);
      break;
    }
  return MOE_OK;
}

int ensure_scratch_impl(moe_weights* w, int n_tok) {
  const size_t d = w->d(), f = w->f(), k = w->k(), L = std::max(1, w->L());
  const size_t n = std::max(1, n_tok);
  TRY(w->xa.ensure(n * d * 4));
  TRY(w->xb.ensure(n * d * 4));
  TRY(w->delta.ensure(n * d * 4));
  TRY(w->xin.ensure(n * d * 4));
  TRY(w->ids.ensure(L * n * k * 4));
  TRY(w->gates.ensure(L * n * k * 4));
  TRY(w->rpart.ensure((size_t)std::max(w->ctx->sm_count, moe::reduce_blocks(w->dims())) * w->E() * 4));
  TRY(w->counter.ensure(64));
  TRY(w->ypart.ensure((size_t)std::max(1, w->ctx->sm_count) * d * 4));
  if (n_tok > 1 || !w->plan.ok) {
    // sized for the grouped prefill's K-split partials up front: growing a
    // buffer later means cudaFree, which synchronizes the device (and with
    // peer-linked ranks on one GPU would wait on a rank's spinning exchange)
    TRY(w->h.ensure(n * k * f * 4));  // generic path (also the sink / counter fallbacks)
    const size_t splits = use_prefill(w, n_tok, nullptr) ? (size_t)std::max(1, w->prefill_splits) : 1;
    TRY(w->y.ensure(n * k * d * 4 * splits));
  }
  return MOE_OK;
}

int allreduce(moe_weights* w, float* buf, size_t count, cudaStream_t s) {
  moe_ctx* c = w->ctx;
  if (!c->ep() || c->virtual_ep) return MOE_OK;  // virtual: caller sums the partials
  NcclApi* api = nccl();
  if (!api || !c->comm) return fail(MOE_ERR_NCCL, "expert parallelism requested without NCCL");
  const int r = api->allReduce(buf, buf, count, kNcclFloat32, kNcclSum, c->comm, s);
  if (r != 0)
    return fail(MOE_ERR_NCCL, std::string("ncclAllReduce: ") + (api->errStr ? api->errStr(r) : "?"));
  return MOE_OK;
}

bool use_decode(const moe_weights* w, int n_tok, const float* post) {
  return n_tok == 1 && w->plan.ok && post == nullptr && w->sp.counts == nullptr;
}

// Peer windows usable by the batch-1 kernels of these weights.
bool peer_ok(const moe_weights* w) {
  const moe_ctx* c = w->ctx;
  return c->peers && w->d() <= c->win_hidden && w->plan.grid <= moe::kPeerSlots;
}

// Whole-token persistent kernel: one GPU, or several linked by peer windows
// (the per-layer exchange then runs inside the kernel).
bool use_stack(const moe_weights* w, int n_tok) {
  // MOE_B200_VIRTUAL_STACK (measurement hook, tools/shard_proxy.py): a
  // virtual rank runs its shard through the persistent kernel with no
  // exchange — one rank's streaming time of an N-GPU step
  const bool virt = moe::debug_options().virtual_stack != 0;
  const moe_ctx* c = w->ctx;
  return use_decode(w, n_tok, nullptr) && (!c->ep() || peer_ok(w) || (c->virtual_ep && virt)) &&
         w->stack_enabled && w->L() > 0;
}

// Recompute rw = R_{l+1} W2 after any weight/router change (outside capture).
int refresh_projection(moe_weights* w) {
  if (!w->rw_enabled || !w->rw_dirty || !use_stack(w, 1)) return MOE_OK;
  cudaStream_t s = w->ctx->stream;
  const Dims dm = w->dims();
  for (int l = 0; l + 1 < w->L(); ++l)
    CU(moe::launch_router_projection(w->layer_mem[l], w->n_local[l], dm,
                                     w->router + (size_t)(l + 1) * dm.E * dm.d,
                                     w->rw_mem[l].as<float>(), s));
  CU(cudaStreamSynchronize(s));
  w->rw_dirty = false;
  return MOE_OK;
}

// The single-barrier fixed-point stack kernel (single GPU, E <= 8, router
// projections on); decode_stack_kernel otherwise.
bool use_stack2(const moe_weights* w) {
  return moe::debug_options().stack_kernel >= 2 && !w->ctx->ep() && w->rw_enabled && w->stack_acc.p != nullptr &&
         moe::stack2_supported(w->plan, w->dims());
}

int enqueue_stack(moe_weights* w, float* x, int32_t* ids, float* gates, cudaStream_t s,
                  unsigned long long* trace = nullptr, float* logits = nullptr) {
  moe::StackDesc sd;
  sd.trace = trace;
  sd.rw = w->rw_enabled ? w->dev_rw.as<const float* const>() : nullptr;
  sd.layer_experts = w->dev_layers.as<const void* const>();
  sd.slot_of = w->dev_slots.as<const int16_t>();
  sd.expert_stride = 3 * w->mat_elems();
  sd.mat_stride = w->mat_elems();
  sd.router = w->router;
  sd.L = w->L();
  if (use_stack2(w)) {
    CU(moe::launch_decode_stack2(w->plan, sd, w->dims(), x, w->stack_acc.p, ids, gates, logits, s));
    return MOE_OK;
  }
  if (logits) return fail(MOE_ERR_UNSUPPORTED, "router logits need the single-barrier stack kernel");
  CU(moe::launch_decode_stack(w->plan, sd, w->dims(), x, w->xbuf2.as<float>(),
                              w->ypart.as<float>(), w->rpart.as<float>(), ids, gates,
                              w->gbar.as<unsigned>(), s, peer_ok(w) ? &w->ctx->pa : nullptr));
  return MOE_OK;
}

bool use_prefill(const moe_weights* w, int n_tok, const float* post) {
  return n_tok > 1 && post == nullptr && w->prefill_enabled && moe::prefill_supported(w->dims()) &&
         (w->sp.counts == nullptr || w->prefill_splits > 0);  // counters: grouped kernel only
}

size_t prefill_h_bytes(const moe_weights* w, int n_tok) {
  return ((size_t)n_tok * w->k() * w->f() * 2 + 255) & ~(size_t)255;
}

int ensure_prefill_scratch(moe_weights* w, int n_tok) {
  const size_t rows = (size_t)n_tok * w->k();
  TRY(w->pf_counts.ensure(4 * (size_t)w->E()));
  TRY(w->pf_offsets.ensure(4 * (size_t)w->E()));
  TRY(w->pf_perm.ensure(4 * rows));
  TRY(w->pf_xg.ensure(2 * rows * w->d()));
  // [H | Y]: the grouped kernel's bf16 H and its fp32 Y partials in ONE
  // allocation, so one persisting-L2 window covers both (H is read back by
  // the down tiles, Y by the combine)
  TRY(w->pf_h.ensure(prefill_h_bytes(w, n_tok) +
                     4 * rows * w->d() * (size_t)std::max(1, w->prefill_splits)));
  TRY(w->pf_sync.ensure(4 * moe::prefill_sync_words(w->E(), n_tok, w->d())));
  TRY(w->pf_route.ensure(4 * (16 + (size_t)moe::route_blocks(n_tok) * w->E())));
  return MOE_OK;
}

// The fused prefill layer (router with dispatch bases -> grouped kernel that
// scatters, computes and combines): single GPU, every expert local, the
// grouped kernel (splits > 0), no post-SiLU capture.
bool use_fused_prefill(const moe_weights* w, int n_tok, const float* post) {
  const Dims dm = w->dims();
  return use_prefill(w, n_tok, post) && moe::debug_options().prefill_fused && !w->ctx->ep() &&
         !w->replicas && w->prefill_splits > 0 && moe::route_dispatch_supported(dm) &&
         moe::route_block_tokens() * dm.k <= 64 && dm.k * w->prefill_splits <= 8;
}

// moe_debug_kernel_timing: a fresh event pair around the grouped kernel
int kernel_events(moe_weights* w, cudaEvent_t& t0, cudaEvent_t& t1) {
  t0 = t1 = nullptr;
  if (!w->ktime_on) return MOE_OK;
  if (w->kev_used == w->kev.size()) {
    cudaEvent_t a = nullptr, b = nullptr;
    CU(cudaEventCreate(&a));
    CU(cudaEventCreate(&b));
    w->kev.emplace_back(a, b);
  }
  t0 = w->kev[w->kev_used].first;
  t1 = w->kev[w->kev_used].second;
  ++w->kev_used;
  return MOE_OK;
}

// Experts + combine + residual for one layer (x may alias x_out only on
// the decode path).  EP: local partials -> all-reduce -> residual.
int experts_forward(moe_weights* w, int l, const float* x, int n_tok, const int32_t* ids,
                    const float* gates, float* x_out, float* post, cudaStream_t s, bool pdl,
                    const float* next_router, int32_t* next_ids, float* next_gates,
                    const float* router_l = nullptr) {
  const Dims dm = w->dims();
  const LayerWeights lw = w->layer(l);
  const bool ep = w->ctx->ep();
  moe::SparsityCounters sp = w->sp;
  if (sp.counts) sp.counts += (size_t)l * sp.n;
  if (router_l) {
    // router_l: route this layer here (ids/gates are outputs) — fused into the
    // prefill layer's first kernel when the fused path applies
    if (!use_fused_prefill(w, n_tok, post)) {
      CU(moe::launch_router_topk(router_l, x, n_tok, dm, const_cast<int32_t*>(ids),
                                 const_cast<float*>(gates), s, false));
      router_l = nullptr;
    }
  }
  if (use_decode(w, n_tok, post)) {
    CU(moe::launch_decode_experts(w->plan, lw, dm, ids, gates, x, w->ypart.as<float>(), s, pdl));
    if (!ep) {
      CU(moe::launch_reduce_residual(w->ypart.as<float>(), w->plan.grid, x, x_out, dm,
                                     next_router, w->rpart.as<float>(),
                                     w->counter.as<unsigned>(), next_ids, next_gates, s, pdl));
      return MOE_OK;
    }
    if (peer_ok(w)) {
      // fused combine over peer memory: reduce + push + rank-ordered sum + residual + router
      CU(moe::launch_reduce_exchange(w->ypart.as<float>(), w->plan.grid, x, x_out, dm, next_router,
                                     w->rpart.as<float>(), w->counter.as<unsigned>(), next_ids,
                                     next_gates, w->ctx->pa, s, pdl));
      return MOE_OK;
    }
    float* delta = w->delta.as<float>();
    CU(moe::launch_reduce_residual(w->ypart.as<float>(), w->plan.grid, nullptr, delta, dm,
                                   nullptr, nullptr, nullptr, nullptr, nullptr, s, pdl));
    TRY(allreduce(w, delta, (size_t)dm.d, s));
    CU(moe::launch_reduce_residual(delta, 1, x, x_out, dm, next_router, w->rpart.as<float>(),
                                   w->counter.as<unsigned>(), next_ids, next_gates, s, false));
    return MOE_OK;
  }
  const float* cgates = gates;
  float* ybuf = w->y.as<float>();  // expert outputs y[pair][d] (+ K-split partials)
  int nsplit = 1;
  const int32_t* split_of = nullptr;  // per-expert K splits of the grouped prefill
  if (use_prefill(w, n_tok, post)) {
    // tcgen05 grouped GEMM: permute -> gather -> up -> down (gate in epilogue)
    TRY(ensure_prefill_scratch(w, n_tok));
    const int rows = n_tok * dm.k;
    int32_t* counts = w->pf_counts.as<int32_t>();
    int32_t* offsets = w->pf_offsets.as<int32_t>();
    int32_t* perm = w->pf_perm.as<int32_t>();
    if (router_l) {
      // fused: router + dispatch bases, then the grouped kernel scatters the
      // rows, runs both GEMMs and writes x_out itself
      moe::PrefillFuse fz;
      fz.router = router_l;
      fz.ids = const_cast<int32_t*>(ids);
      fz.gates = const_cast<float*>(gates);
      fz.route = w->pf_route.as<int32_t>();
      fz.x_out = x_out;
      float* yb = reinterpret_cast<float*>(w->pf_h.as<char>() + prefill_h_bytes(w, n_tok));
      cudaEvent_t kt0 = nullptr, kt1 = nullptr;
      TRY(kernel_events(w, kt0, kt1));
      CU(moe::launch_prefill_experts(lw, w->n_local[l], dm, n_tok, x, counts, offsets, perm, gates,
                                     w->dev_slots.as<int16_t>() + (size_t)l * dm.E,
                                     w->pf_xg.as<__nv_bfloat16>(), w->pf_h.as<__nv_bfloat16>(), yb,
                                     w->pf_sync.as<int>(), w->ctx->sm_count, w->prefill_splits, s, sp,
                                     kt0, kt1, &fz));
      if (next_router)
        CU(moe::launch_router_topk(next_router, x_out, n_tok, dm, next_ids, next_gates, s, pdl));
      return MOE_OK;
    }
    CU(moe::launch_permute(ids, n_tok, dm.k, dm.E, counts, offsets, perm, nullptr, s, pdl));
    const int S = w->prefill_splits;
    const int16_t* slots = w->dev_slots.as<int16_t>() + (size_t)l * dm.E;
    if (w->replicas && S > 0) {
      // replicated experts: this step's min-max share of every expert's rows
      // (identical plan on every rank), over the resident slots
      CU(moe::launch_replica_plan(counts, offsets, dm.E, w->dev_holders.as<uint32_t>() + (size_t)l * dm.E,
                                  w->ctx->world, w->ctx->rank, w->rep_weight_ps, w->rep_row_ps,
                                  w->rep_part_ps,
                                  w->pf_counts2.as<int32_t>(), w->pf_offsets2.as<int32_t>(), s));
      counts = w->pf_counts2.as<int32_t>();
      offsets = w->pf_offsets2.as<int32_t>();
      slots = w->dev_res_slots.as<int16_t>() + (size_t)l * dm.E;
    }
    ybuf = reinterpret_cast<float*>(w->pf_h.as<char>() + prefill_h_bytes(w, n_tok));
    if (w->n_local[l] < dm.E || w->replicas)
      CU(cudaMemsetAsync(ybuf, 0, (size_t)std::max(1, S) * rows * dm.d * 4, s));
    cudaEvent_t kt0 = nullptr, kt1 = nullptr;
    TRY(kernel_events(w, kt0, kt1));
    CU(moe::launch_prefill_experts(lw, w->n_local[l], dm, n_tok, x, counts, offsets, perm, gates,
                                   slots,
                                   w->pf_xg.as<__nv_bfloat16>(), w->pf_h.as<__nv_bfloat16>(),
                                   ybuf, w->pf_sync.as<int>(), w->ctx->sm_count, S,
                                   s, sp, kt0, kt1));
    cgates = nullptr;
    nsplit = std::max(1, S);
    if (S > 0) split_of = moe::prefill_split_of(w->pf_sync.as<int>(), dm.E, n_tok);
  } else {
    CU(moe::launch_generic_up(lw, dm, x, n_tok, ids, w->h.as<float>(), post, s, pdl, sp));
    CU(moe::launch_generic_down(lw, dm, w->h.as<float>(), n_tok, ids, w->y.as<float>(), s, pdl));
  }
  if (!ep) {
    CU(moe::launch_combine(x, ybuf, cgates, n_tok, dm, x_out, s, pdl, nsplit, ids, split_of));
  } else {
    float* delta = w->delta.as<float>();
    CU(moe::launch_combine(nullptr, ybuf, cgates, n_tok, dm, delta, s, pdl, nsplit, ids,
                           split_of));
    const long long nd = (long long)n_tok * dm.d;
    if (w->ctx->peers && nd <= w->ctx->pa.mt_cap) {
      // reduce-scatter + all-gather over the peer windows (no NCCL)
      CU(moe::launch_peer_allreduce(delta, x, x_out, nd, w->ctx->pa, s));
    } else {
      TRY(allreduce(w, delta, (size_t)nd, s));
      CU(moe::launch_add(x, delta, x_out, nd, s, false));
    }
  }
  if (next_router)
    CU(moe::launch_router_topk(next_router, x_out, n_tok, dm, next_ids, next_gates, s, pdl));
  return MOE_OK;
}

// Enqueue the whole L-layer forward on stream s (x in place).
int enqueue_forward(moe_weights* w, float* x, int n_tok, int32_t* ids, float* gates,
                    cudaStream_t s, float* post_all) {
  const int L = w->L();
  const Dims dm = w->dims();
  const size_t tk = (size_t)n_tok * dm.k;
  const bool pdl = true;
  // fused prefill: every layer routes inside its own first kernel
  const bool fused = use_fused_prefill(w, n_tok, post_all);
  if (!fused) CU(moe::launch_router_topk(w->router, x, n_tok, dm, ids, gates, s, false));
  const float* cur = x;
  for (int l = 0; l < L; ++l) {
    float* nxt = (l == L - 1) ? x : ((l % 2 == 0) ? w->xa.as<float>() : w->xb.as<float>());
    const bool more = l + 1 < L && !fused;
    float* post = post_all ? post_all + (size_t)l * tk * dm.f : nullptr;
    TRY(experts_forward(w, l, cur, n_tok, ids + (size_t)l * tk, gates + (size_t)l * tk, nxt,
                        post, s, pdl,
                        more ? w->router + (size_t)(l + 1) * dm.E * dm.d : nullptr,
                        more ? ids + (size_t)(l + 1) * tk : nullptr,
                        more ? gates + (size_t)(l + 1) * tk : nullptr,
                        fused ? w->router + (size_t)l * dm.E * dm.d : nullptr));
    cur = nxt;
  }
  return MOE_OK;
}

// The batch-1 forward as a CUDA graph, captured once per (x, ids, gates) on a
// private stream (the caller's stream may be the legacy default stream,
// which cannot be captured) and launched on the caller's stream.
// host_io (optional, pinned): the graph also copies in_bytes host -> x before
// the forward and out_bytes x -> host after (the host-buffer API's batch-1
// step as ONE launch; x, ids, gates contiguous on both sides).  The host
// pointer is part of the key (in the stream slot).
int forward_graph(moe_weights* w, float* x, int32_t* ids, float* gates, cudaStream_t s,
                  void* host_io = nullptr, size_t in_bytes = 0, size_t out_bytes = 0) {
  auto key = std::make_tuple(x, ids, gates, reinterpret_cast<cudaStream_t>(host_io),
                             moe::debug_options().stack_kernel);
  auto it = w->graphs.find(key);
  if (it == w->graphs.end()) {
    cudaStream_t cs = w->cap_stream;  // created with the weights (creation may synchronize)
    cudaGraph_t g = nullptr;
    CU(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    int rc = MOE_OK;
    if (host_io && cudaMemcpyAsync(x, host_io, in_bytes, cudaMemcpyHostToDevice, cs) != cudaSuccess)
      rc = fail(MOE_ERR_CUDA, "capture of the token copy failed");
    if (rc == MOE_OK)
      rc = use_stack(w, 1) ? enqueue_stack(w, x, ids, gates, cs)
                           : enqueue_forward(w, x, 1, ids, gates, cs, nullptr);
    if (rc == MOE_OK && host_io &&
        cudaMemcpyAsync(host_io, x, out_bytes, cudaMemcpyDeviceToHost, cs) != cudaSuccess)
      rc = fail(MOE_ERR_CUDA, "capture of the result copy failed");
    cudaError_t e = cudaStreamEndCapture(cs, &g);
    if (rc != MOE_OK) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    CU(e);
    GraphEntry ge;
    e = cudaGraphInstantiate(&ge.exec, g, 0);
    cudaGraphDestroy(g);
    CU(e);
    it = w->graphs.emplace(key, ge).first;
  }
  CU(cudaGraphLaunch(it->second.exec, s));
  return MOE_OK;
}

int host_pinned(moe_weights* w, size_t bytes, void** out) {
  if (w->host_pin_bytes < bytes) {
    if (w->host_pin) cudaFreeHost(w->host_pin);
    w->host_pin = nullptr;
    w->host_pin_bytes = 0;
    drop_graphs(w);  // batch-1 host-buffer graphs copy to / from the old buffer
    CU(cudaMallocHost(&w->host_pin, bytes));
    w->host_pin_bytes = bytes;
  }
  *out = w->host_pin;
  return MOE_OK;
}

}  // namespace

// ===========================================================================
extern "C" {

int moe_version(void) { return 1; }

// Debug / A-B switches (kernels.h DebugOptions): the only way to change the
// product's code path besides the shape and the world (no environment reads).
static int* option_slot(const char* name) {
  moe::DebugOptions& o = moe::debug_options();
  static const std::pair<const char*, int moe::DebugOptions::*> table[] = {
      {"stack", &moe::DebugOptions::stack},
      {"stack_kernel", &moe::DebugOptions::stack_kernel},
      {"rw", &moe::DebugOptions::rw},
      {"prefill", &moe::DebugOptions::prefill},
      {"prefill_splits", &moe::DebugOptions::prefill_splits},
      {"stack_grid", &moe::DebugOptions::stack_grid},
      {"virtual_stack", &moe::DebugOptions::virtual_stack},
      {"noncoop", &moe::DebugOptions::noncoop},
      {"force_ep", &moe::DebugOptions::force_ep},
      {"no_pdl", &moe::DebugOptions::no_pdl},
      {"combine4", &moe::DebugOptions::combine4},
      {"prefill_fused", &moe::DebugOptions::prefill_fused},
      {"pf_debug", &moe::DebugOptions::pf_debug},
      {"pf_evict", &moe::DebugOptions::pf_evict},
      {"pf_lag", &moe::DebugOptions::pf_lag},
      {"pf_late8", &moe::DebugOptions::pf_late8},
      {"pf_slo", &moe::DebugOptions::pf_slo},
      {"pf_persist", &moe::DebugOptions::pf_persist},
  };
  if (!name) return nullptr;
  for (const auto& e : table)
    if (std::strcmp(e.first, name) == 0) return &(o.*(e.second));
  return nullptr;
}

int moe_debug_set_option(const char* name, int64_t value) {
  int* p = option_slot(name);
  if (!p) return fail(MOE_ERR_ARG, std::string("unknown debug option: ") + (name ? name : "(null)"));
  *p = (int)value;
  return MOE_OK;
}

int moe_debug_get_option(const char* name, int64_t* value) {
  int* p = option_slot(name);
  if (!p || !value) return fail(MOE_ERR_ARG, std::string("unknown debug option: ") + (name ? name : "(null)"));
  *value = *p;
  return MOE_OK;
}

int moe_debug_set_trace_path(const char* path) {
  moe::trace_path_store() = path ? path : "";
  return MOE_OK;
}
const char* moe_last_error(void) { return g_err.c_str(); }
int moe_shape_validate(const moe_shape* s) { return check_shape(s); }

int moe_ctx_create(int device, moe_ctx** out) {
  if (!out) return fail(MOE_ERR_ARG, "null out");
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    return fail(MOE_ERR_NO_DEVICE, "no CUDA device visible (the product has no CPU path)");
  if (device < 0 || device >= n) return fail(MOE_ERR_ARG, "device index out of range");
  cudaDeviceProp prop;
  CU(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(MOE_ERR_NO_DEVICE, std::string("needs an sm_100 (B200) device, found ") + prop.name);
  auto* c = new moe_ctx();
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    return fail(MOE_ERR_CUDA, cudaGetErrorString(e));
  }
  *out = c;
  return MOE_OK;
}

int moe_ctx_destroy(moe_ctx* c) {
  if (!c) return MOE_OK;
  cudaSetDevice(c->device);
  if (c->comm && nccl() && nccl()->commDestroy) nccl()->commDestroy(c->comm);
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  if (c->win) cudaFree(c->win);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return MOE_OK;
}

void* moe_ctx_stream(moe_ctx* c) { return c ? (void*)c->stream : nullptr; }

int moe_ctx_synchronize(moe_ctx* c) {
  if (!c) return fail(MOE_ERR_ARG, "null ctx");
  TRY(set_device(c));
  CU(cudaStreamSynchronize(c->stream));
  return MOE_OK;
}

int moe_ctx_sm_count(moe_ctx* c) { return c ? c->sm_count : 0; }

int moe_ep_unique_id(void* uid128) {
  if (!uid128) return fail(MOE_ERR_ARG, "null uid");
  NcclApi* api = nccl();
  if (!api) return fail(MOE_ERR_NCCL, "libnccl.so.2 not loadable");
  const int r = api->getUniqueId(uid128);
  if (r) return fail(MOE_ERR_NCCL, "ncclGetUniqueId failed");
  return MOE_OK;
}

int moe_ctx_init_ep(moe_ctx* c, int world, int rank, const void* uid128) {
  if (!c || !uid128) return fail(MOE_ERR_ARG, "null argument");
  if (world < 1 || rank < 0 || rank >= world) return fail(MOE_ERR_ARG, "bad world/rank");
  if (world == 1 && !moe::debug_options().force_ep) {
    c->world = 1;
    c->rank = 0;
    return MOE_OK;
  }
  c->ep_forced = world == 1;  // 1-rank communicator: exercises the EP path on one GPU
  NcclApi* api = nccl();
  if (!api) return fail(MOE_ERR_NCCL, "libnccl.so.2 not loadable");
  TRY(set_device(c));
  NcclUid uid;
  std::memcpy(uid.internal, uid128, 128);
  void* comm = nullptr;
  const int r = reinterpret_cast<CommInitRankFn>(api->commInitRankSym)(&comm, world, uid, rank);
  if (r) return fail(MOE_ERR_NCCL, std::string("ncclCommInitRank: ") + (api->errStr ? api->errStr(r) : "?"));
  c->comm = comm;
  c->world = world;
  c->rank = rank;
  return MOE_OK;
}

int moe_ctx_set_virtual_rank(moe_ctx* c, int world, int rank) {
  if (!c) return fail(MOE_ERR_ARG, "null ctx");
  if (world < 1 || rank < 0 || rank >= world) return fail(MOE_ERR_ARG, "bad world/rank");
  if (c->comm) return fail(MOE_ERR_ARG, "context already has a communicator");
  c->world = world;
  c->rank = rank;
  c->virtual_ep = world > 1;
  return MOE_OK;
}

static int alloc_window(moe_ctx* c, int world, int max_hidden, int max_tokens) {
  if (world < 1 || world > moe::kMaxRanks) return fail(MOE_ERR_ARG, "world must be 1..8");
  if (max_hidden < 1) return fail(MOE_ERR_ARG, "max_hidden < 1");
  if (max_tokens < 0) return fail(MOE_ERR_ARG, "max_tokens < 0");
  if (c->win && (c->win_world != world || c->win_hidden < max_hidden || c->win_tokens < max_tokens))
    return fail(MOE_ERR_ARG, "peer window already allocated with another geometry");
  if (!c->win) {
    TRY(set_device(c));
    const size_t bytes = moe::peer_window_bytes(world, max_hidden, max_tokens);
    CU(cudaMalloc(&c->win, bytes));
    CU(cudaMemset(c->win, 0, bytes));
    CU(cudaDeviceSynchronize());
    c->win_world = world;
    c->win_hidden = max_hidden;
    c->win_tokens = max_tokens;
  }
  return MOE_OK;
}

static void set_peer_parts(moe_ctx* c, int r, void* base) {
  const moe::PeerParts q = moe::peer_window_parts(base, c->win_world, c->win_hidden, c->win_tokens);
  c->pa.inbox[r] = q.inbox;
  c->pa.flags[r] = q.flags;
  c->pa.zbox[r] = q.zbox;
  c->pa.zflags[r] = q.zflags;
  c->pa.mt_recv[r] = q.mt_recv;
  c->pa.mt_gath[r] = q.mt_gath;
  c->pa.mt_pflag[r] = q.mt_pflag;
  c->pa.mt_gflag[r] = q.mt_gflag;
}

static void set_own_parts(moe_ctx* c, int world, int rank) {
  const moe::PeerParts q = moe::peer_window_parts(c->win, world, c->win_hidden, c->win_tokens);
  set_peer_parts(c, rank, c->win);
  c->pa.seq = q.seq;
  c->pa.zseq = q.zseq;
  c->pa.err = q.err;
  c->pa.mt_seq = q.mt_seq;
  c->pa.mt_cap = (long long)c->win_tokens * c->win_hidden;
  c->pa.world = world;
  c->pa.rank = rank;
}

int moe_ctx_peer_window(moe_ctx* c, int world, int max_hidden, void* ipc_handle) {
  return moe_ctx_peer_window_tokens(c, world, max_hidden, 0, ipc_handle);
}

int moe_ctx_peer_window_tokens(moe_ctx* c, int world, int max_hidden, int max_tokens,
                               void* ipc_handle) {
  if (!c) return fail(MOE_ERR_ARG, "null ctx");
  TRY(alloc_window(c, world, max_hidden, max_tokens));
  if (ipc_handle) {
    cudaIpcMemHandle_t h;
    CU(cudaIpcGetMemHandle(&h, c->win));
    std::memcpy(ipc_handle, &h, sizeof(h));
  }
  return MOE_OK;
}

int moe_ctx_open_peers(moe_ctx* c, int world, int rank, const void* handles) {
  if (!c || !handles) return fail(MOE_ERR_ARG, "null argument");
  if (!c->win || c->win_world != world) return fail(MOE_ERR_ARG, "call moe_ctx_peer_window first");
  if (rank < 0 || rank >= world) return fail(MOE_ERR_ARG, "bad rank");
  if (c->comm && (c->world != world || c->rank != rank))
    return fail(MOE_ERR_ARG, "world/rank differ from the NCCL communicator's");
  TRY(set_device(c));
  set_own_parts(c, world, rank);
  for (int r = 0; r < world; ++r) {
    if (r == rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(handles) + (size_t)r * sizeof(h), sizeof(h));
    void* p = nullptr;
    CU(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c->ipc_opened.push_back(p);
    set_peer_parts(c, r, p);
  }
  c->world = world;
  c->rank = rank;
  c->virtual_ep = false;
  c->peers = true;
  return MOE_OK;
}

int moe_ctx_link_peers(moe_ctx* const* ctxs, int world, int max_hidden) {
  return moe_ctx_link_peers_tokens(ctxs, world, max_hidden, 0);
}

int moe_ctx_link_peers_tokens(moe_ctx* const* ctxs, int world, int max_hidden, int max_tokens) {
  if (!ctxs) return fail(MOE_ERR_ARG, "null ctxs");
  if (world < 2 || world > moe::kMaxRanks) return fail(MOE_ERR_ARG, "world must be 2..8");
  for (int r = 0; r < world; ++r) {
    if (!ctxs[r]) return fail(MOE_ERR_ARG, "null ctx");
    if (ctxs[r]->comm) return fail(MOE_ERR_ARG, "context already has a communicator");
    TRY(alloc_window(ctxs[r], world, max_hidden, max_tokens));
  }
  for (int r = 0; r < world; ++r)
    for (int q = 0; q < world; ++q) {
      const int dr = ctxs[r]->device, dq = ctxs[q]->device;
      if (dr == dq) continue;
      int ok = 0;
      CU(cudaDeviceCanAccessPeer(&ok, dr, dq));
      if (!ok) return fail(MOE_ERR_UNSUPPORTED, "no peer access between the contexts' devices");
      CU(cudaSetDevice(dr));
      const cudaError_t e = cudaDeviceEnablePeerAccess(dq, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CU(e);
      cudaGetLastError();
    }
  for (int r = 0; r < world; ++r) {
    moe_ctx* c = ctxs[r];
    set_own_parts(c, world, r);
    for (int q = 0; q < world; ++q) {
      if (q == r) continue;
      set_peer_parts(c, q, ctxs[q]->win);
    }
    c->world = world;
    c->rank = r;
    c->virtual_ep = false;
    c->peers = true;
  }
  return MOE_OK;
}

// diagnostics: this rank's exchange counters (out[0] = zseq, out[1..n-1] = seq[0..n-2])
extern "C" int moe_debug_peer_counters(moe_ctx* c, unsigned* out, int n) {
  if (!c || !out || n < 1) return fail(MOE_ERR_ARG, "bad argument");
  if (!c->peers) return fail(MOE_ERR_ARG, "no peer window");
  TRY(set_device(c));
  CU(cudaMemcpy(out, c->pa.zseq, 4, cudaMemcpyDeviceToHost));
  if (n > 1) CU(cudaMemcpy(out + 1, c->pa.seq, 4 * (size_t)std::min(n - 1, moe::kPeerSlots), cudaMemcpyDeviceToHost));
  return MOE_OK;
}

int moe_ctx_peer_check(moe_ctx* c) {
  if (!c) return fail(MOE_ERR_ARG, "null ctx");
  if (!c->peers) return MOE_OK;
  TRY(set_device(c));
  unsigned err = 0;
  CU(cudaMemcpy(&err, c->pa.err, 4, cudaMemcpyDeviceToHost));
  if (err) return fail(MOE_ERR_NCCL, "peer exchange timed out: a rank never published its slice");
  return MOE_OK;
}

int moe_ctx_world(moe_ctx* c, int* world, int* rank) {
  if (!c) return fail(MOE_ERR_ARG, "null ctx");
  if (world) *world = c->world;
  if (rank) *rank = c->rank;
  return MOE_OK;
}

static int weights_create(moe_ctx* c, const moe_shape* shape, int dtype,
                          const int32_t* owner_rank, bool tensor_parallel, moe_weights** out,
                          const uint32_t* replica_mask = nullptr) {
  if (!c || !out) return fail(MOE_ERR_ARG, "null argument");
  *out = nullptr;
  TRY(check_shape(shape));
  if (tensor_parallel && owner_rank)
    return fail(MOE_ERR_ARG, "tensor parallelism shards every expert: no owner map");
  if (tensor_parallel && shape->ffn_dim % c->world != 0)
    return fail(MOE_ERR_SHAPE, "ffn_dim must be divisible by the tensor-parallel world");
  if (dtype != MOE_DTYPE_BF16 && dtype != MOE_DTYPE_F32) return fail(MOE_ERR_ARG, "bad dtype");
  if (shape->experts_per_layer > moe::kMaxExperts)
    return fail(MOE_ERR_UNSUPPORTED, "experts_per_layer > 256");
  TRY(set_device(c));
  auto* w = new moe_weights();
  w->ctx = c;
  w->shape = *shape;
  w->dtype = dtype;
  w->esize = dtype == MOE_DTYPE_BF16 ? 2 : 4;
  w->tp = tensor_parallel ? c->world : 1;
  w->tp_rank = tensor_parallel ? c->rank : 0;
  w->f_local = shape->ffn_dim / w->tp;
  const int L = shape->num_layers, E = shape->experts_per_layer;
  w->owner.assign((size_t)L * E, tensor_parallel ? c->rank : 0);
  if (owner_rank) {
    for (int i = 0; i < L * E; ++i) {
      if (owner_rank[i] < 0 || owner_rank[i] >= c->world) {
        delete w;
        return fail(MOE_ERR_ARG, "owner rank out of range");
      }
      w->owner[i] = owner_rank[i];
    }
  }
  if (replica_mask && c->world > moe::kReplicaMaxRanks) {
    delete w;
    return fail(MOE_ERR_UNSUPPORTED, "replicas need world <= 8");
  }
  w->holders.assign((size_t)L * E, 0u);
  for (size_t i = 0; i < (size_t)L * E; ++i) {
    const uint32_t extra = replica_mask ? replica_mask[i] : 0u;
    if (c->world < 32 && (extra >> c->world) != 0) {
      delete w;
      return fail(MOE_ERR_ARG, "replica mask names a rank >= world");
    }
    w->holders[i] = (c->world <= 32 ? (1u << w->owner[i]) : 0u) | extra;
    if (extra & ~(1u << w->owner[i])) w->replicas = true;
  }
  // default split cost, from the grouped kernel on B200 (tools/replica_proxy.py):
  // weights at the 6.54 TB/s copy peak (3*d*f*esize B), rows at 1.25 PFLOP/s
  // (6*d*f flop; the 8192-token layer rate), and a fixed ~35 us per expert
  // part (a 256-row part of a Mixtral expert measured ~90 us, not 54)
  w->rep_weight_ps = (long long)(3.0 * shape->hidden_dim * w->f_local * w->esize * 1000.0 / 6540.0);
  w->rep_row_ps = (long long)(6.0 * shape->hidden_dim * w->f_local / 1250.0);
  w->rep_part_ps = w->rep_weight_ps * 2 / 3;
  w->slot_of.assign((size_t)L * E, -1);
  w->exec_slot.assign((size_t)L * E, -1);
  w->n_local.assign(L, 0);
  w->layer_mem.assign(L, nullptr);
  auto cleanup = [&](int rc) {
    moe_weights_destroy(w);
    return rc;
  };
  for (int l = 0; l < L; ++l) {
    int n = 0;
    for (int e = 0; e < E; ++e)
      if (w->owner[(size_t)l * E + e] == c->rank || ((w->holders[(size_t)l * E + e] >> c->rank) & 1u)) {
        w->slot_of[(size_t)l * E + e] = (int16_t)n;
        if (w->owner[(size_t)l * E + e] == c->rank) w->exec_slot[(size_t)l * E + e] = (int16_t)n;
        ++n;
      }
    w->n_local[l] = n;
    const size_t bytes = (size_t)n * 3 * w->mat_elems() * w->esize;
    if (bytes) {
      cudaError_t e = cudaMalloc(&w->layer_mem[l], bytes);
      if (e != cudaSuccess)
        return cleanup(fail(MOE_ERR_OOM, "cudaMalloc experts: " + std::string(cudaGetErrorString(e))));
      w->device_bytes += bytes;
    }
  }
  const size_t rbytes = (size_t)std::max(1, L) * E * shape->hidden_dim * 4;
  if (cudaMalloc(&w->router, rbytes) != cudaSuccess)
    return cleanup(fail(MOE_ERR_OOM, "cudaMalloc router"));
  if (cudaMemset(w->router, 0, rbytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
    return cleanup(fail(MOE_ERR_CUDA, "router memset failed"));
  w->device_bytes += rbytes;
  w->plan = moe::plan_decode(w->dims(), c->sm_count);
  {
    w->rw_enabled = w->plan.ok && (!c->ep() || c->peers) && L >= 2 && E <= 8 &&
                    (size_t)E * shape->hidden_dim * 4 <= 200 * 1024 && moe::debug_options().rw;
    if (w->rw_enabled) {
      w->rw_mem.resize(L - 1);
      std::vector<const float*> ptrs(L, nullptr);
      for (int l = 0; l + 1 < L; ++l) {
        if (w->rw_mem[l].ensure(sizeof(float) * (size_t)std::max(1, w->n_local[l]) * w->f() * E))
          return cleanup(fail(MOE_ERR_OOM, "cudaMalloc router projections"));
        ptrs[l] = w->rw_mem[l].as<float>();
        w->device_bytes += (int64_t)w->rw_mem[l].bytes;
      }
      if (w->dev_rw.ensure(sizeof(void*) * L) ||
          cudaMemcpy(w->dev_rw.p, ptrs.data(), sizeof(void*) * L, cudaMemcpyHostToDevice))
        return cleanup(fail(MOE_ERR_CUDA, "upload projection table"));
    }
  }
  if (cudaStreamCreateWithFlags(&w->cap_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&w->io_stream, cudaStreamNonBlocking) != cudaSuccess)
    return cleanup(fail(MOE_ERR_CUDA, "create streams"));
  w->stack_enabled = moe::debug_options().stack != 0;
  if (w->rw_enabled && !c->ep() && moe::stack2_supported(w->plan, w->dims())) {
    if (w->stack_acc.ensure(moe::stack2_acc_bytes(w->dims())))  // zeroed: the kernel's invariant
      return cleanup(fail(MOE_ERR_OOM, "cudaMalloc stack accumulators"));
    w->device_bytes += (int64_t)w->stack_acc.bytes;
  }
  w->prefill_enabled = moe::debug_options().prefill != 0;
  w->prefill_splits = moe::debug_options().prefill_splits;
  {
    // device-side tables for the persistent stack kernel
    const int Lm = std::max(1, L);
    if (w->dev_layers.ensure(sizeof(void*) * Lm) || w->dev_slots.ensure(sizeof(int16_t) * Lm * E) ||
        w->dev_res_slots.ensure(sizeof(int16_t) * Lm * E) || w->dev_holders.ensure(4 * (size_t)Lm * E) ||
        w->pf_counts2.ensure(4 * (size_t)E) || w->pf_offsets2.ensure(4 * (size_t)E) ||
        w->xbuf2.ensure(sizeof(float) * 2 * shape->hidden_dim) || w->gbar.ensure(256) ||
        w->rpart.ensure(sizeof(float) * (size_t)std::max(c->sm_count, moe::reduce_blocks(w->dims())) * E))
      return cleanup(fail(MOE_ERR_OOM, "cudaMalloc stack tables"));
    if (L > 0 &&
        (cudaMemcpy(w->dev_layers.p, w->layer_mem.data(), sizeof(void*) * L, cudaMemcpyHostToDevice) ||
         cudaMemcpy(w->dev_slots.p, w->exec_slot.data(), sizeof(int16_t) * L * E, cudaMemcpyHostToDevice) ||
         cudaMemcpy(w->dev_res_slots.p, w->slot_of.data(), sizeof(int16_t) * L * E, cudaMemcpyHostToDevice) ||
         cudaMemcpy(w->dev_holders.p, w->holders.data(), 4 * (size_t)L * E, cudaMemcpyHostToDevice)))
      return cleanup(fail(MOE_ERR_CUDA, "upload stack tables"));
  }
  *out = w;
  return MOE_OK;
}

int moe_weights_create(moe_ctx* c, const moe_shape* shape, int dtype, const int32_t* owner_rank,
                       moe_weights** out) {
  return weights_create(c, shape, dtype, owner_rank, false, out);
}

int moe_weights_create_tp(moe_ctx* c, const moe_shape* shape, int dtype, moe_weights** out) {
  return weights_create(c, shape, dtype, nullptr, true, out);
}

int moe_weights_create_ep(moe_ctx* c, const moe_shape* shape, int dtype, const int32_t* owner_rank,
                          const uint32_t* replica_mask, moe_weights** out) {
  return weights_create(c, shape, dtype, owner_rank, false, out, replica_mask);
}

int moe_debug_kernel_timing(moe_weights* w, int enable, double* total_us, int64_t* launches) {
  if (!w) return fail(MOE_ERR_ARG, "null weights");
  std::lock_guard<std::mutex> lk(w->mu);
  TRY(set_device(w->ctx));
  if (enable) {
    w->ktime_on = true;
    w->kev_used = 0;
    return MOE_OK;
  }
  w->ktime_on = false;
  double tot = 0.0;
  for (size_t i = 0; i < w->kev_used; ++i) {
    CU(cudaEventSynchronize(w->kev[i].second));
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, w->kev[i].first, w->kev[i].second));
    tot += ms * 1e3;
  }
  if (total_us) *total_us = tot;
  if (launches) *launches = (int64_t)w->kev_used;
  return MOE_OK;
}

int moe_weights_set_replica_cost(moe_weights* w, int64_t weight_ps, int64_t row_ps,
                                 int64_t part_ps) {
  if (!w) return fail(MOE_ERR_ARG, "null weights");
  if (weight_ps < 0 || row_ps < 0 || part_ps < 0) return fail(MOE_ERR_ARG, "negative cost");
  w->rep_weight_ps = weight_ps;
  w->rep_row_ps = row_ps;
  w->rep_part_ps = part_ps;
  return MOE_OK;
}

int moe_weights_replica_cost(const moe_weights* w, int64_t* weight_ps, int64_t* row_ps,
                             int64_t* part_ps) {
  if (!w) return fail(MOE_ERR_ARG, "null weights");
  if (weight_ps) *weight_ps = w->rep_weight_ps;
  if (row_ps) *row_ps = w->rep_row_ps;
  if (part_ps) *part_ps = w->rep_part_ps;
  return MOE_OK;
}

int moe_replica_plan(const int32_t* counts, int E, const uint32_t* holders, int world,
                     int64_t weight_ps, int64_t row_ps, int64_t part_ps, int chunk, int rank,
                     int32_t* lo, int32_t* hi, int64_t* makespan) {
  if (!counts || !holders || !lo || !hi) return fail(MOE_ERR_ARG, "null argument");
  if (E < 1 || E > moe::kMaxExperts || world < 1 || world > moe::kReplicaMaxRanks || rank < 0 ||
      rank >= world || chunk < 1 || weight_ps < 0 || row_ps < 0 || part_ps < 0)
    return fail(MOE_ERR_ARG, "bad replica plan arguments");
  std::vector<int32_t> order(E);
  for (int e = 0; e < E; ++e) {
    if (counts[e] < 0) return fail(MOE_ERR_ARG, "negative count");
    order[moe::replica_order_pos(counts, E, e)] = e;
  }
  const moe::ReplicaCost c{weight_ps, row_ps, part_ps, chunk};
  const long long mk = moe::replica_split_plan(counts, order.data(), E, holders, world, c, rank, lo, hi);
  if (makespan) *makespan = mk;
  return MOE_OK;
}

int moe_weights_reserve(moe_weights* w, int max_tokens) {
  if (!w) return fail(MOE_ERR_ARG, "null weights");
  if (max_tokens < 1) return fail(MOE_ERR_ARG, "max_tokens < 1");
  std::lock_guard<std::mutex> lk(w->mu);
  TRY(set_device(w->ctx));
  TRY(ensure_scratch(w, max_tokens));
  if (max_tokens > 1 && use_prefill(w, max_tokens, nullptr)) TRY(ensure_prefill_scratch(w, max_tokens));
  if (w->plan.ok) TRY(ensure_scratch(w, 1));
  TRY(refresh_projection(w));
  return MOE_OK;
}

int moe_weights_tp(const moe_weights* w, int* tp_world, int* tp_rank, int* ffn_local) {
  if (!w) return fail(MOE_ERR_ARG, "null weights");
  if (tp_world) *tp_world = w->tp;
  if (tp_rank) *tp_rank = w->tp_rank;
  if (ffn_local) *ffn_local = w->f_local;
  return MOE_OK;
}

int moe_weights_destroy(moe_weights* w) {
  if (!w) return MOE_OK;
  cudaSetDevice(w->ctx->device);
  for (auto& kv : w->graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  if (w->cap_stream) cudaStreamDestroy(w->cap_stream);
  if (w->io_stream) cudaStreamDestroy(w->io_stream);
  if (w->order_ev) cudaEventDestroy(w->order_ev);
  if (w->ha.cin) cudaStreamSynchronize(w->ha.cin);
  if (w->ha.cout) cudaStreamSynchronize(w->ha.cout);
  for (int i = 0; i < 2; ++i) {
    for (cudaEvent_t e : {w->ha.in_done[i], w->ha.comp_done[i], w->ha.out_done[i]})
      if (e) cudaEventDestroy(e);
    for (DevBuf* b : {&w->ha.x[i], &w->ha.y[i], &w->ha.ids[i], &w->ha.gates[i]}) b->release();
  }
  if (w->ha.cin) cudaStreamDestroy(w->ha.cin);
  if (w->ha.cout) cudaStreamDestroy(w->ha.cout);
  for (DevBuf& b : w->rw_mem) b.release();
  w->dev_rw.release();
  for (void* p : w->layer_mem)
    if (p) cudaFree(p);
  if (w->router) cudaFree(w->router);
  for (DevBuf* b : {&w->ypart, &w->rpart, &w->counter, &w->xa, &w->xb, &w->xin, &w->h, &w->y, &w->delta,
                    &w->ids, &w->gates, &w->post, &w->stage_d, &w->xbuf2, &w->gbar,
                    &w->dev_layers, &w->dev_slots, &w->pf_counts, &w->pf_offsets, &w->pf_perm,
                    &w->pf_xg, &w->pf_h, &w->pf_sync, &w->pf_route})
    b->release();
  for (DevBuf* b : {&w->dev_holders, &w->dev_res_slots, &w->pf_counts2, &w->pf_offsets2, &w->io,
                    &w->stack_acc})
    b->release();
  for (cudaEvent_t e : w->io_ev)
    if (e) cudaEventDestroy(e);
  for (auto& p : w->kev) {
    cudaEventDestroy(p.first);
    cudaEventDestroy(p.second);
  }
  if (w->host_pin) cudaFreeHost(w->host_pin);
  delete w;
  return MOE_OK;
}

int64_t moe_weights_device_bytes(const moe_weights* w) { return w ? w->device_bytes : 0; }

static int check_le(moe_weights* w, int layer, int expert) {
  if (!w) return fail(MOE_ERR_ARG, "null weights");
  if (layer < 0 || layer >= w->L()) return fail(MOE_ERR_SHAPE, "layer index out of range");
  if (expert < 0 || expert >= w->E()) return fail(MOE_ERR_SHAPE, "expert index out of range");
  return MOE_OK;
}

int moe_weights_upload_expert(moe_weights* w, int layer, int expert, const double* w_in,
                              const double* w_gate, const double* w_out) {
  TRY(check_le(w, layer, expert));
  w->rw_dirty = true;
  if (!w_in || !w_gate || !w_out) return fail(MOE_ERR_ARG, "null matrix");
  std::lock_guard<std::mutex> lk(w->mu);
  if (w->slot_of[(size_t)layer * w->E() + expert] < 0) return MOE_OK;  // remote
  TRY(set_device(w->ctx));
  const long long n = w->mat_elems();
  TRY(w->stage_d.ensure((size_t)n * 8));
  cudaStream_t s = w->ctx->stream;
  const double* src[3] = {w_in, w_gate, w_out};
  for (int m = 0; m < 3; ++m) {
    if (m < 2)  // this rank's rows [r0, r0 + f_local) of the [f x d] matrix
      CU(cudaMemcpyAsync(w->stage_d.p, src[m] + w->r0() * w->d(), (size_t)n * 8,
                         cudaMemcpyHostToDevice, s));
    else  // columns [r0, r0 + f_local) of w_out [d x f]
      CU(cudaMemcpy2DAsync(w->stage_d.p, (size_t)w->f() * 8, src[m] + w->r0(),
                           (size_t)w->f_glob() * 8, (size_t)w->f() * 8, (size_t)w->d(),
                           cudaMemcpyHostToDevice, s));
    if (m < 2)
      CU(moe::launch_convert(w->stage_d.as<double>(), w->expert_ptr(layer, expert, m), w->dtype,
                             w->f(), w->d(), false, s));
    else  // w_out [d x f] -> W2T [f x d]
      CU(moe::launch_convert(w->stage_d.as<double>(), w->expert_ptr(layer, expert, m), w->dtype,
                             w->d(), w->f(), true, s));
    CU(cudaStreamSynchronize(s));
  }
  return MOE_OK;
}

int moe_weights_upload_router(moe_weights* w, int layer, const double* router) {
  TRY(check_le(w, layer, 0));
  w->rw_dirty = true;
  if (!router) return fail(MOE_ERR_ARG, "null router");
  std::lock_guard<std::mutex> lk(w->mu);
  TRY(set_device(w->ctx));
  const long long n = (long long)w->E() * w->d();
  TRY(w->stage_d.ensure((size_t)n * 8));
  cudaStream_t s = w->ctx->stream;
  CU(cudaMemcpyAsync(w->stage_d.p, router, (size_t)n * 8, cudaMemcpyHostToDevice, s));
  CU(moe::launch_convert_f32(w->stage_d.as<double>(), w->router + (size_t)layer * n, n, s));
  CU(cudaStreamSynchronize(s));
  return MOE_OK;
}

int moe_weights_random(moe_weights* w, uint64_t seed) {
  if (!w) return fail(MOE_ERR_ARG, "null weights");
  w->rw_dirty = true;
  std::lock_guard<std::mutex> lk(w->mu);
  TRY(set_device(w->ctx));
  cudaStream_t s = w->ctx->stream;
  const float scale = (float)(1.0 / std::sqrt((double)w->d()));
  for (int l = 0; l < w->L(); ++l) {
    for (int e = 0; e < w->E(); ++e) {
      if (w->slot_of[(size_t)l * w->E() + e] < 0) continue;
      for (int m = 0; m < 3; ++m) {
        const uint64_t tag = ((uint64_t)l << 40) | ((uint64_t)e << 8) | (uint64_t)m;
        if (m < 2)
          CU(moe::launch_random(w->expert_ptr(l, e, m), w->dtype, w->f(), w->d(), false, seed,
                                tag, scale, s, w->d(), w->r0() * w->d()));
        else  // w_out [d x f]: this rank's columns, stored transposed
          CU(moe::launch_random(w->expert_ptr(l, e, m), w->dtype, w->d(), w->f(), true, seed,
                                tag, scale, s, w->f_glob(), w->r0()));
      }
    }
    const uint64_t rtag = ((uint64_t)l << 40) | (0xFFFFull << 8) | 3ull;
    CU(moe::launch_random(w->router + (size_t)l * w->E() * w->d(), MOE_DTYPE_F32, w->E(), w->d(),
                          false, seed, rtag, scale, s));
  }
  CU(cudaStreamSynchronize(s));
  return MOE_OK;
}

int moe_weights_download_expert(moe_weights* w, int layer, int expert, double* w_in,
                                double* w_gate, double* w_out) {
  TRY(check_le(w, layer, expert));
  std::lock_guard<std::mutex> lk(w->mu);
  if (w->slot_of[(size_t)layer * w->E() + expert] < 0)
    return fail(MOE_ERR_ARG, "expert not resident on this rank");
  TRY(set_device(w->ctx));
  const long long n = w->mat_elems();
  TRY(w->stage_d.ensure((size_t)n * 8));
  cudaStream_t s = w->ctx->stream;
  double* dst[3] = {w_in, w_gate, w_out};
  for (int m = 0; m < 3; ++m) {
    if (!dst[m]) continue;
    if (m < 2)
      CU(moe::launch_to_double(w->expert_ptr(layer, expert, m), w->dtype, w->stage_d.as<double>(),
                               w->f(), w->d(), false, s));
    else
      CU(moe::launch_to_double(w->expert_ptr(layer, expert, m), w->dtype, w->stage_d.as<double>(),
                               w->d(), w->f(), true, s));
    if (m < 2)  // tensor parallel: only this rank's slice of the full-size buffer
      CU(cudaMemcpyAsync(dst[m] + w->r0() * w->d(), w->stage_d.p, (size_t)n * 8,
                         cudaMemcpyDeviceToHost, s));
    else
      CU(cudaMemcpy2DAsync(dst[m] + w->r0(), (size_t)w->f_glob() * 8, w->stage_d.p,
                           (size_t)w->f() * 8, (size_t)w->f() * 8, (size_t)w->d(),
                           cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
  }
  return MOE_OK;
}

int moe_weights_download_router(moe_weights* w, int layer, double* router) {
  TRY(check_le(w, layer, 0));
  if (!router) return fail(MOE_ERR_ARG, "null router");
  std::lock_guard<std::mutex> lk(w->mu);
  TRY(set_device(w->ctx));
  const size_t n = (size_t)w->E() * w->d();
  std::vector<float> tmp(n);
  CU(cudaMemcpy(tmp.data(), w->router + (size_t)layer * n, n * 4, cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < n; ++i) router[i] = tmp[i];
  return MOE_OK;
}

int moe_router_topk(moe_weights* w, int layer, const float* x, int n_tok, int32_t* ids,
                    float* gates, void* stream) {
  TRY(check_le(w, layer, 0));
  if (n_tok < 0) return fail(MOE_ERR_ARG, "n_tok < 0");
  if (n_tok == 0) return MOE_OK;
  if (!x || !ids || !gates) return fail(MOE_ERR_ARG, "null pointer");
  TRY(set_device(w->ctx));
  CU(moe::launch_router_topk(w->router + (size_t)layer * w->E() * w->d(), x, n_tok, w->dims(),
                             ids, gates, pick(w->ctx, stream), false));
  return MOE_OK;
}

int moe_permute(moe_ctx* c, const int32_t* ids, int n_tok, int top_k, int n_experts,
                int32_t* counts, int32_t* offsets, int32_t* perm, int32_t* inv_perm,
                void* stream) {
  if (!c || !counts || !offsets || (n_tok > 0 && (!ids || !perm)))
    return fail(MOE_ERR_ARG, "null pointer");
  if (n_tok < 0 || top_k < 1 || n_experts < 1 || n_experts > moe::kMaxExperts)
    return fail(MOE_ERR_SHAPE, "bad permute geometry");
  TRY(set_device(c));
  CU(moe::launch_permute(ids, n_tok, top_k, n_experts, counts, offsets, perm, inv_perm,
                         pick(c, stream)));
  return MOE_OK;
}

int moe_routing_histogram(moe_ctx* c, const int32_t* ids, int n_layers, int n_tok, int top_k,
                          int n_experts, int64_t* counts, void* stream) {
  if (!c || !counts || (n_layers > 0 && n_tok > 0 && !ids)) return fail(MOE_ERR_ARG, "null pointer");
  if (n_layers < 0 || n_tok < 0 || top_k < 1 || n_experts < 1 || n_experts > moe::kMaxExperts)
    return fail(MOE_ERR_SHAPE, "bad histogram geometry");
  TRY(set_device(c));
  CU(moe::launch_routing_histogram(ids, n_layers, n_tok, top_k, n_experts, counts,
                                   pick(c, stream)));
  return MOE_OK;
}

int moe_routing_trace_step(moe_ctx* c, const int32_t* ids, const float* gates, int n_layers,
                           int n_tok, int top_k, int n_experts, int32_t* token_count,
                           double* gate_weight) {
  if (!c || !token_count || !gate_weight || (n_layers > 0 && n_tok > 0 && (!ids || !gates)))
    return fail(MOE_ERR_ARG, "null pointer");
  if (n_layers < 0 || n_tok < 1 || top_k < 1 || n_experts < 1 || n_experts > moe::kMaxExperts)
    return fail(MOE_ERR_SHAPE, "bad trace geometry");
  TRY(set_device(c));
  const size_t le = (size_t)n_layers * n_experts;
  if (le == 0) return MOE_OK;
  // [counts int32, padded to 8 B][gate sums fp64]
  const size_t dg_off = (le * 4 + 7) & ~(size_t)7;
  void* buf = nullptr;
  CU(cudaMallocAsync(&buf, dg_off + le * 8, c->stream));
  int32_t* dc = static_cast<int32_t*>(buf);
  double* dg = reinterpret_cast<double*>(static_cast<char*>(buf) + dg_off);
  cudaError_t e = moe::launch_trace_step(ids, gates, n_layers, n_tok, top_k, n_experts, dc, dg,
                                         c->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(token_count, dc, le * 4, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(gate_weight, dg, le * 8, cudaMemcpyDeviceToHost, c->stream);
  cudaFreeAsync(buf, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  CU(e);
  for (size_t i = 0; i < le; ++i)
    gate_weight[i] = token_count[i] > 0 ? gate_weight[i] / token_count[i] : 0.0;
  return MOE_OK;
}

int moe_experts_forward(moe_weights* w, int layer, const float* x, int n_tok, const int32_t* ids,
                        const float* gates, float* x_out, float* post_silu, void* stream) {
  TRY(check_le(w, layer, 0));
  if (post_silu && w->tp > 1)
    return fail(MOE_ERR_UNSUPPORTED, "post-SiLU capture of a tensor-parallel shard");
  if (n_tok < 0) return fail(MOE_ERR_ARG, "n_tok < 0");
  if (n_tok == 0) return MOE_OK;
  if (!x || !ids || !gates || !x_out) return fail(MOE_ERR_ARG, "null pointer");
  std::lock_guard<std::mutex> lk(w->mu);
  TRY(set_device(w->ctx));
  TRY(ensure_scratch(w, n_tok));
  StreamOrder so(w, pick(w->ctx, stream));
  return experts_forward(w, layer, x, n_tok, ids, gates, x_out, post_silu, so.s, false, nullptr,
                         nullptr, nullptr);
}

int moe_decode_experts_partial(moe_weights* w, int layer, const float* x, const int32_t* ids,
                               const float* gates, float* ypart, void* stream) {
  TRY(check_le(w, layer, 0));
  if (!x || !ids || !gates || !ypart) return fail(MOE_ERR_ARG, "null pointer");
  if (!w->plan.ok) return fail(MOE_ERR_UNSUPPORTED, "shape has no streaming decode plan");
  TRY(set_device(w->ctx));
  CU(moe::launch_decode_experts(w->plan, w->layer(layer), w->dims(), ids, gates, x, ypart,
                                pick(w->ctx, stream), false));
  return MOE_OK;
}

int moe_layer_forward(moe_weights* w, int layer, const float* x, float* x_out, int n_tok,
                      int32_t* ids, float* gates, void* stream) {
  TRY(check_le(w, layer, 0));
  if (n_tok < 0) return fail(MOE_ERR_ARG, "n_tok < 0");
  if (n_tok == 0) return MOE_OK;
  if (!x || !ids || !gates || !x_out) return fail(MOE_ERR_ARG, "null pointer");
  std::lock_guard<std::mutex> lk(w->mu);
  TRY(set_device(w->ctx));
  TRY(ensure_scratch(w, n_tok));
  StreamOrder so(w, pick(w->ctx, stream));
  cudaStream_t s = so.s;
  return experts_forward(w, layer, x, n_tok, ids, gates, x_out, nullptr, s, true, nullptr, nullptr,
                         nullptr, w->router + (size_t)layer * w->E() * w->d());
}

int moe_forward(moe_weights* w, float* x, int n_tok, int32_t* ids, float* gates, void* stream) {
  if (!w) return fail(MOE_ERR_ARG, "null weights");
  if (n_tok < 0) return fail(MOE_ERR_ARG, "n_tok < 0");
  if (n_tok == 0 || w->L() == 0) return MOE_OK;
  if (!x || !ids || !gates) return fail(MOE_ERR_ARG, "null pointer");
  std::lock_guard<std::mutex> lk(w->mu);
  TRY(set_device(w->ctx));
  TRY(ensure_scratch(w, n_tok));
  TRY(refresh_projection(w));
  StreamOrder so(w, pick(w->ctx, stream));
  cudaStream_t s = so.s;
  if (n_tok == 1 && w->plan.ok) {
    return forward_graph(w, x, ids, gates, s);
  }
  return enqueue_forward(w, x, n_tok, ids, gates, s, nullptr);
}

// Pipelined host-buffer steps: H2D of call i+1 and D2H of call i-1 run on
// their own copy streams while call i computes (two device staging slots).
int moe_forward_host_async(moe_weights* w, int layer, const float* x_host, int n_tok,
                           float* out_host, int32_t* ids_host, float* gates_host, int64_t* ticket) {
  if (!w) return fail(MOE_ERR_ARG, "null weights");
  if (layer < -1 || layer >= w->L()) return fail(MOE_ERR_ARG, "layer out of range");
  if (n_tok < 0) return fail(MOE_ERR_ARG, "n_tok < 0");
  if (n_tok > 0 && (!x_host || !out_host || !ids_host || !gates_host))
    return fail(MOE_ERR_ARG, "null pointer");
  std::lock_guard<std::mutex> lk(w->mu);
  TRY(set_device(w->ctx));
  moe_weights::MoeHostAsync& ha = w->ha;
  if (!ha.cin) {
    if (cudaStreamCreateWithFlags(&ha.cin, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ha.cout, cudaStreamNonBlocking) != cudaSuccess)
      return fail(MOE_ERR_CUDA, "create copy streams");
    for (int i = 0; i < 2; ++i)
      for (cudaEvent_t* e : {&ha.in_done[i], &ha.comp_done[i], &ha.out_done[i]})
        CU(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  }
  const int64_t t = ha.next;
  if (ticket) *ticket = t;
  if (n_tok == 0) return MOE_OK;
  const int slot = (int)(t & 1);
  const int nl = layer < 0 ? w->L() : 1;
  const size_t nx = (size_t)n_tok * w->d(), nr = (size_t)nl * n_tok * w->k();
  TRY(ensure_scratch(w, n_tok));
  TRY(refresh_projection(w));
  // a slot's buffers are reused only after its previous D2H landed (the
  // compute below waits for that too)
  const size_t ny = layer >= 0 ? nx : 0;  // one layer: separate output (the stack runs in place)
  if (ha.x[slot].bytes < nx * 4 || ha.y[slot].bytes < ny * 4 || ha.ids[slot].bytes < nr * 4 ||
      ha.gates[slot].bytes < nr * 4) {
    CU(cudaEventSynchronize(ha.out_done[slot]));
    TRY(ha.x[slot].ensure(nx * 4));
    if (ny) TRY(ha.y[slot].ensure(ny * 4));
    TRY(ha.ids[slot].ensure(nr * 4));
    TRY(ha.gates[slot].ensure(nr * 4));
  }
  float* dx = ha.x[slot].as<float>();
  float* dy = layer >= 0 ? ha.y[slot].as<float>() : dx;
  int32_t* dids = ha.ids[slot].as<int32_t>();
  float* dg = ha.gates[slot].as<float>();
  // in: the slot's previous compute has consumed its tokens and its previous
  // results have left (the layer writes them in place)
  CU(cudaStreamWaitEvent(ha.cin, ha.comp_done[slot], 0));
  CU(cudaStreamWaitEvent(ha.cin, ha.out_done[slot], 0));
  CU(cudaMemcpyAsync(dx, x_host, nx * 4, cudaMemcpyHostToDevice, ha.cin));
  CU(cudaEventRecord(ha.in_done[slot], ha.cin));
  {
    StreamOrder so(w, w->io_stream);
    cudaStream_t s = so.s;
    CU(cudaStreamWaitEvent(s, ha.in_done[slot], 0));
    if (layer >= 0) {
      TRY(experts_forward(w, layer, dx, n_tok, dids, dg, dy, nullptr, s, true, nullptr, nullptr,
                          nullptr, w->router + (size_t)layer * w->E() * w->d()));
    } else if (n_tok == 1 && w->plan.ok) {
      TRY(forward_graph(w, dx, dids, dg, s));
    } else {
      TRY(enqueue_forward(w, dx, n_tok, dids, dg, s, nullptr));
    }
    CU(cudaEventRecord(ha.comp_done[slot], s));
  }
  CU(cudaStreamWaitEvent(ha.cout, ha.comp_done[slot], 0));
  CU(cudaMemcpyAsync(out_host, dy, nx * 4, cudaMemcpyDeviceToHost, ha.cout));
  CU(cudaMemcpyAsync(ids_host, dids, nr * 4, cudaMemcpyDeviceToHost, ha.cout));
  CU(cudaMemcpyAsync(gates_host, dg, nr * 4, cudaMemcpyDeviceToHost, ha.cout));
  CU(cudaEventRecord(ha.out_done[slot], ha.cout));
  ha.next = t + 1;
  return MOE_OK;
}

int moe_host_wait(moe_weights* w, int64_t ticket) {
  if (!w) return fail(MOE_ERR_ARG, "null weights");
  std::lock_guard<std::mutex> lk(w->mu);
  if (!w->ha.cout || ticket >= w->ha.next) return MOE_OK;
  TRY(set_device(w->ctx));
  // out is in-order: the slot's latest D2H covers every earlier ticket of it
  if (ticket < 0) CU(cudaStreamSynchronize(w->ha.cout));
  else CU(cudaEventSynchronize(w->ha.out_done[ticket & 1]));
  return MOE_OK;
}

int moe_forward_sparsity(moe_weights* w, float* x, int n_tok, int32_t* ids, float* gates,
                         const double* thresholds, int n_thresholds, int64_t* counts,
                         void* stream) {
  if (!w) return fail(MOE_ERR_ARG, "null weights");
  if (n_tok < 0) return fail(MOE_ERR_ARG, "n_tok < 0");
  if (!thresholds || !counts) return fail(MOE_ERR_ARG, "null pointer");
  if (n_thresholds < 1 || n_thresholds > moe::kMaxThresholds)
    return fail(MOE_ERR_ARG, "1..8 thresholds");
  for (int i = 1; i < n_thresholds; ++i)  // placement.cpp:130-132
    if (thresholds[i] <= thresholds[i - 1])
      return fail(MOE_ERR_VALIDATION, "thresholds must be strictly increasing");
  if (n_tok == 0 || w->L() == 0) return MOE_OK;
  if (!x || !ids || !gates) return fail(MOE_ERR_ARG, "null pointer");
  std::lock_guard<std::mutex> lk(w->mu);
  TRY(set_device(w->ctx));
  TRY(ensure_scratch(w, n_tok));
  w->sp.counts = reinterpret_cast<unsigned long long*>(counts);
  w->sp.n = n_thresholds;
  for (int i = 0; i < n_thresholds; ++i) w->sp.thr[i] = (float)thresholds[i];
  int rc;
  {
    StreamOrder so(w, pick(w->ctx, stream));
    rc = enqueue_forward(w, x, n_tok, ids, gates, so.s, nullptr);
  }
  w->sp = moe::SparsityCounters();
  return rc;
}

int moe_forward_host(moe_weights* w, const double* tokens, int n_tok, double* out, int32_t* ids,
                     double* gates, double* post_silu) {
  if (!w) return fail(MOE_ERR_ARG, "null weights");
  if (n_tok < 0) return fail(MOE_ERR_ARG, "n_tok < 0");
  const int L = w->L(), d = w->d(), k = w->k(), f = w->f();
  if (n_tok == 0) return MOE_OK;
  if (!tokens || !out) return fail(MOE_ERR_ARG, "null pointer");
  if (L == 0) {
    std::memcpy(out, tokens, sizeof(double) * (size_t)n_tok * d);
    return MOE_OK;
  }
  std::lock_guard<std::mutex> lk(w->mu);
  TRY(set_device(w->ctx));
  TRY(ensure_scratch(w, n_tok));
  TRY(refresh_projection(w));
  StreamOrder so(w, w->io_stream);
  cudaStream_t s = so.s;
  const size_t nx = (size_t)n_tok * d, nr = (size_t)L * n_tok * k;
  if (post_silu && w->tp > 1)
    return fail(MOE_ERR_UNSUPPORTED, "post-SiLU capture of a tensor-parallel shard");
  const size_t npost = post_silu ? (size_t)L * n_tok * k * f : 0;
  void* pin = nullptr;
  TRY(host_pinned(w, nx * 4 + nr * 8 + npost * 4, &pin));
  float* hx = static_cast<float*>(pin);
  int32_t* hids = reinterpret_cast<int32_t*>(hx + nx);
  float* hg = reinterpret_cast<float*>(hids + nr);
  float* hpost = hg + nr;
  if (n_tok == 1 && w->plan.ok && !post_silu) {
    // batch 1: token in, forward, result + routing out — one graph launch
    // and one host wait (x, ids, gates contiguous in w->io as in the pinned
    // buffer)
    TRY(w->io.ensure(nx * 4 + nr * 8));
    float* iox = w->io.as<float>();
    int32_t* ioids = reinterpret_cast<int32_t*>(iox + nx);
    float* iog = reinterpret_cast<float*>(ioids + nr);
    moe_host::to_f32_dma(hx, tokens, nx);
    TRY(refresh_projection(w));
    TRY(forward_graph(w, iox, ioids, iog, s, hx, nx * 4, nx * 4 + nr * 8));
    CU(cudaStreamSynchronize(s));
    moe_host::to_f64(out, hx, nx);
    if (ids) std::memcpy(ids, hids, nr * 4);
    if (gates)
      for (size_t i = 0; i < nr; ++i) gates[i] = hg[i];
    return MOE_OK;
  }
  float* dx = w->xin.as<float>();  // device copy of the tokens (in/out)
  int32_t* dids = w->ids.as<int32_t>();
  float* dg = w->gates.as<float>();
  // prefill-sized calls move the tokens in chunks: the copy engine carries
  // chunk c while the host pool converts chunk c+1 (and the reverse on the
  // way out)
  const int nch = nx >= ((size_t)1 << 20) ? kIoChunks : 1;
  auto lo = [&](int c) { return c == 0 ? (size_t)0 : (nx * c / nch) & ~(size_t)15; };
  auto hi = [&](int c) { return c == nch - 1 ? nx : (nx * (c + 1) / nch) & ~(size_t)15; };
  for (int c = 0; c < nch; ++c) {
    moe_host::to_f32_dma(hx + lo(c), tokens + lo(c), hi(c) - lo(c));
    CU(cudaMemcpyAsync(dx + lo(c), hx + lo(c), (hi(c) - lo(c)) * 4, cudaMemcpyHostToDevice, s));
  }
  if (post_silu) {
    TRY(w->post.ensure(npost * 4));
    // the sink path needs silu(w_in x) per (token, slot): generic kernels, no graph
    TRY(enqueue_forward(w, dx, n_tok, dids, dg, s, w->post.as<float>()));
    CU(cudaMemcpyAsync(hpost, w->post.p, npost * 4, cudaMemcpyDeviceToHost, s));
  } else if (n_tok == 1 && w->plan.ok) {
    TRY(refresh_projection(w));
    TRY(forward_graph(w, dx, dids, dg, s));
  } else {
    TRY(enqueue_forward(w, dx, n_tok, dids, dg, s, nullptr));
  }
  if (nch > 1 && !w->io_ev[0])
    for (auto& e : w->io_ev) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (int c = 0; c < nch; ++c) {
    CU(cudaMemcpyAsync(hx + lo(c), dx + lo(c), (hi(c) - lo(c)) * 4, cudaMemcpyDeviceToHost, s));
    if (nch > 1) CU(cudaEventRecord(w->io_ev[c], s));
  }
  CU(cudaMemcpyAsync(hids, dids, nr * 4, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(hg, dg, nr * 4, cudaMemcpyDeviceToHost, s));
  for (int c = 0; c < nch; ++c) {
    if (nch > 1) CU(cudaEventSynchronize(w->io_ev[c]));
    else CU(cudaStreamSynchronize(s));
    moe_host::to_f64(out + lo(c), hx + lo(c), hi(c) - lo(c));
  }
  CU(cudaStreamSynchronize(s));
  if (ids) std::memcpy(ids, hids, nr * 4);
  if (gates)
    for (size_t i = 0; i < nr; ++i) gates[i] = hg[i];
  if (post_silu) {
    // device layout [l][t][j][r] -> reference sink order [t][l][j][r]
    for (int l = 0; l < L; ++l)
      for (int t = 0; t < n_tok; ++t)
        for (int j = 0; j < k; ++j) {
          const float* src = hpost + (((size_t)l * n_tok + t) * k + j) * f;
          double* dst = post_silu + (((size_t)t * L + l) * k + j) * f;
          for (int r = 0; r < f; ++r) dst[r] = src[r];
        }
  }
  return MOE_OK;
}

int moe_expert_ffn_host(moe_ctx* c, int dtype, int hidden, int ffn, const double* w_in,
                        const double* w_gate, const double* w_out, const double* x, double* y) {
  if (!c || !w_in || !w_gate || !w_out || !x || !y) return fail(MOE_ERR_ARG, "null pointer");
  moe_shape sh{1, 1, 1, hidden, ffn, dtype == MOE_DTYPE_BF16 ? 2 : 4};
  moe_weights* w = nullptr;
  TRY(moe_weights_create(c, &sh, dtype, nullptr, &w));
  int rc = moe_weights_upload_expert(w, 0, 0, w_in, w_gate, w_out);
  if (rc == MOE_OK) {
    std::lock_guard<std::mutex> lk(w->mu);
    cudaStream_t s = c->stream;
    rc = ensure_scratch(w, 1);
    float* dx = w->xa.as<float>();
    float* dy = w->xb.as<float>();
    int32_t* dids = w->ids.as<int32_t>();
    float* dg = w->gates.as<float>();
    std::vector<float> hx(hidden);
    for (int i = 0; i < hidden; ++i) hx[i] = (float)x[i];
    const int32_t id0 = 0;
    const float one = 1.0f;
    if (rc == MOE_OK && (cudaMemcpyAsync(dx, hx.data(), hidden * 4, cudaMemcpyHostToDevice, s) ||
                         cudaMemcpyAsync(dids, &id0, 4, cudaMemcpyHostToDevice, s) ||
                         cudaMemcpyAsync(dg, &one, 4, cudaMemcpyHostToDevice, s)))
      rc = fail(MOE_ERR_CUDA, "H2D failed");
    // y = 1 * expert(x): generic kernels with a zero residual
    if (rc == MOE_OK) {
      const Dims dm = w->dims();
      const LayerWeights lw = w->layer(0);
      if (w->h.ensure((size_t)ffn * 4) || w->y.ensure((size_t)hidden * 4))
        rc = MOE_ERR_OOM;
      else if (moe::launch_generic_up(lw, dm, dx, 1, dids, w->h.as<float>(), nullptr, s, false) ||
          moe::launch_generic_down(lw, dm, w->h.as<float>(), 1, dids, w->y.as<float>(), s, false) ||
          moe::launch_combine(nullptr, w->y.as<float>(), dg, 1, dm, dy, s, false))
        rc = fail(MOE_ERR_CUDA, "expert kernels failed");
    }
    if (rc == MOE_OK) {
      if (cudaMemcpyAsync(hx.data(), dy, hidden * 4, cudaMemcpyDeviceToHost, s) ||
          cudaStreamSynchronize(s))
        rc = fail(MOE_ERR_CUDA, "D2H failed");
      else
        for (int i = 0; i < hidden; ++i) y[i] = hx[i];
    }
  }
  moe_weights_destroy(w);
  return rc;
}

int moe_gate_topk_host(moe_ctx* c, int n_experts, int hidden, const double* router,
                       const double* x, int top_k, int32_t* ids, double* gates) {
  if (!c || !router || !x || !ids || !gates) return fail(MOE_ERR_ARG, "null pointer");
  if (top_k < 1 || top_k > n_experts) return fail(MOE_ERR_SHAPE, "top_k out of range");
  moe_shape sh{1, n_experts, top_k, hidden, 1, 4};
  moe_weights* w = nullptr;
  TRY(moe_weights_create(c, &sh, MOE_DTYPE_F32, nullptr, &w));
  int rc = moe_weights_upload_router(w, 0, router);
  if (rc == MOE_OK) rc = ensure_scratch(w, 1);
  if (rc == MOE_OK) {
    cudaStream_t s = c->stream;
    std::vector<float> hx(hidden), hg(top_k);
    for (int i = 0; i < hidden; ++i) hx[i] = (float)x[i];
    if (cudaMemcpyAsync(w->xa.p, hx.data(), hidden * 4, cudaMemcpyHostToDevice, s) ||
        moe::launch_router_topk(w->router, w->xa.as<float>(), 1, w->dims(), w->ids.as<int32_t>(),
                                w->gates.as<float>(), s, false) ||
        cudaMemcpyAsync(ids, w->ids.p, top_k * 4, cudaMemcpyDeviceToHost, s) ||
        cudaMemcpyAsync(hg.data(), w->gates.p, top_k * 4, cudaMemcpyDeviceToHost, s) ||
        cudaStreamSynchronize(s))
      rc = fail(MOE_ERR_CUDA, "router kernel failed");
    else
      for (int j = 0; j < top_k; ++j) gates[j] = hg[j];
  }
  moe_weights_destroy(w);
  return rc;
}

int moe_expert_path(moe_weights* w, int n_tok) {
  if (!w) return 0;
  if (use_decode(w, n_tok, nullptr)) return 1;
  return use_prefill(w, n_tok, nullptr) ? 3 : 2;
}

int moe_debug_trace_forward(moe_weights* w, float* x, int32_t* ids, float* gates,
                            uint64_t* trace, int64_t cap) {
  if (!w || !x || !ids || !gates || !trace) return fail(MOE_ERR_ARG, "null pointer");
  if (!use_stack(w, 1)) return fail(MOE_ERR_UNSUPPORTED, "no persistent stack plan");
  const size_t n = (size_t)w->L() * w->ctx->sm_count * 16;
  if ((size_t)cap < n) return fail(MOE_ERR_ARG, "trace buffer too small");
  std::lock_guard<std::mutex> lk(w->mu);
  TRY(set_device(w->ctx));
  TRY(ensure_scratch(w, 1));
  TRY(refresh_projection(w));
  DevBuf buf;
  TRY(buf.ensure(n * 8));
  cudaStream_t s = w->ctx->stream;
  int rc = enqueue_stack(w, x, ids, gates, s, buf.as<unsigned long long>());
  if (rc == MOE_OK && (cudaMemcpyAsync(trace, buf.p, n * 8, cudaMemcpyDeviceToHost, s) ||
                       cudaStreamSynchronize(s)))
    rc = fail(MOE_ERR_CUDA, "trace copy failed");
  buf.release();
  return rc;
}

int moe_forward_logits(moe_weights* w, float* x, int32_t* ids, float* gates, float* logits,
                       void* stream) {
  if (!w || !x || !ids || !gates || !logits) return fail(MOE_ERR_ARG, "null pointer");
  if (!use_stack(w, 1) || !use_stack2(w))
    return fail(MOE_ERR_UNSUPPORTED, "no single-barrier persistent stack plan for these weights");
  std::lock_guard<std::mutex> lk(w->mu);
  TRY(set_device(w->ctx));
  TRY(ensure_scratch(w, 1));
  TRY(refresh_projection(w));
  StreamOrder so(w, pick(w->ctx, stream));
  return enqueue_stack(w, x, ids, gates, so.s, nullptr, logits);
}

int moe_forward_launches(moe_weights* w, int n_tok) {
  if (!w || n_tok <= 0 || w->L() == 0) return 0;
  const int L = w->L();
  const bool ep = w->ctx->ep();
  if (use_stack(w, n_tok)) return 1;
  if (use_decode(w, n_tok, nullptr))  // experts + reduce (+ NCCL all-reduce + residual)
    return 1 + L * (ep && !peer_ok(w) ? 3 : 2);
  // per layer: [permute, gather, up, down] or [up, down], combine, (+add for EP),
  // and the next layer's router
  if (use_fused_prefill(w, n_tok, nullptr)) return 2 * L;  // router(+dispatch bases), grouped kernel
  const int experts =
      use_prefill(w, n_tok, nullptr) ? (w->prefill_splits > 0 ? 3 : 4) : 2;  // grouped: permute, gather, GEMM
  return 1 + L * (experts + 1 + (ep ? 1 : 0)) + (L - 1);
}

}  // extern "C"
