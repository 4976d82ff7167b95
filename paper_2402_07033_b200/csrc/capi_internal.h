// capi_internal.h — shared internals of the C-ABI translation units
// (capi_ctx.cu: context, options, EP / peer windows; capi_weights.cu: device
// weight store; capi_orch.cu: the layer-major orchestration; capi_forward.cu:
// the forward / host-buffer entry points).  Not installed; include/moe_b200.h
// is the interface.
#pragma once

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

using moe::Dims;
using moe::LayerWeights;

namespace capi {

// the message of this thread's last failure (moe_last_error)
extern thread_local std::string g_err;
int fail(int code, const std::string& msg);

#define CU(expr)                                                                      \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess) {                                                          \
      return capi::fail(_e == cudaErrorMemoryAllocation ? MOE_ERR_OOM : MOE_ERR_CUDA, \
                        std::string(#expr) + ": " + cudaGetErrorString(_e));          \
    }                                                                                 \
  } while (0)

#define TRY(expr)                  \
  do {                             \
    int _rc = (expr);              \
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
NcclApi* nccl();  // nullptr when libnccl is not loadable
constexpr int kNcclFloat32 = 7;
constexpr int kNcclSum = 0;

}  // namespace capi

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
  unsigned fc_seq = 0;  // multi-token peer exchanges issued (fused EP combine or delta
                        // all-reduce; the same count on every rank) -> their data parity
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
    if (e != cudaSuccess) return capi::fail(MOE_ERR_OOM, "cudaMalloc scratch failed");
    // legacy-stream memset, waited for on that stream only (the kernels run on
    // non-blocking streams; a device-wide sync would also wait for a peer-linked
    // rank's exchange kernel that is spinning on this process's other ranks)
    if (cudaMemset(p, 0, n) != cudaSuccess || cudaStreamSynchronize(cudaStreamLegacy) != cudaSuccess)
      return capi::fail(MOE_ERR_CUDA, "scratch memset failed");
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
  DevBuf pf_route;  // fused prefill: per-router-block expert counts
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
  bool stack2_ok = false;  // the single-barrier stack kernel fits (accumulators allocated)
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

namespace capi {

inline cudaStream_t pick(moe_ctx* c, void* s) { return s ? static_cast<cudaStream_t>(s) : c->stream; }

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

// ---- shared helpers (capi_orch.cu unless noted) ---------------------------------
int check_shape(const moe_shape* s);
int set_device(moe_ctx* c);
int check_le(moe_weights* w, int layer, int expert);  // capi_weights.cu
void drop_graphs(moe_weights* w);
int ensure_scratch(moe_weights* w, int n_tok);
int ensure_scratch_impl(moe_weights* w, int n_tok);
int allreduce(moe_weights* w, float* buf, size_t count, cudaStream_t s);
bool use_decode(const moe_weights* w, int n_tok, const float* post);
bool peer_ok(const moe_weights* w);
bool use_stack(const moe_weights* w, int n_tok);
int refresh_projection(moe_weights* w);
bool use_stack2(const moe_weights* w);
bool use_layer_stack(const moe_weights* w, int n_tok, const float* post);
int enqueue_layer_stack(moe_weights* w, int l, const float* x, float* x_out, int32_t* ids,
                        float* gates, cudaStream_t s);
int enqueue_stack(moe_weights* w, float* x, int32_t* ids, float* gates, cudaStream_t s,
                  unsigned long long* trace = nullptr, float* logits = nullptr);
bool use_prefill(const moe_weights* w, int n_tok, const float* post);
size_t prefill_h_bytes(const moe_weights* w, int n_tok);
int ensure_prefill_scratch(moe_weights* w, int n_tok);
bool use_fused_prefill(const moe_weights* w, int n_tok, const float* post);
int kernel_events(moe_weights* w, cudaEvent_t& t0, cudaEvent_t& t1);
int experts_forward(moe_weights* w, int l, const float* x, int n_tok, const int32_t* ids,
                    const float* gates, float* x_out, float* post, cudaStream_t s, bool pdl,
                    const float* next_router, int32_t* next_ids, float* next_gates,
                    const float* router_l = nullptr);
int enqueue_forward(moe_weights* w, float* x, int n_tok, int32_t* ids, float* gates,
                    cudaStream_t s, float* post_all);
int forward_graph(moe_weights* w, float* x, int32_t* ids, float* gates, cudaStream_t s,
                  void* host_io = nullptr, size_t in_bytes = 0, size_t out_bytes = 0);
int host_pinned(moe_weights* w, size_t bytes, void** out);

}  // namespace capi

using namespace capi;
