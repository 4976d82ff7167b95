// capi_ctx.cu — C-ABI: version / errors / debug options, the device context,
// expert parallelism (NCCL, dlopen'ed) and the NVLink peer-memory windows.
#include <dlfcn.h>

#include "capi_internal.h"

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

namespace capi {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

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

}  // namespace capi

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
      {"pf_cut16", &moe::DebugOptions::pf_cut16},
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
  c->pa.mt_cflag[r] = q.mt_cflag;
  c->pa.mt_tflag[r] = q.mt_tflag;
  c->pa.mt_done[r] = q.mt_seq ? q.mt_seq + 1 : nullptr;
}

static void set_own_parts(moe_ctx* c, int world, int rank) {
  const moe::PeerParts q = moe::peer_window_parts(c->win, world, c->win_hidden, c->win_tokens);
  set_peer_parts(c, rank, c->win);
  c->pa.seq = q.seq;
  c->pa.zseq = q.zseq;
  c->pa.err = q.err;
  c->pa.mt_seq = q.mt_seq;
  c->pa.mt_cap = (long long)c->win_tokens * c->win_hidden;
  c->pa.mt_tokens = c->win_tokens;
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

}  // extern "C"
