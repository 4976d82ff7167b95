// capi_orch.cu — the layer-major orchestration of the reference's
// model_forward (model.cpp:103-161) on the device: per-call scratch, path
// selection (persistent stack / per-layer decode / fused or unfused tcgen05
// prefill / generic), the expert-parallel combine, batch-1 CUDA graphs.
#include "capi_internal.h"

namespace capi {


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
  return moe::debug_options().stack_kernel >= 2 && !w->ctx->ep() && w->stack2_ok && w->stack_acc.p != nullptr;
}

// One layer at batch 1 (moe_layer_forward) through the single-barrier
// persistent kernel as a 1-layer stack: routing, both projections, the
// combine and the residual in ONE launch instead of router + experts +
// reduce (the layer's tables are the stack's, offset to layer l).
bool use_layer_stack(const moe_weights* w, int n_tok, const float* post) {
  return n_tok == 1 && post == nullptr && w->sp.counts == nullptr && use_stack(w, 1) && use_stack2(w);
}

int enqueue_layer_stack(moe_weights* w, int l, const float* x, float* x_out, int32_t* ids,
                        float* gates, cudaStream_t s) {
  moe::StackDesc sd;
  sd.rw = w->rw_enabled ? w->dev_rw.as<const float* const>() + l : nullptr;  // not read: L = 1
  sd.layer_experts = w->dev_layers.as<const void* const>() + l;
  sd.slot_of = w->dev_slots.as<const int16_t>() + (size_t)l * w->E();
  sd.expert_stride = 3 * w->mat_elems();
  sd.mat_stride = w->mat_elems();
  sd.router = w->router + (size_t)l * w->E() * w->d();
  sd.L = 1;
  CU(moe::launch_decode_stack2(w->plan, sd, w->dims(), const_cast<float*>(x), w->stack_acc.p, ids,
                               gates, nullptr, s, x_out));
  return MOE_OK;
}

int enqueue_stack(moe_weights* w, float* x, int32_t* ids, float* gates, cudaStream_t s,
                  unsigned long long* trace, float* logits) {
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
  TRY(w->pf_route.ensure(4 * (size_t)moe::route_blocks(n_tok) * w->E()));
  return MOE_OK;
}

// The fused prefill layer (router with dispatch bases -> grouped kernel that
// scatters, computes and combines): single GPU, every expert local, the
// grouped kernel (splits > 0), no post-SiLU capture.
bool use_fused_prefill(const moe_weights* w, int n_tok, const float* post) {
  const Dims dm = w->dims();
  const moe_ctx* c = w->ctx;
  // expert / tensor parallelism: the combine is the streamed peer-window
  // reduction (ep_combine_kernel), so the windows must hold the step
  const bool ep_ok = !c->ep() || (peer_ok(w) && n_tok <= c->win_tokens && c->pa.mt_cap > 0 &&
                                  (long long)n_tok * dm.d <= c->pa.mt_cap);
  return use_prefill(w, n_tok, post) && moe::debug_options().prefill_fused && ep_ok &&
         !w->replicas && w->prefill_splits > 0 && moe::route_dispatch_supported(dm) &&
         moe::route_block_tokens() * dm.k <= 64;
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
                    const float* router_l) {
  const Dims dm = w->dims();
  const LayerWeights lw = w->layer(l);
  const bool ep = w->ctx->ep();
  moe::SparsityCounters sp = w->sp;
  if (sp.counts) sp.counts += (size_t)l * sp.n;
  if (router_l) {
    // router_l: route this layer here (ids/gates are outputs) — inside the
    // batch-1 persistent kernel, or fused into the prefill layer's first
    // kernel, when those paths apply
    if (use_layer_stack(w, n_tok, post))
      return enqueue_layer_stack(w, l, x, x_out, const_cast<int32_t*>(ids), const_cast<float*>(gates), s);
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
      if (ep) {
        fz.pa = &w->ctx->pa;
        fz.holders = w->tp > 1 ? nullptr : w->dev_holders.as<uint32_t>() + (size_t)l * dm.E;
        fz.seq = ++w->ctx->fc_seq;
      }
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
      CU(moe::launch_peer_allreduce(delta, x, x_out, nd, w->ctx->pa, ++w->ctx->fc_seq, s));
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
                  void* host_io, size_t in_bytes, size_t out_bytes) {
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

}  // namespace capi
