// capi_forward.cu — C-ABI: router / permutation / histogram / trace-step
// entry points, the layer and model forwards (device pointers), the
// host-buffer entry points (synchronous drop-in and pipelined) and
// introspection.
#include "capi_internal.h"
#include "host_io.h"

extern "C" {

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

int moe_routing_pair_histogram(moe_ctx* c, const int32_t* ids, int n_layers, int n_tok, int top_k,
                               int n_experts, int64_t* pairs, void* stream) {
  if (!c || !pairs || (n_layers > 0 && n_tok > 0 && !ids)) return fail(MOE_ERR_ARG, "null pointer");
  if (n_layers < 0 || n_tok < 0 || top_k < 1 || n_experts < 1 || n_experts > moe::kMaxExperts)
    return fail(MOE_ERR_SHAPE, "bad histogram geometry");
  TRY(set_device(c));
  CU(moe::launch_routing_pair_histogram(ids, n_layers, n_tok, top_k, n_experts, pairs,
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
// their own copy streams while call i computes (two device staging slots);
// batch-1 steps keep their copies on the compute stream.
// Device alias of a page-locked host buffer (cudaHostAlloc / torch
// pin_memory / cudaHostRegister), or nullptr for pageable memory.
static void* mapped_alias(const void* h) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, h) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;
  }
  return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
}

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
  if (n_tok == 1) {
    // a decode step waits on its own result before the next token exists:
    // nothing to overlap, so the copies ride the compute stream (no
    // cross-stream event hand-offs on the latency path)
    StreamOrder so(w, w->io_stream);
    cudaStream_t s = so.s;
    // both slots' earlier D2H first: tickets stay completed in order
    CU(cudaStreamWaitEvent(s, ha.out_done[0], 0));
    CU(cudaStreamWaitEvent(s, ha.out_done[1], 0));
    CU(cudaMemcpyAsync(dx, x_host, nx * 4, cudaMemcpyHostToDevice, s));
    if (layer >= 0 && use_layer_stack(w, 1, nullptr)) {
      // one persistent launch whose CTA 0 alone writes the token's output,
      // ids and gates: into pinned caller buffers it writes them directly
      // (device aliases of the host pages), replacing three small D2H copies
      // on the latency path; pageable buffers keep the copies
      void* mo = mapped_alias(out_host);
      void* mi = mapped_alias(ids_host);
      void* mg = mapped_alias(gates_host);
      if (mo && mi && mg) {
        TRY(enqueue_layer_stack(w, layer, dx, static_cast<float*>(mo), static_cast<int32_t*>(mi),
                                static_cast<float*>(mg), s));
        CU(cudaEventRecord(ha.comp_done[slot], s));
        CU(cudaEventRecord(ha.out_done[slot], s));
        ha.next = t + 1;
        return MOE_OK;
      }
    }
    if (layer >= 0) {
      TRY(experts_forward(w, layer, dx, n_tok, dids, dg, dy, nullptr, s, true, nullptr, nullptr,
                          nullptr, w->router + (size_t)layer * w->E() * w->d()));
    } else if (w->plan.ok) {
      TRY(forward_graph(w, dx, dids, dg, s));
    } else {
      TRY(enqueue_forward(w, dx, n_tok, dids, dg, s, nullptr));
    }
    CU(cudaMemcpyAsync(out_host, dy, nx * 4, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(ids_host, dids, nr * 4, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(gates_host, dg, nr * 4, cudaMemcpyDeviceToHost, s));
    CU(cudaEventRecord(ha.comp_done[slot], s));
    CU(cudaEventRecord(ha.out_done[slot], s));
    ha.next = t + 1;
    return MOE_OK;
  }
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
  // results land in ticket order (multi-token D2H in order on the out
  // stream; a batch-1 step's copies ride the compute stream after every
  // earlier D2H), so the slot's latest out event covers every earlier ticket
  if (ticket < 0) ticket = w->ha.next - 1;
  CU(cudaEventSynchronize(w->ha.out_done[ticket & 1]));
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

int moe_layer_launches(moe_weights* w, int n_tok) {
  if (!w || n_tok <= 0 || w->L() == 0) return 0;
  if (use_layer_stack(w, n_tok, nullptr)) return 1;         // the 1-layer persistent stack
  if (use_decode(w, n_tok, nullptr))                         // router, experts, reduce (+ EP exchange)
    return w->ctx->ep() && !peer_ok(w) ? 4 : 3;
  if (use_fused_prefill(w, n_tok, nullptr)) return 3;      // router(+bases), grouped, combine_ready
  const int experts = use_prefill(w, n_tok, nullptr) ? (w->prefill_splits > 0 ? 3 : 4) : 2;
  return 1 + experts + 1 + (w->ctx->ep() ? 1 : 0);
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
  if (use_fused_prefill(w, n_tok, nullptr)) return 3 * L;  // router(+block counts), grouped kernel, combine
  const int experts =
      use_prefill(w, n_tok, nullptr) ? (w->prefill_splits > 0 ? 3 : 4) : 2;  // grouped: permute, gather, GEMM
  return 1 + L * (experts + 1 + (ep ? 1 : 0)) + (L - 1);
}

}  // extern "C"
