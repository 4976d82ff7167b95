// capi_weights.cu — C-ABI: the device weight store (create / destroy /
// reserve, expert + router upload, device random init, download, the
// replicated-expert cost model, live kernel timing).
#include "capi_internal.h"
#include "replica_plan.h"
#include "shard_plan.h"

namespace capi {

int check_le(moe_weights* w, int layer, int expert) {
  if (!w) return fail(MOE_ERR_ARG, "null weights");
  if (layer < 0 || layer >= w->L()) return fail(MOE_ERR_SHAPE, "layer index out of range");
  if (expert < 0 || expert >= w->E()) return fail(MOE_ERR_SHAPE, "expert index out of range");
  return MOE_OK;
}

}  // namespace capi

extern "C" {

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
  // the single-barrier kernel: its next-layer logits come from the
  // projections, so L >= 2 needs them; a 1-layer model has no next layer
  w->stack2_ok = w->plan.ok && !c->ep() && E <= 8 && (size_t)E * shape->hidden_dim * 4 <= 200 * 1024 &&
                 moe::debug_options().rw && (L == 1 || w->rw_enabled) &&
                 moe::stack2_supported(w->plan, w->dims());
  if (w->stack2_ok) {
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

int moe_ep_shard_map_coselect(const int64_t* counts, const int64_t* pairs, int n_layers, int n_experts,
                              int world, int32_t* owner, int32_t* exact) {
  if (!counts || !pairs || !owner) return fail(MOE_ERR_ARG, "null argument");
  if (n_layers < 0 || n_experts < 1 || n_experts > moe::kMaxExperts || world < 1)
    return fail(MOE_ERR_ARG, "bad shard map arguments");
  const size_t E = (size_t)n_experts;
  for (size_t i = 0; i < (size_t)n_layers * E; ++i)
    if (counts[i] < 0) return fail(MOE_ERR_VALIDATION, "negative routing count");
  for (size_t i = 0; i < (size_t)n_layers * E * E; ++i)
    if (pairs[i] < 0) return fail(MOE_ERR_VALIDATION, "negative co-selection count");
  std::vector<int> o(E);
  for (int l = 0; l < n_layers; ++l) {
    const bool ex = moe::coselect_layer(pairs + (size_t)l * E * E, counts + (size_t)l * E, n_experts, world,
                                        o.data());
    for (size_t e = 0; e < E; ++e) owner[(size_t)l * E + e] = o[e];
    if (exact) exact[l] = ex ? 1 : 0;
  }
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

}  // extern "C"
