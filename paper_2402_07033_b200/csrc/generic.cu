// generic.cu — shape-agnostic CUDA kernels: router top-k, SwiGLU experts for
// any (hidden, ffn, tokens), combine + residual, and the deterministic
// token permutation.  These serve the reference's tiny test geometries
// (hidden 2..6, ffn 2..8, toy 32/64) and any shape the streaming / tcgen05
// kernels do not take.  Still GPU code: there is no CPU path in the product.
#include <algorithm>
#include <cstdlib>

#include "../../include/moe_b200.h"
#include "common.cuh"
#include "kernels.h"

namespace moe {

static cudaLaunchConfig_t make_cfg(dim3 grid, dim3 block, cudaStream_t s, bool pdl,
                                   cudaLaunchAttribute* attr, size_t smem = 0) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl && !debug_options().no_pdl) ? 1 : 0;
  return cfg;
}

// ---- router: gate_topk (model.cpp:69-101) ----------------------------------
// kRouterTok tokens per block; the 256 threads stride the hidden dimension
// (column c belongs to thread c % 256), each thread holding 8 experts x
// kRouterTok fp32 partial dot products, so a token's GEMV is spread over the
// whole block (short dependent chains: latency, not one warp's serial loop,
// bounds it).  Per (token, expert) the summation order is fixed — per-thread
// chain in ascending c, warp butterfly, then the 8 warp partials in warp
// order — and does not depend on n_tok or the token's slot in the block, so
// every caller of this kernel (the per-layer batch-1 path, prefill, any
// chunking) routes a token bit for bit identically.  The persistent stack
// kernels (decode.cu) assemble their logits with their own reductions (a
// different fp32 summation order); their routing is checked against the
// oracle directly (tests/test_gpu_parity_full.py, every layer of the stack).
constexpr int kRouterTok = 4;
__global__ void __launch_bounds__(256) router_topk_kernel(const float* __restrict__ router,
                                                          const float* __restrict__ x, int n_tok,
                                                          int d, int E, int k, int32_t* ids,
                                                          float* gates) {
  __shared__ float part[8][kRouterTok][8];
  __shared__ float logits[kRouterTok][kMaxExperts];
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = warp_uniform(tid >> 5);
  griddep_wait();
  griddep_launch_dependents();
  const int t0 = blockIdx.x * kRouterTok;
  const int nt = min(kRouterTok, n_tok - t0);
  const float* xt = x + (size_t)t0 * d;
  for (int e0 = 0; e0 < E; e0 += 8) {
    const int ne = min(8, E - e0);
    float acc[8][kRouterTok];
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int t = 0; t < kRouterTok; ++t) acc[j][t] = 0.f;
#pragma unroll 4
    for (int c = tid; c < d; c += 256) {
      float xv[kRouterTok];
#pragma unroll
      for (int t = 0; t < kRouterTok; ++t) xv[t] = t < nt ? __ldg(xt + (size_t)t * d + c) : 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < ne) {
          const float r = __ldg(router + (size_t)(e0 + j) * d + c);
#pragma unroll
          for (int t = 0; t < kRouterTok; ++t) acc[j][t] = fmaf(r, xv[t], acc[j][t]);
        }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int t = 0; t < kRouterTok; ++t) {
        const float v = warp_sum(acc[j][t]);
        if (lane == 0) part[warp][t][j] = v;
      }
    __syncthreads();
    if (tid < 8 * kRouterTok) {
      const int j = tid & 7, t = tid >> 3;
      if (j < ne && t < nt) {
        float sum = part[0][t][j];
#pragma unroll
        for (int w = 1; w < 8; ++w) sum += part[w][t][j];
        logits[t][e0 + j] = sum;
      }
    }
    __syncthreads();
  }
  for (int t = warp; t < nt; t += 8)
    warp_topk_softmax(logits[t], E, k, ids + (size_t)(t0 + t) * k, gates + (size_t)(t0 + t) * k);
}

// Same arithmetic, for d % 256 == 0: the block's token rows and router rows
// are staged in shared memory by bulk copies (cp.async.bulk) through a
// 2-stage ring of column chunks — both chunks of a d=4096 row are in flight at
// once — instead of each thread's 16+ dependent global loads, which left the
// per-thread loop latency-bound (~30 us at 512 tokens).
//
// Optional dispatch output (rd.blk_count != nullptr; the fused prefill path,
// launch_route_dispatch): every block records how many of its (token, slot)
// pairs chose each expert.  The grouped kernel turns those into the stable
// counting sort's positions (offsets[e] + the counts of the blocks before +
// the rank within the block: exactly permute_kernel's order) and scatters
// each block's pairs itself, without a permute launch.
constexpr int kRouterChunk = 2048;  // columns per chunk (multiple of 256)
constexpr int kRouterStages = 2;
__global__ void __launch_bounds__(256, 1) router_topk_bulk_kernel(const float* __restrict__ router,
                                                                  const float* __restrict__ x,
                                                                  int n_tok, int d, int E, int k,
                                                                  int32_t* ids, float* gates,
                                                                  RouteDispatch rd) {
  extern __shared__ float4 rt_smem4[];
  constexpr int kStageFloats = (kRouterTok + 8) * kRouterChunk;  // [tok rows | router rows]
  float* stage_base = reinterpret_cast<float*>(rt_smem4);
  __shared__ float part[8][kRouterTok][8];
  __shared__ float logits[kRouterTok][kMaxExperts];
  __shared__ __align__(8) uint64_t bar[kRouterStages];
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = warp_uniform(tid >> 5);
  if (tid == 0) {
    for (int i = 0; i < kRouterStages; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  griddep_wait();
  griddep_launch_dependents();
  const int t0 = blockIdx.x * kRouterTok;
  const int nt = min(kRouterTok, n_tok - t0);
  if (rd.zero != nullptr)  // the grouped kernel's sync words (it starts after this grid)
    for (int i = blockIdx.x * 256 + tid; i < rd.n_zero; i += gridDim.x * 256) rd.zero[i] = 0;
  uint64_t pol_keep, pol_norm;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_norm));
  // steps: (expert group of 8, column chunk), group-major
  const int nch = (d + kRouterChunk - 1) / kRouterChunk;
  const int nsteps = ((E + 7) / 8) * nch;
  auto issue = [&](int st) {
    if (tid != 0 || st >= nsteps) return;
    const int e0 = (st / nch) * 8, c0 = (st % nch) * kRouterChunk;
    const int ne = min(8, E - e0), cw = min(kRouterChunk, d - c0);
    float* xs = stage_base + (st % kRouterStages) * kStageFloats;
    float* rs = xs + kRouterTok * kRouterChunk;
    uint64_t* b = &bar[st % kRouterStages];
    mbar_arrive_expect_tx(b, (uint32_t)((nt + ne) * cw * 4));
    for (int t = 0; t < nt; ++t)
      bulk_g2s(xs + t * kRouterChunk, x + (size_t)(t0 + t) * d + c0, cw * 4, b, pol_norm);
    for (int j = 0; j < ne; ++j)
      bulk_g2s(rs + j * kRouterChunk, router + (size_t)(e0 + j) * d + c0, cw * 4, b, pol_keep);
  };
  for (int st = 0; st < kRouterStages; ++st) issue(st);
  int st = 0;
  for (int e0 = 0; e0 < E; e0 += 8) {
    const int ne = min(8, E - e0);
    float acc[8][kRouterTok];
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int t = 0; t < kRouterTok; ++t) acc[j][t] = 0.f;
    for (int c0 = 0; c0 < d; c0 += kRouterChunk, ++st) {
      const int cw = min(kRouterChunk, d - c0);
      const float* xs = stage_base + (st % kRouterStages) * kStageFloats;
      const float* rs = xs + kRouterTok * kRouterChunk;
      mbar_wait(&bar[st % kRouterStages], (uint32_t)((st / kRouterStages) & 1));
#pragma unroll 2
      for (int c = tid; c < cw; c += 256) {
        float xv[kRouterTok];
#pragma unroll
        for (int t = 0; t < kRouterTok; ++t) xv[t] = xs[t * kRouterChunk + c];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float r = rs[j * kRouterChunk + c];
#pragma unroll
          for (int t = 0; t < kRouterTok; ++t) acc[j][t] = fmaf(r, xv[t], acc[j][t]);
        }
      }
      __syncthreads();  // this stage is refilled next
      issue(st + kRouterStages);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int t = 0; t < kRouterTok; ++t) {
        const float v = warp_sum(acc[j][t]);
        if (lane == 0) part[warp][t][j] = v;
      }
    __syncthreads();
    if (tid < 8 * kRouterTok) {
      const int j = tid & 7, t = tid >> 3;
      if (j < ne && t < nt) {
        float sum = part[0][t][j];
#pragma unroll
        for (int w = 1; w < 8; ++w) sum += part[w][t][j];
        logits[t][e0 + j] = sum;
      }
    }
    __syncthreads();
  }
  for (int t = warp; t < nt; t += 8)
    warp_topk_softmax(logits[t], E, k, ids + (size_t)(t0 + t) * k, gates + (size_t)(t0 + t) * k);
  if (rd.blk_count == nullptr) return;

  // ---- per-block expert counts (fused prefill path) ----
  __shared__ int32_t s_pid[kRouterTok * 256];  // this block's expert ids (k <= E <= 256)
  __syncthreads();  // this block's ids (global) visible to the whole block
  const int npair = nt * k;
  for (int p = tid; p < npair; p += 256) s_pid[p] = ids[(size_t)t0 * k + p];
  __syncthreads();
  for (int e = tid; e < E; e += 256) {
    int c = 0;
    for (int p = 0; p < npair; ++p) c += s_pid[p] == e;
    rd.blk_count[(size_t)blockIdx.x * E + e] = c;
  }
}

cudaError_t launch_router_topk(const float* router, const float* x, int n_tok, const Dims& dm,
                               int32_t* ids, float* gates, cudaStream_t s, bool pdl) {
  if (n_tok <= 0) return cudaSuccess;
  cudaLaunchAttribute attr[1];
  const dim3 grid((n_tok + kRouterTok - 1) / kRouterTok);
  if (dm.d % 256 == 0) {
    const size_t smem = (size_t)kRouterStages * (kRouterTok + 8) * kRouterChunk * sizeof(float);
    cudaError_t e = cudaFuncSetAttribute(router_topk_bulk_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = make_cfg(grid, dim3(256), s, pdl, attr, smem);
    return cudaLaunchKernelEx(&cfg, router_topk_bulk_kernel, router, x, n_tok, dm.d, dm.E, dm.k,
                              ids, gates, RouteDispatch{});
  }
  cudaLaunchConfig_t cfg = make_cfg(grid, dim3(256), s, pdl, attr);
  return cudaLaunchKernelEx(&cfg, router_topk_kernel, router, x, n_tok, dm.d, dm.E, dm.k, ids,
                            gates);
}

bool route_dispatch_supported(const Dims& dm) { return dm.d % 256 == 0 && dm.E <= 256; }
int route_blocks(int n_tok) { return (n_tok + kRouterTok - 1) / kRouterTok; }
int route_block_tokens() { return kRouterTok; }

cudaError_t launch_route_dispatch(const float* router, const float* x, int n_tok, const Dims& dm,
                                  int32_t* ids, float* gates, const RouteDispatch& rd,
                                  cudaStream_t s, bool pdl) {
  if (n_tok <= 0) return cudaSuccess;
  if (!route_dispatch_supported(dm) || rd.blk_count == nullptr) return cudaErrorInvalidValue;
  cudaLaunchAttribute attr[1];
  const size_t smem = (size_t)kRouterStages * (kRouterTok + 8) * kRouterChunk * sizeof(float);
  cudaError_t e = cudaFuncSetAttribute(router_topk_bulk_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = make_cfg(dim3(route_blocks(n_tok)), dim3(256), s, pdl, attr, smem);
  return cudaLaunchKernelEx(&cfg, router_topk_bulk_kernel, router, x, n_tok, dm.d, dm.E, dm.k, ids,
                            gates, rd);
}

// ---- generic SwiGLU up: one warp per (ffn row, token, slot) ---------------
template <typename W>
__global__ void __launch_bounds__(256) generic_up_kernel(LayerWeights lw, int d, int f, int k,
                                                         const float* __restrict__ x,
                                                         const int32_t* __restrict__ ids,
                                                         float* h, float* post_silu,
                                                         SparsityCounters sp) {
  __shared__ unsigned sp_blk[kMaxThresholds];
  const int warp = warp_uniform(threadIdx.x >> 5), lane = threadIdx.x & 31;
  griddep_wait();
  griddep_launch_dependents();
  if (sp.counts) {
    if (threadIdx.x < kMaxThresholds) sp_blk[threadIdx.x] = 0u;
    __syncthreads();
  }
  const int r = blockIdx.x * 8 + warp;
  const int tj = blockIdx.y;
  if (r >= f) {
    if (sp.counts) {
      __syncthreads();
      if (threadIdx.x < sp.n && sp_blk[threadIdx.x])
        atomicAdd(&sp.counts[threadIdx.x], (unsigned long long)sp_blk[threadIdx.x]);
    }
    return;
  }
  const int t = tj / k;
  const int slot = lw.slot_of[ids[tj]];
  float a = 0.f, b = 0.f;
  if (slot >= 0) {
    const W* w1 = reinterpret_cast<const W*>(lw.experts) + slot * lw.expert_stride + (size_t)r * d;
    const W* w3 = w1 + lw.mat_stride;
    const float* xt = x + (size_t)t * d;
    for (int c = lane; c < d; c += 32) {
      const float xv = xt[c];
      a = fmaf(Elem<W>::to_float(w1[c]), xv, a);
      b = fmaf(Elem<W>::to_float(w3[c]), xv, b);
    }
    a = warp_sum(a);
    b = warp_sum(b);
  }
  if (lane == 0) {
    const float sa = slot >= 0 ? silu_f(a) : 0.f;
    h[(size_t)tj * f + r] = sa * b;
    if (post_silu) post_silu[(size_t)tj * f + r] = sa;
    if (sp.counts && slot >= 0)
      for (int i = 0; i < sp.n; ++i)
        if (fabsf(sa) < sp.thr[i]) atomicAdd(&sp_blk[i], 1u);
  }
  if (sp.counts) {
    __syncthreads();
    if (threadIdx.x < sp.n && sp_blk[threadIdx.x])
      atomicAdd(&sp.counts[threadIdx.x], (unsigned long long)sp_blk[threadIdx.x]);
  }
}

// ---- generic SwiGLU down: y[t][j][i] = sum_r W2T[r][i] h[t][j][r] ----------
template <typename W>
__global__ void __launch_bounds__(256) generic_down_kernel(LayerWeights lw, int d, int f, int k,
                                                           const float* __restrict__ h,
                                                           const int32_t* __restrict__ ids,
                                                           float* y) {
  griddep_wait();
  griddep_launch_dependents();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d) return;
  const int tj = blockIdx.y;
  const int slot = lw.slot_of[ids[tj]];
  float acc = 0.f;
  if (slot >= 0) {
    const W* w2t =
        reinterpret_cast<const W*>(lw.experts) + slot * lw.expert_stride + 2 * lw.mat_stride + i;
    const float* hr = h + (size_t)tj * f;
    for (int r = 0; r < f; ++r) acc = fmaf(Elem<W>::to_float(w2t[(size_t)r * d]), hr[r], acc);
  }
  y[(size_t)tj * d + i] = acc;
}

cudaError_t launch_generic_up(const LayerWeights& lw, const Dims& dm, const float* x, int n_tok,
                              const int32_t* ids, float* h, float* post_silu, cudaStream_t s,
                              bool pdl, const SparsityCounters& sp) {
  if (n_tok <= 0) return cudaSuccess;
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg =
      make_cfg(dim3((dm.f + 7) / 8, n_tok * dm.k), dim3(256), s, pdl, attr);
  if (dm.dtype == MOE_DTYPE_BF16)
    return cudaLaunchKernelEx(&cfg, generic_up_kernel<__nv_bfloat16>, lw, dm.d, dm.f, dm.k, x,
                              ids, h, post_silu, sp);
  return cudaLaunchKernelEx(&cfg, generic_up_kernel<float>, lw, dm.d, dm.f, dm.k, x, ids, h,
                            post_silu, sp);
}

cudaError_t launch_generic_down(const LayerWeights& lw, const Dims& dm, const float* h,
                                int n_tok, const int32_t* ids, float* y, cudaStream_t s,
                                bool pdl) {
  if (n_tok <= 0) return cudaSuccess;
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg =
      make_cfg(dim3((dm.d + 127) / 128, n_tok * dm.k), dim3(128), s, pdl, attr);
  if (dm.dtype == MOE_DTYPE_BF16)
    return cudaLaunchKernelEx(&cfg, generic_down_kernel<__nv_bfloat16>, lw, dm.d, dm.f, dm.k, h,
                              ids, y);
  return cudaLaunchKernelEx(&cfg, generic_down_kernel<float>, lw, dm.d, dm.f, dm.k, h, ids, y);
}

// ---- combine + residual (model.cpp:128, 143, 147) ---------------------------
// combined = 0; combined += g_j * y_j over slots (ids ascending); x += combined.
// x == nullptr writes the bare combined delta (expert-parallel partials).
__global__ void __launch_bounds__(256) combine_kernel(const float* x, const float* __restrict__ y,
                                                      const float* __restrict__ gates, int k, int d,
                                                      float* x_out, int nsplit, long long sstride,
                                                      const int32_t* __restrict__ ids,
                                                      const int32_t* __restrict__ split_of) {
  griddep_wait();
  griddep_launch_dependents();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d) return;
  const int t = blockIdx.y;
  float c = 0.f;
  // gates == nullptr: y already carries the gate (tcgen05 prefill epilogue)
  for (int j = 0; j < k; ++j) {
    const float g = gates ? gates[(size_t)t * k + j] : 1.0f;
    const int ns = split_of ? split_of[ids[(size_t)t * k + j]] : nsplit;
    for (int sp = 0; sp < ns; ++sp)  // K-split partials, fixed order
      c += g * y[sp * sstride + ((size_t)t * k + j) * d + i];
  }
  x_out[(size_t)t * d + i] = (x ? x[(size_t)t * d + i] : 0.f) + c;
}

// float4 variant (d % 4 == 0): same per-element arithmetic order.  One block
// per token: the slot gates / split counts are read once into smem, and each
// thread keeps several float4 columns' loads in flight (the per-pair split
// lookup used to be a dependent load chain per element).
constexpr int kCombineCols = 4;  // float4 columns per thread per pass
__global__ void __launch_bounds__(256) combine4_kernel(const float* x, const float* __restrict__ y,
                                                       const float* __restrict__ gates, int k, int d,
                                                       float* x_out, int nsplit, long long sstride,
                                                       const int32_t* __restrict__ ids,
                                                       const int32_t* __restrict__ split_of) {
  __shared__ float s_g[32];
  __shared__ int s_ns[32];
  griddep_wait();
  griddep_launch_dependents();
  const int t = blockIdx.x;
  if (threadIdx.x < k) {
    const int j = threadIdx.x;
    s_g[j] = gates ? gates[(size_t)t * k + j] : 1.0f;
    s_ns[j] = split_of ? split_of[ids[(size_t)t * k + j]] : nsplit;
  }
  __syncthreads();
  const int n4 = d / 4;
  const float4* y4 = reinterpret_cast<const float4*>(y);
  for (int c0 = threadIdx.x; c0 < n4; c0 += blockDim.x * kCombineCols) {
    float4 acc[kCombineCols];
#pragma unroll
    for (int u = 0; u < kCombineCols; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = 0; j < k; ++j) {
      const float g = s_g[j];
      const int ns = s_ns[j];
      for (int sp = 0; sp < ns; ++sp) {
        const float4* row = y4 + (sp * sstride + ((size_t)t * k + j) * d) / 4;
        float4 v[kCombineCols];
#pragma unroll
        for (int u = 0; u < kCombineCols; ++u) {
          const int i4 = c0 + u * blockDim.x;
          v[u] = i4 < n4 ? __ldg(row + i4) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < kCombineCols; ++u) {
          acc[u].x += g * v[u].x;
          acc[u].y += g * v[u].y;
          acc[u].z += g * v[u].z;
          acc[u].w += g * v[u].w;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kCombineCols; ++u) {
      const int i4 = c0 + u * blockDim.x;
      if (i4 >= n4) continue;
      float4 o = acc[u];
      if (x) {
        const float4 xv = reinterpret_cast<const float4*>(x + (size_t)t * d)[i4];
        o = make_float4(xv.x + o.x, xv.y + o.y, xv.z + o.z, xv.w + o.w);
      }
      reinterpret_cast<float4*>(x_out + (size_t)t * d)[i4] = o;
    }
  }
}

// top-2 with at most 2 K-split partials per slot (the tcgen05 prefill's
// default): every load of the token's row (x, 2 slots x 2 partials) is issued
// before the first add, instead of one dependent round per (slot, partial) —
// the same adds in the same order as combine4_kernel, so bit-identical.
__global__ void __launch_bounds__(256) combine_k2_kernel(const float* x, const float* __restrict__ y,
                                                         const float* __restrict__ gates, int d,
                                                         float* x_out, int nsplit, long long sstride,
                                                         const int32_t* __restrict__ ids,
                                                         const int32_t* __restrict__ split_of) {
  griddep_wait();
  griddep_launch_dependents();
  const int t = blockIdx.x;
  const float g0 = gates ? gates[(size_t)t * 2] : 1.0f;
  const float g1 = gates ? gates[(size_t)t * 2 + 1] : 1.0f;
  const int ns0 = split_of ? split_of[ids[(size_t)t * 2]] : nsplit;
  const int ns1 = split_of ? split_of[ids[(size_t)t * 2 + 1]] : nsplit;
  const int n4 = d / 4;
  const float4* r00 = reinterpret_cast<const float4*>(y + ((size_t)t * 2) * d);
  const float4* r10 = reinterpret_cast<const float4*>(y + ((size_t)t * 2 + 1) * d);
  const float4* r01 = reinterpret_cast<const float4*>(y + sstride + ((size_t)t * 2) * d);
  const float4* r11 = reinterpret_cast<const float4*>(y + sstride + ((size_t)t * 2 + 1) * d);
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int c0 = threadIdx.x; c0 < n4; c0 += blockDim.x * kCombineCols) {
    float4 v00[kCombineCols], v01[kCombineCols], v10[kCombineCols], v11[kCombineCols],
        xv[kCombineCols];
#pragma unroll
    for (int u = 0; u < kCombineCols; ++u) {
      const int i4 = c0 + u * blockDim.x;
      const bool in = i4 < n4;
      v00[u] = in ? __ldg(r00 + i4) : z;
      v10[u] = in ? __ldg(r10 + i4) : z;
      v01[u] = in && ns0 > 1 ? __ldg(r01 + i4) : z;
      v11[u] = in && ns1 > 1 ? __ldg(r11 + i4) : z;
      xv[u] = in && x ? reinterpret_cast<const float4*>(x + (size_t)t * d)[i4] : z;
    }
#pragma unroll
    for (int u = 0; u < kCombineCols; ++u) {
      const int i4 = c0 + u * blockDim.x;
      if (i4 >= n4) continue;
      float4 acc = z;
      acc.x += g0 * v00[u].x;
      acc.y += g0 * v00[u].y;
      acc.z += g0 * v00[u].z;
      acc.w += g0 * v00[u].w;
      if (ns0 > 1) {
        acc.x += g0 * v01[u].x;
        acc.y += g0 * v01[u].y;
        acc.z += g0 * v01[u].z;
        acc.w += g0 * v01[u].w;
      }
      acc.x += g1 * v10[u].x;
      acc.y += g1 * v10[u].y;
      acc.z += g1 * v10[u].z;
      acc.w += g1 * v10[u].w;
      if (ns1 > 1) {
        acc.x += g1 * v11[u].x;
        acc.y += g1 * v11[u].y;
        acc.z += g1 * v11[u].z;
        acc.w += g1 * v11[u].w;
      }
      float4 o = acc;
      if (x) o = make_float4(xv[u].x + o.x, xv[u].y + o.y, xv[u].z + o.z, xv[u].w + o.w);
      reinterpret_cast<float4*>(x_out + (size_t)t * d)[i4] = o;
    }
  }
}

cudaError_t launch_combine(const float* x, const float* y, const float* gates, int n_tok,
                           const Dims& dm, float* x_out, cudaStream_t s, bool pdl, int nsplit,
                           const int32_t* ids, const int32_t* split_of) {
  if (n_tok <= 0) return cudaSuccess;
  cudaLaunchAttribute attr[1];
  const bool k2_off = debug_options().combine4 != 0;  // A/B: the looped kernel
  if (dm.d % 4 == 0 && dm.k == 2 && nsplit <= 2 && !k2_off) {
    cudaLaunchConfig_t cfg = make_cfg(dim3(n_tok), dim3(256), s, pdl, attr);
    const long long sstride = (long long)n_tok * dm.k * dm.d;
    return cudaLaunchKernelEx(&cfg, combine_k2_kernel, x, y, gates, dm.d, x_out, nsplit, sstride,
                              ids, split_of);
  }
  if (dm.d % 4 == 0 && dm.k <= 32) {
    cudaLaunchConfig_t cfg = make_cfg(dim3(n_tok), dim3(256), s, pdl, attr);
    const long long sstride = (long long)n_tok * dm.k * dm.d;
    return cudaLaunchKernelEx(&cfg, combine4_kernel, x, y, gates, dm.k, dm.d, x_out, nsplit,
                              sstride, ids, split_of);
  }
  cudaLaunchConfig_t cfg = make_cfg(dim3((dm.d + 255) / 256, n_tok), dim3(256), s, pdl, attr);
  const long long sstride = (long long)n_tok * dm.k * dm.d;
  return cudaLaunchKernelEx(&cfg, combine_kernel, x, y, gates, dm.k, dm.d, x_out, nsplit, sstride,
                            ids, split_of);
}

// Fused prefill combine (kernels.h launch_combine_ready).  Y is written by
// the concurrently running grouped kernel, so it is read through L2 (ld.cg)
// after the queue flag's acquire.
__global__ void __launch_bounds__(256) combine_ready_kernel(const float* x, const float* y, int d,
                                                            int k, float* x_out, int n_tok,
                                                            long long sstride,
                                                            const int32_t* ids,
                                                            const int32_t* split_of, int* queue) {
  __shared__ int s_t;
  const int n4 = d / 4;
  int slot = threadIdx.x == 0 ? atomicAdd(queue, 1) : 0;  // thread 0 claims one slot ahead
  while (true) {
    if (threadIdx.x == 0) {
      int t = -1;
      if (slot < n_tok) {
        int f;
        do {
          asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(f) : "l"(queue + 4 + slot) : "memory");
          if (!f) __nanosleep(128);
        } while (!f);
        t = f - 1;
        slot = atomicAdd(queue, 1);
      }
      s_t = t;
    }
    __syncthreads();
    const int t = s_t;
    __syncthreads();
    if (t < 0) break;
    for (int c0 = threadIdx.x; c0 < n4; c0 += blockDim.x * kCombineCols) {
      float4 acc[kCombineCols], xv[kCombineCols];
#pragma unroll
      for (int u = 0; u < kCombineCols; ++u) {
        acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        const int i4 = c0 + u * blockDim.x;
        xv[u] = i4 < n4 ? __ldcg(reinterpret_cast<const float4*>(x + (size_t)t * d) + i4) : acc[u];
      }
      for (int j = 0; j < k; ++j) {
        const size_t p = (size_t)t * k + j;
        const int ns = __ldcg(split_of + __ldcg(ids + p));
        for (int sp = 0; sp < ns; ++sp) {
          const float4* r = reinterpret_cast<const float4*>(y + sp * sstride + p * d);
          float4 v[kCombineCols];
#pragma unroll
          for (int u = 0; u < kCombineCols; ++u) {
            const int i4 = c0 + u * blockDim.x;
            v[u] = i4 < n4 ? __ldcg(r + i4) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int u = 0; u < kCombineCols; ++u) {
            acc[u].x += v[u].x;
            acc[u].y += v[u].y;
            acc[u].z += v[u].z;
            acc[u].w += v[u].w;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kCombineCols; ++u) {
        const int i4 = c0 + u * blockDim.x;
        if (i4 < n4)
          reinterpret_cast<float4*>(x_out + (size_t)t * d)[i4] =
              make_float4(xv[u].x + acc[u].x, xv[u].y + acc[u].y, xv[u].z + acc[u].z, xv[u].w + acc[u].w);
      }
    }
  }
  griddep_wait();  // completion of this grid implies the grouped kernel's
}

cudaError_t launch_combine_ready(const float* x, const float* y, int n_tok, const Dims& dm,
                                 float* x_out, int nsplit, const int32_t* ids, const int32_t* split_of,
                                 int* queue, int blocks, cudaStream_t s, bool pdl) {
  if (n_tok <= 0) return cudaSuccess;
  if (dm.d % 4) return cudaErrorInvalidValue;
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = make_cfg(dim3(std::max(1, std::min(blocks, n_tok))), dim3(256), s, pdl, attr);
  const long long sstride = (long long)n_tok * dm.k * dm.d;
  (void)nsplit;
  return cudaLaunchKernelEx(&cfg, combine_ready_kernel, x, y, dm.d, dm.k, x_out, n_tok, sstride, ids,
                            split_of, queue);
}

__global__ void add_kernel(const float* a, const float* __restrict__ b, float* out, long long n) {
  griddep_wait();
  griddep_launch_dependents();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = a[i] + b[i];
}

cudaError_t launch_add(const float* a, const float* b, float* out, long long n, cudaStream_t s,
                       bool pdl) {
  if (n <= 0) return cudaSuccess;
  cudaLaunchAttribute attr[1];
  const int blocks = (int)((n + 255) / 256 < 1184 ? (n + 255) / 256 : 1184);
  cudaLaunchConfig_t cfg = make_cfg(dim3(blocks), dim3(256), s, pdl, attr);
  return cudaLaunchKernelEx(&cfg, add_kernel, a, b, out, n);
}

// ---- deterministic permutation ------------------------------
// Flatten (token t, slot j) -> p = t*k+j, stable counting sort by expert:
// perm[offsets[e] + rank] = p with ranks ascending in p.  One block; each
// 1024-pair chunk ranks its pairs with warp match + per-warp counts, so the
// result never depends on atomic order.
__global__ void __launch_bounds__(1024) permute_kernel(const int32_t* __restrict__ ids, int n,
                                                       int E, int32_t* counts, int32_t* offsets,
                                                       int32_t* perm, int32_t* inv_perm) {
  extern __shared__ int32_t sm[];
  int32_t* run = sm;             // [E] running count per expert
  int32_t* off = run + E;        // [E] exclusive offsets
  int32_t* wcnt = off + E;       // [32][E] per-warp counts of the chunk
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = warp_uniform(tid >> 5);
  griddep_wait();
  griddep_launch_dependents();
  for (int e = tid; e < E; e += blockDim.x) run[e] = 0;
  __syncthreads();
  // pass 1: counts
  for (int p = tid; p < n; p += blockDim.x) atomicAdd(&run[ids[p]], 1);
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    for (int e = 0; e < E; ++e) {
      off[e] = acc;
      counts[e] = run[e];
      offsets[e] = acc;
      acc += run[e];
    }
  }
  __syncthreads();
  for (int e = tid; e < E; e += blockDim.x) run[e] = 0;
  __syncthreads();
  // pass 2: stable ranks, chunk by chunk
  for (int base = 0; base < n; base += blockDim.x) {
    for (int q = tid; q < 32 * E; q += blockDim.x) wcnt[q] = 0;
    __syncthreads();
    const int p = base + tid;
    const bool valid = p < n;
    const int e = valid ? ids[p] : -1;
    const unsigned active = __ballot_sync(MOE_FULL_MASK, valid);
    const unsigned same = __match_any_sync(MOE_FULL_MASK, e) & active;
    const int rank_w = __popc(same & ((1u << lane) - 1u));
    if (valid && rank_w == 0) wcnt[warp * E + e] = __popc(same);
    __syncthreads();
    if (valid) {
      int before = run[e];
      for (int w = 0; w < warp; ++w) before += wcnt[w * E + e];
      const int pos = off[e] + before + rank_w;
      perm[pos] = p;
      if (inv_perm) inv_perm[p] = pos;
    }
    __syncthreads();
    for (int q = tid; q < E; q += blockDim.x) {
      int add = 0;
      for (int w = 0; w < 32; ++w) add += wcnt[w * E + q];
      run[q] += add;
    }
    __syncthreads();
  }
}

cudaError_t launch_permute(const int32_t* ids, int n_tok, int k, int E, int32_t* counts,
                           int32_t* offsets, int32_t* perm, int32_t* inv_perm, cudaStream_t s,
                           bool pdl) {
  const int n = n_tok * k;
  const size_t smem = sizeof(int32_t) * (size_t)(2 * E + 32 * E);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(permute_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = make_cfg(dim3(1), dim3(1024), s, pdl, attr, smem);
  return cudaLaunchKernelEx(&cfg, permute_kernel, ids, n, E, counts, offsets, perm, inv_perm);
}

// ---- routing histogram (profile_from_trace, placement.cpp:30-43) -------------
// counts[l][e] += |{(t, j) : ids[l][t][j] == e}|: the per-(layer, expert)
// selection counts a PopularityProfile accumulates, kept on the device across
// forwards (integer atomics: order-independent, exact).
__global__ void __launch_bounds__(256) routing_histogram_kernel(const int32_t* __restrict__ ids,
                                                                int n, int E,
                                                                unsigned long long* counts) {
  extern __shared__ unsigned hist_sm[];
  const int l = blockIdx.y;
  for (int e = threadIdx.x; e < E; e += blockDim.x) hist_sm[e] = 0u;
  __syncthreads();
  const int32_t* row = ids + (size_t)l * n;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int e = row[i];
    if (e >= 0 && e < E) atomicAdd(&hist_sm[e], 1u);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    if (hist_sm[e]) atomicAdd(&counts[(size_t)l * E + e], (unsigned long long)hist_sm[e]);
}

cudaError_t launch_routing_histogram(const int32_t* ids, int L, int n_tok, int k, int E,
                                     int64_t* counts, cudaStream_t s) {
  const int n = n_tok * k;
  if (L <= 0 || n <= 0) return cudaSuccess;
  const int bx = std::min((n + 255) / 256, 64);
  routing_histogram_kernel<<<dim3(bx, L), 256, E * sizeof(unsigned), s>>>(
      ids, n, E, reinterpret_cast<unsigned long long*>(counts));
  return cudaGetLastError();
}

// ---- co-selection histogram (shard_plan.h) ----------------------
// pairs[l][a][b] (a < b) += |{t : experts a and b both among token t's top-k
// at layer l}| — what the co-selection-aware shard map separates.
__global__ void __launch_bounds__(256) routing_pair_histogram_kernel(const int32_t* __restrict__ ids,
                                                                     int n_tok, int k, int E,
                                                                     unsigned long long* pairs,
                                                                     bool in_smem) {
  extern __shared__ unsigned pair_sm[];
  const int l = blockIdx.y;
  unsigned long long* gl = pairs + (size_t)l * E * E;
  if (in_smem)
    for (int i = threadIdx.x; i < E * E; i += blockDim.x) pair_sm[i] = 0u;
  __syncthreads();
  const int32_t* row = ids + (size_t)l * n_tok * k;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n_tok; t += gridDim.x * blockDim.x)
    for (int j1 = 0; j1 < k; ++j1)
      for (int j2 = j1 + 1; j2 < k; ++j2) {
        const int a = row[(size_t)t * k + j1], b = row[(size_t)t * k + j2];
        if (a >= 0 && a < E && b >= 0 && b < E && a != b) {
          const int i = min(a, b) * E + max(a, b);
          if (in_smem)
            atomicAdd(&pair_sm[i], 1u);
          else
            atomicAdd(&gl[i], 1ull);
        }
      }
  if (!in_smem) return;
  __syncthreads();
  for (int i = threadIdx.x; i < E * E; i += blockDim.x)
    if (pair_sm[i]) atomicAdd(&gl[i], (unsigned long long)pair_sm[i]);
}

cudaError_t launch_routing_pair_histogram(const int32_t* ids, int L, int n_tok, int k, int E,
                                          int64_t* pairs, cudaStream_t s) {
  if (L <= 0 || n_tok <= 0 || k < 2) return cudaSuccess;
  const int bx = std::min((n_tok + 255) / 256, 64);
  const bool in_smem = E <= 64;  // 16 KB of shared counters; beyond, global atomics
  routing_pair_histogram_kernel<<<dim3(bx, L), 256, in_smem ? (size_t)E * E * sizeof(unsigned) : 0, s>>>(
      ids, n_tok, k, E, reinterpret_cast<unsigned long long*>(pairs), in_smem);
  return cudaGetLastError();
}

// ---- one RoutingTrace step (model.cpp:120-158) -------------------------------
// For each (layer, expert): the number of (token, slot) pairs routed to it and
// the sum of their gates, accumulated in fp64 in token order — the order of
// the reference's tally / gate_sum loop — so gate_weight = sum / count.
__global__ void trace_step_kernel(const int32_t* __restrict__ ids, const float* __restrict__ gates,
                                  int L, int n, int k, int E, int32_t* count, double* gsum) {
  const int le = blockIdx.x * blockDim.x + threadIdx.x;
  if (le >= L * E) return;
  const int l = le / E, e = le - l * E;
  const int32_t* id = ids + (size_t)l * n * k;
  const float* g = gates + (size_t)l * n * k;
  int c = 0;
  double sacc = 0.0;
  for (int i = 0; i < n * k; ++i)
    if (id[i] == e) {
      ++c;
      sacc += (double)g[i];
    }
  count[le] = c;
  gsum[le] = sacc;
}

cudaError_t launch_trace_step(const int32_t* ids, const float* gates, int L, int n_tok, int k,
                              int E, int32_t* count, double* gsum, cudaStream_t s) {
  if (L <= 0) return cudaSuccess;
  trace_step_kernel<<<(L * E + 127) / 128, 128, 0, s>>>(ids, gates, L, n_tok, k, E, count, gsum);
  return cudaGetLastError();
}

}  // namespace moe
