// decode.cu — batch-1 MoE decode on sm_100a.
//
// Replaces the reference's per-token expert loop (model.cpp:125-147:
// gate_topk -> expert_ffn x k -> gate-weighted combine -> residual), whose
// cost is matvec's inner loop (model.cpp:26).  At batch 1 the layer is a pure
// weight stream (704.8 MB per Mixtral layer), so the kernel is
// built around HBM bandwidth:
//
//  * One persistent CTA per SM.  The k selected experts' ffn rows
//    (k*f "rows", each = W1 row, W3 row, W2T row of d elements) are split
//    evenly over the CTAs (split over ffn, not over hidden).
//  * A producer warp streams each CTA's rows into a shared-memory ring with
//    1-D TMA bulk copies (cp.async.bulk, L2 evict_first) completing on
//    mbarriers — ~190 KB in flight per SM, independent of register pressure.
//  * Consumer warps keep their slice of x in registers, dot W1/W3 rows in
//    batches of 16 ffn rows, reduce with a 32-value butterfly shuffle +
//    one cross-warp smem step, apply silu(a)*b*gate, then immediately AXPY
//    the matching W2T rows into per-thread partial outputs.  h never leaves
//    the SM; each CTA emits one partial d-vector.
//  * reduce_residual_kernel sums the per-CTA partials in a fixed order
//    (deterministic), adds the residual (model.cpp:147) and computes the next
//    layer's router logits + top-k (model.cpp:69-101) with a last-block-done
//    reduction, so a layer is 2 launches chained with PDL inside one graph.
#include <algorithm>

#include "../../include/moe_b200.h"
#include "common.cuh"
#include "kernels.h"

namespace moe {

constexpr int kBatch = 16;      // ffn rows per up/down batch
constexpr int kMaxSlots = 16;   // top_k limit of the streaming kernel
constexpr int kMaxConsWarps = 8;

struct DecodeArgs {
  LayerWeights lw;
  const int32_t* ids;
  const float* gates;
  const float* x;
  float* ypart;
  int d, f, k;
  int row_bytes, rps, stages, stage_bytes;
};

template <typename W, int NV>
__global__ void __launch_bounds__(kMaxConsWarps * 32 + 32, 1)
    decode_experts_kernel(const __grid_constant__ DecodeArgs a) {
  constexpr int VEC = Elem<W>::kVec;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)a.stages * a.stage_bytes);
  uint64_t* empty = full + a.stages;
  float* red = reinterpret_cast<float*>(empty + a.stages);  // [kMaxConsWarps][32]
  float* h_s = red + kMaxConsWarps * 32;                      // [kBatch]
  __shared__ int s_slot[kMaxSlots];
  __shared__ float s_gate[kMaxSlots];
  __shared__ int s_nloc;

  const int ncons = blockDim.x - 32;
  const int ncw = ncons >> 5;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], ncw);
    }
    fence_mbar_init();
  }
  __syncthreads();
  griddep_wait();
  griddep_launch_dependents();
  if (tid == 0) {
    int n = 0;
    for (int j = 0; j < a.k; ++j) {
      const int slot = a.lw.slot_of[a.ids[j]];
      if (slot >= 0) {
        s_slot[n] = slot;
        s_gate[n] = a.gates[j];
        ++n;
      }
    }
    s_nloc = n;
  }
  __syncthreads();

  const long long T = (long long)s_nloc * a.f;
  const long long g0 = (long long)blockIdx.x * T / gridDim.x;
  const long long g1 = (long long)(blockIdx.x + 1) * T / gridDim.x;
  const int total_vec = (int)(3 * (g1 - g0));
  const W* wbase = reinterpret_cast<const W*>(a.lw.experts);

  if (warp == ncw) {
    // ===== producer: one lane streams the CTA's rows into the ring =====
    if (lane == 0 && total_vec > 0) {
      const uint64_t pol = l2_evict_first_policy();
      int c_slot = 0, c_stage = 0, p = 0;
      uint32_t c_phase = 0;
      for (long long g = g0; g < g1;) {
        const int jj = (int)(g / a.f);
        const int r = (int)(g - (long long)jj * a.f);
        const int nb = (int)min((long long)kBatch, min(g1 - g, (long long)(a.f - r)));
        const W* eb = wbase + (long long)s_slot[jj] * a.lw.expert_stride;
        for (int m = 0; m < 3; ++m) {
          const W* src = eb + m * a.lw.mat_stride + (long long)r * a.d;
          for (int q = 0; q < nb; ++q) {
            if (c_slot == 0) {
              mbar_wait(&empty[c_stage], c_phase ^ 1);
              const int nvec = min(a.rps, total_vec - p);
              mbar_arrive_expect_tx(&full[c_stage], (uint32_t)(nvec * a.row_bytes));
            }
            bulk_g2s(ring + (size_t)c_stage * a.stage_bytes + (size_t)c_slot * a.row_bytes,
                     src + (long long)q * a.d, (uint32_t)a.row_bytes, &full[c_stage], pol);
            ++p;
            if (++c_slot == a.rps) {
              c_slot = 0;
              if (++c_stage == a.stages) {
                c_stage = 0;
                c_phase ^= 1;
              }
            }
          }
        }
        g += nb;
      }
    }
    return;
  }

  // ===== consumers =====
  float xr[NV * VEC];
#pragma unroll
  for (int m = 0; m < NV; ++m) {
    const float4* xp = reinterpret_cast<const float4*>(a.x + (size_t)(tid + m * ncons) * VEC);
#pragma unroll
    for (int v = 0; v < VEC / 4; ++v) {
      const float4 t = xp[v];
      xr[m * VEC + 4 * v + 0] = t.x;
      xr[m * VEC + 4 * v + 1] = t.y;
      xr[m * VEC + 4 * v + 2] = t.z;
      xr[m * VEC + 4 * v + 3] = t.w;
    }
  }
  float yacc[NV * VEC];
#pragma unroll
  for (int i = 0; i < NV * VEC; ++i) yacc[i] = 0.f;

  int c_slot = 0, c_stage = 0, p = 0;
  uint32_t c_phase = 0;
  auto acquire = [&]() -> const uint8_t* {
    if (c_slot == 0) mbar_wait(&full[c_stage], c_phase);
    return ring + (size_t)c_stage * a.stage_bytes + (size_t)c_slot * a.row_bytes;
  };
  auto release = [&]() {
    ++p;
    if (++c_slot == a.rps || p == total_vec) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[c_stage]);
      c_slot = 0;
      if (++c_stage == a.stages) {
        c_stage = 0;
        c_phase ^= 1;
      }
    }
  };

  for (long long g = g0; g < g1;) {
    const int jj = (int)(g / a.f);
    const int r = (int)(g - (long long)jj * a.f);
    const int nb = (int)min((long long)kBatch, min(g1 - g, (long long)(a.f - r)));
    const float gate = s_gate[jj];

    // -- up: W1 rows [0,nb) then W3 rows [0,nb) of this batch
    float acc[2 * kBatch];
#pragma unroll
    for (int q = 0; q < 2 * kBatch; ++q) {
      acc[q] = 0.f;
      if ((q & (kBatch - 1)) < nb) {
        const uint8_t* row = acquire();
        float s = 0.f;
#pragma unroll
        for (int m = 0; m < NV; ++m) {
          const uint4 v = lds128(row + (size_t)(tid + m * ncons) * 16);
          float w[VEC];
          Elem<W>::unpack(v, w);
#pragma unroll
          for (int i = 0; i < VEC; ++i) s = fmaf(w[i], xr[m * VEC + i], s);
        }
        acc[q] = s;
        release();
      }
    }
    // butterfly reduce-scatter: lane l ends with the warp sum of item l
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
      const bool hi = (lane & s) != 0;
#pragma unroll
      for (int i = 0; i < s; ++i) {
        const float send = hi ? acc[i] : acc[i + s];
        const float keep = hi ? acc[i + s] : acc[i];
        acc[i] = keep + __shfl_xor_sync(MOE_FULL_MASK, send, s);
      }
    }
    red[warp * 32 + lane] = acc[0];
    named_bar_sync(1, ncons);
    if (warp == 0) {
      float tot = 0.f;
      for (int w = 0; w < ncw; ++w) tot += red[w * 32 + lane];
      const float b = __shfl_down_sync(MOE_FULL_MASK, tot, kBatch);
      if (lane < nb) h_s[lane] = gate * (silu_f(tot) * b);
    }
    named_bar_sync(1, ncons);

    // -- down: W2T rows [0,nb): y += h[q] * W2T[r+q][:]
#pragma unroll
    for (int q = 0; q < kBatch; ++q) {
      if (q < nb) {
        const uint8_t* row = acquire();
        const float hq = h_s[q];
#pragma unroll
        for (int m = 0; m < NV; ++m) {
          const uint4 v = lds128(row + (size_t)(tid + m * ncons) * 16);
          float w[VEC];
          Elem<W>::unpack(v, w);
#pragma unroll
          for (int i = 0; i < VEC; ++i) yacc[m * VEC + i] = fmaf(hq, w[i], yacc[m * VEC + i]);
        }
        release();
      }
    }
    g += nb;
  }

  float* out = a.ypart + (size_t)blockIdx.x * a.d;
#pragma unroll
  for (int m = 0; m < NV; ++m) {
    float4* op = reinterpret_cast<float4*>(out + (size_t)(tid + m * ncons) * VEC);
#pragma unroll
    for (int v = 0; v < VEC / 4; ++v)
      op[v] = make_float4(yacc[m * VEC + 4 * v], yacc[m * VEC + 4 * v + 1],
                          yacc[m * VEC + 4 * v + 2], yacc[m * VEC + 4 * v + 3]);
  }
}

// Fixed-order reduction of the per-CTA partials + residual, fused with the
// next layer's router GEMV/top-k.  32 hidden columns per block.
__global__ void __launch_bounds__(256) reduce_residual_kernel(
    const float* __restrict__ ypart, int nparts, const float* x, float* x_out, int d,
    const float* __restrict__ next_router, int E, int k, float* rpart, unsigned* counter,
    int32_t* next_ids, float* next_gates) {
  __shared__ float red[8][33];
  __shared__ float xs[32];
  __shared__ float logits[kMaxExperts];
  __shared__ int s_last;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  griddep_wait();
  griddep_launch_dependents();
  const int i = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (i < d)
    for (int p = warp; p < nparts; p += 8) s += ypart[(size_t)p * d + i];
  red[warp][lane] = s;
  __syncthreads();
  if (warp == 0) {
    float tot = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) tot += red[w][lane];
    float xo = 0.f;
    if (i < d) {
      xo = (x ? x[i] : 0.f) + tot;
      x_out[i] = xo;
    }
    xs[lane] = xo;
  }
  if (next_router == nullptr) return;
  __syncthreads();
  for (int e = warp; e < E; e += 8) {
    const float v = (i < d) ? next_router[(size_t)e * d + i] * xs[lane] : 0.f;
    const float t = warp_sum(v);
    if (lane == 0) rpart[(size_t)blockIdx.x * E + e] = t;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int e = tid; e < E; e += blockDim.x) {
    float l = 0.f;
    for (int b = 0; b < (int)gridDim.x; ++b) l += __ldcg(&rpart[(size_t)b * E + e]);
    logits[e] = l;
  }
  __syncthreads();
  if (tid == 0) {
    topk_softmax(logits, E, k, next_ids, next_gates);
    *counter = 0u;
  }
}

int reduce_blocks(const Dims& dm) { return (dm.d + 31) / 32; }

DecodePlan plan_decode(const Dims& dm, int sm_count) {
  DecodePlan p;
  const int esize = dm.dtype == MOE_DTYPE_BF16 ? 2 : 4;
  const int vec = 16 / esize;
  if (dm.k > kMaxSlots || dm.E > kMaxExperts || dm.d % vec) return p;
  const int nvec = dm.d / vec;
  for (int nv = 1; nv <= 4; ++nv) {
    if (nvec % nv) continue;
    const int nc = nvec / nv;
    if (nc % 32 == 0 && nc <= kMaxConsWarps * 32) {
      p.nv = nv;
      p.ncons = nc;
      break;
    }
  }
  if (!p.nv) return p;
  const int row_bytes = dm.d * esize;
  p.rps = std::max(1, 32768 / row_bytes);
  const int stage = p.rps * row_bytes;
  const int budget = 200 * 1024;
  p.stages = std::min(8, budget / stage);
  if (p.stages < 2) return p;
  p.smem = p.stages * stage + 2 * p.stages * 8 + (kMaxConsWarps * 32 + kBatch) * 4;
  p.grid = sm_count;
  p.ok = true;
  return p;
}

template <typename W, int NV>
static cudaError_t launch_decode_t(const DecodePlan& p, const DecodeArgs& a, cudaStream_t s,
                                   bool pdl) {
  auto kern = decode_experts_kernel<W, NV>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.grid);
  cfg.blockDim = dim3(p.ncons + 32);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

template <typename W>
static cudaError_t dispatch_nv(const DecodePlan& p, const DecodeArgs& a, cudaStream_t s,
                               bool pdl) {
  switch (p.nv) {
    case 1: return launch_decode_t<W, 1>(p, a, s, pdl);
    case 2: return launch_decode_t<W, 2>(p, a, s, pdl);
    case 3: return launch_decode_t<W, 3>(p, a, s, pdl);
    case 4: return launch_decode_t<W, 4>(p, a, s, pdl);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_decode_experts(const DecodePlan& p, const LayerWeights& lw, const Dims& dm,
                                  const int32_t* ids, const float* gates, const float* x,
                                  float* ypart, cudaStream_t s, bool pdl) {
  DecodeArgs a;
  a.lw = lw;
  a.ids = ids;
  a.gates = gates;
  a.x = x;
  a.ypart = ypart;
  a.d = dm.d;
  a.f = dm.f;
  a.k = dm.k;
  a.row_bytes = dm.d * (dm.dtype == MOE_DTYPE_BF16 ? 2 : 4);
  a.rps = p.rps;
  a.stages = p.stages;
  a.stage_bytes = p.rps * a.row_bytes;
  if (dm.dtype == MOE_DTYPE_BF16) return dispatch_nv<__nv_bfloat16>(p, a, s, pdl);
  return dispatch_nv<float>(p, a, s, pdl);
}

cudaError_t launch_reduce_residual(const float* ypart, int nparts, const float* x, float* x_out,
                                   const Dims& dm, const float* next_router, float* rpart,
                                   unsigned* counter, int32_t* next_ids, float* next_gates,
                                   cudaStream_t s, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(reduce_blocks(dm));
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, reduce_residual_kernel, ypart, nparts, x, x_out, dm.d,
                            next_router, dm.E, dm.k, rpart, counter, next_ids, next_gates);
}

}  // namespace moe
