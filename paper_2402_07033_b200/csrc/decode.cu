// decode.cu — batch-1 MoE decode on sm_100a.
//
// Replaces the reference's per-token expert loop (model.cpp:125-147:
// gate_topk -> expert_ffn x k -> gate-weighted combine -> residual), whose
// cost is matvec's inner loop (model.cpp:26).  At batch 1 the layer is a pure
// weight stream (704.8 MB per Mixtral layer), so the kernels are
// built around HBM bandwidth:
//
//  * One CTA per SM.  The k selected experts' ffn rows (k*f "rows", each =
//    W1 row, W3 row, W2T row of d elements) are split evenly over the CTAs
//    (split over ffn, not over hidden).
//  * A producer warp streams each CTA's rows into a shared-memory ring with
//    1-D TMA bulk copies (cp.async.bulk, L2 evict_first) completing on
//    mbarriers — ~190 KB in flight per SM, independent of register pressure.
//  * Consumer warps keep their slice of x in registers, dot W1/W3 rows in
//    batches of 16 ffn rows, reduce with a 32-value butterfly shuffle +
//    one cross-warp smem step, apply silu(a)*b*gate, then immediately AXPY
//    the matching W2T rows into per-thread partial outputs.  h never leaves
//    the SM; each CTA emits one partial d-vector.
//
// Two drivers share that core:
//  * decode_experts_kernel + reduce_residual_kernel: one layer = 2 launches
//    (PDL-chained); the reduce sums the per-CTA partials in a fixed order,
//    adds the residual (model.cpp:147) and fuses the next layer's router +
//    top-k (model.cpp:69-101) via last-block-done.  Used per layer and for
//    expert parallelism (an NCCL all-reduce sits between the two).
//  * decode_stack_kernel: the whole L-layer token in ONE persistent
//    cooperative launch with two grid barriers per layer; routing of layer
//    l+1 is computed redundantly by every CTA from per-CTA router partials,
//    so the producer warps start streaming layer l+1 without another launch.
#include <algorithm>
#include <cstdlib>

#include "../../include/moe_b200.h"
#include "common.cuh"
#include "kernels.h"

namespace moe {

constexpr int kBatch = 16;      // ffn rows per up/down batch
constexpr int kMaxSlots = 16;   // top_k limit of the streaming kernels
constexpr int kMaxConsWarps = 8;

// ---------------------------------------------------------------------------
// shared streaming core
struct Ring {
  uint8_t* buf;
  uint64_t* full;
  uint64_t* empty;
  int rps, stages, stage_bytes, row_bytes;
};
struct Cursor {
  int slot = 0, stage = 0;
  uint32_t phase = 0;
  __device__ __forceinline__ void next_stage(int stages) {
    slot = 0;
    if (++stage == stages) {
      stage = 0;
      phase ^= 1;
    }
  }
};

// Producer: stream rows [g0, g1) of the layer (row g = slot j, ffn index r)
// as [W1 rows | W3 rows | W2T rows] per batch of <= kBatch rows.
template <typename W>
__device__ __forceinline__ void produce_rows(const Ring& R, Cursor& cur, const W* wbase,
                                             long long expert_stride, long long mat_stride,
                                             const int* s_slot, int f, int d, long long g0,
                                             long long g1, uint64_t pol) {
  const int total_vec = (int)(3 * (g1 - g0));
  int p = 0;
  for (long long g = g0; g < g1;) {
    const int jj = (int)(g / f);
    const int r = (int)(g - (long long)jj * f);
    const int nb = (int)min((long long)kBatch, min(g1 - g, (long long)(f - r)));
    const W* eb = wbase + (long long)s_slot[jj] * expert_stride;
    for (int m = 0; m < 3; ++m) {
      const W* src = eb + m * mat_stride + (long long)r * d;
      for (int q = 0; q < nb; ++q) {
        if (cur.slot == 0) {
          mbar_wait(&R.empty[cur.stage], cur.phase ^ 1);
          const int nvec = min(R.rps, total_vec - p);
          mbar_arrive_expect_tx(&R.full[cur.stage], (uint32_t)(nvec * R.row_bytes));
        }
        bulk_g2s(R.buf + (size_t)cur.stage * R.stage_bytes + (size_t)cur.slot * R.row_bytes,
                 src + (long long)q * d, (uint32_t)R.row_bytes, &R.full[cur.stage], pol);
        ++p;
        if (++cur.slot == R.rps) cur.next_stage(R.stages);
      }
    }
    g += nb;
  }
  if (cur.slot != 0) cur.next_stage(R.stages);
}

// Consumers: accumulate yacc += sum over rows of gate*silu(W1 x)*(W3 x)*W2T.
// Optional router projection (z): with rw = R_{l+1} W2 precomputed per expert
// as [f][E] fp32 (E <= kZMax), warp 0 also accumulates
//   z[e] += sum_r h'_r * rw[r][e]        (h'_r = gate * silu(a_r) * b_r)
// i.e. this CTA's share of the next layer's router logits, with no extra
// pass over W2 and the rw rows prefetched at batch start.
constexpr int kZMax = 8;
template <typename W, int NV>
__device__ __forceinline__ void consume_rows(const Ring& R, Cursor& cur, const float* xr,
                                             float* yacc, const float* s_gate, int f,
                                             long long g0, long long g1, float* red, float* h_s,
                                             int tid, int ncons, int bar_id,
                                             unsigned long long* t_first = nullptr,
                                             const float* rw = nullptr, const int* s_slot = nullptr,
                                             int E = 0, float* zreg = nullptr) {
  constexpr int VEC = Elem<W>::kVec;
  const int warp = warp_uniform(tid >> 5), lane = tid & 31, ncw = ncons >> 5;
  const int total_vec = (int)(3 * (g1 - g0));
  int p = 0;
  auto acquire = [&]() -> const uint8_t* {
    if (cur.slot == 0) mbar_wait(&R.full[cur.stage], cur.phase);
    if (t_first != nullptr && p == 0 && tid == 0) *t_first = clock64();
    return R.buf + (size_t)cur.stage * R.stage_bytes + (size_t)cur.slot * R.row_bytes;
  };
  auto release = [&]() {
    ++p;
    if (++cur.slot == R.rps || p == total_vec) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&R.empty[cur.stage]);
      cur.next_stage(R.stages);
    }
  };
  for (long long g = g0; g < g1;) {
    const int jj = (int)(g / f);
    const int r = (int)(g - (long long)jj * f);
    const int nb = (int)min((long long)kBatch, min(g1 - g, (long long)(f - r)));
    const float gate = s_gate[jj];
    float rwv[kZMax];
    if (rw != nullptr && warp == 0) {  // prefetch: consumed after this batch's up phase
      const float* rp = rw + ((size_t)s_slot[jj] * f + r + lane) * E;
#pragma unroll
      for (int e = 0; e < kZMax; ++e) rwv[e] = (lane < nb && e < E) ? __ldg(rp + e) : 0.f;
    }

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
    named_bar_sync(bar_id, ncons);
    float hq = 0.f;
    if (warp == 0) {
      float tot = 0.f;
      for (int w = 0; w < ncw; ++w) tot += red[w * 32 + lane];
      const float b = __shfl_down_sync(MOE_FULL_MASK, tot, kBatch);
      hq = lane < nb ? gate * (silu_f(tot) * b) : 0.f;
      if (lane < nb) h_s[lane] = hq;
    }
    named_bar_sync(bar_id, ncons);
    // z accumulation after the barrier: the other warps are not held up
    if (rw != nullptr && warp == 0) {
#pragma unroll
      for (int e = 0; e < kZMax; ++e) zreg[e] += warp_sum(hq * rwv[e]);
    }

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
}

template <typename W, int NV>
__device__ __forceinline__ void load_x(const float* x, float* xr, int tid, int ncons) {
  constexpr int VEC = Elem<W>::kVec;
#pragma unroll
  for (int m = 0; m < NV; ++m) {
    const float4* xp = reinterpret_cast<const float4*>(x + (size_t)(tid + m * ncons) * VEC);
#pragma unroll
    for (int v = 0; v < VEC / 4; ++v) {
      const float4 t = __ldcg(xp + v);
      xr[m * VEC + 4 * v + 0] = t.x;
      xr[m * VEC + 4 * v + 1] = t.y;
      xr[m * VEC + 4 * v + 2] = t.z;
      xr[m * VEC + 4 * v + 3] = t.w;
    }
  }
}

template <typename W, int NV>
__device__ __forceinline__ void store_y(float* out, const float* yacc, int tid, int ncons) {
  constexpr int VEC = Elem<W>::kVec;
#pragma unroll
  for (int m = 0; m < NV; ++m) {
    float4* op = reinterpret_cast<float4*>(out + (size_t)(tid + m * ncons) * VEC);
#pragma unroll
    for (int v = 0; v < VEC / 4; ++v)
      op[v] = make_float4(yacc[m * VEC + 4 * v], yacc[m * VEC + 4 * v + 1],
                          yacc[m * VEC + 4 * v + 2], yacc[m * VEC + 4 * v + 3]);
  }
}

// ---------------------------------------------------------------------------
// per-layer kernel
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
  Ring R;
  R.buf = smem;
  R.full = reinterpret_cast<uint64_t*>(smem + (size_t)a.stages * a.stage_bytes);
  R.empty = R.full + a.stages;
  R.rps = a.rps;
  R.stages = a.stages;
  R.stage_bytes = a.stage_bytes;
  R.row_bytes = a.row_bytes;
  __shared__ float red[kMaxConsWarps * 32];
  __shared__ float h_s[kBatch];
  __shared__ int s_slot[kMaxSlots];
  __shared__ float s_gate[kMaxSlots];
  __shared__ int s_nloc;

  const int ncons = blockDim.x - 32;
  const int ncw = ncons >> 5;
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = warp_uniform(tid >> 5);  // provably warp-uniform: no collective fallback

  if (tid == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&R.full[s], 1);
      mbar_init(&R.empty[s], ncw);
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
  Cursor cur;
  if (warp == ncw) {
    if (lane == 0 && g1 > g0)
      produce_rows<W>(R, cur, reinterpret_cast<const W*>(a.lw.experts), a.lw.expert_stride,
                      a.lw.mat_stride, s_slot, a.f, a.d, g0, g1, l2_evict_first_policy());
    return;
  }
  float xr[NV * VEC];
  load_x<W, NV>(a.x, xr, tid, ncons);
  float yacc[NV * VEC];
#pragma unroll
  for (int i = 0; i < NV * VEC; ++i) yacc[i] = 0.f;
  consume_rows<W, NV>(R, cur, xr, yacc, s_gate, a.f, g0, g1, red, h_s, tid, ncons, 1);
  store_y<W, NV>(a.ypart + (size_t)blockIdx.x * a.d, yacc, tid, ncons);
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
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = warp_uniform(tid >> 5);  // provably warp-uniform: no collective fallback
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
  if (warp == 0) warp_topk_softmax(logits, E, k, next_ids, next_gates);
  if (tid == 0) *counter = 0u;
}

// Expert-parallel variant: the reduced 32-column slice of this rank's delta
// is pushed to every rank's inbox, and the residual adds the rank-ordered sum
// of all ranks' slices (see launch_reduce_exchange in kernels.h).
__global__ void __launch_bounds__(256) reduce_exchange_kernel(
    const float* __restrict__ ypart, int nparts, const float* x, float* x_out, int d,
    const float* __restrict__ next_router, int E, int k, float* rpart, unsigned* counter,
    int32_t* next_ids, float* next_gates, PeerArgs pa) {
  __shared__ float red[8][33];
  __shared__ float xs[32];
  __shared__ float logits[kMaxExperts];
  __shared__ int s_last;
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = warp_uniform(tid >> 5);
  const int b = blockIdx.x;
  griddep_wait();
  const int i = b * 32 + lane;
  float s = 0.f;
  if (i < d)
    for (int p = warp; p < nparts; p += 8) s += ypart[(size_t)p * d + i];
  red[warp][lane] = s;
  __syncthreads();
  if (warp == 0) {
    float tot = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) tot += red[w][lane];
    const unsigned seq = __shfl_sync(MOE_FULL_MASK, lane == 0 ? pa.seq[b] + 1u : 0u, 0);
    const size_t par = seq & 1u;
    // push this rank's slice to every rank (P2P stores), then release flags
    if (i < d)
      for (int r = 0; r < pa.world; ++r) pa.inbox[r][(par * pa.world + pa.rank) * d + i] = tot;
    __threadfence_system();
    __syncwarp();
    if (lane < pa.world) st_release_sys(pa.flags[lane] + (size_t)pa.rank * kPeerSlots + b, seq);
    // wait for every rank's slice of this block (bounded: a missing peer is
    // reported through pa.err instead of hanging the GPU)
    if (lane < pa.world) peer_wait(pa.flags[pa.rank] + (size_t)lane * kPeerSlots + b, seq, pa.err);
    __syncwarp();
    float all = 0.f;
    if (i < d) {
      const float* in = pa.inbox[pa.rank] + par * pa.world * d + i;
      for (int r = 0; r < pa.world; ++r) all += __ldcv(in + (size_t)r * d);  // rank order
    }
    float xo = 0.f;
    if (i < d) {
      xo = (x ? x[i] : 0.f) + all;
      x_out[i] = xo;
    }
    xs[lane] = xo;
    if (lane == 0) pa.seq[b] = seq;
  }
  __syncthreads();
  griddep_launch_dependents();  // only after the peers arrived (see launch_reduce_exchange)
  if (next_router == nullptr) return;
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
    for (int bb = 0; bb < (int)gridDim.x; ++bb) l += __ldcg(&rpart[(size_t)bb * E + e]);
    logits[e] = l;
  }
  __syncthreads();
  if (warp == 0) warp_topk_softmax(logits, E, k, next_ids, next_gates);
  if (tid == 0) *counter = 0u;
}

// ---------------------------------------------------------------------------
// persistent whole-stack kernel
struct StackArgs {
  const void* const* layer_experts;  // [L] expert base per layer
  const int16_t* slot_of;            // [L][E]
  long long expert_stride, mat_stride;
  const float* router;               // [L][E][d]
  float* x;                          // in: x_0, out: x_L
  float* xbuf;                       // [2][d]
  float* ypart;                      // [G][d]
  float* rpart;                      // [G][E]
  int32_t* ids_out;                  // [L][k]
  float* gates_out;                  // [L][k]
  unsigned* gbar;                    // grid barrier counter (0 at launch)
  unsigned long long* trace;         // optional [L][G][16] clock64 stamps
  const float* const* rw;            // [L] R_{l+1} W2 per local expert [f][E] (nullptr: off)
  PeerArgs pa;                       // peer windows (peer != 0)
  int peer;
  int L, d, f, E, k;
  int row_bytes, rps, stages, stage_bytes;
};

__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned target, int ncons) {
  // bar.sync orders the CTA's prior writes before thread 0's release (the
  // release is cumulative); cross-CTA data is then read with ld.cg (L2).
  named_bar_sync(2, ncons);
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while ((int)(v - target) < 0);  // modulo 2^32: decode_stack2_kernel's counter never resets
  }
  named_bar_sync(2, ncons);
}

// Fixed-order sum of strided values with all loads in flight at once (one L2
// round trip instead of one per value).
constexpr int kSumUnroll = 24;
__device__ __forceinline__ float strided_sum(const float* base, int first, int count, int step,
                                             size_t stride) {
  float s = 0.f;
  for (int p0 = first; p0 < count; p0 += kSumUnroll * step) {
    float v[kSumUnroll];
#pragma unroll
    for (int i = 0; i < kSumUnroll; ++i) {
      const int p = p0 + i * step;
      v[i] = p < count ? __ldcg(base + (size_t)p * stride) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < kSumUnroll; ++i) s += v[i];
  }
  return s;
}

// Routing is linear in x, so the next layer's logits are assembled from
// per-CTA partials written BEFORE the first grid barrier:
//   logits_{l+1} = R_{l+1} x_{l+1} = R_{l+1} x_l + sum_c R_{l+1} ypart_c,
// CTA c contributing z_c = R_{l+1} (ypart_c [+ x_l if c == 0]).  Right after
// barrier 1 every CTA sums the G partials in a fixed order, picks the top-k
// and releases its producer warp — the residual reduction and the second
// barrier (needed only by the consumers, for x_{l+1}) overlap the ring fill.
template <typename W, int NV>
__global__ void __launch_bounds__(kMaxConsWarps * 32 + 32, 1)
    decode_stack_kernel(const __grid_constant__ StackArgs a) {
  constexpr int VEC = Elem<W>::kVec;
  extern __shared__ __align__(128) uint8_t smem[];
  Ring R;
  R.buf = smem;
  R.full = reinterpret_cast<uint64_t*>(smem + (size_t)a.stages * a.stage_bytes);
  R.empty = R.full + a.stages;
  R.rps = a.rps;
  R.stages = a.stages;
  R.stage_bytes = a.stage_bytes;
  R.row_bytes = a.row_bytes;
  __shared__ uint64_t route_bar;
  __shared__ float red[kMaxConsWarps * 32];
  __shared__ float h_s[kBatch];
  __shared__ float logits[kMaxExperts];
  __shared__ float zred[kMaxConsWarps * kMaxExperts];
  __shared__ int32_t s_ids[kMaxSlots];
  __shared__ float s_g[kMaxSlots];
  __shared__ int s_slot[kMaxSlots];
  __shared__ float s_gate[kMaxSlots];
  __shared__ int s_nloc;
  __shared__ int16_t s_so[kMaxExperts];  // slot map of the layer being routed

  const int ncons = blockDim.x - 32;
  const int ncw = ncons >> 5;
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = warp_uniform(tid >> 5);  // provably warp-uniform: no collective fallback
  const int G = gridDim.x, c = blockIdx.x;
  const int d = a.d, E = a.E, k = a.k;

  if (tid == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&R.full[s], 1);
      mbar_init(&R.empty[s], ncw);
    }
    mbar_init(&route_bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  griddep_wait();

  if (warp == ncw) {
    // ===== producer =====
    if (lane != 0) return;
    const uint64_t pol = l2_evict_first_policy();
    Cursor cur;
    for (int l = 0; l < a.L; ++l) {
      mbar_wait_sleep(&route_bar, (uint32_t)(l & 1));
      if (a.trace) a.trace[((size_t)l * G + c) * 16 + 6] = clock64();
      const long long T = (long long)s_nloc * a.f;
      const long long g0 = (long long)c * T / G, g1 = (long long)(c + 1) * T / G;
      if (g1 > g0)
        produce_rows<W>(R, cur, reinterpret_cast<const W*>(a.layer_experts[l]), a.expert_stride,
                        a.mat_stride, s_slot, a.f, d, g0, g1, pol);
      if (a.trace) a.trace[((size_t)l * G + c) * 16 + 7] = clock64();
    }
    return;
  }

  // ===== consumers =====
  // top-k of `logits` for layer l -> smem routing + release of the producer
  auto commit_route = [&](int l) {  // called by warp 0
    warp_topk_softmax(logits, E, k, s_ids, s_g);
    if (lane != 0) return;
    int n = 0;
    for (int j = 0; j < k; ++j) {
      const int slot = s_so[s_ids[j]];
      if (slot >= 0) {
        s_slot[n] = slot;
        s_gate[n] = s_g[j];
        ++n;
      }
      if (c == 0) {
        a.ids_out[(size_t)l * k + j] = s_ids[j];
        a.gates_out[(size_t)l * k + j] = s_g[j];
      }
    }
    s_nloc = n;
    mbar_arrive(&route_bar);
  };

  unsigned gen = 0;
  Cursor cur;
  const int cc0 = (int)((long long)c * d / G), cc1 = (int)((long long)(c + 1) * d / G);
  if (a.trace && tid == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (a.L > 1) a.trace[((size_t)1 * G + c) * 16 + 13] = smid;  // layer-1 row, slot 13
    a.trace[(size_t)c * 16 + 12] = clock64();
    a.trace[(size_t)c * 16 + 13] = globaltimer();
    a.trace[(size_t)c * 16 + 0] = clock64();
  }
  // multi-GPU: every rank runs this kernel; slot c's exchange counter and the
  // router-partial counter advance by one per layer on all ranks alike
  const bool peer = a.peer != 0;
  const unsigned seq0 = peer ? a.pa.seq[c] : 0u;
  const unsigned zseq0 = peer ? *a.pa.zseq : 0u;
  const int NR = peer ? a.pa.world : 1, rk = peer ? a.pa.rank : 0;
  // routing of layer 0: the router GEMV itself, redundantly in every CTA
  for (int e = tid; e < E; e += ncons) s_so[e] = a.slot_of[e];
  for (int e = warp; e < E; e += ncw) {
    const float* re = a.router + (size_t)e * d;
    float s = 0.f;
    for (int i = lane; i < d; i += 32) s = fmaf(re[i], __ldcg(&a.x[i]), s);
    s = warp_sum(s);
    if (lane == 0) logits[e] = s;
  }
  named_bar_sync(2, ncons);
  if (warp == 0) commit_route(0);
  named_bar_sync(2, ncons);

  // z bookkeeping (warp 0 registers): zreg = this CTA's sum_r h'_r rw[r][:],
  // xt = R_{l+1}[:, chunk] . x_l[chunk] (its share of the x_l term)
  const bool use_rw = a.rw != nullptr;
  float zreg[kZMax], xt[kZMax];
#pragma unroll
  for (int e = 0; e < kZMax; ++e) zreg[e] = xt[e] = 0.f;
  if (use_rw && warp == 0 && a.L > 1) {
    const float* r1 = a.router + (size_t)E * d;
    for (int base = cc0; base < cc1; base += 32) {
      const int col = base + lane;
      const float xv = col < cc1 ? __ldcg(&a.x[col]) : 0.f;
#pragma unroll
      for (int e = 0; e < kZMax; ++e)
        xt[e] += warp_sum((col < cc1 && e < E) ? r1[(size_t)e * d + col] * xv : 0.f);
    }
  }

  for (int l = 0; l < a.L; ++l) {
    const bool more = l + 1 < a.L;
    const float* xl = (l == 0) ? a.x : a.xbuf + (size_t)(l & 1) * d;
    float* xn = more ? a.xbuf + (size_t)((l + 1) & 1) * d : a.x;
    unsigned long long* tr = a.trace ? a.trace + ((size_t)l * G + c) * 16 : nullptr;
    if (more)
      for (int e = tid; e < E; e += ncons) s_so[e] = a.slot_of[(size_t)(l + 1) * E + e];

    // ---- B: stream this CTA's rows of layer l ----
    float xr[NV * VEC];
    load_x<W, NV>(xl, xr, tid, ncons);
    float yacc[NV * VEC];
#pragma unroll
    for (int i = 0; i < NV * VEC; ++i) yacc[i] = 0.f;
    const long long T = (long long)s_nloc * a.f;
    const long long g0 = (long long)c * T / G, g1 = (long long)(c + 1) * T / G;
    const float* rwl = (use_rw && more) ? a.rw[l] : nullptr;
    consume_rows<W, NV>(R, cur, xr, yacc, s_gate, a.f, g0, g1, red, h_s, tid, ncons, 1,
                        tr ? tr + 1 : nullptr, rwl, s_slot, E, zreg);
    if (tr && tid == 0) tr[2] = clock64();
    store_y<W, NV>(a.ypart + (size_t)c * d, yacc, tid, ncons);

    // ---- z_c: this CTA's partial of the next layer's router logits ----
    if (more && use_rw) {
      if (warp == 0) {
#pragma unroll
        for (int e = 0; e < kZMax; ++e) {
          if (lane == e && e < E) a.rpart[(size_t)e * G + c] = zreg[e] + (rk == 0 ? xt[e] : 0.f);
          zreg[e] = 0.f;
          xt[e] = 0.f;
        }
      }
    } else if (more) {  // fallback (E > kZMax): z_c = R_{l+1} (ypart_c [+ x_l])
      const float* rn = a.router + (size_t)(l + 1) * E * d;
      float v[NV * VEC];
#pragma unroll
      for (int i = 0; i < NV * VEC; ++i) v[i] = (c == 0 && rk == 0) ? yacc[i] + xr[i] : yacc[i];
      for (int e0 = 0; e0 < E; e0 += 8) {
        float part[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          part[q] = 0.f;
          if (e0 + q < E) {
            const float* re = rn + (size_t)(e0 + q) * d;
#pragma unroll
            for (int m = 0; m < NV; ++m) {
              const float4* rp = reinterpret_cast<const float4*>(re + (size_t)(tid + m * ncons) * VEC);
#pragma unroll
              for (int u = 0; u < VEC / 4; ++u) {
                const float4 rv = __ldg(rp + u);
                const float* vv = v + m * VEC + 4 * u;
                part[q] = fmaf(rv.x, vv[0], part[q]);
                part[q] = fmaf(rv.y, vv[1], part[q]);
                part[q] = fmaf(rv.z, vv[2], part[q]);
                part[q] = fmaf(rv.w, vv[3], part[q]);
              }
            }
          }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float t = warp_sum(part[q]);
          if (lane == 0 && e0 + q < E) zred[warp * kMaxExperts + e0 + q] = t;
        }
      }
      named_bar_sync(2, ncons);
      for (int e = tid; e < E; e += ncons) {
        float t = 0.f;
        for (int w = 0; w < ncw; ++w) t += zred[w * kMaxExperts + e];
        a.rpart[(size_t)e * G + c] = t;
      }
    }
    if (tr && tid == 0) tr[11] = clock64();
    grid_sync(a.gbar, (++gen) * (unsigned)G, ncons);
    if (tr && tid == 0) tr[3] = clock64();

    // ---- A(l+1): route the next layer and release the producer ----
    if (more) {
      for (int e = warp; e < E; e += ncw) {
        float s = strided_sum(a.rpart + (size_t)e * G, lane, G, 32, 1);
        s = warp_sum(s);
        if (lane == 0) logits[e] = s;
      }
      if (tr && tid == 0) tr[8] = clock64();
      named_bar_sync(2, ncons);
      if (peer) {
        // this rank's router partial -> every rank (CTA 0 pushes), then the
        // rank-ordered sum of all ranks' partials, identical everywhere
        const unsigned zs = zseq0 + (unsigned)l + 1u;
        const int zp = (int)(zs & 1u);
        if (c == 0) {
          for (int e = tid; e < E; e += ncons)
            for (int r = 0; r < NR; ++r)
              a.pa.zbox[r][((size_t)zp * NR + rk) * kMaxExperts + e] = logits[e];
          __threadfence_system();
          named_bar_sync(2, ncons);
          if (tid < NR) st_release_sys(a.pa.zflags[tid] + rk, zs);
        }
        if (tid < NR) peer_wait(a.pa.zflags[rk] + tid, zs, a.pa.err);
        named_bar_sync(2, ncons);
        for (int e = tid; e < E; e += ncons) {
          float t = 0.f;
          for (int r = 0; r < NR; ++r) t += __ldcv(a.pa.zbox[rk] + ((size_t)zp * NR + r) * kMaxExperts + e);
          logits[e] = t;
        }
        named_bar_sync(2, ncons);
      }
      if (tr && tid == 0) tr[9] = clock64();
      if (warp == 0) commit_route(l + 1);
      if (tr && tid == 0) tr[10] = clock64();
      // keep the other warps' phase-C loads out of the MIO queue while warp 0
      // routes (the top-k's shuffles would queue behind them)
      named_bar_sync(2, ncons);
    }

    // ---- C: this CTA's column chunk of x_{l+1} = x_l + sum_c ypart_c ----
    const bool next_xt = use_rw && l + 2 < a.L;
    const float* r2 = next_xt ? a.router + (size_t)(l + 2) * E * d : nullptr;
    if (peer) {
      // multi-GPU: the chunk of this rank's delta goes to every rank, then
      // x_{l+1} = x_l + sum over ranks (rank order) — bit-identical everywhere
      const unsigned sq = seq0 + (unsigned)l + 1u;
      const size_t par = sq & 1u;
      for (int base = cc0; base < cc1; base += 32) {
        const int col = base + lane;
        const bool valid = col < cc1;
        const float s = valid ? strided_sum(a.ypart + col, warp, G, ncw, (size_t)d) : 0.f;
        red[warp * 32 + lane] = s;
        named_bar_sync(2, ncons);
        if (warp == 0 && valid) {
          float tot = 0.f;
          for (int w = 0; w < ncw; ++w) tot += red[w * 32 + lane];
          for (int r = 0; r < NR; ++r) a.pa.inbox[r][(par * NR + rk) * d + col] = tot;
        }
        named_bar_sync(2, ncons);
      }
      __threadfence_system();
      named_bar_sync(2, ncons);
      if (tid < NR) {
        st_release_sys(a.pa.flags[tid] + (size_t)rk * kPeerSlots + c, sq);
        peer_wait(a.pa.flags[rk] + (size_t)tid * kPeerSlots + c, sq, a.pa.err);
      }
      named_bar_sync(2, ncons);
      if (warp == 0) {
        for (int base = cc0; base < cc1; base += 32) {
          const int col = base + lane;
          const bool valid = col < cc1;
          float xo = 0.f;
          if (valid) {
            float all = 0.f;
            const float* in = a.pa.inbox[rk] + par * NR * d + col;
            for (int r = 0; r < NR; ++r) all += __ldcv(in + (size_t)r * d);
            xo = __ldcg(&xl[col]) + all;
            xn[col] = xo;
          }
          if (next_xt) {
#pragma unroll
            for (int e = 0; e < kZMax; ++e) {
              const float rv = (valid && e < E) ? __ldg(r2 + (size_t)e * d + col) : 0.f;
              xt[e] += warp_sum(rv * xo);
            }
          }
        }
      }
      named_bar_sync(2, ncons);
    } else
    for (int base = cc0; base < cc1; base += 32) {
      const int col = base + lane;
      const bool valid = col < cc1;
      float rv[kZMax];
      if (next_xt && warp == 0) {  // issued before the partial sums: latency overlaps
#pragma unroll
        for (int e = 0; e < kZMax; ++e) rv[e] = (valid && e < E) ? __ldg(r2 + (size_t)e * d + col) : 0.f;
      }
      const float s = valid ? strided_sum(a.ypart + col, warp, G, ncw, (size_t)d) : 0.f;
      red[warp * 32 + lane] = s;
      named_bar_sync(2, ncons);
      if (warp == 0) {
        float xo = 0.f;
        if (valid) {
          float tot = 0.f;
          for (int w = 0; w < ncw; ++w) tot += red[w * 32 + lane];
          xo = __ldcg(&xl[col]) + tot;
          xn[col] = xo;
        }
        if (next_xt) {
#pragma unroll
          for (int e = 0; e < kZMax; ++e) xt[e] += warp_sum(rv[e] * xo);
        }
      }
      named_bar_sync(2, ncons);
    }
    if (tr && tid == 0) tr[4] = clock64();
    if (more) grid_sync(a.gbar, (++gen) * (unsigned)G, ncons);
    if (tr && tid == 0) {
      tr[5] = clock64();
      if (!more) {  // calibration pair at the end (row of layer 0)
        a.trace[(size_t)c * 16 + 14] = clock64();
        a.trace[(size_t)c * 16 + 15] = globaltimer();
      }
      if (more) a.trace[((size_t)(l + 1) * G + c) * 16 + 0] = tr[3];
    }
  }
  if (peer && tid == 0) {
    a.pa.seq[c] = seq0 + (unsigned)a.L;
    if (c == 0) *a.pa.zseq = zseq0 + (unsigned)(a.L - 1);
  }
}

// ---------------------------------------------------------------------------
// persistent whole-stack kernel with ONE grid barrier per layer
//
// decode_stack_kernel sums the per-CTA partials in a fixed float order, which
// needs a column-chunk reduction pass and a second grid barrier before any CTA
// holds x_{l+1} (~6 us of every ~115 us layer, tools/trace_stack.py).  Here
// every CTA adds its partial into an L2-resident accumulator with 64-bit
// integer atomics in fixed point (2^-32): integer addition is associative, so
// the sum — and x_{l+1}, and the routing — is bit-identical whatever order
// the contributions land in, and right after the one barrier every CTA reads
// the finished accumulator.  The next layer's router logits are assembled the
// same way: R_{l+1} x_l (split over CTAs and threads, one column per thread)
// plus the z partials of R_{l+1} W2 accumulated during the stream.
//
// Range: a partial |v| >= 2^22 (so the 148-CTA sum could leave the 2^31
// fixed-point range) is counted in an overflow word; that layer's x and
// logits then become NaN (loud, never a silently wrapped sum).
//
// Accumulators rotate over 3 buffers (layer l uses buf(l)); buf(l+2) is
// zeroed after layer l's barrier, which orders the zeroing before any use of
// that buffer (at layer l+2, after barrier l+1).  The barrier counter and the
// rotation carry across launches in `state`, so nothing is reset per launch.
constexpr float kFix = 4294967296.0f;               // 2^32
constexpr float kFixInv = 2.3283064365386963e-10f;  // 2^-32
constexpr float kFixMax = 4194304.0f;               // 2^22
constexpr int kZStride = 16;                        // zacc words per buffer: kZMax logits + overflow
constexpr int kStateBase = 32;                      // state[32] barrier base, state[33] rotation

struct Stack2Args {
  const void* const* layer_experts;
  const int16_t* slot_of;
  long long expert_stride, mat_stride;
  const float* router;               // [L][E][d]
  const float* const* rw;            // [L] R_{l+1} W2 per local expert [f][E]
  float* x;                          // in: x_0 (out: x_L when x_out == x)
  float* x_out;                      // out: x_L
  unsigned long long* acc;           // [3][d] fixed point
  unsigned long long* zacc;          // [3][kZStride]
  unsigned* state;                   // [0] barrier counter, [32] base, [33] rotation
  int32_t* ids_out;                  // [L][k]
  float* gates_out;                  // [L][k]
  float* logits_out;                 // optional [L][E]
  unsigned long long* trace;         // optional [L][G][16]
  int L, d, f, E, k;
  int row_bytes, rps, stages, stage_bytes;
};

__device__ __forceinline__ unsigned long long to_fix(float v) {
  return (unsigned long long)__float2ll_rn(v * kFix);
}
__device__ __forceinline__ float from_fix(unsigned long long a) {
  return __ll2float_rn((long long)a) * kFixInv;
}

template <typename W, int NV>
__global__ void __launch_bounds__(kMaxConsWarps * 32 + 32, 1)
    decode_stack2_kernel(const __grid_constant__ Stack2Args a) {
  constexpr int VEC = Elem<W>::kVec;
  constexpr int S = NV * VEC;
  extern __shared__ __align__(128) uint8_t smem[];
  Ring R;
  R.buf = smem;
  R.full = reinterpret_cast<uint64_t*>(smem + (size_t)a.stages * a.stage_bytes);
  R.empty = R.full + a.stages;
  R.rps = a.rps;
  R.stages = a.stages;
  R.stage_bytes = a.stage_bytes;
  R.row_bytes = a.row_bytes;
  float* stg = reinterpret_cast<float*>(smem + (size_t)a.stages * a.stage_bytes + 2 * a.stages * 8);
  __shared__ uint64_t route_bar;
  __shared__ float red[kMaxConsWarps * 32];
  __shared__ float h_s[kBatch];
  __shared__ float logits[kMaxExperts];
  __shared__ int32_t s_ids[kMaxSlots];
  __shared__ float s_g[kMaxSlots];
  __shared__ int s_slot[kMaxSlots];
  __shared__ float s_gate[kMaxSlots];
  __shared__ int s_nloc;
  __shared__ int16_t s_so[kMaxExperts];
  __shared__ unsigned s_state[2];

  const int ncons = blockDim.x - 32;
  const int ncw = ncons >> 5;
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = warp_uniform(tid >> 5);
  const int G = gridDim.x, c = blockIdx.x;
  const int d = a.d, E = a.E, k = a.k;

  if (tid == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&R.full[s], 1);
      mbar_init(&R.empty[s], ncw);
    }
    mbar_init(&route_bar, 1);
    fence_mbar_init();
  }
  griddep_wait();
  if (tid == 32) {
    s_state[0] = __ldcg(&a.state[kStateBase]);
    s_state[1] = __ldcg(&a.state[kStateBase + 1]);
  }
  __syncthreads();
  const unsigned bar0 = s_state[0], rot = s_state[1];

  if (warp == ncw) {
    if (lane != 0) return;
    const uint64_t pol = l2_evict_first_policy();
    Cursor cur;
    for (int l = 0; l < a.L; ++l) {
      mbar_wait_sleep(&route_bar, (uint32_t)(l & 1));
      if (a.trace) a.trace[((size_t)l * G + c) * 16 + 6] = clock64();
      const long long T = (long long)s_nloc * a.f;
      const long long g0 = (long long)c * T / G, g1 = (long long)(c + 1) * T / G;
      if (g1 > g0)
        produce_rows<W>(R, cur, reinterpret_cast<const W*>(a.layer_experts[l]), a.expert_stride,
                        a.mat_stride, s_slot, a.f, d, g0, g1, pol);
      if (a.trace) a.trace[((size_t)l * G + c) * 16 + 7] = clock64();
    }
    return;
  }

  auto commit_route = [&](int l) {
    if (c == 0 && a.logits_out != nullptr && lane < E) a.logits_out[(size_t)l * E + lane] = logits[lane];
    warp_topk_softmax(logits, E, k, s_ids, s_g);
    if (lane != 0) return;
    int n = 0;
    for (int j = 0; j < k; ++j) {
      const int slot = s_so[s_ids[j]];
      if (slot >= 0) {
        s_slot[n] = slot;
        s_gate[n] = s_g[j];
        ++n;
      }
      if (c == 0) {
        a.ids_out[(size_t)l * k + j] = s_ids[j];
        a.gates_out[(size_t)l * k + j] = s_g[j];
      }
    }
    s_nloc = n;
    mbar_arrive(&route_bar);
  };
  auto buf = [&](int l) { return (int)((rot + (unsigned)l) % 3u); };
  auto col_of = [&](int q) { return (tid + (q / VEC) * ncons) * VEC + (q % VEC); };
  unsigned long long* const ovf_words = a.zacc + kZMax;
  float rv[2];
  auto load_rv = [&](int lr) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int p = c + j * G;
      rv[j] = (lr < a.L && p < S * E) ? __ldg(a.router + ((size_t)lr * E + p / S) * d + col_of(p % S)) : 0.f;
    }
  };
  auto add_xpart = [&](int lr, int b, const float* xr) {
    if (lr >= a.L) return;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int p = c + j * G;
      if (p < S * E) {
        const int q = p % S;
        float xv = 0.f;
#pragma unroll
        for (int i = 0; i < S; ++i) xv = (i == q) ? xr[i] : xv;
        const float v = warp_sum(rv[j] * xv);
        if (lane == 0) {
          atomicAdd(&a.zacc[(size_t)b * kZStride + p / S], to_fix(v));
          if (!(fabsf(v) < kFixMax)) atomicAdd(&ovf_words[(size_t)b * kZStride], 1ull);
        }
      }
    }
  };

  for (int e = tid; e < E; e += ncons) s_so[e] = a.slot_of[e];
  for (int e = warp; e < E; e += ncw) {
    const float* re = a.router + (size_t)e * d;
    float s = 0.f;
    for (int i = lane; i < d; i += 32) s = fmaf(re[i], __ldcg(&a.x[i]), s);
    s = warp_sum(s);
    if (lane == 0) logits[e] = s;
  }
  named_bar_sync(2, ncons);
  if (warp == 0) commit_route(0);
  float xr[S];
  load_x<W, NV>(a.x, xr, tid, ncons);
  load_rv(1);
  add_xpart(1, buf(0), xr);
  load_rv(2);
  named_bar_sync(2, ncons);

  float zreg[kZMax];
#pragma unroll
  for (int e = 0; e < kZMax; ++e) zreg[e] = 0.f;
  Cursor cur;
  for (int l = 0; l < a.L; ++l) {
    const bool more = l + 1 < a.L;
    const int b = buf(l);
    unsigned long long* tr = a.trace ? a.trace + ((size_t)l * G + c) * 16 : nullptr;
    if (tr && tid == 0) tr[0] = clock64();
    if (more)
      for (int e = tid; e < E; e += ncons) s_so[e] = a.slot_of[(size_t)(l + 1) * E + e];
    float yacc[S];
#pragma unroll
    for (int i = 0; i < S; ++i) yacc[i] = 0.f;
    const long long T = (long long)s_nloc * a.f;
    const long long g0 = (long long)c * T / G, g1 = (long long)(c + 1) * T / G;
    consume_rows<W, NV>(R, cur, xr, yacc, s_gate, a.f, g0, g1, red, h_s, tid, ncons, 1,
                        tr ? tr + 1 : nullptr, more ? a.rw[l] : nullptr, s_slot, E, zreg);
    if (tr && tid == 0) tr[2] = clock64();
    store_y<W, NV>(stg, yacc, tid, ncons);
    named_bar_sync(2, ncons);
    bool ov = false;
    unsigned long long* accb = a.acc + (size_t)b * d;
    for (int i = tid; i < d; i += ncons) {
      const float v = stg[i];
      ov |= !(fabsf(v) < kFixMax);
      atomicAdd(&accb[i], to_fix(v));
    }
    if (more && warp == 0) {
      float zv = 0.f;
#pragma unroll
      for (int e = 0; e < kZMax; ++e) {
        zv = (lane == e) ? zreg[e] : zv;
        zreg[e] = 0.f;
      }
      if (lane < E) {
        atomicAdd(&a.zacc[(size_t)b * kZStride + lane], to_fix(zv));
        ov |= !(fabsf(zv) < kFixMax);
      }
    }
    if (__any_sync(MOE_FULL_MASK, ov) && lane == 0) atomicAdd(&ovf_words[(size_t)b * kZStride], 1ull);
    if (tr && tid == 0) tr[11] = clock64();
    grid_sync(a.state, bar0 + (unsigned)((l + 1) * G), ncons);
    if (tr && tid == 0) tr[3] = clock64();
    unsigned long long av[S];
#pragma unroll
    for (int m = 0; m < NV; ++m) {
      const ulonglong2* ap = reinterpret_cast<const ulonglong2*>(accb + (size_t)(tid + m * ncons) * VEC);
#pragma unroll
      for (int v = 0; v < VEC / 2; ++v) {
        const ulonglong2 t = __ldcg(ap + v);
        av[m * VEC + 2 * v] = t.x;
        av[m * VEC + 2 * v + 1] = t.y;
      }
    }
    const bool bad = __ldcg(&ovf_words[(size_t)b * kZStride]) != 0ull;
    if (more && warp == 0) {
      const unsigned long long zl = lane < E ? __ldcg(&a.zacc[(size_t)b * kZStride + lane]) : 0ull;
      if (lane < E) logits[lane] = bad ? 0.f : from_fix(zl);
      __syncwarp();
      commit_route(l + 1);
      if (tr && lane == 0) tr[10] = clock64();
    }
#pragma unroll
    for (int i = 0; i < S; ++i) xr[i] = bad ? __int_as_float(0x7fffffff) : xr[i] + from_fix(av[i]);
    if (tr && tid == 0) tr[4] = clock64();
    {
      const int b2 = buf(l + 2);
      const int c0 = (int)((long long)c * d / G), c1 = (int)((long long)(c + 1) * d / G);
      for (int i = c0 + tid; i < c1; i += ncons) a.acc[(size_t)b2 * d + i] = 0ull;
      if (c == 0 && tid < kZStride) a.zacc[(size_t)b2 * kZStride + tid] = 0ull;
    }
    if (l + 2 < a.L) {
      add_xpart(l + 2, buf(l + 1), xr);
      load_rv(l + 3);
    }
    if (!more && c == 0) store_y<W, NV>(a.x_out, xr, tid, ncons);
    named_bar_sync(2, ncons);  // routing of l+1 visible to every consumer warp
    if (tr && tid == 0) tr[5] = clock64();
  }
  if (c == 0 && tid == 0) {
    a.state[kStateBase] = bar0 + (unsigned)(a.L * G);
    a.state[kStateBase + 1] = (rot + (unsigned)a.L) % 3u;
  }
}

// ---------------------------------------------------------------------------
// persistent whole-stack kernel, routing off the critical path
//
// decode_stack2_kernel interleaves up and down rows batch by batch, so the
// next layer's logits are complete only when the slowest CTA has streamed its
// last W2T row; then the grid barrier, the top-k and the first TMA round trip
// of layer l+1 all sit on an idle HBM (~13 us of a ~109 us layer).
//
// Routing needs only h: logits_{l+1} = R_{l+1} x_l + sum_r h_r (R_{l+1} W2)[r]
// (the projection is precomputed per expert), so here every CTA streams ALL
// its W1/W3 rows first (2/3 of the bytes; h parked in smem), publishes its z
// partial, then streams its W2T rows.  The producer thread, after issuing the
// last W2T copy of layer l, waits on a grid counter for all z partials (long
// since in: the down phase is ~1/3 of the layer), picks layer l+1's top-k
// itself and keeps issuing — the ring holds layer l+1's first rows while the
// consumers reduce x_{l+1} across the barrier.  Same per-CTA row split, same
// per-row arithmetic and the same fixed-point sums as decode_stack2_kernel:
// outputs, ids and gates are bit-identical to it.
constexpr int kStateRoute = 64;      // state[64]: route counter (own 128 B line)
constexpr int kStateRouteBase = 34;  // state[34]: its value at launch

// Scalar restatement of warp_topk_softmax for E <= 32 (same rank predicate,
// same ascending-id sequential denominator): bit-identical gates.
__device__ __forceinline__ int thread_topk_softmax(const float* lg, int E, int k, int32_t* ids,
                                                   float* gates) {
  int n = 0;
  float mx = -INFINITY;
  for (int e = 0; e < E; ++e) {
    const float v = lg[e];
    int rank = 0;
    for (int e2 = 0; e2 < E; ++e2) {
      const float o = lg[e2];
      rank += (int)((o > v) | ((o == v) & (e2 < e)));
    }
    if (rank < k) {
      ids[n++] = e;
      mx = fmaxf(mx, v);
    }
  }
  float denom = 0.f;
  for (int j = 0; j < n; ++j) denom += expf(lg[ids[j]] - mx);
  for (int j = 0; j < n; ++j) gates[j] = expf(lg[ids[j]] - mx) / denom;
  return n;
}

// Producer, phase-split order: W1/W3 rows of every batch, then the W2T rows.
template <typename W>
__device__ __forceinline__ void produce_rows_split(const Ring& R, Cursor& cur, const W* wbase,
                                                   long long expert_stride, long long mat_stride,
                                                   const int* s_slot, int f, int d, long long g0,
                                                   long long g1, uint64_t pol,
                                                   unsigned long long* t_up,
                                                   unsigned long long* t_ring = nullptr) {
  const int total_vec = (int)(3 * (g1 - g0));
  int p = 0;
  const int ring_rows = R.stages * R.rps;
  auto put = [&](const W* src) {
    if (cur.slot == 0) {
      mbar_wait(&R.empty[cur.stage], cur.phase ^ 1);
      if (t_ring != nullptr && (p == 0 || p == ring_rows)) t_ring[p == 0 ? 0 : 1] = clock64();
      const int nvec = min(R.rps, total_vec - p);
      mbar_arrive_expect_tx(&R.full[cur.stage], (uint32_t)(nvec * R.row_bytes));
    }
    bulk_g2s(R.buf + (size_t)cur.stage * R.stage_bytes + (size_t)cur.slot * R.row_bytes, src,
             (uint32_t)R.row_bytes, &R.full[cur.stage], pol);
    ++p;
    if (++cur.slot == R.rps) cur.next_stage(R.stages);
  };
  for (long long g = g0; g < g1;) {
    const int jj = (int)(g / f);
    const int r = (int)(g - (long long)jj * f);
    const int nb = (int)min((long long)kBatch, min(g1 - g, (long long)(f - r)));
    const W* eb = wbase + (long long)s_slot[jj] * expert_stride + (long long)r * d;
    for (int q = 0; q < nb; ++q) put(eb + (long long)q * d);
    for (int q = 0; q < nb; ++q) put(eb + mat_stride + (long long)q * d);
    g += nb;
  }
  if (t_up) *t_up = clock64();
  for (long long g = g0; g < g1;) {
    const int jj = (int)(g / f);
    const int r = (int)(g - (long long)jj * f);
    const int nb = (int)min(g1 - g, (long long)(f - r));
    const W* eb = wbase + (long long)s_slot[jj] * expert_stride + 2 * mat_stride + (long long)r * d;
    for (int q = 0; q < nb; ++q) put(eb + (long long)q * d);
    g += nb;
  }
  if (cur.slot != 0) cur.next_stage(R.stages);
}

struct RowCount {
  int p, total;
};

// Consumers, up phase: h'_r = gate * silu(W1_r x) * (W3_r x) into hbuf, and
// warp 0's z accumulation — decode_stack2's arithmetic, batch for batch.
// red is double-buffered, so one CTA barrier per batch suffices.
template <typename W, int NV>
__device__ __forceinline__ void consume_up(const Ring& R, Cursor& cur, RowCount& rc, const float* xr,
                                           const float* s_gate, int f, long long g0, long long g1,
                                           float* red, float* hbuf, int tid, int ncons, int bar_id,
                                           unsigned long long* t_first, const float* rw,
                                           const int* s_slot, int E, float* zreg) {
  constexpr int VEC = Elem<W>::kVec;
  const int warp = warp_uniform(tid >> 5), lane = tid & 31, ncw = ncons >> 5;
  int bi = 0;
  for (long long g = g0; g < g1;) {
    const int jj = (int)(g / f);
    const int r = (int)(g - (long long)jj * f);
    const int nb = (int)min((long long)kBatch, min(g1 - g, (long long)(f - r)));
    float rwv[kZMax];
    if (rw != nullptr && warp == 0) {
      const float* rp = rw + ((size_t)s_slot[jj] * f + r + lane) * E;
#pragma unroll
      for (int e = 0; e < kZMax; ++e) rwv[e] = (lane < nb && e < E) ? __ldg(rp + e) : 0.f;
    }
    float acc[2 * kBatch];
#pragma unroll
    for (int q = 0; q < 2 * kBatch; ++q) {
      acc[q] = 0.f;
      if ((q & (kBatch - 1)) < nb) {
        if (cur.slot == 0) mbar_wait(&R.full[cur.stage], cur.phase);
        if (t_first != nullptr && rc.p == 0 && tid == 0) *t_first = clock64();
        const uint8_t* row = R.buf + (size_t)cur.stage * R.stage_bytes + (size_t)cur.slot * R.row_bytes;
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
        ++rc.p;
        if (++cur.slot == R.rps || rc.p == rc.total) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&R.empty[cur.stage]);
          cur.next_stage(R.stages);
        }
      }
    }
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
    float* rb = red + (bi & 1) * (kMaxConsWarps * 32);
    rb[warp * 32 + lane] = acc[0];
    named_bar_sync(bar_id, ncons);
    if (warp == 0) {
      float tot = 0.f;
      for (int w = 0; w < ncw; ++w) tot += rb[w * 32 + lane];
      const float b = __shfl_down_sync(MOE_FULL_MASK, tot, kBatch);
      const float hq = lane < nb ? s_gate[jj] * (silu_f(tot) * b) : 0.f;
      if (lane < nb) hbuf[g - g0 + lane] = hq;
      if (rw != nullptr) {
#pragma unroll
        for (int e = 0; e < kZMax; ++e) zreg[e] += warp_sum(hq * rwv[e]);
      }
    }
    ++bi;
    g += nb;
  }
}

// Consumers, down phase: y += h'_r * W2T_r over the CTA's rows in order.
template <typename W, int NV>
__device__ __forceinline__ void consume_down(const Ring& R, Cursor& cur, RowCount& rc, float* yacc,
                                             const float* hbuf, int n, int tid, int ncons) {
  constexpr int VEC = Elem<W>::kVec;
  const int lane = tid & 31;
#pragma unroll 4
  for (int i = 0; i < n; ++i) {
    if (cur.slot == 0) mbar_wait(&R.full[cur.stage], cur.phase);
    const uint8_t* row = R.buf + (size_t)cur.stage * R.stage_bytes + (size_t)cur.slot * R.row_bytes;
    const float hq = hbuf[i];
#pragma unroll
    for (int m = 0; m < NV; ++m) {
      const uint4 v = lds128(row + (size_t)(tid + m * ncons) * 16);
      float w[VEC];
      Elem<W>::unpack(v, w);
#pragma unroll
      for (int j = 0; j < VEC; ++j) yacc[m * VEC + j] = fmaf(hq, w[j], yacc[m * VEC + j]);
    }
    ++rc.p;
    if (++cur.slot == R.rps || rc.p == rc.total) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&R.empty[cur.stage]);
      cur.next_stage(R.stages);
    }
  }
}

template <typename W, int NV>
__global__ void __launch_bounds__(kMaxConsWarps * 32 + 64, 1)
    decode_stack3_kernel(const __grid_constant__ Stack2Args a) {
  constexpr int VEC = Elem<W>::kVec;
  constexpr int S = NV * VEC;
  extern __shared__ __align__(128) uint8_t smem[];
  Ring R;
  R.buf = smem;
  R.full = reinterpret_cast<uint64_t*>(smem + (size_t)a.stages * a.stage_bytes);
  R.empty = R.full + a.stages;
  R.rps = a.rps;
  R.stages = a.stages;
  R.stage_bytes = a.stage_bytes;
  R.row_bytes = a.row_bytes;
  float* stg = reinterpret_cast<float*>(smem + (size_t)a.stages * a.stage_bytes + 2 * a.stages * 8);
  float* hbuf = stg + a.d;
  __shared__ uint64_t route_bar;
  __shared__ float red[2 * kMaxConsWarps * 32];
  __shared__ float logits[kMaxExperts];
  __shared__ int32_t s_ids[kMaxSlots];
  __shared__ float s_g[kMaxSlots];
  __shared__ int s_slot[2][kMaxSlots];
  __shared__ float s_gate[2][kMaxSlots];
  __shared__ int s_nloc[2];
  __shared__ unsigned s_state[3];

  const int ncons = blockDim.x - 64;  // + producer warp + router warp
  const int ncw = ncons >> 5;
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = warp_uniform(tid >> 5);
  const int G = gridDim.x, c = blockIdx.x;
  const int d = a.d, E = a.E, k = a.k;
  unsigned long long* const trace = a.trace;
  auto tslot = [&](int l, int i) { return trace + ((size_t)l * G + c) * 16 + i; };

  if (tid == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&R.full[s], 1);
      mbar_init(&R.empty[s], ncw);
    }
    mbar_init(&route_bar, 1);
    fence_mbar_init();
  }
  griddep_wait();
  if (tid == 32) {
    s_state[0] = __ldcg(&a.state[kStateBase]);
    s_state[1] = __ldcg(&a.state[kStateBase + 1]);
    s_state[2] = __ldcg(&a.state[kStateRouteBase]);
  }
  __syncthreads();
  const unsigned bar0 = s_state[0], rot = s_state[1], rbase = s_state[2];
  auto buf = [&](int l) { return (int)((rot + (unsigned)l) % 3u); };
  unsigned long long* const ovf_words = a.zacc + kZMax;

  if (warp == ncw) {  // producer: one elected lane issues every bulk copy
    if (lane != 0) return;
    if (trace) {
      *tslot(0, 12) = clock64();
      *tslot(0, 13) = globaltimer();
    }
    const uint64_t pol = l2_evict_first_policy();
    Cursor cur;
    for (int l = 0; l < a.L; ++l) {
      mbar_wait_sleep(&route_bar, (uint32_t)(l & 1));  // layer l's routing (ready long before, l >= 1)
      if (trace) *tslot(l, 10) = clock64();
      const int set = l & 1;
      const long long T = (long long)s_nloc[set] * a.f;
      const long long g0 = (long long)c * T / G, g1 = (long long)(c + 1) * T / G;
      if (g1 > g0)
        produce_rows_split<W>(R, cur, reinterpret_cast<const W*>(a.layer_experts[l]), a.expert_stride,
                              a.mat_stride, s_slot[set], a.f, d, g0, g1, pol,
                              trace ? tslot(l, 8) : nullptr,
                              (trace && l > 0) ? tslot(l, 12) : nullptr);
      if (trace) *tslot(l, 9) = clock64();
    }
    if (trace) {
      *tslot(0, 14) = clock64();
      *tslot(0, 15) = globaltimer();
    }
    return;
  }
  if (warp == ncw + 1) {  // router: layer l+1's top-k as soon as every z partial is in
    for (int l = 0; l + 1 < a.L; ++l) {
      const int so = lane < E ? __ldg(a.slot_of + (size_t)(l + 1) * E + lane) : -1;
      if (lane == 0) {
        const unsigned target = rbase + (unsigned)((l + 1) * G);
        unsigned v;
        for (;;) {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.state + kStateRoute) : "memory");
          if ((int)(v - target) >= 0) break;
          __nanosleep(128);
        }
      }
      __syncwarp();
      const unsigned long long* zb = a.zacc + (size_t)buf(l) * kZStride;
      const bool bad = __ldcg(&ovf_words[(size_t)buf(l) * kZStride]) != 0ull;
      if (lane < E) logits[lane] = bad ? 0.f : from_fix(__ldcg(zb + lane));
      __syncwarp();
      if (c == 0 && a.logits_out != nullptr && lane < E) a.logits_out[(size_t)(l + 1) * E + lane] = logits[lane];
      warp_topk_softmax(logits, E, k, s_ids, s_g);
      // slot of each selected expert: lane j of the warp holds slot_of[j]
      const int nset = (l + 1) & 1;
      int nl = 0;
      for (int j = 0; j < k; ++j) {
        const int slot = __shfl_sync(MOE_FULL_MASK, so, s_ids[j] & 31);
        if (slot >= 0) {
          if (lane == 0) {
            s_slot[nset][nl] = slot;
            s_gate[nset][nl] = s_g[j];
          }
          ++nl;
        }
      }
      if (c == 0 && lane < k) {
        a.ids_out[(size_t)(l + 1) * k + lane] = s_ids[lane];
        a.gates_out[(size_t)(l + 1) * k + lane] = s_g[lane];
      }
      if (lane == 0) {
        s_nloc[nset] = nl;
        mbar_arrive(&route_bar);  // producer and consumers of layer l+1
        if (trace) *tslot(l, 11) = clock64();
      }
      __syncwarp();
    }
    return;
  }

  auto col_of = [&](int q) { return (tid + (q / VEC) * ncons) * VEC + (q % VEC); };
  float rv[2];
  auto load_rv = [&](int lr) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int p = c + j * G;
      rv[j] = (lr < a.L && p < S * E) ? __ldg(a.router + ((size_t)lr * E + p / S) * d + col_of(p % S)) : 0.f;
    }
  };
  auto add_xpart = [&](int lr, int b, const float* xr) {
    if (lr >= a.L) return;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int p = c + j * G;
      if (p < S * E) {
        const int q = p % S;
        float xv = 0.f;
#pragma unroll
        for (int i = 0; i < S; ++i) xv = (i == q) ? xr[i] : xv;
        const float v = warp_sum(rv[j] * xv);
        if (lane == 0) {
          atomicAdd(&a.zacc[(size_t)b * kZStride + p / S], to_fix(v));
          if (!(fabsf(v) < kFixMax)) atomicAdd(&ovf_words[(size_t)b * kZStride], 1ull);
        }
      }
    }
  };

  // layer 0's routing from x_0 (consumer warps; same arithmetic as stack2)
  for (int e = warp; e < E; e += ncw) {
    const float* re = a.router + (size_t)e * d;
    float s = 0.f;
    for (int i = lane; i < d; i += 32) s = fmaf(re[i], __ldcg(&a.x[i]), s);
    s = warp_sum(s);
    if (lane == 0) logits[e] = s;
  }
  named_bar_sync(2, ncons);
  if (warp == 0) {
    if (c == 0 && a.logits_out != nullptr && lane < E) a.logits_out[lane] = logits[lane];
    warp_topk_softmax(logits, E, k, s_ids, s_g);
    if (lane == 0) {
      int n = 0;
      for (int j = 0; j < k; ++j) {
        const int slot = a.slot_of[s_ids[j]];
        if (slot >= 0) {
          s_slot[0][n] = slot;
          s_gate[0][n] = s_g[j];
          ++n;
        }
        if (c == 0) {
          a.ids_out[j] = s_ids[j];
          a.gates_out[j] = s_g[j];
        }
      }
      s_nloc[0] = n;
      mbar_arrive(&route_bar);
    }
  }
  float xr[S];
  load_x<W, NV>(a.x, xr, tid, ncons);
  load_rv(1);
  add_xpart(1, buf(0), xr);
  load_rv(2);
  named_bar_sync(2, ncons);

  float zreg[kZMax];
#pragma unroll
  for (int e = 0; e < kZMax; ++e) zreg[e] = 0.f;
  Cursor cur;
  for (int l = 0; l < a.L; ++l) {
    const bool more = l + 1 < a.L;
    const int b = buf(l), set = l & 1;
    const bool tr0 = trace != nullptr && tid == 0;
    if (tr0) *tslot(l, 0) = clock64();
    if (l > 0) mbar_wait(&route_bar, (uint32_t)(l & 1));
    const long long T = (long long)s_nloc[set] * a.f;
    const long long g0 = (long long)c * T / G, g1 = (long long)(c + 1) * T / G;
    RowCount rc{0, (int)(3 * (g1 - g0))};
    consume_up<W, NV>(R, cur, rc, xr, s_gate[set], a.f, g0, g1, red, hbuf, tid, ncons, 1,
                      tr0 ? tslot(l, 1) : nullptr, more ? a.rw[l] : nullptr, s_slot[set], E, zreg);
    named_bar_sync(2, ncons);  // hbuf complete; every warp's R x share (add_xpart) issued
    if (tr0) *tslot(l, 2) = clock64();
    if (more && warp == 0) {
      float zv = 0.f;
#pragma unroll
      for (int e = 0; e < kZMax; ++e) {
        zv = (lane == e) ? zreg[e] : zv;
        zreg[e] = 0.f;
      }
      if (lane < E) {
        atomicAdd(&a.zacc[(size_t)b * kZStride + lane], to_fix(zv));
        if (!(fabsf(zv) < kFixMax)) atomicAdd(&ovf_words[(size_t)b * kZStride], 1ull);
      }
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.state + kStateRoute) : "memory");
        if (trace) *tslot(l, 3) = clock64();
      }
    }
    float yacc[S];
#pragma unroll
    for (int i = 0; i < S; ++i) yacc[i] = 0.f;
    consume_down<W, NV>(R, cur, rc, yacc, hbuf, (int)(g1 - g0), tid, ncons);
    if (tr0) *tslot(l, 4) = clock64();
    store_y<W, NV>(stg, yacc, tid, ncons);
    named_bar_sync(2, ncons);
    bool ov = false;
    unsigned long long* accb = a.acc + (size_t)b * d;
    for (int i = tid; i < d; i += ncons) {
      const float v = stg[i];
      ov |= !(fabsf(v) < kFixMax);
      atomicAdd(&accb[i], to_fix(v));
    }
    if (__any_sync(MOE_FULL_MASK, ov) && lane == 0) atomicAdd(&ovf_words[(size_t)b * kZStride], 1ull);
    if (tr0) *tslot(l, 5) = clock64();
    grid_sync(a.state, bar0 + (unsigned)((l + 1) * G), ncons);
    if (tr0) *tslot(l, 6) = clock64();
    unsigned long long av[S];
#pragma unroll
    for (int m = 0; m < NV; ++m) {
      const ulonglong2* ap = reinterpret_cast<const ulonglong2*>(accb + (size_t)(tid + m * ncons) * VEC);
#pragma unroll
      for (int v = 0; v < VEC / 2; ++v) {
        const ulonglong2 t = __ldcg(ap + v);
        av[m * VEC + 2 * v] = t.x;
        av[m * VEC + 2 * v + 1] = t.y;
      }
    }
    const bool bad = __ldcg(&ovf_words[(size_t)b * kZStride]) != 0ull;
#pragma unroll
    for (int i = 0; i < S; ++i) xr[i] = bad ? __int_as_float(0x7fffffff) : xr[i] + from_fix(av[i]);
    {
      const int b2 = buf(l + 2);
      const int c0 = (int)((long long)c * d / G), c1 = (int)((long long)(c + 1) * d / G);
      for (int i = c0 + tid; i < c1; i += ncons) a.acc[(size_t)b2 * d + i] = 0ull;
      if (c == 0 && tid < kZStride) a.zacc[(size_t)b2 * kZStride + tid] = 0ull;
    }
    if (l + 2 < a.L) {
      add_xpart(l + 2, buf(l + 1), xr);
      load_rv(l + 3);
    }
    if (!more && c == 0) store_y<W, NV>(a.x_out, xr, tid, ncons);
    if (tr0) *tslot(l, 7) = clock64();
  }
  if (c == 0 && tid == 0) {
    a.state[kStateBase] = bar0 + (unsigned)(a.L * G);
    a.state[kStateBase + 1] = (rot + (unsigned)a.L) % 3u;
    a.state[kStateRouteBase] = rbase + (unsigned)((a.L - 1) * G);
  }
}

// ---------------------------------------------------------------------------
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
  p.smem = p.stages * stage + 2 * p.stages * 8;
  p.grid = sm_count;
  // testing hook: fewer CTAs, so that several linked ranks' persistent kernels
  // fit one GPU side by side (tests/test_gpu_ep_peers.py)
  if (debug_options().stack_grid > 0) p.grid = std::min(sm_count, debug_options().stack_grid);
  p.ok = true;
  return p;
}

static void fill_ring_args(const DecodePlan& p, const Dims& dm, int& row_bytes, int& rps,
                           int& stages, int& stage_bytes) {
  row_bytes = dm.d * (dm.dtype == MOE_DTYPE_BF16 ? 2 : 4);
  rps = p.rps;
  stages = p.stages;
  stage_bytes = p.rps * row_bytes;
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

template <typename W, int NV>
static cudaError_t launch_stack_t(const DecodePlan& p, const StackArgs& a, cudaStream_t s) {
  auto kern = decode_stack_kernel<W, NV>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.grid);
  cfg.blockDim = dim3(p.ncons + 32);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = debug_options().noncoop ? 0 : 1;  // diagnostics
  return cudaLaunchKernelEx(&cfg, kern, a);
}

#define MOE_DISPATCH_NV(FN, W, ...)        \
  switch (p.nv) {                         \
    case 1: return FN<W, 1>(__VA_ARGS__); \
    case 2: return FN<W, 2>(__VA_ARGS__); \
    case 3: return FN<W, 3>(__VA_ARGS__); \
    case 4: return FN<W, 4>(__VA_ARGS__); \
  }                                       \
  return cudaErrorInvalidValue;

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
  fill_ring_args(p, dm, a.row_bytes, a.rps, a.stages, a.stage_bytes);
  if (dm.dtype == MOE_DTYPE_BF16) {
    MOE_DISPATCH_NV(launch_decode_t, __nv_bfloat16, p, a, s, pdl)
  }
  MOE_DISPATCH_NV(launch_decode_t, float, p, a, s, pdl)
}

cudaError_t launch_decode_stack(const DecodePlan& p, const StackDesc& sd, const Dims& dm,
                                float* x, float* xbuf, float* ypart, float* rpart,
                                int32_t* ids_out, float* gates_out, unsigned* gbar,
                                cudaStream_t s, const PeerArgs* pa) {
  StackArgs a;
  a.peer = pa != nullptr && pa->world > 1;
  if (pa) a.pa = *pa;
  a.layer_experts = sd.layer_experts;
  a.slot_of = sd.slot_of;
  a.expert_stride = sd.expert_stride;
  a.mat_stride = sd.mat_stride;
  a.router = sd.router;
  a.x = x;
  a.xbuf = xbuf;
  a.ypart = ypart;
  a.rpart = rpart;
  a.ids_out = ids_out;
  a.gates_out = gates_out;
  a.gbar = gbar;
  a.trace = sd.trace;
  a.rw = sd.rw;
  a.L = sd.L;
  a.d = dm.d;
  a.f = dm.f;
  a.E = dm.E;
  a.k = dm.k;
  fill_ring_args(p, dm, a.row_bytes, a.rps, a.stages, a.stage_bytes);
  cudaError_t e = cudaMemsetAsync(gbar, 0, 256, s);  // arrival counter + release line
  if (e != cudaSuccess) return e;
  if (dm.dtype == MOE_DTYPE_BF16) {
    MOE_DISPATCH_NV(launch_stack_t, __nv_bfloat16, p, a, s)
  }
  MOE_DISPATCH_NV(launch_stack_t, float, p, a, s)
}

int stack2_smem(const DecodePlan& p, const Dims& dm) { return p.smem + dm.d * 4; }

bool stack2_supported(const DecodePlan& p, const Dims& dm) {
  if (!p.ok || dm.E > kZMax) return false;
  const int vec = dm.dtype == MOE_DTYPE_BF16 ? 8 : 4;
  return p.nv * vec * dm.E <= 2 * p.grid && stack2_smem(p, dm) <= 227 * 1024;
}

size_t stack2_acc_bytes(const Dims& dm) { return 3 * (size_t)dm.d * 8 + 3 * kZStride * 8 + 512; }

// decode_stack3_kernel: the ring, the partial-y staging and h for the CTA's
// rows (at most ceil(k*f/G)).
static int stack3_hcap(const DecodePlan& p, const Dims& dm) {
  return (int)(((long long)dm.k * dm.f + p.grid - 1) / p.grid) + 1;
}
int stack3_smem(const DecodePlan& p, const Dims& dm) { return stack2_smem(p, dm) + 4 * stack3_hcap(p, dm); }
bool stack3_supported(const DecodePlan& p, const Dims& dm) {
  return stack2_supported(p, dm) && dm.E <= 32 && stack3_smem(p, dm) <= 227 * 1024;
}

template <typename W, int NV>
static cudaError_t launch_stack2_t(const DecodePlan& p, const Dims& dm, const Stack2Args& a,
                                   cudaStream_t s) {
  const bool v3 = debug_options().stack_kernel == 3 && stack3_supported(p, dm);
  auto kern = v3 ? decode_stack3_kernel<W, NV> : decode_stack2_kernel<W, NV>;
  const int smem = v3 ? stack3_smem(p, dm) : stack2_smem(p, dm);
  const int threads = p.ncons + (v3 ? 64 : 32);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = debug_options().noncoop ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

cudaError_t launch_decode_stack2(const DecodePlan& p, const StackDesc& sd, const Dims& dm, float* x,
                                 void* accbuf, int32_t* ids_out, float* gates_out,
                                 float* logits_out, cudaStream_t s, float* x_out) {
  // (the projections are read only for a next layer)
  if (!stack2_supported(p, dm) || (sd.rw == nullptr && sd.L > 1)) return cudaErrorInvalidValue;
  Stack2Args a;
  a.layer_experts = sd.layer_experts;
  a.slot_of = sd.slot_of;
  a.expert_stride = sd.expert_stride;
  a.mat_stride = sd.mat_stride;
  a.router = sd.router;
  a.rw = sd.rw;
  a.x = x;
  a.x_out = x_out ? x_out : x;
  a.acc = static_cast<unsigned long long*>(accbuf);
  a.zacc = a.acc + 3 * (size_t)dm.d;
  a.state = reinterpret_cast<unsigned*>(a.zacc + 3 * kZStride);
  a.ids_out = ids_out;
  a.gates_out = gates_out;
  a.logits_out = logits_out;
  a.trace = sd.trace;
  a.L = sd.L;
  a.d = dm.d;
  a.f = dm.f;
  a.E = dm.E;
  a.k = dm.k;
  fill_ring_args(p, dm, a.row_bytes, a.rps, a.stages, a.stage_bytes);
  if (dm.dtype == MOE_DTYPE_BF16) {
    MOE_DISPATCH_NV(launch_stack2_t, __nv_bfloat16, p, dm, a, s)
  }
  MOE_DISPATCH_NV(launch_stack2_t, float, p, dm, a, s)
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

// Pacing of the multi-token exchanges (peer_allreduce_kernel,
// ep_combine_kernel): their data copies alternate by parity, so a rank may
// write call c's copy only once every rank has finished reading call c-2's.
// The all-reduce alone keeps the ranks within one call of each other, but
// in the streamed combine a rank that holds none of a call's tokens' experts
// and is home to none of them (n_tok < world) is waited on by nobody, so
// without this a peer could run two calls ahead and overwrite the gather
// copy it is still reading.  Each kernel starts by waiting for every rank's
// mt_done >= seq - 2 (in its own window) and its last block to finish
// stores mt_done = seq into every rank's window.
__device__ __forceinline__ void mt_pace_wait(const PeerArgs& pa, unsigned seq) {
  if (threadIdx.x < (unsigned)pa.world) peer_wait(pa.mt_done[pa.rank] + threadIdx.x, seq - 2u, pa.err);
  __syncthreads();
}
__device__ __forceinline__ void mt_pace_done(const PeerArgs& pa, unsigned seq) {
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(pa.mt_seq, 1u) + 1u) % (unsigned)gridDim.x == 0u;
  __syncthreads();
  if (s_last && threadIdx.x < (unsigned)pa.world) {
    __threadfence_system();
    st_release_sys(pa.mt_done[threadIdx.x] + pa.rank, seq);
  }
}

static size_t mt_bytes(int world, int max_hidden, int max_tokens) {
  if (max_tokens <= 0) return 0;
  const size_t cap = (size_t)max_tokens * max_hidden;
  return 2 * (size_t)world * cap * 4 + 2 * cap * 4 + (size_t)(world + 2) * kMtBlocks * 4 +
         (size_t)(world + 1) * max_tokens * 4;
}

size_t peer_window_bytes(int world, int max_hidden, int max_tokens) {
  return 2 * (size_t)world * max_hidden * 4 + (size_t)world * kPeerSlots * 4 +
         2 * (size_t)world * kMaxExperts * 4 + 64 + kPeerSlots * 4 + 64 +
         mt_bytes(world, max_hidden, max_tokens);
}

PeerParts peer_window_parts(void* base, int world, int max_hidden, int max_tokens) {
  PeerParts q;
  char* p = static_cast<char*>(base);
  q.inbox = reinterpret_cast<float*>(p);
  p += 2 * (size_t)world * max_hidden * 4;
  q.flags = reinterpret_cast<unsigned*>(p);
  p += (size_t)world * kPeerSlots * 4;
  q.zbox = reinterpret_cast<float*>(p);
  p += 2 * (size_t)world * kMaxExperts * 4;
  q.zflags = reinterpret_cast<unsigned*>(p);
  p += 64;
  q.seq = reinterpret_cast<unsigned*>(p);
  p += kPeerSlots * 4;
  q.zseq = reinterpret_cast<unsigned*>(p);
  q.err = q.zseq + 1;
  p += 64;
  q.mt_recv = q.mt_gath = nullptr;
  q.mt_pflag = q.mt_gflag = q.mt_seq = nullptr;
  q.mt_cflag = q.mt_tflag = nullptr;
  if (max_tokens > 0) {
    const size_t cap = (size_t)max_tokens * max_hidden;
    q.mt_recv = reinterpret_cast<float*>(p);
    p += 2 * (size_t)world * cap * 4;
    q.mt_gath = reinterpret_cast<float*>(p);
    p += 2 * cap * 4;
    q.mt_pflag = reinterpret_cast<unsigned*>(p);
    p += (size_t)world * kMtBlocks * 4;
    q.mt_gflag = reinterpret_cast<unsigned*>(p);
    p += kMtBlocks * 4;
    q.mt_seq = reinterpret_cast<unsigned*>(p);
    p += kMtBlocks * 4;
    q.mt_cflag = reinterpret_cast<unsigned*>(p);
    p += (size_t)world * max_tokens * 4;
    q.mt_tflag = reinterpret_cast<unsigned*>(p);
  }
  return q;
}

// Multi-token peer allreduce.  Block b owns elements [b*n/B, (b+1)*n/B).
//  1 every rank pushes its delta chunk into the owner's recv[par][rank],
//    fence.sys, releases pflag[rank][b] on the owner;
//  2 the owner (rank b % world) waits for all ranks' pflag, sums recv in rank
//    order, pushes the sum into every rank's gath[par], releases gflag[b];
//  3 every rank waits for its gflag[b] and writes x_out = x + gath.
// Parity = the call's sequence number & 1 (the context's multi-token
// exchange counter, shared with ep_combine_kernel so that the two kinds of
// call alternate the same two data copies); mt_pace_wait / mt_pace_done keep
// every rank from writing call c's copy before all ranks finished call c-2.
__global__ void __launch_bounds__(256) peer_allreduce_kernel(const float* __restrict__ delta,
                                                             const float* x, float* x_out,
                                                             long long n, PeerArgs pa, unsigned seq) {
  const int b = blockIdx.x, B = gridDim.x, tid = threadIdx.x;
  const int W = pa.world, rk = pa.rank, owner = b % W;
  const long long e0 = n * b / B, e1 = n * (b + 1) / B;
  const long long cap = pa.mt_cap;
  const long long par = seq & 1u;
  mt_pace_wait(pa, seq);
  // 1: scatter this rank's chunk to its owner
  float* dst = pa.mt_recv[owner] + (par * W + rk) * cap;
  for (long long i = e0 + tid; i < e1; i += blockDim.x) dst[i] = delta[i];
  __threadfence_system();
  __syncthreads();
  if (tid == 0) st_release_sys(pa.mt_pflag[owner] + (size_t)rk * kMtBlocks + b, seq);
  // 2: the owner reduces in rank order and gathers to everyone
  if (rk == owner) {
    if (tid < W) peer_wait(pa.mt_pflag[rk] + (size_t)tid * kMtBlocks + b, seq, pa.err);
    __syncthreads();
    const float* in = pa.mt_recv[rk] + par * W * cap;
    for (long long i = e0 + tid; i < e1; i += blockDim.x) {
      float sum = 0.f;
      for (int r = 0; r < W; ++r) sum += __ldcv(in + (size_t)r * cap + i);
      for (int r = 0; r < W; ++r) pa.mt_gath[r][par * cap + i] = sum;
    }
    __threadfence_system();
    __syncthreads();
    if (tid < W) st_release_sys(pa.mt_gflag[tid] + b, seq);
  }
  // 3: residual
  if (tid == 0) peer_wait(pa.mt_gflag[rk] + b, seq, pa.err);
  __syncthreads();
  const float* g = pa.mt_gath[rk] + par * cap;
  for (long long i = e0 + tid; i < e1; i += blockDim.x) x_out[i] = x[i] + __ldcv(g + i);
  mt_pace_done(pa, seq);
}

// Expert-parallel prefill combine, streamed beside the grouped kernel (fused
// prefill under EP with peer windows).  Every rank routes all n tokens and
// runs only its experts; token t's final row is reduced by its home rank
// t % W.  Per call (sequence number seq, data parity seq & 1):
//  1 the local completion queue (tokens whose local partials have all
//    landed) is drained: the token's local delta (its local slots ascending,
//    K splits ascending) goes straight into the home's receive box
//    recv[par][this rank][t / W] and the home's contribution flag is released;
//  2 home tokens are claimed; each waits for the ranks that own one of its
//    experts (known from the replicated routing), sums their deltas in rank
//    order, adds x and pushes the row into every rank's gather area + flag;
//  3 every rank copies the gathered rows into x_out.
// The same adds as delta -> peer_allreduce (which adds the other ranks'
// exact zeros), so ranks agree bit for bit with each other and with the
// unfused EP path.  Waits are bounded (pa.err).  Completion of this grid
// implies the grouped kernel's (griddep_wait at the end).
__global__ void __launch_bounds__(256) ep_combine_kernel(
    const float* x, const float* y, int d, int k, float* x_out, int n_tok, long long sstride,
    const int32_t* ids, const int32_t* split_of, const int16_t* slot_of, const uint32_t* holders,
    int* queue, PeerArgs pa, unsigned seq) {
  __shared__ int s_t, s_nq, s_i;
  __shared__ unsigned s_mask;
  const int tid = threadIdx.x;
  const int W = pa.world, rk = pa.rank;
  const long long cap = pa.mt_cap;
  const int mt = pa.mt_tokens;
  const unsigned par = seq & 1u;
  const int n4 = d / 4;
  mt_pace_wait(pa, seq);
  // the local queue's length: tokens with at least one expert on this rank
  if (tid == 0) s_nq = 0;
  __syncthreads();
  {
    int c = 0;
    for (int t = tid; t < n_tok; t += blockDim.x) {
      bool loc = false;
      for (int j = 0; j < k; ++j) loc |= slot_of[__ldg(ids + (size_t)t * k + j)] >= 0;
      c += loc;
    }
    atomicAdd(&s_nq, c);
  }
  __syncthreads();
  const int nq = s_nq;
  // 1: local deltas -> home ranks
  int slot = tid == 0 ? atomicAdd(queue, 1) : 0;
  while (true) {
    if (tid == 0) {
      int t = -1;
      if (slot < nq) {
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
    const int home = t % W, hi = t / W;
    float4* dst = reinterpret_cast<float4*>(pa.mt_recv[home] + ((size_t)par * W + rk) * cap + (size_t)hi * d);
    for (int c4 = tid; c4 < n4; c4 += blockDim.x) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int j = 0; j < k; ++j) {
        const size_t p = (size_t)t * k + j;
        const int e = __ldcg(ids + p);
        if (slot_of[e] < 0) continue;
        const int ns = __ldcg(split_of + e);
        for (int sp = 0; sp < ns; ++sp) {
          const float4 v = __ldcg(reinterpret_cast<const float4*>(y + sp * sstride + p * d) + c4);
          acc.x += v.x;
          acc.y += v.y;
          acc.z += v.z;
          acc.w += v.w;
        }
      }
      dst[c4] = acc;
    }
    __threadfence_system();
    __syncthreads();
    if (tid == 0) st_release_sys(pa.mt_cflag[home] + (size_t)rk * mt + hi, seq);
  }
  // 2: this rank's home tokens t = rk + W i
  while (true) {
    if (tid == 0) {
      const int i = atomicAdd(queue + 2, 1);
      const int t = rk + W * i;
      // contributing ranks: the holders of the token's experts (every rank
      // under tensor parallelism, holders == nullptr)
      unsigned m = holders ? 0u : (1u << W) - 1u;
      if (t < n_tok && holders)
        for (int j = 0; j < k; ++j) m |= __ldg(holders + __ldg(ids + (size_t)t * k + j));
      s_i = t < n_tok ? i : -1;
      s_mask = m;
    }
    __syncthreads();
    const int i = s_i;
    const unsigned m = s_mask;
    if (i < 0) break;
    if (tid < W && ((m >> tid) & 1u)) peer_wait(pa.mt_cflag[rk] + (size_t)tid * mt + i, seq, pa.err);
    __syncthreads();
    const int t = rk + W * i;
    const float* in = pa.mt_recv[rk] + (size_t)par * W * cap + (size_t)i * d;
    for (int c4 = tid; c4 < n4; c4 += blockDim.x) {
      float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int r = 0; r < W; ++r) {
        if (!((m >> r) & 1u)) continue;
        const float4 v = __ldcv(reinterpret_cast<const float4*>(in + (size_t)r * cap) + c4);
        sum.x += v.x;
        sum.y += v.y;
        sum.z += v.z;
        sum.w += v.w;
      }
      const float4 xv = __ldg(reinterpret_cast<const float4*>(x + (size_t)t * d) + c4);
      const float4 o = make_float4(xv.x + sum.x, xv.y + sum.y, xv.z + sum.z, xv.w + sum.w);
      for (int r = 0; r < W; ++r)
        reinterpret_cast<float4*>(pa.mt_gath[r] + (size_t)par * cap + (size_t)t * d)[c4] = o;
    }
    __threadfence_system();
    __syncthreads();
    if (tid < W) st_release_sys(pa.mt_tflag[tid] + t, seq);
    __syncthreads();
  }
  // 3: every token's row into x_out
  while (true) {
    if (tid == 0) {
      const int t = atomicAdd(queue + 3, 1);
      if (t < n_tok) peer_wait(pa.mt_tflag[rk] + t, seq, pa.err);
      s_t = t < n_tok ? t : -1;
    }
    __syncthreads();
    const int t = s_t;
    __syncthreads();
    if (t < 0) break;
    const float4* g = reinterpret_cast<const float4*>(pa.mt_gath[rk] + (size_t)par * cap + (size_t)t * d);
    for (int c4 = tid; c4 < n4; c4 += blockDim.x)
      reinterpret_cast<float4*>(x_out + (size_t)t * d)[c4] = __ldcv(g + c4);
  }
  mt_pace_done(pa, seq);
  griddep_wait();
}

cudaError_t launch_ep_combine(const float* x, const float* y, int n_tok, const Dims& dm, float* x_out,
                              const int32_t* ids, const int32_t* split_of, const int16_t* slot_of,
                              const uint32_t* holders, int* queue, const PeerArgs& pa, unsigned seq,
                              cudaStream_t s, bool pdl) {
  if (n_tok <= 0) return cudaSuccess;
  if (dm.d % 4 || n_tok > pa.mt_tokens || (long long)n_tok * dm.d > pa.mt_cap) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kMtBlocks);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  const long long sstride = (long long)n_tok * dm.k * dm.d;
  return cudaLaunchKernelEx(&cfg, ep_combine_kernel, x, y, dm.d, dm.k, x_out, n_tok, sstride, ids, split_of,
                            slot_of, holders, queue, pa, seq);
}

cudaError_t launch_peer_allreduce(const float* delta, const float* x, float* x_out, long long n,
                                  const PeerArgs& pa, unsigned seq, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  peer_allreduce_kernel<<<kMtBlocks, 256, 0, s>>>(delta, x, x_out, n, pa, seq);
  return cudaGetLastError();
}

cudaError_t launch_reduce_exchange(const float* ypart, int nparts, const float* x, float* x_out,
                                   const Dims& dm, const float* next_router, float* rpart,
                                   unsigned* counter, int32_t* next_ids, float* next_gates,
                                   const PeerArgs& pa, cudaStream_t s, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(reduce_blocks(dm));
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, reduce_exchange_kernel, ypart, nparts, x, x_out, dm.d,
                            next_router, dm.E, dm.k, rpart, counter, next_ids, next_gates, pa);
}

}  // namespace moe
