// common.cuh — shared device helpers for the sm_100a MoE kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define MOE_FULL_MASK 0xffffffffu

namespace moe {

// ---- element conversion ----------------------------------------------------
template <typename W>
struct Elem;
template <>
struct Elem<__nv_bfloat16> {
  static constexpr int kVec = 8;  // elements per 16-byte vector
  __device__ __forceinline__ static void unpack(const uint4& v, float* f) {
    const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 t = __bfloat1622float2(p[i]);
      f[2 * i] = t.x;
      f[2 * i + 1] = t.y;
    }
  }
  __device__ __forceinline__ static float to_float(__nv_bfloat16 v) { return __bfloat162float(v); }
  __device__ __forceinline__ static __nv_bfloat16 from_double(double v) { return __double2bfloat16(v); }
  __device__ __forceinline__ static __nv_bfloat16 from_float(float v) { return __float2bfloat16_rn(v); }
};
template <>
struct Elem<float> {
  static constexpr int kVec = 4;
  __device__ __forceinline__ static void unpack(const uint4& v, float* f) {
    f[0] = __uint_as_float(v.x);
    f[1] = __uint_as_float(v.y);
    f[2] = __uint_as_float(v.z);
    f[3] = __uint_as_float(v.w);
  }
  __device__ __forceinline__ static float to_float(float v) { return v; }
  __device__ __forceinline__ static float from_double(double v) { return (float)v; }
  __device__ __forceinline__ static float from_float(float v) { return v; }
};

__device__ __forceinline__ float silu_f(float a) { return a / (1.0f + expf(-a)); }

// Broadcast from lane 0: the compiler then treats the value (and branches on
// it) as warp-uniform, so shuffles under `if (warp == ...)` need no
// WARPSYNC.COLLECTIVE emulation.
__device__ __forceinline__ int warp_uniform(int v) { return __shfl_sync(MOE_FULL_MASK, v, 0); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) v += __shfl_xor_sync(MOE_FULL_MASK, v, s);
  return v;
}

// ---- programmatic dependent launch -----------------------------------------
// Every kernel waits for its predecessor before touching global memory; only
// smem / mbarrier setup runs before the wait (overlapping the previous tail).
__device__ __forceinline__ void griddep_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// ---- shared-memory mbarrier + bulk copy (TMA 1-D) --------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// For long waits (a producer idling across a layer boundary): the thread is
// suspended in try_wait (suspend-time hint) instead of re-polling, so its
// SYNCS/MIO traffic does not slow the other warps' shuffles and loads.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
        : "memory");
  }
}
// L2 policy for weights that are streamed exactly once.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// cp.async.bulk global -> shared (UBLKCP), completes tx bytes on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src, uint32_t bytes,
                                        uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst_smem)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint4 lds128(const void* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem_u32(p)));
  return v;
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---- system-scope flags between peer GPUs (NVLink P2P / CUDA IPC windows) --
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Bounded wait for a peer's flag to reach `target` (sequence numbers compare
// modulo 2^32): a rank that never arrives sets *err instead of hanging.
// Bounded wait for a peer's flag.  Once any wait of this rank has timed out
// (err set) the others give up at their next check instead of each spinning
// to its own bound, so a missing peer costs one timeout, not one per wait.
__device__ __forceinline__ void peer_wait(const unsigned* f, unsigned target, unsigned* err) {
  unsigned spins = 0;
  while ((int)(ld_acquire_sys(f) - target) < 0) {
    if (++spins > (1u << 22)) {
      atomicExch(err, 1u);
      break;
    }
    if (spins > 64) {
      if ((spins & 63) == 0 && *reinterpret_cast<volatile unsigned*>(err)) break;
      __nanosleep(128);
    }
  }
}

// ---- warp-wide top-k (registers only; no local-memory arrays) --------------
// Same semantics as topk_softmax below / gate_topk (model.cpp:79-99): k
// rounds of a warp argmax with (logit desc, id asc) ordering, ids emitted
// ascending, softmax over the selected logits with the denominator summed
// sequentially in ascending-id order.  Called by all 32 lanes of one warp;
// logits in shared/global memory, E <= 256, any k <= E (k <= 32 when E <=
// 32).  Slot j is written by lane j % 32.
__device__ __forceinline__ void warp_topk_softmax(const float* logits, int E, int k,
                                                  int32_t* ids, float* gates) {
  const int lane = threadIdx.x & 31;
  if (E <= 32) {
    // all-pairs rank: rank(e) = #{e' : l[e'] > l[e] or (l[e'] == l[e] and e' < e)};
    // the E shuffles are independent (no dependent argmax chain).
    // Fixed-trip, fully unrolled loops: the shuffles sit in provably
    // convergent code (no collective fallback) and issue back to back.
    const float v = lane < E ? logits[lane] : 0.f;
    // branch-free predicate arithmetic: the 32 shuffles issue back to back
    // (a short-circuit condition here compiled to 32 BSSY/BRA/BSYNC diamonds,
    // ~1.5 us on the decode layer boundary)
    int rank = 0;
#pragma unroll
    for (int e2 = 0; e2 < 32; ++e2) {
      const float o = __shfl_sync(MOE_FULL_MASK, v, e2);
      rank += (int)((e2 < E) & ((o > v) | ((o == v) & (e2 < lane))));
    }
    const bool sel = (lane < E) & (rank < k);
    const unsigned m = __ballot_sync(MOE_FULL_MASK, sel);
    const int pos = __popc(m & ((1u << lane) - 1u));  // ascending-id slot
    float mx = sel ? v : -INFINITY;
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) mx = fmaxf(mx, __shfl_xor_sync(MOE_FULL_MASK, mx, s));
    const float w = sel ? expf(v - mx) : 0.f;
    // ascending-id sequential sum over the selected lanes only: the other
    // lanes would add exact zeros, so this equals the full 0..31 sum bit for
    // bit (m is warp-uniform: k iterations, convergent)
    float denom = 0.f;
    for (unsigned mm = m; mm; mm &= mm - 1u) denom += __shfl_sync(MOE_FULL_MASK, w, __ffs(mm) - 1);
    if (sel) {
      ids[pos] = lane;
      gates[pos] = w / denom;
    }
    __syncwarp();
    return;
  }
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int e = lane + 32 * i;
    v[i] = e < E ? logits[e] : 0.f;
  }
  unsigned taken = 0u;  // bit i: expert lane+32i selected
  for (int j = 0; j < k; ++j) {
    float bv = 0.f;
    int be = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = lane + 32 * i;
      if (e < E && !(taken & (1u << i)) && (be == 0x7fffffff || v[i] > bv)) {
        bv = v[i];
        be = e;
      }
    }
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
      const float ov = __shfl_xor_sync(MOE_FULL_MASK, bv, s);
      const int oe = __shfl_xor_sync(MOE_FULL_MASK, be, s);
      const bool better = (oe != 0x7fffffff) &&
                          (be == 0x7fffffff || ov > bv || (ov == bv && oe < be));
      if (better) {
        bv = ov;
        be = oe;
      }
    }
    if ((be & 31) == lane) taken |= 1u << (be >> 5);
  }
  // emit ids ascending: block i of 32 experts in lane order
  int base = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const unsigned m = __ballot_sync(MOE_FULL_MASK, (taken >> i) & 1u);
    if ((taken >> i) & 1u) {
      const int pos = base + __popc(m & ((1u << lane) - 1u));
      ids[pos] = lane + 32 * i;
    }
    base += __popc(m);
  }
  __syncwarp();
  // any k <= E: slots j = lane, lane+32, ... (k > 32 is legal in the
  // reference, model.cpp:77); the denominator is the same ascending-id
  // sequential sum in every lane
  float mx = -INFINITY;
  for (int j = lane; j < k; j += 32) mx = fmaxf(mx, logits[ids[j]]);
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) mx = fmaxf(mx, __shfl_xor_sync(MOE_FULL_MASK, mx, s));
  float denom = 0.f;
  for (int j = 0; j < k; ++j) denom += expf(logits[ids[j]] - mx);
  for (int j = lane; j < k; j += 32) gates[j] = expf(logits[ids[j]] - mx) / denom;
  __syncwarp();
}

}  // namespace moe
