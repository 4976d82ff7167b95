// prefill.cu — multi-token (prefill) MoE layer on the 5th-gen tensor cores.
//
// The reference runs every token through expert_ffn one at a time
// (model.cpp:125-147); token-major and layer-major orders are identical
// because tokens never interact, so a prefill layer becomes a
// grouped GEMM over the experts' token sets:
//
//   permute (generic.cu)  ->  gather x rows by expert (bf16)
//   up   : H_e  = silu(X_e W1_e^T) * (X_e W3_e^T)        [tokens_e x ffn]
//   down : Y_e  = g * (H_e W2_e^T)                      [tokens_e x hidden]
//   combine (generic.cu): x += sum_j Y[t, j]  in ascending-id order
//
// The default (fused) layer is three launches: the router also counts each
// 4-token block's pairs per expert; the persistent grouped kernel derives
// the stable permutation from those counts and its epilogue warps scatter
// the bf16 rows themselves (dynamically claimed blocks) while the producer
// streams the first weights; each down epilogue counts the partials it
// landed per (token, 256 columns), and a token whose last partial lands is
// queued for the combine kernel running alongside (combine_ready_kernel, or
// ep_combine_kernel under expert / tensor parallelism).
//
// Both GEMMs are "swap-AB": the WEIGHT tile is the UMMA A operand (M = 128
// weight rows) and the expert's tokens are the N dimension (<= 256), so every
// weight byte is streamed from HBM exactly once per token chunk — at 512
// tokens (~128 per expert) the layer is HBM-bound.
//
// Per CTA: warp 4 issues TMA (cp.async.bulk.tensor, SWIZZLE_128B) into a
// 3/4-stage smem ring, warp 5 issues tcgen05.mma (kind::f16, bf16 in, fp32
// accumulate in TMEM) from one elected lane and commits to mbarriers, warps
// 0-3 drain TMEM with tcgen05.ld and run the fused epilogue
// (silu*mul -> bf16 H, or gate-scale -> fp32 Y).  W1/W3 tiles are K-major;
// the W2 tile is read from the decode layout W2T [ffn x hidden] as an
// MN-major operand (a_major = 1), so one weight copy serves both paths.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../include/moe_b200.h"
#include "common.cuh"
#include "kernels.h"
#include "replica_plan.h"

namespace moe {

constexpr int PF_BM = 128;    // UMMA M: weight rows per tile
constexpr int PF_BK = 64;     // K per stage: one 128-byte swizzle row of bf16
constexpr int PF_MAXN = 256;  // tokens per CTA (UMMA N <= 256)
constexpr int PF_BOXN = 64;   // token rows per TMA box
constexpr int PF_THREADS = 192;

// ---- tcgen05 / TMA PTX wrappers ------------------------------------------------
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// Same with an L2 cache-policy hint: the expert weights are streamed once per
// token chunk, so they are loaded evict_first and do not push the reused
// tensors (X and H tiles, the fp32 Y partials read back by the combine) out
// of the 126 MB L2.
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, int c0, int c1,
                                                 uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
// smem matrix descriptor (tcgen05 "version 1"), SWIZZLE_128B
__device__ __forceinline__ uint64_t umma_desc(const void* smem, uint32_t lbo_bytes,
                                              uint32_t sbo_bytes) {
  const uint64_t addr = smem_u32(smem);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;  // version
  d |= 2ull << 61;  // SWIZZLE_128B
  return d;
}
// instruction descriptor, kind::f16: bf16 x bf16 -> f32, M = 128
__device__ __forceinline__ uint32_t umma_idesc(int n, bool a_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn_major ? 1u : 0u) << 15) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(PF_BM >> 4) << 24);
}
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_free(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
// 32 lanes x 32 bit, 16 consecutive columns -> 16 registers per thread
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 lanes x 32 bit, 32 consecutive columns; call tmem_ld_wait() before use
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// TMEM double buffering for the grouped kernel: 2 buffers x 256 columns.  A
// tile takes one buffer (down; up with N <= 128 as D1|D3) or both (up with
// N > 128: D1 in one, D3 in the other).  The MMA warp and the epilogue warps
// replay the same assignment from the same tile sequence.
struct TmemSched {
  uint32_t next = 0, uses0 = 0, uses1 = 0;
  __device__ __forceinline__ int take(bool wide, int* b, uint32_t* par) {
    b[0] = next;
    b[1] = next ^ 1;
    const int n = wide ? 2 : 1;
    for (int i = 0; i < n; ++i) {
      uint32_t& u = b[i] ? uses1 : uses0;
      par[i] = u & 1;
      ++u;
    }
    if (!wide) next ^= 1;
    return n;
  }
};

struct PrefillArgs {
  const int32_t* counts;   // [E] tokens per expert
  const int32_t* offsets;  // [E] first sorted row of each expert
  const int32_t* perm;     // [n*k] sorted row -> pair p = t*k + j
  const float* gates;      // [n*k]
  const int16_t* slot_of;  // [E] local slot or -1 (this layer)
  __nv_bfloat16* h;        // [n*k, f] sorted rows (up output, down input)
  float* y;                // [n*k, d] by pair index (down output)
  int d, f, k;
};

// Shared-memory plan (1024-B aligned tiles for SWIZZLE_128B).
template <int STAGES, int A_TILES>
struct PfSmem {
  static constexpr int kA = PF_BM * PF_BK * 2;        // 16 KB per weight tile
  static constexpr int kB = PF_MAXN * PF_BK * 2;      // 32 KB token tile
  static constexpr int kStage = A_TILES * kA + kB;
  static constexpr int kBytes = STAGES * kStage + 1024 /*align*/ + 256 /*barriers*/;
};

// ===== up: H = silu(X W1^T) * (X W3^T) =======================================
// grid (f/128, token chunks, E).  TMEM: D1 cols [0,256), D3 cols [256,512).
template <int STAGES>
__global__ void __launch_bounds__(PF_THREADS, 1)
    prefill_up_kernel(const __grid_constant__ CUtensorMap wmap,  // layer [3*E_loc*f, d], box 64x128
                      const __grid_constant__ CUtensorMap xmap,  // Xg [n*k, d], box 64x64
                      PrefillArgs a) {
  using SM = PfSmem<STAGES, 2>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * SM::kStage);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_base_s = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int e = blockIdx.z;
  const int warp = warp_uniform(threadIdx.x >> 5), lane = threadIdx.x & 31;
  griddep_wait();
  const int count = a.counts[e];
  const int row0 = blockIdx.y * PF_MAXN;
  const int slot = a.slot_of[e];
  if (row0 >= count || slot < 0) return;
  const int nvalid = min(PF_MAXN, count - row0);
  const int N = (nvalid + 15) & ~15;
  const int nboxes = (N + PF_BOXN - 1) / PF_BOXN;
  const int srow = a.offsets[e] + row0;            // first sorted token row
  const int f0 = blockIdx.x * PF_BM;
  const int w1row = (slot * 3 + 0) * a.f + f0;
  const int w3row = (slot * 3 + 1) * a.f + f0;
  const int nkb = a.d / PF_BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_mbar_init();
  }
  if (warp == 5) tmem_alloc(tmem_base_s, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_base_s;

  if (warp == 4 && lane == 0) {
    // ---- TMA producer ----
    tma_prefetch_desc(&wmap);
    tma_prefetch_desc(&xmap);
    const uint32_t bytes = 2 * SM::kA + nboxes * PF_BOXN * PF_BK * 2;
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&empty[s], ((kb / STAGES) & 1) ^ 1);
      uint8_t* st = smem + s * SM::kStage;
      mbar_arrive_expect_tx(&full[s], bytes);
      tma_load_2d(st, &wmap, kb * PF_BK, w1row, &full[s]);
      tma_load_2d(st + SM::kA, &wmap, kb * PF_BK, w3row, &full[s]);
      for (int b = 0; b < nboxes; ++b)
        tma_load_2d(st + 2 * SM::kA + b * PF_BOXN * PF_BK * 2, &xmap, kb * PF_BK,
                    srow + b * PF_BOXN, &full[s]);
    }
  } else if (warp == 5 && lane == 0) {
    // ---- MMA issuer ----
    const uint32_t idesc = umma_idesc(N, false);
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&full[s], (kb / STAGES) & 1);
      tc_fence_after();
      const uint8_t* st = smem + s * SM::kStage;
#pragma unroll
      for (int kk = 0; kk < PF_BK / 16; ++kk) {
        const uint64_t a1 = umma_desc(st + kk * 32, 16, 1024);
        const uint64_t a3 = umma_desc(st + SM::kA + kk * 32, 16, 1024);
        const uint64_t b = umma_desc(st + 2 * SM::kA + kk * 32, 16, 1024);
        const uint32_t acc = (kb | kk) != 0;
        umma_f16(tmem, a1, b, idesc, acc);
        umma_f16(tmem + 256, a3, b, idesc, acc);
      }
      umma_commit(&empty[s]);
    }
    umma_commit(tmem_full);
  } else if (warp < 4) {
    // ---- epilogue: TMEM -> silu(D1)*D3 -> bf16 H[sorted row][f0 + lane row] ----
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    const int frow = f0 + warp * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
    for (int c0 = 0; c0 < N; c0 += 16) {
      float d1[16], d3[16];
      tmem_ld16(lane_base + c0, d1);
      tmem_ld16(lane_base + 256 + c0, d3);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int j = c0 + i;
        if (j < nvalid)
          a.h[(size_t)(srow + j) * a.f + frow] = __float2bfloat16_rn(silu_f(d1[i]) * d3[i]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) tmem_free(tmem, 512);
}

// ===== down: Y[pair] = g * (H W2^T), W2 read MN-major from W2T ================
// grid (d/128, token chunks, E).  TMEM: D cols [0,256).
template <int STAGES>
__global__ void __launch_bounds__(PF_THREADS, 1)
    prefill_down_kernel(const __grid_constant__ CUtensorMap w2map,  // layer [3*E_loc*f, d], box 64x64
                        const __grid_constant__ CUtensorMap hmap,   // H [n*k, f], box 64x64
                        PrefillArgs a) {
  using SM = PfSmem<STAGES, 1>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * SM::kStage);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_base_s = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int e = blockIdx.z;
  const int warp = warp_uniform(threadIdx.x >> 5), lane = threadIdx.x & 31;
  griddep_wait();
  const int count = a.counts[e];
  const int row0 = blockIdx.y * PF_MAXN;
  const int slot = a.slot_of[e];
  if (row0 >= count || slot < 0) return;
  const int nvalid = min(PF_MAXN, count - row0);
  const int N = (nvalid + 15) & ~15;
  const int nboxes = (N + PF_BOXN - 1) / PF_BOXN;
  const int srow = a.offsets[e] + row0;
  const int d0 = blockIdx.x * PF_BM;
  const int w2row = (slot * 3 + 2) * a.f;  // W2T rows = ffn index
  const int nkb = a.f / PF_BK;
  constexpr int kHalf = PF_BK * 64 * 2;  // one 64(d) x 64(f) box = 8 KB

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_mbar_init();
  }
  if (warp == 5) tmem_alloc(tmem_base_s, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_base_s;

  if (warp == 4 && lane == 0) {
    tma_prefetch_desc(&w2map);
    tma_prefetch_desc(&hmap);
    const uint32_t bytes = SM::kA + nboxes * PF_BOXN * PF_BK * 2;
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&empty[s], ((kb / STAGES) & 1) ^ 1);
      uint8_t* st = smem + s * SM::kStage;
      mbar_arrive_expect_tx(&full[s], bytes);
      // A: W2T rows [kb*64, +64) x cols [d0, d0+128) as two 64-col boxes (MN-major)
      tma_load_2d(st, &w2map, d0, w2row + kb * PF_BK, &full[s]);
      tma_load_2d(st + kHalf, &w2map, d0 + 64, w2row + kb * PF_BK, &full[s]);
      for (int b = 0; b < nboxes; ++b)
        tma_load_2d(st + SM::kA + b * PF_BOXN * PF_BK * 2, &hmap, kb * PF_BK, srow + b * PF_BOXN,
                    &full[s]);
    }
  } else if (warp == 5 && lane == 0) {
    const uint32_t idesc = umma_idesc(N, true);
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&full[s], (kb / STAGES) & 1);
      tc_fence_after();
      const uint8_t* st = smem + s * SM::kStage;
#pragma unroll
      for (int kk = 0; kk < PF_BK / 16; ++kk) {
        // MN-major A: 16 K-rows = 2 groups of 8 rows (SBO = 1024 B); the two
        // 64-wide M groups are the two boxes (LBO = 8 KB)
        const uint64_t adesc = umma_desc(st + kk * 2048, kHalf, 1024);
        const uint64_t bdesc = umma_desc(st + SM::kA + kk * 32, 16, 1024);
        umma_f16(tmem, adesc, bdesc, idesc, (kb | kk) != 0);
      }
      umma_commit(&empty[s]);
    }
    umma_commit(tmem_full);
  } else if (warp < 4) {
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    const int drow = d0 + warp * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
    for (int c0 = 0; c0 < N; c0 += 16) {
      float v[16];
      tmem_ld16(lane_base + c0, v);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int j = c0 + i;
        if (j < nvalid) {
          const int p = a.perm[srow + j];
          a.y[(size_t)p * a.d + drow] = a.gates[p] * v[i];
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) tmem_free(tmem, 256);
}

// ===== persistent grouped kernel: up AND down tiles of all experts =========
// One CTA per SM pulls tiles from a global atomic counter (dynamic balance,
// no wave quantisation).  Tile order: every up tile (expert-major, then token
// chunk, then ffn tile), then every down tile (expert, chunk, hidden tile,
// K split).  A down tile of (e, chunk) waits until all ffn tiles of that
// (e, chunk) have published H (per-(e,chunk) counter, release/acquire +
// fence.proxy.async before its TMA reads).  Up tiles never wait, so the
// schedule cannot deadlock.  The producer warp runs ahead into the next tile
// while the epilogue warps drain TMEM, so the ring refills behind the epilogue.
// Token chunk of the grouped kernel (kernels.h kPrefillChunk, UMMA N): 256.
// Measured against 128 (4 x 48 KB stages, 128 KB of weights in flight, no
// wide TMEM tiles): 128 is 11 % slower at 512 tokens and 18-25 % slower at
// 2048-8192 (twice the tiles, weight tiles re-read from L2 per chunk, half
// the MMA N).  An expert with more tokens becomes several chunks whose tiles
// run back to back, so the second read of a weight tile comes from L2.
constexpr int GP_MAXN = kPrefillChunk;
constexpr int kRouteItemPairs = 64;  // fused dispatch: max (token, slot) pairs of one router block
constexpr int kMaxItemTok = 4;       // ... and its tokens (route_block_tokens())
constexpr int GP_STAGE = 2 * PF_BM * PF_BK * 2 + GP_MAXN * PF_BK * 2;
constexpr int GP_STAGES = (192 * 1024) / GP_STAGE;
constexpr int GP_QN = 2;
// epilogue staging: 32 token rows x 128 columns, fp32 (down) or bf16 (up)
constexpr int GP_STG = 32 * PF_BM * 4;  // 16 KB
constexpr int GP_SMEM = GP_STAGES * GP_STAGE + GP_STG + 1024 /*align*/ + 256 /*barriers, queue*/ +
                        (8 * kMaxExperts + 1) * 4 /*schedule segments [3E+1] + [3E], splits, chunks [E]*/ +
                        2 * GP_MAXN * 4 /*down tile: pair index + gate per token row*/ +
                        (2 * kRouteItemPairs + kMaxExperts / 32 + 2) * 4 /*fused dispatch*/ +
                        2 * kMaxExperts * 4 /*counts, offsets*/;

struct GroupedArgs {
  const int32_t* counts;
  const int32_t* offsets;
  const int32_t* perm;
  const float* gates;
  const int16_t* slot_of;  // [E] of this layer
  __nv_bfloat16* h;        // [rows, f]
  float* y;                // [S][rows, d]
  int* done;               // [E][max_chunks], zero at launch
  int* split_of;           // [E] out: K splits used for each expert's down tiles (combine reads it)
  unsigned* tile_counter;  // zero at launch
  int d, f, k, E, rows, S, max_chunks;
  int debug;  // timing experiments only: bit0 skip up epilogue, bit1 skip down epilogue
  // diagnostics (MOE_B200_PF_TRACE): per CTA, per tile, 4 x u64:
  // [tile | N << 32], producer got tile, MMA issued last MMA, epilogue done
  unsigned long long* trace;
  int trace_cap;  // tiles per CTA
  SparsityCounters sp;  // fused |silu(w_in x)| < thr counters (off: sp.counts == nullptr)
  int lag;              // schedule: expert i's down tiles follow expert i+lag's up tiles
  int late8;            // eighths of the active experts whose downs take the finest split
  int s_lo;             // K split of the other experts' downs (0: S / 2)
  int cut16;            // > 0: a 2-way K split cuts at cut16/16 of K, and every
                        // expert's small second pieces go last (LPT tail)
  int evict_first;      // weights loaded with an L2 evict_first hint
  // fused path (fused != 0): the router kernel's blocks are dispatched here
  // (perm + bf16 Xg scatter, claimed dynamically by the epilogue warps before
  // their first tile), up tiles wait for their expert's rows, and the down
  // epilogues count each token's landed partials for the combine kernel,
  // which runs concurrently (launch_combine with ready flags).
  int fused;
  const float* xin;         // [n_tok][d] layer input
  const int32_t* ids;       // [n_tok][k]
  const int32_t* blk_base;  // [nblk][E] per-block expert counts (launch_route_dispatch)
  int32_t* perm_w;          // == perm, written by the dispatch
  __nv_bfloat16* xg;        // [rows][d], written by the dispatch
  unsigned* disp_ctr;       // dispatch items claimed (zero at launch)
  int* x_ready;             // [E] sorted rows written (zero at launch)
  int* tok_cnt;             // [n_tok][d/256] partials landed (zero at launch)
  int* tok_ready;           // [n_tok] hidden blocks complete (zero at launch)
  int* cq;                  // combine queue [head][tail][2 spare claims][slot: token + 1, n_tok] (zero at launch)
  int n_tok, nblk, blk_tok;
};

__device__ __forceinline__ void gp_stamp(const GroupedArgs& a, int i, int field,
                                         unsigned long long v) {
  if (a.trace && i < a.trace_cap)
    a.trace[((size_t)blockIdx.x * a.trace_cap + i) * 4 + field] = v;
}

struct GTile {
  int up, e, c, t1, s;  // t1: ffn tile (up) or hidden tile (down)
};

// The tile schedule is a list of segments, each the up or the down tiles of
// one expert: seg_start[i] = first tile of segment i, seg_code[i] = 4 e + mode
// (mode 1: up tiles; 0: down tiles, every K piece; 2 / 3: only the first /
// second piece of a 2-way uneven K split, see dn_krange).
// Token chunks (experts with > GP_MAXN tokens) are the fastest-varying index, so
// the chunks' tiles of one weight tile run back to back on different SMs and
// all but the first read it from L2.
__device__ __forceinline__ GTile gp_decode(int t, const int* seg_start, const int* seg_code,
                                           int n_ft, int n_dt, const int* split, const int* nch) {
  GTile g;
  int i = 0;
  while (seg_start[i + 1] <= t) ++i;
  const int loc = t - seg_start[i];
  g.e = seg_code[i] >> 2;
  const int mode = seg_code[i] & 3;
  g.up = mode == 1;
  const int ch = nch[g.e];
  g.c = loc % ch;
  const int rem = loc / ch;
  if (mode != 0) {
    g.t1 = rem;
    g.s = mode == 3 ? 1 : 0;
  } else {
    const int S = split[g.e];
    g.t1 = rem / S;
    g.s = rem % S;
  }
  return g;
}

// K-block range [kb0, kb1) of piece s of a down tile split S ways: even,
// or for S = 2 with cut16 > 0 a large first piece of cut16/16 of K and a
// small second one (the small pieces are scheduled last and fill the tail)
__device__ __forceinline__ void dn_krange(int s, int S, int nkb, int cut16, int& kb0, int& kb1) {
  if (S == 2 && cut16 > 0) {
    const int c = max(1, min(nkb - 1, nkb * cut16 / 16));
    kb0 = s ? c : 0;
    kb1 = s ? nkb : c;
  } else {
    kb0 = s * nkb / S;
    kb1 = (s + 1) * nkb / S;
  }
}

template <bool kSparsity>
__global__ void __launch_bounds__(PF_THREADS, 1)
    prefill_grouped_kernel(const __grid_constant__ CUtensorMap wmap_up,  // box 64 x 128
                           const __grid_constant__ CUtensorMap wmap_dn,  // box 64 x 64
                           const __grid_constant__ CUtensorMap xmap,     // Xg, box 64 x 64
                           const __grid_constant__ CUtensorMap hmap,     // H,  box 64 x 64
                           GroupedArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* stg = smem + GP_STAGES * GP_STAGE;  // epilogue staging (GP_STG bytes)
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + GP_STG);
  uint64_t* empty = full + GP_STAGES;
  uint64_t* tmem_full = empty + GP_STAGES;  // [2]
  uint64_t* tmem_empty = tmem_full + 2;      // [2]
  uint64_t* qfull = tmem_empty + 2;
  uint64_t* qempty = qfull + GP_QN;
  uint32_t* tmem_base_s = reinterpret_cast<uint32_t*>(qempty + GP_QN);
  int* q_tile = reinterpret_cast<int*>(tmem_base_s + 1);
  int* seg_start = q_tile + GP_QN;                  // [3E + 1]
  int* seg_code = seg_start + 3 * kMaxExperts + 1;   // [3E]
  int* s_split = seg_code + 3 * kMaxExperts;         // [E]
  int* s_nch = s_split + kMaxExperts;                // [E] token chunks per expert
  int* s_pair = s_nch + kMaxExperts;                              // [GP_MAXN]
  float* s_gate = reinterpret_cast<float*>(s_pair + GP_MAXN);     // [GP_MAXN]
  int* s_dpos = reinterpret_cast<int*>(s_gate + GP_MAXN);         // [kRouteItemPairs] dispatch: sorted row
  int* s_eid = s_dpos + kRouteItemPairs;                          // [kRouteItemPairs] dispatch: expert id
  unsigned* s_xrdy = reinterpret_cast<unsigned*>(s_eid + kRouteItemPairs);  // [E/32] producer's bitmask
  int* s_misc = reinterpret_cast<int*>(s_xrdy + kMaxExperts / 32);          // [2]: claimed item
  int* s_cnt = s_misc + 2;                                                   // [E] rows per expert
  int* s_off = s_cnt + kMaxExperts;                                          // [E] first sorted row
  __shared__ int s_total;

  const int warp = warp_uniform(threadIdx.x >> 5), lane = threadIdx.x & 31;
  // down tiles cover 2 x 128 hidden rows (two weight tiles per stage, like
  // up's W1/W3 pair), so both tile kinds stream 32 KB of weights per K-block
  const int n_ft = a.f / PF_BM, n_dt = a.d / (2 * PF_BM);
  griddep_wait();
  if (a.fused) {
    // per-expert totals from the router's per-block counts (all threads: one
    // segment of blocks each, then a fixed-order sum), offsets by thread 0
    const int nseg = max(1, PF_THREADS / a.E);
    for (int q = threadIdx.x; q < a.E * nseg; q += PF_THREADS) {
      const int e = q % a.E, sg = q / a.E;
      int t = 0;
      for (int b = sg; b < a.nblk; b += nseg) t += __ldcg(a.blk_base + (size_t)b * a.E + e);
      s_pair[q] = t;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < a.E; e += PF_THREADS) {
      int t = 0;
      for (int sg = 0; sg < nseg; ++sg) t += s_pair[sg * a.E + e];
      s_cnt[e] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0;
      for (int e = 0; e < a.E; ++e) {
        s_off[e] = acc;
        acc += s_cnt[e];
      }
    }
  } else {
    for (int e = threadIdx.x; e < a.E; e += PF_THREADS) {
      s_cnt[e] = a.counts[e];
      s_off[e] = a.offsets[e];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // Schedule: the active experts' up tiles in order, with expert i's down
    // tiles placed after expert i+lag's up tiles (a.lag; the default puts
    // all downs after all ups), the remaining downs last.  Down tiles of
    // expert e only wait for e's up tiles, which precede them in the list,
    // and up tiles never wait, so any lag is deadlock-free.  The last ~3/8
    // of the experts' downs — the final wave — take the finest K split
    // (a.S), the others half of it: large tiles early, small ones in the tail.
    int act[kMaxExperts];
    int n_act = 0;
    for (int e = 0; e < a.E; ++e)
      if (a.slot_of[e] >= 0 && s_cnt[e] > 0) act[n_act++] = e;
    const int n_late = (a.late8 * n_act + 7) / 8;
    int dn_tiles = 0;  // down tiles without K splits
    for (int e = 0; e < a.E; ++e) {
      s_split[e] = 1;
      s_nch[e] = max(1, (s_cnt[e] + GP_MAXN - 1) / GP_MAXN);
      if (a.slot_of[e] >= 0 && s_cnt[e] > 0) dn_tiles += s_nch[e] * n_dt;
    }
    // K splits only pay while the down tiles are few per SM (tail); with many
    // (large batches) they only add fp32 Y partial traffic for the combine
    const int s_hi = dn_tiles >= 4 * (int)gridDim.x ? 1 : min(a.S, a.f / PF_BK);
    const int s_lo = a.s_lo > 0 ? min(a.s_lo, s_hi) : max(1, s_hi / 2);
    for (int i = 0; i < n_act; ++i) s_split[act[i]] = i >= n_act - n_late ? s_hi : s_lo;
    // (every CTA writes the same values: the fused combine reads them after
    // acquiring flags released by whichever CTA finished a token)
    for (int e = 0; e < a.E; ++e) a.split_of[e] = s_split[e];
    const int kLag = a.lag;
    int ns = 0, tot = 0;
    const bool uneven = a.cut16 > 0;
    auto push = [&](int e, int mode) {
      if (mode == 0 && uneven && s_split[e] == 2) mode = 2;  // big pieces here, small ones last
      const int ch = (s_cnt[e] + GP_MAXN - 1) / GP_MAXN;
      seg_start[ns] = tot;
      seg_code[ns++] = 4 * e + mode;
      tot += mode == 1 ? ch * n_ft : ch * n_dt * (mode == 0 ? s_split[e] : 1);
    };
    for (int i = 0; i < n_act; ++i) {
      push(act[i], 1);
      if (i >= kLag) push(act[i - kLag], 0);
    }
    for (int i = max(0, n_act - kLag); i < n_act; ++i) push(act[i], 0);
    if (uneven)
      for (int i = 0; i < n_act; ++i)
        if (s_split[act[i]] == 2) push(act[i], 3);
    seg_start[ns] = tot;
    s_total = tot;
    for (int i = 0; i < GP_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tmem_full[i], 1);
      mbar_init(&tmem_empty[i], 1);
    }
    for (int i = 0; i < GP_QN; ++i) {
      mbar_init(&qfull[i], 1);
      mbar_init(&qempty[i], 2);  // MMA lane + epilogue thread 0
    }
    fence_mbar_init();
  }
  if (warp == 5) tmem_alloc(tmem_base_s, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_base_s;
  const int total = s_total;
  if (a.fused) griddep_launch_dependents();  // the combine kernel runs alongside (ready queue)
  if (a.fused && warp == 4 && lane == 0)
    for (int i = 0; i < kMaxExperts / 32; ++i) s_xrdy[i] = 0u;
  if (a.fused && warp < 4) {
    // ---- dispatch: router blocks claimed one at a time by the epilogue warps
    // (the producer meanwhile streams the first tile's weights)
    const int tpb = a.blk_tok * a.k;
    while (true) {
      if (threadIdx.x == 0) s_misc[0] = (int)atomicAdd(a.disp_ctr, 1u);
      named_bar_sync(3, 128);
      const int b = s_misc[0];
      if (b >= a.nblk) break;
      const int p0 = b * tpb;
      const int np = min(tpb, a.n_tok * a.k - p0);
      // base of this block's rows in each expert's segment: the offset plus
      // the counts of the blocks before it (128 threads, one segment each)
      int* part = s_pair;                            // [128] (free until the first down tile)
      int* s_base = reinterpret_cast<int*>(s_gate);  // [E]
      const int nseg = max(1, 128 / a.E);
      for (int q = threadIdx.x; q < a.E * nseg; q += 128) {
        const int e = q % a.E, sg = q / a.E;
        int t = 0;
        for (int bb = sg; bb < b; bb += nseg) t += __ldcg(a.blk_base + (size_t)bb * a.E + e);
        part[q] = t;
      }
      if (threadIdx.x < np) s_eid[threadIdx.x] = __ldg(a.ids + p0 + threadIdx.x);
      named_bar_sync(3, 128);
      for (int e = threadIdx.x; e < a.E; e += 128) {
        int t = s_off[e];
        for (int sg = 0; sg < nseg; ++sg) t += part[sg * a.E + e];
        s_base[e] = t;
      }
      named_bar_sync(3, 128);
      const int base = threadIdx.x < np ? s_base[s_eid[threadIdx.x]] : 0;
      if (threadIdx.x < np) {
        const int p = p0 + threadIdx.x;
        const int e = s_eid[threadIdx.x];
        int rank = 0;
        for (int q = 0; q < (int)threadIdx.x; ++q) rank += s_eid[q] == e;
        const int pos = base + rank;
        const bool local = a.slot_of[e] >= 0;  // (expert parallelism: other ranks' experts are skipped)
        if (local) a.perm_w[pos] = p;
        s_dpos[threadIdx.x] = local ? pos : -1;
      }
      named_bar_sync(3, 128);
      // the item's token rows, each read once (all its loads in flight), the
      // bf16 copy written to every sorted row of the token's pairs
      const int n4 = a.d / 4;
      const int tb = p0 / a.k, nt = (np + a.k - 1) / a.k;
      for (int c0 = threadIdx.x; c0 < n4; c0 += 128 * 2) {
        float4 v[kMaxItemTok][2];
#pragma unroll
        for (int tt = 0; tt < kMaxItemTok; ++tt)
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int c4 = c0 + u * 128;
            v[tt][u] = (tt < nt && c4 < n4)
                           ? __ldg(reinterpret_cast<const float4*>(a.xin + (size_t)(tb + tt) * a.d) + c4)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
        for (int tt = 0; tt < kMaxItemTok; ++tt) {
          if (tt >= nt) break;
          for (int j = 0; j < a.k; ++j) {
            const int i = tt * a.k + j;
            if (i >= np) break;
            if (s_dpos[i] < 0) continue;
            uint2* dst = reinterpret_cast<uint2*>(a.xg + (size_t)s_dpos[i] * a.d);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int c4 = c0 + u * 128;
              if (c4 < n4) {
                const __nv_bfloat162 lo = __floats2bfloat162_rn(v[tt][u].x, v[tt][u].y),
                                     hi = __floats2bfloat162_rn(v[tt][u].z, v[tt][u].w);
                dst[c4] = make_uint2(*reinterpret_cast<const uint32_t*>(&lo),
                                     *reinterpret_cast<const uint32_t*>(&hi));
              }
            }
          }
        }
      }
      __threadfence();
      named_bar_sync(3, 128);
      if (threadIdx.x < np) {  // the expert's first pair in this item publishes the item's count
        const int e = s_eid[threadIdx.x];
        int before = 0, n_e = 0;
        for (int q = 0; q < np; ++q) {
          before += (q < (int)threadIdx.x) & (s_eid[q] == e);
          n_e += s_eid[q] == e;
        }
        if (before == 0 && a.slot_of[e] >= 0)
          asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(a.x_ready + e), "r"(n_e) : "memory");
      }
    }
  }
  const int nkb_up = a.d / PF_BK, nkb_dn = a.f / PF_BK;
  constexpr int kA = PF_BM * PF_BK * 2;
  constexpr int kBox = PF_BOXN * PF_BK * 2;

  auto chunk_geom = [&](const GTile& g, int& nvalid, int& N, int& nboxes, int& srow) {
    const int row0 = g.c * GP_MAXN;
    nvalid = min(GP_MAXN, s_cnt[g.e] - row0);
    N = (nvalid + 15) & ~15;
    nboxes = (N + PF_BOXN - 1) / PF_BOXN;
    srow = s_off[g.e] + row0;
  };

  if (warp == 4) {
    // ===== producer =====
    if (lane == 0) {
      tma_prefetch_desc(&wmap_up);
      tma_prefetch_desc(&wmap_dn);
      tma_prefetch_desc(&xmap);
      tma_prefetch_desc(&hmap);
      uint64_t wpol;
      if (a.evict_first)
        wpol = l2_evict_first_policy();
      else
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(wpol));
      uint32_t kc = 0;
      int qi = 0, ntile = 0;
      uint32_t qph = 0;
      while (true) {
        const int t = (int)atomicAdd(a.tile_counter, 1u);
        mbar_wait(&qempty[qi], qph ^ 1);
        q_tile[qi] = t;
        mbar_arrive(&qfull[qi]);
        if (++qi == GP_QN) {
          qi = 0;
          qph ^= 1;
        }
        if (t >= total) break;
        const GTile g = gp_decode(t, seg_start, seg_code, n_ft, n_dt, s_split, s_nch);
        int nvalid, N, nboxes, srow;
        chunk_geom(g, nvalid, N, nboxes, srow);
        gp_stamp(a, ntile, 0,
                 (unsigned long long)t | ((unsigned long long)N << 32) | ((unsigned long long)g.up << 48));
        gp_stamp(a, ntile, 1, globaltimer());
        ++ntile;
        const int slot = a.slot_of[g.e];
        if (g.up) {
          const int w1row = (slot * 3 + 0) * a.f + g.t1 * PF_BM;
          const int w3row = (slot * 3 + 1) * a.f + g.t1 * PF_BM;
          const uint32_t bytes = 2 * kA + nboxes * kBox;
          int kb = 0;
          if (a.fused && !((s_xrdy[g.e >> 5] >> (g.e & 31)) & 1u)) {
            // first tile of this expert here: weights of the first stages go
            // out now, the token boxes once every row of the expert is written
            const int pre = min(nkb_up, GP_STAGES);
            for (; kb < pre; ++kb) {
              const int st = (kc + kb) % GP_STAGES;
              mbar_wait(&empty[st], (((kc + kb) / GP_STAGES) & 1) ^ 1);
              uint8_t* sp = smem + st * GP_STAGE;
              mbar_arrive_expect_tx(&full[st], bytes);
              tma_load_2d_hint(sp, &wmap_up, kb * PF_BK, w1row, &full[st], wpol);
              tma_load_2d_hint(sp + kA, &wmap_up, kb * PF_BK, w3row, &full[st], wpol);
            }
            const int want = s_cnt[g.e];
            int v;
            do {
              asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(a.x_ready + g.e) : "memory");
              if (v < want) __nanosleep(32);
            } while (v < want);
            asm volatile("fence.proxy.async.global;" ::: "memory");
            s_xrdy[g.e >> 5] |= 1u << (g.e & 31);
            for (int j = 0; j < pre; ++j) {
              const int st = (kc + j) % GP_STAGES;
              uint8_t* sp = smem + st * GP_STAGE;
              for (int b = 0; b < nboxes; ++b)
                tma_load_2d(sp + 2 * kA + b * kBox, &xmap, j * PF_BK, srow + b * PF_BOXN, &full[st]);
            }
            kc += pre;
          }
          for (; kb < nkb_up; ++kb, ++kc) {
            const int st = kc % GP_STAGES;
            mbar_wait(&empty[st], ((kc / GP_STAGES) & 1) ^ 1);
            uint8_t* sp = smem + st * GP_STAGE;
            mbar_arrive_expect_tx(&full[st], bytes);
            tma_load_2d_hint(sp, &wmap_up, kb * PF_BK, w1row, &full[st], wpol);
            tma_load_2d_hint(sp + kA, &wmap_up, kb * PF_BK, w3row, &full[st], wpol);
            for (int b = 0; b < nboxes; ++b)
              tma_load_2d(sp + 2 * kA + b * kBox, &xmap, kb * PF_BK, srow + b * PF_BOXN, &full[st]);
          }
        } else {
          // wait for every ffn tile of (e, chunk): H complete
          const int* flag = a.done + g.e * a.max_chunks + g.c;
          int v;
          do {
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
            if (v < n_ft) __nanosleep(64);
          } while (v < n_ft);
          asm volatile("fence.proxy.async.global;" ::: "memory");
          const int d0 = g.t1 * 2 * PF_BM;
          const int w2row = (slot * 3 + 2) * a.f;
          const int S = s_split[g.e];
          int kb0, kb1;
          dn_krange(g.s, S, nkb_dn, a.cut16, kb0, kb1);
          const uint32_t bytes = 2 * kA + nboxes * kBox;
          for (int kb = kb0; kb < kb1; ++kb, ++kc) {
            const int st = kc % GP_STAGES;
            mbar_wait(&empty[st], ((kc / GP_STAGES) & 1) ^ 1);
            uint8_t* sp = smem + st * GP_STAGE;
            mbar_arrive_expect_tx(&full[st], bytes);
            // W2T rows [kb*64, +64) x hidden cols [d0, d0+256): 4 boxes of 64 cols
#pragma unroll
            for (int q = 0; q < 4; ++q)
              tma_load_2d_hint(sp + q * (kA / 2), &wmap_dn, d0 + q * 64, w2row + kb * PF_BK, &full[st],
                               wpol);
            for (int b = 0; b < nboxes; ++b)
              tma_load_2d(sp + 2 * kA + b * kBox, &hmap, kb * PF_BK, srow + b * PF_BOXN, &full[st]);
          }
        }
      }
    }
  } else if (warp == 5) {
    // ===== MMA issuer =====
    if (lane == 0) {
      uint32_t kc = 0;
      TmemSched ts;
      int qi = 0, ntile = 0;
      uint32_t qph = 0;
      while (true) {
        mbar_wait(&qfull[qi], qph);
        const int t = q_tile[qi];
        mbar_arrive(&qempty[qi]);
        if (++qi == GP_QN) {
          qi = 0;
          qph ^= 1;
        }
        if (t >= total) break;
        const GTile g = gp_decode(t, seg_start, seg_code, n_ft, n_dt, s_split, s_nch);
        int nvalid, N, nboxes, srow;
        chunk_geom(g, nvalid, N, nboxes, srow);
        int bufs[2];
        uint32_t par[2];
        const int nb = ts.take(N > 128, bufs, par);
        for (int i = 0; i < nb; ++i) mbar_wait(&tmem_empty[bufs[i]], par[i] ^ 1);
        tc_fence_after();
        const uint32_t c1 = tmem + bufs[0] * 256;
        const uint32_t c3 = nb == 2 ? tmem + bufs[1] * 256 : c1 + 128;
        if (g.up) {
          const uint32_t idesc = umma_idesc(N, false);
          for (int kb = 0; kb < nkb_up; ++kb, ++kc) {
            const int st = kc % GP_STAGES;
            mbar_wait(&full[st], (kc / GP_STAGES) & 1);
            tc_fence_after();
            const uint8_t* sp = smem + st * GP_STAGE;
#pragma unroll
            for (int kk = 0; kk < PF_BK / 16; ++kk) {
              const uint64_t b = umma_desc(sp + 2 * kA + kk * 32, 16, 1024);
              const uint32_t acc = (kb | kk) != 0;
              umma_f16(c1, umma_desc(sp + kk * 32, 16, 1024), b, idesc, acc);
              umma_f16(c3, umma_desc(sp + kA + kk * 32, 16, 1024), b, idesc, acc);
            }
            umma_commit(&empty[st]);
          }
        } else {
          const uint32_t idesc = umma_idesc(N, true);
          const int S = s_split[g.e];
          int kb0, kb1;
          dn_krange(g.s, S, nkb_dn, a.cut16, kb0, kb1);
          const int nk = kb1 - kb0;
          for (int kb = 0; kb < nk; ++kb, ++kc) {
            const int st = kc % GP_STAGES;
            mbar_wait(&full[st], (kc / GP_STAGES) & 1);
            tc_fence_after();
            const uint8_t* sp = smem + st * GP_STAGE;
#pragma unroll
            for (int kk = 0; kk < PF_BK / 16; ++kk) {
              // MN-major A: 16 K-rows = 2 groups of 8 rows (SBO = 1024 B); the
              // two 64-wide M groups of a 128-row tile are adjacent boxes (LBO = 8 KB)
              const uint64_t b = umma_desc(sp + 2 * kA + kk * 32, 16, 1024);
              const uint32_t acc = (kb | kk) != 0;
              umma_f16(c1, umma_desc(sp + kk * 2048, kA / 2, 1024), b, idesc, acc);
              umma_f16(c3, umma_desc(sp + kA + kk * 2048, kA / 2, 1024), b, idesc, acc);
            }
            umma_commit(&empty[st]);
          }
        }
        for (int i = 0; i < nb; ++i) umma_commit(&tmem_full[bufs[i]]);
        gp_stamp(a, ntile++, 2, globaltimer());
      }
    }
  } else {
    // ===== epilogue (warps 0-3) =====
    TmemSched ts;
    int qi = 0, ntile = 0;
    uint32_t qph = 0;
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    while (true) {
      mbar_wait(&qfull[qi], qph);
      const int t = q_tile[qi];
      named_bar_sync(3, 128);
      if (threadIdx.x == 0) mbar_arrive(&qempty[qi]);
      if (++qi == GP_QN) {
        qi = 0;
        qph ^= 1;
      }
      if (t >= total) break;
      const GTile g = gp_decode(t, seg_start, seg_code, n_ft, n_dt, s_split, s_nch);
      int nvalid, N, nboxes, srow;
      chunk_geom(g, nvalid, N, nboxes, srow);
      if (!g.up) {
        if (a.fused) {  // perm rows of this expert were written by the dispatch
          if (threadIdx.x == 0) {
            int v;
            do {
              asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(a.x_ready + g.e) : "memory");
            } while (v < s_cnt[g.e]);
          }
          named_bar_sync(3, 128);
        }
        // the rows' pair indices and gates, fetched while the MMAs still run
        for (int j = threadIdx.x; j < nvalid; j += 128) {
          const int p = __ldg(a.perm + srow + j);
          s_pair[j] = p;
          s_gate[j] = __ldg(a.gates + p);
        }
      }
      int bufs[2];
      uint32_t par[2];
      const int nb = ts.take(N > 128, bufs, par);
      for (int i = 0; i < nb; ++i) mbar_wait(&tmem_full[bufs[i]], par[i]);
      tc_fence_after();
      const uint32_t c1 = tmem + lane_off + bufs[0] * 256;
      const uint32_t c3 = nb == 2 ? tmem + lane_off + bufs[1] * 256 : c1 + 128;
      unsigned sp_cnt[kMaxThresholds] = {};
      if (g.up && (a.debug & 1)) {
      } else if (!g.up && (a.debug & 2)) {
      } else if (g.up) {
        // silu(D1)*D3 -> bf16, transposed through smem so that each token row
        // of H (128 contiguous ffn values = 256 B) leaves as 16 B vector stores
        const int f0 = g.t1 * PF_BM;
        __nv_bfloat16* st16 = reinterpret_cast<__nv_bfloat16*>(stg);
        for (int c0 = 0; c0 < N; c0 += 32) {
          uint32_t r1[32], r3[32];
          tmem_ld32_nowait(c1 + c0, r1);
          tmem_ld32_nowait(c3 + c0, r3);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float u = __uint_as_float(r1[i]);
            const float sv = __fdividef(u, 1.0f + __expf(-u));
            st16[i * PF_BM + warp * 32 + lane] = __float2bfloat16_rn(sv * __uint_as_float(r3[i]));
            if (kSparsity && c0 + i < nvalid) {
#pragma unroll
              for (int q = 0; q < kMaxThresholds; ++q)
                if (q < a.sp.n) sp_cnt[q] += fabsf(sv) < a.sp.thr[q];
            }
          }
          named_bar_sync(3, 128);
          const int nrow = min(32, nvalid - c0);
#pragma unroll
          for (int it = 0; it < 4; ++it) {
            const int u = it * 128 + threadIdx.x;  // 32 rows x 16 x 16 B
            const int row = u >> 4, c16 = u & 15;
            if (row < nrow)
              *reinterpret_cast<uint4*>(a.h + (size_t)(srow + c0 + row) * a.f + f0 + c16 * 8) =
                  lds128(st16 + row * PF_BM + c16 * 8);
          }
          named_bar_sync(3, 128);
        }
      } else {
        // gate * D -> fp32 Y[pair], same transpose: 512 B per token row, for
        // the tile's two 128-row hidden halves (D in c1 and c3)
        float* st32 = reinterpret_cast<float*>(stg);
        for (int half = 0; half < 2; ++half) {
          const uint32_t cd = half ? c3 : c1;
          float* ys = a.y + (size_t)g.s * a.rows * a.d + g.t1 * 2 * PF_BM + half * PF_BM;
          for (int c0 = 0; c0 < N; c0 += 32) {
            uint32_t r[32];
            tmem_ld32_nowait(cd + c0, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) st32[i * PF_BM + warp * 32 + lane] = __uint_as_float(r[i]);
            named_bar_sync(3, 128);
            const int nrow = min(32, nvalid - c0);
#pragma unroll
            for (int it = 0; it < 8; ++it) {
              const int row = it * 4 + warp;  // one token row per warp per step
              if (row < nrow) {
                const int p = s_pair[c0 + row];
                const float gt = s_gate[c0 + row];
                float4 v = *reinterpret_cast<const float4*>(st32 + row * PF_BM + lane * 4);
                v.x *= gt;
                v.y *= gt;
                v.z *= gt;
                v.w *= gt;
                *reinterpret_cast<float4*>(ys + (size_t)p * a.d + lane * 4) = v;
              }
            }
            named_bar_sync(3, 128);
          }
        }
        if (a.fused) {
          // (token, hidden tile) blocks whose last partial this tile landed:
          // once all of a token's blocks are in, tok_ready[t] reaches d/256
          // and the concurrently running combine kernel (launched early, PDL)
          // sums that token's partials
          __threadfence();
          named_bar_sync(3, 128);
          const int n_ht = a.d / (2 * PF_BM);
          for (int j = threadIdx.x; j < nvalid; j += 128) {
            const int t = s_pair[j] / a.k;
            int target = 0;
            for (int jj = 0; jj < a.k; ++jj) {  // this rank's experts of the token (all on one GPU)
              const int e = __ldg(a.ids + (size_t)t * a.k + jj);
              if (a.slot_of[e] >= 0) target += s_split[e];
            }
            if (atomicAdd(a.tok_cnt + (size_t)t * n_ht + g.t1, 1) == target - 1) {
              __threadfence();  // acquire the other tiles' partials, release them onwards
              if (atomicAdd(a.tok_ready + t, 1) == n_ht - 1) {
                // the token's last block: publish it to the combine queue
                __threadfence();
                const int qi = atomicAdd(a.cq + 1, 1);
                asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(a.cq + 4 + qi), "r"(t + 1) : "memory");
              }
            }
          }
        }
      }
      if (kSparsity && g.up) {
#pragma unroll
        for (int q = 0; q < kMaxThresholds; ++q)
          if (q < a.sp.n) {
            const unsigned v = __reduce_add_sync(MOE_FULL_MASK, sp_cnt[q]);
            if (lane == 0 && v) atomicAdd(&a.sp.counts[q], (unsigned long long)v);
          }
      }
      tc_fence_before();
      named_bar_sync(3, 128);
      if (threadIdx.x == 0) {
        for (int i = 0; i < nb; ++i) mbar_arrive(&tmem_empty[bufs[i]]);
        gp_stamp(a, ntile, 3, globaltimer());
        ++ntile;
        if (g.up) {
          __threadfence();
          asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(a.done + g.e * a.max_chunks + g.c)
                       : "memory");
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) tmem_free(tmem, 512);
}

// Xg[sorted row] = bf16(x[token of that pair]); float4 in, 4 x bf16 out.
// Block 0 also zeroes the grouped kernel's sync words (tile counter + done
// flags): the grouped kernel is launched programmatically dependent on this
// one and reads them only after its griddep_wait.
__global__ void gather_rows_kernel(const float* __restrict__ x, const int32_t* __restrict__ perm,
                                   int nrows, int k, int d, __nv_bfloat16* xg, int* zero,
                                   int n_zero) {
  griddep_wait();
  griddep_launch_dependents();
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i < n_zero; i += blockDim.x) zero[i] = 0;
  const int row = blockIdx.x;
  if (row >= nrows) return;
  const int t = perm[row] / k;
  const float4* src = reinterpret_cast<const float4*>(x + (size_t)t * d);
  uint2* dst = reinterpret_cast<uint2*>(xg + (size_t)row * d);
  for (int i = threadIdx.x; i < d / 4; i += blockDim.x) {
    const float4 v = __ldg(src + i);
    const __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    dst[i] = make_uint2(*reinterpret_cast<const uint32_t*>(&a), *reinterpret_cast<const uint32_t*>(&b));
  }
}

// This rank's share of every replicated expert's rows for one step
// (replica_plan.h): order by (count desc, id asc) in parallel, then one
// thread runs the min-max split (E <= 256, world <= 8: a few us at most).
__global__ void __launch_bounds__(256) replica_plan_kernel(
    const int32_t* __restrict__ counts, const int32_t* __restrict__ offsets, int E,
    const uint32_t* __restrict__ holders, int world, int rank, ReplicaCost cost,
    int32_t* counts_out, int32_t* offsets_out) {
  __shared__ int32_t s_counts[kMaxExperts], s_order[kMaxExperts], s_lo[kMaxExperts],
      s_hi[kMaxExperts];
  __shared__ uint32_t s_hold[kMaxExperts];
  griddep_wait();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    s_counts[e] = counts[e];
    s_hold[e] = holders[e];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) s_order[replica_order_pos(s_counts, E, e)] = e;
  __syncthreads();
  if (threadIdx.x == 0) replica_split_plan(s_counts, s_order, E, s_hold, world, cost, rank, s_lo, s_hi);
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    counts_out[e] = s_hi[e] - s_lo[e];
    offsets_out[e] = offsets[e] + s_lo[e];
  }
}

cudaError_t launch_replica_plan(const int32_t* counts, const int32_t* offsets, int E,
                                const uint32_t* holders, int world, int rank, long long weight_ps,
                                long long row_ps, long long part_ps, int32_t* counts_out,
                                int32_t* offsets_out, cudaStream_t s) {
  if (E <= 0 || E > kMaxExperts || world < 1 || world > kReplicaMaxRanks) return cudaErrorInvalidValue;
  const ReplicaCost c{weight_ps, row_ps, part_ps, kPrefillChunk};
  replica_plan_kernel<<<1, 256, 0, s>>>(counts, offsets, E, holders, world, rank, c, counts_out,
                                        offsets_out);
  return cudaGetLastError();
}

// ---- host side -----------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D bf16 tensor [rows x cols] (row-major), box = box_cols x box_rows, 128B swizzle
static bool make_map(CUtensorMap* m, const void* base, long long rows, long long cols,
                     int box_cols, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool prefill_supported(const Dims& dm) {
  return dm.dtype == MOE_DTYPE_BF16 && dm.d % (2 * PF_BM) == 0 && dm.f % PF_BM == 0 &&
         dm.d % PF_BK == 0 && dm.f % PF_BK == 0 && encode_fn() != nullptr;
}

constexpr int kUpStages = 3;
constexpr int kDownStages = 4;

cudaError_t launch_prefill_experts(const LayerWeights& lw, int n_local, const Dims& dm,
                                   int n_tok, const float* x, const int32_t* counts,
                                   const int32_t* offsets, const int32_t* perm,
                                   const float* gates, const int16_t* slot_of_dev,
                                   __nv_bfloat16* xg, __nv_bfloat16* h, float* y, int* sync,
                                   int sm_count, int splits, cudaStream_t s,
                                   const SparsityCounters& sp, cudaEvent_t t0, cudaEvent_t t1,
                                   const PrefillFuse* fz) {
  const int rows = n_tok * dm.k;
  if (rows == 0 || n_local == 0) return cudaSuccess;
  if (fz && (splits <= 0 || (n_local != dm.E && fz->pa == nullptr) || !route_dispatch_supported(dm) ||
             route_block_tokens() * dm.k > kRouteItemPairs || route_block_tokens() > kMaxItemTok))
    return cudaErrorInvalidValue;
  // an expert holds <= n_tok tokens; the grouped kernel's done flags are per
  // GP_MAXN-token chunk, the two-kernel path's grid per PF_MAXN
  const int chunks = (n_tok + GP_MAXN - 1) / GP_MAXN;
  // PDL chain permute -> gather -> grouped kernel: each launch overlaps the
  // previous kernel's tail and waits (griddep_wait) before touching its data
  const bool no_pdl = debug_options().no_pdl != 0;
  cudaLaunchAttribute pdl_attr[1];
  pdl_attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl_attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t gcfg = {};
  gcfg.gridDim = dim3(rows);
  gcfg.blockDim = dim3(128);
  gcfg.stream = s;
  gcfg.attrs = pdl_attr;
  gcfg.numAttrs = no_pdl ? 0 : 1;
  const int n_zero = splits > 0 ? 1 + dm.E * chunks : 0;
  cudaError_t err;
  int* const fsync = sync + 1 + dm.E * chunks + dm.E;  // fused: [dispatch][x_ready E][combine counters]
  if (fz) {
    RouteDispatch rd;
    rd.blk_count = fz->route;
    rd.zero = sync;
    rd.n_zero = (int)prefill_sync_words(dm.E, n_tok, dm.d);
    err = launch_route_dispatch(fz->router, x, n_tok, dm, fz->ids, fz->gates, rd, s, !no_pdl);
  } else {
    err = cudaLaunchKernelEx(&gcfg, gather_rows_kernel, x, perm, rows, dm.k, dm.d, xg, sync,
                             n_zero);  // d % 128 == 0
  }
  if (err != cudaSuccess) return err;
  CUtensorMap wmap_up, wmap_dn, xmap, hmap;
  const long long wrows = 3LL * n_local * dm.f;
  if (!make_map(&wmap_up, lw.experts, wrows, dm.d, 64, PF_BM) ||
      !make_map(&wmap_dn, lw.experts, wrows, dm.d, 64, PF_BK) ||
      !make_map(&xmap, xg, rows, dm.d, 64, PF_BOXN) || !make_map(&hmap, h, rows, dm.f, 64, PF_BOXN))
    return cudaErrorInvalidValue;
  if (splits > 0) {
    // persistent grouped kernel (default)
    GroupedArgs g;
    g.counts = counts;
    g.offsets = offsets;
    g.perm = perm;
    g.gates = gates;
    g.slot_of = slot_of_dev;
    g.h = h;
    g.y = y;
    g.done = sync + 1;
    g.split_of = sync + 1 + dm.E * chunks;  // see prefill_split_of()
    g.tile_counter = reinterpret_cast<unsigned*>(sync);
    g.d = dm.d;
    g.f = dm.f;
    g.k = dm.k;
    g.E = dm.E;
    g.rows = rows;
    g.S = splits;
    g.max_chunks = chunks;
    g.debug = debug_options().pf_debug;
    g.sp = sp;
    // measured A/B (512 tokens): evict_first keeps H/Y in L2 (-33 MB DRAM,
    // combine 11.5 -> 9.6 us) but slows the weight stream by ~5 us: off
    g.evict_first = debug_options().pf_evict;
    // measured (tools/prof_prefill.py, Mixtral 512 tokens): interleaving
    // downs among ups is slower (lag 1/2/3: +33/+12/+24 us) than all ups
    // first, so the default lag puts every down after every up
    g.lag = debug_options().pf_lag;
    g.late8 = debug_options().pf_late8;
    g.s_lo = debug_options().pf_slo;
    g.cut16 = debug_options().pf_cut16;
    g.fused = fz != nullptr;
    g.xin = x;
    g.ids = fz ? fz->ids : nullptr;
    g.blk_base = fz ? fz->route : nullptr;
    g.perm_w = const_cast<int32_t*>(perm);
    g.xg = xg;
    g.disp_ctr = reinterpret_cast<unsigned*>(fsync);
    g.x_ready = fsync + 1;
    g.tok_cnt = fsync + 1 + dm.E;
    g.tok_ready = fsync + 1 + dm.E + n_tok * (dm.d / 256);
    g.cq = g.tok_ready + n_tok;
    g.n_tok = n_tok;
    g.nblk = route_blocks(n_tok);
    g.blk_tok = route_block_tokens();
    g.trace = nullptr;
    g.trace_cap = 0;
    const char* trace_path = debug_trace_path()[0] ? debug_trace_path() : nullptr;
    static unsigned long long* trace_buf = nullptr;
    if (trace_path) {
      g.trace_cap = 32;
      const size_t tb = (size_t)sm_count * g.trace_cap * 4 * sizeof(unsigned long long);
      if (!trace_buf && cudaMalloc(&trace_buf, tb) != cudaSuccess) return cudaErrorMemoryAllocation;
      if ((err = cudaMemsetAsync(trace_buf, 0, tb, s)) != cudaSuccess) return err;
      g.trace = trace_buf;
    }
    // (sync words zeroed by the gather kernel, or by the router on the fused path)
    auto kern = sp.counts ? prefill_grouped_kernel<true> : prefill_grouped_kernel<false>;
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, GP_SMEM);
    if (err != cudaSuccess) return err;
    cudaLaunchConfig_t kcfg = {};
    kcfg.gridDim = dim3(sm_count);
    kcfg.blockDim = dim3(PF_THREADS);
    kcfg.dynamicSmemBytes = GP_SMEM;
    kcfg.stream = s;
    // t0/t1 (moe_debug_kernel_timing): events on this stream right around
    // the grouped kernel — its live duration (the event breaks the PDL edge)
    cudaLaunchAttribute kattr[2];
    int nk = 0;
    if (!(no_pdl || trace_path || t0)) kattr[nk++] = pdl_attr[0];
    static int persist_off = 0;  // set once persisting L2 proved unavailable
    int persist = debug_options().pf_persist && !persist_off;
    if (persist) {
      // keep H (written by the up tiles, read back by the down tiles) and Y
      // (read by the combine; the caller places it right after H) in a
      // persisting L2 window so the weight stream does not evict them to
      // DRAM — only when the whole window fits the persisting set-aside:
      // measured -3..-9 us at 512 tokens (62.5 MB), but a clamped window
      // at 2048-8192 tokens cost 2-5 % and a 73 MB one at 640 tokens 1-2 %
      static size_t limit_set = 0;
      static int maxp = -1, maxw = 0, l2 = 0;
      if (maxp < 0) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev) != cudaSuccess)
          maxp = maxw = l2 = 0;
        // at most half the L2 set aside: 73 MB at 640 tokens already cost
        // 6-12 us (the rest of the kernel's L2 traffic loses the space)
        maxp = std::min(maxp, l2 / 2);
      }
      size_t wbytes = (size_t)rows * dm.f * 2;
      const size_t ybytes = (size_t)std::max(1, splits) * rows * dm.d * 4;
      const char* hb = reinterpret_cast<const char*>(h);
      const char* yb = reinterpret_cast<const char*>(y);
      if (yb >= hb + wbytes && yb <= hb + wbytes + 256) wbytes = (size_t)(yb - hb) + ybytes;
      if (wbytes <= (size_t)std::min(maxp, maxw)) {
        if (limit_set < wbytes) {
          if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, wbytes) != cudaSuccess) {
            // no persisting L2 here (e.g. under MPS): clear the non-sticky
            // error so a later cudaGetLastError() does not report it, and
            // run without the window from now on
            (void)cudaGetLastError();
            persist = 0;
            persist_off = 1;
            wbytes = 0;
          }
          limit_set = wbytes;
        }
      }
      if (persist && wbytes && wbytes <= (size_t)std::min(maxp, maxw)) {
        kattr[nk].id = cudaLaunchAttributeAccessPolicyWindow;
        kattr[nk].val.accessPolicyWindow.base_ptr = h;
        kattr[nk].val.accessPolicyWindow.num_bytes = wbytes;
        kattr[nk].val.accessPolicyWindow.hitRatio = 1.0f;
        kattr[nk].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        kattr[nk].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        ++nk;
      } else if (persist && limit_set) {
        // a larger batch after a windowed one: give the set-aside back
        if (cudaCtxResetPersistingL2Cache() != cudaSuccess ||
            cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0) != cudaSuccess)
          (void)cudaGetLastError();
        limit_set = 0;
      }
    }
    kcfg.attrs = kattr;
    kcfg.numAttrs = nk;
    if (t0 && (err = cudaEventRecord(t0, s)) != cudaSuccess) return err;
    err = cudaLaunchKernelEx(&kcfg, kern, wmap_up, wmap_dn, xmap, hmap, g);
    if (err == cudaSuccess && t1) err = cudaEventRecord(t1, s);
    if (err == cudaSuccess && fz && fz->pa)
      err = launch_ep_combine(x, y, n_tok, dm, fz->x_out, fz->ids, g.split_of, slot_of_dev, fz->holders, g.cq,
                              *fz->pa, fz->seq, s, !no_pdl && !t1);
    else if (err == cudaSuccess && fz)
      err = launch_combine_ready(x, y, n_tok, dm, fz->x_out, splits, fz->ids, g.split_of, g.cq,
                                 sm_count, s, !no_pdl && !t1);
    if (err != cudaSuccess || !trace_path) return err;
    // diagnostics only: synchronous dump (appends one record per launch)
    const size_t n = (size_t)sm_count * g.trace_cap * 4;
    std::vector<unsigned long long> h(n);
    if ((err = cudaMemcpyAsync(h.data(), trace_buf, n * 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
        (err = cudaStreamSynchronize(s)) != cudaSuccess)
      return err;
    if (FILE* fp = fopen(trace_path, "ab")) {
      const int hdr[4] = {sm_count, g.trace_cap, 0, 0};
      fwrite(hdr, sizeof(int), 4, fp);
      fwrite(h.data(), 8, n, fp);
      fclose(fp);
    }
    return cudaSuccess;
  }
  PrefillArgs a;
  a.counts = counts;
  a.offsets = offsets;
  a.perm = perm;
  a.gates = gates;
  a.slot_of = slot_of_dev;
  a.h = h;
  a.y = y;
  a.d = dm.d;
  a.f = dm.f;
  a.k = dm.k;
  {
    const int smem = PfSmem<kUpStages, 2>::kBytes;
    auto kern = prefill_up_kernel<kUpStages>;
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err != cudaSuccess) return err;
    kern<<<dim3(dm.f / PF_BM, chunks, dm.E), PF_THREADS, smem, s>>>(wmap_up, xmap, a);
    if ((err = cudaGetLastError()) != cudaSuccess) return err;
  }
  {
    const int smem = PfSmem<kDownStages, 1>::kBytes;
    auto kern = prefill_down_kernel<kDownStages>;
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err != cudaSuccess) return err;
    kern<<<dim3(dm.d / PF_BM, chunks, dm.E), PF_THREADS, smem, s>>>(wmap_dn, hmap, a);
    if ((err = cudaGetLastError()) != cudaSuccess) return err;
  }
  return cudaSuccess;
}

}  // namespace moe
