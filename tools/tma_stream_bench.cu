// tma_stream_bench.cu — HBM streaming rate of the two weight-access patterns
// the product kernels use, with no math (measurement tool, not product code).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda \
//        -o tools/tma_stream_bench tools/tma_stream_bench.cu && tools/tma_stream_bench
//
// A bf16 matrix of 3 x 8 x 14336 rows x 4096 columns (all W1/W3/W2T rows of
// one Mixtral layer, 2.82 GB) is streamed once per pass by a persistent grid
// (one CTA per SM) through a shared-memory ring:
//   rows1d  : each CTA copies contiguous 32 KB row chunks (cp.async.bulk), the
//             decode kernel's pattern;
//   tile2d  : each CTA takes 128-row tiles and walks K in 64-column boxes,
//             two boxes (two 128-row groups) per 32 KB stage — the grouped
//             prefill kernel's weight pattern (TMA 2-D, SWIZZLE_128B);
//   tile2dK2: the same with two adjacent K boxes of ONE 128-row group per
//             stage (256 B contiguous per row per stage).
//   tile2dX : tile2d plus, per stage, the token boxes the grouped kernel
//             also loads: 3 x (64 tokens x 64 columns) of an L2-resident
//             bf16 activation matrix (24 KB; ~160 tokens per expert at 512
//             tokens) — does the L2->SM token traffic slow the weight stream?
// The consumer warp only waits for each stage and frees it.  Ring depth is
// a parameter (stages x 32 KB).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2402_07033_b200/csrc/common.cuh"
using namespace moe;

constexpr int kStage = 32 * 1024;

__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// mode 0: rows1d, 1: tile2d (2 row groups per stage), 2: tile2dK2 (2 K boxes per stage)
constexpr int kXBytes = 3 * 64 * 128;  // mode 3: token boxes per stage
__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap map,
                                                      const __grid_constant__ CUtensorMap xmap,
                                                      const char* base, long long rows, int K,
                                                      int stages, int mode) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t full[16], empty[16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const long long row_bytes = (long long)K * 2;
  const long long total = rows * row_bytes;
  // work items: mode 0 = 32 KB chunks of the flat matrix; modes 1/2 = (tile, kblock pairs)
  long long n_items, per;
  const int sbytes = kStage + (mode == 3 ? kXBytes : 0);
  if (mode == 0) {
    n_items = total / kStage;
  } else {
    const long long tiles = rows / (mode == 1 || mode == 3 ? 256 : 128);
    per = mode == 1 || mode == 3 ? K / 64 : K / 128;
    n_items = tiles * per;
  }
  const long long i0 = n_items * blockIdx.x / gridDim.x, i1 = n_items * (blockIdx.x + 1) / gridDim.x;
  if (warp == 0) {
    if (lane != 0) return;
    int st = 0;
    uint32_t ph = 0;
    for (long long i = i0; i < i1; ++i) {
      mbar_wait(&empty[st], ph ^ 1);
      unsigned char* dst = sm + (size_t)st * sbytes;
      mbar_arrive_expect_tx(&full[st], sbytes);
      if (mode == 0) {
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(dst)),
            "l"(base + i * kStage), "r"(kStage), "r"(smem_u32(&full[st]))
            : "memory");
      } else {
        const long long tile = i / per, kb = i % per;
        if (mode == 1 || mode == 3) {
          tma2d(dst, &map, (int)(kb * 64), (int)(tile * 256), &full[st]);
          tma2d(dst + 16384, &map, (int)(kb * 64), (int)(tile * 256 + 128), &full[st]);
          if (mode == 3)
            for (int b = 0; b < 3; ++b)
              tma2d(dst + kStage + b * 8192, &xmap, (int)(kb * 64), (int)((tile % 4) * 192 + b * 64), &full[st]);
        } else {
          tma2d(dst, &map, (int)(kb * 128), (int)(tile * 128), &full[st]);
          tma2d(dst + 16384, &map, (int)(kb * 128 + 64), (int)(tile * 128), &full[st]);
        }
      }
      if (++st == stages) {
        st = 0;
        ph ^= 1;
      }
    }
  } else {
    if (lane != 0) return;
    int st = 0;
    uint32_t ph = 0;
    for (long long i = i0; i < i1; ++i) {
      mbar_wait(&full[st], ph);
      mbar_arrive(&empty[st]);
      if (++st == stages) {
        st = 0;
        ph ^= 1;
      }
    }
  }
}

int main() {
  const long long rows = 3LL * 8 * 14336;
  const int K = 4096;
  const size_t bytes = (size_t)rows * K * 2;
  void* base = nullptr;
  if (cudaMalloc(&base, bytes) != cudaSuccess) return 1;
  cudaMemset(base, 1, bytes);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return 2;
  // L2-resident activations for mode 3: 768 tokens x K bf16 (6 MB)
  void* xbase = nullptr;
  if (cudaMalloc(&xbase, (size_t)768 * K * 2) != cudaSuccess) return 1;
  cudaMemset(xbase, 1, (size_t)768 * K * 2);
  CUtensorMap xmap;
  cuuint64_t xdims[2] = {(cuuint64_t)K, 768};
  cuuint32_t xbox[2] = {64, 64};
  if (enc(&xmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, xbase, xdims, strides, xbox, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return 2;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
  const char* names[4] = {"rows1d  ", "tile2d  ", "tile2dK2", "tile2dX "};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int stages : {3, 4, 6}) {
    for (int mode = 0; mode < 4; ++mode) {
      const int smem = stages * (kStage + (mode == 3 ? kXBytes : 0));
      if (smem > 225 * 1024) continue;
      for (int w = 0; w < 2; ++w)
        stream_kernel<<<sms, 64, smem>>>(map, xmap, (const char*)base, rows, K, stages, mode);
      cudaEventRecord(e0);
      const int reps = 10;
      for (int r = 0; r < reps; ++r)
        stream_kernel<<<sms, 64, smem>>>(map, xmap, (const char*)base, rows, K, stages, mode);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const cudaError_t err = cudaGetLastError();
      printf("%s stages %d: %.1f us per pass, %.0f GB/s of weights %s\n", names[mode], stages, ms * 1e3 / reps,
             bytes / (ms / reps * 1e-3) / 1e9, err == cudaSuccess ? "" : cudaGetErrorString(err));
    }
  }
  return 0;
}
