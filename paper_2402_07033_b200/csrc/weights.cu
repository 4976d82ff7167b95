// weights.cu — device-side weight conversion and counter-based init.
//
// Upload: the reference holds fp64 row-major matrices (model.hpp:14-26).  The
// device stores W1 = w_in, W3 = w_gate ([f x d], as-is) and W2T = w_out^T
// ([f x d]) in bf16 (RNE) or fp32.  Random init: Philox4x32-10 + Box-Muller,
// N(0, 1/sqrt(d)) like random_model (model.cpp:37), keyed by (seed, tag,
// logical index) so EP shards reproduce the unsharded weights exactly.
#include <algorithm>

#include "../../include/moe_b200.h"
#include "common.cuh"
#include "kernels.h"

namespace moe {

template <typename W>
__global__ void convert_kernel(const double* __restrict__ src, W* __restrict__ dst,
                               long long rows, long long cols, bool transpose) {
  // 32x32 tile transpose through smem (coalesced both ways); plain copy
  // when !transpose.
  __shared__ double tile[32][33];
  const long long r0 = (long long)blockIdx.y * 32, c0 = (long long)blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int j = ty; j < 32; j += 8) {
    const long long r = r0 + j, c = c0 + tx;
    if (r < rows && c < cols) tile[j][tx] = src[r * cols + c];
  }
  __syncthreads();
  if (!transpose) {
    for (int j = ty; j < 32; j += 8) {
      const long long r = r0 + j, c = c0 + tx;
      if (r < rows && c < cols) dst[r * cols + c] = Elem<W>::from_double(tile[j][tx]);
    }
  } else {
    // dst is [cols x rows]
    for (int j = ty; j < 32; j += 8) {
      const long long c = c0 + j, r = r0 + tx;
      if (r < rows && c < cols) dst[c * rows + r] = Elem<W>::from_double(tile[tx][j]);
    }
  }
}

template <typename W>
__global__ void to_double_kernel(const W* __restrict__ src, double* __restrict__ dst,
                                 long long rows, long long cols, bool transpose) {
  // inverse of convert_kernel: dst [rows x cols] (reference layout); src is
  // [rows x cols], or [cols x rows] when transpose.
  __shared__ double tile[32][33];
  const long long r0 = (long long)blockIdx.y * 32, c0 = (long long)blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  if (!transpose) {
    for (int j = ty; j < 32; j += 8) {
      const long long r = r0 + j, c = c0 + tx;
      if (r < rows && c < cols) dst[r * cols + c] = (double)Elem<W>::to_float(src[r * cols + c]);
    }
    return;
  }
  for (int j = ty; j < 32; j += 8) {
    const long long c = c0 + j, r = r0 + tx;
    if (r < rows && c < cols) tile[tx][j] = (double)Elem<W>::to_float(src[c * rows + r]);
  }
  __syncthreads();
  for (int j = ty; j < 32; j += 8) {
    const long long r = r0 + j, c = c0 + tx;
    if (r < rows && c < cols) dst[r * cols + c] = tile[j][tx];
  }
}

static dim3 tiles(long long rows, long long cols) {
  return dim3((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
}

cudaError_t launch_convert(const double* src, void* dst, int dtype, long long rows,
                           long long cols, bool transpose, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  if (dtype == MOE_DTYPE_BF16)
    convert_kernel<__nv_bfloat16><<<tiles(rows, cols), dim3(32, 8), 0, s>>>(
        src, static_cast<__nv_bfloat16*>(dst), rows, cols, transpose);
  else
    convert_kernel<float><<<tiles(rows, cols), dim3(32, 8), 0, s>>>(
        src, static_cast<float*>(dst), rows, cols, transpose);
  return cudaGetLastError();
}

cudaError_t launch_to_double(const void* src, int dtype, double* dst, long long rows,
                             long long cols, bool transpose, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  if (dtype == MOE_DTYPE_BF16)
    to_double_kernel<__nv_bfloat16><<<tiles(rows, cols), dim3(32, 8), 0, s>>>(
        static_cast<const __nv_bfloat16*>(src), dst, rows, cols, transpose);
  else
    to_double_kernel<float><<<tiles(rows, cols), dim3(32, 8), 0, s>>>(
        static_cast<const float*>(src), dst, rows, cols, transpose);
  return cudaGetLastError();
}

__global__ void convert_f32_kernel(const double* __restrict__ src, float* __restrict__ dst,
                                   long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = (float)src[i];
}

cudaError_t launch_convert_f32(const double* src, float* dst, long long n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 4096);
  convert_f32_kernel<<<blocks, 256, 0, s>>>(src, dst, n);
  return cudaGetLastError();
}

// ---- router projection: rw[slot][r][:] = R_next · W2T[slot][r][:] ---------------
// The next layer's router applied to each ffn column of W2 (decode.cu uses it
// to assemble the next layer's logits during the down projection).  R_next is
// staged in shared memory; one warp per ffn row, fixed summation order.
constexpr int kProjE = 8;
template <typename W>
__global__ void __launch_bounds__(256) router_projection_kernel(const W* __restrict__ experts,
                                                                long long expert_stride,
                                                                long long mat_stride, int d, int f,
                                                                int E, const float* __restrict__ rn,
                                                                float* __restrict__ rw) {
  extern __shared__ float rs[];  // [E][d]
  for (int i = threadIdx.x; i < E * d; i += blockDim.x) rs[i] = rn[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = blockIdx.y;
  const W* w2t = experts + slot * expert_stride + 2 * mat_stride;
  for (int r = blockIdx.x * 8 + warp; r < f; r += gridDim.x * 8) {
    float acc[kProjE];
#pragma unroll
    for (int e = 0; e < kProjE; ++e) acc[e] = 0.f;
    const W* row = w2t + (size_t)r * d;
    for (int i = lane; i < d; i += 32) {
      const float w = Elem<W>::to_float(row[i]);
#pragma unroll
      for (int e = 0; e < kProjE; ++e)
        if (e < E) acc[e] = fmaf(w, rs[e * d + i], acc[e]);
    }
#pragma unroll
    for (int e = 0; e < kProjE; ++e) {
      const float v = warp_sum(acc[e]);
      if (lane == 0 && e < E) rw[((size_t)slot * f + r) * E + e] = v;
    }
  }
}

cudaError_t launch_router_projection(const void* layer_experts, int n_local, const Dims& dm,
                                     const float* router_next, float* rw, cudaStream_t s) {
  if (n_local == 0) return cudaSuccess;
  if (dm.E > kProjE) return cudaErrorInvalidValue;
  const size_t smem = sizeof(float) * (size_t)dm.E * dm.d;
  const dim3 grid((unsigned)std::min(148 * 2, (dm.f + 7) / 8), (unsigned)n_local);
  const long long es = 3LL * dm.f * dm.d, ms = (long long)dm.f * dm.d;
  cudaError_t e;
  if (dm.dtype == MOE_DTYPE_BF16) {
    e = cudaFuncSetAttribute(router_projection_kernel<__nv_bfloat16>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    router_projection_kernel<__nv_bfloat16><<<grid, 256, smem, s>>>(
        static_cast<const __nv_bfloat16*>(layer_experts), es, ms, dm.d, dm.f, dm.E, router_next, rw);
  } else {
    e = cudaFuncSetAttribute(router_projection_kernel<float>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    router_projection_kernel<float><<<grid, 256, smem, s>>>(
        static_cast<const float*>(layer_experts), es, ms, dm.d, dm.f, dm.E, router_next, rw);
  }
  return cudaGetLastError();
}

// ---- Philox4x32-10 ----------------------------------------------------------
__device__ __forceinline__ uint4 philox(uint4 c, uint2 k) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

// Normal variate #n of the stream (seed, tag): pair q = n/2 from one Philox
// block, Box-Muller, element n&1.
__device__ __forceinline__ float normal_at(uint64_t seed, uint64_t tag, unsigned long long n) {
  const unsigned long long q = n >> 1;
  const uint4 r = philox(make_uint4((uint32_t)q, (uint32_t)(q >> 32), (uint32_t)tag,
                                    (uint32_t)(tag >> 32)),
                         make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
  const float u1 = ((float)r.x + 1.0f) * 2.3283064365386963e-10f;  // (0, 1]
  const float u2 = (float)r.y * 2.3283064365386963e-10f;           // [0, 1)
  const float rad = sqrtf(-2.0f * logf(u1));
  float sv, cv;
  sincospif(2.0f * u2, &sv, &cv);
  return (n & 1) ? rad * sv : rad * cv;
}

template <typename W>
__global__ void random_kernel(W* __restrict__ dst, long long rows, long long cols, bool transpose,
                              uint64_t seed, uint64_t tag, float scale, long long ld,
                              long long off) {
  const long long n = rows * cols;
  for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < n;
       o += (long long)gridDim.x * blockDim.x) {
    // o indexes the STORED layout; recover the logical (reference) index.
    // (r, c) is the element of this [rows x cols] block, which sits at column
    // offset / row stride (off, ld) inside the full reference matrix (a
    // tensor-parallel rank holds a slice of every expert).
    long long r, c;
    if (transpose) {
      c = o / rows;  // stored [cols x rows]
      r = o - c * rows;
    } else {
      r = o / cols;
      c = o - r * cols;
    }
    const long long logical = r * ld + c + off;
    dst[o] = Elem<W>::from_float(normal_at(seed, tag, (unsigned long long)logical) * scale);
  }
}

cudaError_t launch_random(void* dst, int dtype, long long rows, long long cols, bool transpose,
                          uint64_t seed, uint64_t tag, float scale, cudaStream_t s, long long ld,
                          long long off) {
  if (ld <= 0) ld = cols;
  const long long n = rows * cols;
  if (n <= 0) return cudaSuccess;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 148 * 16);
  if (dtype == MOE_DTYPE_BF16)
    random_kernel<__nv_bfloat16><<<blocks, 256, 0, s>>>(static_cast<__nv_bfloat16*>(dst), rows,
                                                         cols, transpose, seed, tag, scale, ld,
                                                         off);
  else
    random_kernel<float><<<blocks, 256, 0, s>>>(static_cast<float*>(dst), rows, cols, transpose,
                                                seed, tag, scale, ld, off);
  return cudaGetLastError();
}

}  // namespace moe
