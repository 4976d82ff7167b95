// red_bench.cu — L2 fixed-point reduction micro-benchmark for the stack
// kernel's layer boundary: G CTAs each add a d-vector into an accumulator with
// red.global.add.u64 (the decode_stack3 pattern), vs R address-spread replicas
// (CTA c adds into replica c % R; a reader sums R values per column).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_bench tools/red_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void red_kernel(unsigned long long* acc, int d, int R, int iters) {
  const int c = blockIdx.x;
  unsigned long long* a = acc + (size_t)(c % R) * d;
  for (int it = 0; it < iters; ++it)
    for (int i = threadIdx.x; i < d; i += blockDim.x)
      atomicAdd(&a[i], (unsigned long long)(c + i + it));
}
__global__ void read_kernel(const unsigned long long* acc, int d, int R, unsigned long long* sink) {
  unsigned long long s = 0;
  for (int i = threadIdx.x; i < d; i += blockDim.x)
    for (int r = 0; r < R; ++r) s += __ldcg(&acc[(size_t)r * d + i]);
  if (s == 42) *sink = s;
}
// Epilogue pattern of a split-K down tile: each CTA (4 warps, like the
// grouped kernel's epilogue) adds / stores a 128-token x 256-column block of
// a [tokens][d] accumulator, one row per warp iteration (lane = column).
// mode 0: red.add.u64 (fixed point), 1: fp32 stores (the partials today),
// 2: red.add.f32.
__global__ void tile_kernel(void* acc, int n_tok, int d, int tiles_per_cta, int mode) {
  const int ncb = d / 256, ntb = n_tok / 128;
  for (int t = 0; t < tiles_per_cta; ++t) {
    const int tile = (blockIdx.x * tiles_per_cta + t) % (ncb * ntb);
    const int c0 = (tile % ncb) * 256, r0 = (tile / ncb) * 128;
    for (int r = threadIdx.x >> 5; r < 128; r += blockDim.x >> 5)
      for (int c = threadIdx.x & 31; c < 256; c += 32) {
        const size_t i = (size_t)(r0 + r) * d + c0 + c;
        if (mode == 0)
          asm volatile("red.global.add.u64 [%0], %1;" ::"l"((unsigned long long*)acc + i), "l"((unsigned long long)(r + c + t)) : "memory");
        else if (mode == 1)
          ((float*)acc)[i] = (float)(r + c + t);
        else
          atomicAdd((float*)acc + i, 1.0f);
      }
  }
}
int main() {
  const int d = 4096, G = 148;
  unsigned long long* acc;
  cudaMalloc(&acc, 64ull * d * 8);
  cudaMemset(acc, 0, 64ull * d * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int R : {1, 2, 4, 8, 16, 32}) {
    for (int threads : {256}) {
      const int iters = 20;
      red_kernel<<<G, threads>>>(acc, d, R, 2);
      cudaEventRecord(e0);
      red_kernel<<<G, threads>>>(acc, d, R, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      read_kernel<<<G, 256>>>(acc, d, R, acc + 63ull * d);
      cudaEventRecord(e0);
      for (int i = 0; i < iters; ++i) read_kernel<<<G, 256>>>(acc, d, R, acc + 63ull * d);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms2;
      cudaEventElapsedTime(&ms2, e0, e1);
      printf("R=%2d threads=%d: %6.2f us per %d x %d REDs (%.1f G atom/s) | reader (all CTAs sum R replicas): %.2f us/launch\n",
             R, threads, ms * 1e3 / iters, G, d, (double)G * d * iters / (ms * 1e-3) / 1e9, ms2 * 1e3 / iters);
    }
  }
  {
    const int n_tok = 512, tpc = 8;
    void* big;
    cudaMalloc(&big, (size_t)n_tok * d * 8);
    cudaMemset(big, 0, (size_t)n_tok * d * 8);
    const char* names[3] = {"red.add.u64", "st.f32", "red.add.f32"};
    for (int mode = 0; mode < 3; ++mode) {
      tile_kernel<<<G, 128>>>(big, n_tok, d, 1, mode);
      cudaEventRecord(e0);
      tile_kernel<<<G, 128>>>(big, n_tok, d, tpc, mode);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double n = (double)G * tpc * 128 * 256;
      printf("tile epilogue %-12s: %7.2f us per CTA tile (128 x 256), %.1f G elem/s over %d CTAs\n", names[mode],
             ms * 1e3 / tpc, n / (ms * 1e-3) / 1e9, G);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
