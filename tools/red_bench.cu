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
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
