// Micro-benchmarks that drive design choices: MATCH.ANY throughput, FP64 dependent latency,
// shared-memory random 64-bit RMW throughput.  Build: nvcc -arch=sm_100a -O3 -o micro micro.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_match(unsigned* out, int iters, unsigned seed) {
  unsigned v = threadIdx.x * 2654435761u + seed, acc = 0;
  for (int i = 0; i < iters; ++i) { acc += __match_any_sync(0xffffffffu, v & 511); v = v * 1664525u + 1013904223u; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_lcg(unsigned* out, int iters, unsigned seed) {
  unsigned v = threadIdx.x * 2654435761u + seed, acc = 0;
  for (int i = 0; i < iters; ++i) { acc += (v & 511); v = v * 1664525u + 1013904223u; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_dadd_chain(double* out, int iters, double a) {
  double x = threadIdx.x;
  for (int i = 0; i < iters; ++i) x = __dadd_rn(x, a);
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}
__global__ void k_dfma_chain(double* out, int iters, double a) {
  double x = threadIdx.x;
  for (int i = 0; i < iters; ++i) x = __fma_rn(x, a, a);
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}
__global__ void k_smem_rmw(double* out, int iters, unsigned seed) {
  extern __shared__ double h[];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) h[i] = 0;
  __syncthreads();
  double* mine = h;  // single table, we only measure LSU throughput (races ignored)
  unsigned v = threadIdx.x * 2654435761u + seed;
  for (int i = 0; i < iters; ++i) { unsigned b = (v >> 8) & 4095; mine[b] = mine[b] + 1.0; v = v * 1664525u + 1013904223u; }
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = h[threadIdx.x];
}
template <class F> float timeit(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms;
}
int main() {
  void* buf; cudaMalloc(&buf, 148 * 1024 * 8 * 4);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 1 << 16;
  for (int warps : {1, 4, 8, 16, 32}) {
    float m1 = timeit([&] { k_match<<<148, warps * 32>>>((unsigned*)buf, iters, 1); });
    float m0 = timeit([&] { k_lcg<<<148, warps * 32>>>((unsigned*)buf, iters, 1); });
    double cyc = (m1 - m0) * 1e-3 * clk * 1e3;  // cycles at nominal clock
    printf("MATCH.ANY warps/SM=%2d: %.2f cycles per warp-instr per SM (loop %.3f ms vs %.3f ms)\n", warps, cyc / ((double)iters * warps), m1, m0);
  }
  {
    float t = timeit([&] { k_dadd_chain<<<148, 32>>>((double*)buf, iters, 1e-9); });
    printf("DADD dependent latency: %.1f cycles\n", t * 1e-3 * clk * 1e3 / iters);
    t = timeit([&] { k_dfma_chain<<<148, 32>>>((double*)buf, iters, 1.0000001); });
    printf("DFMA dependent latency: %.1f cycles\n", t * 1e-3 * clk * 1e3 / iters);
    for (int warps : {4, 8, 16, 32}) {
      t = timeit([&] { k_dadd_chain<<<148, warps * 32>>>((double*)buf, iters, 1e-9); });
      printf("DADD chain, %2d warps/SM: %.2f cycles per warp-instr per SMSP\n", warps, t * 1e-3 * clk * 1e3 / iters / (warps / 4.0));
    }
  }
  for (int warps : {1, 4, 8, 16}) {
    float t = timeit([&] { k_smem_rmw<<<148, warps * 32, 4096 * 8>>>((double*)buf, iters / 4, 1); });
    printf("smem random RMW (LDS.64+DADD+STS.64) warps/SM=%2d: %.1f cycles per warp-RMW per SM\n", warps, t * 1e-3 * clk * 1e3 / (iters / 4.0 * warps));
  }
  return 0;
}
