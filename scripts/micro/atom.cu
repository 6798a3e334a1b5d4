// Micro-benchmark: shared-memory FP64 accumulation into a 500-bin row, 8 rows per CTA (the V-Sample table shape):
// plain read-modify-write (races ignored: throughput only) vs atomicAdd(double) (CAS loop) vs 64-bit integer atomicAdd.
// Build: nvcc -arch=sm_100a -O3 -o atom atom.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double* out, int iters, unsigned seed, int window) {
  extern __shared__ double h[];
  for (int i = threadIdx.x; i < 8 * 512; i += blockDim.x) h[i] = 0;
  __syncthreads();
  unsigned v = (threadIdx.x + blockIdx.x * blockDim.x) * 2654435761u + seed;
  const int lane = threadIdx.x & 31;
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      v = v * 1664525u + 1013904223u;
      // lane l sits in stratification window (l mod 12): 42 bins wide, like g = 12, n_bins = 500
      unsigned b = window ? ((lane % 12) * 41 + (v >> 8) % 43) : (v >> 8) % 500;
      double w = 1.0 + (v & 255);
      double* p = h + j * 512 + b;
      if (MODE == 0) *p = *p + w;
      else if (MODE == 1) atomicAdd(p, w);
      else atomicAdd(reinterpret_cast<unsigned long long*>(p), (unsigned long long)w);
    }
  }
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = h[threadIdx.x] + acc;
}
template <class F> float timeit(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms;
}
int main() {
  void* buf; cudaMalloc(&buf, 148 * 2 * 1024 * 8);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 1 << 12;
  const char* names[3] = {"plain RMW (racy)", "atomicAdd(double)", "atomicAdd(u64)"};
  for (int window = 0; window < 2; ++window)
    for (int warps : {8, 16}) {
      float t[3];
      t[0] = timeit([&] { k<0><<<148 * (warps / 8), 256, 8 * 512 * 8>>>((double*)buf, iters, 1, window); });
      t[1] = timeit([&] { k<1><<<148 * (warps / 8), 256, 8 * 512 * 8>>>((double*)buf, iters, 1, window); });
      t[2] = timeit([&] { k<2><<<148 * (warps / 8), 256, 8 * 512 * 8>>>((double*)buf, iters, 1, window); });
      for (int m = 0; m < 3; ++m)
        printf("%s warps/SM=%2d %-18s: %.3f ms, %.1f SM-cycles per warp-update (32 updates)\n", window ? "windowed" : "uniform ", warps, names[m], t[m],
               t[m] * 1e-3 * clk * 1e3 / ((double)iters * 8 * warps));
    }
  return 0;
}
