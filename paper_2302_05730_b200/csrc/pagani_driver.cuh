// Device side of the PAGANI refinement driver (reference: pagani.py:300-391):
// fixed-shape tree reductions, threshold classification, stable compaction and bisection.
// All of these are HBM-bound streaming kernels over the SoA region list [d][ld].
#pragma once

#include "pcb_device.cuh"

namespace pcb {

constexpr int kTreeBlock = 256;                 // threads
constexpr int kTreeSpan = kTreeBlock * 4;       // elements per CTA: one aligned 2^10 subtree

// One level of engine.tree_sum (engine.py:69-86): CTA b reduces the aligned subtree
// [b*1024, (b+1)*1024) of `in` (zero beyond n) with the adjacent-pair tree and writes out[b].
// Iterating until one value remains reproduces tree_sum bit for bit, because zero-padding
// each odd level is the same as zero-padding the input to a power of two.
__global__ void __launch_bounds__(kTreeBlock) tree_level_kernel(const double* __restrict__ in, long long n,
                                                                double* __restrict__ out) {
  __shared__ double s[kTreeBlock / 32];
  const long long base = (long long)blockIdx.x * kTreeSpan + 4LL * threadIdx.x;
  double a0 = base + 0 < n ? in[base + 0] : 0.0;
  double a1 = base + 1 < n ? in[base + 1] : 0.0;
  double a2 = base + 2 < n ? in[base + 2] : 0.0;
  double a3 = base + 3 < n ? in[base + 3] : 0.0;
  double v = (a0 + a1) + (a2 + a3);
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) v = v + __shfl_xor_sync(PCB_FULL_MASK, v, m);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
    out[blockIdx.x] = t;
  }
}

// max over a double array (only needed for the "force progress" fallback, pagani.py:364-365)
__global__ void max_kernel(const double* __restrict__ in, long long n, double* __restrict__ out) {
  __shared__ double s[32];
  double v = -1.0;  // error estimates are non-negative
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    v = fmax(v, in[i]);
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v = fmax(v, __shfl_xor_sync(PCB_FULL_MASK, v, m));
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < (blockDim.x >> 5) ? s[threadIdx.x] : -1.0;
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) v = fmax(v, __shfl_xor_sync(PCB_FULL_MASK, v, m));
    if (threadIdx.x == 0) {
      // non-negative doubles order like their bit patterns
      atomicMax((unsigned long long*)out, (unsigned long long)__double_as_longlong(fmax(v, 0.0)));
    }
  }
}

constexpr int kScanBlock = 1024;

struct ClassifyArgs {
  long long n, ld;
  int d;
  int mode;            // 0: err > budget*vol (pagani.py:361-363)   1: err >= emax (pagani.py:365)
  double budget;
  double emax;
  const double* lengths;  // [d][ld]
  const double* errors;
  unsigned char* flags;
  unsigned int* block_counts;  // per 1024-region CTA
};

// split_mask and per-CTA counts
__global__ void __launch_bounds__(kScanBlock) classify_kernel(const __grid_constant__ ClassifyArgs a) {
  __shared__ unsigned int s_cnt[32];
  const long long r = (long long)blockIdx.x * kScanBlock + threadIdx.x;
  bool split = false;
  if (r < a.n) {
    const double e = a.errors[r];
    if (a.mode == 0) {
      double vol = a.lengths[r];
      for (int j = 1; j < a.d; ++j) vol = vol * a.lengths[j * a.ld + r];  // np.prod, left to right
      split = e > a.budget * vol;
    } else {
      split = e >= a.emax;
    }
    a.flags[r] = split;
  }
  unsigned int ballot = __ballot_sync(PCB_FULL_MASK, split);
  if ((threadIdx.x & 31) == 0) s_cnt[threadIdx.x >> 5] = __popc(ballot);
  __syncthreads();
  if (threadIdx.x < 32) {
    unsigned int c = s_cnt[threadIdx.x];
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) c += __shfl_xor_sync(PCB_FULL_MASK, c, m);
    if (threadIdx.x == 0) a.block_counts[blockIdx.x] = c;
  }
}

// exclusive scan of the per-CTA counts (<= 2^16 entries for 2^26 regions): one CTA, serial chunks
__global__ void __launch_bounds__(1024) scan_counts_kernel(const unsigned int* __restrict__ counts, int nb,
                                                           unsigned long long* __restrict__ offsets,
                                                           unsigned long long* __restrict__ total) {
  __shared__ unsigned long long s_warp[32];
  __shared__ unsigned long long s_carry;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < nb; base += 1024) {
    int i = base + threadIdx.x;
    unsigned long long v = i < nb ? counts[i] : 0, x = v;
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) {
      unsigned long long y = __shfl_up_sync(PCB_FULL_MASK, x, m);
      if ((threadIdx.x & 31) >= m) x += y;
    }
    if ((threadIdx.x & 31) == 31) s_warp[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      unsigned long long w = s_warp[threadIdx.x], z = w;
#pragma unroll
      for (int m = 1; m < 32; m <<= 1) {
        unsigned long long y = __shfl_up_sync(PCB_FULL_MASK, z, m);
        if (threadIdx.x >= m) z += y;
      }
      s_warp[threadIdx.x] = z - w;  // exclusive warp offsets
    }
    __syncthreads();
    unsigned long long incl = x + s_warp[threadIdx.x >> 5] + s_carry;
    if (i < nb) offsets[i] = incl - v;
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = s_carry;
}

struct SplitArgs {
  long long n, ld_in, ld_out;
  int d;
  const double* lefts;
  const double* lengths;
  const double* integrals;
  const double* errors;
  const int32_t* axes;
  const unsigned char* flags;
  const unsigned long long* block_offsets;
  double* out_lefts;     // [d][ld_out], children 2k (lower half) and 2k+1 (upper half)
  double* out_lengths;
  double* retired_i;     // compacted estimates of the regions that are not split, parent order
  double* retired_e;
};

// stable compaction + bisection (pagani.py:282-297, 371-377)
__global__ void __launch_bounds__(kScanBlock) split_kernel(const __grid_constant__ SplitArgs a) {
  __shared__ unsigned int s_warp[32];
  const long long r = (long long)blockIdx.x * kScanBlock + threadIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const bool split = r < a.n && a.flags[r];
  const unsigned int ballot = __ballot_sync(PCB_FULL_MASK, split);
  if (lane == 0) s_warp[w] = __popc(ballot);
  __syncthreads();
  if (threadIdx.x < 32) {
    unsigned int c = s_warp[threadIdx.x], z = c;
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) {
      unsigned int y = __shfl_up_sync(PCB_FULL_MASK, z, m);
      if (threadIdx.x >= m) z += y;
    }
    s_warp[threadIdx.x] = z - c;
  }
  __syncthreads();
  if (r >= a.n) return;
  const unsigned long long rank = a.block_offsets[blockIdx.x] + s_warp[w] + __popc(ballot & ((1u << lane) - 1u));
  if (split) {
    const int axis = a.axes[r];
    const unsigned long long c = 2ULL * rank;
    for (int j = 0; j < a.d; ++j) {
      const double left = a.lefts[j * a.ld_in + r];
      double len = a.lengths[j * a.ld_in + r];
      double upper = left;
      if (j == axis) {
        len = len * 0.5;        // half = length * 0.5
        upper = left + len;     // hi_left = left + half
      }
      *reinterpret_cast<double2*>(a.out_lefts + j * a.ld_out + c) = make_double2(left, upper);
      *reinterpret_cast<double2*>(a.out_lengths + j * a.ld_out + c) = make_double2(len, len);
    }
  } else {
    const unsigned long long k = (unsigned long long)r - rank;
    a.retired_i[k] = a.integrals[r];
    a.retired_e[k] = a.errors[r];
  }
}

// lexicographic uniform tiling, axis 0 slowest: left = idx * (1/g), length = 1/g (core.py:265-268)
__global__ void tiling_kernel(int d, int g, long long first, long long n, long long ld, double h, double* lefts, double* lengths) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    long long rem = first + r;  // global tile index
    for (int j = d - 1; j >= 0; --j) {
      lefts[j * ld + r] = (double)(rem % g) * h;
      lengths[j * ld + r] = h;
      rem /= g;
    }
  }
}

// (n,d) row-major host layout <-> [d][ld] device layout
__global__ void rows_to_soa_kernel(int d, long long n, long long ld, const double* __restrict__ rows, double* __restrict__ soa) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x)
    for (int j = 0; j < d; ++j) soa[j * ld + r] = rows[r * d + j];
}

__global__ void soa_to_rows_kernel(int d, long long begin, long long n, long long ld, const double* __restrict__ soa, double* __restrict__ rows) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x)
    for (int j = 0; j < d; ++j) rows[r * d + j] = soa[j * ld + begin + r];
}

// dst[j][dst_off + r] = src[j][src_off + r]
__global__ void soa_copy_kernel(int d, long long n, long long ld_src, long long src_off, const double* __restrict__ src,
                                long long ld_dst, long long dst_off, double* __restrict__ dst) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x)
    for (int j = 0; j < d; ++j) dst[j * ld_dst + dst_off + r] = src[j * ld_src + src_off + r];
}

__global__ void rows_to_soa_at_kernel(int d, long long n, long long ld, long long off, const double* __restrict__ rows, double* __restrict__ soa) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x)
    for (int j = 0; j < d; ++j) soa[j * ld + off + r] = rows[r * d + j];
}

__global__ void widen_axes_kernel(long long n, const int32_t* __restrict__ in, long long* __restrict__ out) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x)
    out[r] = in[r];
}

}  // namespace pcb
