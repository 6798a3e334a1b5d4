// Device side of the PAGANI refinement driver (reference: pagani.py:300-391):
// fixed-shape tree reductions, threshold classification, stable compaction and bisection.
// All of these are HBM-bound streaming kernels over the SoA region list [d][ld].
#pragma once

#include "pcb_device.cuh"

namespace pcb {

// errorest target and per-unit-volume split budget (pagani.py:350, 362).  With abs_tol = 0 (the reference) these are
// the reference's own expressions, rel_tol*|estimate| and 0.8*rel_tol*|estimate| in that association; a positive
// abs_tol (epsabs extension) takes over where it is the larger target.
__host__ __device__ inline double tolerance_target(double rel_tol, double abs_tol, double estimate) {
  const double rel = rel_tol * fabs(estimate);
  return abs_tol > rel ? abs_tol : rel;
}
__host__ __device__ inline double split_budget(double rel_tol, double abs_tol, double estimate) {
  return abs_tol > rel_tol * fabs(estimate) ? 0.8 * abs_tol : 0.8 * rel_tol * fabs(estimate);
}

constexpr int kTreeBlock = 256;                 // threads
constexpr int kTreeSpan = kTreeBlock * 4;       // elements per CTA: one aligned 2^10 subtree

// One level of engine.tree_sum (engine.py:69-86): CTA b reduces the aligned subtree
// [b*1024, (b+1)*1024) of `in` (zero beyond n) with the adjacent-pair tree and writes out[b].
// Iterating until one value remains reproduces tree_sum bit for bit, because zero-padding
// each odd level is the same as zero-padding the input to a power of two.
__global__ void __launch_bounds__(kTreeBlock) tree_level_kernel(const double* __restrict__ in, long long n,
                                                                double* __restrict__ out) {
  pdl_wait();   // may be launched with programmatic serialisation behind its producer (a no-op otherwise)
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

// The same level for TWO arrays of equal length in one launch (blockIdx.y selects the array): the refinement always
// sums integrals and errors together, and a launch boundary costs more than a level of a short list.
__global__ void __launch_bounds__(kTreeBlock) tree_level2_kernel(const double* __restrict__ in0, const double* __restrict__ in1,
                                                                 long long n, double* __restrict__ out0, double* __restrict__ out1) {
  pdl_wait();
  __shared__ double s[kTreeBlock / 32];
  const double* __restrict__ in = blockIdx.y ? in1 : in0;
  double* __restrict__ out = blockIdx.y ? out1 : out0;
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
  pdl_wait();   // may be launched with programmatic serialisation behind its producer (a no-op otherwise)
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
  // Budget taken on the device (mode 0, `scalars` != NULL): the host's own expressions on the scalars it is about to
  // read -- fin = fin_i [+ scalars[slot_ret_i]], estimate = fin + scalars[slot_sum_i] -- so that the classification can
  // be enqueued BEFORE the host has seen the sums and one round trip per iteration carries sums and split count.
  const double* scalars = nullptr;
  double fin_i = 0.0, rel_tol = 0.0, abs_tol = 0.0;
  int have_retired = 0, slot_sum_i = 0, slot_ret_i = 0;
};

// split_mask and per-CTA counts
__global__ void __launch_bounds__(kScanBlock) classify_kernel(const __grid_constant__ ClassifyArgs a) {
  pdl_wait();   // may be launched with programmatic serialisation behind its producer (a no-op otherwise)
  __shared__ unsigned int s_cnt[32];
  const long long r = (long long)blockIdx.x * kScanBlock + threadIdx.x;
  bool split = false;
  double budget = a.budget;
  if (a.scalars) {
    double fin = a.fin_i;
    if (a.have_retired) fin = fin + a.scalars[a.slot_ret_i];
    budget = split_budget(a.rel_tol, a.abs_tol, fin + a.scalars[a.slot_sum_i]);
  }
  if (r < a.n) {
    const double e = a.errors[r];
    if (a.mode == 0) {
      double vol = a.lengths[r];
      for (int j = 1; j < a.d; ++j) vol = vol * a.lengths[j * a.ld + r];  // np.prod, left to right
      split = e > budget * vol;
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
  pdl_wait();   // may be launched with programmatic serialisation behind its producer (a no-op otherwise)
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
  unsigned long long* rearm_bad = nullptr;   // non-finite flag of the evaluation that follows (set to ~0 here), or NULL
};

// Hand `count` scalar slots to the host through pinned memory: values first, then the sequence word the host polls.
// Replaces a device->host copy plus a stream synchronisation per read (two per iteration of the general refine path).
__global__ void publish_scalars_kernel(const unsigned long long* __restrict__ scalars, int first, int count,
                                       volatile unsigned long long* pinned, volatile unsigned long long* seq_word, unsigned long long seq) {
  pdl_wait();
  if (threadIdx.x < count) pinned[first + threadIdx.x] = scalars[first + threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    *seq_word = seq;
  }
}

// stable compaction + bisection (pagani.py:282-297, 371-377)
__global__ void __launch_bounds__(kScanBlock) split_kernel(const __grid_constant__ SplitArgs a) {
  pdl_wait();   // may be launched with programmatic serialisation behind its producer (a no-op otherwise)
  __shared__ unsigned int s_warp[32];
  const long long r = (long long)blockIdx.x * kScanBlock + threadIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (a.rearm_bad && r == 0) *a.rearm_bad = ~0ULL;   // the host has read the previous evaluation's flag before it launched this kernel
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
  pdl_wait();   // may be launched with programmatic serialisation behind its producer (a no-op otherwise)
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

// ------------------------------------------------------------------------------------------------------------
// One refinement iteration of a SHORT list (n <= 1024 regions) in one CTA: global sums, stop tests, threshold
// classification (with the forced-progress fallback), stable compaction + bisection and the retired sums
// (pagani.py:336-378) -- the work of ten launches and two host round trips of the general path.  The arithmetic
// is the general path's: 1024-leaf adjacent-pair trees (= engine.tree_sum with zero padding), serial volume
// products, the same comparisons.  The host passes the running totals in and reads one record back from pinned
// memory; `bad` is the evaluate kernel's non-finite flag, re-armed here for the next evaluation.
// ------------------------------------------------------------------------------------------------------------
struct ShortIterRecord {       // pinned host memory
  double estimate, errorest;   // of this iteration (pagani.py:336-337)
  double fin_i, fin_e;         // finished totals after this iteration's retirements
  long long n_split;           // regions bisected (children = 2 * n_split)
  unsigned long long bad;      // first non-finite evaluation (region * f_eval + point) or ~0
  int action;                  // 0: continue with the children   1: tolerance met   2: max iterations   3: region cap
  int pad;
  volatile unsigned long long seq;
};

struct ShortIterArgs {
  int n, d;
  long long ld_in, ld_out_unused;
  const double* lefts;         // [d][ld_in]
  const double* lengths;
  const double* integrals;
  const double* errors;
  const int32_t* axes;
  double* out_lefts;           // [d][ld_out], ld_out = round_up(2 * n_split, 32), capacity for n_split = n
  double* out_lengths;
  double fin_i, fin_e;
  long long processed, region_cap;
  double rel_tol, abs_tol;
  int iteration, max_iterations;
  unsigned long long* bad;     // device flag of the evaluate kernel
  ShortIterRecord* record;
  unsigned long long seq;
  // device-resident chain (ShortState, pcb_device.cuh): the kernel always leaves the next iteration's inputs in
  // `state`; with from_state it also TAKES n, ld_in, fin_i, fin_e and processed from there (the host enqueued it before
  // it knew them) and returns at once when the chain has stopped
  ShortState* state = nullptr;
  int from_state = 0;
  int short_max = 1024;        // longest list the chain continues with
};

// adjacent-pair tree over 1024 values, one per thread (zeros beyond the data); every thread gets the sum
__device__ __forceinline__ double tree1024(double v, double* s_warp /* [32] */) {
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) v = v + __shfl_xor_sync(PCB_FULL_MASK, v, m);
  __syncthreads();   // s_warp may still be read from a previous call
  if ((threadIdx.x & 31) == 0) s_warp[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = s_warp[threadIdx.x & 31];
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) t = t + __shfl_xor_sync(PCB_FULL_MASK, t, m);
  return t;
}

// ------------------------------------------------------------------------------------------------------------
// Sharded refinement (multi-GPU): the global tree sums of refine (pagani.py:336-337, 371-372) from per-rank pieces.
// The ordered global list is the concatenation of the ranks' slices.  Every rank packs ONE row per iteration:
//   header   [0] first non-finite evaluation of its slice (8-byte integer, ~0 = none), [1] n_active, [2] n_retired
//   section  x 4 (active integrals, active errors, retired integrals, retired errors):
//            counts [4] = n_head, n_blocks, n_tail, 0;  head[1024]: raw values before the first 1024-aligned GLOBAL
//            index;  tail[1024]: raw values behind the last complete aligned block;  blocks[width]: pair-tree sums
//            of the complete aligned 1024-blocks (tree_level_kernel)
// The rows are all-gathered and every rank rebuilds the ordered list of 1024-block sums (a block that straddles
// ranks is re-assembled from one tail and the following heads) and finishes the tree: bit-identical to a
// single-device tree_sum over the concatenation, for any number of ranks.
// ------------------------------------------------------------------------------------------------------------
__host__ __device__ inline long long shard_section_doubles(long long width) { return 4 + 2 * kTreeSpan + width; }
__host__ __device__ inline long long shard_row_doubles(long long width) { return 4 + 4 * shard_section_doubles(width); }

struct ShardPackArgs {
  double* row;
  long long width;
  const double* src[4];
  long long n[4];        // elements of the section on this rank (0: empty section)
  long long head[4];     // (-global offset) mod 1024
  const unsigned long long* bad;
};

// grid = 4 sections: raw head / tail values and the counts (the block sums are written by tree_level_kernel)
__global__ void __launch_bounds__(kTreeSpan) shard_pack_kernel(const __grid_constant__ ShardPackArgs a) {
  const int s = blockIdx.x, t = threadIdx.x;
  double* sec = a.row + 4 + (long long)s * shard_section_doubles(a.width);
  const long long n = a.n[s];
  const long long h = a.head[s] < n ? a.head[s] : n;
  const long long nb = (n - h) / kTreeSpan, tail = n - h - nb * kTreeSpan;
  sec[4 + t] = t < h ? a.src[s][t] : 0.0;
  sec[4 + kTreeSpan + t] = t < tail ? a.src[s][h + nb * kTreeSpan + t] : 0.0;
  if (t == 0) {
    sec[0] = (double)h;
    sec[1] = (double)nb;
    sec[2] = (double)tail;
    sec[3] = 0.0;
    if (s == 0) {
      *reinterpret_cast<unsigned long long*>(a.row) = *a.bad;
      a.row[1] = (double)a.n[0];
      a.row[2] = (double)a.n[2];
      a.row[3] = 0.0;
    }
  }
}

struct ShardAssembleArgs {
  const double* gathered;   // world rows
  int world;
  long long row_doubles, width;
  double* lists[4];         // per section: the ordered 1024-block sums of the GLOBAL array
};

// grid = (world, 4): CTA (r, s) places rank r's complete-block sums of section s at their global block indices and,
// when r has a tail, re-assembles the block that starts with it (its tail, then the heads of the following ranks)
__global__ void __launch_bounds__(kTreeSpan) shard_assemble_kernel(const __grid_constant__ ShardAssembleArgs a) {
  __shared__ double s_warp[32];
  const int r = blockIdx.x, s = blockIdx.y, t = threadIdx.x;
  auto section = [&](int q) { return a.gathered + (long long)q * a.row_doubles + 4 + (long long)s * shard_section_doubles(a.width); };
  long long off = 0;   // global element offset of rank r's slice of this section
  for (int q = 0; q < r; ++q) {
    const double* c = section(q);
    off += (long long)c[0] + (long long)c[1] * kTreeSpan + (long long)c[2];
  }
  const double* me = section(r);
  const long long h = (long long)me[0], nb = (long long)me[1], tail = (long long)me[2];
  const long long first_block = (off + h) / kTreeSpan;
  double* list = a.lists[s];
  for (long long i = t; i < nb; i += kTreeSpan) list[first_block + i] = me[4 + 2 * kTreeSpan + i];
  if (tail == 0) return;
  double leaf = 0.0;
  if (t < tail) {
    leaf = me[4 + kTreeSpan + t];
  } else {
    long long pos = tail;
    for (int q = r + 1; q < a.world && pos < kTreeSpan; ++q) {
      const double* c = section(q);
      const long long hq = (long long)c[0];
      if (t < pos + hq) { leaf = c[4 + (t - pos)]; break; }
      pos += hq;
      if ((long long)c[1] > 0 || (long long)c[2] > 0) break;   // rank q reaches beyond this block: it ends here
    }
  }
  const double sum = tree1024(leaf, s_warp);
  if (t == 0) list[first_block + nb] = sum;
}

// (split count, largest error) of the local list, as the two doubles the ranks all-gather
__global__ void shard_pack_counts_kernel(const unsigned long long* n_split, const double* emax, double* row) {
  row[0] = (double)*n_split;
  row[1] = *emax;
}

__global__ void __launch_bounds__(1024) short_iteration_kernel(const __grid_constant__ ShortIterArgs a) {
  __shared__ double s_warp[32];
  __shared__ unsigned int s_cnt[32];
  __shared__ double s_ret_i[1024], s_ret_e[1024];
  __shared__ double s_emax;
  const int r = threadIdx.x, lane = r & 31, w = r >> 5;
  pdl_wait();   // launched behind the evaluate kernel with programmatic serialisation: its results are visible from here
  int n = a.n;
  long long ld_in = a.ld_in, processed = a.processed;
  double fin_i0 = a.fin_i, fin_e0 = a.fin_e;
  if (a.from_state) {
    if (a.state->status != 0) return;   // CTA-uniform: the chain stopped before this iteration
    n = (int)a.state->n;
    ld_in = a.state->ld;
    processed = a.state->processed;
    fin_i0 = a.state->fin_i;
    fin_e0 = a.state->fin_e;
  }
  const bool have = r < n;
  const double my_i = have ? a.integrals[r] : 0.0, my_e = have ? a.errors[r] : 0.0;
  const double sum_i = tree1024(my_i, s_warp);
  const double sum_e = tree1024(my_e, s_warp);
  const double estimate = fin_i0 + sum_i, errorest = fin_e0 + sum_e;
  const unsigned long long bad = *a.bad;
  __syncthreads();   // every thread holds the flag before thread 0 may re-arm it below: `action` is CTA-uniform
  int action = 0;
  if (bad != ~0ULL) action = 4;   // the host raises; nothing else matters
  else if (errorest <= tolerance_target(a.rel_tol, a.abs_tol, estimate)) action = 1;
  else if (a.iteration == a.max_iterations) action = 2;
  long long n_split = 0;
  double fin_i = fin_i0, fin_e = fin_e0;
  if (action == 0) {
    // classification (pagani.py:361-365)
    const double budget = split_budget(a.rel_tol, a.abs_tol, estimate);
    bool split = false;
    if (have) {
      double vol = a.lengths[r];
      for (int j = 1; j < a.d; ++j) vol = vol * a.lengths[j * ld_in + r];  // np.prod, left to right
      split = my_e > budget * vol;
    }
    unsigned total = __syncthreads_count(split);
    if (total == 0) {  // nothing exceeds its budget: force progress on the worst regions, ties included
      double m = have ? my_e : -1.0;
#pragma unroll
      for (int k = 16; k >= 1; k >>= 1) m = fmax(m, __shfl_xor_sync(PCB_FULL_MASK, m, k));
      if (lane == 0) s_warp[w] = m;
      __syncthreads();
      if (w == 0) {
        double t = s_warp[lane];
#pragma unroll
        for (int k = 16; k >= 1; k >>= 1) t = fmax(t, __shfl_xor_sync(PCB_FULL_MASK, t, k));
        if (lane == 0) s_emax = fmax(t, 0.0);
      }
      __syncthreads();
      split = have && my_e >= s_emax;
      total = __syncthreads_count(split);
    }
    n_split = total;
    if (processed + 2 * n_split > a.region_cap) {
      action = 3;
    } else {
      // stable ranks: exclusive scan of the split flags
      const unsigned ballot = __ballot_sync(PCB_FULL_MASK, split);
      if (lane == 0) s_cnt[w] = __popc(ballot);
      __syncthreads();
      if (w == 0) {
        unsigned c = s_cnt[lane], z = c;
#pragma unroll
        for (int m = 1; m < 32; m <<= 1) {
          unsigned y = __shfl_up_sync(PCB_FULL_MASK, z, m);
          if (lane >= m) z += y;
        }
        s_cnt[lane] = z - c;
      }
      s_ret_i[r] = 0.0;
      s_ret_e[r] = 0.0;
      __syncthreads();
      const unsigned rank = s_cnt[w] + __popc(ballot & ((1u << lane) - 1u));
      const long long ld_out = (2 * n_split + 31) / 32 * 32;
      if (have) {
        if (split) {
          const int axis = a.axes[r];
          const unsigned c = 2u * rank;
          for (int j = 0; j < a.d; ++j) {
            const double left = a.lefts[j * ld_in + r];
            double len = a.lengths[j * ld_in + r];
            double upper = left;
            if (j == axis) {
              len = len * 0.5;        // half = length * 0.5
              upper = left + len;     // hi_left = left + half
            }
            *reinterpret_cast<double2*>(a.out_lefts + j * ld_out + c) = make_double2(left, upper);
            *reinterpret_cast<double2*>(a.out_lengths + j * ld_out + c) = make_double2(len, len);
          }
        } else {
          const unsigned k = (unsigned)r - rank;   // parent order among the retired
          s_ret_i[k] = my_i;
          s_ret_e[k] = my_e;
        }
      }
      __syncthreads();
      // fin += tree_sum(act[~mask]) (pagani.py:371-372)
      const double ret_i = tree1024(s_ret_i[r], s_warp);
      const double ret_e = tree1024(s_ret_e[r], s_warp);
      fin_i = fin_i0 + ret_i;
      fin_e = fin_e0 + ret_e;
    }
  }
  if (r == 0) {
    *a.bad = ~0ULL;   // re-arm for the next evaluation
    if (a.state) {    // every thread read the old state before the barriers above
      ShortState* st = a.state;
      st->n = 2 * n_split;
      st->ld = (2 * n_split + 31) / 32 * 32;
      st->fin_i = fin_i;
      st->fin_e = fin_e;
      st->processed = processed + 2 * n_split;
      st->status = action != 0 ? action : (2 * n_split > a.short_max ? 5 : 0);
    }
    ShortIterRecord* rec = a.record;
    rec->estimate = estimate;
    rec->errorest = errorest;
    rec->fin_i = fin_i;
    rec->fin_e = fin_e;
    rec->n_split = n_split;
    rec->bad = bad;
    rec->action = action;
    __threadfence_system();
    rec->seq = a.seq;
  }
}

}  // namespace pcb
