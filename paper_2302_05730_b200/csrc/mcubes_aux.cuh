// m-Cubes auxiliary kernels (not templated on the integrand): table merge, work-group trees,
// grid refinement (reference: mcubes.py:255-265, 292-298; vegas_grid.py:133-193).
#pragma once

#include "mcubes_kernels.cuh"
#include "pcb_device.cuh"

namespace pcb {

// CTA tables -> contribution table in a fixed order: a CTA owns 32 bins; thread (chunk c, bin i) adds the
// tables of blocks [c*per, (c+1)*per) serially, then the chunk sums of a bin are added in chunk order.
__device__ __forceinline__ void raw_stamp(unsigned long long* tl, bool who, int k) {
  if (tl && who && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tl[k] = t;
  }
}
// Asynchronous global -> shared copies: fire-and-forget, so a thread has a whole batch of loads in flight before it
// waits once (ptxas pairs plain loads with their additions two at a time -- 28 dependent round trips of ~0.25 us
// for a 56-table chunk -- whatever the source order).
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
constexpr int kReduceThreads = 256;
constexpr int kMergeChunks = kReduceThreads / 32;
constexpr int kMergeBatch = 32;   // table rows a thread keeps in flight (staged in shared memory: 8 B x 256 threads each)
constexpr int kGroupBatch = 8;    // (I, Var) pairs a thread keeps in flight
__host__ __device__ inline size_t reduce_parts_doubles(int pow2) {
  const size_t x = (size_t)kMergeChunks * 33 > (size_t)2 * pow2 ? (size_t)kMergeChunks * 33 : (size_t)2 * pow2;
  return (x + 1) & ~(size_t)1;
}
__host__ __device__ inline size_t reduce_smem_bytes(int pow2) {
  return (reduce_parts_doubles(pow2) + (size_t)kMergeBatch * kReduceThreads) * sizeof(double);
}
__device__ __forceinline__ void merge_hist_cta(int cta, const double* __restrict__ block_hist, int nblocks, int nbins_total,
                                               double* __restrict__ out, double* __restrict__ out_copy, double* s_part /* [kMergeChunks][33] */,
                                               double2* s_stage /* [kMergeBatch / 2][kReduceThreads] */) {
  const int lane = threadIdx.x & 31, c = threadIdx.x >> 5;
  const int i = cta * 32 + lane;
  const int per = (nblocks + kMergeChunks - 1) / kMergeChunks;
  const int b0 = c * per, b1 = min(nblocks, b0 + per);
  double t = 0.0;
  if ((nbins_total & 1) == 0) {
    // Rows are 16-B aligned: a warp fetches its chunk's rows two at a time with 16-byte copies that bypass L1 (lanes
    // 0-15 one row, lanes 16-31 the next; half the requests of the 8-byte form), kMergeBatch rows in flight, and
    // then every lane adds its bin over the rows in the same serial order as ever.
    double* rows = reinterpret_cast<double*>(s_stage) + (size_t)c * kMergeBatch * 32;   // this warp's [kMergeBatch][32]
    const int cnt = max(b1 - b0, 0), pair = (lane & 15) * 2, sub = lane >> 4;
    const bool fetch = cta * 32 + pair < nbins_total;
    for (int base = 0; base < cnt; base += kMergeBatch) {
      const int nbatch = min(kMergeBatch, cnt - base);
      for (int k = sub; k < nbatch; k += 2)
        if (fetch) cp_async16(rows + k * 32 + pair, block_hist + (size_t)(b0 + base + k) * nbins_total + cta * 32 + pair);
      cp_async_wait_all();
      __syncwarp();
      if (i < nbins_total)
        for (int k = 0; k < nbatch; ++k) {
          const double v = rows[k * 32 + lane];
          t = (base + k == 0) ? v : t + v;
        }
      __syncwarp();
    }
  } else if (i < nbins_total && b0 < b1) {
    // The kernel is bound by the latency of its loads (tables just written by other SMs), not by bandwidth: a thread
    // puts up to kMergeBatch rows of its chunk in flight, waits once and adds them in the same serial order as ever.
    const double* src = block_hist + (size_t)b0 * nbins_total + i;
    const int cnt = b1 - b0;
    double2* mine = s_stage + threadIdx.x;
    for (int base = 0; base < cnt; base += kMergeBatch) {
      const int nbatch = min(kMergeBatch, cnt - base);
      for (int k = 0; k < nbatch; ++k)
        cp_async8(reinterpret_cast<double*>(mine + (k >> 1) * kReduceThreads) + (k & 1), src + (size_t)(base + k) * nbins_total);
      cp_async_wait_all();
      int k = 0;
      for (; k + 1 < nbatch; k += 2) {
        const double2 v = mine[(k >> 1) * kReduceThreads];
        t = (base + k == 0) ? v.x : t + v.x;
        t = t + v.y;
      }
      if (k < nbatch) {
        const double v = mine[(k >> 1) * kReduceThreads].x;
        t = (base + k == 0) ? v : t + v;
      }
    }
  }
  s_part[c * 33 + lane] = t;
  __syncthreads();
  if (c == 0 && i < nbins_total) {
    double r = s_part[lane];
    const int used = (nblocks + per - 1) / per;
    for (int k = 1; k < used; ++k) r = r + s_part[k * 33 + lane];
    out[i] = r;
    if (out_copy) out_copy[i] = r;
  }
}

// per logical thread: serial sum of its segment partials; then the CTA reduces the work-group's threads with
// the adjacent-pair tree (mcubes.py:255-259).  group_out[g][0..1] = (I_g, E_g).  s: [2][pow2] doubles.
__device__ __forceinline__ void group_tree_cta(int group, const double* __restrict__ seg_partials, int nseg, long long n_local_threads,
                                               int group_size, int pow2, double* __restrict__ group_out, double* s, double2* s_stage) {
  const long long t0 = (long long)group * group_size;
  for (int i = threadIdx.x; i < pow2; i += blockDim.x) {
    double e = 0.0, v = 0.0;
    const long long t = t0 + i;
    if (i < group_size && t < n_local_threads) {
      // (I, Var) pairs of the thread's segments, kGroupBatch pairs in flight at a time, added in order
      const double2* src = reinterpret_cast<const double2*>(seg_partials) + t * nseg;
      double2* mine = s_stage + threadIdx.x;
      for (int base = 0; base < nseg; base += kGroupBatch) {
        const int nbatch = min(kGroupBatch, nseg - base);
        for (int k = 0; k < nbatch; ++k) cp_async16(mine + k * kReduceThreads, src + base + k);
        cp_async_wait_all();
        for (int k = 0; k < nbatch; ++k) {
          const double2 r = mine[k * kReduceThreads];
          e = (base + k == 0) ? r.x : e + r.x;
          v = (base + k == 0) ? r.y : v + r.y;
        }
      }
    }
    s[i] = e;
    s[pow2 + i] = v;
  }
  __syncthreads();
  for (int half = pow2 >> 1; half >= 1; half >>= 1) {
    // adjacent pairs: element i of the next level = s[2i] + s[2i+1]; done in place via a staging read
    double e[8], v[8];
    int cnt = 0;
    for (int i = threadIdx.x; i < half; i += blockDim.x, ++cnt) { e[cnt] = s[2 * i] + s[2 * i + 1]; v[cnt] = s[pow2 + 2 * i] + s[pow2 + 2 * i + 1]; }
    __syncthreads();
    cnt = 0;
    for (int i = threadIdx.x; i < half; i += blockDim.x, ++cnt) { s[i] = e[cnt]; s[pow2 + i] = v[cnt]; }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    group_out[2 * group] = s[0];
    group_out[2 * group + 1] = s[pow2];
  }
}

// One launch after the accumulation: CTAs [0, merge_ctas) merge the per-CTA tables into the contribution
// table (and into the run's per-iteration history slot), CTAs [merge_ctas, merge_ctas + n_groups) reduce one
// work-group each.
struct ReduceArgs {
  const int* stop;               // iteration at which the run stopped (INT_MAX while running); may be NULL
  int iteration;
  const double* block_hist;
  int nblocks, nbins_total, merge_ctas;
  double* contrib;
  double* contrib_copy;          // optional
  const double* seg_partials;
  int nseg, group_size, pow2;
  long long n_local_threads;
  double* group_out;
  unsigned long long* timeline;  // debug stamps or NULL
  // sharded runs: the pass scalars (first non-finite sample, clamp count) are copied behind the group pairs of this
  // rank's packed row, which the ranks then all-gather (NULL otherwise)
  const unsigned long long* pass_scalars;
  unsigned long long* row_tail;
};
__global__ void __launch_bounds__(kReduceThreads) reduce_kernel(const __grid_constant__ ReduceArgs a) {
  pdl_launch_dependents();
  tl_stamp(a.timeline, a.iteration, 1, 0);
  if (a.timeline && a.iteration == 1 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(a.timeline + 220, ~t);   // latest entry
  }
  pdl_wait();
  tl_stamp(a.timeline, a.iteration, 1, 1);
  if (a.timeline && a.iteration == 1 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(a.timeline + 221, ~t);   // latest return from the wait
  }
  if (a.stop && a.iteration > *a.stop) return;
  extern __shared__ __align__(16) double s_dyn[];  // reduce_smem_bytes(pow2): the parts / tree area, then the load staging
  double2* s_stage = reinterpret_cast<double2*>(s_dyn + reduce_parts_doubles(a.pow2));
  unsigned long long* ph = (a.timeline && a.iteration == 1) ? a.timeline + 210 : nullptr;
  raw_stamp(ph, blockIdx.x == 0, 0);
  raw_stamp(ph, (int)blockIdx.x == a.merge_ctas - 1, 2);
  raw_stamp(ph, (int)blockIdx.x == a.merge_ctas, 4);
  raw_stamp(ph, blockIdx.x == gridDim.x - 1, 6);
  if (a.row_tail && blockIdx.x == 0 && threadIdx.x == 0) {
    a.row_tail[0] = a.pass_scalars[0];
    a.row_tail[1] = a.pass_scalars[1];
  }
  if ((int)blockIdx.x < a.merge_ctas) {
    merge_hist_cta(blockIdx.x, a.block_hist, a.nblocks, a.nbins_total, a.contrib, a.contrib_copy, s_dyn, s_stage);
    raw_stamp(ph, blockIdx.x == 0, 1);
    raw_stamp(ph, (int)blockIdx.x == a.merge_ctas - 1, 3);
  } else {
    group_tree_cta(blockIdx.x - a.merge_ctas, a.seg_partials, a.nseg, a.n_local_threads, a.group_size, a.pow2, a.group_out, s_dyn, s_stage);
    raw_stamp(ph, (int)blockIdx.x == a.merge_ctas, 5);
    raw_stamp(ph, blockIdx.x == gridDim.x - 1, 7);
  }
  tl_stamp(a.timeline, a.iteration, 1, 2);
}

// final reduction of the per-work-group (I, E) pairs in group order with the pair tree of engine.tree_sum
// (mcubes.py:292-293), for up to 1024 groups in one CTA; returns (integral, variance sum) on thread 0.
// s: [2][1024] doubles; blockDim.x >= 512.
// `world` > 0: the pairs come from the all-gathered rows of a sharded run -- rank r owns groups
// [n*r/world, n*(r+1)/world) and its row starts at pairs + r*row_stride (group_shards in sharded.py).
__device__ __forceinline__ void group_pairs_tree_cta(const double* __restrict__ pairs, int n, double* s, double& integral, double& variance,
                                                     int world = 0, long long row_stride = 0) {
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
    const double* src = pairs + 2 * i;
    if (world > 0 && i < n) {
      const int r = (int)((((long long)i + 1) * world - 1) / n);          // owner of group i
      const long long first = (long long)n * r / world;
      src = pairs + r * row_stride + 2 * (i - first);
    }
    s[i] = i < n ? src[0] : 0.0;
    s[1024 + i] = i < n ? src[1] : 0.0;
  }
  __syncthreads();
  for (int half = 512; half >= 1; half >>= 1) {
    double e = 0.0, v = 0.0;
    const bool act = threadIdx.x < half;
    if (act) { e = s[2 * threadIdx.x] + s[2 * threadIdx.x + 1]; v = s[1024 + 2 * threadIdx.x] + s[1024 + 2 * threadIdx.x + 1]; }
    __syncthreads();
    if (act) { s[threadIdx.x] = e; s[1024 + threadIdx.x] = v; }
    __syncthreads();
  }
  integral = s[0];
  variance = s[1024];
}

// start of pcb_mcubes_run: uniform grid (init_grid, vegas_grid.py:77-84: k / n_bins), run not stopped, pass scalars armed
__global__ void run_init_kernel(int nb, double* __restrict__ bounds, int* __restrict__ stop, unsigned long long* __restrict__ scalars) {
  pdl_launch_dependents();
  double* row = bounds + (size_t)blockIdx.x * (nb + 1);
  for (int k = threadIdx.x; k <= nb; k += blockDim.x) row[k] = (double)k / (double)nb;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *stop = 0x7fffffff;
    scalars[0] = ~0ULL;   // M_BAD
    scalars[1] = 0ULL;    // M_CLAMPS
  }
}

// transform_many (vegas_grid.py:99-114) for caller-supplied points; flags[0] set on y outside [0,1)
__global__ void grid_transform_kernel(int d, int nb, const double* __restrict__ bnd, long long n, const double* __restrict__ y,
                                      double* __restrict__ x, double* __restrict__ jac, long long* __restrict__ bins, int* flags) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double jj = 1.0;
    for (int j = 0; j < d; ++j) {
      const double yy = y[i * d + j];
      if (!(yy >= 0.0 && yy < 1.0)) { flags[0] = 1; x[i * d + j] = yy; bins[i * d + j] = 0; continue; }
      const double z = yy * (double)nb;
      const double zi = __dadd_rz(z, 4503599627370496.0);
      int b = __double2loint(zi);
      const double frac = z - (zi - 4503599627370496.0);
      const double lo = bnd[j * (nb + 1) + b];
      const double w = bnd[j * (nb + 1) + b + 1] - lo;
      x[i * d + j] = lo + frac * w;
      const double jw = (double)nb * w;
      jj = (j == 0) ? jw : jj * jw;
      bins[i * d + j] = b;
    }
    jac[i] = jj;
  }
}

// sample_cube (mcubes.py:143-164), points: sample k of one sub-cube from caller-drawn uniforms u[k][j] --
// y = (coord + u) / g (IEEE division, mcubes.py:152), then transform_many.  One thread per sample.
__global__ void cube_points_kernel(int d, int nb, int p, long long cube, int g, const double* __restrict__ bnd,
                                   const double* __restrict__ u, double* __restrict__ x, double* __restrict__ jac,
                                   long long* __restrict__ bins) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= p) return;
  int coord[PCB_MAX_DIM];
  long long rem = cube;
  for (int j = d - 1; j >= 0; --j) { coord[j] = (int)(rem % g); rem /= g; }   // axis 0 most significant (mcubes.py:132-140)
  double jj = 1.0;
  for (int j = 0; j < d; ++j) {
    const double yy = __ddiv_rn((double)coord[j] + u[k * d + j], (double)g);
    const double z = yy * (double)nb;
    const double zi = __dadd_rz(z, 4503599627370496.0);
    int b = __double2loint(zi);
    b = b < nb ? b : nb - 1;
    const double frac = z - (zi - 4503599627370496.0);
    const double lo = bnd[j * (nb + 1) + b];
    const double w = bnd[j * (nb + 1) + b + 1] - lo;
    x[k * d + j] = lo + frac * w;
    const double jw = (double)nb * w;
    jj = (j == 0) ? jw : jj * jw;
    bins[k * d + j] = b;
  }
  jac[k] = jj;
}

// sample_cube, values: v = f(x) * jac, v^2, and the first non-finite sample (mcubes.py:154-162)
__global__ void cube_values_kernel(int p, const double* __restrict__ fx, const double* __restrict__ jac, double* __restrict__ v,
                                   double* __restrict__ v2, int* first_bad) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= p) return;
  const double f = fx[k];
  if (!isfinite(f)) atomicMin(first_bad, k);
  const double vv = f * jac[k];
  v[k] = vv;
  v2[k] = vv * vv;
}

__global__ void debug_divide_kernel(long long n, const double* __restrict__ x, double g, double rg, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = g > 0.0 ? div_by_const(x[i], g, rg) : rcp_normal(x[i]);
}

__global__ void deinterleave2_kernel(const double* __restrict__ in, int n, double* __restrict__ a, double* __restrict__ b) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) { a[i] = in[2 * i]; b[i] = in[2 * i + 1]; }
}

// ------------------------------------------------------------------------------------------
// refine_grid (vegas_grid.py:142-193): one CTA per axis.
// numpy's pairwise float sum of an n-vector restated for ONE WARP (all 32 lanes call it with the same
// arguments): numpy splits recursively down to blocks of <= 128 elements, sums a block with 8 strided
// accumulators combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) and adds the tail serially.  Lanes 0..7
// play the 8 accumulators (their chains are independent), the combine is three xor-shuffles.
// ------------------------------------------------------------------------------------------
// one block of numpy's pairwise sum (n <= 128), by one warp
__device__ __forceinline__ double np_block_sum_warp(const double* a, int n) {
  const int lane = threadIdx.x & 31;
  if (n < 8) {
    double r = 0.0;  // numpy starts from the first element; 0.0 + a[0] == a[0] for these inputs (a >= 0)
    for (int i = 0; i < n; ++i) r = (i == 0) ? a[0] : r + a[i];
    return r;
  }
  const int k = lane & 7, body = n - (n % 8);
  double r = a[k];
  int i = 8;
  for (; i + 24 < body; i += 32) {   // loads batched: only the DADD chain is exposed
    const double v0 = a[i + k], v1 = a[i + 8 + k], v2 = a[i + 16 + k], v3 = a[i + 24 + k];
    r = r + v0; r = r + v1; r = r + v2; r = r + v3;
  }
  for (; i < body; i += 8) r = r + a[i + k];
  r = r + __shfl_xor_sync(PCB_FULL_MASK, r, 1);
  r = r + __shfl_xor_sync(PCB_FULL_MASK, r, 2);
  r = r + __shfl_xor_sync(PCB_FULL_MASK, r, 4);
  for (int i = body; i < n; ++i) r = r + a[i];
  return r;
}

// The same sum by a whole CTA (every thread calls it; blockDim.x a multiple of 32, `a` in shared memory, n <= 4096),
// bit-identical to the warp version below.  numpy's recursion tree depends on n only: it is laid out level by level
// (a node of more than 128 elements splits at n/2 rounded down to a multiple of 8), its blocks are summed by
// different warps at the same time and the block sums are combined bottom-up in the tree's own association.  The
// recursive form costs ~5 us per 500-element sum (real calls with register spills, generic loads, one warp doing all
// blocks one after the other) -- two of them were two thirds of the grid refinement.
constexpr int kPwLevels = 6;                 // 4096 elements need at most 6 levels of splits
constexpr int kPwSlots = 1 << kPwLevels;
constexpr int kPwMaxN = 4096;
__device__ __forceinline__ double np_pairwise_sum_cta(const double* a, int n) {
  __shared__ int s_off[2][kPwSlots], s_len[2][kPwSlots];
  __shared__ unsigned char s_split[kPwLevels][kPwSlots / 2];
  __shared__ double s_val[kPwSlots];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  __syncthreads();   // the previous call's s_val[0] has been read by everybody
  if (tid == 0) { s_off[0][0] = 0; s_len[0][0] = n; }
  int levels = 0, cur = 0;
  for (;;) {
    __syncthreads();
    const int cnt = 1 << levels;
    int big = 0;
    if (tid < cnt) big = s_len[cur][tid] > 128;
    if (levels == kPwLevels || !__syncthreads_or(big)) break;
    if (tid < cnt) {
      const int o = s_off[cur][tid], l = s_len[cur][tid];
      int n2 = l / 2;
      n2 -= n2 % 8;
      s_split[levels][tid] = (unsigned char)big;
      s_off[cur ^ 1][2 * tid] = o;
      s_len[cur ^ 1][2 * tid] = big ? n2 : l;
      s_off[cur ^ 1][2 * tid + 1] = o + n2;
      s_len[cur ^ 1][2 * tid + 1] = big ? l - n2 : 0;   // 0: no right child, the node is carried down unchanged
    }
    cur ^= 1;
    ++levels;
  }
  const int cnt = 1 << levels;
  for (int slot = warp; slot < cnt; slot += nwarps) {
    const int l = s_len[cur][slot];
    if (l > 0) {
      const double r = np_block_sum_warp(a + s_off[cur][slot], l);
      if (lane == 0) s_val[slot] = r;
    }
  }
  __syncthreads();
  if (warp == 0) {
    for (int lev = levels - 1; lev >= 0; --lev) {
      double x = 0.0;
      if (lane < (1 << lev)) {
        x = s_val[2 * lane];
        if (s_split[lev][lane]) x = x + s_val[2 * lane + 1];
      }
      __syncwarp();
      if (lane < (1 << lev)) s_val[lane] = x;
      __syncwarp();
    }
  }
  __syncthreads();
  return s_val[0];
}

__device__ inline double np_pairwise_sum_warp(const double* a, int n) {
  if (n <= 128) return np_block_sum_warp(a, n);
  int n2 = n / 2;
  n2 -= n2 % 8;
  const double lo = np_pairwise_sum_warp(a, n2);
  const double hi = np_pairwise_sum_warp(a + n2, n - n2);
  return lo + hi;
}

struct RefineArgs {
  int d, n;
  double alpha;
  int smoothing;
  const double* boundaries;     // [d][n+1]
  const double* contrib;        // [d][n]
  double* new_boundaries;       // [d][n+1]
  unsigned long long* phase_tl = nullptr;  // debug: raw %globaltimer per phase of axis 0 (PCB_TIMELINE)
};
__device__ __forceinline__ void phase_stamp(unsigned long long* tl, int j, int k) {
  if (tl && j == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tl[k] = t;
  }
}

// index of element i in an array padded by one slot per 16 elements: a lane that walks a run of 16 consecutive
// elements then sits 17 doubles from its neighbour instead of 16 (= 128 B, i.e. all 32 lanes in the same banks)
__device__ __forceinline__ int pad16(int i) { return i + (i >> 4); }
__host__ __device__ inline size_t refine_smem_doubles(int n) {
  const size_t padded = (size_t)n + 1 + (size_t)(n + 1) / 16 + 1;
  return padded + (size_t)n + padded + (size_t)(n + 1) + 2;
}

// sh: refine_smem_doubles(n) doubles of shared memory; blockDim.x threads cooperate on axis j
__device__ __forceinline__ void refine_axis_cta(const RefineArgs& a, int j, double* sh) {
  const int n = a.n, tid = threadIdx.x;
  const int padded = n + 1 + (n + 1) / 16 + 1;
  double* c = sh;              // [n]   smoothed contributions; later the padded copy of w
  double* w = c + padded;      // [n]   damped weights
  double* cw = w + n;          // [n+1] cumulative weights, padded (pad16)
  double* row = cw + padded;   // [n+1] new boundaries
  double* s_scal = row + n + 1;  // [2] total, wsum
  const double* src = a.contrib + (size_t)j * n;
  const double* old = a.boundaries + (size_t)j * (n + 1);
  double* dst = a.new_boundaries + (size_t)j * (n + 1);

  phase_stamp(a.phase_tl, j, 0);
  int any = 0;
  for (int i = tid; i < n; i += blockDim.x) any |= (src[i] > 0.0);
  if (!__syncthreads_or(any)) {  // axis untouched (vegas_grid.py:156-157)
    for (int i = tid; i <= n; i += blockDim.x) dst[i] = old[i];
    return;
  }
  for (int i = tid; i < n; i += blockDim.x) {
    double v;
    if (a.smoothing && n >= 2) {
      if (i == 0) v = (src[0] + src[1]) / 2.0;
      else if (i == n - 1) v = (src[n - 2] + src[n - 1]) / 2.0;
      else v = (src[i - 1] + src[i] + src[i + 1]) / 3.0;
    } else {
      v = src[i];
    }
    c[i] = v;
  }
  __syncthreads();
  phase_stamp(a.phase_tl, j, 1);
  double total;
  if (n <= kPwMaxN) {
    total = np_pairwise_sum_cta(c, n);
  } else {
    if (tid < 32) {
      const double t = np_pairwise_sum_warp(c, n);
      if (tid == 0) s_scal[0] = t;
    }
    __syncthreads();
    total = s_scal[0];
  }
  phase_stamp(a.phase_tl, j, 2);
  for (int i = tid; i < n; i += blockDim.x) {
    const double r = c[i] / total;
    double ww = 0.0;
    if (r > 0.0 && r < 1.0) {
      const double base = (1.0 - r) / log(1.0 / r);
      // the default damping exponent 3/2 as x * sqrt(x) (both correctly rounded operations; pow() is ~10x the
      // instructions and itself only accurate to 1-2 ulp); any other exponent goes through pow
      ww = a.alpha == 1.5 ? base * sqrt(base) : pow(base, a.alpha);
    }
    else if (r >= 1.0) ww = 1.0;
    w[i] = ww;
  }
  __syncthreads();
  phase_stamp(a.phase_tl, j, 3);
  const double wsum_cta = n <= kPwMaxN ? np_pairwise_sum_cta(w, n) : 0.0;
  double* wp = c;   // c is dead: padded copy of w for the scan below
  for (int i = tid; i < n; i += blockDim.x) wp[pad16(i)] = w[i];
  __syncthreads();
  if (tid < 32) {
    const double wsum = n <= kPwMaxN ? wsum_cta : np_pairwise_sum_warp(w, n);
    if (tid == 0) s_scal[1] = wsum;
    // np.cumsum as a warp scan: lane l owns a run of consecutive bins (serial prefix inside the run, shuffle scan
    // across the runs).  The association differs from numpy's serial chain by rounding only (~1e-16 relative,
    // the boundaries are compared to 1e-12: log/sqrt are not numpy's either); a 500-long dependent DADD chain
    // would be a quarter of this kernel.
    const int per = (n + 31) / 32, i0 = tid * per, i1 = min(n, i0 + per);
    double run = 0.0;
    for (int i = i0; i < i1; ++i) run = (i == i0) ? wp[pad16(i)] : run + wp[pad16(i)];
    double incl = run;
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) {
      const double y = __shfl_up_sync(PCB_FULL_MASK, incl, m);
      if (tid >= m) incl = y + incl;
    }
    double acc = __shfl_up_sync(PCB_FULL_MASK, incl, 1);   // sum of the runs before mine
    if (tid == 0) acc = 0.0;
    for (int i = i0; i < i1; ++i) {
      acc = acc + wp[pad16(i)];
      cw[pad16(i + 1)] = acc;
    }
    if (tid == 0) cw[0] = 0.0;
    __syncwarp();
    if (tid == 0) cw[pad16(n)] = wsum;
  }
  __syncthreads();
  phase_stamp(a.phase_tl, j, 4);
  const double wsum = s_scal[1];
  if (!(wsum > 0.0)) {
    for (int i = tid; i <= n; i += blockDim.x) dst[i] = old[i];
    return;
  }
  for (int k = tid + 1; k < n; k += blockDim.x) {
    const double target = wsum * (double)k / (double)n;
    // searchsorted(cw, target, side="right") - 1, clipped to [0, n-1]
    int lo = 0, hi = n + 1;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (cw[pad16(mid)] <= target) lo = mid + 1; else hi = mid;
    }
    int idx = lo - 1;
    idx = idx < 0 ? 0 : (idx > n - 1 ? n - 1 : idx);
    const double cw_lo = cw[pad16(idx)];
    const double seg = cw[pad16(idx + 1)] - cw_lo;
    const double frac = seg > 0.0 ? (target - cw_lo) / seg : 0.0;
    row[k] = old[idx] + frac * (old[idx + 1] - old[idx]);
  }
  if (tid == 0) { row[0] = 0.0; row[n] = 1.0; }
  __syncthreads();
  phase_stamp(a.phase_tl, j, 5);
  // the serial repair below is a no-op unless some boundary collapsed: test that in parallel first
  int broken = 0;
  for (int k = tid + 1; k <= n; k += blockDim.x) broken |= (row[k] <= row[k - 1]);
  broken = __syncthreads_or(broken);
  if (broken && tid == 0) {  // restore strict monotonicity (vegas_grid.py:183-192)
    for (int k = 1; k <= n; ++k)
      if (row[k] <= row[k - 1]) row[k] = nextafter(row[k - 1], 2.0);
    if (row[n] != 1.0) {
      row[n] = 1.0;
      for (int k = n; k > 0; --k)
        if (row[k - 1] >= row[k]) row[k - 1] = nextafter(row[k], -1.0);
    }
  }
  __syncthreads();
  phase_stamp(a.phase_tl, j, 6);
  for (int i = tid; i <= n; i += blockDim.x) dst[i] = row[i];
  phase_stamp(a.phase_tl, j, 7);
}

__global__ void __launch_bounds__(512) refine_grid_kernel(const __grid_constant__ RefineArgs a) {
  extern __shared__ double sh[];
  refine_axis_cta(a, blockIdx.x, sh);
}

// ------------------------------------------------------------------------------------------
// End of an m-Cubes iteration, one launch: CTA j < n_refine refines axis j of the grid
// (vegas_grid.py:142-193); the last CTA finishes the group-order pair tree (mcubes.py:292-293),
// publishes the iteration record to pinned host memory, re-arms the pass scalars and decides
// whether the run has reached its tolerance (combine_iterations, mcubes.py:311-329).
// ------------------------------------------------------------------------------------------
struct McRecord {               // host-visible (pinned) record of one iteration
  double integral, variance;
  unsigned long long clamps, bad;
  int stop, pad;
  volatile unsigned long long seq;  // written last: run token << 20 | (iteration + 1)
};

struct FinishArgs {
  RefineArgs refine;
  int n_refine;                 // d when the grid adapts, else 0
  int* stop;                    // iteration at which the run stopped (INT_MAX while running); NULL outside pcb_mcubes_run
  const double* group_pairs;    // [n_groups][2]
  int n_groups;                 // <= 1024, or 0 when the sums are already in scalars[M_INTEGRAL..]
  unsigned long long* scalars;  // pass scalars: bad, clamps, integral, variance
  double* hist_i;               // run history of (integral, variance), capacity = iterations
  double* hist_v;
  int iteration;
  double rel_tol, abs_tol;
  McRecord* record;             // pinned host memory (nullptr: leave the results in scalars only)
  unsigned long long seq;
  unsigned long long* timeline; // debug stamps or NULL
  // sharded runs: group_pairs points at the all-gathered rows (world rows of row_stride doubles: the rank's group
  // pairs, then its first-non-finite index and clamp count); world = 0 otherwise
  int world;
  long long row_stride;
};

__global__ void __launch_bounds__(512) finish_kernel(const __grid_constant__ FinishArgs a) {
  // kernels of iteration `it` run iff it <= *stop, so the refinement CTAs of the stopping iteration itself are
  // unaffected by the decision taken by the last CTA of this very launch
  // no early trigger here: the next pass's CTAs must start together on an empty device.  Trickling in while this
  // kernel runs, they land unevenly on the SMs (the CTAs with one more unit batch share an SM) and the pass is 10 %
  // slower (measured with the device timeline).
  tl_stamp(a.timeline, a.iteration, 2, 0);
  pdl_wait();
  tl_stamp(a.timeline, a.iteration, 2, 1);
  if (a.stop && a.iteration > *a.stop) return;
  extern __shared__ double sh[];
  if ((int)blockIdx.x < a.n_refine) {
    refine_axis_cta(a.refine, blockIdx.x, sh);
    tl_stamp(a.timeline, a.iteration, 2, 2);
    return;
  }
  double integral, variance;
  double* sc_d = reinterpret_cast<double*>(a.scalars);
  if (a.n_groups > 0) {
    group_pairs_tree_cta(a.group_pairs, a.n_groups, sh, integral, variance, a.world, a.row_stride);
  } else {
    integral = sc_d[2];
    variance = sc_d[3];
  }
  if (threadIdx.x != 0) return;
  sc_d[2] = integral;
  sc_d[3] = variance;
  unsigned long long bad = a.scalars[0], clamps = a.scalars[1];
  if (a.world > 0) {   // every rank takes the same minimum / sum over the gathered rows
    bad = ~0ULL;
    clamps = 0ULL;
    for (int r = 0; r < a.world; ++r) {
      const unsigned long long* tail = reinterpret_cast<const unsigned long long*>(a.group_pairs + (r + 1) * a.row_stride) - 2;
      bad = tail[0] < bad ? tail[0] : bad;
      clamps += tail[1];
    }
  }
  int stop = bad != ~0ULL;
  if (a.hist_i) {
    const double var = fmax(variance, 0.0);
    a.hist_i[a.iteration] = integral;
    a.hist_v[a.iteration] = var;
    if (a.rel_tol > 0.0 || a.abs_tol > 0.0) {
      double wsum = 0.0, dot = 0.0;
      for (int i = 0; i <= a.iteration; ++i) {
        const double w = 1.0 / fmax(a.hist_v[i], 1e-30);
        wsum = wsum + w;
        dot = dot + w * a.hist_i[i];
      }
      const double est = dot / wsum, err = 1.0 / sqrt(wsum);
      if (err <= fmax(a.abs_tol, a.rel_tol * fabs(est))) stop = 1;
    }
    // re-arm the scalars for the next pass of the run
    a.scalars[0] = ~0ULL;
    a.scalars[1] = 0ULL;
  }
  if (a.record) {
    a.record->integral = integral;
    a.record->variance = variance;
    a.record->clamps = clamps;
    a.record->bad = bad;
    a.record->stop = stop;
    __threadfence_system();
    a.record->seq = a.seq;
  }
  if (a.stop && stop) {
    __threadfence();
    *a.stop = a.iteration;
  }
  tl_stamp(a.timeline, a.iteration, 2, 3);
}

}  // namespace pcb
