// m-Cubes V-Sample on the device (reference: mcubes.py:210-308, vegas_grid.py:99-114; arithmetic
// restated in SURVEY.md appendix A.4).
//
// Work decomposition: the reference's logical thread T owns sub-cubes [T*s, (T+1)*s) and RNG
// stream T.  A physical warp processes 32 logical threads at a time (lane <-> logical thread,
// lanes strided far apart in T so their sub-cubes sit in different grid bands), a segment of each
// thread's cube range per work unit (load balance for huge s).  Every draw is
// uniform(seed, T, (L*p + k)*d + j), so the sample set is identical to the reference's for any
// partition of threads over warps, segments or GPUs.
//
// The pass is two kernels:
//   vsample_kernel  pure compute at 16 warps/SM: hash -> stratified y -> grid transform -> f -> per-cube
//                   (S1, S2, estimate, variance); it emits one compact record per sample
//                   (contribution, d bin ids) to HBM instead of touching a histogram;
//   bin_kernel      streams the records and accumulates the (d x n_bins) contribution table.
// Shared-memory FP64 atomicAdd is a CAS loop on sm_100 (ATOMS.CAST.SPIN), so in bin_kernel each warp
// owns a private table in shared memory, arbitrates intra-warp collisions with one tag round and lets
// the few losers use the CAS atomic; tables are merged warp -> CTA -> grid in a fixed order.
// Keeping the table out of the sampling kernel is what lifts it from 5 to 16 resident warps per SM.
#pragma once

#include "pcb_device.cuh"

namespace pcb {

// x / d and x % d for a loop-invariant d by one multiply-high (m = floor(2^64 / d)): the quotient estimate is
// at most 2 short, fixed by the loop.  64-bit division is ~100 instructions on this part and the per-unit
// setup of a small pass would otherwise cost as much as one sample.
struct FastDiv {
  unsigned long long d, m;
};
__host__ inline FastDiv make_fastdiv(unsigned long long d) {
  FastDiv f;
  f.d = d;
  f.m = d <= 1 ? ~0ULL : (unsigned long long)((((unsigned __int128)1) << 64) / d);
  return f;
}
__device__ __forceinline__ unsigned long long fast_divmod(unsigned long long x, const FastDiv& f, unsigned long long& rem) {
  unsigned long long q = __umul64hi(x, f.m);
  unsigned long long r = x - q * f.d;
  while (r >= f.d) { r -= f.d; ++q; }
  rem = r;
  return q;
}

struct SampleArgs {
  pcb_integrand f;
  int g, p, nb, squared_weighted;
  long long m, s;
  long long n_threads;          // logical threads of the whole plan
  long long t_begin, t_end;     // this launch's shard of logical threads
  // Work item = segment sigma = (T - t_begin) * nseg + q of seg_len sub-cubes; lane l of unit u takes
  // sigma = ((u * 32 + l) * seg_mul) mod n_segments.  The multiplier spreads the 32 lanes of a warp over
  // different sub-cube coordinates on EVERY axis (lane-to-lane offset ~ (1,1,...,1) in base g), so their
  // samples fall into different windows of the importance grid and rarely collide in the accumulation.
  long long n_segments;         // (t_end - t_begin) * nseg
  unsigned long long seg_mul;   // coprime to n_segments
  FastDiv div_segments, div_nseg, div_g;
  int nseg;                     // segments per logical thread
  int rng_kind;
  long long seg_len;
  unsigned long long seed;
  const double* injected;       // PCB_RNG_INJECTED: table[(cube*p + k)*d + j]
  const double* boundaries;     // [d][nb+1]
  double gd, rg;                // (double)g and RN(1/g)
  double den_est, den_var;      // p*m and p*(p-1)*m*m, exact integers rounded once (mcubes.py:247-248)
  double* seg_partials;         // [(t - t_begin) * nseg + q][2]
  unsigned long long* clamps;
  unsigned long long* bad;      // min over non-finite samples of cube*p + k
  // sample records of this launch's units [unit_begin, unit_end): record r of unit u sits at
  // (u - unit_begin) * rec_per_unit + r with r = (cube_step * p + k) * 32 + lane
  long long unit_begin, unit_end, rec_per_unit, rec_capacity;
  double* rec_w;                // [rec_capacity] contribution (v^2, or f^2 when not squared_weighted)
  unsigned short* rec_b;        // [d][rec_capacity] bin ids
  const int* stop;              // iteration at which the run stopped (INT_MAX while running); may be NULL
  int iteration;
};

struct BinArgs {
  int nb;
  long long n_groups;           // record groups of 32
  long long rec_capacity;
  const double* rec_w;
  const unsigned short* rec_b;
  double* block_hist;           // [gridDim.x][d*nb], accumulated across launches
  int accumulate;               // 0: overwrite block_hist, 1: add to it
  const int* stop;
  int iteration;
};

// One sample: draw u per axis, stratify, push through the grid, evaluate (mcubes.py:224-243).
template <class F, int D, int RNG>
__device__ __forceinline__ void draw_sample(const SampleArgs& a, const double* s_b, const double (&coord)[D],
                                            unsigned long long kc, unsigned long long T, unsigned long long ctr,
                                            unsigned long long inj_base, bool active, int (&bin)[D], double& fx,
                                            double& v) {
  const int nb = a.nb, nb1 = a.nb + 1;
  const double nbd = (double)nb;
  double x[D];
  double jac = 1.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    double uu;
    if constexpr (RNG == PCB_RNG_REFERENCE_HASH) {
      uu = u53_to_unit(mix64(kc + (unsigned long long)j * kGolden));
    } else {
      if (a.rng_kind == PCB_RNG_PHILOX) uu = philox_uniform(a.seed, T, ctr + j);
      else uu = active ? a.injected[inj_base + j] : 0.5;
    }
    const double y = div_by_const(coord[j] + uu, a.gd, a.rg);   // (coord + u) / g
    const double z = y * nbd;
    const double zi = __dadd_rz(z, 4503599627370496.0);         // 2^52 + floor(z)
    int b = __double2loint(zi);
    b = b < nb ? b : nb - 1;
    const double frac = z - (zi - 4503599627370496.0);
    const double lo = s_b[j * nb1 + b];
    const double wd = s_b[j * nb1 + b + 1] - lo;
    x[j] = lo + frac * wd;
    const double jw = nbd * wd;
    jac = (j == 0) ? jw : jac * jw;
    bin[j] = b;
  }
  fx = eval_at<F, D>(x, a.f);
  v = fx * jac;
}

constexpr int kSampleWarps = 8;  // warps per sampling CTA; two CTAs per SM at 128 registers

template <int FAM, int D, int RNG>
__global__ void __launch_bounds__(kSampleWarps * 32, 2) vsample_kernel(const __grid_constant__ SampleArgs a) {
  using F = Family<FAM>;
  if (a.stop && a.iteration > *a.stop) return;  // run already converged: a speculatively enqueued pass is a no-op
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nb1 = a.nb + 1;
  double* s_b = reinterpret_cast<double*>(smem_raw);            // [D][nb+1]
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < D * nb1; i += blockDim.x) s_b[i] = a.boundaries[i];
  __syncthreads();

  const int p = a.p;
  const double pd = (double)p;
  unsigned long long clamp_count = 0;

  for (long long u = a.unit_begin + (long long)blockIdx.x * kSampleWarps + wib; u < a.unit_end;
       u += (long long)gridDim.x * kSampleWarps) {
    const unsigned long long sin = (unsigned long long)u * 32ULL + (unsigned long long)lane;
    const bool live = sin < (unsigned long long)a.n_segments;
    unsigned long long sigma = 0, qq_seg = 0;
    if (live) fast_divmod(sin * a.seg_mul, a.div_segments, sigma);
    const long long T = a.t_begin + (long long)fast_divmod(sigma, a.div_nseg, qq_seg);
    const int q = (int)qq_seg;
    long long c_begin = 0, count = 0;
    if (live) {
      const long long l0 = (long long)q * a.seg_len;
      long long l1 = l0 + a.seg_len;
      if (l1 > a.s) l1 = a.s;
      c_begin = T * a.s + l0;
      long long c_end = T * a.s + l1;
      if (c_end > a.m) c_end = a.m;
      count = c_end > c_begin ? c_end - c_begin : 0;
    }
    // sub-cube coordinates (axis 0 most significant, mcubes.py:132-140), kept as doubles
    double coord[D];
    {
      unsigned long long rem = (unsigned long long)c_begin;
#pragma unroll
      for (int j = D - 1; j >= 0; --j) {
        unsigned long long digit;
        rem = fast_divmod(rem, a.div_g, digit);
        coord[j] = (double)(int)digit;
      }
    }
    const unsigned long long key = stream_key(a.seed, (unsigned long long)T);
    // hash input key + (counter+1)*GOLDEN for counter = (L*p + k)*D + j, advanced incrementally
    unsigned long long ctr = (unsigned long long)(q * a.seg_len) * (unsigned long long)p * D;
    unsigned long long kc = key + (ctr + 1ULL) * kGolden;
    double sum_est = 0.0, sum_var = 0.0;
    double* rw = a.rec_w + (u - a.unit_begin) * a.rec_per_unit + lane;
    unsigned short* rb = a.rec_b + (u - a.unit_begin) * a.rec_per_unit + lane;

    // every lane walks the full segment so that the record block of the unit is completely written;
    // lanes past their own cube range emit empty records
    for (long long i = 0; i < a.seg_len; ++i) {
      const bool active = i < count;
      const unsigned long long inj_cube = (unsigned long long)(c_begin + i) * (unsigned long long)p;
      double s1 = 0.0, s2 = 0.0;
      int k = 0;
      // two samples at a time: independent dependency chains keep the FP64 and integer pipes busy
      if constexpr (RNG == PCB_RNG_REFERENCE_HASH)
      for (; k + 1 < p; k += 2) {
        int bin[2][D];
        double fx[2], v[2];
        draw_sample<F, D, RNG>(a, s_b, coord, kc, (unsigned long long)T, ctr, (inj_cube + k) * D, active, bin[0], fx[0], v[0]);
        draw_sample<F, D, RNG>(a, s_b, coord, kc + (unsigned long long)D * kGolden, (unsigned long long)T, ctr + D,
                               (inj_cube + k + 1) * D, active, bin[1], fx[1], v[1]);
        kc += 2ULL * D * kGolden;
        ctr += 2 * D;
        if (active && !(isfinite(fx[0]) && isfinite(fx[1])))
          atomicMin(a.bad, inj_cube + (unsigned long long)k + (isfinite(fx[0]) ? 1ULL : 0ULL));
        const double v2[2] = {v[0] * v[0], v[1] * v[1]};
        // sample order (numpy's order for p < 8, mcubes.py:245-246; from p = 8 on numpy uses an
        // 8-accumulator tree -- only the rounding differs)
        s1 = (k == 0) ? v[0] + v[1] : (s1 + v[0]) + v[1];
        s2 = (k == 0) ? v2[0] + v2[1] : (s2 + v2[0]) + v2[1];
#pragma unroll
        for (int q2 = 0; q2 < 2; ++q2) {
          const long long r = (i * p + k + q2) * 32;
          rw[r] = active ? (a.squared_weighted ? v2[q2] : fx[q2] * fx[q2]) : 0.0;
#pragma unroll
          for (int j = 0; j < D; ++j) rb[(long long)j * a.rec_capacity + r] = (unsigned short)bin[q2][j];
        }
      }
      for (; k < p; ++k) {
        int bin[D];
        double fx, v;
        draw_sample<F, D, RNG>(a, s_b, coord, kc, (unsigned long long)T, ctr, (inj_cube + k) * D, active, bin, fx, v);
        kc += (unsigned long long)D * kGolden;
        ctr += D;
        if (active && !isfinite(fx)) atomicMin(a.bad, inj_cube + (unsigned long long)k);
        const double v2 = v * v;
        s1 = (k == 0) ? v : s1 + v;
        s2 = (k == 0) ? v2 : s2 + v2;
        const long long r = (i * p + k) * 32;
        rw[r] = active ? (a.squared_weighted ? v2 : fx * fx) : 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) rb[(long long)j * a.rec_capacity + r] = (unsigned short)bin[j];
      }
      if (active) {
        const double est = s1 / a.den_est;
        const double raw = (s2 - s1 * s1 / pd) / a.den_var;
        if (raw < 0.0) ++clamp_count;
        const double var = fmax(raw, 0.0);
        sum_est = (i == 0) ? est : sum_est + est;
        sum_var = (i == 0) ? var : sum_var + var;
      }
      // odometer: next sub-cube
#pragma unroll
      for (int j = D - 1; j >= 0; --j) {
        coord[j] = coord[j] + 1.0;
        if (coord[j] < a.gd) break;
        coord[j] = 0.0;
      }
    }
    if ((a.seg_len * p) & 1) {  // units hold an even number of 32-record groups: blank the padding group
      const long long r = a.seg_len * p * 32;
      rw[r] = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) rb[(long long)j * a.rec_capacity + r] = 0;
    }
    if (live) {
      double* out = a.seg_partials + sigma * 2;
      out[0] = sum_est;
      out[1] = sum_var;
    }
  }
  if (clamp_count) atomicAdd(a.clamps, clamp_count);
}

}  // namespace pcb
