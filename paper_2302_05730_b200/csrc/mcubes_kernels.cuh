// m-Cubes V-Sample and grid refinement on the device (reference: mcubes.py:210-308,
// vegas_grid.py:99-193; arithmetic restated in SURVEY.md appendix A.4).
//
// Work decomposition: the reference's logical thread T owns sub-cubes [T*s, (T+1)*s) and RNG
// stream T.  A physical warp processes 32 logical threads at a time (lane <-> logical thread,
// lanes strided far apart in T so their sub-cubes sit in different grid bands), optionally only
// a segment of each thread's cube range (load balance for huge s).  Every draw is
// uniform(seed, T, (L*p + k)*d + j), so the sample set is identical to the reference's for any
// partition of threads over warps, segments or GPUs.
//
// Bin contributions: shared-memory FP64 atomicAdd is a CAS loop on sm_100 (ATOMS.CAST.SPIN), so
// each warp owns a private (d x n_bins) table in shared memory and resolves intra-warp collisions
// with a tag-and-retry round; tables are merged warp -> CTA -> grid in a fixed order.
#pragma once

#include "pcb_device.cuh"

namespace pcb {

struct SampleArgs {
  pcb_integrand f;
  int g, p, nb, squared_weighted;
  long long m, s;
  long long n_threads;          // logical threads of the whole plan
  long long t_begin, t_end;     // this launch's shard of logical threads
  long long n_lw;               // logical warps in the shard = ceil((t_end - t_begin) / 32)
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
  double* block_hist;           // [gridDim.x][d*nb]
};

// Add one or two samples' contributions to the warp-private table.  One tag round arbitrates lanes
// that hit the same bin: every contender writes its lane id, whoever reads its own id back owns the
// bin and does a plain read-modify-write.  The few losers (about one lane per axis) then add theirs
// with the shared-memory CAS atomic, which is only slow when many lanes use it.  When both samples of
// a lane fall into the same bin their contributions are merged into one update.
template <int D, int NS>
__device__ __forceinline__ void hist_add(double* hist, unsigned char* tags, const int (&bin)[NS][D], int nb,
                                         const double (&w2)[NS], bool on, int lane) {
  int off[NS][D];
  double add[NS][D];
  bool use[NS][D];
#pragma unroll
  for (int j = 0; j < D; ++j) {
    off[0][j] = j * nb + bin[0][j];
    add[0][j] = w2[0];
    use[0][j] = on;
    if constexpr (NS == 2) {
      off[1][j] = j * nb + bin[1][j];
      const bool same = bin[1][j] == bin[0][j];
      add[0][j] = same ? w2[0] + w2[1] : w2[0];
      add[1][j] = w2[1];
      use[1][j] = on && !same;
    }
  }
#pragma unroll
  for (int q = 0; q < NS; ++q)
#pragma unroll
    for (int j = 0; j < D; ++j)
      if (use[q][j]) tags[off[q][j]] = (unsigned char)lane;
  __syncwarp();
  unsigned lost = 0;
#pragma unroll
  for (int q = 0; q < NS; ++q)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const bool win = use[q][j] && tags[off[q][j]] == lane;
      const double updated = hist[off[q][j]] + add[q][j];
      if (win) hist[off[q][j]] = updated;
      lost |= (use[q][j] && !win) ? (1u << (q * D + j)) : 0u;
    }
  __syncwarp();
  if (__any_sync(PCB_FULL_MASK, lost)) {
#pragma unroll
    for (int q = 0; q < NS; ++q)
#pragma unroll
      for (int j = 0; j < D; ++j)
        if ((lost >> (q * D + j)) & 1u) atomicAdd(hist + off[q][j], add[q][j]);
    __syncwarp();
  }
}

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

// warps per CTA are bounded by shared memory (one private table each); from d = 4 on at most 8 fit usefully,
// which lets the compiler use up to 255 registers for the two-sample interleave
__host__ __device__ constexpr int vsample_max_warps(int d) { return d >= 4 ? 8 : 16; }

template <int FAM, int D, int RNG>
__global__ void __launch_bounds__(vsample_max_warps(D) * 32) vsample_kernel(const __grid_constant__ SampleArgs a) {
  using F = Family<FAM>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nb = a.nb, nb1 = a.nb + 1;
  const int W = blockDim.x >> 5;
  double* s_b = reinterpret_cast<double*>(smem_raw);            // [D][nb+1]
  double* s_hist = s_b + D * nb1;                               // [W][D*nb]
  unsigned char* s_tag = reinterpret_cast<unsigned char*>(s_hist + (size_t)W * D * nb);  // [W][D*nb]
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;

  for (int i = threadIdx.x; i < D * nb1; i += blockDim.x) s_b[i] = a.boundaries[i];
  for (int i = threadIdx.x; i < W * D * nb; i += blockDim.x) s_hist[i] = 0.0;
  __syncthreads();
  double* hist = s_hist + (size_t)wib * D * nb;
  unsigned char* tags = s_tag + (size_t)wib * D * nb;

  const long long n_units = a.n_lw * a.nseg;
  const int p = a.p;
  const double pd = (double)p;
  unsigned long long clamp_count = 0;

  for (long long u = (long long)blockIdx.x * W + wib; u < n_units; u += (long long)gridDim.x * W) {
    const long long lw = u % a.n_lw;
    const int q = (int)(u / a.n_lw);
    const long long T = a.t_begin + lw + (long long)lane * a.n_lw;
    long long c_begin = 0, count = 0;
    if (T < a.t_end) {
      const long long l0 = (long long)q * a.seg_len;
      long long l1 = l0 + a.seg_len;
      if (l1 > a.s) l1 = a.s;
      c_begin = T * a.s + l0;
      long long c_end = T * a.s + l1;
      if (c_end > a.m) c_end = a.m;
      count = c_end > c_begin ? c_end - c_begin : 0;
    }
    long long max_count = count;
#pragma unroll
    for (int mm = 16; mm >= 1; mm >>= 1) {
      long long o = __shfl_xor_sync(PCB_FULL_MASK, max_count, mm);
      max_count = o > max_count ? o : max_count;
    }
    // sub-cube coordinates (axis 0 most significant, mcubes.py:132-140), kept as doubles
    double coord[D];
    {
      long long rem = c_begin;
#pragma unroll
      for (int j = D - 1; j >= 0; --j) {
        long long qq = rem / a.g;
        coord[j] = (double)(rem - qq * a.g);
        rem = qq;
      }
    }
    const unsigned long long key = stream_key(a.seed, (unsigned long long)T);
    // hash input key + (counter+1)*GOLDEN for counter = (L*p + k)*D + j, advanced incrementally
    unsigned long long ctr = (unsigned long long)(q * a.seg_len) * (unsigned long long)p * D;
    unsigned long long kc = key + (ctr + 1ULL) * kGolden;
    double sum_est = 0.0, sum_var = 0.0;

    for (long long i = 0; i < max_count; ++i) {
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
        const double w2[2] = {a.squared_weighted ? v2[0] : fx[0] * fx[0], a.squared_weighted ? v2[1] : fx[1] * fx[1]};
        hist_add<D, 2>(hist, tags, bin, nb, w2, active, lane);
      }
      for (; k < p; ++k) {
        int bin[1][D];
        double fx, v;
        draw_sample<F, D, RNG>(a, s_b, coord, kc, (unsigned long long)T, ctr, (inj_cube + k) * D, active, bin[0], fx, v);
        kc += (unsigned long long)D * kGolden;
        ctr += D;
        if (active && !isfinite(fx)) atomicMin(a.bad, inj_cube + (unsigned long long)k);
        const double v2 = v * v;
        s1 = (k == 0) ? v : s1 + v;
        s2 = (k == 0) ? v2 : s2 + v2;
        const double w2[1] = {a.squared_weighted ? v2 : fx * fx};
        hist_add<D, 1>(hist, tags, bin, nb, w2, active, lane);
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
    if (T < a.t_end) {
      double* out = a.seg_partials + ((T - a.t_begin) * a.nseg + q) * 2;
      out[0] = sum_est;
      out[1] = sum_var;
    }
  }
  if (clamp_count) atomicAdd(a.clamps, clamp_count);
  __syncthreads();
  // warp tables -> CTA table, fixed warp order
  double* dst = a.block_hist + (size_t)blockIdx.x * D * nb;
  for (int i = threadIdx.x; i < D * nb; i += blockDim.x) {
    double t = s_hist[i];
    for (int w = 1; w < W; ++w) t = t + s_hist[(size_t)w * D * nb + i];
    dst[i] = t;
  }
}

}  // namespace pcb
