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
// The pass is ONE kernel.  A CTA (8 warps) works in rounds, and in every round each warp does two things at once:
//   draw      two samples per lane (hash -> stratified y -> grid transform -> f -> per-cube S1, S2, estimate,
//             variance), staged as one record per sample -- contribution and D bin ids -- in shared memory;
//   bin       warp w serves axis w (w + 8 for D > 8): it adds the records the CTA staged in the PREVIOUS round to
//             ITS private row of the contribution table (n_bins doubles in shared memory).  Shared-memory FP64
//             atomicAdd is a CAS loop on sm_100 (ATOMS.CAST.SPIN), so same-bin lanes are arbitrated by a tag round
//             (the winner does a plain read-modify-write); a loser keeps its record in a one-deep pending slot that
//             takes part in its next call (d >= 7) or is flushed at the end of the round (d <= 6); a second loss
//             before the slot is free uses the CAS atomic (bin_pair_carry / bin_pair_flush below).
// The staging is double-buffered and the accumulation is dealt over the axis steps of the draw as straight-line
// code, so the shared-memory round trips of `bin` hide behind the integer / FP64 arithmetic of `draw` inside every
// warp; one barrier per round.  No sample record ever travels to HBM.  Rows are merged CTA -> grid in a fixed
// order (reduce_kernel).  The ORDER in which same-bin contributions of one warp are added is decided by which
// lane's tag store lands last (and, for the rare CAS path, by the order of the compare-and-swaps): fixed by the
// hardware for a given launch configuration -- the tests find the table bit-reproducible run to run on the B200 --
// but not by the CUDA memory model.  The contract is therefore "contribution table to summation order" (1e-12
// against the reference); (integral, variance), which never pass through this path, are bit-reproducible by design.
#pragma once

#include <type_traits>

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

// the same for 32-bit operands (m = floor(2^32 / d)): sub-cube indices below 2^32 take their base-g digits this way
__device__ __forceinline__ unsigned fast_divmod32(unsigned x, unsigned d, unsigned m, unsigned& rem) {
  unsigned q = __umulhi(x, m);
  unsigned r = x - q * d;
  while (r >= d) { r -= d; ++q; }
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
  unsigned g_m32;               // floor(2^32 / g) when m < 2^32 (digits by 32-bit arithmetic), else 0
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
  long long n_units;            // work units (32 segments each)
  double* block_hist;           // [gridDim.x][d*nb]: the CTA's rows of the contribution table
  const int* stop;              // iteration at which the run stopped (INT_MAX while running); may be NULL
  int iteration;
  unsigned long long* timeline; // debug stamps (tl_stamp) or NULL
};

// One axis of one sample: draw u, stratify, push through the grid (mcubes.py:224-236, vegas_grid.py:99-114).
template <int RNG>
__device__ __forceinline__ void draw_axis(const SampleArgs& a, const double* s_b, int j, double coord_j,
                                          unsigned long long kc, unsigned long long T, unsigned long long ctr,
                                          unsigned long long inj_base, bool active, double& xj, double& jac, int& bin_j) {
  const int nb = a.nb, nb1 = a.nb + 1;
  const double nbd = (double)nb;
  double uu;
  if constexpr (RNG == PCB_RNG_REFERENCE_HASH) {
    uu = u53_to_unit(mix64(kc + (unsigned long long)j * kGolden));
  } else {
    if (a.rng_kind == PCB_RNG_PHILOX) uu = philox_uniform(a.seed, T, ctr + j);
    else uu = active ? a.injected[inj_base + j] : 0.5;
  }
  const double y = div_by_const(coord_j + uu, a.gd, a.rg);   // (coord + u) / g
  const double z = y * nbd;
  const double zi = __dadd_rz(z, 4503599627370496.0);         // 2^52 + floor(z)
  int b = __double2loint(zi);
  b = b < nb ? b : nb - 1;
  const double frac = z - (zi - 4503599627370496.0);
#ifdef PCB_EXP_NOCONFLICT_B   // experiment (wrong results): what would conflict-free boundary gathers buy?
  const int bb = (b & ~15) | (int)(threadIdx.x & 15);
  const double lo = s_b[j * nb1 + (bb < nb ? bb : b)];
  const double wd = s_b[j * nb1 + (bb < nb ? bb : b) + 1] - lo;
#else
  const double lo = s_b[j * nb1 + b];
  const double wd = s_b[j * nb1 + b + 1] - lo;
#endif
  xj = lo + frac * wd;
  const double jw = nbd * wd;
  jac = (j == 0) ? jw : jac * jw;
  bin_j = b;
}

#ifndef PCB_SAMPLE_WARPS
#define PCB_SAMPLE_WARPS 8
#endif
constexpr int kSampleWarps = PCB_SAMPLE_WARPS;  // warps per CTA; two CTAs per SM at 128 registers
constexpr int kSlot = kSampleWarps * 32;   // records per staged sample slot

// shared memory of one CTA: boundaries, one table row + tag bytes per axis, the staged records of TWO rounds
// (the round being drawn and the round being added to the rows)
__host__ __device__ inline size_t vsample_stage_bytes(int d) { return (size_t)2 * kSlot * 8 + (size_t)d * 2 * kSlot * 2; }
__host__ __device__ inline size_t vsample_smem_bytes(int d, int nb) {
  const size_t tags = (size_t)((nb + 15) & ~15);
  return (size_t)d * (nb + 1) * 8 + 8 /* pad */ + (size_t)d * ((size_t)nb * 8 + tags) + 2 * vsample_stage_bytes(d);
}

// Add two staged records per lane into the warp's private row (see the header comment).  Straight-line code: the
// caller interleaves it with the arithmetic of the round being drawn, which hides the shared-memory round trips.
// One arbitration round per call: same-bin lanes are arbitrated by a tag store (exactly one lane reads its own id
// back per bin), the winner does a plain read-modify-write whose LOAD is issued together with the tag load (the
// row entry is fetched speculatively: one shared-memory round trip less on the dependent chain), and a lane that
// lost keeps its record in a one-deep pending slot (`pend_b` < 0: empty), which simply takes part in the lane's
// next call as a third candidate -- no second arbitration round, no vote, no loop.  (Until round 2 of this build
// every call ran a second, mostly idle arbitration round plus a vote: 43 % of the pass's stall samples sat on those
// dependent round trips, profiles/r2_ncu_vsample_config4_before.txt.)  A lane that loses while its slot is still
// occupied -- a few calls in a hundred warp-wide -- falls back to the CAS atomic.
__device__ __forceinline__ void bin_pair_carry(double* __restrict__ hist, unsigned char* __restrict__ tags, int lane, double w0, int b0,
                                         double w1, int b1, int& pend_b, double& pend_w) {
#ifdef PCB_EXP_NOCONFLICT_H   // experiment (wrong results): conflict-free table and tag accesses
  b0 = (b0 & ~31) | lane; b1 = ((b1 & ~31) | lane) ^ 32;
  if (b0 >= 480) b0 = lane; if (b1 >= 480) b1 = lane + 32;
#endif
  // a zero contribution leaves the table unchanged: skip it (empty records, f = 0 samples);
  // records of one lane in the same bin become one update
  const bool same = b0 == b1;
  double add0 = same ? w0 + w1 : w0;
  double add1 = w1;
  const bool hit0 = pend_b == b0, hit1 = !same && pend_b == b1;   // the pending record meets a new one of its own lane
  add0 = hit0 ? add0 + pend_w : add0;
  add1 = hit1 ? add1 + pend_w : add1;
  const bool wantp = pend_b >= 0 && !hit0 && !hit1;
  const bool want0 = add0 != 0.0, want1 = !same && add1 != 0.0;
  const int bp = wantp ? pend_b : b0;                  // always a valid bin: the loads below are unconditional
  if (wantp) tags[bp] = (unsigned char)lane;
  if (want0) tags[b0] = (unsigned char)lane;
  if (want1) tags[b1] = (unsigned char)lane;
  __syncwarp();
  const double hp = hist[bp], h0 = hist[b0], h1 = hist[b1];   // speculative: only a winner uses its value
  const unsigned char tp = tags[bp], t0 = tags[b0], t1 = tags[b1];
  const bool winp = wantp && tp == lane, win0 = want0 && t0 == lane, win1 = want1 && t1 == lane;
  if (winp) hist[bp] = hp + pend_w;
  if (win0) hist[b0] = h0 + add0;
  if (win1) hist[b1] = h1 + add1;
  __syncwarp();
  const bool lostp = wantp && !winp, lost0 = want0 && !win0, lost1 = want1 && !win1;
  const bool ovf0 = lostp && lost0, ovf1 = lost1 && (lostp || lost0);
  pend_w = lostp ? pend_w : (lost0 ? add0 : add1);
  pend_b = lostp ? pend_b : (lost0 ? b0 : (lost1 ? b1 : -1));
  if (ovf0 || ovf1) {
    if (ovf0) atomicAdd(hist + b0, add0);
    if (ovf1) atomicAdd(hist + b1, add1);
  }
}

// The same with the pending slot emptied at the end of every round (flush_pending) instead of taking part in the next
// call: two candidates per call, fewer live registers -- the form the 80-register kernels (D <= 6, three CTAs per
// SM) take, where the third candidate spills (d = 6, 9.6e8 samples: 31.4 ms against 34.2 ms; d >= 7 at 128
// registers prefers the carried form: d = 8 33.9 against 34.9 ms, d = 10 62.7 against 65.6 ms).
__device__ __forceinline__ void bin_pair_flush(double* __restrict__ hist, unsigned char* __restrict__ tags, int lane, double w0, int b0,
                                               double w1, int b1, int& pend_b, double& pend_w) {
  const bool same = b0 == b1;
  const double add0 = same ? w0 + w1 : w0, add1 = w1;
  const bool want0 = add0 != 0.0, want1 = !same && add1 != 0.0;
  if (want0) tags[b0] = (unsigned char)lane;
  if (want1) tags[b1] = (unsigned char)lane;
  __syncwarp();
  const double h0 = hist[b0], h1 = hist[b1];           // speculative: only a winner uses its value
  const bool win0 = want0 && tags[b0] == lane, win1 = want1 && tags[b1] == lane;
  if (win0) hist[b0] = h0 + add0;
  if (win1) hist[b1] = h1 + add1;
  __syncwarp();
  if (want0 && !win0) {
    if (pend_b < 0) { pend_b = b0; pend_w = add0; }
    else atomicAdd(hist + b0, add0);
  }
  if (want1 && !win1) {
    if (pend_b < 0) { pend_b = b1; pend_w = add1; }
    else atomicAdd(hist + b1, add1);
  }
}

// apply the pending records of the warp's lanes to its row: tag-arbitrated rounds until none is left (usually one)
__device__ __forceinline__ void flush_pending(double* __restrict__ hist, unsigned char* __restrict__ tags, int lane, int& pend_b,
                                              double& pend_w) {
  while (__any_sync(PCB_FULL_MASK, pend_b >= 0)) {
    if (pend_b >= 0) tags[pend_b] = (unsigned char)lane;
    __syncwarp();
    if (pend_b >= 0 && tags[pend_b] == lane) {
      hist[pend_b] = hist[pend_b] + pend_w;
      pend_b = -1;
    }
    __syncwarp();
  }
}

// resident CTAs per SM the register allocation leaves room for: low dimensions need fewer registers and less shared
// memory, and the accumulation (a warp per axis) keeps fewer of their warps busy
#ifndef PCB_VS_CTAS_LOW
#define PCB_VS_CTAS_LOW 4
#endif
#ifndef PCB_VS_CTAS_MID
#define PCB_VS_CTAS_MID 3
#endif
__host__ __device__ constexpr int vsample_ctas_per_sm(int d) { return d <= 4 ? PCB_VS_CTAS_LOW : (d <= 6 ? PCB_VS_CTAS_MID : 2); }

template <int FAM, int D, int RNG>
__global__ void __launch_bounds__(kSampleWarps * 32, vsample_ctas_per_sm(D)) vsample_kernel(const __grid_constant__ SampleArgs a) {
  using F = Family<FAM>;
  pdl_launch_dependents();
#ifdef PCB_TIMELINE_PASS
  tl_stamp(a.timeline, a.iteration, 0, 0);
#endif
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nb = a.nb, nb1 = a.nb + 1;
  const size_t tag_bytes = (size_t)((nb + 15) & ~15);
  double* s_b = reinterpret_cast<double*>(smem_raw);                                   // [D][nb+1]
  double* s_hist = s_b + (((size_t)D * nb1 + 1) & ~(size_t)1);                         // [D][nb]
  unsigned char* s_tag = reinterpret_cast<unsigned char*>(s_hist + (size_t)D * nb);    // [D][tag_bytes]
  // staging buffer q at s_stage + q * stage_bytes: weights [2][kSampleWarps][32], bin ids [D][2][kSampleWarps][32]
  unsigned char* s_stage = s_tag + (size_t)D * tag_bytes;
  constexpr size_t kStageBytes = (size_t)2 * kSlot * 8 + (size_t)D * 2 * kSlot * 2;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < D * nb; i += blockDim.x) s_hist[i] = 0.0;
  // both staging buffers start as empty records (weight 0, bin 0)
  for (int i = threadIdx.x; i < (int)(2 * kStageBytes / 8); i += blockDim.x) reinterpret_cast<double*>(s_stage)[i] = 0.0;
  // the CTA is resident and its tables are clear while the previous kernel of the stream (the grid refinement of the
  // iteration before) is still finishing; its results -- boundaries, stop decision -- are read from here on
  pdl_wait();
#ifdef PCB_TIMELINE_PASS
  tl_stamp(a.timeline, a.iteration, 0, 1);
#endif
  if (a.stop && a.iteration > *a.stop) return;  // run already converged: a speculatively enqueued pass is a no-op
  {  // boundaries: 16-byte asynchronous copies, all in flight at once (one round trip instead of one per 256 doubles)
    const int total = D * nb1, pairs = total >> 1;
    for (int i = threadIdx.x; i < pairs; i += blockDim.x) {
      const unsigned dst = (unsigned)__cvta_generic_to_shared(s_b + 2 * i);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(a.boundaries + 2 * i) : "memory");
    }
    if ((total & 1) && threadIdx.x == 0) s_b[total - 1] = a.boundaries[total - 1];
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  __syncthreads();
  // debug: phases of the pass, earliest and latest CTA.  Experiment builds only (PCB_NVCC_EXTRA="-DPCB_TIMELINE_PASS
  // -DPCB_DEBUG_ROUNDS"): with the stamps compiled in, the d=8 kernel is 850 instructions longer, allocates its
  // registers differently and the 8.6e8-sample pass takes 39.4 instead of 37.2 ms.
  auto ph_stamp = [&](int k) {
#ifdef PCB_TIMELINE_PASS
    if (a.timeline && a.iteration == 1 && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      atomicMin(a.timeline + 230 + 2 * k, t);        // earliest CTA
      atomicMin(a.timeline + 231 + 2 * k, ~t);       // latest CTA
    }
#endif
  };
  ph_stamp(0);

  const int p = a.p;
  const double pd = (double)p;
  unsigned long long clamp_count = 0;
  // the round being drawn is staged in `cur`; `prev` holds the records of the round before, which this warp adds to
  // its row(s) while it draws
  unsigned char* cur = s_stage;
  unsigned char* prev = s_stage + kStageBytes;
  const int my = wib * 32 + lane;
  constexpr int kRows = (D + kSampleWarps - 1) / kSampleWarps;   // rows of the table this warp serves
#ifndef PCB_VS_CARRY_MIN_D
#define PCB_VS_CARRY_MIN_D 7
#endif
  constexpr bool kCarry = D >= PCB_VS_CARRY_MIN_D;   // pending records take part in the next call (bin_pair_carry) or are flushed per round
  int pend_b[kRows];
  double pend_w[kRows];
#pragma unroll
  for (int q = 0; q < kRows; ++q) { pend_b[q] = -1; pend_w[q] = 0.0; }
  auto stage = [&](int slot, double w, const int (&bin)[D]) {
    reinterpret_cast<double*>(cur)[slot * kSlot + my] = w;
    unsigned short* rb = reinterpret_cast<unsigned short*>(cur + 2 * kSlot * 8);
#pragma unroll
    for (int j = 0; j < D; ++j) rb[(j * 2 + slot) * kSlot + my] = (unsigned short)bin[j];
  };
  // add the records that source warps [w_lo, w_hi) staged in the previous round to the row(s) of this warp
  auto bin_rows = [&](int w_lo, int w_hi, auto unrolled) {
#ifdef PCB_EXPERIMENT_NO_BIN   // experiment builds: how long is a round without the accumulation (results are wrong)
    return;
#endif
    const double* rw = reinterpret_cast<const double*>(prev);
    const unsigned short* rb = reinterpret_cast<const unsigned short*>(prev + 2 * kSlot * 8);
#pragma unroll
    for (int q = 0; q < kRows; ++q) {
      const int j = wib + q * kSampleWarps;
      if (j >= D) break;
      double* hist = s_hist + (size_t)j * nb;
      unsigned char* tags = s_tag + (size_t)j * tag_bytes;
      auto one = [&](int w) {
        if constexpr (kCarry)
          bin_pair_carry(hist, tags, lane, rw[w * 32 + lane], rb[(j * 2) * kSlot + w * 32 + lane], rw[kSlot + w * 32 + lane],
                         rb[(j * 2 + 1) * kSlot + w * 32 + lane], pend_b[q], pend_w[q]);
        else
          bin_pair_flush(hist, tags, lane, rw[w * 32 + lane], rb[(j * 2) * kSlot + w * 32 + lane], rw[kSlot + w * 32 + lane],
                         rb[(j * 2 + 1) * kSlot + w * 32 + lane], pend_b[q], pend_w[q]);
      };
      if constexpr (decltype(unrolled)::value) {
#pragma unroll
        for (int w = w_lo; w < w_hi; ++w) one(w);
      } else {
#pragma unroll 1
        for (int w = w_lo; w < w_hi; ++w) one(w);
      }
    }
  };
  // inside the draw of a sample pair: straight-line, so that the compiler interleaves it with the draw's arithmetic
  auto bin_from = [&](int w_lo, int w_hi) { bin_rows(w_lo, w_hi, std::true_type{}); };
  // everything at once, compact code (single-sample rounds: odd p and the generic generators; the last round)
  auto bin_all = [&]() { bin_rows(0, kSampleWarps, std::false_type{}); };
  // the round is staged: publish it, and take the other buffer (whose records every warp has consumed) for the next
  auto flush_rows = [&]() {
#pragma unroll
    for (int q = 0; q < kRows; ++q) {
      const int j = wib + q * kSampleWarps;
      if (j >= D) break;
      flush_pending(s_hist + (size_t)j * nb, s_tag + (size_t)j * tag_bytes, lane, pend_b[q], pend_w[q]);
    }
  };
  auto end_round = [&]() {   // carried pending records stay in their lanes' slots across rounds (flushed once, at the end)
    if constexpr (!kCarry) flush_rows();
    __syncthreads();
    unsigned char* t = cur; cur = prev; prev = t;
  };

  // the CTA takes kSampleWarps units at a time (one per warp); all units have the same number of rounds
  // debug (PCB_TIMELINE): CTA 0 of iteration 1 stamps the start of each unit batch and the end of each of its rounds
  auto round_stamp = [&](long long ub, int slot) {
#ifdef PCB_DEBUG_ROUNDS   // costs registers in the hot loop: experiment builds only (PCB_NVCC_EXTRA=-DPCB_DEBUG_ROUNDS)
    if (a.timeline && a.iteration == 1 && blockIdx.x == 0 && threadIdx.x == 0) {
      const int idx = 240 + (int)(ub / ((long long)gridDim.x * kSampleWarps)) * 4 + slot;
      if (idx < 256 && slot < 4) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.timeline[idx] = t;
      }
    }
#endif
  };
  for (long long ub = (long long)blockIdx.x * kSampleWarps; ub < a.n_units; ub += (long long)gridDim.x * kSampleWarps) {
    round_stamp(ub, 0);
    const long long u = ub + wib;
    const unsigned long long sin = (unsigned long long)u * 32ULL + (unsigned long long)lane;
    const bool live = u < a.n_units && sin < (unsigned long long)a.n_segments;
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
    if (a.g_m32) {
      unsigned rem = (unsigned)c_begin;
#pragma unroll
      for (int j = D - 1; j >= 0; --j) {
        unsigned digit;
        rem = fast_divmod32(rem, (unsigned)a.g, a.g_m32, digit);
        coord[j] = (double)(int)digit;
      }
    } else {
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

    // every lane of every warp walks the full segment (the rounds are CTA-wide); lanes past their own cube
    // range stage empty records
    for (long long i = 0; i < a.seg_len; ++i) {
      const bool active = i < count;
      const unsigned long long inj_cube = (unsigned long long)(c_begin + i) * (unsigned long long)p;
      double s1 = 0.0, s2 = 0.0;
      int k = 0;
      // two samples at a time: independent dependency chains keep the FP64 and integer pipes busy.  Axis step j of
      // the draw carries its share of the accumulation of the previous round (source warps j*W/D .. (j+1)*W/D).
      if constexpr (RNG == PCB_RNG_REFERENCE_HASH)
      for (; k + 1 < p; k += 2) {
        int bin[2][D];
        double x[2][D], jac[2] = {1.0, 1.0};
#pragma unroll
        for (int j = 0; j < D; ++j) {
          draw_axis<RNG>(a, s_b, j, coord[j], kc, (unsigned long long)T, ctr, (inj_cube + k) * D, active, x[0][j], jac[0], bin[0][j]);
          draw_axis<RNG>(a, s_b, j, coord[j], kc + (unsigned long long)D * kGolden, (unsigned long long)T, ctr + D,
                         (inj_cube + k + 1) * D, active, x[1][j], jac[1], bin[1][j]);
          bin_from(j * kSampleWarps / D, (j + 1) * kSampleWarps / D);
        }
        double fx[2];
        if constexpr (kHasFastSampler<F>) {   // branch-free evaluation where the host established the domain (pcb_device.cuh)
          if (a.f.reserved & PCB_FAST_DOMAIN) {
            fx[0] = eval_at_sampler<F, D, true>(x[0], a.f);
            fx[1] = eval_at_sampler<F, D, true>(x[1], a.f);
          } else {
            fx[0] = eval_at_sampler<F, D>(x[0], a.f);
            fx[1] = eval_at_sampler<F, D>(x[1], a.f);
          }
        } else {
          fx[0] = eval_at_sampler<F, D>(x[0], a.f);
          fx[1] = eval_at_sampler<F, D>(x[1], a.f);
        }
        const double v[2] = {fx[0] * jac[0], fx[1] * jac[1]};
        kc += 2ULL * D * kGolden;
        ctr += 2 * D;
        if (active && !(isfinite(fx[0]) && isfinite(fx[1])))
          atomicMin(a.bad, inj_cube + (unsigned long long)k + (isfinite(fx[0]) ? 1ULL : 0ULL));
        const double v2[2] = {v[0] * v[0], v[1] * v[1]};
        // sample order (numpy's order for p < 8, mcubes.py:245-246; from p = 8 on numpy uses an
        // 8-accumulator tree -- only the rounding differs)
        s1 = (k == 0) ? v[0] + v[1] : (s1 + v[0]) + v[1];
        s2 = (k == 0) ? v2[0] + v2[1] : (s2 + v2[0]) + v2[1];
        stage(0, active ? (a.squared_weighted ? v2[0] : fx[0] * fx[0]) : 0.0, bin[0]);
        stage(1, active ? (a.squared_weighted ? v2[1] : fx[1] * fx[1]) : 0.0, bin[1]);
        end_round();
        round_stamp(ub, (int)i * (p >> 1) + (k >> 1) + 1);
      }
      for (; k < p; ++k) {
        int bin[D];
        double x[D], jac = 1.0;
        bin_all();
#pragma unroll
        for (int j = 0; j < D; ++j)
          draw_axis<RNG>(a, s_b, j, coord[j], kc, (unsigned long long)T, ctr, (inj_cube + k) * D, active, x[j], jac, bin[j]);
        const double fx = eval_at_sampler<F, D>(x, a.f);
        const double v = fx * jac;
        kc += (unsigned long long)D * kGolden;
        ctr += D;
        if (active && !isfinite(fx)) atomicMin(a.bad, inj_cube + (unsigned long long)k);
        const double v2 = v * v;
        s1 = (k == 0) ? v : s1 + v;
        s2 = (k == 0) ? v2 : s2 + v2;
        stage(0, active ? (a.squared_weighted ? v2 : fx * fx) : 0.0, bin);
        stage(1, 0.0, bin);
        end_round();
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
    if (live) {
      double* out = a.seg_partials + sigma * 2;
      out[0] = sum_est;
      out[1] = sum_var;
    }
  }
  ph_stamp(1);
  bin_all();   // the last round's records
  flush_rows();
  if (clamp_count) atomicAdd(a.clamps, clamp_count);
  __syncthreads();
  ph_stamp(2);
  double* dst = a.block_hist + (size_t)blockIdx.x * D * nb;
  for (int i = threadIdx.x; i < D * nb; i += blockDim.x) dst[i] = s_hist[i];
  ph_stamp(3);
#ifdef PCB_TIMELINE_PASS
  tl_stamp(a.timeline, a.iteration, 0, 2);
#endif
}

}  // namespace pcb
