// PAGANI region evaluation for MULTIPLICATIVE integrand families (reference: pagani.py:195-224).
//
// Four of the reference's Genz families factor over the axes up to a final real part:
//   f1  cos(sum_j (j+1) x_j)          = Re prod_j exp(i (j+1) x_j)          integrands.py:38-39
//   f4  exp(-rate * sum_j (x_j-.5)^2) = prod_j exp(-rate (x_j-.5)^2)        integrands.py:79-81
//   f5  exp(-rate * sum_j |x_j-.5|)   = prod_j exp(-rate |x_j-.5|)          integrands.py:91-92
//   f6  exp(sum_j (j+4) x_j) [x < t]  = prod_j [x_j < t_j] exp((j+4) x_j)   integrands.py:113-118
// A Genz-Malik region has only 7 distinct abscissae per axis, so the transcendental is evaluated 7*D
// times per region (D=8: 56) instead of once per rule point (401); a rule point is a short product of
// tabulated factors.  The same products reach the reference value to a few ulp (these families go
// through numpy's SIMD exp/cos in the reference and are compared to 1e-12, never bit-for-bit; the
// families without a transcendental keep the exact-order kernel in pagani_eval.cuh).
//
// Per region (one warp):
//   1. factor table   phi[j][c] = factor_j(left_j + length_j * offset_c), c = 0..6      (7*D entries)
//   2. centre products E[a][b] = prod_{a <= k < b} phi[k][0]                             ((D+1)(D+2)/2)
//   3. rule points, lane l playing virtual threads l and l+32 of the G-wide strided schedule exactly as
//      in the generic kernel (pagani.py:175-192):
//        centre / axial point on axis a:  E[0][a] * phi[a][c] * E[a+1][D]
//        pair point on axes a < b:         E[0][a] * phi[a][ca] * E[a+1][b] * phi[b][cb] * E[b+1][D]
//        corner point:                     prod_j phi[j][5 + bit_j]; with G = 64 the product over axes 0..5
//                                          is constant per virtual thread and hoisted out of the step loop
//   4. schedule tree, volume scaling, error estimate and split axis: shared with the generic kernel.
#pragma once

#include "pagani_eval.cuh"

namespace pcb {

template <bool CPLX>
struct MVal;
template <>
struct MVal<false> {
  double re;
};
template <>
struct __align__(16) MVal<true> {
  double re, im;
};
__device__ __forceinline__ MVal<false> mmul(MVal<false> a, MVal<false> b) { return MVal<false>{a.re * b.re}; }
__device__ __forceinline__ MVal<true> mmul(MVal<true> a, MVal<true> b) {
  return MVal<true>{__fma_rn(a.re, b.re, -(a.im * b.im)), __fma_rn(a.re, b.im, a.im * b.re)};
}
// conjugate: the inverse of a unit-modulus factor
__device__ __forceinline__ MVal<false> mshfl(MVal<false> a, int src) { return MVal<false>{__shfl_sync(PCB_FULL_MASK, a.re, src)}; }
__device__ __forceinline__ MVal<true> mshfl(MVal<true> a, int src) {
  return MVal<true>{__shfl_sync(PCB_FULL_MASK, a.re, src), __shfl_sync(PCB_FULL_MASK, a.im, src)};
}
__device__ __forceinline__ MVal<false> mconj(MVal<false> a) { return a; }
__device__ __forceinline__ MVal<true> mconj(MVal<true> a) { return MVal<true>{a.re, -a.im}; }
__device__ __forceinline__ MVal<false> mone(MVal<false>) { return MVal<false>{1.0}; }
__device__ __forceinline__ MVal<true> mone(MVal<true>) { return MVal<true>{1.0, 0.0}; }

template <int FAM>
struct MultFamily {
  static constexpr bool enabled = false;
  static constexpr bool cplx = false;
  // unit-modulus factors (f1: exp(i theta)) have their conjugate as inverse, so a pair point is
  // Full * rho_a * rho_b with Full = prod_j phi[j][0] and rho_x = conj(phi[x][0]) * phi[x][c]: no table of
  // "everything but axes a and b" (D(D-1)/2 entries per region) is needed
  static constexpr bool unit = false;
  __device__ static MVal<false> factor(int, double, const pcb_integrand&) { return MVal<false>{1.0}; }
};
template <>
struct MultFamily<PCB_F1_OSCILLATORY> {
  static constexpr bool enabled = true;
  static constexpr bool cplx = true;
  static constexpr bool unit = true;
  __device__ static MVal<true> factor(int j, double x, const pcb_integrand&) {
    double s, c;
    sincos((double)(j + 1) * x, &s, &c);
    return MVal<true>{c, s};
  }
};
template <>
struct MultFamily<PCB_F4_GAUSSIAN> {
  static constexpr bool enabled = true;
  static constexpr bool cplx = false;
  static constexpr bool unit = false;
  __device__ static MVal<false> factor(int, double x, const pcb_integrand& f) {
    const double u = x - 0.5;
    return MVal<false>{exp(-f.param[0] * (u * u))};
  }
};
template <>
struct MultFamily<PCB_F5_KINKED> {
  static constexpr bool enabled = true;
  static constexpr bool cplx = false;
  static constexpr bool unit = false;
  __device__ static MVal<false> factor(int, double x, const pcb_integrand& f) { return MVal<false>{exp(-f.param[0] * fabs(x - 0.5))}; }
};
template <>
struct MultFamily<PCB_F6_DISCONTINUOUS> {
  static constexpr bool enabled = true;
  static constexpr bool cplx = false;
  static constexpr bool unit = false;
  __device__ static MVal<false> factor(int j, double x, const pcb_integrand& f) {
    return MVal<false>{(x < f.param[j]) ? exp((double)(j + 5) * x) : 0.0};
  }
};

// index layout of the per-warp table (units of V)
template <int D>
struct MultLayout {
  static constexpr int kPhi = 0;                          // phi[j][c] at j*8 + c; slot c = 7 holds 1
  static constexpr int kE = 8 * D;                        // E[a][b] at kE + a*(D+1) + b, 0 <= a <= b <= D
  static constexpr int kPairs = D * (D - 1) / 2;
  static constexpr int kRab = kE + (D + 1) * (D + 1);     // Rab[pair] = E[0][a] * E[a+1][b] * E[b+1][D]
  static constexpr int kGroups = (D + 2) / 3;             // corner groups of <= 3 axes
  static constexpr int kGrp = kRab + (kPairs > 0 ? kPairs : 1);  // Grp[g][combo] at kGrp + g*8 + combo
  static constexpr int kSize = kGrp + 8 * kGroups;
};

// Unit-modulus families whose phase is LINEAR in x (f1: phi_j(x) = exp(i (j+1) x)) need no transcendental per abscissa:
// the rule's abscissae are centre +- delta_k, so phi(centre +- delta) = phi(centre) * R(+-delta) with R(-delta) =
// conj(R(delta)): three sincos per axis and region (centre, the pair offset, the corner offset) instead of five, and the
// pair candidates' rho = conj(phi(centre)) * phi(centre +- delta) IS R(+-delta) -- no product at all.  The factors move
// by the rounding of one argument (as they do between any two ways of writing the sum); the lane kernel and the warp
// kernel build them with the same operations, so they keep agreeing bit for bit.  PCB_F1_SHARED_TRIG=0: one sincos per
// abscissa (round 1).
#ifndef PCB_F1_SHARED_TRIG
#define PCB_F1_SHARED_TRIG 1
#endif
template <class MF>
__device__ __forceinline__ auto unit_rotation(int j, double len, double off_c, double off_0, const pcb_integrand& f) {
  double dx = len * (off_c - off_0);
  if (f.bounded) dx = f.width[j] * dx;
  return MF::factor(j, dx, f);
}

template <int FAM, int D>
__global__ void __launch_bounds__(kEvalWarps * 32) pagani_eval_mult_kernel(const __grid_constant__ EvalArgs args) {
  pdl_wait();   // region list and flags come from the kernels before it in the stream (programmatic serialisation)
  using F = Family<FAM>;
  using MF = MultFamily<FAM>;
  using V = MVal<MF::cplx>;
  using L = MultLayout<D>;
  constexpr int kStore = 4 * D + 1;                // f(centre), f(+-l2 e_j), f(+-l3 e_j): split-axis inputs
  constexpr int kCorner0 = 2 * D * D + 2 * D + 1;  // first corner point
  constexpr int kHeadGroups = D >= 6 ? 2 : L::kGroups;  // groups whose corner bits are fixed per virtual thread when G = 64
  __shared__ V s_tab[kEvalWarps][L::kSize];
  __shared__ __align__(16) double s_term[kEvalWarps][D * 8];  // generic per-axis terms, for the centre/axial points
  __shared__ double s_store[kEvalWarps][kStore + 1];
  __shared__ double s_geo[kEvalWarps][2][2 * D];   // double-buffered left[0..D), length[0..D)
  __shared__ __align__(16) double s_w[6][8];       // orbit weights (+pad); rows 4/5 = corners with even/odd bit count
  __shared__ double s_off[8];
  __shared__ unsigned s_pair[L::kPairs > 0 ? L::kPairs : 1];  // per axis pair: a | b << 8

  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const pcb_rule& rule = args.rule;
  if (threadIdx.x < 30) {
    int o = threadIdx.x / 5, k = threadIdx.x % 5;
    double w = rule.weights[k][o < 5 ? o : 4];
    if (o == 5 && rule.corner_parity[k]) w = -w;
    s_w[o][k] = w;
  }
  if (threadIdx.x < 7) s_off[threadIdx.x] = rule.offsets[threadIdx.x];
  for (int e = threadIdx.x; e < L::kPairs; e += blockDim.x) {
    int idx = 0;
    for (int j = 0; j < D; ++j)
      for (int k = j + 1; k < D; ++k, ++idx)
        if (idx == e) s_pair[e] = (unsigned)j | ((unsigned)k << 8);
  }
  __syncthreads();

  const int fe = rule.f_eval, G = args.group;
  const double jac = args.f.bounded ? args.f.jac : 1.0;   // x * 1.0 == x: no branch per point
  V* tab = s_tab[wib];
  double* term = s_term[wib];
  const char* term_b = reinterpret_cast<const char*>(term);
  double* store = s_store[wib];
  long long n_regions = args.n, ld = args.ld;
  if (args.state) {   // launched before the host knew the list: length and stride come from the previous iteration kernel
    if (args.state->status != 0) return;
    n_regions = args.state->n;
    ld = args.state->ld;
  }
  const long long stride = (long long)gridDim.x * kEvalWarps;
  long long r = (long long)blockIdx.x * kEvalWarps + wib;
  int buf = 0;
  if (r < n_regions && lane < 2 * D)
    s_geo[wib][0][lane] = (lane < D) ? args.lefts[lane * ld + r] : args.lengths[(lane - D) * ld + r];
  __syncwarp();

  for (; r < n_regions; r += stride, buf ^= 1) {
    const double* geo = s_geo[wib][buf];
    // prefetch the next region's geometry (consumed at the bottom of the loop)
    const long long rn = r + stride;
    double next_geo = 0.0;
    if (rn < n_regions && lane < 2 * D) next_geo = (lane < D) ? args.lefts[lane * ld + rn] : args.lengths[(lane - D) * ld + rn];

    // ---- 1. per-axis tables at the 7 distinct abscissae (quadrature.py:301-302: mul, then add)
#pragma unroll
    for (int e0 = 0; e0 < 8 * D; e0 += 32) {
      const int e = e0 + lane, j = e >> 3, c = e & 7;
      const bool mine = e < 8 * D;
      V v = mone(V{});
      if (mine && c < 7) {
        double x = geo[j] + geo[D + j] * s_off[c];
        if (args.f.bounded) x = args.f.low[j] + args.f.width[j] * x;
        if constexpr (MF::unit && PCB_F1_SHARED_TRIG) {
          // centre factor (c = 0) or the rotation of the offset pair c belongs to (the operations of unit_rotation();
          // one call site for the whole warp); completed below
          double arg = x;
          if (c >= 3) {
            arg = geo[D + j] * (s_off[c < 5 ? 3 : 5] - s_off[0]);
            if (args.f.bounded) arg = args.f.width[j] * arg;
          }
          if (c == 0 || c >= 3) v = MF::factor(j, arg, args.f);
        } else {
          v = MF::factor(j, x, args.f);
        }
        term[e] = F::term(j, x, args.f);
      }
      if constexpr (MF::unit && PCB_F1_SHARED_TRIG) {
        // lane 8 (j mod 4) of this round holds the centre factor of the axis: rho(-delta) = conj(rho(delta)),
        // phi(centre +- delta) = phi(centre) * rho(+-delta) -- as in the lane kernel, operand for operand
        const V e0 = mshfl(v, lane & ~7);
        if (c == 4) v = mconj(v);
        else if (c == 5) v = mmul(e0, v);
        else if (c == 6) v = mmul(e0, mconj(v));
      }
      if (mine) tab[e] = v;   // slot c = 7 of every axis holds 1
    }
    double vol = geo[D];
#pragma unroll
    for (int j = 1; j < D; ++j) vol = vol * geo[D + j];  // np.prod, left to right
    __syncwarp();

    // ---- 2a. centre products E[a][b] = prod_{a <= k < b} phi[k][0]: lane a walks row a;
    //          corner group tables Grp[g][combo] = prod_{axes j of group g} phi[j][5 + bit]
    if (lane <= D) {
      V run = mone(V{});
      tab[L::kE + lane * (D + 1) + lane] = run;
#pragma unroll
      for (int b = 1; b <= D; ++b) {
        if (b > lane) {
          run = mmul(run, tab[(b - 1) * 8]);
          tab[L::kE + lane * (D + 1) + b] = run;
        }
      }
    }
#pragma unroll
    for (int e0 = 0; e0 < 8 * L::kGroups; e0 += 32) {
      const int e = e0 + lane, g = e >> 3, combo = e & 7;
      if (e < 8 * L::kGroups) {
        const int j0 = 3 * g;
        V v = tab[j0 * 8 + 5 + (combo & 1)];
        if (j0 + 1 < D) v = mmul(v, tab[(j0 + 1) * 8 + 5 + ((combo >> 1) & 1)]);
        if (j0 + 2 < D) v = mmul(v, tab[(j0 + 2) * 8 + 5 + ((combo >> 2) & 1)]);
        tab[L::kGrp + e] = v;
      }
    }
    __syncwarp();
    // ---- 2b. unit-modulus factors: rho[j][c] = conj(phi[j][0]) * phi[j][c] for the pair candidates c = 3, 4 (in place)
    if constexpr (MF::unit) {
      if (!PCB_F1_SHARED_TRIG && lane < 2 * D) {   // with shared rotations the slots already hold rho
        const int j = lane >> 1, c = 3 + (lane & 1);
        tab[j * 8 + c] = mmul(mconj(tab[j * 8]), tab[j * 8 + c]);
      }
      __syncwarp();
    } else
    // ---- 2b. Rab[pair] = E[0][a] * E[a+1][b] * E[b+1][D]: everything of a pair point but its two moved axes
    if constexpr (L::kPairs > 0) {
#pragma unroll
      for (int e0 = 0; e0 < L::kPairs; e0 += 32) {
        const int e = e0 + lane;
        if (e < L::kPairs) {
          const unsigned ab = s_pair[e];
          const int a = ab & 255u, b = ab >> 8;
          tab[L::kRab + e] = mmul(mmul(tab[L::kE + a], tab[L::kE + (a + 1) * (D + 1) + b]), tab[L::kE + (b + 1) * (D + 1) + D]);
        }
      }
      __syncwarp();
    }

    // ---- 3. rule points of my two virtual threads.  Partial sums start from -0.0: (-0.0) + x == x for every x,
    //         so "first product, then adds" (pagani.py:189-191) needs no special case; a virtual thread without
    //         points keeps the +0.0 of the reference's zero padding.
    double acc[2][5];
    unsigned badpt = 0xffffffffu;
#pragma unroll
    for (int set = 0; set < 2; ++set) {
      const int vt = lane + 32 * set;
      const double init = (vt < G && vt < fe) ? -0.0 : 0.0;
#pragma unroll
      for (int k = 0; k < 5; ++k) acc[set][k] = init;
      if (vt >= G) continue;
      int i = vt;
      // centre and axial points: evaluated in the reference's own association (these are the split-axis inputs,
      // whose fourth differences cancel to rounding level: pagani.py:215-223)
      for (; i <= 4 * D; i += G) {
        const int q = i - 1;
        const int a = i == 0 ? -1 : ((q >= 2 * D ? q - 2 * D : q) >> 1);
        const unsigned cand = i == 0 ? 0u : (unsigned)(8 * (1 + (q & 1) + (q >= 2 * D ? 2 : 0)));
        double t[D];
#pragma unroll
        for (int j = 0; j < D; ++j) t[j] = term_at<D>(term_b, j, j == a ? cand : 0u);
        double fx = F::template finish<D>(combine_terms<F, D>(t), args.f) * jac;
        if (!isfinite(fx)) badpt = min(badpt, (unsigned)i);
        store[i] = fx;
        const double* w = s_w[i == 0 ? 0 : (q >= 2 * D ? 2 : 1)];
#pragma unroll
        for (int k = 0; k < 5; ++k) acc[set][k] = acc[set][k] + w[k] * fx;
      }
      // pair points: Rab * phi[a][3 or 4] * phi[b][3 or 4]; point i = 4D + 1 + 4*pair + sign bits
      if constexpr (L::kPairs > 0) {
        for (; i < kCorner0; i += G) {
          const int q = i - 1 - 4 * D, e = q >> 2;
          const unsigned ab = s_pair[e];
          const int a = ab & 255u, b = ab >> 8;
          const V v = mmul(mmul(tab[MF::unit ? L::kE + D : L::kRab + e], tab[a * 8 + 3 + (q & 1)]), tab[b * 8 + 3 + ((q >> 1) & 1)]);
          const double fx = v.re * jac;
          if (!isfinite(fx)) badpt = min(badpt, (unsigned)i);
#pragma unroll
          for (int k = 0; k < 5; ++k) acc[set][k] = acc[set][k] + rule.weights[k][3] * fx;
        }
      }
      // corner points: bit j of (i - kCorner0) set => abscissa candidate 6 (minus), else 5 (plus)
      if (G == 64) {
        V head = mone(V{});
        if (i < fe) {
          const unsigned bits = (unsigned)(i - kCorner0);
          head = tab[L::kGrp + (bits & 7u)];
          if constexpr (kHeadGroups > 1) head = mmul(head, tab[L::kGrp + 8 + ((bits >> 3) & 7u)]);
        }
        for (; i < fe; i += 64) {
          const unsigned bits = (unsigned)(i - kCorner0);
          V v = head;
#pragma unroll
          for (int g = kHeadGroups; g < L::kGroups; ++g) v = mmul(v, tab[L::kGrp + 8 * g + ((bits >> (3 * g)) & 7u)]);
          const double fx = v.re * jac;
          if (!isfinite(fx)) badpt = min(badpt, (unsigned)i);
          const double* w = s_w[4 + (__popc(bits) & 1)];
#pragma unroll
          for (int k = 0; k < 5; ++k) acc[set][k] = acc[set][k] + w[k] * fx;
        }
      } else {
        for (; i < fe; i += G) {
          const unsigned bits = (unsigned)(i - kCorner0);
          V v = tab[L::kGrp + (bits & 7u)];
#pragma unroll
          for (int g = 1; g < L::kGroups; ++g) v = mmul(v, tab[L::kGrp + 8 * g + ((bits >> (3 * g)) & 7u)]);
          const double fx = v.re * jac;
          if (!isfinite(fx)) badpt = min(badpt, (unsigned)i);
          const double* w = s_w[4 + (__popc(bits) & 1)];
#pragma unroll
          for (int k = 0; k < 5; ++k) acc[set][k] = acc[set][k] + w[k] * fx;
        }
      }
    }
    if (__any_sync(PCB_FULL_MASK, badpt != 0xffffffffu)) {
      if (badpt != 0xffffffffu) atomicMin(args.bad, (unsigned long long)r * (unsigned long long)fe + (unsigned long long)badpt);
    }

    // ---- 4. schedule tree, volume scaling / error / split axis (as in the generic kernel)
    double sums[5];
    schedule_tree(acc[0], acc[1], lane, sums);
    double v[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) v[k] = vol * sums[k];
    __syncwarp();
    int axis = 0;
    if constexpr (D > 1) axis = split_axis_warp<D>(store, rule, lane);
    const double err = region_error_warp(v, rule, args.err_mode, args.rel_floor, lane);
    if (lane == 0) {
      args.integrals[r] = v[0];
      args.errors[r] = err;
      args.split_axes[r] = axis;
    }
    if (lane < 2 * D) s_geo[wib][buf ^ 1][lane] = next_geo;
    __syncwarp();
  }
}

}  // namespace pcb
