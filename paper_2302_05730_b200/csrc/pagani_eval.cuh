// PAGANI region evaluation: one warp per region (reference: pagani.py:195-224, A.1 of SURVEY.md).
//
// Per region the kernel
//   1. tabulates, per axis, the integrand's per-axis term at the 7 distinct abscissae
//      left + length*offset (quadrature.py:301-302; mul then add) -- 7*D terms instead of F*D;
//   2. evaluates the F rule points: lane l plays the reference's virtual threads l and l+32 of
//      the G-wide strided schedule (point indices t, t+G, ...; pagani.py:175-192).  A point's
//      terms are gathered from the table and combined in numpy's order:
//        * centre/axial/pair points through a per-point code word (one byte per axis = byte offset
//          of the abscissa candidate), built once per CTA;
//        * corner points straight from the point's bit pattern; with G = 64 the low six bits are
//          constant per virtual thread, so the partial combine over axes 0..5 is hoisted out of
//          the step loop;
//   3. reduces the 2x5 partial sums with a reduce-scatter butterfly whose add tree is exactly the
//      adjacent-pair tree of engine.tree_sum over 64 virtual threads (xor 1,2,4,8,16, then A+B);
//   4. scales by the volume, forms the error estimate (pagani.py:104-132) and the split axis
//      (pagani.py:215-223, first maximum wins).
// The next region's geometry is prefetched while the current one is evaluated.
#pragma once

#include "pcb_device.cuh"

namespace pcb {

// The lane kernels take the rule whose corner weights alternate with the bit count in exactly one rule, the parity
// null rule (quadrature.py:199-203); the host sends every other table to the warp-per-region kernels.
constexpr int kParityRule = 2;


struct EvalArgs {
  pcb_integrand f;
  pcb_rule rule;
  long long n, ld;
  const double* lefts;    // [d][ld]
  const double* lengths;  // [d][ld]
  double* integrals;
  double* errors;
  int32_t* split_axes;
  unsigned long long* bad;  // min over non-finite evaluations of region*F + point
  int group;
  int err_mode;
  double rel_floor;
  const ShortState* state = nullptr;   // warp-per-region kernels only: take n and ld from the device (speculative launch)
};

constexpr int kEvalWarps = 4;  // warps per CTA

// error estimate from the five volume-scaled rule values (pagani.py:104-132)
__device__ __forceinline__ double region_error(const double (&v)[5], const pcb_rule& rule, int mode,
                                               double rel_floor) {
  double nul[4] = {fabs(v[1]), fabs(v[2]), fabs(v[3]), fabs(v[4])};
  double err;
  if (mode == PCB_ERR_MAX_NULL) {
    err = fmax(fmax(nul[0], nul[1]), fmax(nul[2], nul[3]));
  } else if (mode == PCB_ERR_MAX_PAIRWISE) {
    err = 0.0;
#pragma unroll
    for (int a = 1; a < 5; ++a)
#pragma unroll
      for (int b = 1; b < 5; ++b) err = fmax(err, fabs(v[a] - v[b]));
  } else {
    double e_high = -1.0, e_low = -1.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (rule.null_high[k]) e_high = fmax(e_high, nul[k]);
      else e_low = fmax(e_low, nul[k] / rule.null_scale[k]);
    }
    double corr = (e_low > 0.0) ? (10.0 * e_high) / e_low : 1.0;
    err = e_high * fmin(1.0, corr);
  }
  return fmax(err, rel_floor * fabs(v[0]));
}

__device__ __forceinline__ double shfl_xor_d(double v, int m) { return __shfl_xor_sync(PCB_FULL_MASK, v, m); }
__device__ __forceinline__ double shfl_idx_d(double v, int l) { return __shfl_sync(PCB_FULL_MASK, v, l); }

// region_error with the divisions of the two-level mode spread over the lanes: every lane holds v[0..4];
// lane k < 4 forms nul[k] / scale[k] (x / 1.0 == x, so unit scales skip the ~25-instruction division), the
// maxima are gathered with shuffles.  Same operations and roundings as region_error, a third of the issue slots.
__device__ __forceinline__ double region_error_warp(const double (&v)[5], const pcb_rule& rule, int mode, double rel_floor,
                                                    int lane) {
  if (mode != PCB_ERR_TWO_LEVEL) return region_error(v, rule, mode, rel_floor);
  const int k = lane & 3;
  const double mine = fabs(k == 0 ? v[1] : k == 1 ? v[2] : k == 2 ? v[3] : v[4]);
  const bool high = rule.null_high[k] != 0;
  const double scale = rule.null_scale[k];
  double hi = high ? mine : -1.0;
  double lo = high ? -1.0 : (scale == 1.0 ? mine : mine / scale);
  hi = fmax(hi, shfl_xor_d(hi, 1));
  lo = fmax(lo, shfl_xor_d(lo, 1));
  hi = fmax(hi, shfl_xor_d(hi, 2));
  lo = fmax(lo, shfl_xor_d(lo, 2));
  const double corr = (lo > 0.0) ? (10.0 * hi) / lo : 1.0;
  const double err = hi * fmin(1.0, corr);
  return fmax(err, rel_floor * fabs(v[0]));
}

// split axis (pagani.py:215-223): argmax_j |c0 * d2(l2, j) - c1 * d2(l3, j)| over the stored centre/axial
// evaluations, first maximum wins.  All lanes return the axis.
template <int D>
__device__ __forceinline__ int split_axis_warp(const double* store, const pcb_rule& rule, int lane) {
  double ind = -1.0;
  if (lane < D) {
    double two_f0 = 2.0 * store[0];
    double d2a = (store[1 + 2 * lane] + store[2 + 2 * lane]) - two_f0;
    double d2b = (store[1 + 2 * D + 2 * lane] + store[2 + 2 * D + 2 * lane]) - two_f0;
    ind = fabs(rule.split_weights[0] * d2a - rule.split_weights[1] * d2b);
  }
  int idx = lane;
#pragma unroll
  for (int m = 8; m >= 1; m >>= 1) {  // argmax over lanes 0..15, lowest index wins ties
    double o = shfl_xor_d(ind, m);
    int oi = __shfl_xor_sync(PCB_FULL_MASK, idx, m);
    if (o > ind || (o == ind && oi < idx)) { ind = o; idx = oi; }
  }
  return __shfl_sync(PCB_FULL_MASK, idx, 0);
}

// Reduce 2 sets x 5 columns over the 32 lanes with the adjacent-pair tree, then add the two sets.
// On return every lane holds all five sums.
__device__ __forceinline__ void schedule_tree(const double (&a)[5], const double (&b)[5], int lane,
                                              double (&out)[5]) {
  const bool b0 = lane & 1, b1 = lane & 2, b2 = lane & 4, b3 = lane & 8;
  double c5[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) {  // level 1: lanes (l, l^1); even lanes keep set A, odd lanes set B
    double keep = b0 ? b[k] : a[k];
    double send = b0 ? a[k] : b[k];
    c5[k] = keep + shfl_xor_d(send, 1);
  }
  double c4[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {  // level 2: bit1 = 0 keeps columns 0..3, bit1 = 1 keeps 4..7 (5..7 are padding)
    double hi = (i == 0) ? c5[4] : 0.0;
    double keep = b1 ? hi : c5[i];
    double send = b1 ? c5[i] : hi;
    c4[i] = keep + shfl_xor_d(send, 2);
  }
  double c2[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {  // level 3
    double keep = b2 ? c4[2 + i] : c4[i];
    double send = b2 ? c4[i] : c4[2 + i];
    c2[i] = keep + shfl_xor_d(send, 4);
  }
  double keep = b3 ? c2[1] : c2[0];  // level 4
  double send = b3 ? c2[0] : c2[1];
  double c1 = keep + shfl_xor_d(send, 8);
  c1 = c1 + shfl_xor_d(c1, 16);      // level 5
  c1 = c1 + shfl_xor_d(c1, 1);       // level 6: virtual threads 0..31 + 32..63
  // column held by lane l: (bit1<<2) | (bit2<<1) | bit3
  out[0] = shfl_idx_d(c1, 0);
  out[1] = shfl_idx_d(c1, 8);
  out[2] = shfl_idx_d(c1, 4);
  out[3] = shfl_idx_d(c1, 12);
  out[4] = shfl_idx_d(c1, 2);
}

// term table row of axis j starts at byte j*64; candidate c sits at byte offset c*8
template <int D>
__device__ __forceinline__ double term_at(const char* table, int j, unsigned byte_off) {
  return *reinterpret_cast<const double*>(table + j * 64 + byte_off);
}

// ---- corner points: combine over all axes, split into a hoistable part (axes < LO) and the rest.
// The split reproduces numpy's association exactly for every combine kind.
template <class F, int D, int LO>
struct CornerCombine {
  // partial state after the first LO axes
  double p0, p1;  // seq kinds: p0 = t0 (+) ... (+) t_{LO-1};  numpy-sum with D >= 8 and LO == 6: p0 = (a0+a1)+(a2+a3), p1 = a4+a5
  __device__ __forceinline__ void head(const char* table, unsigned bits) {
    double t[LO > 0 ? LO : 1];
#pragma unroll
    for (int j = 0; j < LO; ++j) t[j] = term_at<D>(table, j, 40u + ((bits >> j) & 1u) * 8u);
    if constexpr (LO == 0) {
      p0 = 0.0; p1 = 0.0;
    } else if constexpr (F::combine == kSumNumpy && D >= 8) {
      static_assert(LO == 6 || LO == 0, "hoisting is laid out for six lane-constant axes");
      p0 = (t[0] + t[1]) + (t[2] + t[3]);
      p1 = t[4] + t[5];
    } else {
      double s = t[0];
#pragma unroll
      for (int j = 1; j < LO; ++j) s = (F::combine == kProdSeq) ? s * t[j] : s + t[j];
      p0 = s; p1 = 0.0;
    }
  }
  __device__ __forceinline__ double tail(const char* table, unsigned bits) const {
    if constexpr (LO == 0) {
      double t[D];
#pragma unroll
      for (int j = 0; j < D; ++j) t[j] = term_at<D>(table, j, 40u + ((bits >> j) & 1u) * 8u);
      return combine_terms<F, D>(t);
    } else if constexpr (F::combine == kSumNumpy && D >= 8) {
      const double a6 = term_at<D>(table, 6, 40u + ((bits >> 6) & 1u) * 8u);
      const double a7 = term_at<D>(table, 7, 40u + ((bits >> 7) & 1u) * 8u);
      double s = p0 + (p1 + (a6 + a7));
#pragma unroll
      for (int j = 8; j < D; ++j) s = s + term_at<D>(table, j, 40u + ((bits >> j) & 1u) * 8u);
      return s;
    } else {
      double s = p0;
#pragma unroll
      for (int j = LO; j < D; ++j) {
        const double t = term_at<D>(table, j, 40u + ((bits >> j) & 1u) * 8u);
        s = (F::combine == kProdSeq) ? s * t : s + t;
      }
      return s;
    }
  }
};

// WIDE = true: schedule widths G > 64 (pagani.py:56,66 accept any G >= 1).  The warp walks the virtual threads in
// blocks of 64; a block's 64-leaf pair tree is the butterfly above, and the block sums are merged by a binary
// counter -- complete aligned subtrees of 64 * 2^h leaves -- which is engine.tree_sum's adjacent-pair tree over
// the G partials (zero leaves beyond the last virtual thread that owns a point: x + 0.0 == x).
template <int FAM, int D, bool WIDE = false>
__global__ void __launch_bounds__(kEvalWarps * 32) pagani_eval_kernel(const __grid_constant__ EvalArgs args) {
  pdl_wait();   // region list and flags come from the kernels before it in the stream (programmatic serialisation)
  using F = Family<FAM>;
  constexpr int kStore = 4 * D + 1;            // f(centre), f(+-l2 e_j), f(+-l3 e_j): split-axis inputs
  constexpr int kCorner0 = 2 * D * D + 2 * D + 1;  // first corner point
  constexpr int kWords = (D + 7) / 8;          // 64-bit code words per non-corner point
  constexpr int kLo = D < 6 ? D : 6;           // axes whose corner bit is fixed per virtual thread when G = 64
  __shared__ __align__(16) double s_term[kEvalWarps][D * 8];
  __shared__ double s_store[kEvalWarps][kStore + 1];
  __shared__ double s_geo[kEvalWarps][2][2 * D];   // double-buffered left[0..D), length[0..D)
  __shared__ __align__(16) double s_w[6][8];   // orbit weights (+pad); rows 4/5 = corners with even/odd bit count
  __shared__ double s_off[8];
  __shared__ unsigned long long s_code[kCorner0][kWords];  // byte j: candidate byte offset on axis j; bits 6-7 of byte 0: orbit
  __shared__ double s_lvl[WIDE ? kEvalWarps : 1][WIDE ? 8 : 1][5];   // WIDE: the binary counter of block sums

  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const pcb_rule& rule = args.rule;
  if (threadIdx.x < 30) {
    int o = threadIdx.x / 5, k = threadIdx.x % 5;
    double w = rule.weights[k][o < 5 ? o : 4];
    if (o == 5 && rule.corner_parity[k]) w = -w;
    s_w[o][k] = w;
  }
  if (threadIdx.x < 7) s_off[threadIdx.x] = rule.offsets[threadIdx.x];
  for (int i = threadIdx.x; i < kCorner0; i += blockDim.x) {
    // decode point i (centre | +-l2 e_j | +-l3 e_j | l4 pairs) once per CTA
    int a = -1, b = -1, ca = 0, cb = 0, orbit = 0;
    if (i == 0) {
    } else if (i <= 2 * D) {
      int q = i - 1; a = q >> 1; ca = 1 + (q & 1); orbit = 1;
    } else if (i <= 4 * D) {
      int q = i - 1 - 2 * D; a = q >> 1; ca = 3 + (q & 1); orbit = 2;
    } else {
      int q = i - 1 - 4 * D, pr = q >> 2, sg = q & 3, idx = 0;
      for (int j = 0; j < D; ++j)
        for (int k = j + 1; k < D; ++k, ++idx)
          if (idx == pr) { a = j; b = k; }
      ca = 3 + (sg & 1); cb = 3 + (sg >> 1); orbit = 3;
    }
    unsigned long long w[kWords];
    for (int q = 0; q < kWords; ++q) w[q] = 0;
    if (a >= 0) w[a >> 3] |= (unsigned long long)(ca * 8) << (8 * (a & 7));
    if (b >= 0) w[b >> 3] |= (unsigned long long)(cb * 8) << (8 * (b & 7));
    w[0] |= (unsigned long long)orbit << 6;
    for (int q = 0; q < kWords; ++q) s_code[i][q] = w[q];
  }
  __syncthreads();

  const int fe = rule.f_eval, G = args.group;
  const double jac = args.f.bounded ? args.f.jac : 1.0;   // x * 1.0 == x: no branch per point
  const char* term_b = reinterpret_cast<const char*>(s_term[wib]);
  double* term = s_term[wib];
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
  // geometry of the first region
  if (r < n_regions && lane < 2 * D)
    s_geo[wib][0][lane] = (lane < D) ? args.lefts[lane * ld + r] : args.lengths[(lane - D) * ld + r];
  __syncwarp();

  for (; r < n_regions; r += stride, buf ^= 1) {
    const double* geo = s_geo[wib][buf];
    // prefetch the next region's geometry (consumed at the bottom of the loop)
    const long long rn = r + stride;
    double next_geo = 0.0;
    if (rn < n_regions && lane < 2 * D) next_geo = (lane < D) ? args.lefts[lane * ld + rn] : args.lengths[(lane - D) * ld + rn];

    // ---- 1. per-axis term table at the 7 distinct abscissae
#pragma unroll
    for (int e0 = 0; e0 < 8 * D; e0 += 32) {
      const int e = e0 + lane, j = e >> 3, c = e & 7;
      if (e < 8 * D && c < 7) {
        const double x = geo[j] + geo[D + j] * s_off[c];
        term[e] = axis_term<F>(j, x, args.f);
      }
    }
    double vol = geo[D];
#pragma unroll
    for (int j = 1; j < D; ++j) vol = vol * geo[D + j];  // np.prod, left to right
    __syncwarp();

    // ---- 2. rule points of my two virtual threads.  Partial sums start from -0.0: (-0.0) + x == x for every
    //         x, so "first product, then adds" (pagani.py:189-191) needs no special case; a virtual thread
    //         without points keeps the +0.0 of the reference's zero padding.
    double acc[2][5];
    unsigned badpt = 0xffffffffu;
    // the (up to) 64 virtual threads vt0 .. vt0 + 63: lane l plays vt0 + l and vt0 + l + 32
    auto play_block = [&](const int vt0) {
  #pragma unroll
      for (int set = 0; set < 2; ++set) {
        const int vt = vt0 + lane + 32 * set;
        const double init = (vt < G && vt < fe) ? -0.0 : 0.0;
  #pragma unroll
        for (int k = 0; k < 5; ++k) acc[set][k] = init;
        if (vt >= G) continue;
        int i = vt;
        // centre, axial and pair points
        for (; i < kCorner0; i += G) {
          unsigned long long code[kWords];
  #pragma unroll
          for (int q = 0; q < kWords; ++q) code[q] = s_code[i][q];
          const int orbit = (int)((unsigned)code[0] >> 6) & 3;
          code[0] &= ~0xC0ULL;
          double t[D];
  #pragma unroll
          for (int j = 0; j < D; ++j) {
            const unsigned half = (unsigned)(code[j >> 3] >> (32 * ((j >> 2) & 1)));
            t[j] = term_at<D>(term_b, j, __byte_perm(half, 0, 0x4440 + (j & 3)));
          }
          const double fx = F::template finish<D>(combine_terms<F, D>(t), args.f) * jac;
          if (!isfinite(fx)) badpt = min(badpt, (unsigned)i);
          if (i < kStore) store[i] = fx;
          const double* w = s_w[orbit];
  #pragma unroll
          for (int k = 0; k < 5; ++k) acc[set][k] = acc[set][k] + w[k] * fx;
        }
        // corner points: bit j of (i - kCorner0) set => abscissa candidate 6 (minus), else 5 (plus)
        if (G == 64) {
          CornerCombine<F, D, kLo> cc;
          if (i < fe) cc.head(term_b, (unsigned)(i - kCorner0));
          for (; i < fe; i += 64) {
            const unsigned bits = (unsigned)(i - kCorner0);
            const double fx = F::template finish<D>(cc.tail(term_b, bits), args.f) * jac;
            if (!isfinite(fx)) badpt = min(badpt, (unsigned)i);
            const double* w = s_w[4 + (__popc(bits) & 1)];
  #pragma unroll
            for (int k = 0; k < 5; ++k) acc[set][k] = acc[set][k] + w[k] * fx;
          }
        } else {
          CornerCombine<F, D, 0> cc;
          for (; i < fe; i += G) {
            const unsigned bits = (unsigned)(i - kCorner0);
            const double fx = F::template finish<D>(cc.tail(term_b, bits), args.f) * jac;
            if (!isfinite(fx)) badpt = min(badpt, (unsigned)i);
            const double* w = s_w[4 + (__popc(bits) & 1)];
  #pragma unroll
            for (int k = 0; k < 5; ++k) acc[set][k] = acc[set][k] + w[k] * fx;
          }
        }
      }
    };
    double sums[5];
    if constexpr (!WIDE) {
      play_block(0);
      schedule_tree(acc[0], acc[1], lane, sums);
    } else {
      const int leaves = G < fe ? G : fe;           // virtual threads beyond own no point: zero leaves
      unsigned have = 0;
      for (int vt0 = 0; vt0 < leaves; vt0 += 64) {
        play_block(vt0);
        schedule_tree(acc[0], acc[1], lane, sums);
        int h = 0;
        for (; (have >> h) & 1u; ++h) {             // carry: left subtree (stored) + right subtree (new)
#pragma unroll
          for (int k = 0; k < 5; ++k) sums[k] = s_lvl[wib][h][k] + sums[k];
          have &= ~(1u << h);
        }
        if (lane == 0) {
#pragma unroll
          for (int k = 0; k < 5; ++k) s_lvl[wib][h][k] = sums[k];
        }
        have |= 1u << h;
        __syncwarp();
      }
      bool first = true;
      for (int h = 0; h < 8; ++h) {
        if (!((have >> h) & 1u)) continue;
#pragma unroll
        for (int k = 0; k < 5; ++k) sums[k] = first ? s_lvl[wib][h][k] : s_lvl[wib][h][k] + sums[k];
        first = false;
      }
      __syncwarp();
    }
    if (__any_sync(PCB_FULL_MASK, badpt != 0xffffffffu)) {
      if (badpt != 0xffffffffu) atomicMin(args.bad, (unsigned long long)r * (unsigned long long)fe + (unsigned long long)badpt);
    }

    // ---- 3. schedule tree (above), 4. volume scaling / error / split axis
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

// Plain evaluation of the functor at caller-supplied points (Integrand.eval_many).
template <int FAM, int D>
__global__ void eval_points_kernel(const __grid_constant__ pcb_integrand f, long long n, const double* pts, double* out) {
  using F = Family<FAM>;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double x[D];
#pragma unroll
    for (int j = 0; j < D; ++j) x[j] = pts[i * D + j];
    out[i] = eval_at<F, D>(x, f);
  }
}

// Serial integrand invocation micro-benchmark (reference: cli.py:123-153): every
// thread evaluates all n points one after the other and keeps a running sum.
template <int FAM, int D>
__global__ void invoke_kernel(const __grid_constant__ pcb_integrand f, long long n, const double* __restrict__ pts,
                              double* __restrict__ acc_out) {
  using F = Family<FAM>;
  double acc = 0.0;
  for (long long i = 0; i < n; ++i) {
    double x[D];
#pragma unroll
    for (int j = 0; j < D; ++j) x[j] = pts[i * D + j];
    acc = acc + eval_at<F, D>(x, f);
  }
  acc_out[blockIdx.x * (long long)blockDim.x + threadIdx.x] = acc;
}

// Randomly shifted Sobol' average (reference: integrands.py:223-260, the independent QMC oracle): shift s of the
// launch's blockIdx.y, points [0, 2^log2n) in the Gray-code order of the generator (x_{i+1} = x_i ^ V[ctz(i+1)]);
// a thread walks a contiguous run of points, point = frac(sobol + shift) as base + shift - floor(.), and the block's
// sum goes to partial[shift][block] (the host-side driver finishes the per-shift sums with the pair tree).
constexpr int kSobolBits = 30;   // scipy.stats.qmc.Sobol default: coordinates are multiples of 2^-30
template <int FAM, int D>
__global__ void __launch_bounds__(256) qmc_shift_kernel(const __grid_constant__ pcb_integrand f, int log2n,
                                                        const unsigned* __restrict__ dirs /* [D][30] */,
                                                        const double* __restrict__ shifts /* [n_shifts][D] */,
                                                        double* __restrict__ partial /* [n_shifts][gridDim.x] */) {
  using F = Family<FAM>;
  __shared__ double s_warp[8];
  const unsigned long long n = 1ULL << log2n, threads = (unsigned long long)gridDim.x * blockDim.x;
  const unsigned long long per = n / threads, i0 = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) * per;
  unsigned x[D];
#pragma unroll
  for (int j = 0; j < D; ++j) x[j] = 0u;
  for (unsigned long long gray = i0 ^ (i0 >> 1), b = 0; gray; gray >>= 1, ++b)
    if (gray & 1ULL) {
#pragma unroll
      for (int j = 0; j < D; ++j) x[j] ^= dirs[j * kSobolBits + b];
    }
  double sh[D];
#pragma unroll
  for (int j = 0; j < D; ++j) sh[j] = shifts[blockIdx.y * D + j];
  double acc = 0.0;
  for (unsigned long long i = i0; i < i0 + per; ++i) {
    double pt[D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const double v = (double)x[j] * 9.313225746154785e-10 + sh[j];   // base * 2^-30 (exact) + shift
      pt[j] = v - floor(v);
    }
    acc = acc + eval_at<F, D>(pt, f);
    const int c = __ffsll((long long)~i) - 1;     // index of the lowest zero bit of i
    if (c < kSobolBits) {
#pragma unroll
      for (int j = 0; j < D; ++j) x[j] ^= dirs[j * kSobolBits + c];
    }
  }
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) acc = acc + __shfl_xor_sync(PCB_FULL_MASK, acc, m);
  if ((threadIdx.x & 31) == 0) s_warp[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0)
    partial[(size_t)blockIdx.y * gridDim.x + blockIdx.x] =
        ((s_warp[0] + s_warp[1]) + (s_warp[2] + s_warp[3])) + ((s_warp[4] + s_warp[5]) + (s_warp[6] + s_warp[7]));
}

}  // namespace pcb
