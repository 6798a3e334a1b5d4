// PAGANI region evaluation, ONE REGION PER LANE, for the multiplicative families (f1, f4, f5, f6) and the
// default schedule width G = 64 (reference: pagani.py:195-224; arithmetic as in pagani_eval_mult.cuh).
//
// The Genz-Malik point set is the same for every region, so the natural SIMD axis on a GPU is the REGION:
// the 32 lanes of a warp walk the F rule points in lock-step, each on its own region.  Which point comes
// next, which axes it moves, which orbit weights apply -- all of that is warp-uniform and costs (almost)
// nothing per region; what is left per lane and point is three shared-memory gathers from the lane's own
// factor tables, two multiplies and the five weighted accumulations the reference schedule prescribes.
// The warp-per-region kernels spend ~1500 issue slots per region, 3/4 of them on index arithmetic and
// shuffles; this one spends ~500 and is bound by the FP64 pipe.
//
// Per lane (= region):
//   tables     phi[j][c] = factor_j(left_j + length_j * offset_c) for c in {0,3,4,5,6}; from them
//              Rab[a<b] = everything of a pair point but its two moved axes, Grp[g][combo] = corner
//              products over groups of three axes (same association as pagani_eval_mult.cuh, so the
//              two kernels agree bit for bit and a sharded list does not depend on who evaluates it);
//              term[j][c] for c in 0..4: the generic per-axis terms of the 4D+1 centre/axial points,
//              which are evaluated in the reference's own association (split-axis inputs).
//   axial      pre-pass: the 4D+1 centre/axial evaluations (a full transcendental each), dealt point by point
//              to the warps that share the tables; each value replaces the one term slot only it reads.
//              Split axis (first maximum of the fourth-difference indicator) from the stored values.
//   points     virtual thread vt = 0..63 outer, step s inner (point i = vt + 64 s), five partial sums
//              per virtual thread started from -0.0 (see pagani_eval.cuh), merged by a binary counter
//              whose add tree is the adjacent-pair tree of engine.tree_sum.  From D = 7 on the corner
//              points of a block share the table entries and the parity-rule weight of their upper bits.
//   finish     volume scaling, error estimate, coalesced stores.
// A non-finite evaluation poisons the sums; only then the points are walked again to find the first one.
#pragma once

#include <type_traits>

#include "pagani_eval_mult.cuh"

#ifndef PCB_LANES_GENERIC_W
#define PCB_LANES_GENERIC_W 0   // 4 or 8: force the chains per lane of the generic lane kernel (experiments); 0: measured choice
#endif
#ifndef PCB_LANES_AXIAL_UNROLL
#define PCB_LANES_AXIAL_UNROLL 2   // centre / axial evaluations in flight per warp (a full transcendental each)
#endif
#ifndef PCB_LANES_HALVES_REAL
#define PCB_LANES_HALVES_REAL 1   // 2: real families also split the virtual threads over two warps (measured slower: f4 d=8 0.57 vs 0.41 ms)
#endif

namespace pcb {

template <int D, bool UNIT = false, bool HALVES = false>
struct LaneLayout {
  static constexpr int kFe = (1 << D) + 2 * D * D + 2 * D + 1;
  static constexpr int kCorner0 = 2 * D * D + 2 * D + 1;
  static constexpr int kPairs = D * (D - 1) / 2;
  static constexpr int kGroups = (D + 2) / 3;
  static constexpr int kSteps = (kFe + 63) / 64;
  static constexpr int kP34 = 0;                                  // phi[j][3], phi[j][4] at 2j, 2j+1
  static constexpr int kRab = 2 * D;                              // unit-modulus families keep no Rab table (rho form)
  static constexpr int kGrp = kRab + (UNIT ? 0 : (kPairs > 0 ? kPairs : 1));  // Grp[g][combo] at kGrp + 8g + combo
  static constexpr int kTab = kGrp + 8 * kGroups;                 // V entries per lane
  static constexpr int kTerm = 5 * D;                             // doubles per lane: term[j][c], c = 0..4
  // term[j][c], c = 1..4, is replaced in place by the VALUE of the axial point (j, c) once the tables are complete
  // (every slot has exactly one reader, the warp that evaluates that point; the centre terms stay)
  // the two warps of a CTA share the tables of 32 regions and take virtual threads 0..31 and 32..63; the second
  // warp hands over its five sums.  Scratch per lane: the D centre factors while the tables are built, afterwards
  // the hand-over slots
  __host__ __device__ static constexpr size_t scratch_doubles(size_t vsize) {
    const size_t a = D * vsize / 8, b = HALVES ? 5 : 0;
    return a > b ? a : b;
  }
  static constexpr size_t smem_bytes(size_t vsize) {
    return 32 * (kTab * vsize + (size_t)kTerm * 8 + scratch_doubles(vsize) * 8) + 6 * 8 * 8;
  }
};

// Pair point q = 4 * pair + signs of the rule (quadrature.py:186-197) as data: the byte offsets, inside a lane's
// tables, of its three factors -- Rab[pair], phi[a][3 + (q & 1)], phi[b][3 + (q >> 1 & 1)].  Constant memory, indexed by
// loop counters only: the loads and the offsets stay on the uniform datapath and a gather is one shared-memory
// load with a uniform offset (the descriptors used to sit in shared memory: a mask / shift and a multiply-add per gather).
template <int D, bool UNIT, bool HALVES, int VSIZE>
struct PairPointTable {
  using L = LaneLayout<D, UNIT, HALVES>;
  unsigned w[4 * (L::kPairs > 0 ? L::kPairs : 1)][4];
  constexpr PairPointTable() : w{} {
    int e = 0;
    for (int a = 0; a < D; ++a)
      for (int b = a + 1; b < D; ++b, ++e)
        for (int sg = 0; sg < 4; ++sg) {
          unsigned* d = w[4 * e + sg];
          d[0] = (unsigned)(L::kRab + e) * 32u * VSIZE;
          d[1] = (unsigned)(L::kP34 + 2 * a + (sg & 1)) * 32u * VSIZE;
          d[2] = (unsigned)(L::kP34 + 2 * b + ((sg >> 1) & 1)) * 32u * VSIZE;
          d[3] = 0u;
        }
  }
};
template <int D, bool UNIT, bool HALVES, int VSIZE>
__constant__ PairPointTable<D, UNIT, HALVES, VSIZE> kPairPoints = PairPointTable<D, UNIT, HALVES, VSIZE>();

// level LEV of a binary counter over blocks: an odd index closes the pair (left + right) and carries upward
template <int LEV, int NLEV>
__device__ __forceinline__ void counter_merge(int blk, double (&cur)[5], double (&hold)[NLEV][5]) {
  if constexpr (LEV < NLEV) {
    if ((blk >> LEV) & 1) {
#pragma unroll
      for (int k = 0; k < 5; ++k) cur[k] = hold[LEV][k] + cur[k];
      counter_merge<LEV + 1, NLEV>(blk, cur, hold);
    } else {
#pragma unroll
      for (int k = 0; k < 5; ++k) hold[LEV][k] = cur[k];
    }
  }
}

// CTAs per SM the register allocation must leave room for: what the tables allow (227 KB of shared memory per SM),
// capped -- beyond ~10 resident warps the spills cost more than the occupancy brings
template <int FAM, int D>
constexpr int lanes_min_blocks() {
  constexpr bool cplx = MultFamily<FAM>::cplx || PCB_LANES_HALVES_REAL > 1;   // two warps per CTA
  constexpr size_t smem = LaneLayout<D, MultFamily<FAM>::unit, cplx>::smem_bytes(MultFamily<FAM>::cplx ? 16 : 8) + 1024;
  constexpr int by_smem = (int)((227u << 10) / smem);
#ifndef PCB_LANES_CPLX_CAP
#define PCB_LANES_CPLX_CAP 6
#endif
#ifndef PCB_LANES_CPLX_W
#define PCB_LANES_CPLX_W 4
#endif
  constexpr int cap = cplx ? PCB_LANES_CPLX_CAP : 10;
  return by_smem < 1 ? 1 : (by_smem < cap ? by_smem : cap);
}

template <int FAM, int D>
__global__ void __launch_bounds__((PCB_LANES_HALVES_REAL > 1 || MultFamily<FAM>::cplx) ? 64 : 32, lanes_min_blocks<FAM, D>())
pagani_eval_lanes_kernel(const __grid_constant__ EvalArgs args) {
  pdl_wait();   // region list and flags come from the kernels before it in the stream (programmatic serialisation)
  using F = Family<FAM>;
  using MF = MultFamily<FAM>;
  using V = MVal<MF::cplx>;
  using L = LaneLayout<D, MF::unit, (PCB_LANES_HALVES_REAL > 1 || MF::cplx)>;
  // Complex factors (f1) double the tables, and one warp per 48 KB of tables cannot hide the FP64 latency: there two
  // warps ("halves") share the tables of 32 regions and take virtual threads 0..31 and 32..63.  Real families run
  // one warp per CTA with twice the chains per lane (measured faster: no duplicated prologue, no CTA barriers).
  constexpr int kHalves = PCB_LANES_HALVES_REAL > 1 || MF::cplx ? 2 : 1;
  constexpr int kVt = 64 / kHalves;   // virtual threads per half
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // half h takes virtual threads kVt*h .. kVt*h + kVt - 1; read through a shuffle so that the compiler knows it is
  // warp-uniform and keeps the point bookkeeping that derives from it on the uniform datapath
  const int lane = threadIdx.x & 31, half = kHalves > 1 ? __shfl_sync(PCB_FULL_MASK, (int)(threadIdx.x >> 5), 0) : 0;
  auto cta_sync = [&]() { if constexpr (kHalves > 1) __syncthreads(); else __syncwarp(); };
  V* tab = reinterpret_cast<V*>(smem_raw) + lane;                                                   // entry e: tab[e * 32]
  double* term = reinterpret_cast<double*>(smem_raw + sizeof(V) * 32 * L::kTab) + lane;             // term[(5j + c) * 32]
  constexpr size_t kScratchD = L::scratch_doubles(sizeof(V));
  double* scratch = term + 32 * L::kTerm;
  V* cen_s = reinterpret_cast<V*>(smem_raw + sizeof(V) * 32 * L::kTab + 8 * 32 * L::kTerm) + lane;   // cen_s[j * 32] (table phase)
  double* xfer = scratch;                                                                           // xfer[k * 32]: the second half's sums
  double* s_w = reinterpret_cast<double*>(smem_raw + 32 * (sizeof(V) * L::kTab + 8 * L::kTerm + 8 * kScratchD));   // [6][8]

  const pcb_rule& rule = args.rule;
  if (threadIdx.x < 30) {  // orbit weights; rows 4 / 5: corners with even / odd bit count (quadrature.py:199-203)
    const int o = threadIdx.x / 5, k = threadIdx.x % 5;
    double w = rule.weights[k][o < 5 ? o : 4];
    if (o == 5 && rule.corner_parity[k]) w = -w;
    s_w[o * 8 + k] = w;
  }
  cta_sync();

  const double jac = args.f.bounded ? args.f.jac : 1.0;   // x * 1.0 == x
  const V one = mone(V{});

  // value of pair / corner points from the lane's tables
  V full = one;   // unit-modulus families: product of the centre factors of the current region
  auto tab_at = [&](unsigned byte_off) -> V {
    return *reinterpret_cast<const V*>(reinterpret_cast<const unsigned char*>(tab) + byte_off);
  };
  auto pair_value = [&](int i) -> double {
    const unsigned* dsc = kPairPoints<D, MF::unit, (PCB_LANES_HALVES_REAL > 1 || MF::cplx), (int)sizeof(V)>.w[i - 1 - 4 * D];
    const V lead = MF::unit ? full : tab_at(dsc[0]);
    const V v = mmul(mmul(lead, tab_at(dsc[1])), tab_at(dsc[2]));
    return v.re * jac;
  };
  auto corner_head = [&](unsigned bits) -> V {   // groups 0 and 1 (all groups when D < 6)
    V h = tab[(L::kGrp + (bits & 7u)) * 32];
    if constexpr (L::kGroups > 1) h = mmul(h, tab[(L::kGrp + 8 + ((bits >> 3) & 7u)) * 32]);
    return h;
  };
  auto corner_value = [&](V head, unsigned bits) -> double {
    V v = head;
#pragma unroll
    for (int g = 2; g < L::kGroups; ++g) v = mmul(v, tab[(L::kGrp + 8 * g + ((bits >> (3 * g)) & 7u)) * 32]);
    return v.re * jac;
  };
  // Centre / axial points keep the reference's own association (they decide the split axis).  Axial point q
  // (0-based: l2 pairs of axis 0, 1, ..., then the l3 pairs) moves axis q/2 to candidate 1 + (q & 1) [+ 2 for l3].
  auto axial_slot = [&](int q) -> int {
    const int a = (q >= 2 * D ? q - 2 * D : q) >> 1;
    return 5 * a + 1 + (q & 1) + (q >= 2 * D ? 2 : 0);
  };
  auto axial_eval = [&](int q) -> double {   // from the term table (before the slot is overwritten)
    const int slot = axial_slot(q), a = slot / 5;
    double t[D];
#pragma unroll
    for (int j = 0; j < D; ++j) t[j] = term[(j == a ? slot : 5 * j) * 32];
    return F::template finish<D>(combine_terms<F, D>(t), args.f) * jac;
  };
  auto centre_eval = [&]() -> double {
    double t[D];
#pragma unroll
    for (int j = 0; j < D; ++j) t[j] = term[(5 * j) * 32];
    return F::template finish<D>(combine_terms<F, D>(t), args.f) * jac;
  };
  double f_centre = 0.0;
  auto direct_value = [&](int i) -> double { return i == 0 ? f_centre : term[axial_slot(i - 1) * 32]; };

  for (long long batch = blockIdx.x; batch * 32 < args.n; batch += gridDim.x) {
    const long long r = batch * 32 + lane;
    const bool live = r < args.n;
    const long long rc = live ? r : args.n - 1;

    // ---- tables (loops over the axis are rolled: the kernel must stay inside the instruction cache)
    // with two halves, half 0 evaluates the centre and pair factors (c = 0, 3, 4) and the generic terms, half 1 the
    // corner factors (c = 5, 6) and the corner group tables: three and two transcendentals per axis
    double vol = 1.0;
    double next_left = args.lefts[rc], next_len = args.lengths[rc];
#pragma unroll 1
    for (int j = 0; j < D; ++j) {
      const double left = next_left, len = next_len;
      if (j + 1 < D) {   // the next axis' geometry travels while this axis' transcendentals are evaluated
        next_left = args.lefts[(j + 1) * args.ld + rc];
        next_len = args.lengths[(j + 1) * args.ld + rc];
      }
      vol = (j == 0) ? len : vol * len;   // np.prod, left to right
      V cg[2];
      if constexpr (MF::unit && PCB_F1_SHARED_TRIG) {
        // linear phase: centre factor and one rotation per offset (unit_rotation, pagani_eval_mult.cuh); half 0 builds
        // the pair candidates (rho = the rotation itself), half 1 the corner factors -- two sincos each
        double x0 = left + len * rule.offsets[0];
        if (args.f.bounded) x0 = args.f.low[j] + args.f.width[j] * x0;
        const V e0 = MF::factor(j, x0, args.f);
        if (kHalves == 1 || half == 0) {
#pragma unroll
          for (int c = 0; c < 5; ++c) {
            double x = left + len * rule.offsets[c];   // quadrature.py:301-302: mul, then add
            if (args.f.bounded) x = args.f.low[j] + args.f.width[j] * x;
            term[(5 * j + c) * 32] = F::term(j, x, args.f);
          }
          cen_s[j * 32] = e0;
          const V r3 = unit_rotation<MF>(j, len, rule.offsets[3], rule.offsets[0], args.f);
          tab[(L::kP34 + 2 * j) * 32] = r3;
          tab[(L::kP34 + 2 * j + 1) * 32] = mconj(r3);
        }
        if (kHalves == 1 || half == 1) {
          const V r5 = unit_rotation<MF>(j, len, rule.offsets[5], rule.offsets[0], args.f);
          cg[0] = mmul(e0, r5);
          cg[1] = mmul(e0, mconj(r5));
        }
      } else {
#pragma unroll
      for (int c = 0; c < 7; ++c) {
        if (kHalves > 1 && (c >= 5) != (half == 1)) continue;
        double x = left + len * rule.offsets[c];   // quadrature.py:301-302: mul, then add
        if (args.f.bounded) x = args.f.low[j] + args.f.width[j] * x;
        if (c < 5) term[(5 * j + c) * 32] = F::term(j, x, args.f);
        if (c == 1 || c == 2) continue;            // axial points never use a factor
        const V v = MF::factor(j, x, args.f);
        if (c == 0) cen_s[j * 32] = v;
        else if (c < 5) tab[(L::kP34 + 2 * j + (c - 3)) * 32] = MF::unit ? mmul(mconj(cen_s[j * 32]), v) : v;
        else cg[c - 5] = v;
      }
      }
      if (kHalves > 1 && half == 0) continue;
      // corner group tables: Grp[g][combo] = phi[3g][.] * phi[3g+1][.] * phi[3g+2][.], left to right
      const int g = j / 3, pos = j - 3 * g;
      V* grp = tab + (L::kGrp + 8 * g) * 32;
      if (pos == 0) {
        grp[0] = cg[0];
        grp[32] = cg[1];
      } else {
        const int half_n = 1 << pos;
#pragma unroll
        for (int combo = 0; combo < 4; ++combo) {
          if (combo < half_n) {
            const V lo = grp[combo * 32];
            grp[combo * 32] = mmul(lo, cg[0]);
            grp[(combo + half_n) * 32] = mmul(lo, cg[1]);
          }
        }
      }
    }
    cta_sync();
    // the 4D + 1 centre / axial evaluations, dealt to the halves point by point; each value replaces the one term
    // that only its own evaluation reads
    constexpr int kAxialUnroll = PCB_LANES_AXIAL_UNROLL;
#pragma unroll kAxialUnroll
    for (int q = half; q < 4 * D; q += kHalves) {
      const double fx = axial_eval(q);
      term[axial_slot(q) * 32] = fx;
    }
    if (!half) f_centre = centre_eval();
    // Rab[a][b] = (E[0][a] * E[a+1][b]) * E[b+1][D] with E[x][y] = ((1 * c_x) * c_{x+1}) ... * c_{y-1}; half h
    // stores the pairs with a = h (mod 2)
    if constexpr (MF::unit) {
      full = one;   // E[0][D] = ((1 * c_0) * c_1) ... * c_{D-1}
#pragma unroll
      for (int j = 0; j < D; ++j) full = mmul(full, cen_s[j * 32]);
    } else if constexpr (L::kPairs > 0) {
      V cen[D], tail[D];   // tail[b] = E[b+1][D]
#pragma unroll
      for (int j = 0; j < D; ++j) cen[j] = cen_s[j * 32];
#pragma unroll
      for (int b = 0; b < D; ++b) {
        V run = one;
#pragma unroll
        for (int k = b + 1; k < D; ++k) run = mmul(run, cen[k]);
        tail[b] = run;
      }
      V pre = one;   // E[0][a]
      int e = 0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        V mid = one;  // E[a+1][b]
#pragma unroll
        for (int b = a + 1; b < D; ++b) {
          if (kHalves == 1 || (a & 1) == half) {
            tab[(L::kRab + e) * 32] = mmul(mmul(pre, mid), tail[b]);
            mid = mmul(mid, cen[b]);
          }
          ++e;
        }
        pre = mmul(pre, cen[a]);
      }
    }
    cta_sync();   // tables and axial values complete; the centre factors' bytes become the hand-over slots

    // ---- rule points.  Virtual threads are taken W at a time (vt = W blk + v).  For a fixed step s the W points
    //      vt + 64 s of a block almost always belong to one orbit class, so the block is straight-line code over W
    //      independent dependency chains (that is what hides the FP64 latency with ~2 warps per scheduler); only
    //      the three blocks that straddle a class boundary take the point-by-point path.  The first log2(W)
    //      levels of the pair tree are fixed-register adds, the remaining ones a binary counter over the blocks.
    // chains per lane: where the tables leave room for >= 10 warps per SM (d <= 6) four chains and more warps win, above
    // that the eight-chain version hides the latency better (measured: f4 d=5 0.50 -> 0.42 ms, d=6 0.185 -> 0.161, d=8 0.41 vs 0.45)
    constexpr int W = kHalves > 1 ? PCB_LANES_CPLX_W : (D <= 6 ? 4 : 8);
    constexpr int kCounterLevels = (kVt / W) == 8 ? 3 : 4;   // log2(kVt / W)
    // split axis (pagani.py:215-223): first maximum over the axes of the fourth-difference indicator
    int axis = 0;
    if constexpr (D > 1) {
      if (!half) {
        const double two_f0 = 2.0 * f_centre;
        double best = -1.0;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const double d2 = (term[(5 * a + 1) * 32] + term[(5 * a + 2) * 32]) - two_f0;
          const double d3 = (term[(5 * a + 3) * 32] + term[(5 * a + 4) * 32]) - two_f0;
          const double ind = fabs(rule.split_weights[0] * d2 - rule.split_weights[1] * d3);
          if (ind > best) { best = ind; axis = a; }
        }
      }
    }
    double hold[kCounterLevels][5];
    double cur[5];
#pragma unroll 1
    for (int blk = 0; blk < kVt / W; ++blk) {
      const int vt0 = kVt * half + W * blk;
      double acc[W][5];
      V head[W];
#pragma unroll
      for (int v = 0; v < W; ++v) {
        const double init = vt0 + v < L::kFe ? -0.0 : 0.0;
#pragma unroll
        for (int k = 0; k < 5; ++k) acc[v][k] = init;
        head[v] = corner_head((unsigned)(vt0 + v - L::kCorner0) & 63u);
      }
      // Corner points of a block: bit pattern = b0 + v + 64 * (step offset).  While the W patterns share their bits
      // above the sixth (no carry inside the block) the tail groups and the sign of the parity rule's weight are the
      // same for all W chains: one table load and one weight per step.  The chain's own share of the parity sign
      // (bit count of its low six bits) is applied by keeping its parity-rule sum negated for the duration of the
      // corner steps -- negation commutes with every rounding, so the sums carry the same bits.
      // from D = 7 on a chain has several corner steps and the corners have upper bits to share; below, a chain meets
      // one corner at most and the plain path is faster (measured, d = 5 / 6: 5-20 %)
      constexpr bool kSharedCorners = D >= 7;
      const unsigned b0 = (unsigned)(vt0 - L::kCorner0) & 63u;
      // b0 = kC0 (mod W): in the one block per 64 / W that carries, chains kSplit .. W-1 have upper bits + 1
      constexpr int kC0 = (int)((64u * 64u - (unsigned)L::kCorner0) % (unsigned)W);
      const bool carry_free = b0 + W - 1 <= 63u;
      bool negated = false;
      // bit v: bit count of (b0 + v) mod 64 is odd (0x6996... is that parity for 0..63, rotated right by b0)
      const unsigned odd_chains = (unsigned)((0x6996966996696996ULL >> b0) | ((0x6996966996696996ULL << 1) << (63u - b0)));
      auto flip_parity_sums = [&]() {
#pragma unroll
        for (int v = 0; v < W; ++v) {
          const int hi = __double2hiint(acc[v][kParityRule]) ^ (int)((odd_chains << (31 - v)) & 0x80000000u);
          acc[v][kParityRule] = __hiloint2double(hi, __double2loint(acc[v][kParityRule]));
        }
        negated = !negated;
      };
      auto corner_step = [&](int lo, auto carries) {
        constexpr int kSplit = decltype(carries)::value ? W - kC0 : W;
        constexpr int kTails = L::kGroups > 2 ? L::kGroups - 2 : 1;
        const unsigned hb = (unsigned)(lo - L::kCorner0) >> 6;
        V tail[2][kTails];
        double w_par[2];
#pragma unroll
        for (int c = 0; c < (kSplit < W ? 2 : 1); ++c) {
#pragma unroll
          for (int g = 2; g < L::kGroups; ++g) tail[c][g - 2] = tab[(L::kGrp + 8 * g + (((hb + c) >> (3 * g - 6)) & 7u)) * 32];
          w_par[c] = (__popc(hb + c) & 1) ? -rule.weights[kParityRule][4] : rule.weights[kParityRule][4];
        }
        double fx[W];
#pragma unroll
        for (int v = 0; v < W; ++v) {
          V val = head[v];
#pragma unroll
          for (int g = 2; g < L::kGroups; ++g) val = mmul(val, tail[v < kSplit ? 0 : 1][g - 2]);
          fx[v] = val.re * jac;
        }
#pragma unroll
        for (int v = 0; v < W; ++v)
#pragma unroll
          for (int k = 0; k < 5; ++k)
            acc[v][k] = acc[v][k] + (k == kParityRule ? w_par[v < kSplit ? 0 : 1] : rule.weights[k][4]) * fx[v];
      };
#pragma unroll 1
      for (int s = 0; s < L::kSteps; ++s) {
        const int lo = vt0 + 64 * s, hi = lo + W - 1;
        if (kSharedCorners && lo >= L::kCorner0 && hi < L::kFe) {  // W corner points
          if (!negated) flip_parity_sums();
          if constexpr (kC0 != 0) {
            if (carry_free) corner_step(lo, std::false_type{});
            else corner_step(lo, std::true_type{});
          } else {
            corner_step(lo, std::false_type{});
          }
          continue;
        }
        if (kSharedCorners && negated) flip_parity_sums();
        if (hi <= 4 * D) {                                         // W centre / axial points
          double fx[W];
#pragma unroll
          for (int v = 0; v < W; ++v) fx[v] = direct_value(lo + v);
#pragma unroll
          for (int v = 0; v < W; ++v) {
            const double* w = s_w + 8 * (lo + v == 0 ? 0 : (lo + v <= 2 * D ? 1 : 2));
#pragma unroll
            for (int k = 0; k < 5; ++k) acc[v][k] = acc[v][k] + w[k] * fx[v];
          }
        } else if (lo > 4 * D && hi < L::kCorner0) {               // W pair points
          if constexpr (L::kPairs > 0) {
            double fx[W];
#pragma unroll
            for (int v = 0; v < W; ++v) fx[v] = pair_value(lo + v);
#pragma unroll
            for (int v = 0; v < W; ++v)
#pragma unroll
              for (int k = 0; k < 5; ++k) acc[v][k] = acc[v][k] + rule.weights[k][3] * fx[v];
          }
        } else if (!kSharedCorners && lo >= L::kCorner0 && hi < L::kFe) {   // W corner points, each with its own weights
          double fx[W];
#pragma unroll
          for (int v = 0; v < W; ++v) fx[v] = corner_value(head[v], (unsigned)(lo + v - L::kCorner0));
#pragma unroll
          for (int v = 0; v < W; ++v) {
            const double* w = s_w + 8 * (4 + (__popc((unsigned)(lo + v - L::kCorner0)) & 1));
#pragma unroll
            for (int k = 0; k < 5; ++k) acc[v][k] = acc[v][k] + w[k] * fx[v];
          }
        } else if (lo < L::kFe) {                                  // the block straddles a class boundary
#pragma unroll
          for (int v = 0; v < W; ++v) {
            const int i = lo + v;
            double fx;
            int row;   // orbit weights: centre, l2, l3, pairs, corners with even / odd bit count
            if (i <= 4 * D) {
              fx = direct_value(i);
              row = i == 0 ? 0 : (i <= 2 * D ? 1 : 2);
            } else if (i < L::kCorner0) {
              fx = L::kPairs > 0 ? pair_value(i) : 0.0;
              row = 3;
            } else if (i < L::kFe) {
              const unsigned bits = (unsigned)(i - L::kCorner0);
              fx = corner_value(head[v], bits);
              row = 4 + (__popc(bits) & 1);
            } else {
              continue;
            }
            const double* w = s_w + 8 * row;
#pragma unroll
            for (int k = 0; k < 5; ++k) acc[v][k] = acc[v][k] + w[k] * fx;
          }
        }
      }
      if (kSharedCorners && negated) flip_parity_sums();
      // pair tree inside the block: (v, v+1), then (v, v+2), ... always left + right (engine.py:80-84)
#pragma unroll
      for (int span = 1; span < W; span *= 2)
#pragma unroll
        for (int v = 0; v < W; v += 2 * span)
#pragma unroll
          for (int k = 0; k < 5; ++k) acc[v][k] = acc[v][k] + acc[v + span][k];
#pragma unroll
      for (int k = 0; k < 5; ++k) cur[k] = acc[0][k];
      // remaining levels: binary counter over the blocks
#ifdef PCB_EXP_COUNTER_LOCAL
      {
        int lev = 0;
#pragma unroll 1
        while ((blk >> lev) & 1) {
#pragma unroll
          for (int k = 0; k < 5; ++k) cur[k] = hold[lev][k] + cur[k];
          ++lev;
        }
#pragma unroll
        for (int k = 0; k < 5; ++k) hold[lev < kCounterLevels ? lev : 0][k] = cur[k];
      }
#else
      counter_merge<0, kCounterLevels>(blk, cur, hold);
#endif
    }
    // top level of the pair tree: virtual threads 0..31 (half 0) + 32..63 (half 1)
    if constexpr (kHalves > 1) {
      if (half) {
#pragma unroll
        for (int k = 0; k < 5; ++k) xfer[k * 32] = cur[k];
      }
      __syncthreads();
      if (!half) {
#pragma unroll
        for (int k = 0; k < 5; ++k) cur[k] = cur[k] + xfer[k * 32];
      }
    }

    double v[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) v[k] = vol * cur[k];
    if (live && !half) {
      if (!(isfinite(v[0]) && isfinite(v[1]) && isfinite(v[2]) && isfinite(v[3]) && isfinite(v[4]))) {
        // rare: find the first non-finite evaluation of this region (pagani.py:206-209)
        for (int i = 0; i < L::kFe; ++i) {
          double fx;
          if (i <= 4 * D) fx = direct_value(i);
          else if (i < L::kCorner0) fx = L::kPairs > 0 ? pair_value(i) : 0.0;
          else fx = corner_value(corner_head((unsigned)(i - L::kCorner0)), (unsigned)(i - L::kCorner0));
          if (!isfinite(fx)) {
            atomicMin(args.bad, (unsigned long long)r * (unsigned long long)L::kFe + (unsigned long long)i);
            break;
          }
        }
      }
      args.integrals[r] = v[0];
      args.errors[r] = region_error(v, rule, args.err_mode, args.rel_floor);
      args.split_axes[r] = axis;
    }
    cta_sync();   // the next batch's tables overwrite what half 0 has just read
  }
}

// ------------------------------------------------------------------------------------------------------------
// One region per lane for the families WITHOUT a multiplicative form (f2, f3, sum, constant): every rule point
// gathers its D per-axis terms from the lane's table term[j][c] (7 abscissae per axis) and combines them in
// numpy's own order, exactly as pagani_eval_kernel does -- the two kernels agree bit for bit, and for the
// families without a transcendental both agree bit for bit with the reference.
// ------------------------------------------------------------------------------------------------------------
template <int D>
struct GenericLaneLayout {
  static constexpr int kFe = (1 << D) + 2 * D * D + 2 * D + 1;
  static constexpr int kCorner0 = 2 * D * D + 2 * D + 1;
  static constexpr int kSteps = (kFe + 63) / 64;
  static constexpr int kTerm = 7 * D;   // doubles per lane
  static constexpr size_t smem_bytes() { return 32 * (size_t)(kTerm + D) * 8 + 6 * 8 * 8; }
};

// Centre / axial / pair point i of the rule (quadrature.py:168-197), as data: which abscissa c_j in 0..4 every axis
// takes (one byte per axis: `__byte_perm` turns byte j into the byte offset c_j * 256 of the lane's term table in ONE
// instruction) and the row of its orbit weights.  The table lives in constant memory and is indexed by loop
// counters only, so the loads, the extraction and the resulting offsets stay on the uniform datapath and the
// D gathers of a point are D shared-memory loads with a uniform offset -- until round 2 of this build the
// descriptor sat in shared memory and every gather paid two compares, two selects and a multiply-add per axis
// (18 % of the kernel's instructions, profiles/r2_ncu_pagani_lanes_f3_d8_before.txt).
template <int D>
struct PlainPointTable {
  unsigned w[2 * D * D + 2 * D + 1][4];   // [i][0..2]: bytes c_0..c_11, [i][3]: orbit row
  constexpr PlainPointTable() : w{} {
    const int n = 2 * D * D + 2 * D + 1;
    for (int i = 0; i < n; ++i) {
      int a = -1, b = -1, ca = 0, cb = 0, orbit = 0;
      if (i == 0) {
      } else if (i <= 2 * D) {
        const int q = i - 1; a = q >> 1; ca = 1 + (q & 1); orbit = 1;
      } else if (i <= 4 * D) {
        const int q = i - 1 - 2 * D; a = q >> 1; ca = 3 + (q & 1); orbit = 2;
      } else {
        const int q = i - 1 - 4 * D, pr = q >> 2, sg = q & 3;
        int idx = 0;
        for (int j = 0; j < D; ++j)
          for (int k = j + 1; k < D; ++k, ++idx)
            if (idx == pr) { a = j; b = k; }
        ca = 3 + (sg & 1); cb = 3 + (sg >> 1); orbit = 3;
      }
      for (int k = 0; k < 4; ++k) w[i][k] = 0u;
      if (a >= 0) w[i][a >> 2] |= (unsigned)ca << (8 * (a & 3));
      if (b >= 0) w[i][b >> 2] |= (unsigned)cb << (8 * (b & 3));
      w[i][3] = (unsigned)orbit;
    }
  }
};
template <int D>
__constant__ PlainPointTable<D> kPlainPoints = PlainPointTable<D>();

// corner combine over the lane's table, same association as CornerCombine (pagani_eval.cuh)
template <class F, int D>
struct LaneCorner {
  static constexpr int LO = D < 6 ? D : 6;
  double p0, p1;
  __device__ __forceinline__ static double at(const double* term, int j, unsigned bit) { return term[(7 * j + 5 + (int)bit) * 32]; }
  __device__ __forceinline__ void head(const double* term, unsigned bits) {
    double t[LO];
#pragma unroll
    for (int j = 0; j < LO; ++j) t[j] = at(term, j, (bits >> j) & 1u);
    if constexpr (F::combine == kSumNumpy && D >= 8) {
      p0 = (t[0] + t[1]) + (t[2] + t[3]);
      p1 = t[4] + t[5];
    } else {
      double s = t[0];
#pragma unroll
      for (int j = 1; j < LO; ++j) s = (F::combine == kProdSeq) ? s * t[j] : s + t[j];
      p0 = s; p1 = 0.0;
    }
  }
  // the terms of the axes above the sixth depend on the upper bits only: shared by the points of a carry-free block
  static constexpr int kUp = D > LO ? D - LO : 1;
  __device__ __forceinline__ static void upper(const double* term, unsigned upper_bits, double (&up)[kUp]) {
#pragma unroll
    for (int j = LO; j < D; ++j) up[j - LO] = at(term, j, (upper_bits >> (j - LO)) & 1u);
  }
  __device__ __forceinline__ double tail_up(const double (&up)[kUp]) const {
    if constexpr (F::combine == kSumNumpy && D >= 8) {
      double s = p0 + (p1 + (up[0] + up[1]));
#pragma unroll
      for (int j = 8; j < D; ++j) s = s + up[j - LO];
      return s;
    } else {
      double s = p0;
#pragma unroll
      for (int j = LO; j < D; ++j) s = (F::combine == kProdSeq) ? s * up[j - LO] : s + up[j - LO];
      return s;
    }
  }
  __device__ __forceinline__ double tail(const double* term, unsigned bits) const {
    double up[kUp];
    upper(term, bits >> LO, up);
    return tail_up(up);
  }
};

#ifndef PCB_LANES_GENERIC_MINB
#define PCB_LANES_GENERIC_MINB 12
#endif
// Independent dependency chains per lane.  Eight chains at 255 registers (8 resident warps per SM) against four at
// 168 (12 warps), measured on lists of 2.5e5 .. 1.7e6 regions after the point descriptors moved to constant memory
// [r2]: f3 gains at every d (its final map is a 19-operation FP64 chain per point: d=8 2.16 -> 2.48e11 evaluations/s,
// d=6 1.45 -> 2.19e11); f2 gains for d = 6..9 (d=8 3.74 -> 4.13e11, d=6 2.72 -> 3.06e11) and loses outside
// (d=5 2.36 -> 2.09e11, d=10 5.68 -> 5.17e11).
template <int FAM, int D>
__host__ __device__ constexpr int generic_lane_chains() {
  if (PCB_LANES_GENERIC_W != 0) return PCB_LANES_GENERIC_W;
  if (FAM == PCB_F3_CORNER_PEAK) return 8;
  return (D >= 6 && D <= 9) ? 8 : 4;
}
template <int FAM, int D>
__global__ void __launch_bounds__(32, generic_lane_chains<FAM, D>() == 8 ? 1 : PCB_LANES_GENERIC_MINB) pagani_eval_lanes_generic_kernel(const __grid_constant__ EvalArgs args) {
  pdl_wait();   // region list and flags come from the kernels before it in the stream (programmatic serialisation)
  using F = Family<FAM>;
  using L = GenericLaneLayout<D>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x;
  double* term = reinterpret_cast<double*>(smem_raw) + lane;               // term[(7j + c) * 32]
  double* stash = term + 32 * L::kTerm;                                    // stash[j * 32]
  double* s_w = reinterpret_cast<double*>(smem_raw + 32 * (size_t)(L::kTerm + D) * 8);   // [6][8]

  const pcb_rule& rule = args.rule;
  if (lane < 30) {  // orbit weights; rows 4 / 5: corners with even / odd bit count (quadrature.py:199-203)
    const int o = lane / 5, k = lane % 5;
    double w = rule.weights[k][o < 5 ? o : 4];
    if (o == 5 && rule.corner_parity[k]) w = -w;
    s_w[o * 8 + k] = w;
  }
  __syncwarp();
  const double jac = args.f.bounded ? args.f.jac : 1.0;   // x * 1.0 == x

  // centre / axial / pair point i: its D terms combined in numpy's order (the final map is applied W points at a time)
  auto plain_sum = [&](int i, int& row) -> double {
    const unsigned* dsc = kPlainPoints<D>.w[i];
    row = (int)dsc[3];
    double t[D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const unsigned off = __byte_perm(dsc[j >> 2], 0u, 0x4404u | ((unsigned)(j & 3) << 4));   // c_j * 256 bytes
      t[j] = *reinterpret_cast<const double*>(reinterpret_cast<const unsigned char*>(term) + 7 * j * 256 + off);
    }
    return combine_terms<F, D>(t);
  };
  // The final map of W independent points.  A family whose map has an off-domain branch (f3: libm semantics for
  // 1 + s <= 0 and the extremes) offers a branch-free form for arguments known to be in the domain; `fast` (warp-
  // uniform: every lane's region keeps all its sums inside the domain) selects it, and the W dependency chains
  // become one straight-line block the compiler interleaves.  With the branch inside every evaluation the chains ran
  // one after the other and the kernel waited on the FP64 latency (f3 d=8: 0.70 -> see DESIGN 4.1).
  bool fast = true;
  auto finish_block = [&](auto& sums) {
    constexpr int N = (int)(sizeof(sums) / sizeof(double));
    if constexpr (HasIndomainFinish<F>::value) {
      if (fast) {
        F::template finish_indomain_many<D, N>(sums, args.f);
#pragma unroll
        for (int v = 0; v < N; ++v) sums[v] = sums[v] * jac;
      } else {
#pragma unroll
        for (int v = 0; v < N; ++v) sums[v] = finish_out_of_line<F, D>(sums[v], args.f) * jac;
      }
    } else {
#pragma unroll
      for (int v = 0; v < N; ++v) sums[v] = F::template finish<D>(sums[v], args.f) * jac;
    }
  };
  auto finish_one = [&](double sum) -> double {
    if constexpr (HasIndomainFinish<F>::value) return finish_out_of_line<F, D>(sum, args.f) * jac;
    else return F::template finish<D>(sum, args.f) * jac;
  };

  for (long long batch = blockIdx.x; batch * 32 < args.n; batch += gridDim.x) {
    const long long r = batch * 32 + lane;
    const bool live = r < args.n;
    const long long rc = live ? r : args.n - 1;
    double vol = 1.0;
    double next_left = args.lefts[rc], next_len = args.lengths[rc];
    double sum_min = 0.0, sum_abs = 0.0;   // bounds of the combined sums of this region (families with a domain)
#pragma unroll 1
    for (int j = 0; j < D; ++j) {
      const double left = next_left, len = next_len;
      if (j + 1 < D) {
        next_left = args.lefts[(j + 1) * args.ld + rc];
        next_len = args.lengths[(j + 1) * args.ld + rc];
      }
      vol = (j == 0) ? len : vol * len;   // np.prod, left to right
      double t_min = 0.0, t_abs = 0.0;
#pragma unroll
      for (int c = 0; c < 7; ++c) {
        const double x = left + len * rule.offsets[c];   // quadrature.py:301-302: mul, then add
        const double t = axis_term<F>(j, x, args.f);
        term[(7 * j + c) * 32] = t;
        if constexpr (HasIndomainFinish<F>::value) {
          t_min = c == 0 ? t : fmin(t_min, t);
          t_abs = c == 0 ? fabs(t) : fmax(t_abs, fabs(t));
        }
      }
      sum_min += t_min;
      sum_abs += t_abs;
    }
    if constexpr (HasIndomainFinish<F>::value) fast = __all_sync(PCB_FULL_MASK, F::sums_indomain(sum_min, sum_abs));

    constexpr int W = generic_lane_chains<FAM, D>();
    constexpr int kLevels = W == 8 ? 3 : 4;   // log2(64 / W)
    double two_f0 = 0.0, first_of_pair = 0.0, best = -1.0;
    int axis = 0;
    auto split_note = [&](int i, double fx) {   // pagani.py:215-223: running first maximum over the axes
      if constexpr (D > 1) {
        if (i > 4 * D) return;
        const int q = i - 1;
        if (i == 0) two_f0 = 2.0 * fx;
        else if (!(q & 1)) first_of_pair = fx;
        else {
          const double d2 = (first_of_pair + fx) - two_f0;
          const int a = (q >= 2 * D ? q - 2 * D : q) >> 1;
          if (q < 2 * D) stash[a * 32] = d2;
          else {
            const double ind = fabs(rule.split_weights[0] * stash[a * 32] - rule.split_weights[1] * d2);
            if (ind > best) { best = ind; axis = a; }
          }
        }
      }
    };
    double hold[kLevels][5];
    double cur[5];
#pragma unroll 1
    for (int blk = 0; blk < 64 / W; ++blk) {
      const int vt0 = W * blk;
      double acc[W][5];
      LaneCorner<F, D> head[W];
#pragma unroll
      for (int v = 0; v < W; ++v) {
        const double init = vt0 + v < L::kFe ? -0.0 : 0.0;
#pragma unroll
        for (int k = 0; k < 5; ++k) acc[v][k] = init;
        head[v].head(term, (unsigned)(vt0 + v - L::kCorner0) & 63u);
      }
      // corner steps: shared upper terms, one parity-rule weight per step, the chain's own parity carried by its
      // negated parity-rule sum (see pagani_eval_lanes_kernel)
      // from D = 7 on a chain has several corner steps and the corners have upper bits to share; below, a chain meets
      // one corner at most and the plain path is faster (measured, d = 5 / 6: 5-20 %)
      constexpr bool kSharedCorners = D >= 7;
      const unsigned b0 = (unsigned)(vt0 - L::kCorner0) & 63u;
      constexpr int kC0 = (int)((64u * 64u - (unsigned)L::kCorner0) % (unsigned)W);
      const bool carry_free = b0 + W - 1 <= 63u;
      bool negated = false;
      // bit v: bit count of (b0 + v) mod 64 is odd (0x6996... is that parity for 0..63, rotated right by b0)
      const unsigned odd_chains = (unsigned)((0x6996966996696996ULL >> b0) | ((0x6996966996696996ULL << 1) << (63u - b0)));
      auto flip_parity_sums = [&]() {
#pragma unroll
        for (int v = 0; v < W; ++v) {
          const int hi = __double2hiint(acc[v][kParityRule]) ^ (int)((odd_chains << (31 - v)) & 0x80000000u);
          acc[v][kParityRule] = __hiloint2double(hi, __double2loint(acc[v][kParityRule]));
        }
        negated = !negated;
      };
      auto corner_step = [&](int lo, auto carries) {
        constexpr int kSplit = decltype(carries)::value ? W - kC0 : W;
        const unsigned hb = (unsigned)(lo - L::kCorner0) >> 6;
        double up[2][LaneCorner<F, D>::kUp];
        double w_par[2];
#pragma unroll
        for (int c = 0; c < (kSplit < W ? 2 : 1); ++c) {
          LaneCorner<F, D>::upper(term, hb + c, up[c]);
          w_par[c] = (__popc(hb + c) & 1) ? -rule.weights[kParityRule][4] : rule.weights[kParityRule][4];
        }
        double fx[W];
#pragma unroll
        for (int v = 0; v < W; ++v) fx[v] = head[v].tail_up(up[v < kSplit ? 0 : 1]);
        finish_block(fx);
#pragma unroll
        for (int v = 0; v < W; ++v)
#pragma unroll
          for (int k = 0; k < 5; ++k)
            acc[v][k] = acc[v][k] + (k == kParityRule ? w_par[v < kSplit ? 0 : 1] : rule.weights[k][4]) * fx[v];
      };
#pragma unroll 1
      for (int s = 0; s < L::kSteps; ++s) {
        const int lo = vt0 + 64 * s, hi = lo + W - 1;
        if (kSharedCorners && lo >= L::kCorner0 && hi < L::kFe) {  // W corner points
          if (!negated) flip_parity_sums();
          if constexpr (kC0 != 0) {
            if (carry_free) corner_step(lo, std::false_type{});
            else corner_step(lo, std::true_type{});
          } else {
            corner_step(lo, std::false_type{});
          }
          continue;
        }
        if (kSharedCorners && negated) flip_parity_sums();
        if (hi < L::kCorner0) {                                    // W centre / axial / pair points
          double fx[W];
          int row[W];
#pragma unroll
          for (int v = 0; v < W; ++v) fx[v] = plain_sum(lo + v, row[v]);
          finish_block(fx);
#pragma unroll
          for (int v = 0; v < W; ++v) {
            split_note(lo + v, fx[v]);
            const double* w = s_w + 8 * row[v];
#pragma unroll
            for (int k = 0; k < 5; ++k) acc[v][k] = acc[v][k] + w[k] * fx[v];
          }
        } else if (!kSharedCorners && lo >= L::kCorner0 && hi < L::kFe) {   // W corner points, each with its own weights
          double fx[W];
#pragma unroll
          for (int v = 0; v < W; ++v) fx[v] = head[v].tail(term, (unsigned)(lo + v - L::kCorner0));
          finish_block(fx);
#pragma unroll
          for (int v = 0; v < W; ++v) {
            const double* w = s_w + 8 * (4 + (__popc((unsigned)(lo + v - L::kCorner0)) & 1));
#pragma unroll
            for (int k = 0; k < 5; ++k) acc[v][k] = acc[v][k] + w[k] * fx[v];
          }
        } else if (lo < L::kFe) {                                  // the block straddles a class boundary
#pragma unroll
          for (int v = 0; v < W; ++v) {
            const int i = lo + v;
            double fx;
            int row;
            if (i < L::kCorner0) {
              fx = finish_one(plain_sum(i, row));
              split_note(i, fx);
            } else if (i < L::kFe) {
              const unsigned bits = (unsigned)(i - L::kCorner0);
              fx = finish_one(head[v].tail(term, bits));
              row = 4 + (__popc(bits) & 1);
            } else {
              continue;
            }
            const double* w = s_w + 8 * row;
#pragma unroll
            for (int k = 0; k < 5; ++k) acc[v][k] = acc[v][k] + w[k] * fx;
          }
        }
      }
      if (kSharedCorners && negated) flip_parity_sums();
#pragma unroll
      for (int span = 1; span < W; span *= 2)
#pragma unroll
        for (int v = 0; v < W; v += 2 * span)
#pragma unroll
          for (int k = 0; k < 5; ++k) acc[v][k] = acc[v][k] + acc[v + span][k];
#pragma unroll
      for (int k = 0; k < 5; ++k) cur[k] = acc[0][k];
      counter_merge<0, kLevels>(blk, cur, hold);
    }

    double v[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) v[k] = vol * cur[k];
    if (live) {
      if (!(isfinite(v[0]) && isfinite(v[1]) && isfinite(v[2]) && isfinite(v[3]) && isfinite(v[4]))) {
        // rare: find the first non-finite evaluation of this region (pagani.py:206-209)
        for (int i = 0; i < L::kFe; ++i) {
          double fx;
          int row;
          if (i < L::kCorner0) fx = finish_one(plain_sum(i, row));
          else {
            LaneCorner<F, D> cc;
            const unsigned bits = (unsigned)(i - L::kCorner0);
            cc.head(term, bits & 63u);
            fx = finish_one(cc.tail(term, bits));
          }
          if (!isfinite(fx)) {
            atomicMin(args.bad, (unsigned long long)r * (unsigned long long)L::kFe + (unsigned long long)i);
            break;
          }
        }
      }
      args.integrals[r] = v[0];
      args.errors[r] = region_error(v, rule, args.err_mode, args.rel_floor);
      args.split_axes[r] = axis;
    }
  }
}

}  // namespace pcb
