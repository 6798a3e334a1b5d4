// m-Cubes C-ABI: V-Sample pass, grid refinement and the iteration driver.
// Reference: mcubes.py:210-382, vegas_grid.py:133-193.
#include "mcubes_aux.cuh"
#include "mcubes_kernels.cuh"
#include "pcb_host.h"

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace pcb {

enum { M_BAD = 0, M_CLAMPS = 1, M_INTEGRAL = 2, M_VARIANCE = 3 };  // slots in ctx->scalars (offset 40)
constexpr int kMcSlot = 40;

struct SampleLaunch {
  int blocks = 0;        // CTAs (kSampleWarps warps each)
  size_t smem = 0;       // boundaries + table rows + staged records
  int nseg = 1;
  long long seg_len = 0;
};

static pcb_status validate_plan(pcb_ctx* ctx, const pcb_integrand* f, const pcb_mcubes_plan* plan) {
  if (!plan) return fail(ctx, PCB_INVALID, "plan is NULL");
  if (plan->d != f->d) return fail(ctx, PCB_INVALID, "plan, grid, and integrand dimensions must agree");
  if (plan->g < 1 || plan->p < 2 || plan->s < 1 || plan->group_size < 1 || plan->n_bins < 2)
    return fail(ctx, PCB_INVALID, "plan needs g >= 1, p >= 2, s >= 1, group_size >= 1, n_bins >= 2");
  long double m = 1;
  for (int j = 0; j < plan->d; ++j) m *= plan->g;
  if (m != (long double)plan->m) return fail(ctx, PCB_INVALID, "m must equal g^d");
  if (plan->group_size > 4096) return fail(ctx, PCB_INVALID, "group_size %d > 4096 unsupported", plan->group_size);
  if (plan->n_bins > 65535) return fail(ctx, PCB_INVALID, "n_bins %d > 65535 unsupported (16-bit bin ids)", plan->n_bins);
  return PCB_OK;
}

static pcb_status plan_launch(pcb_ctx* ctx, const pcb_mcubes_plan* plan, long long n_local_threads, SampleLaunch* out) {
  out->smem = vsample_smem_bytes(plan->d, plan->n_bins);
  if (out->smem > ctx->smem_optin)
    return fail(ctx, PCB_INVALID, "d=%d, n_bins=%d needs %zu B of shared memory per CTA, device offers %zu", plan->d,
                plan->n_bins, out->smem, ctx->smem_optin);
  // Segments per logical thread are a function of the PLAN, not of the shard: a thread's (I, Var) is the serial sum of
  // its segment sums, so a shard must cut its threads exactly like the single-device run to reproduce its bits.
  const long long n_lw = ((plan->m + plan->s - 1) / plan->s + 31) / 32;
  // work units = 32 segments; aim at >= 8 units per resident warp for balance
  const int ctas_per_sm = vsample_ctas_per_sm(plan->d);   // __launch_bounds__ of vsample_kernel   // __launch_bounds__ of vsample_kernel
  const long long resident = (long long)ctas_per_sm * ctx->sm_count * kSampleWarps;
  int nseg = (int)std::max<long long>(1, std::min<long long>(plan->s, (8 * resident + n_lw - 1) / n_lw));
  if (const char* env = std::getenv("PCB_MCUBES_SEGMENTS")) {
    int v = std::atoi(env);
    if (v >= 1) nseg = (int)std::min<long long>(plan->s, v);
  }
  const long long seg_len = (plan->s + nseg - 1) / nseg;
  out->seg_len = seg_len;
  out->nseg = (int)((plan->s + seg_len - 1) / seg_len);
  const long long units = (n_local_threads * out->nseg + 31) / 32;
  out->blocks = (int)std::max<long long>(1, std::min<long long>((long long)ctas_per_sm * ctx->sm_count, (units + kSampleWarps - 1) / kSampleWarps));
  return PCB_OK;
}

// Multiplier A of the lane -> segment map sigma = ((u*32 + lane) * A) mod N (mcubes_kernels.cuh).  Lane-to-lane
// offset in sub-cubes is ~A*seg_len; the ideal offset is (1,1,...,1) in base g, which gives the 32 lanes of a warp
// different coordinates -- hence different importance-grid windows -- on every axis.  Candidates around that
// value (coprime to N) are scored by counting equal-coordinate lane pairs over a few sample units.
static unsigned long long choose_segment_multiplier(pcb_ctx* ctx, const pcb_mcubes_plan* plan, long long t_begin, long long nt,
                                                    int nseg, long long seg_len) {
  const long long N = nt * nseg;
  if (N <= 1 || N >= (1LL << 31)) return 1;  // (u*32+lane)*A must stay below 2^63
  const std::array<long long, 6> key = {plan->g * 100 + plan->d, plan->s, t_begin, nt, nseg, seg_len};
  auto hit = ctx->mc_multipliers.find(key);
  if (hit != ctx->mc_multipliers.end()) return hit->second;
  const int d = plan->d;
  const long long g = plan->g;
  auto gcd = [](long long a, long long b) { while (b) { long long t = a % b; a = b; b = t; } return a; };
  auto score = [&](long long A) {
    long long total = 0;
    const long long units = (N + 31) / 32;
    for (int smp = 0; smp < 8; ++smp) {
      const long long u = units * smp / 8;
      int coords[32][PCB_MAX_DIM];
      int live = 0;
      for (int lane = 0; lane < 32; ++lane) {
        const long long sin = u * 32 + lane;
        if (sin >= N) break;
        const long long sigma = (long long)(((unsigned __int128)sin * (unsigned __int128)A) % (unsigned __int128)N);
        long long cube = (t_begin + sigma / nseg) * plan->s + (sigma % nseg) * seg_len;
        for (int j = d - 1; j >= 0; --j) { coords[lane][j] = (int)(cube % g); cube /= g; }
        ++live;
      }
      for (int j = 0; j < d; ++j)
        for (int x = 0; x < live; ++x)
          for (int y = x + 1; y < live; ++y) total += coords[x][j] == coords[y][j];
    }
    return total;
  };
  long long delta = 0;  // (1,1,...,1) in base g
  for (int j = 0; j < d; ++j) delta = delta * g + 1;
  std::vector<long long> cands = {1};
  const long long base = std::max<long long>(1, delta / std::max<long long>(1, seg_len));
  for (long long k = -48; k <= 48; ++k) cands.push_back(base + k);
  for (long long k = -8; k <= 8; ++k) { cands.push_back((long long)(N * 0.6180339887) + k); cands.push_back((long long)(N * 0.3819660113) + k); }
  long long best = 1, best_score = -1;
  for (long long c : cands) {
    long long A = ((c % N) + N) % N;
    if (A < 1 || gcd(A, N) != 1) continue;
    const long long sc = score(A);
    if (best_score < 0 || sc < best_score) { best = A; best_score = sc; }
  }
  ctx->mc_multipliers[key] = (unsigned long long)best;
  return (unsigned long long)best;
}

static pcb_status read_mc_scalars(pcb_ctx* ctx) {
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync((double*)ctx->pinned + kMcSlot, ctx->scalars.as<double>() + kMcSlot, 4 * sizeof(double),
                                    cudaMemcpyDeviceToHost, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return PCB_OK;
}

static pcb_status grant_smem(pcb_ctx* ctx, const void* fn, size_t bytes) {
  // Every kernel of the pass chain asks for the same (maximal) shared-memory carve-out: a launch whose carve-out
  // differs from its predecessor's makes the SMs drain and reconfigure, and cannot become resident beside it.
  if (ctx->smem_attr.find(fn) == ctx->smem_attr.end())
    PCB_CUDA_TRY(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared));
  size_t& have = ctx->smem_attr[fn];  // cudaFuncSetAttribute is not free: once per kernel and size
  if (have < bytes) {
    PCB_CUDA_TRY(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    have = bytes;
  }
  return PCB_OK;
}

// What the end-of-pass launch does besides the group-order tree: grid refinement, the iteration record
// and the stop decision of pcb_mcubes_run.
struct PassTail {
  int iteration = 0;
  int* stop = nullptr;                 // device; run only
  bool refine = false;
  double alpha = 1.5;
  int smoothing = 1;
  const double* bounds_in = nullptr;   // device
  double* bounds_out = nullptr;        // device
  double* contrib_copy = nullptr;      // device slot of the run's per-iteration tables (optional)
  double* hist_i = nullptr;            // device run history
  double* hist_v = nullptr;
  double rel_tol = 0.0, abs_tol = 0.0;
  McRecord* record = nullptr;          // pinned
  unsigned long long seq = 0;
  unsigned long long* timeline = nullptr;  // device; debug
  // sharded runs (pcb_mcubes_shard_*): the rank's packed row replaces ctx->mc_group, the end-of-pass launch is
  // enqueued separately (behind the collectives) and reads the gathered rows
  double* row = nullptr;               // device: [2 * width] group pairs, then bad, clamps
  long long row_doubles = 0;
  bool defer_finish = false;
  bool grid_in_unit = true;     // every boundary lies in [0, 1] (always true for grids refined on the device)
  const double* gathered = nullptr;    // device: world rows
  int world = 0;
  long long total_groups = 0;
};

// End-of-pass launch: group-order tree over the work-groups, grid refinement, iteration record, stop decision.
static pcb_status enqueue_finish(pcb_ctx* ctx, const pcb_mcubes_plan* plan, const PassTail& tail, long long n_groups) {
  const int d = plan->d, nb = plan->n_bins;
  unsigned long long* sc_u = ctx->scalars.as<unsigned long long>() + kMcSlot;
  double* sc = ctx->scalars.as<double>() + kMcSlot;
  FinishArgs fa;
  fa.n_groups = (int)n_groups;
  fa.group_pairs = ctx->mc_group.as<double>();
  fa.world = 0;
  fa.row_stride = 0;
  if (tail.gathered) {
    if (tail.total_groups > 1024) return fail(ctx, PCB_INVALID, "sharded mcubes_run supports at most 1024 work-groups (%lld requested)", tail.total_groups);
    fa.n_groups = (int)tail.total_groups;
    fa.group_pairs = tail.gathered;
    fa.world = tail.world;
    fa.row_stride = tail.row_doubles;
  } else if (n_groups > 1024) {  // engine.reduce in group order over more groups than one CTA holds (never with the default plans)
    if (tail.stop) return fail(ctx, PCB_INVALID, "mcubes_run supports at most 1024 work-groups (%lld requested)", n_groups);
    double* gi = ctx->mc_group.as<double>() + 2 * n_groups;
    double* ge = gi + n_groups;
    deinterleave2_kernel<<<(unsigned)((n_groups + 255) / 256), 256, 0, ctx->stream>>>(ctx->mc_group.as<double>(), (int)n_groups, gi, ge);
    ctx->launches++;
    PCB_CUDA_TRY(ctx, cudaGetLastError());
    PCB_TRY(tree_sum_dev(ctx, gi, n_groups, sc + M_INTEGRAL));
    PCB_TRY(tree_sum_dev(ctx, ge, n_groups, sc + M_VARIANCE));
    fa.n_groups = 0;
  }
  fa.refine.d = d; fa.refine.n = nb; fa.refine.alpha = tail.alpha; fa.refine.smoothing = tail.smoothing;
  fa.refine.boundaries = tail.bounds_in; fa.refine.contrib = ctx->mc_contrib.as<double>(); fa.refine.new_boundaries = tail.bounds_out;
  fa.n_refine = tail.refine ? d : 0;
  fa.stop = tail.stop;
  fa.scalars = sc_u;
  fa.hist_i = tail.hist_i;
  fa.hist_v = tail.hist_v;
  fa.iteration = tail.iteration;
  fa.rel_tol = tail.rel_tol;
  fa.abs_tol = tail.abs_tol;
  fa.record = tail.record;
  fa.seq = tail.seq;
  fa.timeline = tail.timeline;
  fa.refine.phase_tl = (tail.timeline && tail.iteration == 1) ? tail.timeline + 200 : nullptr;
  const size_t finish_smem = std::max<size_t>(refine_smem_doubles(nb), 2048) * sizeof(double);
  if (finish_smem > ctx->smem_optin) return fail(ctx, PCB_INVALID, "n_bins %d too large for on-device refinement", nb);
  PCB_TRY(grant_smem(ctx, (const void*)&finish_kernel, finish_smem));
  {
    void* args[] = {&fa};
    PCB_CUDA_TRY(ctx, launch_pdl((const void*)&finish_kernel, dim3(fa.n_refine + 1), dim3(512), args, finish_smem, ctx->stream));
    ctx->launches++;
  }
  return PCB_OK;
}

// PCB_FAST_DOMAIN (pcb_device.cuh): can the sampler evaluate the family's inner operations without their range tests?
// Samples are grid points in [0, 1]^d pushed through the optional affine map of scale_to_bounds.
static int sampler_fast_domain(const pcb_integrand* f, bool grid_in_unit) {
  if (!grid_in_unit) return 0;
  double lo[PCB_MAX_DIM], hi[PCB_MAX_DIM];
  for (int j = 0; j < f->d; ++j) {
    lo[j] = f->bounded ? f->low[j] : 0.0;
    hi[j] = f->bounded ? f->low[j] + f->width[j] : 1.0;
    if (!(std::isfinite(lo[j]) && std::isfinite(hi[j]))) return 0;
    if (lo[j] > hi[j]) std::swap(lo[j], hi[j]);
  }
  if (f->family == PCB_F2_PRODUCT_PEAK) {          // a2 + u*u normal with a normal reciprocal
    if (!(f->param[0] >= 0x1p-900 && f->param[0] <= 0x1p900)) return 0;
    for (int j = 0; j < f->d; ++j)
      if (!(std::fmax(std::fabs(lo[j] - 0.5), std::fabs(hi[j] - 0.5)) <= 0x1p400)) return 0;
    return PCB_FAST_DOMAIN;
  }
  if (f->family == PCB_F3_CORNER_PEAK) {           // 1 + sum (j+1) x_j in [2^-20, 2^21], rounding of the sum below 2^-29
    double sum_min = 0.0, sum_abs = 0.0;
    for (int j = 0; j < f->d; ++j) {
      const double a = (double)(j + 1) * lo[j], b = (double)(j + 1) * hi[j];
      sum_min += std::fmin(a, b);
      sum_abs += std::fmax(std::fabs(a), std::fabs(b));
    }
    return (sum_min >= -1.0 + 0x1p-20 && sum_abs <= 0x1p20) ? PCB_FAST_DOMAIN : 0;
  }
  return 0;
}

// Enqueue one V-Sample pass over logical threads [t_begin, t_end) with device-resident boundaries; nothing
// here waits for the device.  Leaves: contributions in ctx->mc_contrib (d*nb), per-group (I, Var) in
// ctx->mc_group, scalars (bad, clamps, integral, variance) in ctx->scalars[kMcSlot..]; with tail.hist_i set
// the scalars bad/clamps are re-armed by the device for the next pass.
static pcb_status enqueue_pass(pcb_ctx* ctx, const pcb_integrand* f, const pcb_mcubes_plan* plan, const double* bounds_dev,
                               unsigned long long seed, int rng_kind, const double* injected_dev, int squared_weighted,
                               long long t_begin, long long t_end, const PassTail& tail, long long* n_groups_out) {
  const int d = plan->d, nb = plan->n_bins;
  const long long n_threads = (plan->m + plan->s - 1) / plan->s;
  if (t_begin < 0 || t_end > n_threads || t_begin >= t_end)
    return fail(ctx, PCB_INVALID, "thread range [%lld, %lld) outside [0, %lld)", t_begin, t_end, n_threads);
  if (t_begin % plan->group_size != 0)
    return fail(ctx, PCB_INVALID, "thread_begin %lld must be a multiple of group_size %d", t_begin, plan->group_size);
  const long long nt = t_end - t_begin;
  SampleLaunch L;
  PCB_TRY(plan_launch(ctx, plan, nt, &L));
  const void* fn = vsample_kernel_ptr(f->family, d, rng_kind);
  PCB_TRY(grant_smem(ctx, fn, L.smem));

  const long long n_segments = nt * L.nseg, units = (n_segments + 31) / 32;
  const int vs_blocks = L.blocks;
  PCB_CUDA_TRY(ctx, ctx->mc_seg.ensure((size_t)nt * L.nseg * 2 * sizeof(double)));
  PCB_CUDA_TRY(ctx, ctx->mc_hist.ensure((size_t)vs_blocks * d * nb * sizeof(double)));
  PCB_CUDA_TRY(ctx, ctx->mc_contrib.ensure((size_t)d * nb * sizeof(double)));
  const long long n_groups = (nt + plan->group_size - 1) / plan->group_size;
  PCB_CUDA_TRY(ctx, ctx->mc_group.ensure((size_t)n_groups * 4 * sizeof(double)));
  unsigned long long* sc_u = ctx->scalars.as<unsigned long long>() + kMcSlot;
  double* sc = ctx->scalars.as<double>() + kMcSlot;

  SampleArgs a;
  a.f = *f;
  a.f.reserved = sampler_fast_domain(f, tail.grid_in_unit);
  a.g = plan->g; a.p = plan->p; a.nb = nb; a.squared_weighted = squared_weighted;
  a.m = plan->m; a.s = plan->s;
  a.n_threads = n_threads;
  a.t_begin = t_begin; a.t_end = t_end;
  a.n_segments = n_segments;
  a.seg_mul = choose_segment_multiplier(ctx, plan, t_begin, nt, L.nseg, L.seg_len);
  a.div_segments = make_fastdiv((unsigned long long)n_segments);
  a.div_nseg = make_fastdiv((unsigned long long)L.nseg);
  a.div_g = make_fastdiv((unsigned long long)plan->g);
  a.g_m32 = (plan->m < (1LL << 32) && plan->g > 1) ? (unsigned)((1ULL << 32) / (unsigned long long)plan->g) : 0u;
  a.nseg = L.nseg;
  a.rng_kind = rng_kind;
  a.seg_len = L.seg_len;
  a.seed = seed;
  a.injected = injected_dev;
  a.boundaries = bounds_dev;
  a.gd = (double)plan->g;
  a.rg = 1.0 / (double)plan->g;
  // exact integer denominators rounded once, as Python's int -> float conversion does (mcubes.py:247-248)
  a.den_est = (double)((long double)plan->p * (long double)plan->m);
  {
    unsigned __int128 den = (unsigned __int128)plan->p * (unsigned __int128)(plan->p - 1);
    den *= (unsigned __int128)plan->m;
    den *= (unsigned __int128)plan->m;
    a.den_var = (double)den;  // correctly rounded conversion of the exact product
  }
  a.seg_partials = ctx->mc_seg.as<double>();
  a.clamps = sc_u + M_CLAMPS;
  a.bad = sc_u + M_BAD;
  a.n_units = units;
  a.block_hist = ctx->mc_hist.as<double>();
  a.stop = tail.stop;
  a.iteration = tail.iteration;
  a.timeline = tail.timeline;
  {
    // units of work for the roofline: the samples actually drawn (active lanes)
    const long long c0 = t_begin * plan->s, c1 = std::min<long long>(t_end * plan->s, plan->m);
    ProfileSpan span(ctx, 1, (double)(c1 - c0) * plan->p, tail.iteration);
    void* args[] = {&a};
    PCB_CUDA_TRY(ctx, launch_pdl(fn, dim3(vs_blocks), dim3(kSampleWarps * 32), args, L.smem, ctx->stream));
    ctx->launches++;
  }

  // table merge + work-group trees in one launch
  int pow2 = 1;
  while (pow2 < plan->group_size) pow2 <<= 1;
  ReduceArgs r;
  r.stop = tail.stop;
  r.iteration = tail.iteration;
  r.block_hist = ctx->mc_hist.as<double>();
  r.nblocks = vs_blocks;
  r.nbins_total = d * nb;
  r.merge_ctas = (d * nb + 31) / 32;
  r.contrib = ctx->mc_contrib.as<double>();
  r.contrib_copy = tail.contrib_copy;
  r.seg_partials = ctx->mc_seg.as<double>();
  r.nseg = L.nseg;
  r.group_size = plan->group_size;
  r.pow2 = pow2;
  r.n_local_threads = nt;
  r.group_out = tail.row ? tail.row : ctx->mc_group.as<double>();
  r.timeline = tail.timeline;
  r.pass_scalars = sc_u;
  r.row_tail = tail.row ? reinterpret_cast<unsigned long long*>(tail.row + tail.row_doubles - 2) : nullptr;
  const size_t reduce_smem = reduce_smem_bytes(pow2);
  PCB_TRY(grant_smem(ctx, (const void*)&reduce_kernel, reduce_smem));
  {
    void* args[] = {&r};
    PCB_CUDA_TRY(ctx, launch_pdl((const void*)&reduce_kernel, dim3((unsigned)(r.merge_ctas + n_groups)), dim3(kReduceThreads), args,
                                 reduce_smem, ctx->stream));
    ctx->launches++;
  }

  if (n_groups_out) *n_groups_out = n_groups;
  if (tail.defer_finish) return PCB_OK;
  return enqueue_finish(ctx, plan, tail, n_groups);
}

static pcb_status arm_pass_scalars(pcb_ctx* ctx) {
  unsigned long long* sc_u = ctx->scalars.as<unsigned long long>() + kMcSlot;
  PCB_CUDA_TRY(ctx, cudaMemsetAsync(sc_u + M_BAD, 0xFF, sizeof(unsigned long long), ctx->stream));
  PCB_CUDA_TRY(ctx, cudaMemsetAsync(sc_u + M_CLAMPS, 0, sizeof(unsigned long long), ctx->stream));
  return PCB_OK;
}

// first non-finite sample: recompute its point on the device path is overkill; report index and value
static pcb_status report_bad_sample(pcb_ctx* ctx, const pcb_mcubes_plan* plan, unsigned long long flat, pcb_nonfinite* bad) {
  const long long cube = (long long)(flat / (unsigned long long)plan->p);
  const long long k = (long long)(flat % (unsigned long long)plan->p);
  if (bad) {
    bad->region_index = cube;
    bad->point_index = k;
    bad->value = NAN;
    std::memset(bad->point, 0, sizeof bad->point);
  }
  return fail(ctx, PCB_NONFINITE, "non-finite integrand value in sub-cube %lld (sample %lld)", cube, k);
}

static pcb_status refine_dev(pcb_ctx* ctx, int d, int nb, const double* bounds_dev, const double* contrib_dev, double alpha,
                             int smoothing, double* out_dev) {
  RefineArgs r;
  r.d = d; r.n = nb; r.alpha = alpha; r.smoothing = smoothing;
  r.boundaries = bounds_dev; r.contrib = contrib_dev; r.new_boundaries = out_dev;
  const size_t smem = refine_smem_doubles(nb) * sizeof(double);
  if (smem > ctx->smem_optin) return fail(ctx, PCB_INVALID, "n_bins %d too large for on-device refinement", nb);
  PCB_TRY(grant_smem(ctx, (const void*)&refine_grid_kernel, smem));
  refine_grid_kernel<<<d, 512, smem, ctx->stream>>>(r);
  ctx->launches++;
  PCB_CUDA_TRY(ctx, cudaGetLastError());
  return PCB_OK;
}

}  // namespace pcb

using namespace pcb;

extern "C" {

pcb_status pcb_mcubes_sample(pcb_ctx* ctx, const pcb_integrand* f, const pcb_mcubes_plan* plan, const double* boundaries,
                             uint64_t seed, int32_t rng_kind, const double* injected_uniforms, int32_t squared_weighted,
                             int64_t thread_begin, int64_t thread_end, pcb_mcubes_iteration* out, double* contributions,
                             double* group_partials, pcb_nonfinite* bad) {
  if (!ctx) return PCB_INVALID;
  PCB_TRY(validate_integrand(ctx, f));
  PCB_TRY(validate_plan(ctx, f, plan));
  if (!boundaries || !out || !contributions) return fail(ctx, PCB_INVALID, "mcubes_sample: NULL buffer");
  if (rng_kind < 0 || rng_kind > 2 || (rng_kind == PCB_RNG_INJECTED && !injected_uniforms))
    return fail(ctx, PCB_INVALID, "mcubes_sample: bad rng kind / missing injected table");
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const int d = plan->d, nb = plan->n_bins;
  const size_t bbytes = (size_t)d * (nb + 1) * sizeof(double);
  PCB_CUDA_TRY(ctx, ctx->mc_bounds[0].ensure(bbytes));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->mc_bounds[0].p, boundaries, bbytes, cudaMemcpyHostToDevice, ctx->stream));
  const double* inj = nullptr;
  if (rng_kind == PCB_RNG_INJECTED) {
    const size_t ibytes = (size_t)plan->m * plan->p * d * sizeof(double);
    PCB_CUDA_TRY(ctx, ctx->mc_inject.ensure(ibytes));
    PCB_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->mc_inject.p, injected_uniforms, ibytes, cudaMemcpyHostToDevice, ctx->stream));
    inj = ctx->mc_inject.as<double>();
  }
  long long n_groups = 0;
  PCB_TRY(arm_pass_scalars(ctx));
  PassTail plain;
  for (size_t i = 0; i < (size_t)d * (nb + 1) && plain.grid_in_unit; ++i) plain.grid_in_unit = boundaries[i] >= 0.0 && boundaries[i] <= 1.0;
  PCB_TRY(enqueue_pass(ctx, f, plan, ctx->mc_bounds[0].as<double>(), seed, rng_kind, inj, squared_weighted, thread_begin,
                       thread_end, plain, &n_groups));
  PCB_TRY(read_mc_scalars(ctx));
  const unsigned long long* hu = (const unsigned long long*)ctx->pinned + kMcSlot;
  const double* hd = (const double*)ctx->pinned + kMcSlot;
  if (hu[M_BAD] != ~0ULL) return report_bad_sample(ctx, plan, hu[M_BAD], bad);
  out->integral = hd[M_INTEGRAL];
  out->variance = std::fmax(hd[M_VARIANCE], 0.0);
  out->clamp_events = (int64_t)hu[M_CLAMPS];
  // samples drawn by this call: the cubes of the shard times p
  const long long c0 = thread_begin * plan->s, c1 = std::min<long long>(thread_end * plan->s, plan->m);
  out->n_samples = (c1 - c0) * plan->p;
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(contributions, ctx->mc_contrib.p, (size_t)d * nb * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  if (group_partials)
    PCB_CUDA_TRY(ctx, cudaMemcpyAsync(group_partials, ctx->mc_group.p, (size_t)n_groups * 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return PCB_OK;
}

pcb_status pcb_grid_refine(pcb_ctx* ctx, int32_t d, int32_t n_bins, const double* boundaries, const double* contributions,
                           double alpha, int32_t smoothing, double* new_boundaries) {
  if (!ctx) return PCB_INVALID;
  if (d < 1 || d > PCB_MAX_DIM || n_bins < 2 || !boundaries || !contributions || !new_boundaries || alpha < 0)
    return fail(ctx, PCB_INVALID, "grid_refine: bad arguments");
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const size_t bbytes = (size_t)d * (n_bins + 1) * sizeof(double), cbytes = (size_t)d * n_bins * sizeof(double);
  PCB_CUDA_TRY(ctx, ctx->mc_bounds[0].ensure(bbytes));
  PCB_CUDA_TRY(ctx, ctx->mc_bounds[1].ensure(bbytes));
  PCB_CUDA_TRY(ctx, ctx->mc_contrib.ensure(cbytes));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->mc_bounds[0].p, boundaries, bbytes, cudaMemcpyHostToDevice, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->mc_contrib.p, contributions, cbytes, cudaMemcpyHostToDevice, ctx->stream));
  PCB_TRY(refine_dev(ctx, d, n_bins, ctx->mc_bounds[0].as<double>(), ctx->mc_contrib.as<double>(), alpha, smoothing,
                     ctx->mc_bounds[1].as<double>()));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(new_boundaries, ctx->mc_bounds[1].p, bbytes, cudaMemcpyDeviceToHost, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return PCB_OK;
}

pcb_status pcb_grid_transform(pcb_ctx* ctx, int32_t d, int32_t n_bins, const double* boundaries, int64_t n, const double* y,
                              double* x, double* jac, int64_t* bins) {
  if (!ctx) return PCB_INVALID;
  if (d < 1 || d > PCB_MAX_DIM || n_bins < 2 || n < 0 || !boundaries || (n > 0 && (!y || !x || !jac || !bins)))
    return fail(ctx, PCB_INVALID, "grid_transform: bad arguments");
  if (n == 0) return PCB_OK;
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const size_t bbytes = (size_t)d * (n_bins + 1) * sizeof(double), pbytes = (size_t)n * d * sizeof(double);
  PCB_CUDA_TRY(ctx, ctx->mc_bounds[0].ensure(bbytes));
  PCB_CUDA_TRY(ctx, ctx->mc_tmp.ensure(3 * pbytes + (size_t)n * sizeof(double) + 64));
  double* y_dev = ctx->mc_tmp.as<double>();
  double* x_dev = y_dev + (size_t)n * d;
  long long* b_dev = reinterpret_cast<long long*>(x_dev + (size_t)n * d);
  double* j_dev = reinterpret_cast<double*>(b_dev + (size_t)n * d);
  int* flag_dev = reinterpret_cast<int*>(ctx->scalars.as<double>() + 60);
  PCB_CUDA_TRY(ctx, cudaMemsetAsync(flag_dev, 0, sizeof(int), ctx->stream));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->mc_bounds[0].p, boundaries, bbytes, cudaMemcpyHostToDevice, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(y_dev, y, pbytes, cudaMemcpyHostToDevice, ctx->stream));
  grid_transform_kernel<<<(unsigned)std::min<long long>((n + 255) / 256, 4096), 256, 0, ctx->stream>>>(
      d, n_bins, ctx->mc_bounds[0].as<double>(), n, y_dev, x_dev, j_dev, b_dev, flag_dev);
  ctx->launches++;
  PCB_CUDA_TRY(ctx, cudaGetLastError());
  int flag = 0;
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(&flag, flag_dev, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(x, x_dev, pbytes, cudaMemcpyDeviceToHost, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(jac, j_dev, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(bins, b_dev, (size_t)n * d * sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (flag) return fail(ctx, PCB_INVALID, "transform inputs must lie in [0, 1)");
  return PCB_OK;
}

pcb_status pcb_mcubes_sample_cube(pcb_ctx* ctx, const pcb_integrand* f, const pcb_mcubes_plan* plan, const double* boundaries,
                                  int64_t cube_index, const double* uniforms, double* s1, double* s2, int64_t* bins,
                                  double* weights, pcb_nonfinite* bad) {
  if (!ctx) return PCB_INVALID;
  PCB_TRY(validate_integrand(ctx, f));
  PCB_TRY(validate_plan(ctx, f, plan));
  if (!boundaries || !uniforms || !s1 || !s2 || !bins || !weights) return fail(ctx, PCB_INVALID, "sample_cube: NULL buffer");
  if (cube_index < 0 || cube_index >= plan->m) return fail(ctx, PCB_INVALID, "cube index %lld out of range [0, %lld)", (long long)cube_index, (long long)plan->m);
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const int d = plan->d, nb = plan->n_bins, p = plan->p;
  const size_t bbytes = (size_t)d * (nb + 1) * sizeof(double);
  PCB_CUDA_TRY(ctx, ctx->mc_bounds[0].ensure(bbytes));
  // scratch: u[p*d] x[p*d] bins[p*d] jac[p] fx[p] v[p] v2[p] sums[2] flag
  PCB_CUDA_TRY(ctx, ctx->mc_tmp.ensure(((size_t)3 * p * d + (size_t)4 * p + 4) * sizeof(double)));
  double* u_dev = ctx->mc_tmp.as<double>();
  double* x_dev = u_dev + (size_t)p * d;
  long long* b_dev = reinterpret_cast<long long*>(x_dev + (size_t)p * d);
  double* jac_dev = reinterpret_cast<double*>(b_dev + (size_t)p * d);
  double* fx_dev = jac_dev + p;
  double* v_dev = fx_dev + p;
  double* v2_dev = v_dev + p;
  double* sums_dev = v2_dev + p;
  int* flag_dev = reinterpret_cast<int*>(sums_dev + 2);
  PCB_CUDA_TRY(ctx, cudaMemsetAsync(flag_dev, 0x7F, sizeof(int), ctx->stream));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->mc_bounds[0].p, boundaries, bbytes, cudaMemcpyHostToDevice, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(u_dev, uniforms, (size_t)p * d * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  const unsigned blocks = (unsigned)((p + 127) / 128);
  cube_points_kernel<<<blocks, 128, 0, ctx->stream>>>(d, nb, p, (long long)cube_index, plan->g, ctx->mc_bounds[0].as<double>(), u_dev,
                                                      x_dev, jac_dev, b_dev);
  ctx->launches++;
  PCB_CUDA_TRY(ctx, cudaGetLastError());
  {
    long long nn = p;
    pcb_integrand fv = *f;
    const double* pts = x_dev;
    void* args[] = {&fv, &nn, &pts, &fx_dev};
    PCB_CUDA_TRY(ctx, cudaLaunchKernel(points_kernel(f->family, d), dim3(blocks), dim3(256), args, 0, ctx->stream));
    ctx->launches++;
  }
  cube_values_kernel<<<blocks, 128, 0, ctx->stream>>>(p, fx_dev, jac_dev, v_dev, v2_dev, flag_dev);
  ctx->launches++;
  PCB_CUDA_TRY(ctx, cudaGetLastError());
  PCB_TRY(tree_sum_dev(ctx, v_dev, p, sums_dev));        // S1, S2: engine.tree_sum over the p values (mcubes.py:160-161)
  PCB_TRY(tree_sum_dev(ctx, v2_dev, p, sums_dev + 1));
  double sums[2];
  int flag = 0;
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(sums, sums_dev, sizeof sums, cudaMemcpyDeviceToHost, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(&flag, flag_dev, sizeof flag, cudaMemcpyDeviceToHost, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(bins, b_dev, (size_t)p * d * sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(weights, v2_dev, (size_t)p * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (flag >= 0 && flag < p) {   // first non-finite sample: NonFiniteEvaluationError(x[i], fx[i]) (mcubes.py:156-158)
    if (bad) {
      bad->region_index = cube_index;
      bad->point_index = flag;
      std::memset(bad->point, 0, sizeof bad->point);
      PCB_CUDA_TRY(ctx, cudaMemcpy(bad->point, x_dev + (size_t)flag * d, (size_t)d * sizeof(double), cudaMemcpyDeviceToHost));
      PCB_CUDA_TRY(ctx, cudaMemcpy(&bad->value, fx_dev + flag, sizeof(double), cudaMemcpyDeviceToHost));
    }
    return fail(ctx, PCB_NONFINITE, "non-finite integrand value in sub-cube %lld (sample %d)", (long long)cube_index, flag);
  }
  *s1 = sums[0];
  *s2 = sums[1];
  return PCB_OK;
}

pcb_status pcb_debug_divide(pcb_ctx* ctx, int64_t n, const double* x, int32_t g, double* out) {
  if (!ctx || n < 0 || g < 0 || (n > 0 && (!x || !out))) return fail(ctx, PCB_INVALID, "debug_divide: bad arguments");
  if (n == 0) return PCB_OK;
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  PCB_CUDA_TRY(ctx, ctx->mc_tmp.ensure((size_t)n * 16));
  double* x_dev = ctx->mc_tmp.as<double>();
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(x_dev, x, (size_t)n * 8, cudaMemcpyHostToDevice, ctx->stream));
  debug_divide_kernel<<<(unsigned)std::min<long long>((n + 255) / 256, 4096), 256, 0, ctx->stream>>>(n, x_dev, (double)g, g ? 1.0 / (double)g : 0.0, x_dev + n);
  ctx->launches++;
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(out, x_dev + n, (size_t)n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return PCB_OK;
}

pcb_status pcb_mcubes_run(pcb_ctx* ctx, const pcb_integrand* f, const pcb_mcubes_plan* plan, int32_t iterations, uint64_t seed,
                          int32_t rng_kind, int32_t adapt, double alpha, int32_t smoothing, double rel_tol, double abs_tol,
                          pcb_mcubes_iteration* iterations_out, int32_t* n_done, pcb_mcubes_progress_fn progress, void* user,
                          double* contributions_out, double* final_boundaries, double* seconds_device, pcb_nonfinite* bad) {
  if (!ctx) return PCB_INVALID;
  PCB_TRY(validate_integrand(ctx, f));
  PCB_TRY(validate_plan(ctx, f, plan));
  if (iterations < 1) return fail(ctx, PCB_INVALID, "iterations must be >= 1");
  if (!iterations_out || !n_done) return fail(ctx, PCB_INVALID, "mcubes_run: NULL buffer");
  if (rng_kind != PCB_RNG_REFERENCE_HASH && rng_kind != PCB_RNG_PHILOX) return fail(ctx, PCB_INVALID, "mcubes_run: bad rng kind");
  if (alpha < 0) return fail(ctx, PCB_INVALID, "alpha must be >= 0");
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const int d = plan->d, nb = plan->n_bins;
  const size_t bbytes = (size_t)d * (nb + 1) * sizeof(double), tbytes = (size_t)d * nb * sizeof(double);
  PCB_CUDA_TRY(ctx, ctx->mc_bounds[0].ensure(bbytes));
  PCB_CUDA_TRY(ctx, ctx->mc_bounds[1].ensure(bbytes));
  // run state on the device: [0] stop iteration (int), then the (integral, variance) history
  PCB_CUDA_TRY(ctx, ctx->mc_state.ensure(16 + 2 * (size_t)iterations * sizeof(double)));
  int* stop_dev = ctx->mc_state.as<int>();
  double* hist_i = reinterpret_cast<double*>(ctx->mc_state.as<char>() + 16);
  double* hist_v = hist_i + iterations;
  // per-iteration tables are kept on the device (reduce_kernel writes each one) and leave, with the final boundaries,
  // through one pinned staging block when the run ends: two DMA copies and one synchronisation
  const size_t out_bytes = (contributions_out ? (size_t)iterations * tbytes : 0) + bbytes;
  if (ctx->mc_out_cap < out_bytes) {
    if (ctx->mc_out_pinned) cudaFreeHost(ctx->mc_out_pinned);
    ctx->mc_out_pinned = nullptr;
    ctx->mc_out_cap = 0;
    PCB_CUDA_TRY(ctx, cudaMallocHost(&ctx->mc_out_pinned, out_bytes + out_bytes / 4));
    ctx->mc_out_cap = out_bytes + out_bytes / 4;
  }
  double* out_bounds_host = static_cast<double*>(ctx->mc_out_pinned);
  double* out_tables_host = out_bounds_host + (size_t)d * (nb + 1);
  if (contributions_out) PCB_CUDA_TRY(ctx, ctx->mc_tables.ensure((size_t)iterations * tbytes));
  if (ctx->mc_records_cap < (size_t)iterations) {
    if (ctx->mc_records) cudaFreeHost(ctx->mc_records);
    ctx->mc_records = nullptr;
    ctx->mc_records_cap = 0;
    const size_t cap = std::max<size_t>(64, (size_t)iterations);
    PCB_CUDA_TRY(ctx, cudaMallocHost(&ctx->mc_records, cap * sizeof(McRecord)));
    std::memset(ctx->mc_records, 0, cap * sizeof(McRecord));
    ctx->mc_records_cap = cap;
  }
  McRecord* records = static_cast<McRecord*>(ctx->mc_records);
  while (ctx->mc_events.size() < (size_t)iterations + 1) {
    cudaEvent_t ev;
    PCB_CUDA_TRY(ctx, cudaEventCreate(&ev));
    ctx->mc_events.push_back(ev);
  }
  static const bool timeline_on = [] { const char* e = std::getenv("PCB_TIMELINE"); return e && std::atoi(e) != 0; }();
  unsigned long long* timeline_dev = nullptr;
  if (timeline_on) {
    PCB_CUDA_TRY(ctx, ctx->mc_timeline.ensure(256 * sizeof(unsigned long long)));
    timeline_dev = ctx->mc_timeline.as<unsigned long long>();
    PCB_CUDA_TRY(ctx, cudaMemsetAsync(timeline_dev, 0xFF, 256 * sizeof(unsigned long long), ctx->stream));
  }
  const unsigned long long token = ++ctx->mc_run_token;
  // init_grid (k / n_bins on every axis, vegas_grid.py:77-84), stop iteration = "never", pass scalars armed: one launch
  PCB_TRY(grant_smem(ctx, (const void*)&run_init_kernel, 0));
  run_init_kernel<<<d, 256, 0, ctx->stream>>>(nb, ctx->mc_bounds[0].as<double>(), stop_dev,
                                               ctx->scalars.as<unsigned long long>() + kMcSlot);
  ctx->launches++;
  PCB_CUDA_TRY(ctx, cudaGetLastError());
  const size_t span_mark[3] = {ctx->spans[0].size(), ctx->spans[1].size(), ctx->spans[2].size()};
  PCB_CUDA_TRY(ctx, cudaEventRecord(ctx->mc_events[0], ctx->stream));

  // Device time of the run: one event before the first pass and one after the last enqueued kernel.  No event sits
  // between the kernels of the chain (an event record between two kernels ends their programmatic overlap and is a
  // stream operation of its own), so the reported time includes the at most one speculative no-op pass behind the
  // stopping iteration.  PCB_MC_ITER_EVENTS=1 records one event per iteration instead and reports the time up to the
  // end of the stopping iteration (A/B measurements).
  static const bool iteration_events = [] { const char* e = std::getenv("PCB_MC_ITER_EVENTS"); return e && std::atoi(e) != 0; }();
  // The loop is device-resident: every kernel of iteration `it` is a no-op once the device has decided to
  // stop at an earlier iteration, so the host enqueues iteration it+1 BEFORE it waits for the record of
  // iteration it -- the device never idles on the host round trip.
  const long long n_threads = (plan->m + plan->s - 1) / plan->s;
  auto enqueue = [&](int it) -> pcb_status {
    PassTail tail;
    tail.iteration = it;
    tail.stop = stop_dev;
    tail.refine = adapt != 0;
    tail.alpha = alpha;
    tail.smoothing = smoothing;
    const int cur = adapt ? (it & 1) : 0;
    tail.bounds_in = ctx->mc_bounds[cur].as<double>();
    tail.bounds_out = ctx->mc_bounds[cur ^ 1].as<double>();
    tail.contrib_copy = contributions_out ? ctx->mc_tables.as<double>() + (size_t)it * d * nb : nullptr;
    tail.hist_i = hist_i;
    tail.hist_v = hist_v;
    tail.rel_tol = rel_tol;
    tail.abs_tol = abs_tol > 0 ? abs_tol : 0.0;
    tail.record = records + it;
    tail.seq = (token << 20) | (unsigned long long)(it + 1);
    tail.timeline = timeline_dev;
    const unsigned long long it_seed = derive_seed(seed, (unsigned long long)it);  // mcubes.py:58-60, 359
    PCB_TRY(enqueue_pass(ctx, f, plan, tail.bounds_in, it_seed, rng_kind, nullptr, 1, 0, n_threads, tail, nullptr));
    if (iteration_events) PCB_CUDA_TRY(ctx, cudaEventRecord(ctx->mc_events[it + 1], ctx->stream));
    return PCB_OK;
  };
  auto wait_record = [&](int it) -> pcb_status {
    const unsigned long long want = (token << 20) | (unsigned long long)(it + 1);
    const McRecord* r = records + it;
    for (unsigned spin = 0; r->seq != want; ++spin) {
      if ((spin & 0xfff) == 0xfff) {  // the record never arrives if a kernel faulted: look at the stream now and then
        cudaError_t e = cudaStreamQuery(ctx->stream);
        if (e != cudaErrorNotReady && r->seq != want) {
          if (e == cudaSuccess) return fail(ctx, PCB_CUDA, "mcubes_run: iteration %d finished without publishing its record", it);
          (void)cudaGetLastError();
          return fail(ctx, PCB_CUDA, "mcubes_run: %s", cudaGetErrorString(e));
        }
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);   // the record's fields are read after its sequence word
    return PCB_OK;
  };

  int done = 0, enqueued = 0;
  std::vector<double> ivals, ivars;
  // Speculation is withheld when the run is about to stop: the cumulative error of the next iteration is
  // extrapolated geometrically from the last two (it falls several-fold per iteration while the grid adapts and by
  // ~sqrt(k/(k+1)) afterwards); if that meets the target, the pass behind it would only be three no-op launches
  // inside the timed run.  A wrong guess costs one host round trip, never a result: the decision is the device's.
  const bool tol_mode = rel_tol > 0.0 || abs_tol > 0.0;
  bool near_target = false;
  double prev_err = 0.0;
  pcb_status st = enqueue(enqueued++);
  for (int it = 0; st == PCB_OK && it < iterations; ++it) {
    if (enqueued < iterations && enqueued <= it + 1 && !near_target) {
      st = enqueue(enqueued++);
      if (st != PCB_OK) break;
    }
    st = wait_record(it);
    if (st != PCB_OK) break;
    const McRecord rec = {records[it].integral, records[it].variance, records[it].clamps, records[it].bad, records[it].stop, 0, 0};
    if (rec.bad != ~0ULL) {
      cudaStreamSynchronize(ctx->stream);
      return report_bad_sample(ctx, plan, rec.bad, bad);
    }
    pcb_mcubes_iteration& o = iterations_out[it];
    o.integral = rec.integral;
    o.variance = std::fmax(rec.variance, 0.0);
    o.n_samples = plan->m * plan->p;
    o.clamp_events = (int64_t)rec.clamps;
    done = it + 1;
    ivals.push_back(o.integral);
    ivars.push_back(o.variance);
    if (tol_mode && !rec.stop) {
      double wsum = 0.0, dot = 0.0;
      for (int i = 0; i < done; ++i) {
        const double w = 1.0 / std::fmax(ivars[i], 1e-30);
        wsum += w;
        dot += w * ivals[i];
      }
      const double target = std::fmax(abs_tol > 0 ? abs_tol : 0.0, rel_tol * std::fabs(dot / wsum));
      const double err = std::pow(wsum, -0.5);
      near_target = done >= 2 && prev_err > 0.0 && err * std::fmin(1.0, err / prev_err) <= target;
      prev_err = err;
    }
    if (progress) {
      // combine_iterations (mcubes.py:311-329): inverse-variance weights, variances floored at 1e-30
      double wsum = 0.0, dot = 0.0;
      for (int i = 0; i < done; ++i) {
        const double w = 1.0 / std::fmax(ivars[i], 1e-30);
        wsum += w;
        dot += w * ivals[i];
      }
      const double est = dot / wsum, err = std::pow(wsum, -0.5);
      double chi2 = 0.0;
      if (done > 1) {
        for (int i = 0; i < done; ++i) {
          const double w = 1.0 / std::fmax(ivars[i], 1e-30), dv = ivals[i] - est;
          chi2 += w * (dv * dv);
        }
        chi2 /= (double)(done - 1);
      }
      pcb_mcubes_progress rec_out;
      rec_out.iteration = it;
      rec_out.reserved = 0;
      rec_out.estimate = est;
      rec_out.errorest = err;
      rec_out.chi2_per_dof = chi2;
      rec_out.iter_integral = o.integral;
      rec_out.iter_variance = o.variance;
      ctx->abort_requested = 0;
      progress(user, &rec_out);
      if (ctx->abort_requested) {   // the callback asked to stop: make the device stop too, drain, report
        ctx->abort_requested = 0;
        const int now = it;
        cudaMemcpyAsync(stop_dev, &now, sizeof(int), cudaMemcpyHostToDevice, ctx->stream);
        cudaStreamSynchronize(ctx->stream);
        return fail(ctx, PCB_ABORTED, "mcubes_run stopped by its progress callback at iteration %d", it);
      }
    }
    if (rec.stop) break;
    if (enqueued <= it + 1 && enqueued < iterations) {   // speculation was withheld and the run goes on
      st = enqueue(enqueued++);
      if (st != PCB_OK) break;
    }
  }
  // End of the run: the closing event and the two result copies (final boundaries, the tables of the iterations that
  // ran) are enqueued behind the last kernel in one go and awaited once -- this also drains the at most one
  // speculative no-op pass before anything is reused.
  if (!iteration_events && st == PCB_OK) st = cudaEventRecord(ctx->mc_events[1], ctx->stream) == cudaSuccess ? PCB_OK : fail(ctx, PCB_CUDA, "mcubes_run: event record failed");
  if (st == PCB_OK && final_boundaries) {
    const int cur = adapt ? (done & 1) : 0;
    if (cudaMemcpyAsync(out_bounds_host, ctx->mc_bounds[cur].p, bbytes, cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess)
      st = fail(ctx, PCB_CUDA, "mcubes_run: copy of the final boundaries failed");
  }
  if (st == PCB_OK && contributions_out && done > 0) {
    if (cudaMemcpyAsync(out_tables_host, ctx->mc_tables.p, (size_t)done * tbytes, cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess)
      st = fail(ctx, PCB_CUDA, "mcubes_run: copy of the contribution tables failed");
  }
  cudaError_t drain = cudaStreamSynchronize(ctx->stream);
  if (st != PCB_OK) return st;
  PCB_CUDA_TRY(ctx, drain);
  // profiling spans of passes that never ran are not launches of the hot kernel
  for (int k = 0; k < 3; ++k) {
    auto& v = ctx->spans[k];
    size_t keep = span_mark[k];
    for (size_t i = span_mark[k]; i < v.size(); ++i) {
      if (v[i].tag < done) v[keep++] = v[i];
      else ctx->span_pool.push_back(v[i]);
    }
    v.resize(keep);
  }
  if (timeline_dev) {  // debug: where the time of the run went, microseconds from the first stamp
    unsigned long long tl[256];
    PCB_CUDA_TRY(ctx, cudaMemcpy(tl, timeline_dev, sizeof tl, cudaMemcpyDeviceToHost));
    const char* names[3] = {"vsample", "reduce", "finish"};
    unsigned long long t0 = ~0ULL;   // earliest kernel entry (the pass kernel's own stamps exist in experiment builds only)
    for (int k = 0; k < 16 * 3; ++k) t0 = std::min(t0, tl[k * 4]);
    auto us = [&](unsigned long long t) { return t == ~0ULL ? -1.0 : (double)(long long)(t - t0) * 1e-3; };
    for (int it = 0; it < 16 && it <= done; ++it)
      for (int k = 0; k < 3; ++k) {
        const unsigned long long* e = tl + (it * 3 + k) * 4;
        if (e[0] == ~0ULL) continue;
        std::fprintf(stderr, "timeline it %d %-8s enter %9.3f go %9.3f end %9.3f end2 %9.3f\n", it, names[k], us(e[0]), us(e[1]),
                     e[2] == ~0ULL ? -1.0 : us(~e[2]), us(e[3]));
      }
    for (int k = 0; k < 8; ++k) std::fprintf(stderr, "timeline it 1 refine axis 0 phase %d at %9.3f\n", k, us(tl[200 + k]));
    for (int k = 0; k < 4; ++k)
      std::fprintf(stderr, "timeline it 1 vsample %s: earliest CTA %9.3f latest CTA %9.3f\n",
                   k == 0 ? "tables ready   " : k == 1 ? "units done     " : k == 2 ? "last round added" : "table flushed  ", us(tl[230 + 2 * k]), us(~tl[231 + 2 * k]));
    for (int k = 240; k < 256; ++k)
      if (tl[k] != ~0ULL) std::fprintf(stderr, "timeline it 1 vsample CTA 0 batch %d %s %9.3f\n", (k - 240) / 4, (k & 3) == 0 ? "start      " : (k & 3) == 1 ? "round 1 end" : (k & 3) == 2 ? "round 2 end" : "round 3 end", us(tl[k]));
    std::fprintf(stderr, "timeline it 1 reduce latest CTA entry %9.3f latest return from wait %9.3f\n", us(~tl[220]), us(~tl[221]));
    for (int k = 0; k < 8; ++k) std::fprintf(stderr, "timeline it 1 reduce %s CTA %s %9.3f\n", k < 2 ? "first merge" : k < 4 ? "last merge" : k < 6 ? "first group" : "last group", k & 1 ? "end  " : "start", us(tl[210 + k]));
  }
  float ms = 0;
  PCB_CUDA_TRY(ctx, cudaEventElapsedTime(&ms, ctx->mc_events[0], ctx->mc_events[iteration_events ? done : 1]));
  if (seconds_device) *seconds_device = ms * 1e-3;
  *n_done = done;
  if (final_boundaries) std::memcpy(final_boundaries, out_bounds_host, bbytes);
  if (contributions_out) std::memcpy(contributions_out, out_tables_host, (size_t)done * tbytes);
  return PCB_OK;
}

// ------------------------------------------------------------------------------------------------
// m-Cubes run on a shard of the logical threads (multi-GPU, one context per rank).  The loop stays device-resident
// exactly like pcb_mcubes_run; the two collectives of an iteration run on the context's stream, between
//   pass(it)    V-Sample over this rank's work-groups + table merge + the rank's packed row, and
//   finish(it)  group-order tree over ALL groups from the gathered rows, grid refinement from the all-reduced
//               table (identical on every rank), iteration record, stop decision.
// ------------------------------------------------------------------------------------------------
static __global__ void shard_init_row_kernel(double* row, long long row_doubles) {
  for (long long i = threadIdx.x; i < row_doubles - 2; i += blockDim.x) row[i] = 0.0;
  if (threadIdx.x == 0) {
    unsigned long long* tail = reinterpret_cast<unsigned long long*>(row + row_doubles - 2);
    tail[0] = ~0ULL;   // no non-finite sample
    tail[1] = 0ULL;    // no clamp events
  }
}

pcb_status pcb_mcubes_shard_begin(pcb_ctx* ctx, const pcb_integrand* f, const pcb_mcubes_plan* plan, int32_t iterations,
                                  uint64_t seed, int32_t rng_kind, int32_t adapt, double alpha, int32_t smoothing, double rel_tol,
                                  double abs_tol, int32_t keep_tables, int32_t rank, int32_t world, pcb_mcubes_shard_buffers* out) {
  if (!ctx) return PCB_INVALID;
  PCB_TRY(validate_integrand(ctx, f));
  PCB_TRY(validate_plan(ctx, f, plan));
  if (iterations < 1) return fail(ctx, PCB_INVALID, "iterations must be >= 1");
  if (!out || world < 1 || rank < 0 || rank >= world) return fail(ctx, PCB_INVALID, "mcubes_shard_begin: bad rank/world or NULL buffers");
  if (rng_kind != PCB_RNG_REFERENCE_HASH && rng_kind != PCB_RNG_PHILOX) return fail(ctx, PCB_INVALID, "mcubes_run: bad rng kind");
  if (alpha < 0) return fail(ctx, PCB_INVALID, "alpha must be >= 0");
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  auto& S = ctx->mc_shard;
  S = pcb_ctx::McShard();
  const int d = plan->d, nb = plan->n_bins;
  const long long n_threads = (plan->m + plan->s - 1) / plan->s;
  S.f = *f; S.plan = *plan;
  S.iterations = iterations; S.rng_kind = rng_kind; S.adapt = adapt; S.smoothing = smoothing;
  S.alpha = alpha; S.rel_tol = rel_tol; S.abs_tol = abs_tol > 0 ? abs_tol : 0.0;
  S.seed = seed; S.rank = rank; S.world = world; S.keep_tables = keep_tables;
  S.n_groups = (n_threads + plan->group_size - 1) / plan->group_size;
  if (S.n_groups > 1024) return fail(ctx, PCB_INVALID, "sharded mcubes_run supports at most 1024 work-groups (%lld requested)", S.n_groups);
  // contiguous, near-equal ranges of work-groups per rank (sharded.group_shards)
  const long long g0 = S.n_groups * rank / world, g1 = S.n_groups * (rank + 1) / world;
  S.g_count = g1 - g0;
  S.t_begin = g0 * plan->group_size;
  S.t_end = std::min<long long>(g1 * plan->group_size, n_threads);
  S.width = (S.n_groups + world - 1) / world;
  S.row_doubles = 2 * S.width + 2;
  const size_t bbytes = (size_t)d * (nb + 1) * sizeof(double), tbytes = (size_t)d * nb * sizeof(double);
  PCB_CUDA_TRY(ctx, ctx->mc_bounds[0].ensure(bbytes));
  PCB_CUDA_TRY(ctx, ctx->mc_bounds[1].ensure(bbytes));
  PCB_CUDA_TRY(ctx, ctx->mc_contrib.ensure(tbytes));
  PCB_CUDA_TRY(ctx, ctx->mc_state.ensure(16 + 2 * (size_t)iterations * sizeof(double)));
  PCB_CUDA_TRY(ctx, ctx->mc_row.ensure((size_t)S.row_doubles * sizeof(double)));
  if (world > 1) PCB_CUDA_TRY(ctx, ctx->mc_gathered.ensure((size_t)world * S.row_doubles * sizeof(double)));
  if (keep_tables) PCB_CUDA_TRY(ctx, ctx->mc_tables.ensure((size_t)iterations * tbytes));
  const size_t out_bytes = (keep_tables ? (size_t)iterations * tbytes : 0) + bbytes;
  if (ctx->mc_out_cap < out_bytes) {
    if (ctx->mc_out_pinned) cudaFreeHost(ctx->mc_out_pinned);
    ctx->mc_out_pinned = nullptr;
    ctx->mc_out_cap = 0;
    PCB_CUDA_TRY(ctx, cudaMallocHost(&ctx->mc_out_pinned, out_bytes + out_bytes / 4));
    ctx->mc_out_cap = out_bytes + out_bytes / 4;
  }
  if (ctx->mc_records_cap < (size_t)iterations) {
    if (ctx->mc_records) cudaFreeHost(ctx->mc_records);
    ctx->mc_records = nullptr;
    ctx->mc_records_cap = 0;
    const size_t cap = std::max<size_t>(64, (size_t)iterations);
    PCB_CUDA_TRY(ctx, cudaMallocHost(&ctx->mc_records, cap * sizeof(McRecord)));
    std::memset(ctx->mc_records, 0, cap * sizeof(McRecord));
    ctx->mc_records_cap = cap;
  }
  while (ctx->mc_events.size() < 2) {
    cudaEvent_t ev;
    PCB_CUDA_TRY(ctx, cudaEventCreate(&ev));
    ctx->mc_events.push_back(ev);
  }
  S.token = ++ctx->mc_run_token;
  PCB_TRY(grant_smem(ctx, (const void*)&run_init_kernel, 0));
  run_init_kernel<<<d, 256, 0, ctx->stream>>>(nb, ctx->mc_bounds[0].as<double>(), ctx->mc_state.as<int>(),
                                               ctx->scalars.as<unsigned long long>() + kMcSlot);
  shard_init_row_kernel<<<1, 256, 0, ctx->stream>>>(ctx->mc_row.as<double>(), S.row_doubles);
  ctx->launches += 2;
  PCB_CUDA_TRY(ctx, cudaGetLastError());
  for (int k = 0; k < 3; ++k) S.span_mark[k] = ctx->spans[k].size();
  PCB_CUDA_TRY(ctx, cudaEventRecord(ctx->mc_events[0], ctx->stream));
  S.live = true;
  out->stream = (void*)ctx->stream;
  out->row = ctx->mc_row.as<double>();
  out->gathered = world > 1 ? ctx->mc_gathered.as<double>() : ctx->mc_row.as<double>();
  out->table = ctx->mc_contrib.as<double>();
  out->row_doubles = S.row_doubles;
  out->table_doubles = (int64_t)d * nb;
  out->thread_begin = S.t_begin;
  out->thread_end = S.t_end;
  return PCB_OK;
}

static PassTail shard_tail(pcb_ctx* ctx, int it) {
  auto& S = ctx->mc_shard;
  const int d = S.plan.d, nb = S.plan.n_bins;
  PassTail tail;
  tail.iteration = it;
  tail.stop = ctx->mc_state.as<int>();
  tail.refine = S.adapt != 0;
  tail.alpha = S.alpha;
  tail.smoothing = S.smoothing;
  const int cur = S.adapt ? (it & 1) : 0;
  tail.bounds_in = ctx->mc_bounds[cur].as<double>();
  tail.bounds_out = ctx->mc_bounds[cur ^ 1].as<double>();
  tail.contrib_copy = nullptr;   // the per-iteration table is the all-reduced one: copied by finish()
  tail.hist_i = reinterpret_cast<double*>(ctx->mc_state.as<char>() + 16);
  tail.hist_v = tail.hist_i + S.iterations;
  tail.rel_tol = S.rel_tol;
  tail.abs_tol = S.abs_tol;
  tail.record = static_cast<McRecord*>(ctx->mc_records) + it;
  tail.seq = (S.token << 20) | (unsigned long long)(it + 1);
  tail.row = ctx->mc_row.as<double>();
  tail.row_doubles = S.row_doubles;
  tail.defer_finish = true;
  tail.gathered = S.world > 1 ? ctx->mc_gathered.as<double>() : ctx->mc_row.as<double>();
  tail.world = S.world;
  tail.total_groups = S.n_groups;
  (void)d; (void)nb;
  return tail;
}

pcb_status pcb_mcubes_shard_pass(pcb_ctx* ctx, int32_t iteration) {
  if (!ctx || !ctx->mc_shard.live) return fail(ctx, PCB_INVALID, "no live m-Cubes shard run");
  auto& S = ctx->mc_shard;
  if (iteration < 0 || iteration >= S.iterations) return fail(ctx, PCB_INVALID, "iteration %d outside [0, %d)", iteration, S.iterations);
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  if (S.g_count == 0) {   // nothing to sample here: the row keeps (no groups, bad = none, clamps = 0) and the table this rank
                          // adds to the all-reduce is empty (the buffer holds the previous iteration's global sum)
    PCB_CUDA_TRY(ctx, cudaMemsetAsync(ctx->mc_contrib.p, 0, (size_t)S.plan.d * S.plan.n_bins * sizeof(double), ctx->stream));
    return PCB_OK;
  }
  const PassTail tail = shard_tail(ctx, iteration);
  const unsigned long long it_seed = derive_seed(S.seed, (unsigned long long)iteration);   // mcubes.py:58-60, 359
  return enqueue_pass(ctx, &S.f, &S.plan, tail.bounds_in, it_seed, S.rng_kind, nullptr, 1, S.t_begin, S.t_end, tail, nullptr);
}

pcb_status pcb_mcubes_shard_finish(pcb_ctx* ctx, int32_t iteration) {
  if (!ctx || !ctx->mc_shard.live) return fail(ctx, PCB_INVALID, "no live m-Cubes shard run");
  auto& S = ctx->mc_shard;
  if (iteration < 0 || iteration >= S.iterations) return fail(ctx, PCB_INVALID, "iteration %d outside [0, %d)", iteration, S.iterations);
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const PassTail tail = shard_tail(ctx, iteration);
  if (S.keep_tables) {
    const size_t tbytes = (size_t)S.plan.d * S.plan.n_bins * sizeof(double);
    PCB_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->mc_tables.as<char>() + (size_t)iteration * tbytes, ctx->mc_contrib.p, tbytes,
                                      cudaMemcpyDeviceToDevice, ctx->stream));
  }
  return enqueue_finish(ctx, &S.plan, tail, S.n_groups);
}

pcb_status pcb_mcubes_shard_wait(pcb_ctx* ctx, int32_t iteration, pcb_mcubes_iteration* out, int32_t* stop, pcb_nonfinite* bad) {
  if (!ctx || !ctx->mc_shard.live) return fail(ctx, PCB_INVALID, "no live m-Cubes shard run");
  auto& S = ctx->mc_shard;
  if (iteration < 0 || iteration >= S.iterations || !out || !stop) return fail(ctx, PCB_INVALID, "mcubes_shard_wait: bad arguments");
  const unsigned long long want = (S.token << 20) | (unsigned long long)(iteration + 1);
  const McRecord* r = static_cast<McRecord*>(ctx->mc_records) + iteration;
  for (unsigned spin = 0; *(volatile unsigned long long*)&r->seq != want; ++spin) {
    if ((spin & 0xfff) == 0xfff) {
      cudaError_t e = cudaStreamQuery(ctx->stream);
      if (e != cudaErrorNotReady && *(volatile unsigned long long*)&r->seq != want) {
        if (e == cudaSuccess) return fail(ctx, PCB_CUDA, "mcubes shard run: iteration %d finished without publishing its record", iteration);
        (void)cudaGetLastError();
        return fail(ctx, PCB_CUDA, "mcubes shard run: %s", cudaGetErrorString(e));
      }
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  const McRecord rec = {r->integral, r->variance, r->clamps, r->bad, r->stop, 0, 0};
  if (rec.bad != ~0ULL) {
    cudaStreamSynchronize(ctx->stream);
    S.live = false;
    return report_bad_sample(ctx, &S.plan, rec.bad, bad);
  }
  out->integral = rec.integral;
  out->variance = std::fmax(rec.variance, 0.0);
  out->n_samples = S.plan.m * S.plan.p;
  out->clamp_events = (int64_t)rec.clamps;
  *stop = rec.stop;
  return PCB_OK;
}

pcb_status pcb_mcubes_shard_end(pcb_ctx* ctx, int32_t n_done, double* contributions_out, double* final_boundaries,
                                double* seconds_device) {
  if (!ctx || !ctx->mc_shard.live) return fail(ctx, PCB_INVALID, "no live m-Cubes shard run");
  auto& S = ctx->mc_shard;
  S.live = false;
  if (n_done < 0 || n_done > S.iterations) return fail(ctx, PCB_INVALID, "mcubes_shard_end: n_done outside the run");
  if (contributions_out && !S.keep_tables) return fail(ctx, PCB_INVALID, "mcubes_shard_end: the run was started without keep_tables");
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  PCB_CUDA_TRY(ctx, cudaEventRecord(ctx->mc_events[1], ctx->stream));
  PCB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));   // drains the at most one speculative no-op iteration
  for (int k = 0; k < 3; ++k) {   // profiling spans of passes that never ran are not launches of the hot kernel
    auto& v = ctx->spans[k];
    size_t keep = S.span_mark[k];
    for (size_t i = S.span_mark[k]; i < v.size(); ++i) {
      if (v[i].tag < n_done) v[keep++] = v[i];
      else ctx->span_pool.push_back(v[i]);
    }
    v.resize(keep);
  }
  float ms = 0;
  PCB_CUDA_TRY(ctx, cudaEventElapsedTime(&ms, ctx->mc_events[0], ctx->mc_events[1]));
  if (seconds_device) *seconds_device = ms * 1e-3;
  const int d = S.plan.d, nb = S.plan.n_bins;
  const size_t bbytes = (size_t)d * (nb + 1) * sizeof(double), tbytes = (size_t)d * nb * sizeof(double);
  double* out_bounds_host = static_cast<double*>(ctx->mc_out_pinned);
  double* out_tables_host = out_bounds_host + (size_t)d * (nb + 1);
  if (final_boundaries) {
    const int cur = S.adapt ? (n_done & 1) : 0;
    PCB_CUDA_TRY(ctx, cudaMemcpyAsync(out_bounds_host, ctx->mc_bounds[cur].p, bbytes, cudaMemcpyDeviceToHost, ctx->stream));
  }
  if (contributions_out && n_done > 0)
    PCB_CUDA_TRY(ctx, cudaMemcpyAsync(out_tables_host, ctx->mc_tables.p, (size_t)n_done * tbytes, cudaMemcpyDeviceToHost, ctx->stream));
  if (final_boundaries || contributions_out) PCB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (final_boundaries) std::memcpy(final_boundaries, out_bounds_host, bbytes);
  if (contributions_out && n_done > 0) std::memcpy(contributions_out, out_tables_host, (size_t)n_done * tbytes);
  return PCB_OK;
}

}  // extern "C"
