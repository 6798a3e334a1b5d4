/*
 * parcube_b200.h -- C-ABI of the B200-native PAGANI / m-Cubes hot path.
 *
 * The reference package (`parcube`, /root/reference/pkg/src/parcube) is pure Python and has
 * no FFI of its own; its boundary is the Python function surface re-exported in
 * __init__.py:11-83.  Each entry point below is what a ctypes binding placed behind one of
 * those functions calls (INTEGRATION.md shows the stub).  Plain pointers and sizes only;
 * all buffers are caller-owned HOST memory unless the name ends in `_dev`; one in-flight
 * call per context.  Every function returns a pcb_status; pcb_last_error() gives the text.
 *
 * There is no CPU fallback: every entry point needs a CUDA device (sm_100a build).
 */
#ifndef PARCUBE_B200_H
#define PARCUBE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PCB_MAX_DIM 12 /* reference: core.py:14 */

typedef enum {
  PCB_OK = 0,
  PCB_NONFINITE = 1, /* integrand returned NaN/inf: see pcb_nonfinite (core.py:26-37)   */
  PCB_BUDGET = 2,    /* workload exceeds a cap (core.py:22-23, 262-263)                 */
  PCB_INVALID = 3,   /* bad argument (the reference's ValueError paths)                 */
  PCB_CUDA = 4,      /* CUDA runtime failure                                            */
  PCB_ABORTED = 5    /* pcb_ctx_abort() was called from a progress callback             */
} pcb_status;

/* Integrand families = the reference registry BENCHMARKS (integrands.py:131-139). */
typedef enum {
  PCB_F1_OSCILLATORY = 0,   /* cos(sum i*x_i)                      integrands.py:28-39   */
  PCB_F2_PRODUCT_PEAK = 1,  /* prod 1/(a^2+(x_i-1/2)^2)            integrands.py:42-53   */
  PCB_F3_CORNER_PEAK = 2,   /* (1+sum i*x_i)^(-d-1)                integrands.py:56-67   */
  PCB_F4_GAUSSIAN = 3,      /* exp(-rate*sum (x_i-1/2)^2)          integrands.py:70-81   */
  PCB_F5_KINKED = 4,        /* exp(-10*sum |x_i-1/2|)              integrands.py:84-92   */
  PCB_F6_DISCONTINUOUS = 5, /* exp(sum (i+4)x_i) below thresholds  integrands.py:95-118  */
  PCB_SUM = 6,              /* sum x_i                             integrands.py:121-128 */
  PCB_ONE = 7,              /* constant 1 (SPEC.md known answers)                        */
  PCB_N_FAMILIES = 8         /* built-in families; ids PCB_USER_FAMILY_BASE .. +PCB_MAX_USER_FAMILIES-1 are run-time families */
} pcb_family;

/* Run-time families: a device functor compiled from user source against this library's own kernel templates
 * (paper_2302_05730_b200/userfn.py writes the translation unit and runs nvcc), loaded as a cubin and bound to one
 * dimension.  The reference integrates any Python callable (core.py:72-93); a callable cannot run on the device, its
 * CUDA source can.  The kernels, launch paths and results contracts are the built-in families' own. */
#define PCB_USER_FAMILY_BASE 8
#define PCB_MAX_USER_FAMILIES 8
typedef struct {
  const char* eval;           /* pagani_eval_kernel<family, d>                 */
  const char* eval_wide;      /* pagani_eval_kernel<family, d, true>           */
  const char* lanes;          /* pagani_eval_lanes_generic_kernel<family, d>   */
  const char* points;         /* eval_points_kernel<family, d>                 */
  const char* invoke;         /* invoke_kernel<family, d>                      */
  const char* qmc;            /* qmc_shift_kernel<family, d>                   */
  const char* sample_hash;    /* vsample_kernel<family, d, PCB_RNG_REFERENCE_HASH> */
  const char* sample_generic; /* vsample_kernel<family, d, PCB_RNG_PHILOX>     */
} pcb_user_kernel_names;

/* A compiled device functor is selected by (family, d); `param` carries the family's
 * constants as computed by the host in the reference's own expressions:
 *   f2: param[0] = a^2 (1/2500)   f4: param[0] = rate (625)   f5: param[0] = 10
 *   f6: param[j] = threshold_j = (3 + (j+1)) / 10
 * `bounded` applies scale_to_bounds (core.py:134-148): f(low + width*y) * jac.            */
typedef struct {
  int32_t family;
  int32_t d;
  int32_t bounded;
  int32_t reserved;
  double param[PCB_MAX_DIM];
  double low[PCB_MAX_DIM];
  double width[PCB_MAX_DIM];
  double jac;
} pcb_integrand;

/* Orbit form of a RuleTable (quadrature.py:43-70): the table is input data, compressed by the
 * host after verifying its fully symmetric structure (rules.py:orbit_form).
 * offsets: 1/2, (1+l2)/2, (1-l2)/2, (1+l3)/2, (1-l3)/2, (1+l5)/2, (1-l5)/2 -- the values of
 * (generators + 1.0) / 2.0 (quadrature.py:301).  weights[k][o]: rule k on orbit o
 * (centre, l2-axial, l3-axial, l4-pairs, l5-corners); corner_parity[k] != 0 means the corner
 * weight alternates in sign with the parity of the corner's bit count (quadrature.py:199-203). */
typedef struct {
  int32_t d;
  int32_t f_eval;
  double offsets[7];
  double weights[5][5];
  int32_t corner_parity[5];
  int32_t reserved;
  double split_weights[2]; /* quadrature.py:279 */
  int32_t null_high[4];    /* null_degrees[k] >= 5 (pagani.py:123-124) */
  double null_scale[4];    /* null_scales (pagani.py:126) */
} pcb_rule;

typedef enum { PCB_ERR_TWO_LEVEL = 0, PCB_ERR_MAX_NULL = 1, PCB_ERR_MAX_PAIRWISE = 2 } pcb_err_mode;

/* The numerically relevant part of PaganiConfig (pagani.py:44-69). */
typedef struct {
  double rel_tol;
  int32_t max_iterations;
  int32_t group_size;      /* strided schedule width G >= 1 (pagani.py:175-192); G <= 64 runs one warp per
                              region, wider schedules a generic kernel (one CTA per region) */
  int64_t region_cap;
  int32_t initial_regions;
  int32_t err_mode;        /* pcb_err_mode */
  double rel_floor;
  double abs_tol;          /* extension (epsabs, default 0 = the reference): converged when
                              errorest <= max(abs_tol, rel_tol*|estimate|)                  */
} pcb_pagani_config;

/* First non-finite evaluation in row-major (region, point) order (pagani.py:206-209,
 * mcubes.py:238-241). */
typedef struct {
  int64_t region_index; /* region (PAGANI) or sub-cube (m-Cubes) index */
  int64_t point_index;  /* rule point or sample index inside it */
  double value;
  double point[PCB_MAX_DIM];
} pcb_nonfinite;

/* One record per refinement iteration == the reference's progress dict + history tuple
 * (pagani.py:339-349). */
typedef struct {
  int32_t iteration;
  int32_t reserved;
  int64_t n_regions; /* leaves: finished + active */
  int64_t active;
  double estimate;
  double errorest;
} pcb_pagani_progress;

typedef enum {
  PCB_STOP_TOLERANCE = 0,  /* "tolerance met"            pagani.py:350-353 */
  PCB_STOP_MAX_ITER = 1,   /* "max iterations reached"   pagani.py:354-356 */
  PCB_STOP_NO_ACTIVE = 2,  /* "no active regions left"   pagani.py:357-359 */
  PCB_STOP_REGION_CAP = 3  /* "region cap reached"       pagani.py:367-369 */
} pcb_stop_reason;

/* IntegralResult (pagani.py:89-101); history is returned through the progress records. */
typedef struct {
  double estimate;
  double errorest;
  int32_t iterations;
  int32_t converged;
  int64_t regions_processed;
  int32_t reason; /* pcb_stop_reason */
  int32_t n_records;
  double seconds_device; /* CUDA-event time of the whole refinement, for reporting only */
  int64_t kernel_launches;
} pcb_pagani_result;

typedef void (*pcb_pagani_progress_fn)(void* user, const pcb_pagani_progress* rec);

/* McubesPlan (mcubes.py:77-107). */
typedef struct {
  int32_t d;
  int32_t g;
  int32_t p;
  int32_t group_size;
  int64_t m;
  int64_t s;
  int32_t n_bins;          /* 2..65535 (the pass stages bin ids as 16-bit values); the reference default is 500 */
  int32_t reserved;
} pcb_mcubes_plan;

typedef enum {
  PCB_RNG_REFERENCE_HASH = 0, /* the reference's SplitMix64-style hash (mcubes.py:31-55): bit-exact */
  PCB_RNG_PHILOX = 1,         /* Philox4x32-10 keyed by (seed, stream), counter-indexed             */
  PCB_RNG_INJECTED = 2        /* uniforms read from a caller table, index (cube*p + k)*d + j          */
} pcb_rng_kind;

/* McubesIterationResult (mcubes.py:182-192) minus the table, which is an output array. */
typedef struct {
  double integral;
  double variance;
  int64_t n_samples;
  int64_t clamp_events;
} pcb_mcubes_iteration;

typedef struct {
  int32_t iteration;
  int32_t reserved;
  double estimate;
  double errorest;
  double chi2_per_dof;
  double iter_integral;
  double iter_variance;
} pcb_mcubes_progress;

typedef void (*pcb_mcubes_progress_fn)(void* user, const pcb_mcubes_progress* rec);

typedef struct pcb_ctx pcb_ctx;

/* ---- context ------------------------------------------------------------------------- */
pcb_status pcb_ctx_create(int device_ordinal, pcb_ctx** out);
void pcb_ctx_destroy(pcb_ctx* ctx);
const char* pcb_last_error(const pcb_ctx* ctx);
/* Ask the running refine / mcubes_run of this context to stop: callable from inside a progress callback (the
 * reference's drivers propagate an exception raised by `progress` at once, pagani.py:341-349).  The driver returns
 * PCB_ABORTED after the current iteration's record; nothing else of the context is affected.                       */
void pcb_ctx_abort(pcb_ctx* ctx);
/* Scratch memory of a context (region lists, estimates, contribution tables): every buffer is a reserved virtual
 * address range backed by physical chunks on demand (CUDA virtual memory management); growing maps more chunks, the
 * base never moves, nothing is freed or copied, and the context keeps what it has until it is destroyed.  reserve()
 * creates `bytes` of physical chunks up front, so that the first large call maps them instead of asking the driver for
 * memory inside its loop (a refine() to the default region cap 2^26 at d = 8 peaks at ~11 GB).
 * *reserved_out = bytes held in reserve afterwards.                                                                */
pcb_status pcb_ctx_reserve(pcb_ctx* ctx, uint64_t bytes, uint64_t* reserved_out);
/* name and SM count of the context's device, multiprocessor clock in kHz */
pcb_status pcb_device_info(pcb_ctx* ctx, char* name, int name_len, int32_t* sm_count, int32_t* clock_khz);
/* kernels launched by this context since creation (bench.py "gpu_launches") */
int64_t pcb_launch_count(const pcb_ctx* ctx);
/* Measured FP64 peak: runs a dependent-free DFMA loop on every SM; returns TFLOP/s. */
pcb_status pcb_measure_fp64_peak(pcb_ctx* ctx, double* tflops);

/* ---- per-kernel timing for the roofline report -------------------------------------------
 * Between begin and end every launch of the two dominant kernels (PAGANI evaluate, the m-Cubes
 * V-Sample pass) is bracketed by CUDA events on the launching stream.  `kind` 0 = evaluate (units =
 * regions), 1 = V-Sample pass, sampling and accumulation phases (units = samples); 2 is unused since the
 * accumulation moved into the pass kernel.  end() synchronises and returns the sums.          */
pcb_status pcb_profile_begin(pcb_ctx* ctx);
pcb_status pcb_profile_end(pcb_ctx* ctx, int32_t kind, double* kernel_ms, int64_t* launches, double* units);

/* ---- integrand functors: replaces Integrand.eval_many (core.py:66-68, integrands.py) --- */
pcb_status pcb_eval_points(pcb_ctx* ctx, const pcb_integrand* f, int64_t n, const double* points /* (n,d) */,
                           double* values /* (n) */);

/* ---- independent QMC oracle: replaces the sampling loop of integrands.oracle_integral (integrands.py:223-260) -------
 * sums[s] = sum over the first 2^log2_points points of the unscrambled Sobol' sequence (Joe-Kuo direction numbers, 30
 * bits, Gray-code order: the generator behind scipy.stats.qmc.Sobol) of f(frac(point + shifts[s])).  The caller draws
 * the shifts and forms mean / 3 standard errors from the per-shift averages like the reference.                    */
pcb_status pcb_qmc_shift_sums(pcb_ctx* ctx, const pcb_integrand* f, int32_t log2_points, int32_t n_shifts,
                              const double* shifts /* (n_shifts, d) */, double* sums /* (n_shifts) */);

/* ---- serial integrand invocation micro-benchmark: replaces cli.cmd_bench_invoke's loop (cli.py:134-142;
 * PAPER.md:451-455): blocks*threads device threads each evaluate all n points serially, keeping a running
 * sum; ms_out[repetitions] are CUDA-event times, *accumulator is thread 0's sum (the reference's `acc`). */
pcb_status pcb_bench_invoke(pcb_ctx* ctx, const pcb_integrand* f, int64_t n, const double* points, int32_t blocks,
                            int32_t threads, int32_t repetitions, double* ms_out, double* accumulator);

/* ---- PAGANI evaluate: replaces pagani_kernel (pagani.py:227-257) ------------------------
 * lefts/lengths: (n,d) row-major as in RegionList (core.py:187-207); outputs as in
 * RegionEstimates (core.py:224-247): integrals, errors float64, split_axes int64.            */
pcb_status pcb_pagani_evaluate(pcb_ctx* ctx, const pcb_integrand* f, const pcb_rule* rule,
                               const pcb_pagani_config* cfg, int64_t n, const double* lefts,
                               const double* lengths, double* integrals, double* errors,
                               int64_t* split_axes, pcb_nonfinite* bad);
/* Same on device-resident structure-of-arrays buffers: lefts_dev[j*ld + r]; split_axes int32. */
pcb_status pcb_pagani_evaluate_dev(pcb_ctx* ctx, const pcb_integrand* f, const pcb_rule* rule,
                                   const pcb_pagani_config* cfg, int64_t n, int64_t ld,
                                   const double* lefts_dev, const double* lengths_dev,
                                   double* integrals_dev, double* errors_dev, int32_t* split_axes_dev,
                                   pcb_nonfinite* bad);
/* quadrature.apply_rules (quadrature.py:305-322): one region, plain pair tree over all points */
pcb_status pcb_apply_rules(pcb_ctx* ctx, const pcb_integrand* f, int32_t f_eval, const double* generators,
                           const double* weights, const double* left, const double* length,
                           double values[5], double* stored_evals, pcb_nonfinite* bad);

/* ---- PAGANI refine: replaces refine (pagani.py:300-391), whole loop device-resident -------
 * records: capacity cfg->max_iterations + 1.  progress may be NULL.                            */
pcb_status pcb_pagani_refine(pcb_ctx* ctx, const pcb_integrand* f, const pcb_rule* rule,
                             const pcb_pagani_config* cfg, pcb_pagani_result* result,
                             pcb_pagani_progress* records, pcb_pagani_progress_fn progress, void* user,
                             pcb_nonfinite* bad);

/* ---- PAGANI on a shard of the region list (multi-GPU; one context per rank) ------------------
 * The ordered global region list is the concatenation of the ranks' slices.  These calls run one
 * step of refine (pagani.py:300-391) on the local slice and leave the collectives to the host
 * (paper_2302_05730_b200/sharded.py: torch.distributed over NCCL).
 *   init      local slice [first, first+count) of the g^d uniform tiling (core.py:250-269), then evaluate
 *   reduce    `which` 0/1 = active integrals/errors, 2/3 = integrals/errors retired by the last split.
 *             With `head` = number of local elements before the first 1024-aligned GLOBAL index it returns
 *             the raw head elements, the sums of the full aligned 1024-blocks (pair tree, engine.py:69-86)
 *             and the raw tail elements, so every rank can finish the global tree bit-identically.
 *   classify  split mask (pagani.py:361-365): mode 0 err > budget*vol, mode 1 err >= emax; returns the count
 *   split     stable compaction + bisection of the marked regions (pagani.py:282-297, 371-377); the children
 *             become the local list (not yet evaluated), the rest is retired
 *   export    rows [begin, end) of the local list in the reference's (n,d) row-major layout
 *   rebuild   new local list = front rows ++ local[keep_begin, keep_end) ++ back rows  (rebalancing)
 *   evaluate  evaluate the local list                                                                  */
pcb_status pcb_pagani_shard_init(pcb_ctx* ctx, const pcb_integrand* f, const pcb_rule* rule, const pcb_pagani_config* cfg,
                                 int32_t g, int64_t first, int64_t count, pcb_nonfinite* bad);
pcb_status pcb_pagani_shard_count(pcb_ctx* ctx, int64_t* n_active, int64_t* n_retired);
pcb_status pcb_pagani_shard_reduce(pcb_ctx* ctx, int32_t which, int64_t head, double* head_vals, int64_t* n_blocks,
                                   double* block_sums, double* tail_vals, int64_t* n_tail);
pcb_status pcb_pagani_shard_max_error(pcb_ctx* ctx, double* emax);
pcb_status pcb_pagani_shard_classify(pcb_ctx* ctx, double budget, int32_t mode, double emax, int64_t* n_split);
pcb_status pcb_pagani_shard_split(pcb_ctx* ctx);
pcb_status pcb_pagani_shard_export(pcb_ctx* ctx, int64_t begin, int64_t end, double* lefts_rows, double* lengths_rows);
pcb_status pcb_pagani_shard_rebuild(pcb_ctx* ctx, int64_t keep_begin, int64_t keep_end, int64_t n_front,
                                    const double* front_lefts, const double* front_lengths, int64_t n_back,
                                    const double* back_lefts, const double* back_lengths);
pcb_status pcb_pagani_shard_evaluate(pcb_ctx* ctx, pcb_nonfinite* bad);

/* ---- the same steps with the collectives on DEVICE buffers (NCCL on the context's stream, no host staging) ----
 *   deferred      on: init / evaluate / split only enqueue; the slice's non-finite flag travels in the packed row
 *   pack          this rank's row of the iteration: non-finite flag, counts, and for the active (and, with_retired, the
 *                 just-retired) integrals and errors the raw head / tail values around the 1024-aligned GLOBAL blocks plus
 *                 the pair-tree sums of the complete blocks; `width` >= max over ranks of count/1024 + 1.  The host
 *                 all-gathers `row` into `gathered` (world rows; == row for world 1) on `stream`
 *   global_sums   finishes engine.tree_sum over the concatenated global arrays from the gathered rows, on the device,
 *                 and returns (sum I, sum E, retired I, retired E) -- bit-identical to one device for any world size --
 *                 and the lowest rank that saw a non-finite evaluation (-1: none).  One synchronisation
 *   nonfinite     on that rank: the offending (local region, point, value, abscissa)
 *   classify_dev  split mask + (split count, max error) as two doubles in *row; the host all-gathers them into
 *                 *gathered (2*world doubles) and reads them
 *   split_dev     split with the local count taken from that read
 *   list_dev / rebuild_dev   the local list [d][ld] for rank-to-rank sends; new list = front ++ local[keep) ++ back
 *                 with front/back received blocks laid out [2][d][n] (lefts, lengths)                            */
typedef struct {
  void* stream;
  double* row;
  double* gathered;
  int64_t row_doubles;
} pcb_pagani_shard_rows;
pcb_status pcb_pagani_shard_deferred(pcb_ctx* ctx, int32_t on);
pcb_status pcb_pagani_shard_pack(pcb_ctx* ctx, int64_t head_active, int64_t head_retired, int32_t with_retired, int64_t width,
                                 int32_t world, pcb_pagani_shard_rows* out);
pcb_status pcb_pagani_shard_global_sums(pcb_ctx* ctx, int32_t world, int64_t n_active_total, int64_t n_retired_total,
                                        double sums[4], int32_t* bad_rank);
pcb_status pcb_pagani_shard_nonfinite(pcb_ctx* ctx, pcb_nonfinite* bad);
pcb_status pcb_pagani_shard_classify_dev(pcb_ctx* ctx, double budget, int32_t mode, double emax, int32_t world, double** row,
                                         double** gathered);
pcb_status pcb_pagani_shard_split_dev(pcb_ctx* ctx, int64_t n_split);
pcb_status pcb_pagani_shard_list_dev(pcb_ctx* ctx, double** lefts, double** lengths, int64_t* n, int64_t* ld);
pcb_status pcb_pagani_shard_rebuild_dev(pcb_ctx* ctx, int64_t keep_begin, int64_t keep_end, int64_t n_front,
                                        const double* front_dev, int64_t n_back, const double* back_dev);

/* ---- fixed-shape reductions: replaces engine.tree_sum (engine.py:69-86) --------------- */
pcb_status pcb_tree_sum(pcb_ctx* ctx, int64_t n, const double* values, double* out);

/* ---- m-Cubes V-Sample: replaces mcubes_kernel (mcubes.py:268-308) ------------------------
 * boundaries: (d, n_bins+1) as VegasGrid.boundaries (vegas_grid.py:21-43).
 * Logical threads [thread_begin, thread_end) are processed (whole range = one GPU; a
 * sub-range = one shard, mcubes.py:224-232 makes draws independent of the partition).
 * group_partials (optional, may be NULL): (n_groups_touched, 2) per-work-group (I, Var) partial
 * sums in group order starting at group thread_begin / group_size (mcubes.py:292-293).
 * contributions: (d, n_bins) (mcubes.py:294-298).                                            */
pcb_status pcb_mcubes_sample(pcb_ctx* ctx, const pcb_integrand* f, const pcb_mcubes_plan* plan,
                             const double* boundaries, uint64_t seed, int32_t rng_kind,
                             const double* injected_uniforms, int32_t squared_weighted,
                             int64_t thread_begin, int64_t thread_end, pcb_mcubes_iteration* out,
                             double* contributions, double* group_partials, pcb_nonfinite* bad);

/* ---- single sub-cube sampler: replaces mcubes.sample_cube (mcubes.py:143-164) ----------------
 * The caller draws the p*d uniforms (the reference takes them from a duck-typed `rng.take(p*d)`, reshaped (p, d):
 * the injection route of SURVEY 0.1) and gets back S1 = tree_sum(v), S2 = tree_sum(v*v) (engine.py:69-86 over the
 * p values) and the reference's bin_hits as bins (p, d) int64 + weights (p) = v^2.  A non-finite integrand value
 * returns PCB_NONFINITE with the sample's point and value in `bad`.                                   */
pcb_status pcb_mcubes_sample_cube(pcb_ctx* ctx, const pcb_integrand* f, const pcb_mcubes_plan* plan,
                                  const double* boundaries, int64_t cube_index, const double* uniforms /* (p,d) */,
                                  double* s1, double* s2, int64_t* bins /* (p,d) */, double* weights /* (p) */,
                                  pcb_nonfinite* bad);

/* ---- grid refinement: replaces refine_grid (vegas_grid.py:142-193) --------------------- */
pcb_status pcb_grid_refine(pcb_ctx* ctx, int32_t d, int32_t n_bins, const double* boundaries,
                           const double* contributions, double alpha, int32_t smoothing,
                           double* new_boundaries);

/* ---- grid transform: replaces transform / transform_many (vegas_grid.py:87-114) -------------
 * y: (n,d) in [0,1); outputs x (n,d), jac (n), bins (n,d) int64.  Returns PCB_INVALID when a
 * coordinate lies outside [0,1) (the reference's ValueError).                                   */
pcb_status pcb_grid_transform(pcb_ctx* ctx, int32_t d, int32_t n_bins, const double* boundaries, int64_t n,
                              const double* y, double* x, double* jac, int64_t* bins);

/* ---- m-Cubes driver: replaces run (mcubes.py:332-382), loop device-resident ---------------
 * rel_tol <= 0 and abs_tol <= 0 reproduce the reference (fixed iteration count); otherwise the run stops after
 * the first iteration with errorest <= max(abs_tol, rel_tol*|estimate|).  rel_tol > 0 adds the
 * time-to-epsrel stop of BASELINE.md section 3.  iterations_out: capacity `iterations`.
 * final_boundaries (optional): (d, n_bins+1).                                                 */
/* Limits: the run's group-order tree covers at most 1024 work-groups (the reference's default plans have <= 256,
 * mcubes.py:110-129: target_groups = 256); pcb_mcubes_sample has no such limit.                                     */
pcb_status pcb_mcubes_run(pcb_ctx* ctx, const pcb_integrand* f, const pcb_mcubes_plan* plan,
                          int32_t iterations, uint64_t seed, int32_t rng_kind, int32_t adapt, double alpha,
                          int32_t smoothing, double rel_tol, double abs_tol,
                          pcb_mcubes_iteration* iterations_out,
                          int32_t* n_done, pcb_mcubes_progress_fn progress, void* user,
                          double* contributions_out /* optional (iterations, d, n_bins) */,
                          double* final_boundaries, double* seconds_device, pcb_nonfinite* bad);

/* ---- m-Cubes driver on a shard of the sub-cubes (multi-GPU; one context per rank) ----------------
 * Same device-resident loop as pcb_mcubes_run with the logical threads sharded over `world` ranks on work-group
 * boundaries (rank r owns groups [G*r/world, G*(r+1)/world); any partition draws the same samples,
 * mcubes.py:224-232).  Nothing here waits for the device except wait() and end(); the host issues, per iteration,
 *     pass(it);  all-gather of `row` into `gathered`;  all-reduce (sum) of `table` in place;  finish(it)
 * with the two collectives ON `stream` (NCCL through torch.distributed in paper_2302_05730_b200/sharded.py; none
 * for world == 1), and may enqueue iteration it+1 before it waits for the record of iteration it.
 *   row       this rank's per-work-group (I, Var) partials (mcubes.py:255-259), zero padded to ceil(G/world) pairs,
 *             then its first non-finite sample index and its clamp count (8-byte integers)
 *   gathered  `world` rows in rank order; every rank finishes the reference's group-order pair tree
 *             (mcubes.py:292-293) over all G pairs: (integral, variance) are bit-identical for any world size
 *   table     the pass's (d, n_bins) contribution table (mcubes.py:294-298); after the all-reduce every rank refines
 *             the identical grid                                                                          */
typedef struct {
  void* stream;        /* cudaStream_t of the context */
  double* row;         /* device, row_doubles */
  double* gathered;    /* device, world * row_doubles (== row when world == 1) */
  double* table;       /* device, table_doubles */
  int64_t row_doubles;
  int64_t table_doubles;
  int64_t thread_begin, thread_end; /* this rank's logical threads */
} pcb_mcubes_shard_buffers;
pcb_status pcb_mcubes_shard_begin(pcb_ctx* ctx, const pcb_integrand* f, const pcb_mcubes_plan* plan, int32_t iterations,
                                  uint64_t seed, int32_t rng_kind, int32_t adapt, double alpha, int32_t smoothing,
                                  double rel_tol, double abs_tol, int32_t keep_tables, int32_t rank, int32_t world,
                                  pcb_mcubes_shard_buffers* out);
pcb_status pcb_mcubes_shard_pass(pcb_ctx* ctx, int32_t iteration);
pcb_status pcb_mcubes_shard_finish(pcb_ctx* ctx, int32_t iteration);
/* blocks until iteration's record arrives; *stop != 0: the run's tolerance is met (identical on every rank) */
pcb_status pcb_mcubes_shard_wait(pcb_ctx* ctx, int32_t iteration, pcb_mcubes_iteration* out, int32_t* stop, pcb_nonfinite* bad);
/* drains the stream; contributions_out (n_done, d, n_bins) needs keep_tables; final_boundaries (d, n_bins+1) */
pcb_status pcb_mcubes_shard_end(pcb_ctx* ctx, int32_t n_done, double* contributions_out, double* final_boundaries,
                                double* seconds_device);

/* ---- run-time families ------------------------------------------------------------------------
 * Load `cubin` (compiled for sm_100a from this library's kernel templates) as family `family` in
 * [PCB_USER_FAMILY_BASE, PCB_USER_FAMILY_BASE + PCB_MAX_USER_FAMILIES) for dimension d; every kernel named in
 * `names` must exist in the image.  Process-wide; reloading a slot replaces it.                              */
pcb_status pcb_user_family_load(pcb_ctx* ctx, int32_t family, int32_t d, const void* cubin, uint64_t bytes,
                                const pcb_user_kernel_names* names);
pcb_status pcb_user_family_unload(pcb_ctx* ctx, int32_t family);

/* ---- RNG mirror: replaces mcubes._uniform / derive_seed (mcubes.py:51-60) -------------- */
pcb_status pcb_uniforms(pcb_ctx* ctx, uint64_t seed, int32_t rng_kind, int64_t n, const uint64_t* streams,
                        const uint64_t* counters, double* out);

/* ---- self-test hook: the sampler's division-by-constant sequence, out[i] = x[i] / g (g >= 1), and its
 * branch-free reciprocal, out[i] = 1 / x[i] for normal x (g == 0)
 * (tests compare both bit-for-bit with IEEE division; not part of the reference surface)          */
pcb_status pcb_debug_divide(pcb_ctx* ctx, int64_t n, const double* x, int32_t g, double* out);

#ifdef __cplusplus
}
#endif
#endif /* PARCUBE_B200_H */
