// PAGANI C-ABI: evaluate (host and device buffers), apply_rules, tree_sum and the refinement driver.
// Reference: pagani.py:195-391, engine.py:69-86, quadrature.py:305-322.
#include "pagani_driver.cuh"
#include "pagani_eval.cuh"
#include "pcb_host.h"

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cmath>
#include <cstring>

namespace pcb {

// Every kernel of this file waits for its producers at pdl_wait(), so all of them are launched with programmatic
// stream serialisation: back-to-back kernels of an iteration (evaluate -> tree levels -> classify -> scan, split ->
// tree levels -> evaluate) overlap launch latency with the tail of their predecessor (0.8 us per boundary instead
// of 2.5-3.5 us; ~15 boundaries per iteration of the general path).
template <class... Args>
static cudaError_t launch(pcb_ctx* ctx, const void* fn, dim3 grid, dim3 block, size_t smem, Args... a) {
  void* args[] = {(void*)&a...};
  ctx->launches++;
  return launch_pdl(fn, grid, block, args, smem, ctx->stream);
}

static pcb_status validate_rule(pcb_ctx* ctx, const pcb_integrand* f, const pcb_rule* rule, const pcb_pagani_config* cfg) {
  if (!rule || !cfg) return fail(ctx, PCB_INVALID, "rule/config is NULL");
  if (rule->d != f->d) return fail(ctx, PCB_INVALID, "rule, regions, and integrand dimensions must agree");
  if (rule->f_eval != (1 << rule->d) + 2 * rule->d * rule->d + 2 * rule->d + 1)
    return fail(ctx, PCB_INVALID, "rule f_eval %d is not 2^d + 2d^2 + 2d + 1", rule->f_eval);
  if (cfg->group_size < 1) return fail(ctx, PCB_INVALID, "group_size must be >= 1");
  if (cfg->err_mode < 0 || cfg->err_mode > 2) return fail(ctx, PCB_INVALID, "unknown err_mode %d", cfg->err_mode);
  return PCB_OK;
}

static int eval_grid(pcb_ctx* ctx, const void* fn, long long n) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kEvalWarps * 32, 0);
  if (per_sm < 1) per_sm = 1;
  long long want = (n + kEvalWarps - 1) / kEvalWarps;
  return (int)std::min<long long>(want, (long long)per_sm * ctx->sm_count);
}

// launch the evaluate kernel on SoA device buffers; `bad_dev` must already hold ~0
static pcb_status evaluate_launch(pcb_ctx* ctx, const pcb_integrand* f, const pcb_rule* rule, const pcb_pagani_config* cfg,
                                  long long n, long long ld, const double* lefts, const double* lengths, double* I, double* E,
                                  int32_t* K, unsigned long long* bad_dev, const ShortState* state = nullptr) {
  // state != NULL: a speculative launch for a list of at most n regions whose length and stride the kernel takes from
  // the device (warp-per-region kernels only)
  EvalArgs a;
  a.state = state;
  a.f = *f;
  a.rule = *rule;
  a.n = n;
  a.ld = ld;
  a.lefts = lefts;
  a.lengths = lengths;
  a.integrals = I;
  a.errors = E;
  a.split_axes = K;
  a.bad = bad_dev;
  a.group = cfg->group_size;
  a.err_mode = cfg->err_mode;
  a.rel_floor = cfg->rel_floor;
  // Long lists of a multiplicative family at the default schedule width go to the one-region-per-lane kernel
  // (FP64-bound); short lists keep one warp per region (more parallelism per region).  The two agree bit for
  // bit (tests/test_gpu_pagani.py), so the choice never shows in the results.
  size_t lanes_smem = 0;
  int lanes_threads = 32;
  const void* lanes_fn = cfg->group_size == 64 ? eval_lanes_kernel(f->family, f->d, &lanes_smem, &lanes_threads) : nullptr;
  long long lanes_min = 12288;   // measured crossover: one batch of 32 regions per warp takes ~21 us whatever the list length
  size_t lanes_cap = 56u << 10;
  if (const char* env = std::getenv("PCB_PAGANI_LANES_MIN")) {  // test hook: force either kernel
    lanes_min = std::atoll(env);
    lanes_cap = ctx->smem_optin;
  }
  // below ~4 resident warps per SM (52 KB of tables per warp) the lane kernel no longer hides its latency
  // the lane kernels hard-wire which rule alternates its corner weights with the bit count (kParityRule)
  bool parity_ok = true;
  for (int k = 0; k < 5; ++k) parity_ok = parity_ok && ((rule->corner_parity[k] != 0) == (k == kParityRule));
  if (!state && lanes_fn && parity_ok && lanes_smem <= lanes_cap && n >= lanes_min) {
    size_t& have = ctx->smem_attr[lanes_fn];
    if (have < lanes_smem) {
      PCB_CUDA_TRY(ctx, cudaFuncSetAttribute(lanes_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lanes_smem));
      have = lanes_smem;
    }
    int per_sm = (int)std::min<size_t>(32, (ctx->smem_per_sm - 1024) / (lanes_smem + 1024));
    if (per_sm < 1) per_sm = 1;
    const long long want = (n + 31) / 32;
    ProfileSpan span(ctx, 0, (double)n);
    PCB_CUDA_TRY(ctx, launch(ctx, lanes_fn, dim3((unsigned)std::min<long long>(want, (long long)per_sm * ctx->sm_count)), dim3(lanes_threads), lanes_smem, a));
    return PCB_OK;
  }
  // widths above 64 take the exact-order kernel in its block-walking form (pagani.py:175-192 for any G)
  const void* fn = cfg->group_size > 64 ? eval_wide_kernel(f->family, f->d) : eval_kernel(f->family, f->d);
  ProfileSpan span(ctx, 0, state ? 0.0 : (double)n);
  PCB_CUDA_TRY(ctx, launch(ctx, fn, dim3(eval_grid(ctx, fn, n)), dim3(kEvalWarps * 32), 0, a));
  return PCB_OK;
}

// CUDA loads a kernel's code when it is first launched (lazy module loading): tens of milliseconds for the large
// evaluate kernels, in the middle of whichever run happens to need the kernel first -- the config-5 sweep showed
// it as runs 45x slower than a neighbour with more regions (the lane kernel is first used when a list passes 12288
// regions).  A refinement therefore touches every kernel it may launch before its clock starts; once per kernel
// and context.
static pcb_status preload_refine_kernels(pcb_ctx* ctx, const pcb_integrand* f, const pcb_pagani_config* cfg) {
  size_t lanes_smem = 0;
  int lanes_threads = 32;
  const void* lanes_fn = cfg->group_size == 64 ? eval_lanes_kernel(f->family, f->d, &lanes_smem, &lanes_threads) : nullptr;
  const void* fns[] = {cfg->group_size > 64 ? eval_wide_kernel(f->family, f->d) : eval_kernel(f->family, f->d), lanes_fn,
                       (const void*)&tiling_kernel, (const void*)&tree_level_kernel, (const void*)&tree_level2_kernel, (const void*)&short_iteration_kernel,
                       (const void*)&classify_kernel, (const void*)&scan_counts_kernel, (const void*)&max_kernel,
                       (const void*)&split_kernel, (const void*)&publish_scalars_kernel};
  for (const void* fn : fns) {
    if (!fn || !ctx->preloaded.insert(fn).second) continue;
    cudaFuncAttributes attr;
    PCB_CUDA_TRY(ctx, cudaFuncGetAttributes(&attr, fn));
  }
  if (lanes_fn && lanes_smem <= ctx->smem_optin) {
    size_t& have = ctx->smem_attr[lanes_fn];
    if (have < lanes_smem) {
      PCB_CUDA_TRY(ctx, cudaFuncSetAttribute(lanes_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lanes_smem));
      have = lanes_smem;
    }
  }
  return PCB_OK;
}

// engine.tree_sum of two arrays of the same length, level by level in shared launches (same bits as two tree_sum_dev)
static pcb_status tree_sum2_dev(pcb_ctx* ctx, const double* in0, const double* in1, long long n, double* out0, double* out1) {
  if (n <= 0) {
    PCB_CUDA_TRY(ctx, cudaMemsetAsync(out0, 0, sizeof(double), ctx->stream));
    PCB_CUDA_TRY(ctx, cudaMemsetAsync(out1, 0, sizeof(double), ctx->stream));
    return PCB_OK;
  }
  int which = 0;
  while (true) {
    const long long nb = (n + kTreeSpan - 1) / kTreeSpan;
    double *dst0 = out0, *dst1 = out1;
    if (nb > 1) {   // the two arrays' block sums share one ping-pong buffer, second half for the second array
      PCB_CUDA_TRY(ctx, ctx->tree[which].ensure((size_t)2 * nb * sizeof(double)));
      dst0 = ctx->tree[which].as<double>();
      dst1 = dst0 + nb;
    }
    PCB_CUDA_TRY(ctx, launch(ctx, (const void*)&tree_level2_kernel, dim3((unsigned)nb, 2), dim3(kTreeBlock), 0, in0, in1, n, dst0, dst1));
    if (nb == 1) return PCB_OK;
    in0 = dst0;
    in1 = dst1;
    n = nb;
    which ^= 1;
  }
}

pcb_status tree_sum_dev(pcb_ctx* ctx, const double* in, long long n, double* out) {
  if (n <= 0) {
    PCB_CUDA_TRY(ctx, cudaMemsetAsync(out, 0, sizeof(double), ctx->stream));
    return PCB_OK;
  }
  int which = 0;
  while (true) {
    long long nb = (n + kTreeSpan - 1) / kTreeSpan;
    double* dst = out;
    if (nb > 1) {
      PCB_CUDA_TRY(ctx, ctx->tree[which].ensure((size_t)nb * sizeof(double)));
      dst = ctx->tree[which].as<double>();
    }
    PCB_CUDA_TRY(ctx, launch(ctx, (const void*)&tree_level_kernel, dim3((unsigned)nb), dim3(kTreeBlock), 0, in, n, dst));
    if (nb == 1) return PCB_OK;
    in = dst;
    n = nb;
    which ^= 1;
  }
}

static void point_of(const pcb_rule* rule, int d, long long point, const double* left, const double* length, double* x) {
  // abscissa of rule point `point` in canonical order: left + length*offset (quadrature.py:299-302)
  int cand[PCB_MAX_DIM] = {0};
  const int fe = rule->f_eval, corner0 = fe - (1 << d);
  if (point >= corner0) {
    long long bits = point - corner0;
    for (int j = 0; j < d; ++j) cand[j] = 5 + (int)((bits >> j) & 1);
  } else if (point > 4 * d) {
    long long q = point - 1 - 4 * d, pr = q >> 2, sg = q & 3, idx = 0;
    for (int j = 0; j < d; ++j)
      for (int k = j + 1; k < d; ++k, ++idx)
        if (idx == pr) { cand[j] = 3 + (int)(sg & 1); cand[k] = 3 + (int)(sg >> 1); }
  } else if (point > 2 * d) {
    long long q = point - 1 - 2 * d;
    cand[q >> 1] = 3 + (int)(q & 1);
  } else if (point > 0) {
    long long q = point - 1;
    cand[q >> 1] = 1 + (int)(q & 1);
  }
  for (int j = 0; j < d; ++j) {
    volatile double prod = length[j] * rule->offsets[cand[j]];  // two roundings, never contracted
    x[j] = left[j] + prod;
  }
}

pcb_status fetch_nonfinite_pagani(pcb_ctx* ctx, const pcb_integrand* f, const pcb_rule* rule, long long ld,
                                  const double* lefts_dev, const double* lengths_dev, unsigned long long flat,
                                  pcb_nonfinite* bad) {
  const long long region = (long long)(flat / (unsigned long long)rule->f_eval);
  const long long point = (long long)(flat % (unsigned long long)rule->f_eval);
  double left[PCB_MAX_DIM], length[PCB_MAX_DIM], x[PCB_MAX_DIM], value = NAN;
  for (int j = 0; j < f->d; ++j) {
    PCB_CUDA_TRY(ctx, cudaMemcpyAsync(&left[j], lefts_dev + j * ld + region, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    PCB_CUDA_TRY(ctx, cudaMemcpyAsync(&length[j], lengths_dev + j * ld + region, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  }
  PCB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  point_of(rule, f->d, point, left, length, x);
  pcb_status st = pcb_eval_points(ctx, f, 1, x, &value);
  if (st != PCB_OK) return st;
  if (bad) {
    bad->region_index = region;
    bad->point_index = point;
    bad->value = value;
    std::memset(bad->point, 0, sizeof bad->point);
    std::memcpy(bad->point, x, sizeof(double) * f->d);
  }
  return fail(ctx, PCB_NONFINITE, "non-finite integrand value %g in region %lld (rule point %lld)", value, region, point);
}

static pcb_status read_scalars(pcb_ctx* ctx, int first, int count) {
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync((double*)ctx->pinned + first, ctx->scalars.as<double>() + first, count * sizeof(double),
                                    cudaMemcpyDeviceToHost, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return PCB_OK;
}

// The same read for the refinement loop: a one-warp kernel writes the slots and then a sequence word into pinned
// memory and the host polls the word -- no copy engine, no stream synchronisation (measured on lists of 5e4..3e6
// regions: see DESIGN 4.2).  The stream is queried now and then so that a failed launch surfaces instead of hanging.
static pcb_status publish_scalars(pcb_ctx* ctx, int first, int count) {
  if (!ctx->pg_record) {
    PCB_CUDA_TRY(ctx, cudaMallocHost(&ctx->pg_record, 512));
    std::memset(ctx->pg_record, 0, 512);
  }
  volatile unsigned long long* seq_word = reinterpret_cast<volatile unsigned long long*>(static_cast<char*>(ctx->pg_record) + 256);
  const unsigned long long seq = ++ctx->pg_seq;
  PCB_CUDA_TRY(ctx, launch(ctx, (const void*)&publish_scalars_kernel, dim3(1), dim3(32), 0,
                           (const unsigned long long*)ctx->scalars.as<unsigned long long>(), first, count,
                           (volatile unsigned long long*)ctx->pinned, seq_word, seq));
  for (unsigned spin = 0; *seq_word != seq; ++spin) {
    if ((spin & 0xfff) == 0xfff) {
      cudaError_t e = cudaStreamQuery(ctx->stream);
      if (e != cudaErrorNotReady && *seq_word != seq) {
        (void)cudaGetLastError();
        return fail(ctx, PCB_CUDA, "pagani_refine: the device did not publish its scalars (%s)", cudaGetErrorString(e));
      }
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  return PCB_OK;
}

// scalar slots in ctx->scalars / ctx->pinned
enum { S_BAD = 0, S_SUM_I = 1, S_SUM_E = 2, S_NSPLIT = 3, S_EMAX = 4, S_RET_I = 5, S_RET_E = 6 };

}  // namespace pcb

using namespace pcb;

extern "C" {

pcb_status pcb_tree_sum(pcb_ctx* ctx, int64_t n, const double* values, double* out) {
  if (!ctx || !out || n < 0 || (n > 0 && !values)) return fail(ctx, PCB_INVALID, "tree_sum: bad arguments");
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  if (n > 0) {
    PCB_CUDA_TRY(ctx, ctx->rows_a.ensure((size_t)n * sizeof(double)));
    PCB_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->rows_a.p, values, (size_t)n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  }
  PCB_TRY(tree_sum_dev(ctx, ctx->rows_a.as<double>(), n, ctx->scalars.as<double>() + S_SUM_I));
  PCB_TRY(read_scalars(ctx, S_SUM_I, 1));
  *out = ((double*)ctx->pinned)[S_SUM_I];
  return PCB_OK;
}

pcb_status pcb_pagani_evaluate_dev(pcb_ctx* ctx, const pcb_integrand* f, const pcb_rule* rule, const pcb_pagani_config* cfg,
                                   int64_t n, int64_t ld, const double* lefts_dev, const double* lengths_dev,
                                   double* integrals_dev, double* errors_dev, int32_t* split_axes_dev, pcb_nonfinite* bad) {
  if (!ctx) return PCB_INVALID;
  PCB_TRY(validate_integrand(ctx, f));
  PCB_TRY(validate_rule(ctx, f, rule, cfg));
  if (n <= 0) return fail(ctx, PCB_INVALID, "region list is empty");
  if (ld < n) return fail(ctx, PCB_INVALID, "leading dimension %lld < n %lld", (long long)ld, (long long)n);
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  unsigned long long* bad_dev = ctx->scalars.as<unsigned long long>() + S_BAD;
  PCB_CUDA_TRY(ctx, cudaMemsetAsync(bad_dev, 0xFF, sizeof(unsigned long long), ctx->stream));
  PCB_TRY(evaluate_launch(ctx, f, rule, cfg, n, ld, lefts_dev, lengths_dev, integrals_dev, errors_dev, split_axes_dev, bad_dev));
  PCB_TRY(read_scalars(ctx, S_BAD, 1));
  unsigned long long flat = ((unsigned long long*)ctx->pinned)[S_BAD];
  if (flat != ~0ULL) return fetch_nonfinite_pagani(ctx, f, rule, ld, lefts_dev, lengths_dev, flat, bad);
  return PCB_OK;
}

pcb_status pcb_pagani_evaluate(pcb_ctx* ctx, const pcb_integrand* f, const pcb_rule* rule, const pcb_pagani_config* cfg,
                               int64_t n, const double* lefts, const double* lengths, double* integrals, double* errors,
                               int64_t* split_axes, pcb_nonfinite* bad) {
  if (!ctx) return PCB_INVALID;
  PCB_TRY(validate_integrand(ctx, f));
  PCB_TRY(validate_rule(ctx, f, rule, cfg));
  if (n <= 0) return fail(ctx, PCB_INVALID, "region list is empty");
  if (!lefts || !lengths || !integrals || !errors || !split_axes) return fail(ctx, PCB_INVALID, "pagani_evaluate: NULL buffer");
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const int d = f->d;
  const long long ld = round_up(n, 32);
  const size_t row_bytes = (size_t)n * d * sizeof(double);
  PCB_CUDA_TRY(ctx, ctx->rows_a.ensure(row_bytes));
  PCB_CUDA_TRY(ctx, ctx->rows_b.ensure(row_bytes));
  PCB_CUDA_TRY(ctx, ctx->lefts[0].ensure((size_t)ld * d * sizeof(double)));
  PCB_CUDA_TRY(ctx, ctx->lengths[0].ensure((size_t)ld * d * sizeof(double)));
  PCB_CUDA_TRY(ctx, ctx->est_i.ensure((size_t)n * sizeof(double)));
  PCB_CUDA_TRY(ctx, ctx->est_e.ensure((size_t)n * sizeof(double)));
  PCB_CUDA_TRY(ctx, ctx->est_k.ensure((size_t)n * sizeof(int32_t)));
  PCB_CUDA_TRY(ctx, ctx->k64.ensure((size_t)n * sizeof(long long)));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->rows_a.p, lefts, row_bytes, cudaMemcpyHostToDevice, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->rows_b.p, lengths, row_bytes, cudaMemcpyHostToDevice, ctx->stream));
  const int tb = (int)std::min<long long>((n + 255) / 256, (long long)ctx->sm_count * 8);
  rows_to_soa_kernel<<<tb, 256, 0, ctx->stream>>>(d, n, ld, ctx->rows_a.as<double>(), ctx->lefts[0].as<double>());
  rows_to_soa_kernel<<<tb, 256, 0, ctx->stream>>>(d, n, ld, ctx->rows_b.as<double>(), ctx->lengths[0].as<double>());
  ctx->launches += 2;
  pcb_status st = pcb_pagani_evaluate_dev(ctx, f, rule, cfg, n, ld, ctx->lefts[0].as<double>(), ctx->lengths[0].as<double>(),
                                          ctx->est_i.as<double>(), ctx->est_e.as<double>(), ctx->est_k.as<int32_t>(), bad);
  if (st != PCB_OK) return st;
  widen_axes_kernel<<<tb, 256, 0, ctx->stream>>>(n, ctx->est_k.as<int32_t>(), ctx->k64.as<long long>());
  ctx->launches++;
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(integrals, ctx->est_i.p, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(errors, ctx->est_e.p, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(split_axes, ctx->k64.p, (size_t)n * sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return PCB_OK;
}

pcb_status pcb_pagani_refine(pcb_ctx* ctx, const pcb_integrand* f, const pcb_rule* rule, const pcb_pagani_config* cfg,
                             pcb_pagani_result* result, pcb_pagani_progress* records, pcb_pagani_progress_fn progress,
                             void* user, pcb_nonfinite* bad) {
  if (!ctx) return PCB_INVALID;
  PCB_TRY(validate_integrand(ctx, f));
  PCB_TRY(validate_rule(ctx, f, rule, cfg));
  if (!result) return fail(ctx, PCB_INVALID, "result is NULL");
  if (!(cfg->rel_tol > 0)) return fail(ctx, PCB_INVALID, "rel_tol must be > 0");
  if (!(cfg->abs_tol >= 0)) return fail(ctx, PCB_INVALID, "abs_tol must be >= 0");
  if (cfg->max_iterations < 0 || cfg->initial_regions < 1) return fail(ctx, PCB_INVALID, "bad iteration/initial-region budget");
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const int d = f->d;
  const long long launches0 = ctx->launches;

  // iteration 0: smallest g with g^d >= initial_regions (pagani.py:273-279), uniform tiling (core.py:250-269)
  long long g = 1, n = 1;
  long double exact = 1;
  for (;; ++g) {
    exact = 1;
    for (int j = 0; j < d; ++j) exact *= (long double)g;
    if (exact >= (long double)cfg->initial_regions) break;
  }
  if (exact > (long double)cfg->region_cap)
    return fail(ctx, PCB_BUDGET, "uniform split needs %.0Lf regions, cap is %lld", exact, (long long)cfg->region_cap);
  n = (long long)exact;

  PCB_TRY(preload_refine_kernels(ctx, f, cfg));
  // no list of this run is longer than the region cap: bounds for the buffers that scale with the list
  // (DevBuf::hint_max), withdrawn when the run ends -- the sharded entry points size the same buffers per rank
  struct HintGuard {
    pcb_ctx* c;
    void set(size_t list_bytes, size_t scalar_bytes) const {
      for (int b2 = 0; b2 < 2; ++b2) c->lefts[b2].hint_max = c->lengths[b2].hint_max = list_bytes;
      c->est_i.hint_max = c->est_e.hint_max = c->ret_i.hint_max = c->ret_e.hint_max = scalar_bytes;
    }
    ~HintGuard() { set(0, 0); }
  } hint_guard{ctx};
  {
    const size_t cap_regions = (size_t)round_up(cfg->region_cap, 32);
    hint_guard.set(cap_regions * d * sizeof(double), cap_regions * sizeof(double));
  }
  // scalars travel through pinned memory (publish_scalars); PCB_PAGANI_PUBLISH=0: copy + synchronise (A/B runs)
  static const bool use_publish = [] { const char* e = std::getenv("PCB_PAGANI_PUBLISH"); return !(e && std::atoi(e) == 0); }();
  auto fetch = use_publish ? publish_scalars : read_scalars;
  cudaEvent_t ev0, ev1;
  PCB_CUDA_TRY(ctx, cudaEventCreate(&ev0));
  PCB_CUDA_TRY(ctx, cudaEventCreate(&ev1));
  struct EventGuard {
    cudaEvent_t a, b;
    ~EventGuard() { cudaEventDestroy(a); cudaEventDestroy(b); }
  } guard{ev0, ev1};
  cudaEventRecord(ev0, ctx->stream);

  int cur = 0;
  long long ld = round_up(n, 32);
  PCB_CUDA_TRY(ctx, ctx->lefts[cur].ensure((size_t)ld * d * sizeof(double)));
  PCB_CUDA_TRY(ctx, ctx->lengths[cur].ensure((size_t)ld * d * sizeof(double)));
  PCB_CUDA_TRY(ctx, launch(ctx, (const void*)&tiling_kernel, dim3((unsigned)std::min<long long>((n + 255) / 256, 4096)), dim3(256), 0,
                           d, (int)g, 0LL, n, ld, 1.0 / (double)g, ctx->lefts[cur].as<double>(), ctx->lengths[cur].as<double>()));

  double* sc = ctx->scalars.as<double>();
  unsigned long long* sc_u = ctx->scalars.as<unsigned long long>();
  double* host = (double*)ctx->pinned;
  unsigned long long* host_u = (unsigned long long*)ctx->pinned;
  PCB_CUDA_TRY(ctx, cudaMemsetAsync(sc, 0, 16 * sizeof(double), ctx->stream));

  // arm = false: the short-list iteration kernel has already re-armed the non-finite flag on the device
  auto evaluate = [&](long long count, long long ldim, bool arm = true) -> pcb_status {
    PCB_CUDA_TRY(ctx, ctx->est_i.ensure((size_t)count * sizeof(double)));
    PCB_CUDA_TRY(ctx, ctx->est_e.ensure((size_t)count * sizeof(double)));
    PCB_CUDA_TRY(ctx, ctx->est_k.ensure((size_t)count * sizeof(int32_t)));
    if (arm) PCB_CUDA_TRY(ctx, cudaMemsetAsync(sc_u + S_BAD, 0xFF, sizeof(unsigned long long), ctx->stream));
    return evaluate_launch(ctx, f, rule, cfg, count, ldim, ctx->lefts[cur].as<double>(), ctx->lengths[cur].as<double>(),
                           ctx->est_i.as<double>(), ctx->est_e.as<double>(), ctx->est_k.as<int32_t>(), sc_u + S_BAD);
  };
  PCB_TRY(evaluate(n, ld));

  double fin_i = 0.0, fin_e = 0.0, estimate = 0.0, errorest = 0.0;
  long long fin_count = 0, processed = n;
  int n_rec = 0, reason = PCB_STOP_MAX_ITER;
  bool converged = false, have_retired = false;

  // short lists (<= 1024 regions) run the whole iteration in one CTA and hand one record back through pinned memory
  bool use_short = true;
  if (const char* env = std::getenv("PCB_PAGANI_SHORT")) use_short = std::atoi(env) != 0;
  if (!ctx->pg_record) {   // bytes [0, 256): a ring of four short-iteration records, [256, 512): the sequence word of publish_scalars
    PCB_CUDA_TRY(ctx, cudaMallocHost(&ctx->pg_record, 512));
    std::memset(ctx->pg_record, 0, 512);
  }
  static_assert(sizeof(ShortIterRecord) == 64, "four records fit the ring");
  ShortIterRecord* srec_ring = static_cast<ShortIterRecord*>(ctx->pg_record);
  // The short-list chain is device-resident (ShortState): while it lasts the host enqueues the evaluate kernel and the
  // iteration kernel of iteration it+1 -- which take the list length, the running totals and the stop decision from
  // the device -- BEFORE it polls the record of iteration it, so the device never idles on the round trip.
  // PCB_PAGANI_SPECULATE=0: one iteration at a time (A/B runs).  Not with the lane kernels forced onto short lists.
  bool speculate_short = true;
  if (const char* env = std::getenv("PCB_PAGANI_SPECULATE")) speculate_short = std::atoi(env) != 0;
  if (const char* env = std::getenv("PCB_PAGANI_LANES_MIN")) speculate_short = speculate_short && std::atoll(env) > 1024;
  ShortState* state_dev = reinterpret_cast<ShortState*>(sc + 8);   // slots 8..13 of the scalar block (zeroed above)
  static_assert(sizeof(ShortState) <= 8 * sizeof(double), "the state fits the upper half of the scalar block");
  int short_enqueued_upto = -1;   // newest iteration whose iteration kernel is already in the stream
  const unsigned long long run_token = ++ctx->pg_seq;   // record sequence words: (token << 20) | (iteration + 1)

  for (int it = 0; it <= cfg->max_iterations; ++it) {
    if (use_short && n >= 1 && n <= 1024) {
      if (have_retired) {  // fold the general path's pending retirements first
        PCB_TRY(fetch(ctx, 0, 8));
        fin_i += host[S_RET_I];
        fin_e += host[S_RET_E];
        have_retired = false;
      }
      const int nxt = cur ^ 1;
      // both list buffers hold the children of a full short list (2048 regions), the estimate arrays a full short list
      const long long ld_cap = 2048;
      for (int b2 = 0; b2 < 2; ++b2) {
        PCB_CUDA_TRY(ctx, ctx->lefts[b2].ensure((size_t)ld_cap * d * sizeof(double)));
        PCB_CUDA_TRY(ctx, ctx->lengths[b2].ensure((size_t)ld_cap * d * sizeof(double)));
      }
      PCB_CUDA_TRY(ctx, ctx->est_i.ensure((size_t)1024 * sizeof(double)));
      PCB_CUDA_TRY(ctx, ctx->est_e.ensure((size_t)1024 * sizeof(double)));
      PCB_CUDA_TRY(ctx, ctx->est_k.ensure((size_t)1024 * sizeof(int32_t)));
      // iteration kernel of iteration k reading list buffer `in`; from_state: inputs from the device state
      auto launch_short = [&](int k, int in, bool from_state) -> pcb_status {
        ShortIterArgs sa;
        sa.n = (int)n; sa.d = d; sa.ld_in = ld; sa.ld_out_unused = 0;
        sa.lefts = ctx->lefts[in].as<double>();
        sa.lengths = ctx->lengths[in].as<double>();
        sa.integrals = ctx->est_i.as<double>();
        sa.errors = ctx->est_e.as<double>();
        sa.axes = ctx->est_k.as<int32_t>();
        sa.out_lefts = ctx->lefts[in ^ 1].as<double>();
        sa.out_lengths = ctx->lengths[in ^ 1].as<double>();
        sa.fin_i = fin_i; sa.fin_e = fin_e;
        sa.processed = processed; sa.region_cap = cfg->region_cap;
        sa.rel_tol = cfg->rel_tol;
        sa.abs_tol = cfg->abs_tol;
        sa.iteration = k; sa.max_iterations = cfg->max_iterations;
        sa.bad = sc_u + S_BAD;
        sa.record = srec_ring + (k & 3);
        sa.seq = ((unsigned long long)run_token << 20) | (unsigned long long)(k + 1);
        sa.state = state_dev;
        sa.from_state = from_state ? 1 : 0;
        sa.short_max = 1024;
        void* args[] = {&sa};   // dependent launch: resident behind the evaluate kernel, waits for its results (pdl_wait)
        PCB_CUDA_TRY(ctx, launch_pdl((const void*)&short_iteration_kernel, dim3(1), dim3(1024), args, 0, ctx->stream));
        ctx->launches++;
        short_enqueued_upto = k;
        return PCB_OK;
      };
      if (short_enqueued_upto < it) PCB_TRY(launch_short(it, cur, false));
      bool next_enqueued = short_enqueued_upto > it;
      long spec_span = -1;
      if (speculate_short && !next_enqueued && it < cfg->max_iterations) {
        // iteration it+1 on the state iteration it leaves behind: evaluate the children (list buffer nxt), then iterate
        PCB_TRY(evaluate_launch(ctx, f, rule, cfg, 1024, 0, ctx->lefts[nxt].as<double>(), ctx->lengths[nxt].as<double>(),
                                ctx->est_i.as<double>(), ctx->est_e.as<double>(), ctx->est_k.as<int32_t>(), sc_u + S_BAD, state_dev));
        spec_span = ctx->profiling ? (long)ctx->spans[0].size() - 1 : -1;   // its region count is filled in below
        PCB_TRY(launch_short(it + 1, nxt, true));
        next_enqueued = true;
      }
      const ShortIterRecord* srec = srec_ring + (it & 3);
      const unsigned long long want_seq = ((unsigned long long)run_token << 20) | (unsigned long long)(it + 1);
      for (unsigned spin = 0; srec->seq != want_seq; ++spin) {
        if ((spin & 0xfff) == 0xfff) {
          cudaError_t e = cudaStreamQuery(ctx->stream);
          if (e != cudaErrorNotReady && srec->seq != want_seq) {
            (void)cudaGetLastError();
            return fail(ctx, PCB_CUDA, "pagani_refine: short iteration did not publish its record (%s)", cudaGetErrorString(e));
          }
        }
      }
      std::atomic_thread_fence(std::memory_order_acquire);   // the record's fields are read after its sequence word
      if (srec->action == 4)
        return fetch_nonfinite_pagani(ctx, f, rule, ld, ctx->lefts[cur].as<double>(), ctx->lengths[cur].as<double>(), srec->bad, bad);
      estimate = srec->estimate;
      errorest = srec->errorest;
      pcb_pagani_progress rec;
      rec.iteration = it;
      rec.reserved = 0;
      rec.n_regions = fin_count + n;
      rec.active = n;
      rec.estimate = estimate;
      rec.errorest = errorest;
      if (records) records[n_rec] = rec;
      ++n_rec;
      if (progress) {
        ctx->abort_requested = 0;
        progress(user, &rec);
        if (ctx->abort_requested) {
          ctx->abort_requested = 0;
          cudaStreamSynchronize(ctx->stream);
          return fail(ctx, PCB_ABORTED, "refine stopped by its progress callback at iteration %d", it);
        }
      }
      if (srec->action == 1) { converged = true; reason = PCB_STOP_TOLERANCE; break; }
      if (srec->action == 2) { reason = PCB_STOP_MAX_ITER; break; }
      if (srec->action == 3) { reason = PCB_STOP_REGION_CAP; break; }
      const long long n_split = srec->n_split;
      fin_i = srec->fin_i;
      fin_e = srec->fin_e;
      fin_count += n - n_split;
      processed += 2 * n_split;
      n = 2 * n_split;
      ld = round_up(n, 32);
      cur = nxt;
      // the chain goes on by itself while the list stays short; a longer list ended it on the device (status 5: the
      // kernels enqueued ahead return at once) and is evaluated from here
      const bool chained = next_enqueued && n >= 1 && n <= 1024;
      if (spec_span >= 0 && chained) ctx->spans[0][spec_span].units = (double)n;   // profiling: what the speculative launch evaluated
      if (!chained) PCB_TRY(evaluate(n, ld, false));
      continue;
    }
    PCB_TRY(tree_sum2_dev(ctx, ctx->est_i.as<double>(), ctx->est_e.as<double>(), n, sc + S_SUM_I, sc + S_SUM_E));
    // classification (pagani.py:361-365), enqueued before the host has seen the sums: the kernel takes its budget from
    // the same scalars with the host's own expressions, so one round trip returns sums AND split count (the
    // classification of the last iteration is the only work that is ever wasted)
    const long long nblk = (n + kScanBlock - 1) / kScanBlock;
    ClassifyArgs ca;
    const bool speculate = it < cfg->max_iterations && n > 0;
    if (speculate) {
      PCB_CUDA_TRY(ctx, ctx->flags.ensure((size_t)n));
      PCB_CUDA_TRY(ctx, ctx->counts.ensure((size_t)nblk * sizeof(unsigned int)));
      PCB_CUDA_TRY(ctx, ctx->offsets.ensure((size_t)nblk * sizeof(unsigned long long)));
      ca.n = n; ca.ld = ld; ca.d = d; ca.mode = 0; ca.budget = 0.0; ca.emax = 0.0;
      ca.lengths = ctx->lengths[cur].as<double>();
      ca.errors = ctx->est_e.as<double>();
      ca.flags = ctx->flags.as<unsigned char>();
      ca.block_counts = ctx->counts.as<unsigned int>();
      ca.scalars = sc; ca.fin_i = fin_i; ca.rel_tol = cfg->rel_tol; ca.abs_tol = cfg->abs_tol;
      ca.have_retired = have_retired ? 1 : 0; ca.slot_sum_i = S_SUM_I; ca.slot_ret_i = S_RET_I;
      PCB_CUDA_TRY(ctx, launch(ctx, (const void*)&classify_kernel, dim3((unsigned)nblk), dim3(kScanBlock), 0, ca));
      PCB_CUDA_TRY(ctx, launch(ctx, (const void*)&scan_counts_kernel, dim3(1), dim3(1024), 0, (const unsigned int*)ctx->counts.as<unsigned int>(),
                               (int)nblk, ctx->offsets.as<unsigned long long>(), sc_u + S_NSPLIT));
    }
    PCB_TRY(fetch(ctx, 0, 8));
    if (host_u[S_BAD] != ~0ULL)
      return fetch_nonfinite_pagani(ctx, f, rule, ld, ctx->lefts[cur].as<double>(), ctx->lengths[cur].as<double>(), host_u[S_BAD], bad);
    if (have_retired) {  // fin += tree_sum(act[~mask]) of the previous iteration (pagani.py:371-372)
      fin_i += host[S_RET_I];
      fin_e += host[S_RET_E];
      have_retired = false;
    }
    estimate = fin_i + host[S_SUM_I];
    errorest = fin_e + host[S_SUM_E];
    pcb_pagani_progress rec;
    rec.iteration = it;
    rec.reserved = 0;
    rec.n_regions = fin_count + n;
    rec.active = n;
    rec.estimate = estimate;
    rec.errorest = errorest;
    if (records) records[n_rec] = rec;
    ++n_rec;
    if (progress) {
        ctx->abort_requested = 0;
        progress(user, &rec);
        if (ctx->abort_requested) {
          ctx->abort_requested = 0;
          cudaStreamSynchronize(ctx->stream);
          return fail(ctx, PCB_ABORTED, "refine stopped by its progress callback at iteration %d", it);
        }
      }
    if (errorest <= tolerance_target(cfg->rel_tol, cfg->abs_tol, estimate)) {
      converged = true;
      reason = PCB_STOP_TOLERANCE;
      break;
    }
    if (it == cfg->max_iterations) { reason = PCB_STOP_MAX_ITER; break; }
    if (n == 0) { reason = PCB_STOP_NO_ACTIVE; break; }

    long long n_split = (long long)host_u[S_NSPLIT];
    if (n_split == 0) {
      // nothing exceeds its budget: force progress on the worst regions, ties included (pagani.py:364-365)
      PCB_CUDA_TRY(ctx, cudaMemsetAsync(sc + S_EMAX, 0, sizeof(double), ctx->stream));
      PCB_CUDA_TRY(ctx, launch(ctx, (const void*)&max_kernel, dim3((unsigned)std::min<long long>((n + 255) / 256, 1024)), dim3(256), 0,
                               (const double*)ctx->est_e.as<double>(), n, sc + S_EMAX));
      PCB_TRY(fetch(ctx, S_EMAX, 1));
      ca.mode = 1;
      ca.emax = host[S_EMAX];
      ca.scalars = nullptr;
      PCB_CUDA_TRY(ctx, launch(ctx, (const void*)&classify_kernel, dim3((unsigned)nblk), dim3(kScanBlock), 0, ca));
      PCB_CUDA_TRY(ctx, launch(ctx, (const void*)&scan_counts_kernel, dim3(1), dim3(1024), 0, (const unsigned int*)ctx->counts.as<unsigned int>(),
                               (int)nblk, ctx->offsets.as<unsigned long long>(), sc_u + S_NSPLIT));
      PCB_TRY(fetch(ctx, S_NSPLIT, 1));
      n_split = (long long)host_u[S_NSPLIT];
    }
    if (processed + 2 * n_split > cfg->region_cap) { reason = PCB_STOP_REGION_CAP; break; }

    // retire the rest, bisect the split regions (pagani.py:371-378)
    const long long n_child = 2 * n_split, n_ret = n - n_split, ld_out = round_up(n_child, 32);
    const int nxt = cur ^ 1;
    PCB_CUDA_TRY(ctx, ctx->lefts[nxt].ensure((size_t)ld_out * d * sizeof(double)));
    PCB_CUDA_TRY(ctx, ctx->lengths[nxt].ensure((size_t)ld_out * d * sizeof(double)));
    PCB_CUDA_TRY(ctx, ctx->ret_i.ensure((size_t)std::max<long long>(n_ret, 1) * sizeof(double)));
    PCB_CUDA_TRY(ctx, ctx->ret_e.ensure((size_t)std::max<long long>(n_ret, 1) * sizeof(double)));
    SplitArgs sa;
    sa.n = n; sa.ld_in = ld; sa.ld_out = ld_out; sa.d = d;
    sa.lefts = ctx->lefts[cur].as<double>();
    sa.lengths = ctx->lengths[cur].as<double>();
    sa.integrals = ctx->est_i.as<double>();
    sa.errors = ctx->est_e.as<double>();
    sa.axes = ctx->est_k.as<int32_t>();
    sa.flags = ctx->flags.as<unsigned char>();
    sa.block_offsets = ctx->offsets.as<unsigned long long>();
    sa.out_lefts = ctx->lefts[nxt].as<double>();
    sa.out_lengths = ctx->lengths[nxt].as<double>();
    sa.retired_i = ctx->ret_i.as<double>();
    sa.retired_e = ctx->ret_e.as<double>();
    sa.rearm_bad = sc_u + S_BAD;   // instead of a memset between the kernels (it would end their programmatic overlap)
    PCB_CUDA_TRY(ctx, launch(ctx, (const void*)&split_kernel, dim3((unsigned)nblk), dim3(kScanBlock), 0, sa));
    PCB_TRY(tree_sum2_dev(ctx, ctx->ret_i.as<double>(), ctx->ret_e.as<double>(), n_ret, sc + S_RET_I, sc + S_RET_E));
    have_retired = true;  // read back together with the next iteration's sums
    fin_count += n_ret;
    processed += n_child;
    n = n_child;
    ld = ld_out;
    cur = nxt;
    PCB_TRY(evaluate(n, ld, false));
  }

  cudaEventRecord(ev1, ctx->stream);
  PCB_CUDA_TRY(ctx, cudaEventSynchronize(ev1));
  float ms = 0;
  cudaEventElapsedTime(&ms, ev0, ev1);
  result->estimate = estimate;
  result->errorest = errorest;
  result->iterations = n_rec - 1;
  result->converged = converged ? 1 : 0;
  result->regions_processed = processed;
  result->reason = reason;
  result->n_records = n_rec;
  result->seconds_device = ms * 1e-3;
  result->kernel_launches = ctx->launches - launches0;
  return PCB_OK;
}

// ------------------------------------------------------------------------------------------------
// PAGANI on a shard of the region list: one refine step at a time, collectives left to the host.
// ------------------------------------------------------------------------------------------------
static int grid_for(long long n) { return (int)std::max<long long>(1, std::min<long long>((n + 255) / 256, 4096)); }

static pcb_status shard_evaluate(pcb_ctx* ctx, pcb_nonfinite* bad) {
  auto& S = ctx->shard;
  S.classified = false;
  if (S.n == 0) {
    if (S.deferred)   // an empty slice reports "no non-finite evaluation"
      PCB_CUDA_TRY(ctx, cudaMemsetAsync(ctx->scalars.as<unsigned long long>() + S_BAD, 0xFF, sizeof(unsigned long long), ctx->stream));
    return PCB_OK;
  }
  PCB_CUDA_TRY(ctx, ctx->est_i.ensure((size_t)S.n * sizeof(double)));
  PCB_CUDA_TRY(ctx, ctx->est_e.ensure((size_t)S.n * sizeof(double)));
  PCB_CUDA_TRY(ctx, ctx->est_k.ensure((size_t)S.n * sizeof(int32_t)));
  unsigned long long* bad_dev = ctx->scalars.as<unsigned long long>() + S_BAD;
  PCB_CUDA_TRY(ctx, cudaMemsetAsync(bad_dev, 0xFF, sizeof(unsigned long long), ctx->stream));
  PCB_TRY(evaluate_launch(ctx, &S.f, &S.rule, &S.cfg, S.n, S.ld, ctx->lefts[S.cur].as<double>(), ctx->lengths[S.cur].as<double>(),
                          ctx->est_i.as<double>(), ctx->est_e.as<double>(), ctx->est_k.as<int32_t>(), bad_dev));
  if (S.deferred) return PCB_OK;   // the flag is packed into the next row (pcb_pagani_shard_pack)
  PCB_TRY(read_scalars(ctx, S_BAD, 1));
  const unsigned long long flat = ((unsigned long long*)ctx->pinned)[S_BAD];
  if (flat != ~0ULL)
    return fetch_nonfinite_pagani(ctx, &S.f, &S.rule, S.ld, ctx->lefts[S.cur].as<double>(), ctx->lengths[S.cur].as<double>(), flat, bad);
  return PCB_OK;
}

pcb_status pcb_pagani_shard_init(pcb_ctx* ctx, const pcb_integrand* f, const pcb_rule* rule, const pcb_pagani_config* cfg,
                                 int32_t g, int64_t first, int64_t count, pcb_nonfinite* bad) {
  if (!ctx) return PCB_INVALID;
  PCB_TRY(validate_integrand(ctx, f));
  PCB_TRY(validate_rule(ctx, f, rule, cfg));
  if (g < 1 || first < 0 || count < 0) return fail(ctx, PCB_INVALID, "shard_init: bad tiling slice");
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  auto& S = ctx->shard;
  const bool deferred = S.deferred;   // set by pcb_pagani_shard_deferred before init
  S = pcb_ctx::Shard();
  S.deferred = deferred;
  S.live = true;
  S.f = *f; S.rule = *rule; S.cfg = *cfg;
  S.n = count;
  S.ld = round_up(std::max<long long>(count, 1), 32);
  const int d = f->d;
  PCB_CUDA_TRY(ctx, ctx->lefts[0].ensure((size_t)S.ld * d * sizeof(double)));
  PCB_CUDA_TRY(ctx, ctx->lengths[0].ensure((size_t)S.ld * d * sizeof(double)));
  if (count > 0) {
    tiling_kernel<<<grid_for(count), 256, 0, ctx->stream>>>(d, g, (long long)first, (long long)count, S.ld, 1.0 / (double)g,
                                                            ctx->lefts[0].as<double>(), ctx->lengths[0].as<double>());
    ctx->launches++;
  }
  return shard_evaluate(ctx, bad);
}

pcb_status pcb_pagani_shard_count(pcb_ctx* ctx, int64_t* n_active, int64_t* n_retired) {
  if (!ctx || !ctx->shard.live) return fail(ctx, PCB_INVALID, "no live shard");
  if (n_active) *n_active = ctx->shard.n;
  if (n_retired) *n_retired = ctx->shard.n_ret;
  return PCB_OK;
}

pcb_status pcb_pagani_shard_reduce(pcb_ctx* ctx, int32_t which, int64_t head, double* head_vals, int64_t* n_blocks,
                                   double* block_sums, double* tail_vals, int64_t* n_tail) {
  if (!ctx || !ctx->shard.live) return fail(ctx, PCB_INVALID, "no live shard");
  if (which < 0 || which > 3 || head < 0 || head >= kTreeSpan || !n_blocks || !n_tail)
    return fail(ctx, PCB_INVALID, "shard_reduce: bad arguments");
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  auto& S = ctx->shard;
  const long long n = which < 2 ? S.n : S.n_ret;
  const double* src = (which == 0 ? ctx->est_i : which == 1 ? ctx->est_e : which == 2 ? ctx->ret_i : ctx->ret_e).as<double>();
  const long long h = std::min<long long>(head, n);
  const long long nb = (n - h) / kTreeSpan, tail = n - h - nb * kTreeSpan;
  if (h > 0) PCB_CUDA_TRY(ctx, cudaMemcpyAsync(head_vals, src, (size_t)h * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  if (nb > 0) {
    PCB_CUDA_TRY(ctx, ctx->tree[0].ensure((size_t)nb * sizeof(double)));
    tree_level_kernel<<<(unsigned)nb, kTreeBlock, 0, ctx->stream>>>(src + h, nb * kTreeSpan, ctx->tree[0].as<double>());
    ctx->launches++;
    PCB_CUDA_TRY(ctx, cudaMemcpyAsync(block_sums, ctx->tree[0].p, (size_t)nb * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  }
  if (tail > 0)
    PCB_CUDA_TRY(ctx, cudaMemcpyAsync(tail_vals, src + h + nb * kTreeSpan, (size_t)tail * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  *n_blocks = nb;
  *n_tail = tail;
  return PCB_OK;
}

pcb_status pcb_pagani_shard_max_error(pcb_ctx* ctx, double* emax) {
  if (!ctx || !ctx->shard.live || !emax) return fail(ctx, PCB_INVALID, "no live shard");
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  auto& S = ctx->shard;
  double* sc = ctx->scalars.as<double>();
  PCB_CUDA_TRY(ctx, cudaMemsetAsync(sc + S_EMAX, 0, sizeof(double), ctx->stream));
  if (S.n > 0) {
    max_kernel<<<(unsigned)std::min<long long>((S.n + 255) / 256, 1024), 256, 0, ctx->stream>>>(ctx->est_e.as<double>(), S.n, sc + S_EMAX);
    ctx->launches++;
  }
  PCB_TRY(read_scalars(ctx, S_EMAX, 1));
  *emax = ((double*)ctx->pinned)[S_EMAX];
  return PCB_OK;
}

pcb_status pcb_pagani_shard_classify(pcb_ctx* ctx, double budget, int32_t mode, double emax, int64_t* n_split) {
  if (!ctx || !ctx->shard.live || !n_split) return fail(ctx, PCB_INVALID, "no live shard");
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  auto& S = ctx->shard;
  S.n_split = 0;
  S.classified = true;
  *n_split = 0;
  if (S.n == 0) return PCB_OK;
  const long long nblk = (S.n + kScanBlock - 1) / kScanBlock;
  PCB_CUDA_TRY(ctx, ctx->flags.ensure((size_t)S.n));
  PCB_CUDA_TRY(ctx, ctx->counts.ensure((size_t)nblk * sizeof(unsigned int)));
  PCB_CUDA_TRY(ctx, ctx->offsets.ensure((size_t)nblk * sizeof(unsigned long long)));
  ClassifyArgs ca;
  ca.n = S.n; ca.ld = S.ld; ca.d = S.f.d; ca.mode = mode; ca.budget = budget; ca.emax = emax;
  ca.lengths = ctx->lengths[S.cur].as<double>();
  ca.errors = ctx->est_e.as<double>();
  ca.flags = ctx->flags.as<unsigned char>();
  ca.block_counts = ctx->counts.as<unsigned int>();
  unsigned long long* sc_u = ctx->scalars.as<unsigned long long>();
  classify_kernel<<<(unsigned)nblk, kScanBlock, 0, ctx->stream>>>(ca);
  scan_counts_kernel<<<1, 1024, 0, ctx->stream>>>(ctx->counts.as<unsigned int>(), (int)nblk, ctx->offsets.as<unsigned long long>(),
                                                  sc_u + S_NSPLIT);
  ctx->launches += 2;
  PCB_TRY(read_scalars(ctx, S_NSPLIT, 1));
  S.n_split = (long long)((unsigned long long*)ctx->pinned)[S_NSPLIT];
  *n_split = S.n_split;
  return PCB_OK;
}

pcb_status pcb_pagani_shard_split(pcb_ctx* ctx) {
  if (!ctx || !ctx->shard.live) return fail(ctx, PCB_INVALID, "no live shard");
  auto& S = ctx->shard;
  if (!S.classified) return fail(ctx, PCB_INVALID, "shard_split needs a preceding shard_classify");
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const int d = S.f.d, nxt = S.cur ^ 1;
  const long long n_child = 2 * S.n_split, n_ret = S.n - S.n_split, ld_out = round_up(std::max<long long>(n_child, 1), 32);
  PCB_CUDA_TRY(ctx, ctx->lefts[nxt].ensure((size_t)ld_out * d * sizeof(double)));
  PCB_CUDA_TRY(ctx, ctx->lengths[nxt].ensure((size_t)ld_out * d * sizeof(double)));
  PCB_CUDA_TRY(ctx, ctx->ret_i.ensure((size_t)std::max<long long>(n_ret, 1) * sizeof(double)));
  PCB_CUDA_TRY(ctx, ctx->ret_e.ensure((size_t)std::max<long long>(n_ret, 1) * sizeof(double)));
  if (S.n > 0) {
    SplitArgs sa;
    sa.n = S.n; sa.ld_in = S.ld; sa.ld_out = ld_out; sa.d = d;
    sa.lefts = ctx->lefts[S.cur].as<double>();
    sa.lengths = ctx->lengths[S.cur].as<double>();
    sa.integrals = ctx->est_i.as<double>();
    sa.errors = ctx->est_e.as<double>();
    sa.axes = ctx->est_k.as<int32_t>();
    sa.flags = ctx->flags.as<unsigned char>();
    sa.block_offsets = ctx->offsets.as<unsigned long long>();
    sa.out_lefts = ctx->lefts[nxt].as<double>();
    sa.out_lengths = ctx->lengths[nxt].as<double>();
    sa.retired_i = ctx->ret_i.as<double>();
    sa.retired_e = ctx->ret_e.as<double>();
    split_kernel<<<(unsigned)((S.n + kScanBlock - 1) / kScanBlock), kScanBlock, 0, ctx->stream>>>(sa);
    ctx->launches++;
    PCB_CUDA_TRY(ctx, cudaGetLastError());
  }
  S.n_ret = n_ret;
  S.n = n_child;
  S.ld = ld_out;
  S.cur = nxt;
  S.classified = false;
  if (!S.deferred) PCB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return PCB_OK;
}

pcb_status pcb_pagani_shard_export(pcb_ctx* ctx, int64_t begin, int64_t end, double* lefts_rows, double* lengths_rows) {
  if (!ctx || !ctx->shard.live) return fail(ctx, PCB_INVALID, "no live shard");
  auto& S = ctx->shard;
  if (begin < 0 || end > S.n || begin > end) return fail(ctx, PCB_INVALID, "shard_export: range outside the local list");
  const long long n = end - begin;
  if (n == 0) return PCB_OK;
  if (!lefts_rows || !lengths_rows) return fail(ctx, PCB_INVALID, "shard_export: NULL buffer");
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const int d = S.f.d;
  const size_t bytes = (size_t)n * d * sizeof(double);
  PCB_CUDA_TRY(ctx, ctx->rows_a.ensure(bytes));
  PCB_CUDA_TRY(ctx, ctx->rows_b.ensure(bytes));
  soa_to_rows_kernel<<<grid_for(n), 256, 0, ctx->stream>>>(d, begin, n, S.ld, ctx->lefts[S.cur].as<double>(), ctx->rows_a.as<double>());
  soa_to_rows_kernel<<<grid_for(n), 256, 0, ctx->stream>>>(d, begin, n, S.ld, ctx->lengths[S.cur].as<double>(), ctx->rows_b.as<double>());
  ctx->launches += 2;
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(lefts_rows, ctx->rows_a.p, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(lengths_rows, ctx->rows_b.p, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return PCB_OK;
}

pcb_status pcb_pagani_shard_rebuild(pcb_ctx* ctx, int64_t keep_begin, int64_t keep_end, int64_t n_front, const double* front_lefts,
                                    const double* front_lengths, int64_t n_back, const double* back_lefts, const double* back_lengths) {
  if (!ctx || !ctx->shard.live) return fail(ctx, PCB_INVALID, "no live shard");
  auto& S = ctx->shard;
  if (keep_begin < 0 || keep_end > S.n || keep_begin > keep_end || n_front < 0 || n_back < 0)
    return fail(ctx, PCB_INVALID, "shard_rebuild: bad ranges");
  if ((n_front > 0 && (!front_lefts || !front_lengths)) || (n_back > 0 && (!back_lefts || !back_lengths)))
    return fail(ctx, PCB_INVALID, "shard_rebuild: NULL rows");
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const int d = S.f.d, nxt = S.cur ^ 1;
  const long long keep = keep_end - keep_begin, n_new = n_front + keep + n_back;
  if (n_front == 0 && n_back == 0 && keep_begin == 0 && keep_end == S.n) return PCB_OK;  // nothing moves
  const long long ld_new = round_up(std::max<long long>(n_new, 1), 32);
  PCB_CUDA_TRY(ctx, ctx->lefts[nxt].ensure((size_t)ld_new * d * sizeof(double)));
  PCB_CUDA_TRY(ctx, ctx->lengths[nxt].ensure((size_t)ld_new * d * sizeof(double)));
  if (keep > 0) {
    soa_copy_kernel<<<grid_for(keep), 256, 0, ctx->stream>>>(d, keep, S.ld, keep_begin, ctx->lefts[S.cur].as<double>(), ld_new, n_front,
                                                             ctx->lefts[nxt].as<double>());
    soa_copy_kernel<<<grid_for(keep), 256, 0, ctx->stream>>>(d, keep, S.ld, keep_begin, ctx->lengths[S.cur].as<double>(), ld_new, n_front,
                                                             ctx->lengths[nxt].as<double>());
    ctx->launches += 2;
  }
  auto upload = [&](long long n, const double* l_rows, const double* h_rows, long long off) -> pcb_status {
    if (n == 0) return PCB_OK;
    const size_t bytes = (size_t)n * d * sizeof(double);
    PCB_CUDA_TRY(ctx, ctx->rows_a.ensure(bytes));
    PCB_CUDA_TRY(ctx, ctx->rows_b.ensure(bytes));
    PCB_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->rows_a.p, l_rows, bytes, cudaMemcpyHostToDevice, ctx->stream));
    PCB_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->rows_b.p, h_rows, bytes, cudaMemcpyHostToDevice, ctx->stream));
    rows_to_soa_at_kernel<<<grid_for(n), 256, 0, ctx->stream>>>(d, n, ld_new, off, ctx->rows_a.as<double>(), ctx->lefts[nxt].as<double>());
    rows_to_soa_at_kernel<<<grid_for(n), 256, 0, ctx->stream>>>(d, n, ld_new, off, ctx->rows_b.as<double>(), ctx->lengths[nxt].as<double>());
    ctx->launches += 2;
    PCB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));  // rows_a/rows_b are reused by the next upload
    return PCB_OK;
  };
  PCB_TRY(upload(n_front, front_lefts, front_lengths, 0));
  PCB_TRY(upload(n_back, back_lefts, back_lengths, n_front + keep));
  PCB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  S.cur = nxt;
  S.n = n_new;
  S.ld = ld_new;
  return PCB_OK;
}

pcb_status pcb_pagani_shard_evaluate(pcb_ctx* ctx, pcb_nonfinite* bad) {
  if (!ctx || !ctx->shard.live) return fail(ctx, PCB_INVALID, "no live shard");
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  return shard_evaluate(ctx, bad);
}

// ---- device-collective mode: the pieces of an iteration stay in device buffers that the ranks exchange with NCCL ----
pcb_status pcb_pagani_shard_deferred(pcb_ctx* ctx, int32_t on) {
  if (!ctx) return PCB_INVALID;
  ctx->shard.deferred = on != 0;
  return PCB_OK;
}

pcb_status pcb_pagani_shard_pack(pcb_ctx* ctx, int64_t head_active, int64_t head_retired, int32_t with_retired, int64_t width,
                                 int32_t world, pcb_pagani_shard_rows* out) {
  if (!ctx || !ctx->shard.live || !out) return fail(ctx, PCB_INVALID, "no live shard");
  if (head_active < 0 || head_active >= kTreeSpan || head_retired < 0 || head_retired >= kTreeSpan || width < 1 || world < 1)
    return fail(ctx, PCB_INVALID, "shard_pack: bad arguments");
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  auto& S = ctx->shard;
  const long long n_ret = with_retired ? S.n_ret : 0;
  if (S.n / kTreeSpan + 1 > width || n_ret / kTreeSpan + 1 > width) return fail(ctx, PCB_INVALID, "shard_pack: width %lld too small", (long long)width);
  const long long row_doubles = shard_row_doubles(width);
  PCB_CUDA_TRY(ctx, ctx->pg_row.ensure((size_t)row_doubles * sizeof(double)));
  if (world > 1) PCB_CUDA_TRY(ctx, ctx->pg_gathered.ensure((size_t)world * row_doubles * sizeof(double)));
  S.width = width;
  ShardPackArgs pa;
  pa.row = ctx->pg_row.as<double>();
  pa.width = width;
  pa.src[0] = ctx->est_i.as<double>(); pa.src[1] = ctx->est_e.as<double>();
  pa.src[2] = ctx->ret_i.as<double>(); pa.src[3] = ctx->ret_e.as<double>();
  pa.n[0] = pa.n[1] = S.n;
  pa.n[2] = pa.n[3] = n_ret;
  pa.head[0] = pa.head[1] = head_active;
  pa.head[2] = pa.head[3] = head_retired;
  pa.bad = ctx->scalars.as<unsigned long long>() + S_BAD;
  shard_pack_kernel<<<4, kTreeSpan, 0, ctx->stream>>>(pa);
  ctx->launches++;
  for (int s = 0; s < 4; ++s) {
    const long long n = pa.n[s], h = std::min<long long>(pa.head[s], n), nb = (n - h) / kTreeSpan;
    if (nb > 0) {
      double* blocks = pa.row + 4 + (long long)s * shard_section_doubles(width) + 4 + 2 * kTreeSpan;
      tree_level_kernel<<<(unsigned)nb, kTreeBlock, 0, ctx->stream>>>(pa.src[s] + h, nb * kTreeSpan, blocks);
      ctx->launches++;
    }
  }
  PCB_CUDA_TRY(ctx, cudaGetLastError());
  out->stream = (void*)ctx->stream;
  out->row = ctx->pg_row.as<double>();
  out->gathered = world > 1 ? ctx->pg_gathered.as<double>() : ctx->pg_row.as<double>();
  out->row_doubles = row_doubles;
  return PCB_OK;
}

pcb_status pcb_pagani_shard_global_sums(pcb_ctx* ctx, int32_t world, int64_t n_active_total, int64_t n_retired_total,
                                        double sums[4], int32_t* bad_rank) {
  if (!ctx || !ctx->shard.live || !sums || !bad_rank) return fail(ctx, PCB_INVALID, "no live shard");
  if (world < 1 || world > 1024 || n_active_total < 0 || n_retired_total < 0) return fail(ctx, PCB_INVALID, "shard_global_sums: bad arguments");
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  auto& S = ctx->shard;
  const long long row_doubles = shard_row_doubles(S.width);
  const double* gathered = world > 1 ? ctx->pg_gathered.as<double>() : ctx->pg_row.as<double>();
  const long long totals[4] = {n_active_total, n_active_total, n_retired_total, n_retired_total};
  const long long cap = std::max<long long>(1, (std::max(n_active_total, n_retired_total) + kTreeSpan - 1) / kTreeSpan);
  PCB_CUDA_TRY(ctx, ctx->pg_lists.ensure((size_t)4 * cap * sizeof(double)));
  ShardAssembleArgs aa;
  aa.gathered = gathered;
  aa.world = world;
  aa.row_doubles = row_doubles;
  aa.width = S.width;
  for (int s = 0; s < 4; ++s) aa.lists[s] = ctx->pg_lists.as<double>() + (size_t)s * cap;
  shard_assemble_kernel<<<dim3((unsigned)world, 4), kTreeSpan, 0, ctx->stream>>>(aa);
  ctx->launches++;
  PCB_CUDA_TRY(ctx, cudaGetLastError());
  double* sc = ctx->scalars.as<double>();
  const int slot[4] = {S_SUM_I, S_SUM_E, S_RET_I, S_RET_E};
  for (int s = 0; s < 4; ++s)
    PCB_TRY(tree_sum_dev(ctx, aa.lists[s], (totals[s] + kTreeSpan - 1) / kTreeSpan, sc + slot[s]));
  // the ranks' non-finite flags: header word 0 of every row
  unsigned long long* flags = (unsigned long long*)ctx->pinned + 64;
  PCB_CUDA_TRY(ctx, cudaMemcpy2DAsync(flags, sizeof(unsigned long long), gathered, (size_t)row_doubles * sizeof(double),
                                      sizeof(unsigned long long), (size_t)world, cudaMemcpyDeviceToHost, ctx->stream));
  PCB_TRY(read_scalars(ctx, 0, 8));
  const double* host = (const double*)ctx->pinned;
  for (int s = 0; s < 4; ++s) sums[s] = host[slot[s]];
  *bad_rank = -1;
  for (int r = 0; r < world; ++r)
    if (flags[r] != ~0ULL) { *bad_rank = r; break; }
  return PCB_OK;
}

pcb_status pcb_pagani_shard_nonfinite(pcb_ctx* ctx, pcb_nonfinite* bad) {
  if (!ctx || !ctx->shard.live || !bad) return fail(ctx, PCB_INVALID, "no live shard");
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  auto& S = ctx->shard;
  PCB_TRY(read_scalars(ctx, S_BAD, 1));
  const unsigned long long flat = ((unsigned long long*)ctx->pinned)[S_BAD];
  if (flat == ~0ULL) return fail(ctx, PCB_INVALID, "shard_nonfinite: this rank holds no non-finite evaluation");
  return fetch_nonfinite_pagani(ctx, &S.f, &S.rule, S.ld, ctx->lefts[S.cur].as<double>(), ctx->lengths[S.cur].as<double>(), flat, bad);
}

pcb_status pcb_pagani_shard_classify_dev(pcb_ctx* ctx, double budget, int32_t mode, double emax, int32_t world, double** row,
                                         double** gathered) {
  if (!ctx || !ctx->shard.live || !row || !gathered || world < 1) return fail(ctx, PCB_INVALID, "no live shard");
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  auto& S = ctx->shard;
  S.n_split = 0;
  S.classified = true;
  PCB_CUDA_TRY(ctx, ctx->pg_rowb.ensure((size_t)(2 + 2 * world) * sizeof(double)));
  double* sc = ctx->scalars.as<double>();
  unsigned long long* sc_u = ctx->scalars.as<unsigned long long>();
  PCB_CUDA_TRY(ctx, cudaMemsetAsync(sc + S_EMAX, 0, sizeof(double), ctx->stream));
  PCB_CUDA_TRY(ctx, cudaMemsetAsync(sc_u + S_NSPLIT, 0, sizeof(unsigned long long), ctx->stream));
  if (S.n > 0) {
    const long long nblk = (S.n + kScanBlock - 1) / kScanBlock;
    PCB_CUDA_TRY(ctx, ctx->flags.ensure((size_t)S.n));
    PCB_CUDA_TRY(ctx, ctx->counts.ensure((size_t)nblk * sizeof(unsigned int)));
    PCB_CUDA_TRY(ctx, ctx->offsets.ensure((size_t)nblk * sizeof(unsigned long long)));
    ClassifyArgs ca;
    ca.n = S.n; ca.ld = S.ld; ca.d = S.f.d; ca.mode = mode; ca.budget = budget; ca.emax = emax;
    ca.lengths = ctx->lengths[S.cur].as<double>();
    ca.errors = ctx->est_e.as<double>();
    ca.flags = ctx->flags.as<unsigned char>();
    ca.block_counts = ctx->counts.as<unsigned int>();
    classify_kernel<<<(unsigned)nblk, kScanBlock, 0, ctx->stream>>>(ca);
    scan_counts_kernel<<<1, 1024, 0, ctx->stream>>>(ctx->counts.as<unsigned int>(), (int)nblk, ctx->offsets.as<unsigned long long>(),
                                                    sc_u + S_NSPLIT);
    max_kernel<<<(unsigned)std::min<long long>((S.n + 255) / 256, 1024), 256, 0, ctx->stream>>>(ctx->est_e.as<double>(), S.n, sc + S_EMAX);
    ctx->launches += 3;
  }
  shard_pack_counts_kernel<<<1, 1, 0, ctx->stream>>>(sc_u + S_NSPLIT, sc + S_EMAX, ctx->pg_rowb.as<double>());
  ctx->launches++;
  PCB_CUDA_TRY(ctx, cudaGetLastError());
  *row = ctx->pg_rowb.as<double>();
  *gathered = world > 1 ? ctx->pg_rowb.as<double>() + 2 : ctx->pg_rowb.as<double>();
  return PCB_OK;
}

pcb_status pcb_pagani_shard_split_dev(pcb_ctx* ctx, int64_t n_split) {
  if (!ctx || !ctx->shard.live) return fail(ctx, PCB_INVALID, "no live shard");
  auto& S = ctx->shard;
  if (!S.classified) return fail(ctx, PCB_INVALID, "shard_split needs a preceding shard_classify");
  if (n_split < 0 || n_split > S.n) return fail(ctx, PCB_INVALID, "shard_split_dev: split count outside the local list");
  S.n_split = n_split;
  return pcb_pagani_shard_split(ctx);
}

pcb_status pcb_pagani_shard_list_dev(pcb_ctx* ctx, double** lefts, double** lengths, int64_t* n, int64_t* ld) {
  if (!ctx || !ctx->shard.live || !lefts || !lengths || !n || !ld) return fail(ctx, PCB_INVALID, "no live shard");
  auto& S = ctx->shard;
  *lefts = ctx->lefts[S.cur].as<double>();
  *lengths = ctx->lengths[S.cur].as<double>();
  *n = S.n;
  *ld = S.ld;
  return PCB_OK;
}

pcb_status pcb_pagani_shard_rebuild_dev(pcb_ctx* ctx, int64_t keep_begin, int64_t keep_end, int64_t n_front, const double* front_dev,
                                        int64_t n_back, const double* back_dev) {
  if (!ctx || !ctx->shard.live) return fail(ctx, PCB_INVALID, "no live shard");
  auto& S = ctx->shard;
  if (keep_begin < 0 || keep_end > S.n || keep_begin > keep_end || n_front < 0 || n_back < 0)
    return fail(ctx, PCB_INVALID, "shard_rebuild_dev: bad ranges");
  if ((n_front > 0 && !front_dev) || (n_back > 0 && !back_dev)) return fail(ctx, PCB_INVALID, "shard_rebuild_dev: NULL rows");
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const int d = S.f.d, nxt = S.cur ^ 1;
  const long long keep = keep_end - keep_begin, n_new = n_front + keep + n_back;
  if (n_front == 0 && n_back == 0 && keep_begin == 0 && keep_end == S.n) return PCB_OK;  // nothing moves
  const long long ld_new = round_up(std::max<long long>(n_new, 1), 32);
  PCB_CUDA_TRY(ctx, ctx->lefts[nxt].ensure((size_t)ld_new * d * sizeof(double)));
  PCB_CUDA_TRY(ctx, ctx->lengths[nxt].ensure((size_t)ld_new * d * sizeof(double)));
  auto place = [&](long long n, long long ld_src, long long src_off, const double* l_src, const double* h_src, long long dst_off) {
    if (n == 0) return;
    soa_copy_kernel<<<grid_for(n), 256, 0, ctx->stream>>>(d, n, ld_src, src_off, l_src, ld_new, dst_off, ctx->lefts[nxt].as<double>());
    soa_copy_kernel<<<grid_for(n), 256, 0, ctx->stream>>>(d, n, ld_src, src_off, h_src, ld_new, dst_off, ctx->lengths[nxt].as<double>());
    ctx->launches += 2;
  };
  // received blocks are [2][d][n]: lefts then lengths, structure of arrays with leading dimension n
  place(n_front, n_front, 0, front_dev, front_dev + (size_t)d * n_front, 0);
  place(keep, S.ld, keep_begin, ctx->lefts[S.cur].as<double>(), ctx->lengths[S.cur].as<double>(), n_front);
  place(n_back, n_back, 0, back_dev, back_dev + (size_t)d * n_back, n_front + keep);
  PCB_CUDA_TRY(ctx, cudaGetLastError());
  S.cur = nxt;
  S.n = n_new;
  S.ld = ld_new;
  return PCB_OK;
}

// quadrature.apply_rules for a single region: generic table, plain pair tree over all points.
__global__ void region_points_kernel(int d, int fe, const double* gen, const double* left, const double* length, double* pts) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= fe * d) return;
  int j = i % d;
  double off = (gen[i] + 1.0) / 2.0;
  pts[i] = left[j] + length[j] * off;
}
__global__ void rule_products_kernel(int fe, const double* w, const double* fx, double* prod) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < 5 * fe) prod[i] = w[i] * fx[i % fe];
}
__global__ void scale_by_volume_kernel(int d, const double* length, double* sums) {
  double vol = length[0];
  for (int j = 1; j < d; ++j) vol = vol * length[j];
  for (int k = 0; k < 5; ++k) sums[k] = vol * sums[k];
}

pcb_status pcb_apply_rules(pcb_ctx* ctx, const pcb_integrand* f, int32_t f_eval, const double* generators, const double* weights,
                           const double* left, const double* length, double values[5], double* stored_evals, pcb_nonfinite* bad) {
  if (!ctx) return PCB_INVALID;
  PCB_TRY(validate_integrand(ctx, f));
  if (f_eval < 1 || !generators || !weights || !left || !length || !values || !stored_evals)
    return fail(ctx, PCB_INVALID, "apply_rules: bad arguments");
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const int d = f->d, fe = f_eval;
  // layout in rows_a: gen[fe*d] | w[5*fe] | left[d] | length[d] | pts[fe*d] | fx[fe] | prod[5*fe]
  const size_t total = (size_t)fe * d * 2 + (size_t)fe * 11 + 2 * d;
  PCB_CUDA_TRY(ctx, ctx->mc_tmp.ensure(total * sizeof(double)));
  double* base = ctx->mc_tmp.as<double>();
  double *g_dev = base, *w_dev = g_dev + (size_t)fe * d, *l_dev = w_dev + 5 * (size_t)fe, *h_dev = l_dev + d;
  double *p_dev = h_dev + d, *fx_dev = p_dev + (size_t)fe * d, *prod_dev = fx_dev + fe;
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(g_dev, generators, (size_t)fe * d * 8, cudaMemcpyHostToDevice, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(w_dev, weights, (size_t)fe * 5 * 8, cudaMemcpyHostToDevice, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(l_dev, left, d * 8, cudaMemcpyHostToDevice, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(h_dev, length, d * 8, cudaMemcpyHostToDevice, ctx->stream));
  region_points_kernel<<<(fe * d + 255) / 256, 256, 0, ctx->stream>>>(d, fe, g_dev, l_dev, h_dev, p_dev);
  ctx->launches++;
  long long nn = fe;
  pcb_integrand fv = *f;
  const double* pts_c = p_dev;
  void* args[] = {&fv, &nn, &pts_c, &fx_dev};
  PCB_CUDA_TRY(ctx, cudaLaunchKernel(points_kernel(f->family, d), dim3((fe + 255) / 256), dim3(256), args, 0, ctx->stream));
  rule_products_kernel<<<(5 * fe + 255) / 256, 256, 0, ctx->stream>>>(fe, w_dev, fx_dev, prod_dev);
  ctx->launches += 2;
  double* sums = ctx->scalars.as<double>() + 16;
  for (int k = 0; k < 5; ++k) PCB_TRY(tree_sum_dev(ctx, prod_dev + (size_t)k * fe, fe, sums + k));
  scale_by_volume_kernel<<<1, 1, 0, ctx->stream>>>(d, h_dev, sums);
  ctx->launches++;
  std::vector<double> pts_host((size_t)fe * d);
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(stored_evals, fx_dev, (size_t)fe * 8, cudaMemcpyDeviceToHost, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(pts_host.data(), p_dev, (size_t)fe * d * 8, cudaMemcpyDeviceToHost, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(values, sums, 5 * 8, cudaMemcpyDeviceToHost, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < fe; ++i) {
    if (!std::isfinite(stored_evals[i])) {
      if (bad) {
        bad->region_index = -1;
        bad->point_index = i;
        bad->value = stored_evals[i];
        std::memset(bad->point, 0, sizeof bad->point);
        std::memcpy(bad->point, &pts_host[(size_t)i * d], sizeof(double) * d);
      }
      return fail(ctx, PCB_NONFINITE, "non-finite integrand value %g at rule point %d", stored_evals[i], i);
    }
  }
  return PCB_OK;
}

}  // extern "C"
