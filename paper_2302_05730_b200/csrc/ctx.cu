// Context, kernel dispatch tables, eval_points, RNG mirror and the FP64 peak probe.
#include "pcb_device.cuh"
#include "pcb_host.h"

#include <cmath>
#include <cstring>
#include <new>

namespace pcb {

#define PCB_DECL(F, _) \
  const void* eval_kernel_fam##F(int d); \
  const void* eval_wide_kernel_fam##F(int d); \
  const void* points_kernel_fam##F(int d); \
  const void* invoke_kernel_fam##F(int d); \
  const void* qmc_kernel_fam##F(int d); \
  const void* lanes_kernel_fam##F(int d, size_t* smem, int* threads); \
  const void* vsample_kernel_fam##F(int d, int rng);
PCB_DECL(0, ) PCB_DECL(1, ) PCB_DECL(2, ) PCB_DECL(3, ) PCB_DECL(4, ) PCB_DECL(5, ) PCB_DECL(6, ) PCB_DECL(7, )
#undef PCB_DECL

static const kernel_getter kEval[PCB_N_FAMILIES] = {eval_kernel_fam0, eval_kernel_fam1, eval_kernel_fam2, eval_kernel_fam3,
                                                    eval_kernel_fam4, eval_kernel_fam5, eval_kernel_fam6, eval_kernel_fam7};
static const kernel_getter kEvalWide[PCB_N_FAMILIES] = {eval_wide_kernel_fam0, eval_wide_kernel_fam1, eval_wide_kernel_fam2, eval_wide_kernel_fam3,
                                                        eval_wide_kernel_fam4, eval_wide_kernel_fam5, eval_wide_kernel_fam6, eval_wide_kernel_fam7};
static const kernel_getter kPoints[PCB_N_FAMILIES] = {points_kernel_fam0, points_kernel_fam1, points_kernel_fam2, points_kernel_fam3,
                                                      points_kernel_fam4, points_kernel_fam5, points_kernel_fam6, points_kernel_fam7};
typedef const void* (*sample_getter)(int d, int rng);
static const sample_getter kSample[PCB_N_FAMILIES] = {vsample_kernel_fam0, vsample_kernel_fam1, vsample_kernel_fam2, vsample_kernel_fam3,
                                                      vsample_kernel_fam4, vsample_kernel_fam5, vsample_kernel_fam6, vsample_kernel_fam7};

static const kernel_getter kInvoke[PCB_N_FAMILIES] = {invoke_kernel_fam0, invoke_kernel_fam1, invoke_kernel_fam2, invoke_kernel_fam3,
                                                      invoke_kernel_fam4, invoke_kernel_fam5, invoke_kernel_fam6, invoke_kernel_fam7};
static const kernel_getter kQmc[PCB_N_FAMILIES] = {qmc_kernel_fam0, qmc_kernel_fam1, qmc_kernel_fam2, qmc_kernel_fam3,
                                                   qmc_kernel_fam4, qmc_kernel_fam5, qmc_kernel_fam6, qmc_kernel_fam7};
typedef const void* (*lanes_getter)(int d, size_t* smem, int* threads);
static const lanes_getter kLanes[PCB_N_FAMILIES] = {lanes_kernel_fam0, lanes_kernel_fam1, lanes_kernel_fam2, lanes_kernel_fam3,
                                                    lanes_kernel_fam4, lanes_kernel_fam5, lanes_kernel_fam6, lanes_kernel_fam7};
// run-time families (pcb_user_family_load): kernels fetched from a loaded cubin, bound to one dimension
struct UserFamily {
  int d = 0;
  cudaLibrary_t lib = nullptr;
  const void* fn[8] = {};   // order of pcb_user_kernel_names
};
static UserFamily g_user[PCB_MAX_USER_FAMILIES];
// bumped by every load / unload: a context drops its per-kernel caches (granted shared memory, preloaded code) when it
// sees a new value -- a reloaded slot may hand out a kernel handle with the address of one that was unloaded
static unsigned long long g_user_generation = 0;
static const UserFamily* user_family(int family, int d) {
  const int slot = family - PCB_USER_FAMILY_BASE;
  if (slot < 0 || slot >= PCB_MAX_USER_FAMILIES || !g_user[slot].lib || g_user[slot].d != d) return nullptr;
  return &g_user[slot];
}
size_t generic_lanes_smem(int d);   // pagani_inst.cu: GenericLaneLayout<d>::smem_bytes()

const void* eval_lanes_kernel(int family, int d, size_t* smem, int* threads) {
  if (family >= PCB_N_FAMILIES) {
    const UserFamily* u = user_family(family, d);
    *smem = u ? generic_lanes_smem(d) : 0;
    *threads = 32;
    return u ? u->fn[2] : nullptr;
  }
  return kLanes[family](d, smem, threads);
}
const void* eval_kernel(int family, int d) {
  if (family >= PCB_N_FAMILIES) { const UserFamily* u = user_family(family, d); return u ? u->fn[0] : nullptr; }
  return kEval[family](d);
}
const void* eval_wide_kernel(int family, int d) {
  if (family >= PCB_N_FAMILIES) { const UserFamily* u = user_family(family, d); return u ? u->fn[1] : nullptr; }
  return kEvalWide[family](d);
}
const void* points_kernel(int family, int d) {
  if (family >= PCB_N_FAMILIES) { const UserFamily* u = user_family(family, d); return u ? u->fn[3] : nullptr; }
  return kPoints[family](d);
}
const void* vsample_kernel_ptr(int family, int d, int rng) {
  if (family >= PCB_N_FAMILIES) {
    const UserFamily* u = user_family(family, d);
    return u ? u->fn[rng == PCB_RNG_REFERENCE_HASH ? 6 : 7] : nullptr;
  }
  return kSample[family](d, rng);
}
static const void* invoke_kernel_ptr(int family, int d) {
  if (family >= PCB_N_FAMILIES) { const UserFamily* u = user_family(family, d); return u ? u->fn[4] : nullptr; }
  return kInvoke[family](d);
}
static const void* qmc_kernel_ptr(int family, int d) {
  if (family >= PCB_N_FAMILIES) { const UserFamily* u = user_family(family, d); return u ? u->fn[5] : nullptr; }
  return kQmc[family](d);
}

pcb_status validate_integrand(pcb_ctx* ctx, const pcb_integrand* f) {
  if (!f) return fail(ctx, PCB_INVALID, "integrand is NULL");
  if (f->d < 1 || f->d > PCB_MAX_DIM) return fail(ctx, PCB_INVALID, "dimension %d outside [1, %d]", f->d, PCB_MAX_DIM);
  if (f->family >= PCB_USER_FAMILY_BASE && f->family < PCB_USER_FAMILY_BASE + PCB_MAX_USER_FAMILIES) {
    if (ctx && ctx->user_generation != g_user_generation) {
      ctx->smem_attr.clear();
      ctx->preloaded.clear();
      ctx->user_generation = g_user_generation;
    }
    if (!user_family(f->family, f->d))
      return fail(ctx, PCB_INVALID, "run-time family %d is not loaded for dimension %d (pcb_user_family_load)", f->family, f->d);
    return PCB_OK;
  }
  if (f->family < 0 || f->family >= PCB_N_FAMILIES) return fail(ctx, PCB_INVALID, "unknown integrand family %d", f->family);
  return PCB_OK;
}

__global__ void fp64_peak_kernel(double* sink, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
    x0 = __fma_rn(x0, a, b); x1 = __fma_rn(x1, a, b); x2 = __fma_rn(x2, a, b); x3 = __fma_rn(x3, a, b);
    x4 = __fma_rn(x4, a, b); x5 = __fma_rn(x5, a, b); x6 = __fma_rn(x6, a, b); x7 = __fma_rn(x7, a, b);
  }
  double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
  if (s == 12345.678) sink[0] = s;
}

__global__ void uniforms_kernel(unsigned long long seed, int kind, long long n, const unsigned long long* streams,
                                const unsigned long long* counters, double* out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = kind == PCB_RNG_PHILOX ? philox_uniform(seed, streams[i], counters[i])
                                    : hash_uniform(stream_key(seed, streams[i]), counters[i]);
}

}  // namespace pcb

using namespace pcb;

extern "C" {

pcb_status pcb_user_family_load(pcb_ctx* ctx, int32_t family, int32_t d, const void* cubin, uint64_t bytes,
                                const pcb_user_kernel_names* names) {
  const int slot = family - PCB_USER_FAMILY_BASE;
  if (slot < 0 || slot >= PCB_MAX_USER_FAMILIES)
    return fail(ctx, PCB_INVALID, "run-time family id %d outside [%d, %d)", family, PCB_USER_FAMILY_BASE, PCB_USER_FAMILY_BASE + PCB_MAX_USER_FAMILIES);
  if (d < 1 || d > PCB_MAX_DIM || !cubin || bytes == 0 || !names) return fail(ctx, PCB_INVALID, "user_family_load: bad arguments");
  if (ctx) PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  cudaLibrary_t lib = nullptr;
  cudaError_t e = cudaLibraryLoadData(&lib, cubin, nullptr, nullptr, 0, nullptr, nullptr, 0);
  if (e != cudaSuccess) return fail(ctx, PCB_CUDA, "user_family_load: the image does not load (%s)", cudaGetErrorString(e));
  const char* wanted[8] = {names->eval, names->eval_wide, names->lanes, names->points,
                           names->invoke, names->qmc, names->sample_hash, names->sample_generic};
  UserFamily u;
  u.d = d;
  u.lib = lib;
  for (int k = 0; k < 8; ++k) {
    cudaKernel_t kern = nullptr;
    e = wanted[k] ? cudaLibraryGetKernel(&kern, lib, wanted[k]) : cudaErrorInvalidValue;
    if (e != cudaSuccess) {
      cudaLibraryUnload(lib);
      (void)cudaGetLastError();
      return fail(ctx, PCB_INVALID, "user_family_load: kernel %s not found in the image (%s)", wanted[k] ? wanted[k] : "(null)", cudaGetErrorString(e));
    }
    u.fn[k] = (const void*)kern;
  }
  if (g_user[slot].lib) cudaLibraryUnload(g_user[slot].lib);
  g_user[slot] = u;
  ++g_user_generation;
  return PCB_OK;
}

pcb_status pcb_user_family_unload(pcb_ctx* ctx, int32_t family) {
  const int slot = family - PCB_USER_FAMILY_BASE;
  if (slot < 0 || slot >= PCB_MAX_USER_FAMILIES) return fail(ctx, PCB_INVALID, "run-time family id %d out of range", family);
  if (g_user[slot].lib) cudaLibraryUnload(g_user[slot].lib);
  g_user[slot] = UserFamily{};
  ++g_user_generation;
  return PCB_OK;
}


pcb_status pcb_ctx_create(int device_ordinal, pcb_ctx** out) {
  if (!out) return PCB_INVALID;
  *out = nullptr;
  pcb_ctx* ctx = new (std::nothrow) pcb_ctx();
  if (!ctx) return PCB_CUDA;
  *out = ctx;  // returned even on failure so the caller can read the error text
  ctx->device = device_ordinal;
  PCB_CUDA_TRY(ctx, cudaSetDevice(device_ordinal));
  cudaDeviceProp prop;
  PCB_CUDA_TRY(ctx, cudaGetDeviceProperties(&prop, device_ordinal));
  if (prop.major < 10)
    return fail(ctx, PCB_CUDA, "device %d (%s, sm_%d%d) is not a Blackwell sm_100 part; this library has no other code path",
                device_ordinal, prop.name, prop.major, prop.minor);
  ctx->sm_count = prop.multiProcessorCount;
  ctx->smem_optin = prop.sharedMemPerBlockOptin;
  ctx->smem_per_sm = prop.sharedMemPerMultiprocessor;
  ctx->total_mem = prop.totalGlobalMem;
  int khz = 0;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, device_ordinal);
  ctx->clock_khz = khz;
  std::strncpy(ctx->name, prop.name, sizeof(ctx->name) - 1);
  PCB_CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  if (!Vmm::get().ok) return fail(ctx, PCB_CUDA, "the driver does not offer the virtual memory management API the scratch buffers are built on");
  PCB_CUDA_TRY(ctx, cudaMallocHost(&ctx->pinned, 1 << 16));
  PCB_CUDA_TRY(ctx, ctx->scalars.ensure(64 * sizeof(double)));
  return PCB_OK;
}

void pcb_ctx_destroy(pcb_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) {
    cudaStreamSynchronize(ctx->stream);
    ctx->release_buffers();
    cudaStreamDestroy(ctx->stream);
    ctx->stream = nullptr;
  }
  for (auto h : ctx->chunk_cache.free_chunks) Vmm::get().release(h);
  ctx->chunk_cache.free_chunks.clear();
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx->mc_records) cudaFreeHost(ctx->mc_records);
  if (ctx->pg_record) cudaFreeHost(ctx->pg_record);
  if (ctx->mc_out_pinned) cudaFreeHost(ctx->mc_out_pinned);
  for (auto ev : ctx->mc_events) cudaEventDestroy(ev);
  for (int k = 0; k < 3; ++k)
    for (auto& sp : ctx->spans[k]) ctx->span_pool.push_back(sp);
  for (auto& sp : ctx->span_pool) {
    cudaEventDestroy(sp.a);
    cudaEventDestroy(sp.b);
  }
  delete ctx;
}

pcb_status pcb_ctx_reserve(pcb_ctx* ctx, uint64_t bytes, uint64_t* reserved_out) {
  if (!ctx) return PCB_INVALID;
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const Vmm& v = Vmm::get();
  auto& cache = ctx->chunk_cache;
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = ctx->device;
  // physical chunks created now, mapped into whichever buffer grows later (DevBuf::ensure)
  while ((uint64_t)cache.free_chunks.size() * ChunkCache::kChunk < bytes) {
    CUmemGenericAllocationHandle h;
    if (v.create(&h, ChunkCache::kChunk, &prop, 0) != CUDA_SUCCESS)
      return fail(ctx, PCB_CUDA, "pcb_ctx_reserve: the device has no room for %llu bytes", (unsigned long long)bytes);
    cache.free_chunks.push_back(h);
  }
  if (reserved_out) *reserved_out = (uint64_t)cache.free_chunks.size() * ChunkCache::kChunk;
  return PCB_OK;
}

void pcb_ctx_abort(pcb_ctx* ctx) {
  if (ctx) ctx->abort_requested = 1;
}

const char* pcb_last_error(const pcb_ctx* ctx) { return ctx ? ctx->err.c_str() : "context is NULL"; }

pcb_status pcb_device_info(pcb_ctx* ctx, char* name, int name_len, int32_t* sm_count, int32_t* clock_khz) {
  if (!ctx) return PCB_INVALID;
  if (name && name_len > 0) {
    std::strncpy(name, ctx->name, name_len - 1);
    name[name_len - 1] = 0;
  }
  if (sm_count) *sm_count = ctx->sm_count;
  if (clock_khz) *clock_khz = ctx->clock_khz;
  return PCB_OK;
}

int64_t pcb_launch_count(const pcb_ctx* ctx) { return ctx ? ctx->launches : 0; }

pcb_status pcb_measure_fp64_peak(pcb_ctx* ctx, double* tflops) {
  if (!ctx || !tflops) return PCB_INVALID;
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const int iters = 1 << 15, threads = 512, blocks = ctx->sm_count * 4;
  cudaEvent_t e0, e1;
  PCB_CUDA_TRY(ctx, cudaEventCreate(&e0));
  PCB_CUDA_TRY(ctx, cudaEventCreate(&e1));
  double best = 0.0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0, ctx->stream);
    fp64_peak_kernel<<<blocks, threads, 0, ctx->stream>>>(ctx->scalars.as<double>() + 32, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1, ctx->stream);
    PCB_CUDA_TRY(ctx, cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    double tf = 2.0 * 8.0 * iters * (double)threads * blocks / (ms * 1e-3) / 1e12;
    if (rep > 0 && tf > best) best = tf;
    ctx->launches++;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *tflops = best;
  return PCB_OK;
}

pcb_status pcb_profile_begin(pcb_ctx* ctx) {
  if (!ctx) return PCB_INVALID;
  for (int k = 0; k < 3; ++k) {
    for (auto& sp : ctx->spans[k]) ctx->span_pool.push_back(sp);
    ctx->spans[k].clear();
  }
  ctx->profiling = true;
  return PCB_OK;
}

pcb_status pcb_profile_end(pcb_ctx* ctx, int32_t kind, double* kernel_ms, int64_t* launches, double* units) {
  if (!ctx || kind < 0 || kind > 2) return PCB_INVALID;
  ctx->profiling = false;
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  PCB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  double total = 0, total_units = 0;
  for (auto& sp : ctx->spans[kind]) {
    float ms = 0;
    PCB_CUDA_TRY(ctx, cudaEventElapsedTime(&ms, sp.a, sp.b));
    total += ms;
    total_units += sp.units;
  }
  if (kernel_ms) *kernel_ms = total;
  if (launches) *launches = (int64_t)ctx->spans[kind].size();
  if (units) *units = total_units;
  return PCB_OK;
}

pcb_status pcb_eval_points(pcb_ctx* ctx, const pcb_integrand* f, int64_t n, const double* points, double* values) {
  if (!ctx) return PCB_INVALID;
  PCB_TRY(validate_integrand(ctx, f));
  if (n < 0 || (n > 0 && (!points || !values))) return fail(ctx, PCB_INVALID, "eval_points: bad buffers");
  if (n == 0) return PCB_OK;
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  PCB_CUDA_TRY(ctx, ctx->rows_a.ensure((size_t)n * f->d * sizeof(double)));
  PCB_CUDA_TRY(ctx, ctx->rows_b.ensure((size_t)n * sizeof(double)));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->rows_a.p, points, (size_t)n * f->d * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  const double* pts = ctx->rows_a.as<double>();
  double* out = ctx->rows_b.as<double>();
  long long nn = n;
  pcb_integrand fv = *f;
  void* args[] = {&fv, &nn, &pts, &out};
  int blocks = (int)std::min<long long>((n + 255) / 256, (long long)ctx->sm_count * 16);
  PCB_CUDA_TRY(ctx, cudaLaunchKernel(points_kernel(f->family, f->d), dim3(blocks), dim3(256), args, 0, ctx->stream));
  ctx->launches++;
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(values, out, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return PCB_OK;
}

pcb_status pcb_bench_invoke(pcb_ctx* ctx, const pcb_integrand* f, int64_t n, const double* points, int32_t blocks,
                            int32_t threads, int32_t repetitions, double* ms_out, double* accumulator) {
  if (!ctx) return PCB_INVALID;
  PCB_TRY(validate_integrand(ctx, f));
  if (n < 1 || !points || blocks < 1 || threads < 1 || threads > 1024 || repetitions < 1 || !ms_out || !accumulator)
    return fail(ctx, PCB_INVALID, "bench_invoke: bad arguments");
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  PCB_CUDA_TRY(ctx, ctx->rows_a.ensure((size_t)n * f->d * sizeof(double)));
  PCB_CUDA_TRY(ctx, ctx->rows_b.ensure((size_t)blocks * threads * sizeof(double)));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->rows_a.p, points, (size_t)n * f->d * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  const double* pts = ctx->rows_a.as<double>();
  double* out = ctx->rows_b.as<double>();
  long long nn = n;
  pcb_integrand fv = *f;
  void* args[] = {&fv, &nn, &pts, &out};
  cudaEvent_t e0, e1;
  PCB_CUDA_TRY(ctx, cudaEventCreate(&e0));
  PCB_CUDA_TRY(ctx, cudaEventCreate(&e1));
  pcb_status st = PCB_OK;
  for (int r = 0; r < repetitions && st == PCB_OK; ++r) {
    cudaEventRecord(e0, ctx->stream);
    cudaError_t err = cudaLaunchKernel(invoke_kernel_ptr(f->family, f->d), dim3(blocks), dim3(threads), args, 0, ctx->stream);
    cudaEventRecord(e1, ctx->stream);
    ctx->launches++;
    if (err == cudaSuccess) err = cudaEventSynchronize(e1);
    if (err != cudaSuccess) { st = fail(ctx, PCB_CUDA, "bench_invoke: %s", cudaGetErrorString(err)); break; }
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms_out[r] = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (st != PCB_OK) return st;
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(accumulator, out, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return PCB_OK;
}

// Sobol' direction numbers of the first 12 dimensions (Joe & Kuo, new-joe-kuo-6.21201: degree s, coefficient word a,
// initial m_i), 30 bits -- the table behind scipy.stats.qmc.Sobol, which the reference's oracle uses
// (integrands.py:247); tests/test_gpu_qmc.py checks the generated points against scipy bit for bit.
static void sobol_directions(int d, unsigned* v /* [d][30] */) {
  static const int kS[12] = {0, 1, 2, 3, 3, 4, 4, 5, 5, 5, 5, 5};
  static const int kA[12] = {0, 0, 1, 1, 2, 1, 4, 2, 4, 7, 11, 13};
  static const int kM[12][5] = {{0}, {1}, {1, 3}, {1, 3, 1}, {1, 1, 1}, {1, 1, 3, 3}, {1, 3, 5, 13}, {1, 1, 5, 5, 17},
                                {1, 1, 5, 5, 5}, {1, 1, 7, 11, 19}, {1, 1, 5, 1, 1}, {1, 1, 1, 3, 11}};
  const int bits = 30;
  for (int j = 0; j < d; ++j) {
    unsigned long long m[30];
    if (j == 0) {
      for (int i = 0; i < bits; ++i) m[i] = 1;
    } else {
      const int s = kS[j], a = kA[j];
      for (int i = 0; i < s; ++i) m[i] = (unsigned long long)kM[j][i];
      for (int i = s; i < bits; ++i) {
        unsigned long long val = m[i - s] ^ (m[i - s] << s);
        for (int k = 1; k < s; ++k) val ^= (unsigned long long)((a >> (s - 1 - k)) & 1) * (m[i - k] << k);
        m[i] = val;
      }
    }
    for (int i = 0; i < bits; ++i) v[j * bits + i] = (unsigned)(m[i] << (bits - 1 - i));
  }
}

pcb_status pcb_qmc_shift_sums(pcb_ctx* ctx, const pcb_integrand* f, int32_t log2_points, int32_t n_shifts, const double* shifts,
                              double* sums) {
  if (!ctx) return PCB_INVALID;
  PCB_TRY(validate_integrand(ctx, f));
  if (log2_points < 10 || log2_points > 30 || n_shifts < 1 || n_shifts > 4096 || !shifts || !sums)
    return fail(ctx, PCB_INVALID, "qmc_shift_sums: 2^10 <= points <= 2^30, 1 <= shifts <= 4096");
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const int d = f->d;
  // 2^17 threads at most (512 CTAs of 256), at least 8 points per thread
  int log2_threads = log2_points - 3;
  if (log2_threads > 17) log2_threads = 17;
  const unsigned blocks = 1u << (log2_threads - 8);
  unsigned dirs[12 * 30];
  sobol_directions(d, dirs);
  const size_t dir_bytes = (size_t)d * 30 * sizeof(unsigned), shift_bytes = (size_t)n_shifts * d * sizeof(double);
  PCB_CUDA_TRY(ctx, ctx->mc_tmp.ensure(dir_bytes + 64 + shift_bytes + ((size_t)n_shifts * blocks + n_shifts) * sizeof(double)));
  unsigned* dirs_dev = ctx->mc_tmp.as<unsigned>();
  double* shifts_dev = reinterpret_cast<double*>(ctx->mc_tmp.as<char>() + ((dir_bytes + 63) & ~(size_t)63));
  double* partial = shifts_dev + (size_t)n_shifts * d;
  double* sums_dev = partial + (size_t)n_shifts * blocks;
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(dirs_dev, dirs, dir_bytes, cudaMemcpyHostToDevice, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(shifts_dev, shifts, shift_bytes, cudaMemcpyHostToDevice, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));   // `dirs` is a stack buffer
  pcb_integrand fv = *f;
  int lg = log2_points;
  const unsigned* dirs_c = dirs_dev;
  const double* shifts_c = shifts_dev;
  void* args[] = {&fv, &lg, &dirs_c, &shifts_c, &partial};
  PCB_CUDA_TRY(ctx, cudaLaunchKernel(qmc_kernel_ptr(f->family, d), dim3(blocks, (unsigned)n_shifts), dim3(256), args, 0, ctx->stream));
  ctx->launches++;
  for (int s = 0; s < n_shifts; ++s) PCB_TRY(tree_sum_dev(ctx, partial + (size_t)s * blocks, blocks, sums_dev + s));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(sums, sums_dev, (size_t)n_shifts * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return PCB_OK;
}

pcb_status pcb_uniforms(pcb_ctx* ctx, uint64_t seed, int32_t rng_kind, int64_t n, const uint64_t* streams,
                        const uint64_t* counters, double* out) {
  if (!ctx) return PCB_INVALID;
  if (n < 0 || (n > 0 && (!streams || !counters || !out))) return fail(ctx, PCB_INVALID, "uniforms: bad buffers");
  if (rng_kind != PCB_RNG_REFERENCE_HASH && rng_kind != PCB_RNG_PHILOX) return fail(ctx, PCB_INVALID, "uniforms: bad rng kind");
  if (n == 0) return PCB_OK;
  PCB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  PCB_CUDA_TRY(ctx, ctx->rows_a.ensure((size_t)n * 16));
  PCB_CUDA_TRY(ctx, ctx->rows_b.ensure((size_t)n * 8));
  unsigned long long* s = ctx->rows_a.as<unsigned long long>();
  unsigned long long* c = s + n;
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(s, streams, (size_t)n * 8, cudaMemcpyHostToDevice, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(c, counters, (size_t)n * 8, cudaMemcpyHostToDevice, ctx->stream));
  int blocks = (int)std::min<long long>((n + 255) / 256, (long long)ctx->sm_count * 16);
  uniforms_kernel<<<blocks, 256, 0, ctx->stream>>>(seed, rng_kind, n, s, c, ctx->rows_b.as<double>());
  ctx->launches++;
  PCB_CUDA_TRY(ctx, cudaGetLastError());
  PCB_CUDA_TRY(ctx, cudaMemcpyAsync(out, ctx->rows_b.p, (size_t)n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  PCB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return PCB_OK;
}

}  // extern "C"
