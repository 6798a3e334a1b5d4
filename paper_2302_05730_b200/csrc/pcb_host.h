// Host-side runtime shared by the C-ABI translation units: context, device buffers, launch helpers.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <array>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "../../include/parcube_b200.h"

namespace pcb {

// ------------------------------------------------------------------------------------------------------------
// Device scratch memory of a context: growable buffers on CUDA's virtual memory management API.
// A DevBuf reserves a (large) virtual address range once and backs it with physical chunks on demand: growing a
// buffer maps more chunks BEHIND the ones in use -- the base pointer never changes, nothing is freed or copied,
// nothing depends on an allocator's free-list state -- and a context never hands memory back before it is
// destroyed.  The region lists of a refinement double every iteration; with this layout the growth of a list to
// 3.4 GB costs ~50 map calls in total, whatever ran before.
// (Round 1 grew buffers with cudaFree + cudaMalloc: a device-wide synchronisation and a driver allocation per step,
// up to 17x on a refine() that outgrew its buffers.  The stream-ordered pool tried first in round 2 removed that but
// showed rare 0.2-1.5 s stalls when a request of several GB met a fragmented pool: profiles/r2_cold_call.txt history.)
// The driver entry points are taken through cudaGetDriverEntryPoint: the library does not link libcuda, so it still
// loads on a machine without a driver (the CPU test-suite checks the exported symbols there).
// ------------------------------------------------------------------------------------------------------------
struct Vmm {
  CUresult (*reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*address_free)(CUdeviceptr, size_t) = nullptr;
  CUresult (*create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
  CUresult (*release)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*unmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*set_access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*granularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
  bool ok = false;
  static const Vmm& get() {
    static const Vmm v = [] {
      Vmm x;
      auto load = [](const char* name, void** fn) {
        cudaDriverEntryPointQueryResult q;
        return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess && *fn;
      };
      x.ok = load("cuMemAddressReserve", (void**)&x.reserve) && load("cuMemAddressFree", (void**)&x.address_free) &&
             load("cuMemCreate", (void**)&x.create) && load("cuMemRelease", (void**)&x.release) && load("cuMemMap", (void**)&x.map) &&
             load("cuMemUnmap", (void**)&x.unmap) && load("cuMemSetAccess", (void**)&x.set_access) &&
             load("cuMemGetAllocationGranularity", (void**)&x.granularity);
      (void)cudaGetLastError();
      return x;
    }();
    return v;
  }
};

// physical chunks created ahead of time (pcb_ctx_reserve) and handed to the buffers that grow
struct ChunkCache {
  static constexpr size_t kChunk = (size_t)64 << 20;   // measured: 256-MiB chunks map several times slower per byte (page-table setup), smaller ones cost ~0.3 ms each
  std::vector<CUmemGenericAllocationHandle> free_chunks;   // each kChunk bytes
};

struct DevBuf {
  void* p = nullptr;      // base of the reserved range; stable once set
  size_t cap = 0;         // bytes backed by physical memory
  const int* device = nullptr;        // the owning context's device ordinal
  ChunkCache* cache = nullptr;        // the owning context's pre-created chunks
  size_t va = 0;
  // Upper bound of what this buffer can ever be asked for in the current run (0: unknown).  Once a request passes
  // kHintFrom the buffer grows straight to the bound: a list that has reached half a gigabyte is on its way to the region
  // cap, and ONE large mapping step per buffer and process is cheaper -- and less erratic -- than one per iteration
  // (steps of gigabytes occasionally stall for 50-150 ms, profiles/r2_sweep_config5.md).
  size_t hint_max = 0;
  static constexpr size_t kHintFrom = (size_t)512 << 20;
  struct Mapped { CUmemGenericAllocationHandle h; size_t bytes; };
  std::vector<Mapped> chunks;
  static constexpr size_t kVirtual = (size_t)1 << 37;   // 128 GiB of address space per buffer
  ~DevBuf() { release(); }
  void release() {
    const Vmm& v = Vmm::get();
    if (p && v.ok) {
      if (cap) v.unmap((CUdeviceptr)p, cap);
      for (auto& c : chunks) v.release(c.h);
      v.address_free((CUdeviceptr)p, va);
    }
    chunks.clear();
    p = nullptr;
    cap = 0;
    va = 0;
  }
  // grow-only; the base pointer and the contents are preserved
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    static const bool debug = std::getenv("PCB_DEBUG_MEM") != nullptr;
    if (!debug) return grow(bytes);
    const auto t0 = std::chrono::steady_clock::now();
    const size_t before = cap, cached = cache ? cache->free_chunks.size() : 0;
    const cudaError_t e = grow(bytes);
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    std::fprintf(stderr, "DevBuf %p: %zu -> %zu MiB (asked %zu MiB, %zu cached chunks used) in %.3f ms\n", p, before >> 20, cap >> 20,
                 bytes >> 20, cached - (cache ? cache->free_chunks.size() : 0), ms);
    return e;
  }
  cudaError_t grow(size_t bytes) {
    const Vmm& v = Vmm::get();
    if (!v.ok || !device) return cudaErrorNotSupported;
    CUmemAllocationProp prop = {};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = *device;
    size_t gran = (size_t)2 << 20;
    if (v.granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM) != CUDA_SUCCESS || gran == 0) gran = (size_t)2 << 20;
    if (!p) {
      CUdeviceptr base = 0;
      if (v.reserve(&base, kVirtual, 0, 0, 0) != CUDA_SUCCESS) return cudaErrorMemoryAllocation;
      p = (void*)base;
      va = kVirtual;
    }
    if (bytes > va) return cudaErrorMemoryAllocation;
    CUmemAccessDesc acc = {};
    acc.location = prop.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    auto map_one = [&](CUmemGenericAllocationHandle h, size_t n) -> bool {
      if (v.map((CUdeviceptr)p + cap, n, 0, h, 0) != CUDA_SUCCESS) return false;
      if (v.set_access((CUdeviceptr)p + cap, n, &acc, 1) != CUDA_SUCCESS) { v.unmap((CUdeviceptr)p + cap, n); return false; }
      chunks.push_back({h, n});
      cap += n;
      return true;
    };
    // geometric growth (a list that doubles per iteration maps ~2 new ranges per step); big steps take the
    // context's pre-created 64-MiB chunks first
    // A mapping step costs ~0.25 ms whatever its size (cuMemCreate + cuMemMap + cuMemSetAccess, measured), and a
    // refinement that outgrows ten buffers by a few MiB per iteration paid more for them than for its kernels:
    // the first step is at least 8 MiB and a step at least doubles the buffer, up to 64 MiB of slack.  No more than
    // that: region lists double per iteration anyway, so a large buffer needs one step per iteration whatever the
    // policy, and creating physical memory is NOT flat in size for gigabytes (mapping 2x ahead made the first run of a
    // process to 6e7 regions 200 ms slower).
    size_t want = bytes - cap;
    if (cap == 0 && want < ((size_t)8 << 20)) want = (size_t)8 << 20;
    const size_t geometric = cap < ((size_t)64 << 20) ? cap : (size_t)64 << 20;
    if (want < geometric) want = geometric;
    if (hint_max > bytes && bytes >= kHintFrom && want < hint_max - cap) want = hint_max - cap;
    want = (want + gran - 1) / gran * gran;
    while (cache && want >= ChunkCache::kChunk && !cache->free_chunks.empty() && cap < bytes + ChunkCache::kChunk) {
      CUmemGenericAllocationHandle h = cache->free_chunks.back();
      if (!map_one(h, ChunkCache::kChunk)) break;
      cache->free_chunks.pop_back();
      want = want > ChunkCache::kChunk ? want - ChunkCache::kChunk : 0;
      if (cap >= bytes && want < ChunkCache::kChunk) break;
    }
    while (cap < bytes || want >= gran) {
      size_t n = want >= gran ? want : (bytes - cap + gran - 1) / gran * gran;
      CUmemGenericAllocationHandle h;
      if (v.create(&h, n, &prop, 0) != CUDA_SUCCESS) {
        if (cap >= bytes) break;                        // the geometric extra is optional
        n = (bytes - cap + gran - 1) / gran * gran;     // exact need only
        if (v.create(&h, n, &prop, 0) != CUDA_SUCCESS) return cudaErrorMemoryAllocation;
      }
      if (!map_one(h, n)) { v.release(h); return cudaErrorMemoryAllocation; }
      want = 0;
    }
    return cap >= bytes ? cudaSuccess : cudaErrorMemoryAllocation;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

}  // namespace pcb

struct pcb_ctx {
  int device = 0;
  int sm_count = 0;
  int clock_khz = 0;
  size_t smem_optin = 0;
  size_t smem_per_sm = 0;
  size_t total_mem = 0;
  std::map<const void*, size_t> smem_attr;  // dynamic shared memory already granted per kernel
  std::set<const void*> preloaded;          // kernels whose code is known to be loaded (lazy module loading)
  unsigned long long user_generation = 0;   // run-time family registry state these two caches were filled under (ctx.cu)
  cudaStream_t stream = nullptr;
  std::string err;
  volatile int abort_requested = 0;   // pcb_ctx_abort(), polled by the drivers after every progress callback
  long long launches = 0;
  char name[256] = {0};
  void* pinned = nullptr;  // 64 KiB staging for small device->host reads
  void* pg_record = nullptr;          // pinned record of the short-list PAGANI iteration kernel
  unsigned long long pg_seq = 0;
  // scratch device buffers, grown on demand and reused across calls
  pcb::DevBuf lefts[2], lengths[2], est_i, est_e, est_k, flags, counts, offsets, ret_i, ret_e, tree[2], scalars;
  pcb::DevBuf rows_a, rows_b, k64;
  // PAGANI shard state (pcb_pagani_shard_*)
  struct Shard {
    bool live = false;
    pcb_integrand f;
    pcb_rule rule;
    pcb_pagani_config cfg;
    int cur = 0;
    long long n = 0, ld = 0, n_ret = 0, n_split = 0;
    bool classified = false;
    bool deferred = false;   // device-collective mode: init/evaluate enqueue only; the non-finite flag travels in the packed row
    long long width = 0;     // block-sum capacity of the current packed row
  } shard;
  pcb::DevBuf pg_row, pg_gathered, pg_lists, pg_rowb;
  // roofline profiling (pcb_profile_begin/end)
  bool profiling = false;
  struct Span { cudaEvent_t a, b; double units; int tag; };
  std::vector<Span> spans[3];
  std::vector<Span> span_pool;
  pcb::DevBuf mc_bounds[2], mc_hist, mc_contrib, mc_seg, mc_group, mc_tmp, mc_inject;
  // pcb_mcubes_run: device run state (stop iteration, history), per-iteration tables, pinned iteration records
  pcb::DevBuf mc_state, mc_tables, mc_timeline;
  void* mc_out_pinned = nullptr;      // pinned staging of the per-iteration tables and the final boundaries
  size_t mc_out_cap = 0;
  void* mc_records = nullptr;
  size_t mc_records_cap = 0;
  unsigned long long mc_run_token = 0;
  std::vector<cudaEvent_t> mc_events;
  std::map<std::array<long long, 6>, unsigned long long> mc_multipliers;  // lane -> segment map, per plan
  // sharded m-Cubes run (pcb_mcubes_shard_*): state between begin and end
  struct McShard {
    bool live = false;
    pcb_integrand f;
    pcb_mcubes_plan plan;
    int iterations = 0, rng_kind = 0, adapt = 1, smoothing = 1, rank = 0, world = 1, keep_tables = 0;
    double alpha = 1.5, rel_tol = 0.0, abs_tol = 0.0;
    unsigned long long seed = 0, token = 0;
    long long t_begin = 0, t_end = 0, n_groups = 0, g_count = 0, width = 0, row_doubles = 0;
    size_t span_mark[3] = {0, 0, 0};
  } mc_shard;
  pcb::DevBuf mc_row, mc_gathered;

  std::vector<pcb::DevBuf*> buffers() {
    return {&lefts[0], &lefts[1], &lengths[0], &lengths[1], &est_i, &est_e, &est_k, &flags, &counts, &offsets,
            &ret_i, &ret_e, &tree[0], &tree[1], &scalars, &rows_a, &rows_b, &k64, &mc_bounds[0], &mc_bounds[1],
            &mc_hist, &mc_contrib, &mc_seg, &mc_group, &mc_tmp, &mc_inject, &mc_state, &mc_tables, &mc_timeline, &mc_row,
            &mc_gathered, &pg_row, &pg_gathered, &pg_lists, &pg_rowb};
  }
  pcb::ChunkCache chunk_cache;
  pcb_ctx() {
    for (pcb::DevBuf* b : buffers()) { b->device = &device; b->cache = &chunk_cache; }
  }
  void release_buffers() {
    for (pcb::DevBuf* b : buffers()) b->release();
  }
  pcb_ctx(const pcb_ctx&) = delete;
  pcb_ctx& operator=(const pcb_ctx&) = delete;
};

namespace pcb {

inline pcb_status fail(pcb_ctx* ctx, pcb_status code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf;
  return code;
}

#define PCB_CUDA_TRY(ctx, expr)                                                                         \
  do {                                                                                                  \
    cudaError_t _e = (expr);                                                                            \
    if (_e != cudaSuccess) {                                                                            \
      (void)cudaGetLastError();                                                                         \
      return pcb::fail(ctx, PCB_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, __LINE__); \
    }                                                                                                   \
  } while (0)

#define PCB_TRY(expr)                     \
  do {                                    \
    pcb_status _s = (expr);               \
    if (_s != PCB_OK) return _s;          \
  } while (0)

// kernel getters, one translation unit per integrand family (pagani_inst.cu / mcubes_inst.cu)
typedef const void* (*kernel_getter)(int d);
const void* eval_kernel(int family, int d);
const void* eval_wide_kernel(int family, int d);   // schedule widths above 64 (exact-order form, every family)
const void* eval_lanes_kernel(int family, int d, size_t* smem, int* threads);  // nullptr: family has no one-region-per-lane kernel
const void* points_kernel(int family, int d);
const void* vsample_kernel_ptr(int family, int d, int rng);

// bracket one dominant-kernel launch with events when profiling is on
struct ProfileSpan {
  pcb_ctx* ctx;
  int kind;
  pcb_ctx::Span span{};
  bool on;
  // `tag` lets a driver that enqueues speculatively (pcb_mcubes_run) discard the spans of passes that never ran
  ProfileSpan(pcb_ctx* c, int k, double units, int tag = 0) : ctx(c), kind(k), on(c->profiling) {
    if (!on) return;
    if (!ctx->span_pool.empty()) {
      span = ctx->span_pool.back();
      ctx->span_pool.pop_back();
    } else {
      cudaEventCreate(&span.a);
      cudaEventCreate(&span.b);
    }
    span.units = units;
    span.tag = tag;
    cudaEventRecord(span.a, ctx->stream);
  }
  ~ProfileSpan() {
    if (!on) return;
    cudaEventRecord(span.b, ctx->stream);
    ctx->spans[kind].push_back(span);
  }
};

// Launch with programmatic stream serialisation (see pdl_wait() in pcb_device.cuh): back-to-back kernels of one
// stream overlap the launch latency and the prologue of the next with the tail of the previous one.
// PCB_NO_PDL=1 launches plainly (A/B measurements).
inline bool pdl_enabled() {
  static const bool on = [] { const char* e = std::getenv("PCB_NO_PDL"); return !(e && std::atoi(e) != 0); }();
  return on;
}
inline cudaError_t launch_pdl(const void* fn, dim3 grid, dim3 block, void** args, size_t smem, cudaStream_t stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

inline long long round_up(long long x, long long m) { return (x + m - 1) / m * m; }

pcb_status validate_integrand(pcb_ctx* ctx, const pcb_integrand* f);

// internal entry points shared between translation units
pcb_status tree_sum_dev(pcb_ctx* ctx, const double* in_dev, long long n, double* out_dev_scalar);
pcb_status fetch_nonfinite_pagani(pcb_ctx* ctx, const pcb_integrand* f, const pcb_rule* rule, long long ld,
                                  const double* lefts_dev, const double* lengths_dev, unsigned long long flat,
                                  pcb_nonfinite* bad);

}  // namespace pcb
