// Instantiations of the PAGANI evaluate / eval_points kernels for ONE integrand family
// (compiled once per family with -DPCB_FAM=<pcb_family>, so the families build in parallel).
#include "pagani_eval.cuh"
#include "pagani_eval_mult.cuh"
#include "pagani_eval_lanes.cuh"

#ifndef PCB_FAM
#error "compile with -DPCB_FAM=<family id>"
#endif
#define PCB_CAT2(a, b) a##b
#define PCB_CAT(a, b) PCB_CAT2(a, b)
#define PCB_DIMS(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12)

namespace pcb {

// multiplicative families (f1, f4, f5, f6) evaluate rule points as products of tabulated per-axis factors;
// the others keep the exact-order kernel
template <int D>
static const void* eval_kernel_for() {
  if constexpr (MultFamily<PCB_FAM>::enabled) return (const void*)&pagani_eval_mult_kernel<PCB_FAM, D>;
  else return (const void*)&pagani_eval_kernel<PCB_FAM, D>;
}

const void* PCB_CAT(eval_kernel_fam, PCB_FAM)(int d) {
  switch (d) {
#define X(D) case D: return (const void*)eval_kernel_for<D>();
    PCB_DIMS(X)
#undef X
  }
  return nullptr;
}

// schedule widths above 64: the exact-order kernel walking the virtual threads in blocks of 64
const void* PCB_CAT(eval_wide_kernel_fam, PCB_FAM)(int d) {
  switch (d) {
#define X(D) case D: return (const void*)&pagani_eval_kernel<PCB_FAM, D, true>;
    PCB_DIMS(X)
#undef X
  }
  return nullptr;
}

// one-region-per-lane kernel (multiplicative or generic form) and its dynamic shared memory
template <int D>
static const void* lanes_kernel_for(size_t* smem, int* threads) {
  if constexpr (MultFamily<PCB_FAM>::enabled) {
    *smem = LaneLayout<D, MultFamily<PCB_FAM>::unit, (MultFamily<PCB_FAM>::cplx || PCB_LANES_HALVES_REAL > 1)>::smem_bytes(sizeof(MVal<MultFamily<PCB_FAM>::cplx>));
    *threads = (MultFamily<PCB_FAM>::cplx || PCB_LANES_HALVES_REAL > 1) ? 64 : 32;   // complex factors: two warps share the tables of 32 regions
    return (const void*)&pagani_eval_lanes_kernel<PCB_FAM, D>;
  } else {
    *smem = GenericLaneLayout<D>::smem_bytes();
    *threads = 32;
    return (const void*)&pagani_eval_lanes_generic_kernel<PCB_FAM, D>;
  }
}

const void* PCB_CAT(lanes_kernel_fam, PCB_FAM)(int d, size_t* smem, int* threads) {
  switch (d) {
#define X(D) case D: return lanes_kernel_for<D>(smem, threads);
    PCB_DIMS(X)
#undef X
  }
  *smem = 0;
  return nullptr;
}

#if PCB_FAM == 0
// dynamic shared memory of the generic lane kernel for a run-time dimension (run-time families, ctx.cu)
size_t generic_lanes_smem(int d) {
  switch (d) {
#define X(D) case D: return GenericLaneLayout<D>::smem_bytes();
    PCB_DIMS(X)
#undef X
  }
  return 0;
}
#endif

const void* PCB_CAT(points_kernel_fam, PCB_FAM)(int d) {
  switch (d) {
#define X(D) case D: return (const void*)&eval_points_kernel<PCB_FAM, D>;
    PCB_DIMS(X)
#undef X
  }
  return nullptr;
}

const void* PCB_CAT(qmc_kernel_fam, PCB_FAM)(int d) {
  switch (d) {
#define X(D) case D: return (const void*)&qmc_shift_kernel<PCB_FAM, D>;
    PCB_DIMS(X)
#undef X
  }
  return nullptr;
}

const void* PCB_CAT(invoke_kernel_fam, PCB_FAM)(int d) {
  switch (d) {
#define X(D) case D: return (const void*)&invoke_kernel<PCB_FAM, D>;
    PCB_DIMS(X)
#undef X
  }
  return nullptr;
}

}  // namespace pcb
