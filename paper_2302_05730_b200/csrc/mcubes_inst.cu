// Instantiations of the m-Cubes V-Sample kernel for ONE integrand family
// (compiled once per family with -DPCB_FAM=<pcb_family>).
#include "mcubes_kernels.cuh"

#ifndef PCB_FAM
#error "compile with -DPCB_FAM=<family id>"
#endif
#define PCB_CAT2(a, b) a##b
#define PCB_CAT(a, b) PCB_CAT2(a, b)
#define PCB_DIMS(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12)

namespace pcb {

// rng 0: the reference counter hash (hot path); any other kind: generic kernel (Philox / injected table)
const void* PCB_CAT(vsample_kernel_fam, PCB_FAM)(int d, int rng) {
  if (rng == PCB_RNG_REFERENCE_HASH) {
    switch (d) {
#define X(D) case D: return (const void*)&vsample_kernel<PCB_FAM, D, PCB_RNG_REFERENCE_HASH>;
      PCB_DIMS(X)
#undef X
    }
  } else {
    switch (d) {
#define X(D) case D: return (const void*)&vsample_kernel<PCB_FAM, D, PCB_RNG_PHILOX>;
      PCB_DIMS(X)
#undef X
    }
  }
  return nullptr;
}

}  // namespace pcb
