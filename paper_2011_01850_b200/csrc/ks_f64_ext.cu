// ks_f64_ext.cu — kernel-table translation unit (see ktab.h): the monitor / chunk-ring / streamed-MGS / ILU / virtual-rank solve kernels (double).
#include "gmres_kernels.cuh"
#include "ktab.h"

namespace g200 {
void* ktab_solve_f64_ext(int variant, int L) {
  const bool l1 = L == 1;
  switch (variant) {
    case 1: return l1 ? (void*)&solve_kernel<double, 1, false, true> : (void*)&solve_kernel<double, 4, false, true>;
    case 2: return l1 ? (void*)&solve_kernel<double, 1, false, false, 1> : (void*)&solve_kernel<double, 4, false, false, 1>;
    case 5: return l1 ? (void*)&solve_kernel<double, 1, false, false, 2> : (void*)&solve_kernel<double, 4, false, false, 2>;
    case 6: return l1 ? (void*)&solve_kernel<double, 1, false, false, 3> : (void*)&solve_kernel<double, 4, false, false, 3>;
    case 3: return l1 ? (void*)&solve_kernel<double, 1, false, false, 0, true>
                      : (void*)&solve_kernel<double, 4, false, false, 0, true>;
    default: return l1 ? (void*)&solve_kernel<double, 1, true> : (void*)&solve_kernel<double, 4, true>;
  }
}
}  // namespace g200
