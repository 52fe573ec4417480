// ks_f64_hi.cu — kernel-table translation unit (see ktab.h): solve_kernel<double, L> for L in [8, 16, 32].
#include "gmres_kernels.cuh"
#include "ktab.h"

namespace g200 {
void* ktab_solve_f64_hi(int L) {
  switch (L) {
    case 8: return (void*)&solve_kernel<double, 8, false>;
    case 16: return (void*)&solve_kernel<double, 16, false>;
    default: return (void*)&solve_kernel<double, 32, false>;
  }
}
}  // namespace g200
