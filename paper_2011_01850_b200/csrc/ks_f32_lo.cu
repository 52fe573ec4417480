// ks_f32_lo.cu — kernel-table translation unit (see ktab.h): solve_kernel<float, L> for L in [1, 2, 4].
#include "gmres_kernels.cuh"
#include "ktab.h"

namespace g200 {
void* ktab_solve_f32_lo(int L) {
  switch (L) {
    case 1: return (void*)&solve_kernel<float, 1, false>;
    case 2: return (void*)&solve_kernel<float, 2, false>;
    default: return (void*)&solve_kernel<float, 4, false>;
  }
}
}  // namespace g200
