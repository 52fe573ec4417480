// ks_f32_hi.cu — kernel-table translation unit (see ktab.h): solve_kernel<float, L> for L in [8, 16, 32].
#include "gmres_kernels.cuh"
#include "ktab.h"

namespace g200 {
void* ktab_solve_f32_hi(int L) {
  switch (L) {
    case 8: return (void*)&solve_kernel<float, 8, false>;
    case 16: return (void*)&solve_kernel<float, 16, false>;
    default: return (void*)&solve_kernel<float, 32, false>;
  }
}
}  // namespace g200
