// kc_f64.cu — kernel-table translation unit (see ktab.h): the per-step component kernels (double).
#include "gmres_kernels.cuh"
#include "ktab.h"

namespace g200 {
void* ktab_comp_f64(int kind, int L) {
  switch (kind) {
    case 0:
      switch (L) {
        case 1: return (void*)&k_spmv_kernel<double, 1>;
        case 2: return (void*)&k_spmv_kernel<double, 2>;
        case 4: return (void*)&k_spmv_kernel<double, 4>;
        case 8: return (void*)&k_spmv_kernel<double, 8>;
        case 16: return (void*)&k_spmv_kernel<double, 16>;
        default: return (void*)&k_spmv_kernel<double, 32>;
      }
    case 1:
      switch (L) {
        case 1: return (void*)&k_resid_kernel<double, 1>;
        case 2: return (void*)&k_resid_kernel<double, 2>;
        case 4: return (void*)&k_resid_kernel<double, 4>;
        case 8: return (void*)&k_resid_kernel<double, 8>;
        case 16: return (void*)&k_resid_kernel<double, 16>;
        default: return (void*)&k_resid_kernel<double, 32>;
      }
    case 2: return (void*)&k_ortho_kernel<double, 0>;
    case 6: return (void*)&k_ortho_kernel<double, 1>;  // chunk-ring MGS
    case 7: return (void*)&k_ortho_kernel<double, 2>;  // streamed MGS
    case 4: return (void*)&k_ilu_apply_kernel<double>;
    default: return (void*)&k_xupdate_kernel<double>;
  }
}
}  // namespace g200
