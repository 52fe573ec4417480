// kc_f32.cu — kernel-table translation unit (see ktab.h): the per-step component kernels (float).
#include "gmres_kernels.cuh"
#include "ktab.h"

namespace g200 {
void* ktab_comp_f32(int kind, int L) {
  switch (kind) {
    case 0:
      switch (L) {
        case 1: return (void*)&k_spmv_kernel<float, 1>;
        case 2: return (void*)&k_spmv_kernel<float, 2>;
        case 4: return (void*)&k_spmv_kernel<float, 4>;
        case 8: return (void*)&k_spmv_kernel<float, 8>;
        case 16: return (void*)&k_spmv_kernel<float, 16>;
        default: return (void*)&k_spmv_kernel<float, 32>;
      }
    case 1:
      switch (L) {
        case 1: return (void*)&k_resid_kernel<float, 1>;
        case 2: return (void*)&k_resid_kernel<float, 2>;
        case 4: return (void*)&k_resid_kernel<float, 4>;
        case 8: return (void*)&k_resid_kernel<float, 8>;
        case 16: return (void*)&k_resid_kernel<float, 16>;
        default: return (void*)&k_resid_kernel<float, 32>;
      }
    case 2: return (void*)&k_ortho_kernel<float, 0>;
    case 6: return (void*)&k_ortho_kernel<float, 1>;  // chunk-ring MGS
    case 7: return (void*)&k_ortho_kernel<float, 2>;  // streamed MGS
    case 4: return (void*)&k_ilu_apply_kernel<float>;
    default: return (void*)&k_xupdate_kernel<float>;
  }
}
}  // namespace g200
