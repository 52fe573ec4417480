// ktab.h — kernel table: the host stubs of the __global__ template
// instantiations, each group defined in its own translation unit (ks_*.cu,
// kc_*.cu) so that build.py compiles them in parallel; gmres_capi.cu launches
// through these pointers.
#pragma once

namespace g200 {
// fused solve kernels (gmres_kernels.cuh solve_kernel<W, L, VR, MON, CH, PC>)
void* ktab_solve_f32_lo(int L);   // default instantiation, L ∈ {1, 2, 4}
void* ktab_solve_f32_hi(int L);   // default instantiation, L ∈ {8, 16, 32}
void* ktab_solve_f64_lo(int L);
void* ktab_solve_f64_hi(int L);
// variant: 1 orthogonality monitor (MON), 2 chunk-ring MGS (CH = 1), 3 ILU(0) (PC), 4 virtual ranks (VR),
// 5 streamed MGS (CH = 2), 6 MGS global sweep (CH = 3); L ∈ {1, 4}
void* ktab_solve_f32_ext(int variant, int L);
void* ktab_solve_f64_ext(int variant, int L);
// component kernels: kind 0 spmv, 1 resid, 2 ortho (resident MGS / sweep / CGSR), 3 xupdate, 4 ilu apply,
// 6 ortho with the chunk-ring MGS, 7 ortho with the streamed MGS
void* ktab_comp_f32(int kind, int L);
void* ktab_comp_f64(int kind, int L);
}  // namespace g200
