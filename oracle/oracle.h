/* oracle/oracle.h — CPU oracle for mixed-precision restarted GMRES(m).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (paper_2011_01850_b200/) never links, imports or calls it.
 *
 * Plain, slow, single-threaded C++ that follows Alg. 1 of the paper
 * step by step, with the precision split of §4
 * and the readings listed in DESIGN.md §2.
 * `prec`: 0 = fp64 (W = double), 1 = mixed (W = float inside Alg. 1 lines
 * 89–146, fp64 residual and update).  Arrays typed `void*` hold W values.
 * Matrices are CSR (int32 row_ptr/col, fp64 val unless stated).  V is
 * column-major with leading dimension ldv.
 */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORACLE_FP64 = 0, ORACLE_MIXED = 1 };
enum { ORACLE_MGS = 0, ORACLE_CGSR = 1 };
/* ablation flags (Fig. 1/2 behaviour pins; never used by the product) */
enum {
  ORACLE_F_CGS1 = 1,     /* CGSR with one pass only (no re-orthogonalisation) */
  ORACLE_F_RESID32 = 2,  /* residual z = b − A x computed in fp32             */
  ORACLE_F_UPDATE32 = 4, /* solution x stored/updated in fp32                  */
  ORACLE_F_ACC32 = 8,    /* fp32 accumulators for dots/norms (mixed only)      */
  /* preconditioner selection (§8 f2, reading R24): default Jacobi (R11) */
  ORACLE_F_ILU0 = 16,    /* ILU(0) factorised and applied in W                 */
  ORACLE_F_ILU32 = 32    /* fp64 solver with an fp32 ILU(0) ("single-precision
                            ILU"); requires ORACLE_FP64          */
};
enum {
  ORACLE_OK = 0, ORACLE_NOT_CONVERGED = 1, ORACLE_EINVAL = -1, ORACLE_EBADCSR = -2,
  ORACLE_EZERODIAG = -3, ORACLE_EFP32RANGE = -4, ORACLE_ENONFINITE = -5
};

typedef struct {
  int32_t cycles;       /* Arnoldi cycles executed (x-updates)          */
  int32_t inner_iters;  /* total inner iterations                        */
  int32_t history_len;  /* number of per-cycle residuals (cycles + 1)    */
  int32_t inner_len;    /* number of per-inner |s_{j+1}| values          */
  double final_relres;  /* ‖b − A x‖₂ / ‖b‖₂ at exit                     */
} oracle_result;

/* --- component operations (each cites the passage it follows) --- */
void oracle_spmv64(int64_t n, const int32_t* rp, const int32_t* ci, const double* a, const double* x, double* y);
void oracle_spmv32(int64_t n, const int32_t* rp, const int32_t* ci, const float* a, const float* x, float* y);
int oracle_dinv(int64_t n, const int32_t* rp, const int32_t* ci, const double* a, double* dinv64, int64_t* bad_row);
int oracle_cast32(int64_t cnt, const double* in, float* out);
/* §8 f2 (reading R24): ILU(0) of A_W on A's pattern, IKJ order, in W
   (prec): f = factors (strict lower part = L with unit diagonal implicit, rest = U).
   Returns ORACLE_EZERODIAG (bad_row set) on a missing diagonal or a zero pivot. */
int oracle_ilu0(int prec, int64_t n, const int32_t* rp, const int32_t* ci, const void* aW, void* f, int64_t* bad_row);
/* out = U⁻¹ L⁻¹ z in W (forward then backward substitution, k ascending per row) */
void oracle_ilu0_apply(int prec, int64_t n, const int32_t* rp, const int32_t* ci, const void* f, const void* z,
                       void* out);
void oracle_jacobi_spmv(int prec, int64_t n, const int32_t* rp, const int32_t* ci, const void* aW,
                        const void* dinvW, const void* v, void* w);
int oracle_resid(int prec, int64_t n, const int32_t* rp, const int32_t* ci, const double* a64,
                 const double* b, const double* x, const void* dinvW, void* r, double* zz, double* rr);
double oracle_dot(int prec, int64_t n, const void* x, const void* y);
void oracle_mgs(int prec, int64_t n, int j, const void* V, int64_t ldv, void* w, double* h);
void oracle_cgsr(int prec, int64_t n, int j, const void* V, int64_t ldv, void* w, double* h, int passes);
void oracle_scale(int prec, int64_t n, const void* w, double inv, void* v);
void oracle_givens(double a, double b, double* c, double* s, double* rho);
/* a6: apply rotations 1..j−1 to column h[0..j] (h[j] = h_{j+1,j}), form rotation j,
   rotate s; j is 1-based.  Returns |s_{j+1}|. */
double oracle_hess_step(int j, double* h, double* cs, double* sn, double* s);
int oracle_backsolve(int J, const double* R, int64_t ldr, const double* s, double* y);
void oracle_xupdate(int prec, int64_t n, int J, const void* V, int64_t ldv, const double* y, double* x);

/* One Arnoldi cycle (Alg. 1 lines 92–141) from the (unnormalised) preconditioned
 * residual r (W), with exit threshold thr on |s_{j+1}|.  Outputs V (n×(m+1), W),
 * Hbar (unrotated, (m+1)×m, ld m+1), R (rotated, same shape), s (m+1), J.
 * Returns 0, or a negative error. */
int oracle_arnoldi(int prec, int ortho, int flags, int64_t n, const int32_t* rp, const int32_t* ci,
                   const void* aW, const void* dinvW, const void* r, int m, double thr,
                   void* V, int64_t ldv, double* Hbar, double* R, double* s, int32_t* J, int32_t* breakdown,
                   double* inner_hist);

/* Restart policies (readings R6, R22):
 * THRESHOLD  restart at j = m or |s_{j+1}| ≤ β·max(tol‖b‖/‖z‖, δ);
 * TWOSTAGE   the first cycle as THRESHOLD, later cycles at the first cycle's
 *            iteration count J1;
 * STALL      THRESHOLD plus: restart when |s_{j+1}| improved by less than a factor
 *            stall_factor over the last ⌈stall_frac·m⌉ inner iterations
 *            (SURVEY §8 f4). */
enum { ORACLE_POLICY_THRESHOLD = 0, ORACLE_POLICY_TWOSTAGE = 1, ORACLE_POLICY_STALL = 2, ORACLE_POLICY_ORTHLOSS = 3 };
/* ORTHLOSS   THRESHOLD plus a restart when ‖S_k‖ ≥ orth_thresh, S_k = (I+U_k)⁻¹U_k,
 *            U_k = strict upper part of V_kᵀV_k (SURVEY §8
 *            f3); ‖·‖ = Frobenius (orth_kind 0) or spectral by 10 power iterations (1);
 *            orth_hist[t] = the norm after inner step t. */

/* The whole restarted solve (Alg. 1).  x0 may be NULL (= 0).  history[k] =
 * ‖b − A x_k‖/‖b‖, k = 0..cycles; inner[t] = |s_{j+1}|/β per inner step. */
int oracle_gmres_solve(int64_t n, const int32_t* rp, const int32_t* ci, const double* a, const double* b,
                       const double* x0, double* x, int m, double tol, int ortho, int prec, double delta,
                       int max_cycles, int flags, oracle_result* res, double* history, int32_t history_cap,
                       double* inner, int32_t inner_cap);
int oracle_gmres_solve_policy(int64_t n, const int32_t* rp, const int32_t* ci, const double* a, const double* b,
                              const double* x0, double* x, int m, double tol, int ortho, int prec, double delta,
                              int max_cycles, int flags, oracle_result* res, double* history, int32_t history_cap,
                              double* inner, int32_t inner_cap, int policy, double stall_factor, double stall_frac);
int oracle_gmres_solve_orth(int64_t n, const int32_t* rp, const int32_t* ci, const double* a, const double* b,
                            const double* x0, double* x, int m, double tol, int ortho, int prec, double delta,
                            int max_cycles, int flags, oracle_result* res, double* history, int32_t history_cap,
                            double* inner, int32_t inner_cap, int policy, double stall_factor, double stall_frac,
                            int orth_kind, double orth_thresh, double* orth_hist, int32_t orth_cap);

#ifdef __cplusplus
}
#endif
