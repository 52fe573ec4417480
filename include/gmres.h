/* include/gmres.h — C ABI of the B200-native mixed-precision restarted GMRES(m).
 *
 * Method: restarted, left-preconditioned GMRES(m) of Alg. 1
 * with MGS or CGSR (two passes) and the
 * mixed-precision split of §4: the residual z = b − A·x
 * (Alg. 1 line 86) and the update x ← x + u (line 147) in fp64, everything in
 * between (lines 89–146) in fp32 on an fp32 copy of A ("the matrix is stored
 * twice").  Preconditioner: Jacobi M = diag(A) (BASELINE.json)
 * by default; the paper's ILU(0) in W or, for the fp64 solver, in
 * fp32 through gmres_opts.precond.  H, the Givens rotations and
 * s are fp64 on the device (reading R7).
 *
 * All compute runs in hand-written sm_100a kernels (libgmres.so); no
 * cuSPARSE/cuBLAS.  Plain C: no C++ types or exceptions cross this boundary.
 *
 * Conventions
 *  - CSR: int32 row_ptr[n+1], int32 col[nnz], fp64 val[nnz]; row_ptr[0] = 0,
 *    non-decreasing, row_ptr[n] = nnz, columns strictly increasing and < n
 *    within each row.  Every row must hold a non-zero diagonal.
 *  - Ownership: the caller owns every array it passes.  gmres_create COPIES A
 *    to the device; the caller may free its arrays on return.  Outputs are
 *    caller-allocated.  The library never returns memory the caller must free.
 *  - Return codes: 0 = OK, 1 = NOT_CONVERGED (max_cycles reached; x holds the
 *    last iterate), negative = error; gmres_last_error() describes it.
 *  - Concurrency: one solve per context at a time; calls are stream-ordered on
 *    the context's stream (or the stream given to *_device calls).
 */
#ifndef GMRES_H
#define GMRES_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gmres_ctx gmres_ctx;

typedef enum { GMRES_MGS = 0, GMRES_CGSR = 1 } gmres_ortho;
typedef enum { GMRES_FP64 = 0, GMRES_MIXED = 1 } gmres_precision;

typedef enum {
  GMRES_OK = 0,
  GMRES_NOT_CONVERGED = 1,
  GMRES_EINVAL = -1,       /* bad argument: m < 1, tol ≤ 0 or NaN, bad enum, null pointer */
  GMRES_EBADCSR = -2,      /* CSR invariants violated                    */
  GMRES_EZERODIAG = -3,    /* missing or zero diagonal; message names the row            */
  GMRES_EFP32RANGE = -4,   /* mixed mode: |a_ij| or |z_i| exceeds FLT_MAX   */
  GMRES_ENONFINITE = -5,   /* NaN/Inf in the residual or the Arnoldi process             */
  GMRES_ENOMEM = -6,       /* device allocation failed                                   */
  GMRES_ECUDA = -7,        /* CUDA runtime error (message has the CUDA error string)     */
  GMRES_ETIMEOUT = -8      /* device-side watchdog fired in a grid barrier               */
} gmres_status;

typedef struct {
  int32_t status;         /* gmres_status of the solve                                  */
  int32_t cycles;         /* Arnoldi cycles executed = x-updates (0 if x0 converged)    */
  int32_t inner_iters;    /* total inner iterations over all cycles                     */
  int32_t history_len;    /* cycles + 1 per-cycle residuals recorded                    */
  double final_relres;    /* ‖b − A x‖₂/‖b‖₂ of the returned x (fp64, on device)        */
  double device_ms;       /* device time of the solve (CUDA events), incl. the A32 cast */
  double kernel_ms;       /* device time of the fused solve kernel alone (CUDA events)  */
  double final_backward_err; /* ‖b − A x‖₂/(‖A‖_F‖x‖₂ + ‖b‖₂) of the returned x (
                             the paper's unnamed "backward error", PAPER.md:317, 431-433;
                             report only — the stop test is final_relres)              */
} gmres_result;

typedef struct {
  double delta;           /* Arnoldi-improvement restart threshold (PAPER.md:257-264,
                             448); < 0 → default: 1e-6 mixed, 0 fp64                    */
  int32_t max_cycles;     /* ≤ 0 → 10000                                                */
  int32_t record_inner;   /* != 0: keep |s_{j+1}|/β per inner step (gmres_get_inner_history) */
  int32_t lanes_per_row;  /* SpMV lanes per row 1/2/4/8/16/32; 0 = auto from the mean row
                             length.  Virtual ranks, restart_policy 3 and ILU(0): 1 or 4
                             only (EINVAL otherwise)                                  */
  int32_t ctas_per_sm;    /* 0 = auto (occupancy)                                       */
  int32_t profile;        /* != 0: grid barrier after each phase for clean phase timers */
  int32_t tune;           /* developer A/B switches; 0 = production defaults (bit 25: the
                             mixed MGS projections use the fp64 partial all-reduce instead
                             of the exact fixed-point word of DESIGN.md reading R27; bit 28:
                             the resident MGS ring copies the next vector inside the step's
                             all-reduce instead of at the start of the step)               */
  int32_t restart_policy; /* 0 THRESHOLD: restart at j = m or |s_{j+1}| ≤ β·max(tol‖b‖/‖z‖, δ)
                             (PAPER.md:257-264); 1 TWOSTAGE: the first cycle as THRESHOLD,
                             later cycles at the first cycle's iteration count (PAPER.md:
                             251-255, 448); 2 STALL: THRESHOLD plus a restart when |s| improved
                             by less than stall_factor over the last ⌈stall_frac·m⌉ inner
                             iterations (δ defaults to 0)          */
  double stall_factor;    /* ≤ 0 → 1.001; else must be > 1 (EINVAL)      */
  double stall_frac;      /* ≤ 0 → 0.05                                */
  double orth_thresh;     /* restart_policy 3 ORTHLOSS: THRESHOLD plus a restart when
                             ‖S_k‖ ≥ orth_thresh (orth_norm), S_k = (I+U_k)⁻¹U_k, U_k = strict upper
                             part of V_kᵀV_k; ≤ 0 → 1.0.  Adds
                             one pass over the basis per inner iteration               */
  int32_t precond;        /* left preconditioner M: GMRES_PRECOND_JACOBI (0, default;
                             reading R11), GMRES_PRECOND_ILU0 (1: ILU(0) of A_W on A's
                             pattern, factorised on the device inside every timed solve,
                             PAPER.md:291, 427; reading R24) or GMRES_PRECOND_ILU0_FP32
                             (2: precision GMRES_FP64 only — the fp64 solver with an fp32
                             ILU(0) of RN32(A), applied as RN32(in) → fp32 solves → fp64:
                             the paper's "single-precision ILU" arm, PAPER.md:428, 444,
                             463).  ILU(0): single-rank contexts, restart policies 0–2  */
  int32_t orth_norm;      /* restart_policy 3: the norm of S_k — 0 Frobenius (default), 1
                             spectral, estimated by 10 power iterations on S_kᵀS_k from
                             x = (1,…,1)/√k; EINVAL otherwise            */
} gmres_opts;

#define GMRES_PRECOND_JACOBI 0
#define GMRES_PRECOND_ILU0 1
#define GMRES_PRECOND_ILU0_FP32 2

/* Create a solver context on the current CUDA device: validates the CSR on the
 * host, copies A (fp64) to the device and extracts the Jacobi diagonal.
 * Host pointers.  Errors: EINVAL, EBADCSR, EZERODIAG, ENOMEM, ECUDA. */
int gmres_create(const int32_t* row_ptr, const int32_t* col, const double* val, int64_t n, int64_t nnz,
                 gmres_ctx** out);

/* Solve A x = b with host arrays b[n], x0[n] (NULL → x0 = 0) into x_out[n].
 * history (may be NULL) receives ‖b − A x_k‖/‖b‖ for k = 0..cycles (at most
 * history_cap values; *history_len gets the full count).  opts may be NULL.
 * Blocks until done.  Returns the solve status (see gmres_status). */
int gmres_solve(gmres_ctx* ctx, const double* b, const double* x0, double* x_out, int32_t m, double tol,
                int32_t ortho, int32_t precision, const gmres_opts* opts, gmres_result* res, double* history,
                int32_t history_cap, int32_t* history_len);

/* Same with DEVICE arrays d_b, d_x0 (may be NULL), d_x (may alias d_x0),
 * ordered on `stream` (a cudaStream_t; NULL = the context's own stream).
 * history stays a HOST array.  Blocks until the solve finished. */
int gmres_solve_device(gmres_ctx* ctx, const double* d_b, const double* d_x0, double* d_x, int32_t m, double tol,
                       int32_t ortho, int32_t precision, const gmres_opts* opts, gmres_result* res,
                       double* history, int32_t history_cap, int32_t* history_len, void* stream);

/* Per-inner-step |s_{j+1}|/β of the last solve (opts.record_inner != 0). */
int gmres_get_inner_history(gmres_ctx* ctx, double* buf, int32_t cap, int32_t* len);

/* Inner iterations J_k of every cycle k of the last solve (for byte models). */
int gmres_get_cycle_iters(gmres_ctx* ctx, int32_t* buf, int32_t cap, int32_t* len);

/* Device-side phase timers of the last solve (ns, measured by CTA 0 with
 * %globaltimer): [0] residual, [1] SpMV, [2] orthogonalisation, [3] norm +
 * Givens, [4] back-solve + update; with opts.profile: [5] max and [6] mean
 * over CTAs of the CTA's own SpMV time.  Returns the count written. */
int gmres_get_phase_ns(gmres_ctx* ctx, double* buf, int32_t cap);

/* Launch plan of the last solve (host-side choices, for tests and tuning):
 * [0] CTAs, [1] SpMV lanes per row, [2] MGS variant (0 global sweep,
 * 1 whole-vector TMA ring, 2 chunk ring with w partly in shared memory),
 * [3] ring depth (vectors for 1, 8 KB chunk slots for 2), [4] chunks of w in
 * shared memory (variant 2), [5] staging bytes, [6] dynamic shared memory per
 * CTA, [7] CSR stream (0 per-warp chunks, 1 block stream for rows of ≤ 64
 * non-zeros, 2 merge-path tiles for irregular rows), [8] CGSR row-tile height (0: column-major
 * basis).  buf is host memory of cap ≥ 0 entries; returns the count written
 * (≤ GMRES_PLAN_N), or GMRES_EINVAL for a null argument. */
#define GMRES_PLAN_N 9
int gmres_get_plan(gmres_ctx* ctx, int32_t* buf, int32_t cap);

/* Instrumentation (outside any timed region): copy columns [col0, col0+ncols)
 * of the Krylov basis V left by the last solve on ctx — the basis of its last
 * cycle, v_1..v_J in columns 0..J−1 — into d_dst (device, column-major,
 * leading dimension ld ≥ n, element type = that solve's working precision:
 * float for mixed, double for fp64).  Used for ‖I − VᵀV‖ (BASELINE.json C5).
 * EINVAL before any solve or for columns outside [0, m]. */
int gmres_get_basis(gmres_ctx* ctx, int32_t col0, int32_t ncols, void* d_dst, int64_t ld);

/* ------------------------------------------------------------------------
 * Row-partitioned solve over P ranks (the paper's future work,
 * PAPER.md:491-495).  Rank q owns the contiguous global rows
 * [row_begin_q, row_begin_q + n_q) of A, b and x; CSR rows are local, column
 * indices GLOBAL.  Every rank runs the same restarted solve: the Gram–Schmidt
 * dots and norms are all-reduced over all ranks' CTAs inside the persistent
 * kernel (each CTA pushes its partials to every rank and arrives on every
 * rank's counter), and the rows of the Krylov vector / residual / x a peer
 * gathers in its SpMV are pushed into the peer's copy by the owning CTA
 * (peer stores) before that all-reduce publishes them.  All ranks take
 * bit-identical control decisions (same sums in the same order).
 * ---------------------------------------------------------------------- */

/* Host-only planning helpers (no device is touched; usable on any host):
 * gmres_dist_partition: boundaries bounds[0..nranks] (bounds[0] = 0,
 *   bounds[nranks] = n) of a split of the n rows of a global CSR (row_ptr) at
 *   multiples of `align`, balancing rows + nonzeros.
 * gmres_dist_ghosts: the sorted unique global columns of a rank's local rows
 *   (row_ptr/col, n_local rows starting at global row row_begin) outside
 *   those rows; *count = their number, at most cap written.
 * gmres_dist_sends: the local rows of rank [row_begin, row_begin + n_local)
 *   that appear in a peer's ghost list (i.e. what this rank pushes to it). */
int gmres_dist_partition(const int32_t* row_ptr, int64_t n, int32_t nranks, int64_t align, int64_t* bounds);
int gmres_dist_ghosts(const int32_t* row_ptr, const int32_t* col, int64_t n_local, int64_t row_begin, int32_t* ghosts,
                      int64_t cap, int64_t* count);
int gmres_dist_sends(int64_t row_begin, int64_t n_local, const int32_t* peer_ghosts, int64_t n_peer_ghosts,
                     int32_t* rows, int64_t cap, int64_t* count);
/* Host-only: the merge-path tiles of the CSR stream for irregular rows (§8 a2;
 * PAPER.md:100, Alg. 1), as the solves build them for a grid of G CTAs
 * owning rows [cta_rows[g], cta_rows[g+1]) (host arrays, G+1 entries).  A tile
 * starts at non-zero position s, ends at ne ≤ (s & ~7) + 256 and touches ≤ 31
 * rows; rows may span tiles.  tiles: 4 int32 per entry {first row, s, rows
 * touched, 0}, per CTA its tiles then a sentinel {row end, nnz end, 0, 0}
 * (the next entry's s is a tile's ne); tile_off[g] (G+1 entries) = index of
 * CTA g's first entry.  splits: 4 int32 per row that spans tiles {row, tile of
 * its first non-zero, tile of its last, 0} (tile = global entry index);
 * split_off[g] (G+1) likewise.  At most tiles_cap / splits_cap entries are
 * written, *n_tiles / *n_splits receive the full counts; tile_off / split_off
 * may be NULL.  GMRES_EINVAL for an empty row (every row must hold its
 * diagonal) or bad arguments. */
int gmres_plan_mtiles(const int32_t* row_ptr, int64_t n, const int32_t* cta_rows, int32_t G, int32_t* tiles,
                      int64_t tiles_cap, int64_t* n_tiles, int32_t* tile_off, int32_t* splits, int64_t splits_cap,
                      int64_t* n_splits, int32_t* split_off);

/* One rank's share of the matrix (host arrays, copied): n_local rows from
 * global row row_begin (a multiple of 256; n_local a multiple of 256 unless
 * the block ends at n_global), 2 ≤ nranks ≤ 8.  Errors as gmres_create. */
int gmres_create_dist(const int32_t* row_ptr, const int32_t* col, const double* val, int64_t n_global,
                      int64_t row_begin, int64_t n_local, int32_t nranks, int32_t rank, gmres_ctx** out);
/* One process per GPU: export this rank's blob (ghost list + CUDA IPC
 * handles of its exchange buffers; *len = size, blob may be NULL to query),
 * all-gather the blobs (e.g. torch.distributed), then import all of them
 * (offsets[q] = start of rank q's blob, offsets[nranks] = total).  Afterwards
 * gmres_solve_device is collective: every rank calls it with the same m,
 * tol, ortho, precision and options and its own local b, x0, x. */
int gmres_dist_export(gmres_ctx* ctx, void* blob, int64_t cap, int64_t* len);
int gmres_dist_import(gmres_ctx* ctx, const void* blobs, const int64_t* offsets);
/* Several ranks in one process on ONE device ("virtual ranks", 2 ≤ P ≤ 4):
 * link them (peer buffers are the other contexts' allocations) and solve
 * them in one cooperative launch (sms/P CTAs per rank) — the same kernel
 * code as the multi-GPU path.  res[P] receives every rank's result. */
int gmres_dist_link_local(gmres_ctx* const* ctxs, int32_t nranks);
int gmres_solve_virtual(gmres_ctx* const* ctxs, int32_t nranks, const double* const* d_b, const double* const* d_x0,
                        double* const* d_x, int32_t m, double tol, int32_t ortho, int32_t precision,
                        const gmres_opts* opts, gmres_result* res);

const char* gmres_last_error(const gmres_ctx* ctx);  /* "" if none; ctx may be NULL */
void gmres_destroy(gmres_ctx* ctx);

/* ------------------------------------------------------------------------
 * Component entry points (used by the parity tests; device pointers, W =
 * float in mixed mode, double in fp64 mode; blocking).  Each runs the SAME
 * device code the fused solve kernel runs for that step.
 * ---------------------------------------------------------------------- */

/* a2 (Alg. 1): d_w = RN_W(dinv_W ∘ (A_W · d_v)). */
int gmres_k_spmv(gmres_ctx* ctx, int32_t precision, const void* d_v, void* d_w);

/* a1 (Alg. 1 lines 86–90): z = b − A64 x (fp64); d_r = RN_W(dinv_W ∘ RN_W(z));
 * out2[0] = ‖z‖², out2[1] = ‖r‖² (host). */
int gmres_k_resid(gmres_ctx* ctx, int32_t precision, const double* d_b, const double* d_x, void* d_r,
                  double* out2);

/* a3/a4 + a5 (Alg. 1): orthogonalise d_w (n, W) in place against
 * the j columns of d_V (column-major, leading dimension ldv ≥ round_up(n, 256),
 * ldv % 64 == 0, rows ≥ n zero) with MGS or CGSR; h_out (host) receives
 * h_{1..j} and h_out[j] = ‖w‖₂.  CGSR copies V into the row-blocked layout a
 * CGSR solve keeps its basis in and runs on that copy.  Mixed MGS reduces the
 * projections as the mixed solve does (reading R27: exact fixed-point
 * sums, bound B = 2^⌈log2(2‖w‖₂)⌉ from this call's w, for orthonormal V);
 * GMRES_ENONFINITE if a partial falls outside that bound (non-finite data). */
int gmres_k_ortho(gmres_ctx* ctx, int32_t precision, int32_t ortho, int32_t j, const void* d_V, int64_t ldv,
                  void* d_w, double* h_out);
/* The same with the MGS variant chosen: mgs_variant −1 = the one a solve on this
 * context would run (gmres_k_ortho), 0 global sweep, 1 register-resident w with a
 * whole-vector TMA ring, 2 chunk ring, 3 streamed (w off chip); GMRES_EINVAL if the
 * requested variant does not fit.  *variant_used (may be NULL) receives the variant
 * that ran (−1 for CGSR).  All variants perform the same operations in the same
 * order (reading R9), so their results agree bit for bit. */
int gmres_k_ortho_ex(gmres_ctx* ctx, int32_t precision, int32_t ortho, int32_t j, const void* d_V, int64_t ldv,
                     void* d_w, double* h_out, int32_t mgs_variant, int32_t* variant_used);

/* a8 (Alg. 1): d_x += Σ_{i<J} (double)V_i · y_i; y host[J];
 * d_V as for gmres_k_ortho.  blocked != 0: run on a row-blocked copy of V
 * (the layout of a CGSR solve), else on d_V itself (the MGS solves' layout). */
int gmres_k_xupdate(gmres_ctx* ctx, int32_t precision, int32_t J, const void* d_V, int64_t ldv, const double* y,
                    double* d_x, int32_t blocked);

/* a6 + a7 (Alg. 1) on the device: apply the Givens steps to the
 * J columns of the unrotated (m+1)×m Hessenberg Hbar (host, column-major,
 * ld m+1) with s_1 = beta; returns the rotated R (host, same layout), s[J+1]
 * and y[J] = R⁻¹ s_{1..J}. */
int gmres_k_hessenberg(gmres_ctx* ctx, int32_t m, int32_t J, const double* Hbar, double beta, double* R,
                       double* s, double* y);

/* §8 f2 (reading R24): ILU(0) of A_W (W = fp32 for GMRES_MIXED
 * from the fp32 copy of A, fp64 otherwise) on A's pattern, IKJ order, rows in
 * natural order, one launch per level of the lower dependency graph.  d_f
 * (device, nnz W values, may be NULL) receives the factors: strict lower part
 * L (unit diagonal implicit), the rest U, in A's CSR order.  The factors stay
 * in the context for gmres_k_ilu_apply.  EZERODIAG (message names the row) on a
 * missing diagonal or a zero / non-finite pivot; single-rank contexts only. */
int gmres_ilu0_factor(gmres_ctx* ctx, int32_t precision, void* d_f);

/* d_out = U⁻¹ L⁻¹ d_z (device, n W values each; d_out == d_z allowed) with the
 * factors of the last gmres_ilu0_factor of this precision: forward then backward
 * substitution, each row's sum in ascending column order in W, in one cooperative
 * launch.  schedule 0: sync-free (rows poll their inputs' published values — the
 * solve kernel's default); 65536: level-synchronous (a grid barrier per level).
 * Both reproduce the oracle bit for bit. */
int gmres_k_ilu_apply(gmres_ctx* ctx, int32_t precision, const void* d_z, void* d_out, int32_t schedule);

/* Level counts of the ILU(0) triangular solves (lower, upper): the length of
 * the dependency chains a level-scheduled solve serialises over. */
int gmres_ilu0_levels(gmres_ctx* ctx, int32_t* nlev_lower, int32_t* nlev_upper);

/* a0: build the fp32 copy of A on the device (also rebuilt
 * inside every mixed solve, timed).  EFP32RANGE on overflow. */
int gmres_k_cast32(gmres_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* GMRES_H */
