// oracle/oracle.cpp — CPU oracle for mixed-precision restarted GMRES(m).
//
// TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and
// bench.py's CPU-baseline legs; never by the product path.
//
// Plain single-threaded C++ following Alg. 1 in the paper's
// order and notation, with the precision split of PAPER.md:285-289 ("computing
// the residual and updating x in double-precision and computing everything else
// in single-precision") and the readings of DESIGN.md §2 (R1–R24).  Compiled
// -O2 -ffp-contract=off (every W operation rounds on its own), no fast-math.
//
// W is the working precision of Alg. 1 lines 89–146: float in mixed mode,
// double in fp64 mode.  Length-n dot products and norms accumulate in fp64
// (reading R9) unless ORACLE_F_ACC32; short sums (row sums of the SpMV, V·c)
// run in W.  H, the rotations and s are fp64 (reading R7).
#include "oracle.h"

#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <vector>

// Optional OpenMP build (liboracle_omp.so, -fopenmp; BASELINE.md §4 / SURVEY.md
// §8(c) "optional OpenMP build … results bitwise thread-count-invariant"):
// ORACLE_PAR parallelises ONLY loops whose iterations write disjoint outputs and
// contain no cross-iteration reduction (rows of an SpMV, elements of an axpy,
// whole dot products in a set of independent dots).  Every reduction (dots,
// norms, ‖z‖²) stays one sequential loop in index order, so each floating-point
// operation and its operands are the same as in the single-threaded build and
// the two builds agree bit for bit (tests/test_oracle.py::test_omp_build_bitwise).
// Without -fopenmp the pragma is ignored: the default build is plain sequential C++.
#ifdef _OPENMP
#define ORACLE_PAR _Pragma("omp parallel for schedule(static)")
#else
#define ORACLE_PAR
#endif

namespace {

// ---------------------------------------------------------------- helpers
template <class W>
inline W rn(double v) { return (W)v; }  // RN_W: round-to-nearest into W

// Σ_l x_l·y_l with an fp64 accumulator, sequential in l (R9).
template <class W>
double dot(int64_t n, const W* x, const W* y, bool acc32) {
  if (acc32) {
    float s = 0.0f;
    for (int64_t l = 0; l < n; ++l) s = s + (float)x[l] * (float)y[l];
    return (double)s;
  }
  double s = 0.0;
  for (int64_t l = 0; l < n; ++l) s += (double)x[l] * (double)y[l];
  return s;
}

// Alg. 1: w ← M⁻¹ A v_j with M = diag(A) (Jacobi, reading R11).
// Row sum in W in ascending column order, then the Jacobi scale in W.
template <class W>
void jacobi_spmv(int64_t n, const int32_t* rp, const int32_t* ci, const W* a, const W* dinv, const W* v, W* w) {
  ORACLE_PAR
  for (int64_t i = 0; i < n; ++i) {
    W acc = (W)0;
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
      W p = a[e] * v[ci[e]];
      acc = acc + p;
    }
    w[i] = dinv[i] * acc;
  }
}

// ILU(0) ("preconditioned with incomplete LU without fill in";
// reading R24): IKJ elimination restricted to A's pattern, rows in natural
// order, every operation rounded to W:
//   for i, for k < i with a_ik in the pattern (ascending):
//     a_ik ← a_ik / a_kk ;  a_ij ← a_ij − a_ik·a_kj  for j > k with a_ij, a_kj in the pattern.
// The strict lower part then holds L (unit diagonal implicit), the rest U.
template <class W>
int64_t ilu0(int64_t n, const int32_t* rp, const int32_t* ci, W* f) {
  std::vector<int64_t> dpos(n, -1), pos(n, -1);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e)
      if (ci[e] == i) dpos[i] = e;
  for (int64_t i = 0; i < n; ++i) {
    if (dpos[i] < 0) return i;
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) pos[ci[e]] = e;
    for (int64_t e = rp[i]; e < rp[i + 1] && ci[e] < i; ++e) {
      const int64_t k = ci[e];
      f[e] = f[e] / f[dpos[k]];
      for (int64_t q = dpos[k] + 1; q < rp[k + 1]; ++q)
        if (pos[ci[q]] >= 0) f[pos[ci[q]]] = f[pos[ci[q]]] - f[e] * f[q];
    }
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) pos[ci[e]] = -1;
    if (f[dpos[i]] == (W)0 || !std::isfinite((double)f[dpos[i]])) return i;
  }
  return -1;
}

// M⁻¹ z with M = LU (Alg. 1 lines 90 and 100 with the ILU(0) preconditioner):
// L y = z (unit lower), then U x = y, each row's sum sequential in ascending
// column order, in W.
template <class W>
void ilu0_apply(int64_t n, const int32_t* rp, const int32_t* ci, const W* f, const W* z, W* out) {
  std::vector<W> y(n);
  for (int64_t i = 0; i < n; ++i) {
    W t = z[i];
    for (int64_t e = rp[i]; e < rp[i + 1] && ci[e] < i; ++e) t = t - f[e] * y[ci[e]];
    y[i] = t;
  }
  for (int64_t i = n - 1; i >= 0; --i) {
    int64_t d = rp[i];
    while (ci[d] < i) ++d;
    W t = y[i];
    for (int64_t e = d + 1; e < rp[i + 1]; ++e) t = t - f[e] * out[ci[e]];
    out[i] = t / f[d];
  }
}

// MGS procedure: for i = 1..j in order,
//   h_{i,j} ← w·v_i ;  w ← w − h_{i,j} v_i .
template <class W>
void mgs(int64_t n, int j, const W* V, int64_t ldv, W* w, double* h, bool acc32) {
  for (int i = 0; i < j; ++i) {
    const W* vi = V + (int64_t)i * ldv;
    double hij = dot<W>(n, w, vi, acc32);   // line 154
    W hw = rn<W>(hij);
    ORACLE_PAR
    for (int64_t l = 0; l < n; ++l) {        // line 155
      W t = hw * vi[l];
      w[l] = w[l] - t;
    }
    h[i] = hij;
  }
}

// CGSR procedure, performed twice (reading R2):
//   h ← V_jᵀ w ;  w ← w − V_j h ;  accumulate h over the passes.
template <class W>
void cgsr(int64_t n, int j, const W* V, int64_t ldv, W* w, double* h, int passes, bool acc32) {
  std::vector<double> c(j);
  std::vector<W> cw(j);
  for (int i = 0; i < j; ++i) h[i] = 0.0;
  for (int p = 0; p < passes; ++p) {
    ORACLE_PAR
    for (int i = 0; i < j; ++i) c[i] = dot<W>(n, V + (int64_t)i * ldv, w, acc32);  // line 161
    for (int i = 0; i < j; ++i) cw[i] = rn<W>(c[i]);
    ORACLE_PAR
    for (int64_t l = 0; l < n; ++l) {                                                // line 162
      W acc = (W)0;
      for (int i = 0; i < j; ++i) {
        W t = V[(int64_t)i * ldv + l] * cw[i];
        acc = acc + t;
      }
      w[l] = w[l] - acc;
    }
    for (int i = 0; i < j; ++i) h[i] += c[i];                                        // line 163
  }
}

// v ← RN_W(w · RN_W(inv)), inv = 1/‖·‖ computed in fp64 (Alg. 1 lines 94, 105):
// the normalisation is a working-precision scal by the rounded reciprocal —
// inside the single-precision span of the mixed solver (
// DESIGN.md reading R21).  In fp64 mode RN_W is the identity.
template <class W>
void scale(int64_t n, const W* w, double inv, W* v) {
  const W iw = rn<W>(inv);
  ORACLE_PAR
  for (int64_t l = 0; l < n; ++l) v[l] = w[l] * iw;
}

// Back-substitution R y = s (Alg. 1, H⁻¹ s with H upper triangular
// after the rotations), fp64, k ascending inside each row.
int backsolve(int J, const double* R, int64_t ldr, const double* s, double* y) {
  for (int i = J - 1; i >= 0; --i) {
    double acc = s[i];
    for (int k = i + 1; k < J; ++k) acc = acc - R[(int64_t)k * ldr + i] * y[k];
    double d = R[(int64_t)i * ldr + i];
    if (d == 0.0) return ORACLE_ENONFINITE;
    y[i] = acc / d;
  }
  return 0;
}

// x ← x + V_J y (Alg. 1 line 147 with line 145's u = V_J y), fp64 (reading R8):
// u_l = Σ_i (double)v_il · y_i in fp64, i ascending, then x_l ← x_l + u_l.
template <class W>
void xupdate(int64_t n, int J, const W* V, int64_t ldv, const double* y, double* x, bool update32) {
  ORACLE_PAR
  for (int64_t l = 0; l < n; ++l) {
    double u = 0.0;
    for (int i = 0; i < J; ++i) u += (double)V[(int64_t)i * ldv + l] * y[i];
    if (update32) {
      float u32 = (float)u;
      x[l] = (double)((float)x[l] + u32);
    } else {
      x[l] = x[l] + u;
    }
  }
}

}  // namespace

extern "C" {

// ----------------------------------------------------------- components
void oracle_spmv64(int64_t n, const int32_t* rp, const int32_t* ci, const double* a, const double* x, double* y) {
  ORACLE_PAR
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) s += a[e] * x[ci[e]];
    y[i] = s;
  }
}

void oracle_spmv32(int64_t n, const int32_t* rp, const int32_t* ci, const float* a, const float* x, float* y) {
  ORACLE_PAR
  for (int64_t i = 0; i < n; ++i) {
    float s = 0.0f;
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) s = s + a[e] * x[ci[e]];
    y[i] = s;
  }
}

// Jacobi preconditioner M = diag(A) (reading R11): dinv_i = 1/a_ii in fp64.
int oracle_dinv(int64_t n, const int32_t* rp, const int32_t* ci, const double* a, double* dinv64, int64_t* bad_row) {
  for (int64_t i = 0; i < n; ++i) {
    double d = 0.0;
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e)
      if (ci[e] == i) d = a[e];
    if (d == 0.0 || !std::isfinite(d)) {
      if (bad_row) *bad_row = i;
      return ORACLE_EZERODIAG;
    }
    dinv64[i] = 1.0 / d;
  }
  return 0;
}

// "the matrix is stored twice": A32 = RN32(A64); overflow is an error.
int oracle_cast32(int64_t cnt, const double* in, float* out) {
  for (int64_t e = 0; e < cnt; ++e) {
    if (std::isfinite(in[e]) && std::fabs(in[e]) > (double)FLT_MAX) return ORACLE_EFP32RANGE;
    out[e] = (float)in[e];
  }
  return 0;
}

int oracle_ilu0(int prec, int64_t n, const int32_t* rp, const int32_t* ci, const void* aW, void* f, int64_t* bad_row) {
  const int64_t nnz = rp[n];
  int64_t bad;
  if (prec == ORACLE_MIXED) {
    std::memcpy(f, aW, sizeof(float) * nnz);
    bad = ilu0<float>(n, rp, ci, (float*)f);
  } else {
    std::memcpy(f, aW, sizeof(double) * nnz);
    bad = ilu0<double>(n, rp, ci, (double*)f);
  }
  if (bad_row) *bad_row = bad;
  return bad >= 0 ? ORACLE_EZERODIAG : ORACLE_OK;
}

void oracle_ilu0_apply(int prec, int64_t n, const int32_t* rp, const int32_t* ci, const void* f, const void* z,
                       void* out) {
  if (prec == ORACLE_MIXED) ilu0_apply<float>(n, rp, ci, (const float*)f, (const float*)z, (float*)out);
  else ilu0_apply<double>(n, rp, ci, (const double*)f, (const double*)z, (double*)out);
}

void oracle_jacobi_spmv(int prec, int64_t n, const int32_t* rp, const int32_t* ci, const void* aW,
                        const void* dinvW, const void* v, void* w) {
  if (prec == ORACLE_MIXED)
    jacobi_spmv<float>(n, rp, ci, (const float*)aW, (const float*)dinvW, (const float*)v, (float*)w);
  else
    jacobi_spmv<double>(n, rp, ci, (const double*)aW, (const double*)dinvW, (const double*)v, (double*)w);
}

// Alg. 1 lines 86–90: z = b − A x in fp64, then the cast of
// the residual to W and r = M⁻¹ z in W (reading R10:
// r_i = RN_W(dinvW_i · RN_W(z_i))).  Returns ‖z‖², ‖r‖² (fp64 accumulators).
int oracle_resid(int prec, int64_t n, const int32_t* rp, const int32_t* ci, const double* a64,
                 const double* b, const double* x, const void* dinvW, void* r, double* zz, double* rr) {
  double szz = 0.0, srr = 0.0;
  int err = 0;
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) s += a64[e] * x[ci[e]];
    double z = b[i] - s;
    if (!std::isfinite(z)) err = ORACLE_ENONFINITE;
    szz += z * z;
    if (prec == ORACLE_MIXED) {
      if (std::fabs(z) > (double)FLT_MAX && !err) err = ORACLE_EFP32RANGE;
      float z32 = (float)z;
      float ri = ((const float*)dinvW)[i] * z32;
      ((float*)r)[i] = ri;
      srr += (double)ri * (double)ri;
    } else {
      double ri = ((const double*)dinvW)[i] * z;
      ((double*)r)[i] = ri;
      srr += ri * ri;
    }
  }
  *zz = szz;
  *rr = srr;
  return err;
}

double oracle_dot(int prec, int64_t n, const void* x, const void* y) {
  if (prec == ORACLE_MIXED) return dot<float>(n, (const float*)x, (const float*)y, false);
  return dot<double>(n, (const double*)x, (const double*)y, false);
}

void oracle_mgs(int prec, int64_t n, int j, const void* V, int64_t ldv, void* w, double* h) {
  if (prec == ORACLE_MIXED) mgs<float>(n, j, (const float*)V, ldv, (float*)w, h, false);
  else mgs<double>(n, j, (const double*)V, ldv, (double*)w, h, false);
}

void oracle_cgsr(int prec, int64_t n, int j, const void* V, int64_t ldv, void* w, double* h, int passes) {
  if (prec == ORACLE_MIXED) cgsr<float>(n, j, (const float*)V, ldv, (float*)w, h, passes, false);
  else cgsr<double>(n, j, (const double*)V, ldv, (double*)w, h, passes, false);
}

void oracle_scale(int prec, int64_t n, const void* w, double inv, void* v) {
  if (prec == ORACLE_MIXED) scale<float>(n, (const float*)w, inv, (float*)v);
  else scale<double>(n, (const double*)w, inv, (double*)v);
}

// rotation_matrix (reading R4): ρ = hypot(a, b);
// b = 0 → (α, β) = (1, 0), ρ = a; else α = a/ρ, β = b/ρ.
void oracle_givens(double a, double b, double* c, double* s, double* rho) {
  if (b == 0.0) {
    *c = 1.0; *s = 0.0; *rho = a;
    return;
  }
  double r = std::hypot(a, b);
  *c = a / r; *s = b / r; *rho = r;
}

// Alg. 1 lines 108–140 for inner step j (1-based); h[0..j] is column j of H̄
// (h[i-1] = h_{i,j}); cs/sn hold α_i/β_i at [i-1]; s holds s_1.. at [0..].
double oracle_hess_step(int j, double* h, double* cs, double* sn, double* s) {
  for (int i = 1; i <= j - 1; ++i) {  // lines 108–117: apply Givens rotation i
    double t1 = h[i - 1], t2 = h[i];
    double a = cs[i - 1] * t1;
    double b = sn[i - 1] * t2;
    double c = -sn[i - 1] * t1;
    double d = cs[i - 1] * t2;
    h[i - 1] = a + b;
    h[i] = c + d;
  }
  double c, sgn, rho;
  oracle_givens(h[j - 1], h[j], &c, &sgn, &rho);  // lines 118–123
  cs[j - 1] = c;
  sn[j - 1] = sgn;
  double sj = s[j - 1];                            // lines 125–132
  s[j - 1] = c * sj;
  s[j] = -sgn * sj;
  h[j - 1] = rho;                                  // lines 133–140
  h[j] = 0.0;
  return std::fabs(s[j]);
}

int oracle_backsolve(int J, const double* R, int64_t ldr, const double* s, double* y) {
  return backsolve(J, R, ldr, s, y);
}

void oracle_xupdate(int prec, int64_t n, int J, const void* V, int64_t ldv, const double* y, double* x) {
  if (prec == ORACLE_MIXED) xupdate<float>(n, J, (const float*)V, ldv, y, x, false);
  else xupdate<double>(n, J, (const double*)V, ldv, y, x, false);
}

}  // extern "C"

namespace {

// One Arnoldi cycle: Alg. 1 lines 92–141.
// Restart conditions (reading R6 + R22): j = jmax, lucky breakdown,
// |s_{j+1}| ≤ thr, or — with stall_w > 0 — stall: the Arnoldi residual improved
// by less than a factor stall_factor over the last stall_w inner iterations
// (1.001 over 5 % of the restart length).
// Orthogonality-loss monitor (reading R23): U_k = strict upper
// part of V_kᵀV_k, S_k = (I + U_k)⁻¹ U_k, built one column per inner iteration:
// the new column of U is u_i = v_i·v_{k+1} (i ≤ k) and the new column of S is
// (I + U_k)⁻¹ u (unit upper-triangular back-substitution; S's leading block does
// not change).  ‖S‖_F accumulates over columns; ‖S‖₂ is estimated by 10 power
// iterations on SᵀS from x = (1,…,1)/√k.
struct OrthMonitor {
  int kind = 0;          // 0 Frobenius, 1 spectral (10 power iterations)
  double thresh = 1.0;   // restart when the norm reaches it
  int m = 0;
  std::vector<double> U, S;  // column-major (m+1)×(m+1)
  double fro2 = 0.0;
  void init(int m_) { m = m_; U.assign((size_t)(m + 1) * (m + 1), 0.0); S.assign(U.size(), 0.0); fro2 = 0.0; }
  double& u(int i, int l) { return U[(size_t)l * (m + 1) + i]; }
  double& sm(int i, int l) { return S[(size_t)l * (m + 1) + i]; }
  // append column l (0-based: basis vectors 0..l−1 against vector l); returns the norm estimate
  double append(int l, const double* ucol) {
    for (int i = 0; i < l; ++i) u(i, l) = ucol[i];
    for (int i = l - 1; i >= 0; --i) {  // (I + U_l) s = u, U_l = leading l×l block
      double t = ucol[i];
      for (int q = i + 1; q < l; ++q) t -= u(i, q) * sm(q, l);
      sm(i, l) = t;
    }
    for (int i = 0; i < l; ++i) fro2 += sm(i, l) * sm(i, l);
    if (kind == 0) return std::sqrt(fro2);
    const int k = l + 1;  // S is k×k (columns 0..l)
    std::vector<double> x(k, 1.0 / std::sqrt((double)k)), y(k);
    for (int it = 0; it < 10; ++it) {
      for (int i = 0; i < k; ++i) { double t = 0.0; for (int q = i + 1; q < k; ++q) t += sm(i, q) * x[q]; y[i] = t; }
      double nx = 0.0;
      for (int q = 0; q < k; ++q) { double t = 0.0; for (int i = 0; i < q; ++i) t += sm(i, q) * y[i]; x[q] = t; nx += t * t; }
      nx = std::sqrt(nx);
      if (nx == 0.0) return 0.0;
      for (int q = 0; q < k; ++q) x[q] /= nx;
    }
    double ny = 0.0;
    for (int i = 0; i < k; ++i) { double t = 0.0; for (int q = i + 1; q < k; ++q) t += sm(i, q) * x[q]; ny += t * t; }
    return std::sqrt(ny);
  }
};

template <class W>
int arnoldi(int ortho, int flags, int64_t n, const int32_t* rp, const int32_t* ci, const W* aW, const W* dinvW,
            const W* r, int m, double thr, W* V, int64_t ldv, double* Hbar, double* R, double* s, int32_t* Jout,
            int32_t* bd_out, double* inner_hist, int jmax = 0, int stall_w = 0, double stall_factor = 1.0,
            OrthMonitor* mon = nullptr, double* mon_hist = nullptr,
            const std::function<void(const W*, W*)>* ilu = nullptr) {
  if (jmax <= 0 || jmax > m) jmax = m;
  std::vector<double> sabs_hist(m + 1), ucol(mon ? m + 1 : 0);
  if (mon) mon->init(m);
  const bool acc32 = (flags & ORACLE_F_ACC32) != 0;
  const int passes = (flags & ORACLE_F_CGS1) ? 1 : 2;
  const int64_t ldh = m + 1;
  std::vector<double> cs(m), sn(m), h(m + 1);
  std::vector<W> w(n);
  // line 92: β ← ‖r‖₂ ; s_1 ← β (reading R1) ; v_1 ← r/β
  double beta = std::sqrt(dot<W>(n, r, r, acc32));
  if (!(beta > 0.0) || !std::isfinite(beta)) return ORACLE_ENONFINITE;
  for (int i = 0; i <= m; ++i) s[i] = 0.0;
  s[0] = beta;
  sabs_hist[0] = beta;
  scale<W>(n, r, 1.0 / beta, V);
  int J = 0, breakdown = 0;
  for (int j = 1; j <= m; ++j) {  // lines 98–99
    const W* vj = V + (int64_t)(j - 1) * ldv;
    if (ilu) {  // line 100 with M = LU (reading R24): t = A_W v_j (row sums in W), w = U⁻¹L⁻¹t
      std::vector<W> t(n);
      ORACLE_PAR
      for (int64_t i = 0; i < n; ++i) {
        W acc = 0;
        for (int64_t e = rp[i]; e < rp[i + 1]; ++e) acc = acc + aW[e] * vj[ci[e]];
        t[i] = acc;
      }
      (*ilu)(t.data(), w.data());
    } else {
      jacobi_spmv<W>(n, rp, ci, aW, dinvW, vj, w.data());  // line 100
    }
    for (int i = 0; i <= m; ++i) h[i] = 0.0;
    if (ortho == ORACLE_MGS) mgs<W>(n, j, V, ldv, w.data(), h.data(), acc32);  // line 101
    else cgsr<W>(n, j, V, ldv, w.data(), h.data(), passes, acc32);
    double hn = std::sqrt(dot<W>(n, w.data(), w.data(), acc32));  // line 104
    if (!std::isfinite(hn)) return ORACLE_ENONFINITE;
    h[j] = hn;
    if (hn == 0.0) breakdown = 1;  // lucky breakdown (reading R14)
    else scale<W>(n, w.data(), 1.0 / hn, V + (int64_t)j * ldv);  // line 105
    for (int i = 0; i <= j; ++i) Hbar[(int64_t)(j - 1) * ldh + i] = h[i];
    double sabs = oracle_hess_step(j, h.data(), cs.data(), sn.data(), s);  // lines 108–140
    for (int i = 0; i <= j; ++i) R[(int64_t)(j - 1) * ldh + i] = h[i];
    if (inner_hist) inner_hist[j - 1] = sabs / beta;
    sabs_hist[j] = sabs;
    J = j;
    const bool stall = stall_w > 0 && j >= stall_w && sabs * stall_factor > sabs_hist[j - stall_w];
    bool orth = false;
    if (mon && !breakdown) {  // column j of U: v_i · v_{j+1}, i = 1..j (fp64 accumulation)
      const W* vn = V + (int64_t)j * ldv;
      ORACLE_PAR
      for (int i = 0; i < j; ++i) ucol[i] = dot<W>(n, V + (int64_t)i * ldv, vn, false);
      const double sn = mon->append(j, ucol.data());
      if (mon_hist) mon_hist[j - 1] = sn;
      orth = sn >= mon->thresh;
    }
    if (j == jmax || breakdown || sabs <= thr || stall || orth) break;  // restart (readings R6, R22, R23)
  }
  *Jout = J;
  *bd_out = breakdown;
  return 0;
}

}  // namespace

extern "C" int oracle_arnoldi(int prec, int ortho, int flags, int64_t n, const int32_t* rp, const int32_t* ci,
                              const void* aW, const void* dinvW, const void* r, int m, double thr, void* V,
                              int64_t ldv, double* Hbar, double* R, double* s, int32_t* J, int32_t* breakdown,
                              double* inner_hist) {
  if (prec == ORACLE_MIXED)
    return arnoldi<float>(ortho, flags, n, rp, ci, (const float*)aW, (const float*)dinvW, (const float*)r, m, thr,
                          (float*)V, ldv, Hbar, R, s, J, breakdown, inner_hist);
  return arnoldi<double>(ortho, flags, n, rp, ci, (const double*)aW, (const double*)dinvW, (const double*)r, m, thr,
                         (double*)V, ldv, Hbar, R, s, J, breakdown, inner_hist);
}

namespace {

template <class W>
int solve(int64_t n, const int32_t* rp, const int32_t* ci, const double* a, const double* b, const double* x0,
          double* x, int m, double tol, int ortho, double delta, int max_cycles, int flags, oracle_result* res,
          double* history, int32_t history_cap, double* inner, int32_t inner_cap, int policy = 0,
          double stall_factor = 1.001, double stall_frac = 0.05, int orth_kind = 0, double orth_thresh = 1.0,
          double* orth_hist = nullptr, int32_t orth_cap = 0) {
  const bool mixed = sizeof(W) == 4;
  const bool resid32 = (flags & ORACLE_F_RESID32) != 0;
  const bool update32 = (flags & ORACLE_F_UPDATE32) != 0;
  const int64_t nnz = rp[n];
  // setup: Jacobi M⁻¹ (reading R11) and the working-precision copy of A
  std::vector<double> dinv64(n);
  if (oracle_dinv(n, rp, ci, a, dinv64.data(), nullptr) != 0) return ORACLE_EZERODIAG;
  std::vector<W> aW(nnz), dinvW(n);
  for (int64_t e = 0; e < nnz; ++e) {
    if (mixed && std::fabs(a[e]) > (double)FLT_MAX) return ORACLE_EFP32RANGE;
    aW[e] = (W)a[e];
  }
  ORACLE_PAR
  for (int64_t i = 0; i < n; ++i) dinvW[i] = (W)dinv64[i];
  // ILU(0) preconditioner (§8 f2, reading R24): factors in W from A_W, or in
  // fp32 from RN32(A64) inside the fp64 solver ("single-precision ILU")
  std::vector<W> fW;
  std::vector<float> f32, t32a, t32b;
  std::function<void(const W*, W*)> pc;
  if (flags & ORACLE_F_ILU0) {
    fW = aW;
    if (ilu0<W>(n, rp, ci, fW.data()) >= 0) return ORACLE_EZERODIAG;
    pc = [&](const W* in, W* out) { ilu0_apply<W>(n, rp, ci, fW.data(), in, out); };
  } else if (flags & ORACLE_F_ILU32) {
    if (mixed) return ORACLE_EINVAL;
    f32.resize(nnz); t32a.resize(n); t32b.resize(n);
    for (int64_t e = 0; e < nnz; ++e) {
      if (std::fabs(a[e]) > (double)FLT_MAX) return ORACLE_EFP32RANGE;
      f32[e] = (float)a[e];
    }
    if (ilu0<float>(n, rp, ci, f32.data()) >= 0) return ORACLE_EZERODIAG;
    pc = [&](const W* in, W* out) {
      for (int64_t i = 0; i < n; ++i) t32a[i] = (float)in[i];
      ilu0_apply<float>(n, rp, ci, f32.data(), t32a.data(), t32b.data());
      for (int64_t i = 0; i < n; ++i) out[i] = (W)t32b[i];
    };
  }
  const std::function<void(const W*, W*)>* pcp = pc ? &pc : nullptr;
  std::vector<W> rz(pcp ? n : 0);
  std::vector<float> a32;  // resid32 ablation only
  if (resid32) { a32.resize(nnz); for (int64_t e = 0; e < nnz; ++e) a32[e] = (float)a[e]; }

  double nb = 0.0;
  for (int64_t i = 0; i < n; ++i) nb += b[i] * b[i];
  nb = std::sqrt(nb);
  res->cycles = 0; res->inner_iters = 0; res->history_len = 0; res->inner_len = 0; res->final_relres = 0.0;
  if (nb == 0.0) {  // b = 0 → x = 0 (reading R13)
    for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
    if (history_cap > 0) history[0] = 0.0;
    res->history_len = 1;
    return ORACLE_OK;
  }
  for (int64_t i = 0; i < n; ++i) x[i] = x0 ? x0[i] : 0.0;
  if (update32) for (int64_t i = 0; i < n; ++i) x[i] = (double)(float)x[i];

  const int64_t ldv = n;
  std::vector<W> V((size_t)n * (m + 1)), r(n);
  std::vector<double> zrow(n), zuse_row(n);
  std::vector<double> Hbar((size_t)(m + 1) * m), R((size_t)(m + 1) * m), s(m + 1), y(m), ih(m);
  int k = 0, total_inner = 0, J1 = 0;
  const int stall_w = policy == ORACLE_POLICY_STALL ? std::max(1, (int)std::ceil(stall_frac * m)) : 0;
  OrthMonitor mon;
  mon.kind = orth_kind;
  mon.thresh = orth_thresh;
  std::vector<double> mh(m);
  for (;;) {
    // line 86: z_k ← b − A x_k (fp64); line 90: r_k ← M⁻¹ z_k
    // in W after casting the residual (reading R10).
    // rows (independent), then ‖z‖² and the error checks in row order
    ORACLE_PAR
    for (int64_t i = 0; i < n; ++i) {
      double sacc = 0.0;
      for (int64_t e = rp[i]; e < rp[i + 1]; ++e) sacc += a[e] * x[ci[e]];
      double zi = b[i] - sacc;
      zrow[i] = zi;
      double zuse = zi;
      if (resid32) {  // ablation: the same residual formed in fp32 arithmetic
        float s32 = 0.0f;
        for (int64_t e = rp[i]; e < rp[i + 1]; ++e) s32 = s32 + a32[e] * (float)x[ci[e]];
        zuse = (double)((float)b[i] - s32);
      }
      zuse_row[i] = zuse;
      if (pcp) rz[i] = (W)zuse;
      else r[i] = dinvW[i] * (W)zuse;
    }
    double zz = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const double zi = zrow[i];
      if (!std::isfinite(zi)) return ORACLE_ENONFINITE;
      zz += zi * zi;
      if (mixed && std::fabs(zuse_row[i]) > (double)FLT_MAX) return ORACLE_EFP32RANGE;
    }
    if (pcp) (*pcp)(rz.data(), r.data());  // line 90 with M = LU (reading R24)
    double znorm = std::sqrt(zz);
    double rho = znorm / nb;
    if (res->history_len < history_cap) history[res->history_len] = rho;
    res->history_len++;
    res->final_relres = rho;
    // line 88: stop when ‖z_k‖/‖b‖ ≤ tol (reading R5)
    if (rho <= tol) { res->cycles = k; res->inner_iters = total_inner; return ORACLE_OK; }
    if (k >= max_cycles) { res->cycles = k; res->inner_iters = total_inner; return ORACLE_NOT_CONVERGED; }
    // restart condition threshold (reading R6): |s_{j+1}| ≤ β·max(tol‖b‖/‖z_k‖, δ)
    double beta = std::sqrt(dot<W>(n, r.data(), r.data(), (flags & ORACLE_F_ACC32) != 0));
    double need = tol * nb / znorm;
    // two-stage policy (reading R22): after the first cycle,
    // restart at the first cycle's iteration count instead of the δ test
    const bool repeat = policy == ORACLE_POLICY_TWOSTAGE && k > 0;
    double thr = beta * std::fmax(need, repeat ? 0.0 : delta);
    int32_t J = 0, bd = 0;
    int rc = arnoldi<W>(ortho, flags, n, rp, ci, aW.data(), dinvW.data(), r.data(), m, thr, V.data(), ldv,
                        Hbar.data(), R.data(), s.data(), &J, &bd, ih.data(), repeat ? J1 : m, stall_w, stall_factor,
                        policy == ORACLE_POLICY_ORTHLOSS ? &mon : nullptr, mh.data(), pcp);
    if (rc != 0) return rc;
    if (policy == ORACLE_POLICY_ORTHLOSS && orth_hist)
      for (int t = 0; t < J; ++t)
        if (res->inner_len + t < orth_cap) orth_hist[res->inner_len + t] = mh[t];
    if (k == 0) J1 = J;
    for (int t = 0; t < J; ++t) {
      if (res->inner_len < inner_cap) inner[res->inner_len] = ih[t];
      res->inner_len++;
    }
    total_inner += J;
    // line 145: y = H⁻¹ s ; u = V_J y ; line 147: x ← x + u (fp64)
    if (backsolve(J, R.data(), m + 1, s.data(), y.data()) != 0) return ORACLE_ENONFINITE;
    xupdate<W>(n, J, V.data(), ldv, y.data(), x, update32);
    ++k;
  }
}

}  // namespace

extern "C" int oracle_gmres_solve_policy(int64_t n, const int32_t* rp, const int32_t* ci, const double* a,
                                         const double* b, const double* x0, double* x, int m, double tol, int ortho,
                                         int prec, double delta, int max_cycles, int flags, oracle_result* res,
                                         double* history, int32_t history_cap, double* inner, int32_t inner_cap,
                                         int policy, double stall_factor, double stall_frac);

extern "C" int oracle_gmres_solve(int64_t n, const int32_t* rp, const int32_t* ci, const double* a, const double* b,
                                  const double* x0, double* x, int m, double tol, int ortho, int prec, double delta,
                                  int max_cycles, int flags, oracle_result* res, double* history,
                                  int32_t history_cap, double* inner, int32_t inner_cap) {
  return oracle_gmres_solve_policy(n, rp, ci, a, b, x0, x, m, tol, ortho, prec, delta, max_cycles, flags, res,
                                   history, history_cap, inner, inner_cap, ORACLE_POLICY_THRESHOLD, 1.001, 0.05);
}

extern "C" int oracle_gmres_solve_policy(int64_t n, const int32_t* rp, const int32_t* ci, const double* a,
                                         const double* b, const double* x0, double* x, int m, double tol, int ortho,
                                         int prec, double delta, int max_cycles, int flags, oracle_result* res,
                                         double* history, int32_t history_cap, double* inner, int32_t inner_cap,
                                         int policy, double stall_factor, double stall_frac) {
  return oracle_gmres_solve_orth(n, rp, ci, a, b, x0, x, m, tol, ortho, prec, delta, max_cycles, flags, res, history,
                                 history_cap, inner, inner_cap, policy, stall_factor, stall_frac, 0, 1.0, nullptr, 0);
}

extern "C" int oracle_gmres_solve_orth(int64_t n, const int32_t* rp, const int32_t* ci, const double* a,
                                       const double* b, const double* x0, double* x, int m, double tol, int ortho,
                                       int prec, double delta, int max_cycles, int flags, oracle_result* res,
                                       double* history, int32_t history_cap, double* inner, int32_t inner_cap,
                                       int policy, double stall_factor, double stall_frac, int orth_kind,
                                       double orth_thresh, double* orth_hist, int32_t orth_cap) {
  // StallDetect's factor must exceed 1 (1.001): with 1 the stall test never fires
  if (policy < 0 || policy > 3 || !(stall_factor > 1.0) || !(stall_frac > 0.0)) return ORACLE_EINVAL;
  if (orth_kind < 0 || orth_kind > 1 || !(orth_thresh > 0.0)) return ORACLE_EINVAL;
  if (n < 1 || m < 1 || !(tol > 0.0) || !(delta >= 0.0) || max_cycles < 0) return ORACLE_EINVAL;
  if (rp[0] != 0) return ORACLE_EBADCSR;
  for (int64_t i = 0; i < n; ++i) {
    if (rp[i + 1] < rp[i]) return ORACLE_EBADCSR;
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
      if (ci[e] < 0 || ci[e] >= n) return ORACLE_EBADCSR;
      if (e > rp[i] && ci[e] <= ci[e - 1]) return ORACLE_EBADCSR;
    }
  }
  if (prec == ORACLE_MIXED)
    return solve<float>(n, rp, ci, a, b, x0, x, m, tol, ortho, delta, max_cycles, flags, res, history, history_cap,
                        inner, inner_cap, policy, stall_factor, stall_frac, orth_kind, orth_thresh, orth_hist,
                        orth_cap);
  return solve<double>(n, rp, ci, a, b, x0, x, m, tol, ortho, delta, max_cycles, flags, res, history, history_cap,
                       inner, inner_cap, policy, stall_factor, stall_frac, orth_kind, orth_thresh, orth_hist,
                       orth_cap);
}
