// inputs/gen.cpp — seeded synthetic input generators (BASELINE.json configs C1–C5).
//
// This module is INPUT PLUMBING shared by the oracle tests, the GPU parity tests
// and bench.py.  It holds none of the GMRES method's arithmetic: it builds the
// CSR matrices, the random vectors, and b = A·x_true (the right-hand side that
// BASELINE.json prescribes; plain fp64 row sums written here independently of
// both oracle/ and the CUDA path).
//
// Readings (SURVEY.md §8(c) Q13/Q18–Q21):
//  * stencils: h = 1/(N+1), homogeneous Dirichlet (off-grid neighbours dropped),
//    lexicographic ordering with x fastest, central differences for β·∇u;
//    5-pt/7-pt: (1/h²)(2d·u_P − Σ u_N) + β_k (u_{+k} − u_{−k})/(2h);
//    27-pt: (1/(9h²))(26 u_P − Σ_{26} u_N) + the same central convection on the
//    6 face neighbours.
//  * random diagonally dominant (C3): row length k ~ P(k) ∝ k^−α on [kmin,kmax]
//    (k counts the diagonal), k−1 distinct uniform off-diagonal columns ≠ i,
//    values N(0,1), a_ii = 1.1·Σ|a_ij|.
//  * RNG: counter-based (splitmix64 of (seed, stream, index)); U[0,1) from the
//    top 53 bits; N(0,1) by Box–Muller.  Streams: 0 x_true/b, 1 row lengths,
//    2 columns, 3 values.  Deterministic for any thread count.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#include <algorithm>
#ifdef _OPENMP
#include <omp.h>
#endif

extern "C" {

static inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

uint64_t gen_hash(uint64_t seed, uint64_t stream, uint64_t index) {
  return splitmix64(splitmix64(splitmix64(seed) ^ (stream * 0xD1B54A32D192ED03ULL)) ^ index);
}

double gen_u01(uint64_t seed, uint64_t stream, uint64_t index) {
  return (double)(gen_hash(seed, stream, index) >> 11) * (1.0 / 9007199254740992.0);
}

double gen_normal(uint64_t seed, uint64_t stream, uint64_t index) {
  double u1 = gen_u01(seed, stream, 2 * index);
  double u2 = gen_u01(seed, stream, 2 * index + 1);
  return std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(6.283185307179586 * u2);
}

// out[i] = lo + (hi-lo)·U[0,1)(seed, stream, i)
void gen_uniform(int64_t n, uint64_t seed, uint64_t stream, double lo, double hi, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = lo + (hi - lo) * gen_u01(seed, stream, (uint64_t)i);
}

// ---------------------------------------------------------------- stencils
// kind ∈ {5, 7, 27}; N grid points per dimension.
int64_t gen_stencil_n(int kind, int64_t N) {
  return kind == 5 ? N * N : N * N * N;
}

int64_t gen_stencil_nnz(int kind, int64_t N) {
  if (kind == 5) return 5 * N * N - 4 * N;
  if (kind == 7) return 7 * N * N * N - 6 * N * N;
  if (kind == 27) return (3 * N - 2) * (3 * N - 2) * (3 * N - 2);
  return -1;
}

// Fills row_ptr[n+1], col[nnz], val[nnz].  beta[3] = (βx, βy, βz) (βz ignored for 5-pt).
// Returns 0 on success.
int gen_stencil(int kind, int64_t N, const double* beta, int32_t* row_ptr, int32_t* col, double* val) {
  if (!(kind == 5 || kind == 7 || kind == 27) || N < 2) return -1;
  const int dims = (kind == 5) ? 2 : 3;
  const int64_t n = gen_stencil_n(kind, N);
  const double h = 1.0 / (double)(N + 1);
  const double ih2 = 1.0 / (h * h);
  // per-row nnz, deterministic closed form per row (count in-grid neighbours)
  auto in = [&](int64_t c) { return c >= 0 && c < N; };
  std::vector<int32_t> cnt(n);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < n; ++r) {
    int64_t i = r % N, j = (r / N) % N, k = (dims == 3) ? r / (N * N) : 0;
    int c = 1;
    if (kind == 27) {
      for (int dk = -1; dk <= 1; ++dk)
        for (int dj = -1; dj <= 1; ++dj)
          for (int di = -1; di <= 1; ++di) {
            if (!di && !dj && !dk) continue;
            if (in(i + di) && in(j + dj) && in(k + dk)) ++c;
          }
    } else {
      c += in(i - 1) + in(i + 1) + in(j - 1) + in(j + 1);
      if (dims == 3) c += in(k - 1) + in(k + 1);
    }
    cnt[r] = c;
  }
  row_ptr[0] = 0;
  for (int64_t r = 0; r < n; ++r) row_ptr[r + 1] = row_ptr[r] + cnt[r];
  const double bx = beta[0], by = beta[1], bz = (dims == 3) ? beta[2] : 0.0;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < n; ++r) {
    int64_t i = r % N, j = (r / N) % N, k = (dims == 3) ? r / (N * N) : 0;
    int64_t e = row_ptr[r];
    if (kind == 27) {
      const double c9 = ih2 / 9.0;
      for (int dk = -1; dk <= 1; ++dk)
        for (int dj = -1; dj <= 1; ++dj)
          for (int di = -1; di <= 1; ++di) {
            if (!(in(i + di) && in(j + dj) && in(k + dk))) continue;
            int64_t c = (i + di) + N * ((j + dj) + N * (k + dk));
            double v;
            int nz = (di != 0) + (dj != 0) + (dk != 0);
            if (nz == 0) v = 26.0 * c9;
            else {
              v = -c9;
              if (nz == 1) {  // face neighbour: central convection
                if (di) v += di * bx / (2.0 * h);
                if (dj) v += dj * by / (2.0 * h);
                if (dk) v += dk * bz / (2.0 * h);
              }
            }
            col[e] = (int32_t)c; val[e] = v; ++e;
          }
    } else {
      // ascending column order: −z, −y, −x, P, +x, +y, +z
      const int64_t NN = N * N;
      if (dims == 3 && in(k - 1)) { col[e] = (int32_t)(r - NN); val[e] = -ih2 - bz / (2.0 * h); ++e; }
      if (in(j - 1)) { col[e] = (int32_t)(r - N); val[e] = -ih2 - by / (2.0 * h); ++e; }
      if (in(i - 1)) { col[e] = (int32_t)(r - 1); val[e] = -ih2 - bx / (2.0 * h); ++e; }
      col[e] = (int32_t)r; val[e] = 2.0 * dims * ih2; ++e;
      if (in(i + 1)) { col[e] = (int32_t)(r + 1); val[e] = -ih2 + bx / (2.0 * h); ++e; }
      if (in(j + 1)) { col[e] = (int32_t)(r + N); val[e] = -ih2 + by / (2.0 * h); ++e; }
      if (dims == 3 && in(k + 1)) { col[e] = (int32_t)(r + NN); val[e] = -ih2 + bz / (2.0 * h); ++e; }
    }
  }
  return 0;
}

// ---------------------------------------------------- random diag. dominant
// Row lengths: discrete power law on [kmin, kmax] by inverse CDF; writes
// row_ptr[n+1] and returns nnz (or -1).
int64_t gen_randdd_rowptr(int64_t n, uint64_t seed, double alpha, int kmin, int kmax, int32_t* row_ptr) {
  if (n < 1 || kmin < 1 || kmax < kmin) return -1;
  if (kmax > n) kmax = (int)n;
  if (kmin > kmax) kmin = kmax;
  const int K = kmax - kmin + 1;
  std::vector<double> cdf(K);
  double acc = 0.0;
  for (int t = 0; t < K; ++t) { acc += std::pow((double)(kmin + t), -alpha); cdf[t] = acc; }
  for (int t = 0; t < K; ++t) cdf[t] /= acc;
  std::vector<int32_t> len(n);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < n; ++r) {
    double u = gen_u01(seed, 1, (uint64_t)r);
    int t = (int)(std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
    if (t >= K) t = K - 1;
    len[r] = kmin + t;
  }
  int64_t s = 0;
  row_ptr[0] = 0;
  for (int64_t r = 0; r < n; ++r) {
    s += len[r];
    if (s > 2147483647LL) return -1;
    row_ptr[r + 1] = (int32_t)s;
  }
  return s;
}

// Fills col/val for the row_ptr from gen_randdd_rowptr.
int gen_randdd_fill(int64_t n, uint64_t seed, const int32_t* row_ptr, int32_t* col, double* val) {
  int err = 0;
#pragma omp parallel
  {
    std::vector<int64_t> cols;
#pragma omp for schedule(dynamic, 4096)
    for (int64_t r = 0; r < n; ++r) {
      const int k = row_ptr[r + 1] - row_ptr[r];
      cols.clear();
      uint64_t attempt = 0;
      while ((int)cols.size() < k - 1) {
        uint64_t h = gen_hash(seed, 2, ((uint64_t)r << 24) | attempt);
        ++attempt;
        int64_t c = (int64_t)(h % (uint64_t)n);
        if (c == r) continue;
        if (std::find(cols.begin(), cols.end(), c) != cols.end()) continue;
        cols.push_back(c);
        if (attempt > (1u << 23)) { err = -1; break; }
      }
      cols.push_back(r);
      std::sort(cols.begin(), cols.end());
      int64_t e0 = row_ptr[r];
      double offsum = 0.0;
      int64_t diag_e = -1;
      for (int t = 0; t < k; ++t) {
        col[e0 + t] = (int32_t)cols[t];
        if (cols[t] == r) { diag_e = e0 + t; continue; }
        double v = gen_normal(seed, 3, (uint64_t)(e0 + t));
        val[e0 + t] = v;
        offsum += std::fabs(v);
      }
      val[diag_e] = 1.1 * offsum;
      if (offsum == 0.0) val[diag_e] = 1.0;  // only if k == 1
    }
  }
  return err;
}

// b = A·x in fp64 (right-hand side construction for b = A·x_true).
void gen_matvec(int64_t n, const int32_t* row_ptr, const int32_t* col, const double* val, const double* x, double* b) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < n; ++r) {
    double s = 0.0;
    for (int64_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) s += val[e] * x[col[e]];
    b[r] = s;
  }
}

int gen_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

}  // extern "C"
