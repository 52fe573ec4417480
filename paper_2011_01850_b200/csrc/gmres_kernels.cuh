// gmres_kernels.cuh — sm_100a device code for mixed-precision restarted GMRES(m).
//
// One persistent cooperative kernel runs the WHOLE restarted solve (Alg. 1,
// PAPER.md:78-167): every CTA owns a contiguous row block [r0, r1) of every
// n-vector and of every column of V, and the only cross-CTA traffic is
//   * the gather of v_j / x in the SpMV (after a grid barrier), and
//   * deterministic grid all-reduces of fp64 partial sums (dots and norms).
// Givens rotations, the exit test and s are replicated in every CTA from
// bit-identical reduced inputs (so every CTA takes the same branch); CTA 0
// keeps R for the back-substitution.
//
// W is the working precision of Alg. 1 lines 89–146 (float in mixed mode,
// double in fp64 mode).  Element-wise W operations use the
// explicit _rn intrinsics (no FMA contraction) so that their rounding is the
// single W rounding per operation the oracle performs (R9/R10).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <float.h>

namespace g200 {

constexpr int NT = 512;        // threads per CTA (16 warps)
constexpr int NW = NT / 32;
constexpr int ROWALIGN = 32;   // row-partition granularity (128 B of fp32)
constexpr int LDALIGN = 64;    // leading dimension of V (256 B of fp32)

enum { ST_OK = 0, ST_NOT_CONVERGED = 1, ST_EFP32RANGE = -4, ST_ENONFINITE = -5, ST_ETIMEOUT = -8 };
enum { ERRF_RANGE = 1, ERRF_NONFINITE = 2 };
enum { PH_RESID = 0, PH_SPMV = 1, PH_ORTHO = 2, PH_GIVENS = 3, PH_UPDATE = 4, PH_N = 8 };

struct Dev {
  int n;            // rows
  int m;            // max inner iterations per cycle
  int G;            // CTAs in the grid
  int kmax;         // m + 1 (stride of the partial buffers)
  int ortho;        // 0 MGS, 1 CGSR
  int tile_bytes;   // shared bytes reserved for V tiles
  const int* rp;
  const int* ci;
  const double* a64;
  const void* aW;       // W copy of A's values (== a64 in fp64 mode)
  const void* dinvW;    // W copy of 1/a_ii
  const double* b;
  double* x;
  void* V;              // column-major, ldv rows, m+1 columns (W)
  long long ldv;
  void* w0;             // ping-pong work vectors (W, ldv rows, zero padding)
  void* w1;
  double* partials;     // [2][G][kmax]
  double* R;            // rotated Hessenberg, (m+1) x m, ld m+1 (CTA 0)
  double* y;            // m
  unsigned long long* bar;
  int* abort_flag;
  int* err_flag;
  const int* row_begin; // G+1 row boundaries (multiples of ROWALIGN, last = nvec)
  double tol, delta;
  int max_cycles;
  double* history; int hist_cap;
  double* inner_hist; int inner_cap;
  int* out_int;         // [0] status [1] cycles [2] inner iters [3] history len [4] inner len
  double* out_dbl;      // [0] final relres
  unsigned long long* prof;   // [PH_N] ns accumulated by CTA 0
  long long timeout_ns;
};

// ------------------------------------------------------------ primitives
template <class W> struct VecT;
template <> struct VecT<float> { using T = float4; static constexpr int N = 4; };
template <> struct VecT<double> { using T = double2; static constexpr int N = 2; };

__device__ __forceinline__ float rnw(double v, float*) { return __double2float_rn(v); }
__device__ __forceinline__ double rnw(double v, double*) { return v; }
template <class W> __device__ __forceinline__ W RN(double v) { return rnw(v, (W*)nullptr); }

__device__ __forceinline__ float mulw(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mulw(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float addw(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double addw(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float subw(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double subw(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// per-CTA control block in static shared memory
struct Shm {
  unsigned long long epoch;   // grid barriers passed by this CTA
  int red_epoch;              // all-reduces done (selects the partial slot)
  int abort;
  int flag;
  int status;
  double bc[4];
  double red[NW * 2];
};

// Grid-wide barrier over the co-resident (cooperative) grid: monotone 64-bit
// arrival counter, release/acquire through __threadfence + atomics.  A device
// watchdog (globaltimer) aborts every CTA instead of hanging the GPU.
__device__ __forceinline__ bool grid_sync(const Dev& d, Shm& sh) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long target = (sh.epoch += 1ull) * (unsigned long long)d.G;
    __threadfence();
    atomicAdd(d.bar, 1ull);
    int ab = 0;
    unsigned long long t0 = 0;
    unsigned it = 0;
    while (ld_acquire_u64(d.bar) < target) {
      if (((++it) & 1023u) == 0u) {
        if (*(volatile int*)d.abort_flag) { ab = 1; break; }
        const unsigned long long t = globaltimer();
        if (t0 == 0) t0 = t;
        else if ((long long)(t - t0) > d.timeout_ns) { atomicExch(d.abort_flag, 1); ab = 1; break; }
      }
    }
    __threadfence();
    sh.abort = ab;
  }
  __syncthreads();
  return sh.abort == 0;
}

// Block sum of K doubles (deterministic: warp tree, then warps in order).
template <int K>
__device__ __forceinline__ void block_sum(double (&v)[K], Shm& sh, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double s = warp_sum(v[k]);
    if (lane == 0) sh.red[warp * K + k] = s;
  }
  __syncthreads();
  if (threadIdx.x < K) {
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += sh.red[w * K + threadIdx.x];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

// Grid all-reduce of K fp64 values (s_part → s_out, both shared).  Every CTA
// sums the G partials in the same fixed order, so all CTAs hold bit-identical
// results (replicated control flow).
__device__ __forceinline__ bool grid_allreduce(const Dev& d, Shm& sh, const double* s_part, int K, double* s_out,
                                               double* s_tmp) {
  const int slot = sh.red_epoch & 1;
  double* P = d.partials + (size_t)slot * d.G * d.kmax;
  for (int k = threadIdx.x; k < K; k += NT) P[(size_t)blockIdx.x * d.kmax + k] = s_part[k];
  if (!grid_sync(d, sh)) return false;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k0 = 0; k0 < K; k0 += 32) {
    const int k = k0 + lane;
    if (k < K) {
      double acc = 0.0;
      for (int g = warp; g < d.G; g += NW) acc += __ldcg(P + (size_t)g * d.kmax + k);
      s_tmp[warp * d.kmax + k] = acc;
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += NT) {
    double acc = 0.0;
    for (int w = 0; w < NW; ++w) acc += s_tmp[w * d.kmax + k];
    s_out[k] = acc;
  }
  if (threadIdx.x == 0) sh.red_epoch++;
  __syncthreads();
  return true;
}

// ------------------------------------------------------------------ a1
// Alg. 1 lines 86–90: z = b − A64 x in fp64, then
// r = RN_W(dinv_W · RN_W(z)) (reading R10).  L lanes per row, fp64 row sums.
template <class W, int L>
__device__ void resid_rows(const Dev& d, int r0, int r1, W* __restrict__ r_out, double& zz, double& rr, double& bb,
                           int& err) {
  const int lane = threadIdx.x & (L - 1);
  const int rend = min(r1, d.n);
  const W* dinv = (const W*)d.dinvW;
  for (int base = r0 + (threadIdx.x >> 5) * (32 / L); base < rend; base += NT / L) {
    const int row = base + ((threadIdx.x & 31) / L);
    const bool act = row < rend;
    double acc = 0.0;
    if (act) {
      const int s = __ldg(d.rp + row), e = __ldg(d.rp + row + 1);
      for (int p = s + lane; p < e; p += L) acc += __ldg(d.a64 + p) * d.x[__ldg(d.ci + p)];
    }
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (act && lane == 0) {
      const double bi = d.b[row];
      bb += bi * bi;
      const double z = bi - acc;
      if (!isfinite(z)) err |= ERRF_NONFINITE;
      zz += z * z;
      if (sizeof(W) == 4 && fabs(z) > (double)FLT_MAX) err |= ERRF_RANGE;
      const W ri = mulw(__ldg(dinv + row), RN<W>(z));
      r_out[row] = ri;
      rr += (double)ri * (double)ri;
    }
  }
}

// ------------------------------------------------------------------ a2
// Alg. 1: w = RN_W(dinv_W ∘ (A_W v_j)), with v_j = RN_W(src · inv)
// formed on the fly from the unnormalised previous vector (line 105 fused
// into the gather: identical bits to normalising first).  L lanes per row.
template <class W, int L>
__device__ void spmv_rows(const Dev& d, int r0, int r1, const W* __restrict__ src, double inv, W* __restrict__ dst) {
  const int lane = threadIdx.x & (L - 1);
  const int rend = min(r1, d.n);
  const W* aW = (const W*)d.aW;
  const W* dinv = (const W*)d.dinvW;
  for (int base = r0 + (threadIdx.x >> 5) * (32 / L); base < rend; base += NT / L) {
    const int row = base + ((threadIdx.x & 31) / L);
    const bool act = row < rend;
    W acc = (W)0;
    if (act) {
      const int s = __ldg(d.rp + row), e = __ldg(d.rp + row + 1);
      for (int p = s + lane; p < e; p += L) {
        const W v = RN<W>((double)src[__ldg(d.ci + p)] * inv);
        acc = addw(acc, mulw(__ldg(aW + p), v));
      }
    }
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) acc = addw(acc, __shfl_xor_sync(0xffffffffu, acc, o));
    if (act && lane == 0) dst[row] = mulw(__ldg(dinv + row), acc);
  }
}

// own rows of the new basis column: V[:, j] = RN_W(src · inv) (Alg. 1)
template <class W>
__device__ void write_vcol(int r0, int r1, const W* __restrict__ src, double inv, W* __restrict__ vcol) {
  using V4 = typename VecT<W>::T;
  constexpr int N = VecT<W>::N;
  for (int q = r0 / N + threadIdx.x; q < r1 / N; q += NT) {
    V4 a = reinterpret_cast<const V4*>(src)[q];
    W* pa = reinterpret_cast<W*>(&a);
#pragma unroll
    for (int t = 0; t < N; ++t) pa[t] = RN<W>((double)pa[t] * inv);
    reinterpret_cast<V4*>(vcol)[q] = a;
  }
}

// ------------------------------------------------------------------ a3
// One fused MGS sweep over the CTA's rows:
//   w ← RN_W(w − RN_W(RN_W(h_prev)·v_prev))  (line 155 of step i−1), then
//   the partial of h_i = w·v_next (line 154 of step i), or of ‖w‖² when
//   v_next == nullptr (line 104).  fp64 accumulation (reading R9).
template <class W>
__device__ double mgs_sweep(int r0, int r1, W* __restrict__ w, const W* __restrict__ vprev, W hprev,
                            const W* __restrict__ vnext) {
  using V4 = typename VecT<W>::T;
  constexpr int N = VecT<W>::N;
  double acc = 0.0;
  for (int q = r0 / N + threadIdx.x; q < r1 / N; q += NT) {
    V4 a = reinterpret_cast<V4*>(w)[q];
    W* pa = reinterpret_cast<W*>(&a);
    if (vprev) {
      V4 b = reinterpret_cast<const V4*>(vprev)[q];
      const W* pb = reinterpret_cast<const W*>(&b);
#pragma unroll
      for (int t = 0; t < N; ++t) pa[t] = subw(pa[t], mulw(hprev, pb[t]));
      reinterpret_cast<V4*>(w)[q] = a;
    }
    if (vnext) {
      V4 c = reinterpret_cast<const V4*>(vnext)[q];
      const W* pc = reinterpret_cast<const W*>(&c);
#pragma unroll
      for (int t = 0; t < N; ++t) acc += (double)pa[t] * (double)pc[t];
    } else {
#pragma unroll
      for (int t = 0; t < N; ++t) acc += (double)pa[t] * (double)pa[t];
    }
  }
  return acc;
}

// ------------------------------------------------------------------ a4/a8
// Tiled passes over the CTA's rows with the V tile (T rows × ncols) staged in
// shared memory by cp.async (double-buffered), so each pass reads V once:
//   MODE 1: colacc_i += Σ_r V_ri w_r                       (CGS pass, line 161)
//   MODE 2: w ← RN_W(w − Σ_i V_i c_i), then colacc += Vᵀw   (line 162 + next line 161)
//   MODE 3: w ← RN_W(w − Σ_i V_i c_i), nn += ‖w‖²          (line 162 + line 104)
//   MODE 4: x_r += Σ_i (double)V_ri · y_i                   (lines 145–147, fp64)
// V·c is summed in W with i ascending (reading R2/R9); dots in fp64.
template <class W>
__device__ __forceinline__ int tile_rows(int ncols, int tile_bytes) {
  int T = tile_bytes / (2 * (ncols + 1) * (int)sizeof(W));
  T = (T / ROWALIGN) * ROWALIGN;
  if (T > 1024) T = 1024;
  if (T < ROWALIGN) T = ROWALIGN;
  return T;
}

template <class W, int MODE>
__device__ void tile_pass(const Dev& d, int r0, int r1, const W* __restrict__ V, long long ldv, int ncols,
                          W* __restrict__ w, const W* s_coefW, const double* s_y, double* s_colacc, double& nn,
                          char* s_tiles) {
  constexpr int N = VecT<W>::N;
  const int T = tile_rows<W>(ncols, d.tile_bytes);
  const int nrows = r1 - r0;
  if (nrows <= 0) return;
  const int ntiles = (nrows + T - 1) / T;
  const int stride = (ncols + 1) * T;  // W elements per buffer (V tile + w tile)
  W* buf0 = reinterpret_cast<W*>(s_tiles);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool has_w = MODE != 4;

  auto stage = [&](int t, W* sb) {
    const int t0 = r0 + t * T;
    const int cnt = min(T, r1 - t0);
    const int cpc = cnt / N;  // 16-byte chunks per column
    const int ncol_ld = ncols + (has_w ? 1 : 0);
    for (int idx = threadIdx.x; idx < ncol_ld * cpc; idx += NT) {
      const int c = idx / cpc, q = idx - c * cpc;
      const W* g = (c < ncols) ? (V + (long long)c * ldv + t0 + q * N) : (w + t0 + q * N);
      cp_async16(sb + c * T + q * N, g);
    }
  };

  stage(0, buf0);
  cp_async_commit();
  for (int t = 0; t < ntiles; ++t) {
    W* sb = buf0 + (t & 1) * stride;
    if (t + 1 < ntiles) {
      stage(t + 1, buf0 + ((t + 1) & 1) * stride);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int t0 = r0 + t * T;
    const int cnt = min(T, r1 - t0);
    W* sw = sb + ncols * T;
    if (MODE == 2 || MODE == 3) {
      for (int r = threadIdx.x; r < cnt; r += NT) {
        W acc = (W)0;
        for (int i = 0; i < ncols; ++i) acc = addw(acc, mulw(sb[i * T + r], s_coefW[i]));
        const W wn = subw(sw[r], acc);
        sw[r] = wn;
        w[t0 + r] = wn;
        if (MODE == 3) nn += (double)wn * (double)wn;
      }
      if (MODE == 2) __syncthreads();
    }
    if (MODE == 1 || MODE == 2) {
      for (int i = warp; i < ncols; i += NW) {
        double acc = 0.0;
        for (int r = lane; r < cnt; r += 32) acc += (double)sb[i * T + r] * (double)sw[r];
        acc = warp_sum(acc);
        if (lane == 0) s_colacc[i] += acc;
      }
    }
    if (MODE == 4) {
      for (int r = threadIdx.x; r < cnt; r += NT) {
        const int row = t0 + r;
        if (row < d.n) {
          double u = 0.0;
          for (int i = 0; i < ncols; ++i) u += (double)sb[i * T + r] * s_y[i];
          d.x[row] = d.x[row] + u;
        }
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ a6
// Alg. 1 lines 108–140 for step j (1-based) on h[0..j] (fp64, reading R4/R7):
// apply rotations 1..j−1, form rotation j, rotate s.  Returns |s_{j+1}|.
__device__ __forceinline__ double hess_step(int j, double* h, double* cs, double* sn, double* s) {
  for (int i = 1; i <= j - 1; ++i) {
    const double t1 = h[i - 1], t2 = h[i];
    const double c = cs[i - 1], sg = sn[i - 1];
    h[i - 1] = __dadd_rn(__dmul_rn(c, t1), __dmul_rn(sg, t2));
    h[i] = __dadd_rn(__dmul_rn(-sg, t1), __dmul_rn(c, t2));
  }
  const double a = h[j - 1], b = h[j];
  double c, sg, rho;
  if (b == 0.0) {
    c = 1.0; sg = 0.0; rho = a;
  } else {
    rho = hypot(a, b);
    c = a / rho;
    sg = b / rho;
  }
  cs[j - 1] = c;
  sn[j - 1] = sg;
  const double sj = s[j - 1];
  s[j - 1] = __dmul_rn(c, sj);
  s[j] = __dmul_rn(-sg, sj);
  h[j - 1] = rho;
  h[j] = 0.0;
  return fabs(s[j]);
}

// ------------------------------------------------------------------ a7
// Back-substitution R y = s_{1..J} (Alg. 1), column-oriented over the
// CTA; R (ld = ldr) read from global, s copied into s_rhs.
__device__ void backsolve_cta(int J, const double* R, int ldr, const double* s, double* s_rhs, double* y_out,
                              double* s_y) {
  for (int k = threadIdx.x; k < J; k += NT) s_rhs[k] = s[k];
  __syncthreads();
  for (int i = J - 1; i >= 0; --i) {
    if (threadIdx.x == 0) s_y[i] = s_rhs[i] / __ldcg(R + (size_t)i * ldr + i);
    __syncthreads();
    const double yi = s_y[i];
    for (int k = threadIdx.x; k < i; k += NT) s_rhs[k] = __dsub_rn(s_rhs[k], __dmul_rn(__ldcg(R + (size_t)i * ldr + k), yi));
    __syncthreads();
  }
  for (int k = threadIdx.x; k < J; k += NT) y_out[k] = s_y[k];
  __syncthreads();
}

// ---------------------------------------------------- shared-memory layout
struct SmemLayout {
  int kmax;
  size_t off_part, off_out, off_tmp, off_h, off_cs, off_sn, off_s, off_y, off_rhs, off_coef, off_tiles, total;
  __host__ __device__ SmemLayout(int kmax_, int tile_bytes) : kmax(kmax_) {
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o += (bytes + 15) & ~size_t(15); return r; };
    off_part = take(sizeof(double) * kmax);
    off_out = take(sizeof(double) * kmax);
    off_tmp = take(sizeof(double) * NW * kmax);
    off_h = take(sizeof(double) * (kmax + 1));
    off_cs = take(sizeof(double) * kmax);
    off_sn = take(sizeof(double) * kmax);
    off_s = take(sizeof(double) * (kmax + 1));
    off_y = take(sizeof(double) * kmax);
    off_rhs = take(sizeof(double) * kmax);
    off_coef = take(sizeof(double) * kmax);
    off_tiles = take((size_t)tile_bytes);
    total = o;
  }
};

// ---------------------------------------------------------- the solve
template <class W, int L>
__global__ void __launch_bounds__(NT, 1) solve_kernel(Dev d) {
  extern __shared__ __align__(16) char dsm[];
  __shared__ Shm sh;
  const SmemLayout lay(d.kmax, d.tile_bytes);
  double* s_part = reinterpret_cast<double*>(dsm + lay.off_part);
  double* s_out = reinterpret_cast<double*>(dsm + lay.off_out);
  double* s_tmp = reinterpret_cast<double*>(dsm + lay.off_tmp);
  double* s_h = reinterpret_cast<double*>(dsm + lay.off_h);
  double* s_cs = reinterpret_cast<double*>(dsm + lay.off_cs);
  double* s_sn = reinterpret_cast<double*>(dsm + lay.off_sn);
  double* s_s = reinterpret_cast<double*>(dsm + lay.off_s);
  double* s_y = reinterpret_cast<double*>(dsm + lay.off_y);
  double* s_rhs = reinterpret_cast<double*>(dsm + lay.off_rhs);
  W* s_coefW = reinterpret_cast<W*>(dsm + lay.off_coef);
  char* s_tiles = dsm + lay.off_tiles;

  if (threadIdx.x == 0) { sh.epoch = 0; sh.red_epoch = 0; sh.abort = 0; sh.flag = 0; sh.status = 0; }
  __syncthreads();

  const int r0 = d.row_begin[blockIdx.x], r1 = d.row_begin[blockIdx.x + 1];
  W* const wb0 = reinterpret_cast<W*>(d.w0);
  W* const wb1 = reinterpret_cast<W*>(d.w1);
  W* const V = reinterpret_cast<W*>(d.V);
  const long long ldv = d.ldv;
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  unsigned long long tprev = lead ? globaltimer() : 0ull;
  auto tick = [&](int ph) {
    if (lead) { const unsigned long long t = globaltimer(); d.prof[ph] += t - tprev; tprev = t; }
  };

  int k = 0, total_inner = 0, inner_len = 0, status = ST_OK;
  for (;;) {
    // ---------------- residual, stop test (Alg. 1 lines 86–92)
    double v3[3] = {0.0, 0.0, 0.0};
    int err = 0;
    resid_rows<W, L>(d, r0, r1, wb0, v3[0], v3[1], v3[2], err);
    if (err) atomicOr(d.err_flag, err);
    block_sum<3>(v3, sh, s_part);
    if (!grid_allreduce(d, sh, s_part, 3, s_out, s_tmp)) { status = ST_ETIMEOUT; break; }
    const double ZZ = s_out[0], RR = s_out[1], nb = sqrt(s_out[2]);
    const int ef = *(volatile int*)d.err_flag;
    if (nb == 0.0) {  // b = 0 → x = 0, no cycle (reading R13)
      for (int i = r0 + threadIdx.x; i < min(r1, d.n); i += NT) d.x[i] = 0.0;
      if (lead) { if (d.hist_cap > 0) d.history[0] = 0.0; d.out_int[3] = 1; d.out_dbl[0] = 0.0; }
      status = ST_OK;
      break;
    }
    const double rho = sqrt(ZZ) / nb;
    if (lead) {
      if (k < d.hist_cap) d.history[k] = rho;
      d.out_int[3] = k + 1;
      d.out_dbl[0] = rho;
    }
    tick(PH_RESID);
    if (ef & ERRF_NONFINITE || !isfinite(ZZ) || !isfinite(nb)) { status = ST_ENONFINITE; break; }
    if (ef & ERRF_RANGE) { status = ST_EFP32RANGE; break; }
    if (rho <= d.tol) { status = ST_OK; break; }
    if (k >= d.max_cycles) { status = ST_NOT_CONVERGED; break; }
    const double beta = sqrt(RR);
    if (!(beta > 0.0) || !isfinite(beta)) { status = ST_ENONFINITE; break; }
    const double thr = beta * fmax(d.tol * nb / sqrt(ZZ), d.delta);
    if (threadIdx.x == 0) {
      for (int i = 0; i <= d.m; ++i) s_s[i] = 0.0;
      s_s[0] = beta;
    }
    double inv = 1.0 / beta;
    W* src = wb0;
    W* dst = wb1;
    int J = 0;
    bool fail = false;
    for (int j = 1; j <= d.m; ++j) {
      // ------------ v_j (own rows) and w = M⁻¹ A v_j   (lines 100, 105)
      write_vcol<W>(r0, r1, src, inv, V + (long long)(j - 1) * ldv);
      spmv_rows<W, L>(d, r0, r1, src, inv, dst);
      __syncthreads();
      tick(PH_SPMV);
      // ------------ orthogonalise (line 101) and ‖w‖ (line 104)
      double NN;
      if (d.ortho == 0) {
        W hprev = (W)0;
        for (int i = 1; i <= j; ++i) {
          double p[1] = {mgs_sweep<W>(r0, r1, dst, i > 1 ? V + (long long)(i - 2) * ldv : nullptr, hprev,
                                      V + (long long)(i - 1) * ldv)};
          block_sum<1>(p, sh, s_part);
          if (!grid_allreduce(d, sh, s_part, 1, s_out, s_tmp)) { fail = true; break; }
          if (threadIdx.x == 0) s_h[i - 1] = s_out[0];
          hprev = RN<W>(s_out[0]);
        }
        if (fail) break;
        double p[1] = {mgs_sweep<W>(r0, r1, dst, V + (long long)(j - 1) * ldv, hprev, nullptr)};
        block_sum<1>(p, sh, s_part);
        if (!grid_allreduce(d, sh, s_part, 1, s_out, s_tmp)) { fail = true; break; }
        NN = s_out[0];
      } else {
        double nn = 0.0;
        for (int i = threadIdx.x; i < j; i += NT) s_part[i] = 0.0;
        __syncthreads();
        tile_pass<W, 1>(d, r0, r1, V, ldv, j, dst, s_coefW, s_y, s_part, nn, s_tiles);
        if (!grid_allreduce(d, sh, s_part, j, s_out, s_tmp)) { fail = true; break; }
        for (int i = threadIdx.x; i < j; i += NT) {
          s_h[i] = s_out[i];
          s_coefW[i] = RN<W>(s_out[i]);
          s_part[i] = 0.0;
        }
        __syncthreads();
        tile_pass<W, 2>(d, r0, r1, V, ldv, j, dst, s_coefW, s_y, s_part, nn, s_tiles);
        if (!grid_allreduce(d, sh, s_part, j, s_out, s_tmp)) { fail = true; break; }
        for (int i = threadIdx.x; i < j; i += NT) {
          s_h[i] = s_h[i] + s_out[i];
          s_coefW[i] = RN<W>(s_out[i]);
        }
        __syncthreads();
        nn = 0.0;
        tile_pass<W, 3>(d, r0, r1, V, ldv, j, dst, s_coefW, s_y, s_part, nn, s_tiles);
        double p[1] = {nn};
        block_sum<1>(p, sh, s_part);
        if (!grid_allreduce(d, sh, s_part, 1, s_out, s_tmp)) { fail = true; break; }
        NN = s_out[0];
      }
      tick(PH_ORTHO);
      // ------------ h_{j+1,j}, Givens, exit test (lines 104, 108–140, 98)
      const double hn = sqrt(NN);
      if (threadIdx.x == 0) {
        s_h[j] = hn;
        const double sabs = hess_step(j, s_h, s_cs, s_sn, s_s);
        if (blockIdx.x == 0) {
          for (int i = 0; i <= j; ++i) d.R[(size_t)(j - 1) * (d.m + 1) + i] = s_h[i];
          if (inner_len < d.inner_cap) d.inner_hist[inner_len] = sabs / beta;
        }
        sh.flag = (j == d.m) || (hn == 0.0) || (sabs <= thr) || !isfinite(hn);
      }
      __syncthreads();
      inner_len++;
      tick(PH_GIVENS);
      J = j;
      if (!isfinite(hn)) { status = ST_ENONFINITE; fail = true; break; }
      if (sh.flag) break;
      inv = 1.0 / hn;
      W* t = src; src = dst; dst = t;
    }
    if (fail) { if (status == ST_OK) status = ST_ETIMEOUT; break; }
    total_inner += J;
    // ------------ y = R⁻¹ s, x ← x + V_J y  (lines 143–147)
    if (blockIdx.x == 0) backsolve_cta(J, d.R, d.m + 1, s_s, s_rhs, d.y, s_y);
    if (!grid_sync(d, sh)) { status = ST_ETIMEOUT; break; }
    for (int i = threadIdx.x; i < J; i += NT) s_y[i] = __ldcg(d.y + i);
    __syncthreads();
    double dummy = 0.0;
    tile_pass<W, 4>(d, r0, r1, V, ldv, J, nullptr, s_coefW, s_y, s_part, dummy, s_tiles);
    if (!grid_sync(d, sh)) { status = ST_ETIMEOUT; break; }
    tick(PH_UPDATE);
    ++k;
  }
  if (lead) {
    d.out_int[0] = status;
    d.out_int[1] = k;
    d.out_int[2] = total_inner;
    d.out_int[4] = inner_len;
  }
}

// ------------------------------------------------------ setup kernels
// a0: A32 = RN32(A64), overflow flagged.
__global__ void cast32_kernel(const double* __restrict__ a, float* __restrict__ o, long long cnt, int* err) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < cnt; e += (long long)gridDim.x * blockDim.x) {
    const double v = a[e];
    if (isfinite(v) && fabs(v) > (double)FLT_MAX) atomicOr(err, ERRF_RANGE);
    o[e] = __double2float_rn(v);
  }
}

// Jacobi M = diag(A) (reading R11): dinv64 = 1/a_ii (fp64), dinv32 = RN32(dinv64).
__global__ void dinv_kernel(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                            const double* __restrict__ a, double* dinv64, float* dinv32, int* bad_row) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double dg = 0.0;
    for (int p = rp[i]; p < rp[i + 1]; ++p)
      if (ci[p] == i) dg = a[p];
    if (dg == 0.0 || !isfinite(dg)) {
      atomicMin(bad_row, i);
      dinv64[i] = 0.0;
      dinv32[i] = 0.0f;
    } else {
      const double inv = 1.0 / dg;
      dinv64[i] = inv;
      dinv32[i] = __double2float_rn(inv);
    }
  }
}

// ------------------------------------------------- component kernels
// Each runs the same device functions as solve_kernel for one step.
template <class W, int L>
__global__ void __launch_bounds__(NT, 1) k_spmv_kernel(Dev d, const W* v, W* w) {
  const int r0 = d.row_begin[blockIdx.x], r1 = d.row_begin[blockIdx.x + 1];
  spmv_rows<W, L>(d, r0, r1, v, 1.0, w);
}

template <class W, int L>
__global__ void __launch_bounds__(NT, 1) k_resid_kernel(Dev d, W* r, double* out2) {
  extern __shared__ __align__(16) char dsm[];
  __shared__ Shm sh;
  const SmemLayout lay(d.kmax, d.tile_bytes);
  double* s_part = reinterpret_cast<double*>(dsm + lay.off_part);
  double* s_out = reinterpret_cast<double*>(dsm + lay.off_out);
  double* s_tmp = reinterpret_cast<double*>(dsm + lay.off_tmp);
  if (threadIdx.x == 0) { sh.epoch = 0; sh.red_epoch = 0; sh.abort = 0; }
  __syncthreads();
  const int r0 = d.row_begin[blockIdx.x], r1 = d.row_begin[blockIdx.x + 1];
  double v2[2] = {0.0, 0.0}, bb = 0.0;
  int err = 0;
  resid_rows<W, L>(d, r0, r1, r, v2[0], v2[1], bb, err);
  if (err) atomicOr(d.err_flag, err);
  block_sum<2>(v2, sh, s_part);
  if (!grid_allreduce(d, sh, s_part, 2, s_out, s_tmp)) return;
  if (blockIdx.x == 0 && threadIdx.x < 2) out2[threadIdx.x] = s_out[threadIdx.x];
}

template <class W>
__global__ void __launch_bounds__(NT, 1) k_ortho_kernel(Dev d, int j, const W* V, long long ldv, W* w, double* hout) {
  extern __shared__ __align__(16) char dsm[];
  __shared__ Shm sh;
  const SmemLayout lay(d.kmax, d.tile_bytes);
  double* s_part = reinterpret_cast<double*>(dsm + lay.off_part);
  double* s_out = reinterpret_cast<double*>(dsm + lay.off_out);
  double* s_tmp = reinterpret_cast<double*>(dsm + lay.off_tmp);
  double* s_h = reinterpret_cast<double*>(dsm + lay.off_h);
  double* s_y = reinterpret_cast<double*>(dsm + lay.off_y);
  W* s_coefW = reinterpret_cast<W*>(dsm + lay.off_coef);
  char* s_tiles = dsm + lay.off_tiles;
  if (threadIdx.x == 0) { sh.epoch = 0; sh.red_epoch = 0; sh.abort = 0; }
  __syncthreads();
  const int r0 = d.row_begin[blockIdx.x], r1 = d.row_begin[blockIdx.x + 1];
  double NN;
  if (d.ortho == 0) {
    W hprev = (W)0;
    for (int i = 1; i <= j; ++i) {
      double p[1] = {mgs_sweep<W>(r0, r1, w, i > 1 ? V + (long long)(i - 2) * ldv : nullptr, hprev,
                                  V + (long long)(i - 1) * ldv)};
      block_sum<1>(p, sh, s_part);
      if (!grid_allreduce(d, sh, s_part, 1, s_out, s_tmp)) return;
      if (threadIdx.x == 0) s_h[i - 1] = s_out[0];
      hprev = RN<W>(s_out[0]);
    }
    double p[1] = {mgs_sweep<W>(r0, r1, w, V + (long long)(j - 1) * ldv, hprev, nullptr)};
    block_sum<1>(p, sh, s_part);
    if (!grid_allreduce(d, sh, s_part, 1, s_out, s_tmp)) return;
    NN = s_out[0];
  } else {
    double nn = 0.0;
    for (int i = threadIdx.x; i < j; i += NT) s_part[i] = 0.0;
    __syncthreads();
    tile_pass<W, 1>(d, r0, r1, V, ldv, j, w, s_coefW, s_y, s_part, nn, s_tiles);
    if (!grid_allreduce(d, sh, s_part, j, s_out, s_tmp)) return;
    for (int i = threadIdx.x; i < j; i += NT) { s_h[i] = s_out[i]; s_coefW[i] = RN<W>(s_out[i]); s_part[i] = 0.0; }
    __syncthreads();
    tile_pass<W, 2>(d, r0, r1, V, ldv, j, w, s_coefW, s_y, s_part, nn, s_tiles);
    if (!grid_allreduce(d, sh, s_part, j, s_out, s_tmp)) return;
    for (int i = threadIdx.x; i < j; i += NT) { s_h[i] = s_h[i] + s_out[i]; s_coefW[i] = RN<W>(s_out[i]); }
    __syncthreads();
    nn = 0.0;
    tile_pass<W, 3>(d, r0, r1, V, ldv, j, w, s_coefW, s_y, s_part, nn, s_tiles);
    double p[1] = {nn};
    block_sum<1>(p, sh, s_part);
    if (!grid_allreduce(d, sh, s_part, 1, s_out, s_tmp)) return;
    NN = s_out[0];
  }
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < j; i += NT) hout[i] = s_h[i];
    if (threadIdx.x == 0) hout[j] = sqrt(NN);
  }
}

template <class W>
__global__ void __launch_bounds__(NT, 1) k_xupdate_kernel(Dev d, int J, const W* V, long long ldv, const double* y) {
  extern __shared__ __align__(16) char dsm[];
  const SmemLayout lay(d.kmax, d.tile_bytes);
  double* s_y = reinterpret_cast<double*>(dsm + lay.off_y);
  double* s_part = reinterpret_cast<double*>(dsm + lay.off_part);
  W* s_coefW = reinterpret_cast<W*>(dsm + lay.off_coef);
  char* s_tiles = dsm + lay.off_tiles;
  for (int i = threadIdx.x; i < J; i += NT) s_y[i] = y[i];
  __syncthreads();
  const int r0 = d.row_begin[blockIdx.x], r1 = d.row_begin[blockIdx.x + 1];
  double dummy = 0.0;
  tile_pass<W, 4>(d, r0, r1, V, ldv, J, nullptr, s_coefW, s_y, s_part, dummy, s_tiles);
}

// a6 + a7 on a given unrotated Hessenberg (tests): one CTA.
__global__ void __launch_bounds__(NT, 1) k_hess_kernel(int m, int J, const double* Hbar, double beta, double* R,
                                                     double* s, double* y) {
  extern __shared__ __align__(16) char dsm[];
  double* s_h = reinterpret_cast<double*>(dsm);
  double* s_cs = s_h + (m + 2);
  double* s_sn = s_cs + (m + 1);
  double* s_s = s_sn + (m + 1);
  double* s_rhs = s_s + (m + 2);
  double* s_y = s_rhs + (m + 1);
  if (threadIdx.x == 0) {
    for (int i = 0; i <= m; ++i) s_s[i] = 0.0;
    s_s[0] = beta;
    for (int j = 1; j <= J; ++j) {
      for (int i = 0; i <= j; ++i) s_h[i] = Hbar[(size_t)(j - 1) * (m + 1) + i];
      hess_step(j, s_h, s_cs, s_sn, s_s);
      for (int i = 0; i <= m; ++i) R[(size_t)(j - 1) * (m + 1) + i] = (i <= j) ? s_h[i] : 0.0;
    }
    for (int i = 0; i <= J; ++i) s[i] = s_s[i];
  }
  __syncthreads();
  backsolve_cta(J, R, m + 1, s_s, s_rhs, y, s_y);
}

}  // namespace g200
