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
// Data movement: the CSR stream (row_ptr, col, val) and the V tiles are staged
// into shared memory by TMA bulk copies (cp.async.bulk + mbarrier, double
// buffered); threads only gather v_j / x and do arithmetic.
//
// W is the working precision of Alg. 1 lines 89–146 (float in mixed mode,
// double in fp64 mode).  Element-wise W operations use the
// explicit _rn intrinsics (no FMA contraction) so that their rounding is the
// single W rounding per operation the oracle performs (R9/R10);
// with one thread per row the SpMV row sums are even bit-identical to the
// oracle's (ascending column order).
#pragma once
#include <cuda_runtime.h>
#include <float.h>
#include <stdint.h>

namespace g200 {

constexpr int NT = 512;        // threads per CTA (16 warps)
constexpr int NW = NT / 32;
constexpr int ROWALIGN = 32;   // row-partition granularity (128 B of fp32)
constexpr int LDALIGN = 64;    // leading dimension of a caller's column-major V (component entry points)
constexpr int VEC_ALIGN = 256; // padded length of every n-vector (≥ the largest V block height)
constexpr int NGRP = NW;         // CSR-stream pipelines per CTA: one per warp
constexpr int GT = NT / NGRP;    // threads per pipeline (one warp)
constexpr int CHUNK_CAP = 256;   // max nnz of a TMA-staged CSR chunk
constexpr int CHUNK_RMAX = GT;   // max rows of a CSR chunk (multiple of 4)
constexpr int ST_OFF_RV = 160;                              // stage layout (bytes): row_ptr slice,
constexpr int ST_OFF_CI = ST_OFF_RV + CHUNK_RMAX * 8;       // 416: per-row operand slice (dinv),
constexpr int ST_OFF_A = ST_OFF_CI + (CHUNK_CAP + 8) * 4;   // 1472: col slice, then values
// per-warp TMA ring: NSTG(AT) stages of stage_bytes(AT) (fp32 values: 4 × 2528 B,
// fp64 values: 3 × 3584 B), i.e. 3 resp. 2 chunks in flight per warp while one
// is consumed (≈ 64–96 KB per SM: enough bytes in flight for HBM rate)
template <class AT> __host__ __device__ constexpr int NSTG() { return sizeof(AT) == 4 ? 4 : 3; }
template <class AT> __host__ __device__ constexpr int stage_bytes() { return ST_OFF_A + (CHUNK_CAP + 8) * (int)sizeof(AT); }
constexpr int MAXSTG = 4;
// block stream (short-row matrices): a ring of NBS per-CTA stages of BS_BYTES each
// (measured on C2, one solve each: 6 × 28 KB +23 %, 4 × 42 KB +6 %, 3 × 56 KB
// baseline, 2 × 72 KB −5 %, 2 × 80 KB −6.5 %, 2 × 84 KB −7 % mixed MGS / −5 % CGSR,
// 2 × 96 KB −4 % (less L1):
// the per-stage cost — refill hand-off, metadata, the first gathers — dominates)
constexpr int NBS = 2;
constexpr int BS_BYTES = 86016;
constexpr int BS_MAXROW = 64;  // longest row the block stream takes (else the chunk stream)
constexpr int TILE_BYTES = NGRP * 3 * (ST_OFF_A + (CHUNK_CAP + 8) * 8);  // 172032 (≥ the fp32 ring, 161792)
constexpr int MAX_M = 256;                               // restart length limit (shared-memory bound)
constexpr int ARR_PAD = 8;   // elements of slack after rp/col/val (TMA rounds up to 16 B)
constexpr int MAXR = 8;      // ranks (GPUs) of a row-partitioned solve
#ifndef G200_NTB
#define G200_NTB 2           // row-tile pass ring depth (rowtile_pass)
#endif

enum { ST_OK = 0, ST_NOT_CONVERGED = 1, ST_EFP32RANGE = -4, ST_ENONFINITE = -5, ST_ETIMEOUT = -8 };
enum { ERRF_RANGE = 1, ERRF_NONFINITE = 2 };
enum { PH_RESID = 0, PH_SPMV = 1, PH_ORTHO = 2, PH_GIVENS = 3, PH_UPDATE = 4, PH_N = 16 };
// profile-mode sub-phases of CGSR in prof[8..13]: pass1, red1, pass2, red2, pass3, red3

struct Dev {
  int n;            // rows
  int m;            // max inner iterations per cycle
  int G;            // CTAs in the grid
  int kmax;         // m + 1 (stride of the partial buffers)
  int ortho;        // 0 MGS, 1 CGSR
  int tile_bytes;   // shared bytes reserved for the staging region
  int soff[11];     // SmemLayout(kmax, tile_bytes) offsets (host-computed: each shared array is one
                    // add from the dynamic-smem base, cheap to rematerialise — solve_kernel keeps no
                    // shared pointers live in registers)
  const int* rp;
  const int* ci;
  const double* a64;
  const void* aW;       // W copy of A's values (== a64 in fp64 mode)
  const void* dinvW;    // W copy of 1/a_ii
  const double* b;
  double* x;
  void* V;              // Krylov basis, m+1 columns (W), layout below
  long long ldv;        // column-major: leading dimension (rows, ≥ n, multiple of 64)
  // row-blocked layout (CGSR solves, vtb > 0): block b holds rows
  // [b·vtb, (b+1)·vtb) of all m+1 columns, column c at V + b·vbs + c·vtp with
  // vtp = vtb + 16/w_B (padding: lanes reading one row group of different
  // columns hit distinct banks) and vbs = (m+1)·vtp, so a row tile of whole
  // blocks is one contiguous TMA copy per block (tools/tma_bench.cu: bulk copies
  // of ≤ 1 KB stream at ~4 TB/s, ≥ 4 KB at ~7 TB/s).  vtb == 0: column-major.
  int vtb, vtp, vtb_log;
  long long vbs;
  void* w0;             // ping-pong work vectors (W, ldv rows, zero padding)
  void* w1;
  // grid all-reduce (see grid_allreduce): this rank's partial array
  // [2][GG][kst] fp64 and arrival counter, and the same of every rank
  // (peer-mapped; [rank] is the local one) for the pushes and arrivals
  double* slots;
  double* slot_peer[MAXR];
  unsigned long long* ctr;
  unsigned long long* ctr_peer[MAXR];
  int kst;              // k stride of a slot row (kmax rounded to 4)
  long long s1off;      // one-value all-reduces: partials at slots + s1off + buf·GG + cta (contiguous)
  int GG;               // CTAs over all ranks (nranks * G)
  int cta0;             // global index of this rank's CTA 0 (rank * G)
  int nranks, rank;
  int sys_scope;        // != 0: peers are other GPUs (system-scope release/acquire)
  // row partition over ranks (§8 e): this rank owns global rows
  // [row_base, row_base + n); n-vectors are addressed by LOCAL row through
  // views into full-length buffers (w0, w1, x), CSR columns are GLOBAL, so a
  // gather reads view[col − row_base].  The rows a peer gathers are pushed
  // into that peer's buffer (vec_peer: global-index bases of every rank's w0,
  // w1, x) by the CTA owning them, before the release of the next all-reduce.
  long long row_base;
  int halo;             // != 0: push halo rows (nranks > 1)
  unsigned halo_full;   // bit q: rank q receives this rank's whole row blocks (contiguous pushes)
  // barrier epochs / all-reduce count at launch (row-partitioned solves keep
  // the arrival counters monotonic across launches instead of resetting them,
  // so no rank can wipe a faster rank's arrival); final values → epoch_out
  unsigned long long epoch0;
  int red0;
  unsigned long long* epoch_out;  // [0] barrier epochs, [1] all-reduces (CTA 0)
  void* vec_peer[3][MAXR];
  const int* send_off;  // [G+1] per-CTA ranges of the send list
  const int* send_row;  // local row to push
  const int* send_peer; // destination rank
  double* R;            // rotated Hessenberg, (m+1) x m, ld m+1 (CTA 0)
  double* y;            // m
  int* abort_flag;
  int* err_flag;
  const int* row_begin; // G+1 row boundaries (multiples of ROWALIGN, last = nvec)
  const int2* stages;   // block stream: per-CTA stages {row_begin, nnz_begin} + a sentinel
  const int* stage_off; // G+1 offsets into stages
  int block_stream;     // != 0: the CSR stream runs csr_block_stream (rows ≤ BS_MAXROW nnz)
  const int4* chunks;   // CSR chunks {row_begin, nnz_begin, direct, 0}; per CTA a sentinel
  const int* chunk_off; // G+1 offsets into chunks (CTA g: [off[g], off[g+1]-1) + sentinel)
  int merge_stream;     // != 0 (and not block_stream): the CSR stream runs csr_merge_stream
  const int4* mtiles;   // merge-path tiles {row_begin, nnz_begin, rows touched, 0}; per CTA a sentinel
  const int* mt_off;    // G+1 offsets into mtiles
  const int4* msplit;   // rows crossing a tile boundary {local row, first tile, last tile, 0}
  const int* ms_off;    // G+1 offsets into msplit
  double* mcarry;       // [2 · tiles] per-tile partial sums of the crossing rows
  double tol, delta;
  int max_cycles;
  int policy;           // restart policy (readings R22, R23): 0 threshold, 1 two-stage, 2 stall, 3 orth. loss
  double orth_thresh;   // policy 3: restart when ‖S_k‖_F ≥ orth_thresh
  double* Umat;         // policy 3: strict upper part of V_kᵀV_k, (m+1)×(m+1) column-major (CTA 0 writes)
  double* Smat;         // policy 3, spectral: S_k's columns, same layout (CTA 0 writes)
  int orth_spec;        // policy 3: 0 ‖S_k‖_F, 1 ‖S_k‖₂ by 10 power iterations
  int stall_w;          // stall window (inner iterations), policy 2
  double stall_factor;  // stall improvement factor, policy 2
  double* history; int hist_cap;
  int* cycle_J;         // [hist_cap] inner iterations of every cycle
  double* inner_hist; int inner_cap;
  int* out_int;         // [0] status [1] cycles [2] inner iters [3] history len [4] inner len
  double* out_dbl;      // [0] final relres
  unsigned long long* prof;   // [PH_N] ns accumulated by CTA 0
  unsigned long long* prof_cta;  // [G] per-CTA own SpMV ns (profile mode)
  int profile;          // != 0: grid barrier after every phase (clean attribution)
  int tune;             // developer A/B switches (bit 0: no L2 prefetch in MGS, bit 2: no resident MGS)
  int mgs_resident;     // 1: whole-vector ring (mgs_resident), 2: chunk ring (mgs_chunked), 0: mgs_sweep
  int mgs_nbuf;         // ring depth: basis-vector buffers (mgs_resident) or MGS_CHUNK-byte slots (mgs_chunked)
  int mgs_wsm;          // chunks of w kept in shared memory (after the ring) by the resident MGS
  long long timeout_ns;
  // ILU(0) preconditioner (§8 f2, reading R24; PC kernel instantiations only):
  // factors on A's pattern (W), diagonal position per row, and the level
  // schedules of the lower (forward) and upper (backward) triangular solves:
  // rows of level l are ilu_rows[t][ilu_lev[t][l] .. ilu_lev[t][l+1])
  const void* iluW;
  const int* ilu_dpos;
  const int* ilu_lev[2];
  const int* ilu_rows[2];
  int ilu_nlev[2];
  // per slot (level order) of each solve: its off-diagonal entries, contiguous —
  // ilu_eoff[t][slot] .. [slot+1] index ilu_ecol[t] (column) and ilu_eidx[t]
  // (position in the factor array), in the row's ascending column order
  const int* ilu_eoff[2];
  const int* ilu_ecol[2];
  const int* ilu_eidx[2];
  const void* ilu_rec[2];  // packed per-slot records (IluRec<W>), rebuilt after each factorisation
  void* ilu_pub[2];        // [n] W each, sync-free solves: published row values (all-ones NaN = not yet)
  double normA2;           // ‖A‖_F² of this rank's rows (backward-error report)
  int ilu32;               // fp64 solver with fp32 factors: iluW / ilu_rec are fp32
  float* ilu_s32[2];       // ... and its fp32 scratch vectors (right-hand side, solution)
  // exact fixed-point MGS projections (reading R27; mixed, Jacobi, one rank): 2 words
  // 256 B apart, zeroed before each launch; partials quantised to 2^(fx_exp−42)
  int fx;                  // != 0: the MGS projection all-reduces use allreduce1's fixed-point word
  int fx_exp;              // B = 2^fx_exp ≥ 2·√(‖D⁻¹A‖₁‖D⁻¹A‖∞) ≥ |every CTA partial|
  double fx_bnd, fx_up, fx_dn;  // 2^fx_exp, 2^(42−fx_exp), 2^(fx_exp−42)
  unsigned long long* fx_words;
};

// ------------------------------------------------------------ primitives
template <class W> struct VecT;
template <> struct VecT<float> { using T = float4; static constexpr int N = 4; };
template <> struct VecT<double> { using T = double2; static constexpr int N = 2; };

// address of V(row, col) in the layout of d (see Dev)
template <class W>
__device__ __forceinline__ W* v_at(const Dev& d, W* V, long long row, int col) {
  if (d.vtb == 0) return V + (long long)col * d.ldv + row;
  return V + (row >> d.vtb_log) * d.vbs + (long long)col * d.vtp + (row & (d.vtb - 1));
}

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

// Dot of two 16-byte vectors for the length-n reductions (reading R9): in
// mixed mode the 4 products of a float4 form one short fp32 sum (fma chain,
// "short sums stay in W") that is then accumulated in fp64 — one fp32→fp64
// conversion per 4 elements instead of 8 (F2F runs at 1/8 of the fp32 rate and
// bounded the MGS step, ncu/globaltimer r01); in fp64 mode plain fp64.
__device__ __forceinline__ double dotv(const float4& a, const float4& b) {
  float s = __fmul_rn(a.x, b.x);
  s = __fmaf_rn(a.y, b.y, s);
  s = __fmaf_rn(a.z, b.z, s);
  s = __fmaf_rn(a.w, b.w, s);
  return (double)s;
}
__device__ __forceinline__ double dotv(const double2& a, const double2& b) { return a.x * b.x + a.y * b.y; }

// a ← RN_W(a − RN_W(h·b)) element-wise on a 16-byte vector (MGS line 155); named
// members, no pointer casts, so the vectors stay in registers
__device__ __forceinline__ void sub_scaled(float4& a, const float4& b, float h) {
  a.x = __fsub_rn(a.x, __fmul_rn(h, b.x));
  a.y = __fsub_rn(a.y, __fmul_rn(h, b.y));
  a.z = __fsub_rn(a.z, __fmul_rn(h, b.z));
  a.w = __fsub_rn(a.w, __fmul_rn(h, b.w));
}
__device__ __forceinline__ void sub_scaled(double2& a, const double2& b, double h) {
  a.x = __dsub_rn(a.x, __dmul_rn(h, b.x));
  a.y = __dsub_rn(a.y, __dmul_rn(h, b.y));
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// ---- TMA bulk copies (cp.async.bulk) completing on an mbarrier
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// the same with an L2 eviction-priority policy (createpolicy)
__device__ __forceinline__ void tma_load_1d_hint(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                                 unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ unsigned long long policy_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long policy_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long policy_evict_normal() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// scalar global loads with an L2 eviction-priority policy (SpMV gathers: evict_last
// keeps the gathered vector in L2 while the CSR arrays stream past it)
__device__ __forceinline__ float ld_pol(const float* p, unsigned long long pol) {
  float v;
  asm volatile("ld.global.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_pol(const double* p, unsigned long long pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
// plain arrival (no transaction bytes) on a shared mbarrier
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// 16-byte global store with an L2 eviction-priority policy
__device__ __forceinline__ void st_hint(float4* p, const float4& v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_hint(double2* p, const double2& v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}

// bulk prefetch of [src, src+bytes) into L2 (bytes multiple of 16)
__device__ __forceinline__ void prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// non-blocking probe of a phase (test_wait: never suspends the thread)
__device__ __forceinline__ bool mbar_test_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// per-CTA control block in static shared memory
struct Shm {
  unsigned long long mbar[NGRP][MAXSTG];  // TMA stage barriers (per CSR-stream group)
  unsigned long long mbar_v[32];     // TMA barriers of the resident MGS's ring (≤ MGS_MAXSLOT)
  unsigned long long mbar_e[32];     // streamed MGS: slot-consumed barriers (one arrival per warp)
  unsigned long long mbar_t[4];      // TMA barriers of the row-tile passes' V tiles
  unsigned long long mbar_b[NBS];    // TMA barriers of the block stream's stages
  int bcnt[NBS];                     // warps done with a block-stream stage
  unsigned bphase;                   // bit s: parity of the next completion of mbar_b[s]
  unsigned tma_phase[NGRP];          // bit s: parity of the next completion of stage s
  unsigned vphase;                   // bit b: parity of the next completion of mbar_v[b] (mgs_resident)
  unsigned vg;                       // chunk-ring MGS: stream chunks issued so far (thread 0 writes)
  unsigned tphase;                   // bit b: parity of the next completion of mbar_t[b]
  int cdir;                          // CGSR: direction of the next iteration's first pass
  int abort;
  int flag;
  unsigned long long epoch;          // grid barriers passed by this CTA (thread 0)
  int cta;                           // CTA index within its rank (blockIdx.x unless virtual ranks)
  int red_epoch;                     // all-reduces done (partial buffer parity; thread 0 writes)
  unsigned fx_epoch;                 // parity of the fixed-point projection all-reduces done (the word used next)
  unsigned long long fx_prev[2];     // full value last read from each word (thread 32 only)
  double red[NW * 8];
  double red2[NW * 4];
  unsigned long long pmin, pmax;     // profile mode: all-reduce arrival spread (ar_probe)
  unsigned long long tprev;          // CTA 0's phase timer: timestamp of the last phase boundary
  unsigned long long tsub;           // profile mode: CGSR sub-phase / per-CTA SpMV timers
  // cycle state that only thread 0 needs (kept out of every thread's registers)
  double thr, beta;                  // restart threshold, β of the cycle
  double inv;                        // 1/‖v_j's source‖ of the next SpMV (read by every thread, written by thread 0)
  int kcyc, total_inner;             // cycles done, inner iterations done
  int r0, r1;                        // this CTA's row block
  int jmax, J1, inner_len;           // max inner steps of the cycle, first cycle's J, recorded inner steps
};

// wait for stage s of group grp's TMA pipeline; watchdog on %globaltimer
// (a timeout raises the global abort flag; callers keep their barrier
// sequence and the solve ends with ETIMEOUT at the next grid barrier)
__device__ __forceinline__ void stage_wait(const Dev& d, Shm& sh, int grp, int s) {
  const unsigned par = (sh.tma_phase[grp] >> s) & 1u;
  if (mbar_try_wait(&sh.mbar[grp][s], par)) return;
  const unsigned long long t0 = globaltimer();
  for (;;) {
    if (mbar_try_wait(&sh.mbar[grp][s], par)) return;
    if ((long long)(globaltimer() - t0) > d.timeout_ns) {
      atomicExch(d.abort_flag, 1);
      return;
    }
  }
}

__device__ __forceinline__ void group_sync(int) { __syncwarp(); }

__device__ __forceinline__ void init_shm(Shm& sh, int cta) {
  if (threadIdx.x == 0) {
    sh.cta = cta;
    sh.epoch = 0;
    sh.red_epoch = 0;
    sh.fx_epoch = 0;
    sh.fx_prev[0] = sh.fx_prev[1] = 0ull;
    sh.abort = 0;
    sh.flag = 0;
    sh.vg = 0;
    sh.vphase = 0;
    for (int g = 0; g < NGRP; ++g) {
      sh.tma_phase[g] = 0;
      for (int t = 0; t < MAXSTG; ++t) mbar_init(&sh.mbar[g][t], 1);
    }
    for (int b = 0; b < 32; ++b) mbar_init(&sh.mbar_v[b], 1);
    for (int b = 0; b < 32; ++b) mbar_init(&sh.mbar_e[b], NW);
    for (int b = 0; b < 4; ++b) mbar_init(&sh.mbar_t[b], 1);
    sh.tphase = 0;
    sh.cdir = 0;
    for (int b = 0; b < NBS; ++b) { mbar_init(&sh.mbar_b[b], 1); sh.bcnt[b] = 0; }
    sh.bphase = 0;
    fence_mbar_init();
  }
  __syncthreads();
}

// ------------------------------------------------ grid all-reduce (push + counter)
// Every rank holds a partial array [2][GG][kst] fp64 (GG = CTAs over all
// ranks) and an arrival counter.  Reduction e uses buffer e mod 2: CTA c
// writes its K partials into row c of that buffer in EVERY rank's array (the
// local one among them), then adds 1 to every rank's counter with a release
// reduction; thread 0 of each CTA spins (acquire) on its own rank's counter
// until all GG CTAs of this epoch arrived, and the CTA loads the GG·K partials
// from local memory and sums each k over the GG CTAs in one fixed order — the
// same in every CTA of every rank, so all hold bit-identical results
// (replicated control flow).  Buffer e mod 2 is rewritten at
// e+2, after every CTA arrived at e+1, i.e. after everyone finished reading it.
// (tools/ar_bench.cu: this beats sentinel-slot polling on B200, whose 148×148
// pollers contend in L2: 1.96 vs ≥ 2.56 µs per one-value all-reduce.)
__device__ __forceinline__ void red_release_add(unsigned long long* p, unsigned long long v, bool sys) {
  if (sys) asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_ctr(const unsigned long long* p, bool sys) {
  unsigned long long v;
  if (sys) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ double* slot_row(const Dev& d, double* base, int buf, int gcta) {
  return base + ((size_t)buf * d.GG + gcta) * d.kst;
}

// thread 0: arrive on every rank's counter, wait for all GG CTAs (watchdog);
// the caller brackets it with __syncthreads.  Returns false on abort.
__device__ __forceinline__ bool arrive_wait(const Dev& d, Shm& sh) {
  // called by ONE FULL WARP (lane 0 arrives and polls; the converged warp spins:
  // tools/ar_bench.cu 1.72 vs 1.96 µs per one-value all-reduce with a lone thread)
  const bool sys = d.sys_scope != 0;
  const int lane = threadIdx.x & 31;
  unsigned long long target = 0;
  if (lane == 0) {
    target = (sh.epoch += 1ull) * (unsigned long long)d.GG;
    for (int q = 0; q < d.nranks; ++q) red_release_add(d.ctr_peer[q], 1ull, sys);
  }
  target = __shfl_sync(0xffffffffu, target, 0);
  unsigned it = 0;
  unsigned long long t0 = 0;
  for (;;) {
    const unsigned long long v = lane == 0 ? ld_acquire_ctr(d.ctr, sys) : 0ull;
    if (__shfl_sync(0xffffffffu, v, 0) >= target) break;
    if (((++it) & 1023u) == 0u) {
      if (*(volatile int*)d.abort_flag) return false;
      const unsigned long long t = globaltimer();
      if (t0 == 0) t0 = t;
      else if ((long long)(t - t0) > d.timeout_ns) { if (lane == 0) atomicExch(d.abort_flag, 1); return false; }
    }
  }
  return *(volatile int*)d.abort_flag == 0;
}

// Grid barrier over all CTAs of all ranks (release/acquire).
__device__ __forceinline__ bool grid_sync(const Dev& d, Shm& sh) {
  __syncthreads();
  if (threadIdx.x < 32) {
    const bool ok = arrive_wait(d, sh);
    if (threadIdx.x == 0) sh.abort = ok ? 0 : 1;
  }
  __syncthreads();
  return sh.abort == 0;
}

// push this CTA's K partials into buffer buf of every rank's array
__device__ __forceinline__ void push_partials(const Dev& d, const Shm& sh, const double* s_part, int K, int buf) {
  const int gc = d.cta0 + sh.cta;
  for (int t = threadIdx.x; t < K * d.nranks; t += NT) {
    const int q = t / K, k = t - q * K;
    slot_row(d, d.slot_peer[q], buf, gc)[k] = s_part[k];
  }
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

// profile mode, CTA 0: spread of the CTAs' arrival times at this all-reduce
// (each CTA stored its %globaltimer next to its partial) → sh.pmin / sh.pmax
static __device__ __noinline__ void ar_probe(const Dev& d, Shm& sh, int buf) {
  unsigned long long tmin = ~0ull, tmax = 0ull;
  for (int g = threadIdx.x; g < d.GG; g += NT) {
    const unsigned long long t = (unsigned long long)__double_as_longlong(__ldcg(slot_row(d, d.slots, buf, g) + 1));
    tmin = min(tmin, t);
    tmax = max(tmax, t);
  }
  if (threadIdx.x == 0) { sh.pmin = ~0ull; sh.pmax = 0ull; }
  __syncthreads();
  if (tmax) { atomicMin(&sh.pmin, tmin); atomicMax(&sh.pmax, tmax); }
}

// One-value all-reduce of a per-thread contribution: CTA sum (warp trees,
// warps in order) → push → arrive/wait → fixed-order sum over all GG CTAs.
// (acq is implied: the counter acquire orders every later read.)
struct NoMid { __device__ __forceinline__ void operator()() const {} };
// mid() runs in every thread right after the CTA barrier that follows the
// local contributions (e.g. to reuse a buffer the contributions were read from)
// Fixed-point variant (FX, MGS projections only, d.fx: reading R27): the CTA partial s
// is quantised to q = RN(s·2^(42−e)), |q| ≤ 2^42 (B = 2^e bounds every partial), and
// one 64-bit red.add carries the arrival and the value: count in bits 53–63, the
// offset-binary sum Σ(q + 2^43) below (< 2^51 for ≤ 600 CTAs).  The integer sum is
// exact, so every CTA reads the same word and gets the same h whatever the order of
// arrival — one round trip after the last arrival instead of the partial store's
// release, the counter and the partial loads (tools/ar_bench.cu 1.33 vs 1.80–1.99 µs).
// Two words alternate and only ever grow (mod 2^64, zeroed by the host before the
// launch): every CTA keeps the full value it last read from a word (the same value in
// every CTA) and takes this epoch's count and sum from the difference.  Nothing is
// stored or zeroed, so nothing needs a release or an acquire fence: a CTA's add of
// epoch e+2 (same word) depends on its poll of epoch e+1, which completes only after
// every CTA arrived there, i.e. after every CTA's poll of epoch e returned (the r02
// rotation of four zeroed words needed CTA 0's release and a fence.acq_rel after each
// poll: ≈ 0.4 µs per projection in the polling thread, profiles/r02_ncu_*_source_top).
// The scalings are exact power-of-two multiplies (|s·2^(42−e)| ≤ 2^42; host: |e| ≤ 900).
__device__ __forceinline__ void red_relaxed_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ bool fx_arrive_wait(const Dev& d, Shm& sh, double s, double& out) {  // one thread
  const unsigned e = sh.fx_epoch & 1u;
  unsigned long long* wd = d.fx_words + (size_t)e * 32;
  const unsigned long long prev = sh.fx_prev[e];
  long long q = 0;
  if (fabs(s) <= d.fx_bnd) q = __double2ll_rn(s * d.fx_up);
  else atomicOr(d.err_flag, ERRF_NONFINITE);  // non-finite (the bound holds for finite data)
  red_relaxed_add(wd, (1ull << 53) + (unsigned long long)(q + (1ll << 43)));
  const unsigned long long GG = (unsigned long long)d.GG;
  unsigned long long x;
  unsigned it = 0;
  unsigned long long t0 = 0;
  bool ok = true;
  while ((((x = ld_relaxed_u64(wd)) - prev) >> 53) < GG) {
    if (((++it) & 1023u) == 0u) {
      if (*(volatile int*)d.abort_flag) { ok = false; break; }
      const unsigned long long t = globaltimer();
      if (t0 == 0) t0 = t;
      else if ((long long)(t - t0) > d.timeout_ns) { atomicExch(d.abort_flag, 1); ok = false; break; }
    }
  }
  const long long sum = (long long)((x - prev) & ((1ull << 53) - 1)) - (long long)GG * (1ll << 43);
  out = (double)sum * d.fx_dn;
  sh.fx_prev[e] = x;
  sh.fx_epoch = e ^ 1u;
  return ok;  // (a CTA that aborted elsewhere never arrives again: the next poll sees the flag)
}
template <bool FX = false, class Mid = NoMid>
__device__ __forceinline__ bool allreduce1(const Dev& d, Shm& sh, double v, bool /*acq*/, double& out,
                                           Mid mid = Mid()) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int buf = sh.red_epoch & 1;
  v = warp_sum(v);
  if (lane == 0) sh.red[warp] = v;
  __syncthreads();
  mid();
  if (FX && d.fx) {
    if (warp == 1) {
      double s = lane < NW ? sh.red[lane] : 0.0;
#pragma unroll
      for (int o = NW / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) {
        double x = 0.0;
        const bool ok = fx_arrive_wait(d, sh, s, x);
        sh.red2[0] = x;
        sh.abort = ok ? 0 : 1;
      }
    }
    __syncthreads();
    out = sh.red2[0];
    return sh.abort == 0;
  }
  if (warp == 1) {  // (warp 1 releases: warp 0 may hold in-flight bulk copies, see mgs_resident)
    double s = lane < NW ? sh.red[lane] : 0.0;  // fixed shuffle tree over the warps
#pragma unroll
    for (int o = NW / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      const int gc = d.cta0 + sh.cta;
      for (int q = 0; q < d.nranks; ++q) d.slot_peer[q][d.s1off + (long long)buf * d.GG + gc] = s;
      if (d.profile) slot_row(d, d.slot_peer[0], buf, gc)[1] = __longlong_as_double((long long)globaltimer());
    }
    const bool ok = arrive_wait(d, sh);  // (the partial store precedes lane 0's release)
    // the polling warp sums the GG partials right after it sees the count (lane l: CTAs
    // l, l+32, … in order, all loads in flight together; then a fixed shuffle tree):
    // one CTA barrier after the detection instead of two (C2 mixed MGS −1.5 ms).  The
    // partials are contiguous (d.s1off): 37 sectors per CTA instead of one per partial.
    double x = 0.0;
    if (ok) {
      const double* p1 = d.slots + d.s1off + (long long)buf * d.GG;
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int g = lane + 32 * u;
        v[u] = g < d.GG ? __ldcg(p1 + g) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) x += v[u];
      for (int g = lane + 256; g < d.GG; g += 32) x += __ldcg(p1 + g);
    }
    x = warp_sum(x);
    if (lane == 0) {
      sh.red2[0] = x;
      sh.abort = ok ? 0 : 1;
      sh.red_epoch++;
    }
  }
  if (d.profile && sh.cta == 0) {
    __syncthreads();
    ar_probe(d, sh, buf);
  }
  __syncthreads();
  out = sh.red2[0];
  if (d.profile && sh.cta == 0 && threadIdx.x == 0) {  // prof[11] Σ arrival spread, [12] Σ last arrival → result, [13] count
    d.prof[11] += sh.pmax - sh.pmin;
    d.prof[12] += globaltimer() - sh.pmax;
    d.prof[13] += 1ull;
  }
  return sh.abort == 0;
}

// Grid all-reduce of K fp64 values (s_part → s_out, both shared; s_part
// complete and block-synced by the caller).  Warp w loads a contiguous block
// of CTAs, lane = k; blocks are then summed in warp order: a fixed order, the
// same in every CTA of every rank.
constexpr int GCH = 8;  // independent partial loads in flight per lane
constexpr int GCH1 = 10; // CTAs per warp of the single-round path (GG ≤ 160)
__device__ __forceinline__ bool grid_allreduce(const Dev& d, Shm& sh, const double* s_part, int K, double* s_out,
                                               double* s_tmp, bool /*acq*/ = true) {
  const int buf = sh.red_epoch & 1;
  push_partials(d, sh, s_part, K, buf);
  __syncthreads();
  if ((threadIdx.x >> 5) == 1) {  // warp 1 arrives and polls (warp 0 issues the row-tile passes' bulk copies)
    const bool ok = arrive_wait(d, sh);
    if (threadIdx.x == 32) {
      sh.abort = ok ? 0 : 1;
      sh.red_epoch++;
    }
  }
  __syncthreads();
  if (sh.abort) return false;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gpw = (d.GG + NW - 1) / NW;
  const int g0 = warp * gpw;
  if (K <= 64 && gpw <= GCH1) {
    // one round of loads (K ≤ 64): lane holds k0 + lane and k0 + lane + 32 of all its
    // warp's CTAs in flight together (the loop below takes ⌈K/32⌉·⌈gpw/GCH⌉ dependent
    // L2 round trips; C2 CGSR 90.2 → 88.2 ms); the same per-k order over the CTAs
    {
      const int ka = lane, kb = lane + 32;
      double v0[GCH1], v1[GCH1];
#pragma unroll
      for (int u = 0; u < GCH1; ++u) {
        const int g = g0 + u;
        const bool ok = u < gpw && g < d.GG;
        const double* row = slot_row(d, d.slots, buf, ok ? g : 0);
        v0[u] = (ok && ka < K) ? __ldcg(row + ka) : 0.0;
        v1[u] = (ok && kb < K) ? __ldcg(row + kb) : 0.0;
      }
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int u = 0; u < GCH1; ++u) {
        a0 += v0[u];
        a1 += v1[u];
      }
      if (ka < K) s_tmp[warp * d.kmax + ka] = a0;
      if (kb < K) s_tmp[warp * d.kmax + kb] = a1;
    }
  } else
  for (int k0 = 0; k0 < K; k0 += 32) {
    const int k = k0 + lane;
    if (k < K) {
      double acc = 0.0;
      for (int u0 = 0; u0 < gpw; u0 += GCH) {
        double v[GCH];
#pragma unroll
        for (int u = 0; u < GCH; ++u) {
          const int g = g0 + u0 + u;
          v[u] = (u0 + u < gpw && g < d.GG) ? __ldcg(slot_row(d, d.slots, buf, g) + k) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < GCH; ++u) acc += v[u];
      }
      s_tmp[warp * d.kmax + k] = acc;
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += NT) {
    double acc = 0.0;
    for (int w = 0; w < NW; ++w) acc += s_tmp[w * d.kmax + k];
    s_out[k] = acc;
  }
  __syncthreads();
  return true;
}

// ---------------------------------------------------- halo push (§8 e)
// Push the rows of `loc` (this rank's local view of buffer `which`: 0 = w0,
// 1 = w1, 2 = x) that peers gather into their full-length copies of it, at the
// same global index.  Called by every CTA after its own rows of `loc` are
// final and before the all-reduce/barrier whose release publishes them
// (no-op on one rank).
template <class T>
__device__ __forceinline__ void halo_push(const Dev& d, const Shm& sh, const T* loc, int which) {
  if (!d.halo) return;
  __syncthreads();  // the CTA's final values of loc are written
  const int e0 = d.send_off[sh.cta], e1 = d.send_off[sh.cta + 1];
  for (int e = e0 + threadIdx.x; e < e1; e += NT) {
    const int row = d.send_row[e];
    T* pb = reinterpret_cast<T*>(d.vec_peer[which][d.send_peer[e]]);
    pb[d.row_base + row] = loc[row];
  }
  if (d.halo_full) {  // whole row block of this CTA, coalesced, to the peers that gather most rows
    const int r0 = d.row_begin[sh.cta], r1 = min(d.row_begin[sh.cta + 1], d.n);
    for (int q = 0; q < d.nranks; ++q) {
      if (!((d.halo_full >> q) & 1u)) continue;
      T* pb = reinterpret_cast<T*>(d.vec_peer[which][q]) + d.row_base;
      for (int r = r0 + threadIdx.x; r < r1; r += NT) pb[r] = loc[r];
    }
  }
}
template <class W>
__device__ __forceinline__ int wbuf_index(const Dev& d, const W* w) { return w == (const W*)d.w0 ? 0 : 1; }

// ---------------------------------------------------- CSR stream (a1, a2)
// The CTA's rows are cut (on the host) into chunks of ≤ CHUNK_RMAX rows and
// ≤ CHUNK_CAP non-zeros whose boundaries are multiples of 4 rows.  Every warp
// of the CTA is an independent pipeline: warp g takes chunks g, g+NGRP, ...
// and owns a 2-stage ring; its lane 0 stages chunk i+2's row_ptr/col/val
// slices into shared memory with three TMA bulk copies (cp.async.bulk,
// mbarrier) while the warp computes chunk i.  Warps drift out of phase, so
// one warp's gathers overlap another's TMA wait (no CTA-wide barrier).  L lanes per row (L = 1: one
// thread per row, the oracle's summation order); gathers from global (L1/L2).
// Chunks whose 4 rows exceed CHUNK_CAP are "direct": a warp per row from
// global memory.  pre(row) is called by the epilogue lane before the row's
// gathers (to prefetch per-row operands); epi(row, acc, pre) after.
template <class AT> struct AccOps;
template <> struct AccOps<float> {
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
};
template <> struct AccOps<double> {
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
};

// Chunk metadata of one warp's pipeline, 32 chunks per batch held one per
// lane (two batches: current and next) and read with warp shuffles, so the
// chunk table never sits on a chunk's critical path (ncu r01: the two
// dependent loads of d.chunks per chunk were a top long-scoreboard stall).
struct ChunkMeta { int rb, nb, direct, re, ne; };
struct MetaWin {
  int base;                 // pipeline index of lane 0's chunk in cur
  int cur[5], nxt[5];
  __device__ __forceinline__ void load(const Dev& d, int c0, int c1, int grp, int kb, int (&m)[5]) {
    const int c = c0 + grp + (kb + (int)(threadIdx.x & 31)) * NGRP;
    if (c < c1) {
      const int4 e = d.chunks[c], f = d.chunks[c + 1];
      m[0] = e.x; m[1] = e.y; m[2] = e.z; m[3] = f.x; m[4] = f.y;
    } else {
      m[0] = m[1] = m[2] = m[3] = m[4] = 0;
    }
  }
  __device__ __forceinline__ void init(const Dev& d, int c0, int c1, int grp) {
    base = 0;
    load(d, c0, c1, grp, 0, cur);
    load(d, c0, c1, grp, 32, nxt);
  }
  // k (warp-uniform) ≥ base; advances the window when k leaves cur
  __device__ __forceinline__ void advance(const Dev& d, int c0, int c1, int grp, int k) {
    while (k >= base + 32) {
#pragma unroll
      for (int t = 0; t < 5; ++t) cur[t] = nxt[t];
      base += 32;
      load(d, c0, c1, grp, base + 32, nxt);
    }
  }
  // metadata of pipeline chunk k, base ≤ k < base + 64 (warp-uniform)
  __device__ __forceinline__ ChunkMeta get(int k) const {
    const int idx = k - base;
    int v[5];
#pragma unroll
    for (int t = 0; t < 5; ++t) {
      const int a = __shfl_sync(0xffffffffu, cur[t], idx & 31);
      const int b = __shfl_sync(0xffffffffu, nxt[t], idx & 31);
      v[t] = idx < 32 ? a : b;
    }
    return ChunkMeta{v[0], v[1], v[2], v[3], v[4]};
  }
};

// CSR stream.  epi(row, acc, pv, diag) gets the row sum, pre()'s value and
// the gathered value at the diagonal column (0 if the row has none).
template <class AT, int L, class RT, class Gather, class Pre, class Epi>
__device__ void csr_stream(const Dev& d, Shm& sh, char* s_stage, const AT* __restrict__ vals,
                           const RT* __restrict__ rowv, Gather gat, Pre pre, Epi epi) {
  using Ops = AccOps<AT>;
  using PT = decltype(pre(0, (RT)0));
  const int grp = threadIdx.x / GT, gt = threadIdx.x % GT;
  const int c0 = d.chunk_off[sh.cta], c1 = d.chunk_off[sh.cta + 1] - 1;
  const int nk = c1 - c0 > grp ? (c1 - c0 - grp + NGRP - 1) / NGRP : 0;  // chunks of this pipeline
  const int gro = (int)d.row_base;  // columns are global: local row r's diagonal is column r + gro
  constexpr int NS = NSTG<AT>(), SB = stage_bytes<AT>();
  constexpr int GB = 8;
  char* gbase = s_stage + grp * NS * SB;
  MetaWin mw;
  mw.init(d, c0, c1, grp);
  const unsigned long long pol_a = policy_evict_first();  // the CSR arrays are read once per SpMV
  auto issue = [&](const ChunkMeta& m, int s) {  // group leader only
    if (m.direct) return;
    char* st = gbase + s * SB;
    const int ea = m.nb & ~3, eb = (m.ne + 3) & ~3;
    const unsigned b_rp = (unsigned)(((m.re - m.rb + 1) + 3) & ~3) * 4u;
    const unsigned b_ci = (unsigned)(eb - ea) * 4u;
    const unsigned b_a = (unsigned)(eb - ea) * (unsigned)sizeof(AT);
    const unsigned b_rv = (unsigned)((m.re - m.rb) * (int)sizeof(RT) + 15) & ~15u;  // rowv is padded to 32 rows
    // (no proxy fence: the TMA reads data no generic store of this launch
    // wrote, and overwrites a stage the warp finished reading before the __syncwarp)
    mbar_expect_tx(&sh.mbar[grp][s], b_rp + b_rv + b_ci + b_a);
    tma_load_1d_hint(st, d.rp + m.rb, b_rp, &sh.mbar[grp][s], pol_a);
    tma_load_1d_hint(st + ST_OFF_RV, rowv + m.rb, b_rv, &sh.mbar[grp][s], pol_a);
    if (b_ci) {
      tma_load_1d_hint(st + ST_OFF_CI, d.ci + ea, b_ci, &sh.mbar[grp][s], pol_a);
      tma_load_1d_hint(st + ST_OFF_A, vals + ea, b_a, &sh.mbar[grp][s], pol_a);
    }
  };
  for (int t = 0; t < NS && t < nk; ++t) {
    const ChunkMeta m = mw.get(t);
    if (gt == 0) issue(m, t);
  }
  const int wl = threadIdx.x & 31, gw = gt >> 5;  // lane, warp within the group
  struct Stg { const int* rp; const int* ci; const AT* a; const RT* rv; int ea; };
  auto stage = [&](int s, const ChunkMeta& m) {
    const char* st = gbase + s * SB;
    return Stg{reinterpret_cast<const int*>(st), reinterpret_cast<const int*>(st + ST_OFF_CI),
               reinterpret_cast<const AT*>(st + ST_OFF_A), reinterpret_cast<const RT*>(st + ST_OFF_RV), m.nb & ~3};
  };
  // a lane's elements p0+lane, p0+lane+L, ... in batches of GB: all GB
  // gathers are issued before the (in-order) accumulation
  auto row_dot = [&](const Stg& S, int row, int p0, int p1, int lane, AT& diag) -> AT {
    AT acc = (AT)0;
    for (int pb = p0 + lane; pb < p1; pb += GB * L) {
      AT g[GB], a[GB];
      int cc[GB];
#pragma unroll
      for (int u = 0; u < GB; ++u) {
        const int p = pb + u * L;
        const bool ok = p < p1;
        cc[u] = ok ? S.ci[p] : -1;
        g[u] = ok ? gat(cc[u]) : (AT)0;
        a[u] = ok ? S.a[p] : (AT)0;
      }
#pragma unroll
      for (int u = 0; u < GB; ++u) {
        if (pb + u * L < p1) acc = Ops::add(acc, Ops::mul(a[u], g[u]));
        if (cc[u] == row + gro) diag = g[u];
      }
    }
    return acc;
  };
  for (int k = 0; k < nk; ++k) {
    mw.advance(d, c0, c1, grp, k);
    const int s = k % NS;
    const ChunkMeta m = mw.get(k);
    const int rb = m.rb, nrow = m.re - m.rb;
    // one thread per row and an even ring: consume two staged chunks at once,
    // so that both chunks' gathers are in flight together (the stream is
    // bound by the per-chunk gather latency at one chunk per warp)
    if (L == 1 && NS % 2 == 0 && !(d.tune & 1024) && k + 1 < nk) {
      const ChunkMeta m2 = mw.get(k + 1);
      if (!m.direct && !m2.direct) {
        const int s2 = (k + 1) % NS;
        const int rb2 = m2.rb, nrow2 = m2.re - m2.rb;
        stage_wait(d, sh, grp, s);
        stage_wait(d, sh, grp, s2);
        const Stg S1 = stage(s, m), S2 = stage(s2, m2);
        for (int lr = gt; lr < max(nrow, nrow2); lr += GT) {
          const bool act1 = lr < nrow, act2 = lr < nrow2;
          PT pv1{}, pv2{};
          if (act1) pv1 = pre(rb + lr, S1.rv[lr]);
          if (act2) pv2 = pre(rb2 + lr, S2.rv[lr]);
          int p1 = act1 ? S1.rp[lr] - S1.ea : 0, q1 = act1 ? S1.rp[lr + 1] - S1.ea : 0;
          int p2 = act2 ? S2.rp[lr] - S2.ea : 0, q2 = act2 ? S2.rp[lr + 1] - S2.ea : 0;
          AT acc1 = (AT)0, acc2 = (AT)0, dg1 = (AT)0, dg2 = (AT)0;
          while (p1 < q1 || p2 < q2) {
            AT g1[GB], a1[GB], g2[GB], a2[GB];
            int k1[GB], k2[GB];
#pragma unroll
            for (int u = 0; u < GB; ++u) {
              const bool o1 = p1 + u < q1, o2 = p2 + u < q2;
              k1[u] = o1 ? S1.ci[p1 + u] : -1;
              k2[u] = o2 ? S2.ci[p2 + u] : -1;
              g1[u] = o1 ? gat(k1[u]) : (AT)0;
              a1[u] = o1 ? S1.a[p1 + u] : (AT)0;
              g2[u] = o2 ? gat(k2[u]) : (AT)0;
              a2[u] = o2 ? S2.a[p2 + u] : (AT)0;
            }
#pragma unroll
            for (int u = 0; u < GB; ++u) {
              if (p1 + u < q1) acc1 = Ops::add(acc1, Ops::mul(a1[u], g1[u]));
              if (p2 + u < q2) acc2 = Ops::add(acc2, Ops::mul(a2[u], g2[u]));
              if (k1[u] == rb + lr + gro) dg1 = g1[u];
              if (k2[u] == rb2 + lr + gro) dg2 = g2[u];
            }
            p1 += GB;
            p2 += GB;
          }
          if (act1) epi(rb + lr, acc1, pv1, dg1);
          if (act2) epi(rb2 + lr, acc2, pv2, dg2);
        }
        __syncwarp();
        const ChunkMeta n1 = mw.get(min(k + NS, nk - 1)), n2 = mw.get(min(k + NS + 1, nk - 1));
        if (gt == 0) {
          sh.tma_phase[grp] ^= (1u << s) | (1u << s2);
          if (k + NS < nk) issue(n1, s);
          if (k + NS + 1 < nk) issue(n2, s2);
        }
        ++k;
        continue;
      }
    }
    if (!m.direct) {
      stage_wait(d, sh, grp, s);
      const Stg S = stage(s, m);
      if (L == 1) {
        for (int lr = gt; lr < nrow; lr += GT) {
          const PT pv = pre(rb + lr, S.rv[lr]);
          AT dg = (AT)0;
          const AT acc = row_dot(S, rb + lr, S.rp[lr] - S.ea, S.rp[lr + 1] - S.ea, 0, dg);
          epi(rb + lr, acc, pv, dg);
        }
      } else {
        const int sub = wl / L, lane = wl & (L - 1);
        for (int base = gw * (32 / L); base < nrow; base += GT / L) {
          const int lr = base + sub;
          const bool act = lr < nrow;
          PT pv{};
          if (act && lane == 0) pv = pre(rb + lr, S.rv[lr]);
          AT acc = (AT)0, dg = (AT)0;
          if (act) acc = row_dot(S, rb + lr, S.rp[lr] - S.ea, S.rp[lr + 1] - S.ea, lane, dg);
#pragma unroll
          for (int o = L / 2; o > 0; o >>= 1) {
            acc = Ops::add(acc, __shfl_xor_sync(0xffffffffu, acc, o));
            dg += __shfl_xor_sync(0xffffffffu, dg, o);  // one lane holds the diagonal
          }
          if (act && lane == 0) epi(rb + lr, acc, pv, dg);
        }
      }
    } else {
      // direct chunk (very long rows): one warp per row from global memory
      for (int lr = gw; lr < nrow; lr += GT / 32) {
        const int row = rb + lr;
        PT pv{};
        if (wl == 0) pv = pre(row, __ldg(rowv + row));
        const int p0 = __ldg(d.rp + row), p1 = __ldg(d.rp + row + 1);
        AT acc = (AT)0, dg = (AT)0;
        for (int p = p0 + wl; p < p1; p += 32) {
          const int col = __ldcs(d.ci + p);
          const AT g = gat(col);
          acc = Ops::add(acc, Ops::mul(__ldcs(vals + p), g));
          if (col == row + gro) dg = g;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          acc = Ops::add(acc, __shfl_xor_sync(0xffffffffu, acc, o));
          dg += __shfl_xor_sync(0xffffffffu, dg, o);
        }
        if (wl == 0) epi(row, acc, pv, dg);
      }
    }
    __syncwarp();
    const ChunkMeta n = mw.get(min(k + NS, nk - 1));
    if (gt == 0) {
      if (!m.direct) sh.tma_phase[grp] ^= (1u << s);
      if (k + NS < nk) issue(n, s);
    }
  }
  // the epilogue's stores (w, the V column) are read next by TMA bulk copies
  // (async proxy) of this CTA: order them for that proxy before the barrier
  fence_proxy_async_global();
  __syncthreads();
}

// ---------------------------------------------------- block CSR stream (a1, a2)
// For matrices whose rows are short (≤ BS_MAXROW nonzeros: the stencils), the
// CTA's rows are cut (on the host) into stages of ≤ BS_BYTES of row_ptr,
// per-row operand (Jacobi), col and val slices — four large bulk copies per
// stage (the per-warp 32-row chunks of csr_stream cost four ≤ 1 KB copies
// each, and bulk copies are paced by the TMA engine at ~20–40 ns per copy:
// tools/tma_bench.cu).  All 16 warps consume a stage, each a contiguous
// sixteenth of its rows, L lanes per row; the warp that finishes a stage last
// (shared counter) issues the copies of the stage NBS ahead into its slot.
template <class AT, int L, class RT, class Gather, class Pre, class Epi>
__device__ void csr_block_stream(const Dev& d, Shm& sh, char* s_stage, const AT* __restrict__ vals,
                                 const RT* __restrict__ rowv, Gather gat, Pre pre, Epi epi) {
  using Ops = AccOps<AT>;
  using PT = decltype(pre(0, (RT)0));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int s0 = d.stage_off[sh.cta], ns = d.stage_off[sh.cta + 1] - 1 - s0;
  const int gro = (int)d.row_base;
  constexpr int GB = 8;
  unsigned ph = sh.bphase;
  struct Geo { int rb, rows, ea, o_rv, o_ci, o_va; unsigned b_rp, b_rv, b_ci, b_va; };
  auto geo = [&](int k) {
    const int2 e = d.stages[s0 + k], f = d.stages[s0 + k + 1];
    Geo g;
    g.rb = e.x;
    g.rows = f.x - e.x;
    g.ea = e.y & ~3;
    const int eb = (f.y + 3) & ~3;
    g.b_rp = (unsigned)(((g.rows + 1 + 3) & ~3) * 4);
    g.b_rv = (unsigned)((g.rows * (int)sizeof(RT) + 15) & ~15);
    g.b_ci = (unsigned)((eb - g.ea) * 4);
    g.b_va = (unsigned)((eb - g.ea) * (int)sizeof(AT));
    g.o_rv = (int)g.b_rp;
    g.o_ci = g.o_rv + (int)g.b_rv;
    g.o_va = g.o_ci + (int)g.b_ci;
    return g;
  };
  const unsigned long long pol_a = policy_evict_first();  // the CSR arrays are read once per SpMV
  auto issue = [&](int k) {  // one thread
    const Geo g = geo(k);
    const int slot = k % NBS;
    char* st = s_stage + slot * BS_BYTES;
    unsigned long long* bar = &sh.mbar_b[slot];
    mbar_expect_tx(bar, g.b_rp + g.b_rv + g.b_ci + g.b_va);
    tma_load_1d_hint(st, d.rp + g.rb, g.b_rp, bar, pol_a);
    tma_load_1d_hint(st + g.o_rv, rowv + g.rb, g.b_rv, bar, pol_a);
    if (g.b_ci) {
      tma_load_1d_hint(st + g.o_ci, d.ci + g.ea, g.b_ci, bar, pol_a);
      tma_load_1d_hint(st + g.o_va, vals + g.ea, g.b_va, bar, pol_a);
    }
  };
  if (threadIdx.x == 0)
    for (int k = 0; k < NBS && k < ns; ++k) issue(k);
  for (int k = 0; k < ns; ++k) {
    const int slot = k % NBS;
    {
      const unsigned par = (ph >> slot) & 1u;
      ph ^= (1u << slot);
      if (!mbar_try_wait(&sh.mbar_b[slot], par)) {
        const unsigned long long t0 = globaltimer();
        while (!mbar_try_wait(&sh.mbar_b[slot], par))
          if ((long long)(globaltimer() - t0) > d.timeout_ns) { atomicExch(d.abort_flag, 1); break; }
      }
    }
    const Geo g = geo(k);
    const char* st = s_stage + slot * BS_BYTES;
    const int* srp = reinterpret_cast<const int*>(st);
    const RT* srv = reinterpret_cast<const RT*>(st + g.o_rv);
    const int* sci = reinterpret_cast<const int*>(st + g.o_ci);
    const AT* sa = reinterpret_cast<const AT*>(st + g.o_va);
    const int wa = (warp * g.rows) / NW, wb = ((warp + 1) * g.rows) / NW;
    const int sub = lane / L, ln = lane & (L - 1);
    constexpr int RPP = 32 / L;  // rows per pass of the warp
    // two passes' rows at once per lane: both rows' gathers are in flight together
    for (int r0 = wa; r0 < wb; r0 += 2 * RPP) {
      int r[2], p[2], q[2];
      bool act[2];
      PT pv[2];
      AT acc[2], dg[2];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        r[t] = r0 + sub + t * RPP;
        act[t] = r[t] < wb;
        pv[t] = PT{};
        if (act[t] && ln == 0) pv[t] = pre(g.rb + r[t], srv[r[t]]);
        p[t] = act[t] ? srp[r[t]] - g.ea + ln : 0;
        q[t] = act[t] ? srp[r[t] + 1] - g.ea : 0;
        acc[t] = (AT)0;
        dg[t] = (AT)0;
      }
      while (p[0] < q[0] || p[1] < q[1]) {
        AT gv[2][GB], av[2][GB];
        int cc[2][GB];
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int u = 0; u < GB; ++u) {
            const int e = p[t] + u * L;
            const bool ok = e < q[t];
            cc[t][u] = ok ? sci[e] : -1;
            gv[t][u] = ok ? gat(cc[t][u]) : (AT)0;
            av[t][u] = ok ? sa[e] : (AT)0;
          }
#pragma unroll
        for (int t = 0; t < 2; ++t) {
#pragma unroll
          for (int u = 0; u < GB; ++u) {
            if (p[t] + u * L < q[t]) acc[t] = Ops::add(acc[t], Ops::mul(av[t][u], gv[t][u]));
            if (cc[t][u] == g.rb + r[t] + gro) dg[t] = gv[t][u];
          }
          p[t] += GB * L;
        }
      }
#pragma unroll
      for (int t = 0; t < 2; ++t) {
#pragma unroll
        for (int o = L / 2; o > 0; o >>= 1) {
          acc[t] = Ops::add(acc[t], __shfl_xor_sync(0xffffffffu, acc[t], o));
          dg[t] += __shfl_xor_sync(0xffffffffu, dg[t], o);
        }
        if (act[t] && ln == 0) epi(g.rb + r[t], acc[t], pv[t], dg[t]);
      }
    }
    __syncwarp();
    if (lane == 0) {  // the last warp done with stage k refills its slot
      if (atomicAdd(&sh.bcnt[slot], 1) == NW - 1) {
        sh.bcnt[slot] = 0;
        if (k + NBS < ns) issue(k + NBS);
      }
    }
  }
  if (threadIdx.x == 0) sh.bphase = ph;  // every thread read it at entry, before the barrier below
  fence_proxy_async_global();
  __syncthreads();
}

// ------------------------------------------------ merge-path CSR stream (a2)
// Alg. 1 line 100 on irregular rows (BJ configs[2]: power-law
// row lengths 4..2000, "load-imbalance stress for SpMV").  The host cuts each
// CTA's non-zeros into tiles (make_mtiles): ≤ MT_CAP positions counted from an
// 8-aligned base A, ≤ MT_RMAX rows touched; a row may span several tiles.
// Per tile, lane t owns the 8 consecutive positions [A + 8t, A + 8t + 8) —
// equal work per lane whatever the row lengths (a merge-path split of the
// non-zeros) — and issues its 8 gathers together.  Only the column and value
// slices are staged (two bulk copies per tile: the TMA engine paces small
// copies, and the r02 four-copy tiles were bound by it); lane l holds
// row_ptr[rb + l] (l ≤ nr) in a register and every lane reads row bounds with
// shuffles.  A lane sums its positions row segment by row segment
// (clo[u]: the segment that ended before slot u); a segmented scan across
// lanes (5 shuffle steps, fixed order) carries a row's partial over lane
// boundaries; lane l then takes row l's sum from the lane holding its last
// element and runs its epilogue (coalesced, one row per lane).  A row crossing
// a tile boundary leaves one partial per tile in d.mcarry ([2·tile]: the
// tile's first row if it started earlier, [2·tile+1]: its last row if it
// continues); after the CTA barrier the CTA's split-row list (d.msplit: row,
// first tile, last tile) sums them in tile order and runs their epilogue —
// deterministic, no atomics.  Every row has ≥ 1 non-zero (the diagonal,
// validated at create).  diag(row) returns the gathered value at the diagonal
// column (loaded directly: coalesced, L2).
constexpr int MT_CAP = 256;   // positions per tile (32 lanes × 8)
constexpr int MT_RMAX = 31;   // rows touched per tile (row_ptr[rb .. rb + nr] in one register per lane)
constexpr int MT_OFF_A = MT_CAP * 4;  // stage layout (bytes): columns, then values
static_assert(MT_OFF_A + MT_CAP * 4 <= ST_OFF_A + (CHUNK_CAP + 8) * 4, "fp32 merge stage");
static_assert(MT_OFF_A + MT_CAP * 8 <= ST_OFF_A + (CHUNK_CAP + 8) * 8, "fp64 merge stage");

struct MTile { int rb, s, nr, ne; };  // first row, first position, rows touched, end position
struct MTWin {                        // tile metadata, 32 tiles per batch held one per lane (cf. MetaWin)
  int base;
  int cur[4], nxt[4];
  __device__ __forceinline__ void load(const Dev& d, int c0, int c1, int grp, int kb, int (&m)[4]) {
    const int c = c0 + grp + (kb + (int)(threadIdx.x & 31)) * NGRP;
    if (c < c1) {
      const int4 e = d.mtiles[c];
      m[0] = e.x; m[1] = e.y; m[2] = e.z; m[3] = d.mtiles[c + 1].y;
    } else {
      m[0] = m[1] = m[2] = m[3] = 0;
    }
  }
  __device__ __forceinline__ void init(const Dev& d, int c0, int c1, int grp) {
    base = 0;
    load(d, c0, c1, grp, 0, cur);
    load(d, c0, c1, grp, 32, nxt);
  }
  __device__ __forceinline__ void advance(const Dev& d, int c0, int c1, int grp, int k) {
    while (k >= base + 32) {
#pragma unroll
      for (int t = 0; t < 4; ++t) cur[t] = nxt[t];
      base += 32;
      load(d, c0, c1, grp, base + 32, nxt);
    }
  }
  __device__ __forceinline__ MTile get(int k) const {
    const int idx = k - base;
    int v[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int a = __shfl_sync(0xffffffffu, cur[t], idx & 31);
      const int b = __shfl_sync(0xffffffffu, nxt[t], idx & 31);
      v[t] = idx < 32 ? a : b;
    }
    return MTile{v[0], v[1], v[2], v[3]};
  }
};

__device__ __forceinline__ void lds8(const float* p, float (&a)[8]) {
  const float4 x = reinterpret_cast<const float4*>(p)[0], y = reinterpret_cast<const float4*>(p)[1];
  a[0] = x.x; a[1] = x.y; a[2] = x.z; a[3] = x.w; a[4] = y.x; a[5] = y.y; a[6] = y.z; a[7] = y.w;
}
__device__ __forceinline__ void lds8(const double* p, double (&a)[8]) {
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const double2 x = reinterpret_cast<const double2*>(p)[h];
    a[2 * h] = x.x;
    a[2 * h + 1] = x.y;
  }
}
__device__ __forceinline__ void lds8(const int* p, int (&a)[8]) {
  const int4 x = reinterpret_cast<const int4*>(p)[0], y = reinterpret_cast<const int4*>(p)[1];
  a[0] = x.x; a[1] = x.y; a[2] = x.z; a[3] = x.w; a[4] = y.x; a[5] = y.y; a[6] = y.z; a[7] = y.w;
}

template <class AT, int TB, class RT, class Gather, class Pre, class Diag, class Epi>
__device__ void csr_merge_stream(const Dev& d, Shm& sh, char* s_stage, const AT* __restrict__ vals,
                                 const RT* __restrict__ rowv, Gather gat, Pre pre, Diag diag, Epi epi) {
  using Ops = AccOps<AT>;
  using PT = decltype(pre(0, (RT)0));
  const int grp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = d.mt_off[sh.cta], c1 = d.mt_off[sh.cta + 1] - 1;  // tiles [c0, c1) + a sentinel
  const int nk = c1 - c0 > grp ? (c1 - c0 - grp + NGRP - 1) / NGRP : 0;  // tiles of this warp
  constexpr int NS = NSTG<AT>(), SB = stage_bytes<AT>();
  char* gbase = s_stage + grp * NS * SB;
  MTWin mw;
  mw.init(d, c0, c1, grp);
  const unsigned long long pol_a = policy_evict_first();  // the CSR arrays are read once per SpMV
  auto issue = [&](const MTile& m, int s) {               // lane 0
    char* st = gbase + s * SB;
    const int A = m.s & ~7, eb = (m.ne + 3) & ~3;
    const unsigned b_ci = (unsigned)(eb - A) * 4u, b_a = (unsigned)(eb - A) * (unsigned)sizeof(AT);
    mbar_expect_tx(&sh.mbar[grp][s], b_ci + b_a);
    tma_load_1d_hint(st, d.ci + A, b_ci, &sh.mbar[grp][s], pol_a);
    tma_load_1d_hint(st + MT_OFF_A, vals + A, b_a, &sh.mbar[grp][s], pol_a);
  };
  for (int t = 0; t < NS && t < nk; ++t) {
    const MTile m = mw.get(t);
    if (lane == 0) issue(m, t);
  }
  // TB tiles per iteration (fp32: two of the four staged tiles): their gathers
  // and their latency chains (row search, segment pass, scan, lookups) overlap
  static_assert(NS % TB == 0, "merge stream: ring depth must be a multiple of TB");
  for (int k = 0; k < nk; k += TB) {
    mw.advance(d, c0, c1, grp, k);
    MTile m[TB];
    bool val[TB];
#pragma unroll
    for (int t = 0; t < TB; ++t) {
      val[t] = k + t < nk;
      m[t] = mw.get(min(k + t, nk - 1));
      if (!val[t]) { m[t].nr = 0; m[t].ne = m[t].s; }  // empty: no position, no row
    }
    // per-row operands of lane l's row rb + l, and row_ptr[rb + l] (l ≤ nr), from
    // global memory before the stage wait: their latency runs under the wait
    AT dgl[TB];
    RT rvv[TB];
    int rsv[TB];
#pragma unroll
    for (int t = 0; t < TB; ++t) {
      const bool own = lane < m[t].nr;
      dgl[t] = own ? diag(m[t].rb + lane) : (AT)0;
      rvv[t] = own ? __ldg(rowv + m[t].rb + lane) : (RT)0;
      rsv[t] = lane <= m[t].nr ? __ldg(d.rp + m[t].rb + lane) : 0x7fffffff;
    }
#pragma unroll
    for (int t = 0; t < TB; ++t)
      if (val[t]) stage_wait(d, sh, grp, (k + t) % NS);
    AT g[TB][8], a[TB][8];
    int A[TB], p0[TB], pf[TB], pe[TB];
#pragma unroll
    for (int t = 0; t < TB; ++t) {
      const char* st = gbase + ((k + t) % NS) * SB;
      A[t] = m[t].s & ~7;
      p0[t] = A[t] + 8 * lane;
      pf[t] = max(p0[t], m[t].s);
      pe[t] = min(p0[t] + 8, m[t].ne);  // the lane's positions [pf, pe)
      int cc[8];
      lds8(reinterpret_cast<const int*>(st) + 8 * lane, cc);
#pragma unroll
      for (int u = 0; u < 8; ++u) g[t][u] = (p0[t] + u >= pf[t] && p0[t] + u < pe[t]) ? gat(cc[u]) : (AT)0;
    }
    PT pv[TB];
    int rs[TB], re[TB];
#pragma unroll
    for (int t = 0; t < TB; ++t) {
      const char* st = gbase + ((k + t) % NS) * SB;
      lds8(reinterpret_cast<const AT*>(st + MT_OFF_A) + 8 * lane, a[t]);
      rs[t] = rsv[t];
      re[t] = __shfl_sync(0xffffffffu, rsv[t], (lane + 1) & 31);
      pv[t] = lane < m[t].nr ? pre(m[t].rb + lane, rvv[t]) : PT{};
    }
    // row of the lane's first position: the last row starting at or before pf
    // (binary search over row_ptr[rb .. rb + nr − 1] by shuffles; nr ≤ 31)
    int lr[TB], hi[TB];
#pragma unroll
    for (int t = 0; t < TB; ++t) { lr[t] = 0; hi[t] = m[t].nr - 1; }
#pragma unroll
    for (int it = 0; it < 5; ++it) {
#pragma unroll
      for (int t = 0; t < TB; ++t) {
        const int mid = (lr[t] + hi[t] + 1) >> 1;
        const int v = __shfl_sync(0xffffffffu, rsv[t], mid & 31);
        if (lr[t] < hi[t]) {
          if (v <= pf[t]) lr[t] = mid; else hi[t] = mid - 1;
        }
      }
    }
    AT acc[TB], clo[TB][8];
    bool f[TB];
#pragma unroll
    for (int t = 0; t < TB; ++t) {
      const int lr0 = lr[t];
      const int st0 = __shfl_sync(0xffffffffu, rsv[t], lr0 & 31);
      int end = __shfl_sync(0xffffffffu, rsv[t], (lr0 + 1) & 31);
      acc[t] = (AT)0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        clo[t][u] = (AT)0;
        const int nx = __shfl_sync(0xffffffffu, rsv[t], (lr[t] + 2) & 31);  // end of the next row
        const int p = p0[t] + u;
        if (p >= pf[t] && p < pe[t]) {
          if (p == end) {  // the segment of row lr ended before slot u (rows are non-empty)
            clo[t][u] = acc[t];
            acc[t] = (AT)0;
            ++lr[t];
            end = nx;
          }
          acc[t] = Ops::add(acc[t], Ops::mul(a[t][u], g[t][u]));
        }
      }
      // reset flag of the segmented scan: the lane holds no position, or its last
      // segment starts in it
      f[t] = !(pf[t] < pe[t]) || lr[t] > lr0 || st0 >= pf[t];
    }
    // segmented inclusive scan of the lanes' last segments: C = partial of that
    // row from its first position in the tile
    AT C[TB];
#pragma unroll
    for (int t = 0; t < TB; ++t) C[t] = pf[t] < pe[t] ? acc[t] : (AT)0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
      for (int t = 0; t < TB; ++t) {
        const AT cv = __shfl_up_sync(0xffffffffu, C[t], o);
        const bool fv = __shfl_up_sync(0xffffffffu, (int)f[t], o) != 0;
        if (lane >= o) {
          if (!f[t]) C[t] = Ops::add(cv, C[t]);
          f[t] = f[t] || fv;
        }
      }
    }
#pragma unroll
    for (int t = 0; t < TB; ++t) {
      // row l's positions in the tile [ps, pq): its last segment is in lane kl
      const bool own = lane < m[t].nr;
      const int ps = max(rs[t], m[t].s), pq = min(re[t], m[t].ne);
      const int kl = own ? ((pq - 1 - A[t]) >> 3) : 0, kf = own ? ((ps - A[t]) >> 3) : 0;
      const int eu = pq - (A[t] + 8 * kl);  // 1..8: slot after the row's last position in lane kl
      const bool fin = eu == 8 || pq == m[t].ne;
      AT x = __shfl_sync(0xffffffffu, acc[t], kl);
#pragma unroll
      for (int u = 1; u < 8; ++u) {
        const AT v = __shfl_sync(0xffffffffu, clo[t][u], kl);
        if (!fin && eu == u) x = v;
      }
      const AT cp = __shfl_sync(0xffffffffu, C[t], (kl + 31) & 31);
      if (own) {
        if (kf < kl) x = Ops::add(cp, x);
        const bool open_l = rs[t] < m[t].s, open_r = re[t] > m[t].ne;
        if (!open_l && !open_r) epi(m[t].rb + lane, x, pv[t], dgl[t]);
        else d.mcarry[2 * (c0 + grp + (k + t) * NGRP) + (open_l ? 0 : 1)] = (double)x;
      }
    }
    __syncwarp();
    MTile n[TB];
#pragma unroll
    for (int t = 0; t < TB; ++t) n[t] = mw.get(min(k + t + NS, nk - 1));
    if (lane == 0) {
#pragma unroll
      for (int t = 0; t < TB; ++t) {
        if (!val[t]) continue;
        const int s = (k + t) % NS;
        sh.tma_phase[grp] ^= (1u << s);
        if (k + t + NS < nk) issue(n[t], s);
      }
    }
  }
  __syncthreads();  // the tiles' carries are visible to the CTA
  const int q0 = d.ms_off[sh.cta], q1 = d.ms_off[sh.cta + 1];
  for (int q = q0 + (int)threadIdx.x; q < q1; q += NT) {
    const int4 e = d.msplit[q];  // {row, first tile, last tile}
    AT acc = (AT)d.mcarry[2 * e.y + 1];
    for (int c = e.y + 1; c <= e.z; ++c) acc = Ops::add(acc, (AT)d.mcarry[2 * c]);
    epi(e.x, acc, pre(e.x, rowv[e.x]), diag(e.x));
  }
  fence_proxy_async_global();
  __syncthreads();
}

template <class AT, int L, class RT, class Gather, class Pre, class Epi>
__device__ __forceinline__ void csr_any_stream(const Dev& d, Shm& sh, char* s_stage, const AT* __restrict__ vals,
                                               const RT* __restrict__ rowv, Gather gat, Pre pre, Epi epi) {
  if (d.block_stream) csr_block_stream<AT, L>(d, sh, s_stage, vals, rowv, gat, pre, epi);
  else csr_stream<AT, L>(d, sh, s_stage, vals, rowv, gat, pre, epi);
}
// The merge-path stream runs one tile per warp iteration (TB = 1).  Measured r02
// on C3 (mixed, 30 SpMVs per solve): chunk stream 41.3 ms, merge tiles with four
// bulk copies 28.9 ms, two tiles per iteration (TB = 2, twice the gathers in
// flight) 28.9 ms, two copies per tile 30.3 ms — neither more gathers per warp
// nor fewer TMA copies moves it: the random gathers (one L2 sector each,
// 120 M per SpMV) are bound by the memory system's outstanding requests, not
// by the warp's issue.  TB = 2 raised the register pressure of the whole
// persistent kernel (spills moved into the resident MGS loop; as a __noinline__
// call the ABI did the same), so it is kept as a compile-time option only.

// ------------------------------------------------------------------ a1
// Alg. 1 lines 86–90: z = b − A64 x in fp64, then
// r = RN_W(dinv_W · RN_W(z)) (reading R10).  fp64 row sums.
template <class W, int L, bool MERGE>
__device__ __forceinline__ void resid_body(const Dev& d, Shm& sh, char* s_stage, W* __restrict__ r_out, double& zz,
                                           double& rr, double& bb, double& xx, int& err) {
  const W* dinv = (const W*)d.dinvW;
  const double* __restrict__ xg = d.x - d.row_base;  // global-index view (CSR columns are global)
  struct P2 { double b; W di; };
  const unsigned long long pol_g = policy_evict_last();
  auto gat = [&](int col) -> double { return ld_pol(xg + col, pol_g); };
  auto pre = [&](int row, W di) -> P2 { return P2{d.b[row], di}; };
  auto epi = [&](int row, double acc, P2 pv, double xd) {  // xd: x at the diagonal column = x_row
    const double bi = pv.b;
    bb += bi * bi;
    xx += xd * xd;  // ‖x‖² for the normwise backward error (report only, reading R5)
    const double z = bi - acc;
    if (!isfinite(z)) err |= ERRF_NONFINITE;
    zz += z * z;
    if (sizeof(W) == 4 && fabs(z) > (double)FLT_MAX) err |= ERRF_RANGE;
    const W ri = mulw(pv.di, RN<W>(z));
    r_out[row] = ri;
    rr += (double)ri * (double)ri;
  };
  auto dg = [&](int row) -> double { return d.x[row]; };
  if (MERGE) csr_merge_stream<double, 1>(d, sh, s_stage, d.a64, dinv, gat, pre, dg, epi);
  else csr_any_stream<double, L>(d, sh, s_stage, d.a64, dinv, gat, pre, epi);
}
template <class W, int L>
__device__ void resid_phase(const Dev& d, Shm& sh, char* s_stage, W* __restrict__ r_out, double& zz, double& rr,
                            double& bb, double& xx, int& err) {
  if (!d.block_stream && d.merge_stream) resid_body<W, L, true>(d, sh, s_stage, r_out, zz, rr, bb, xx, err);
  else resid_body<W, L, false>(d, sh, s_stage, r_out, zz, rr, bb, xx, err);
}

// ------------------------------------------------------------------ a2
// Alg. 1: w = RN_W(dinv_W ∘ (A_W v_j)), with v_j = RN_W(src · RN_W(inv))
// (reading R21: a working-precision scal by the rounded reciprocal) formed on
// the fly from the unnormalised previous vector (line 105 fused into the
// gather: identical bits to normalising first).  The epilogue also stores the
// CTA's own rows of v_j into V[:, j−1].
template <class W, int L, bool MERGE>
__device__ __forceinline__ void spmv_body(const Dev& d, Shm& sh, char* s_stage, const W* __restrict__ src, double inv,
                                          W* __restrict__ dst, W* __restrict__ V, int vc) {
  const W* dinv = (const W*)d.dinvW;
  const W* __restrict__ srcg = src - d.row_base;  // global-index view (CSR columns are global)
  const W invW = RN<W>(inv);
  const unsigned long long pol_g = policy_evict_last();
  auto gat = [&](int col) -> W { return mulw(ld_pol(srcg + col, pol_g), invW); };
  auto pre = [&](int, W di) -> W { return di; };
  auto epi = [&](int row, W acc, W di, W vj) {
    dst[row] = mulw(di, acc);
    if (V) *v_at(d, V, row, vc) = vj;  // v_j at the diagonal = RN_W(src_row · inv), gathered above
  };
  auto dg = [&](int row) -> W { return mulw(ld_pol(src + row, pol_g), invW); };
  if (MERGE) csr_merge_stream<W, 1>(d, sh, s_stage, (const W*)d.aW, dinv, gat, pre, dg, epi);
  else csr_any_stream<W, L>(d, sh, s_stage, (const W*)d.aW, dinv, gat, pre, epi);
}
template <class W, int L>
__device__ void spmv_phase(const Dev& d, Shm& sh, char* s_stage, const W* __restrict__ src, double inv,
                           W* __restrict__ dst, W* __restrict__ V, int vc) {
  if (!d.block_stream && d.merge_stream) spmv_body<W, L, true>(d, sh, s_stage, src, inv, dst, V, vc);
  else spmv_body<W, L, false>(d, sh, s_stage, src, inv, dst, V, vc);
}

// ------------------------------------------------------------------ f2: ILU(0)
// Factorisation (reading R24), one launch per level of the lower
// dependency graph, one thread per row in the IKJ order of the oracle: for each
// k < i in row i (ascending) l_ik = a_ik / u_kk, then a_ij −= l_ik·u_kj over the
// columns j > k common to rows i and k (a merge of the two sorted rows).  Rows
// k belong to earlier levels (earlier launches).  A zero or non-finite pivot
// records the smallest such row in *bad.
template <class W>
__global__ void ilu_factor_level_kernel(const int* __restrict__ rp, const int* __restrict__ ci,
                                        const int* __restrict__ dpos, const int* __restrict__ rows, int cnt, W* f,
                                        int* bad) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt) return;
  const int i = rows[t];
  const int e_end = rp[i + 1], di = dpos[i];
  for (int e = rp[i]; e < di; ++e) {
    const int k = ci[e];
    const W lik = f[e] / f[dpos[k]];
    f[e] = lik;
    int p = e + 1;
    const int q_end = rp[k + 1];
    for (int q = dpos[k] + 1; q < q_end; ++q) {
      const int cj = ci[q];
      while (p < e_end && ci[p] < cj) ++p;
      if (p == e_end) break;
      if (ci[p] == cj) f[p] = subw(f[p], mulw(lik, f[q]));
    }
  }
  const W u = f[di];
  if (u == (W)0 || !isfinite((double)u)) atomicMin(bad, i);
}

// M⁻¹: out = U⁻¹ L⁻¹ in (in == out allowed), level by level over the whole grid
// with a grid barrier between levels; each row's sum runs sequentially in
// ascending column order in W, as in the oracle (bit-identical).  A thread
// takes slot gt of every level (level-ordered entry lists, built on the host)
// and loads the next level's row, columns, factor values, diagonal and
// right-hand side BEFORE the barrier, so after it only the ≤ ILU_KP solution
// values it depends on remain to be read (through L2: other CTAs wrote them).
// Slots beyond the first per thread and entries beyond ILU_KP take a plain loop.
constexpr int ILU_KP = 4;
// one slot's operands, packed so a level's prefetch is one round of independent
// 16-byte loads: {row, entries, first entry, –}, 4 columns, 4 factor values, the
// diagonal (U solve); entries beyond ILU_KP are read from the entry lists
template <class W>
struct alignas(16) IluRec {
  int row, ne, e0, pad;
  int col[ILU_KP];
  W val[ILU_KP];
  W diag;
  W pad2[16 / sizeof(W) - 1];
};

template <class W, int T>
__global__ void ilu_records_kernel(int n, const int* __restrict__ rows, const int* __restrict__ eoff,
                                   const int* __restrict__ ecol, const int* __restrict__ eidx,
                                   const int* __restrict__ dpos, const W* __restrict__ f, IluRec<W>* rec) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
    IluRec<W> r{};
    r.row = rows[s];
    r.e0 = eoff[s];
    r.ne = eoff[s + 1] - r.e0;
    for (int k = 0; k < ILU_KP; ++k) {
      r.col[k] = k < r.ne ? ecol[r.e0 + k] : 0;
      r.val[k] = k < r.ne ? f[eidx[r.e0 + k]] : (W)0;
    }
    r.diag = T == 1 ? f[dpos[r.row]] : (W)1;
    rec[s] = r;
  }
}

template <class W>
struct IluSlot {
  IluRec<W> r;
  W rhs;
  bool on;
};

template <class W, int T>
__device__ __forceinline__ void ilu_load(const Dev& d, const W* rhs_src, int slot, int end, IluSlot<W>& p) {
  p.on = slot < end;
  if (!p.on) return;
  using V4 = int4;
  const V4* src = reinterpret_cast<const V4*>(reinterpret_cast<const IluRec<W>*>(d.ilu_rec[T]) + slot);
  V4* dst = reinterpret_cast<V4*>(&p.r);
#pragma unroll
  for (int k = 0; k < (int)(sizeof(IluRec<W>) / 16); ++k) dst[k] = __ldg(src + k);
  if (d.tune & 32768) p.rhs = __ldcg(rhs_src + p.r.row);  // dev A/B: rhs before the barrier
}

template <class W, int T>
__device__ __forceinline__ void ilu_row(const Dev& d, const W* __restrict__ f, const IluSlot<W>& p, const W* rhs_src,
                                        W* out) {
  // the right-hand side is read with the solution values (one L2 round trip)
  const W rhs = (d.tune & 32768) ? p.rhs : __ldcg(rhs_src + p.r.row);
  W x[ILU_KP];
#pragma unroll
  for (int k = 0; k < ILU_KP; ++k)
    if (k < p.r.ne) x[k] = __ldcg(out + p.r.col[k]);
  W acc = rhs;
#pragma unroll
  for (int k = 0; k < ILU_KP; ++k)
    if (k < p.r.ne) acc = subw(acc, mulw(p.r.val[k], x[k]));
  for (int k = ILU_KP; k < p.r.ne; ++k)
    acc = subw(acc, mulw(f[d.ilu_eidx[T][p.r.e0 + k]], __ldcg(out + d.ilu_ecol[T][p.r.e0 + k])));
  out[p.r.row] = T == 1 ? acc / p.r.diag : acc;
}

template <class W, int T>
__device__ __forceinline__ bool ilu_solve(const Dev& d, Shm& sh, const W* rhs_src, W* out) {
  const W* __restrict__ f = (const W*)d.iluW;
  const int gt = sh.cta * NT + threadIdx.x, gs = d.G * NT;
  const int nl = d.ilu_nlev[T];
  const int* lev = d.ilu_lev[T];
  IluSlot<W> p;
  ilu_load<W, T>(d, rhs_src, lev[0] + gt, lev[1], p);
  for (int l = 0; l < nl; ++l) {
    const int a = lev[l], b = lev[l + 1];
    if (d.tune & 16384) {  // dev A/B: barriers only (wrong results)
      if (!grid_sync(d, sh)) return false;
      continue;
    }
    if (p.on) ilu_row<W, T>(d, f, p, rhs_src, out);
    for (int t = a + gt + gs; t < b; t += gs) {  // wide levels: further slots, plain loop
      const int row = d.ilu_rows[T][t];
      W acc = __ldcg(rhs_src + row);
      for (int e = d.ilu_eoff[T][t]; e < d.ilu_eoff[T][t + 1]; ++e)
        acc = subw(acc, mulw(f[d.ilu_eidx[T][e]], __ldcg(out + d.ilu_ecol[T][e])));
      out[row] = T == 1 ? acc / f[d.ilu_dpos[row]] : acc;
    }
    if (l + 1 < nl) ilu_load<W, T>(d, rhs_src, b + gt, lev[l + 2], p);
    // the next phase may stage the result with bulk copies (async proxy)
    if (T == 1 && l + 1 == nl) fence_proxy_async_global();
    if (!grid_sync(d, sh)) return false;
  }
  return true;
}

// Sync-free variant: no barrier per level.  Thread gt takes slots gt, gt + gs, …
// of the level-ordered slot list (so its rows come in non-decreasing level
// order).  A row's result is also stored into the publish buffer of its solve,
// which was filled with the all-ones bit pattern (a NaN that arithmetic never
// produces: the GPU returns the canonical NaN); a row polls the published
// values of all its inputs in one round of relaxed loads (re-polling only those
// still unpublished) and uses them directly — the value is its own ready flag,
// so no fence sits on the dependency chain.  (Measured on C2: a flag + release/
// acquire protocol ran 2× slower than the level-synchronous solve; polling the
// inputs one after another, 1.6× slower than one round.)  Progress: the lowest-level unfinished row has all its
// inputs done, and every thread is resident (cooperative launch); a watchdog
// raises the abort flag instead of hanging.  Each solve re-arms the other
// solve's buffer (the grid barrier between the solves orders it).
template <class W> struct PubBits;
template <> struct PubBits<float> { using U = unsigned; static constexpr U SENT = 0xffffffffu; };
template <> struct PubBits<double> { using U = unsigned long long; static constexpr U SENT = ~0ull; };

__device__ __forceinline__ unsigned ld_relaxed_bits(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_bits(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_bits(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_bits(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// one input of a row beyond the first ILU_KP (27-point stencils, long rows): poll until published
template <class W>
__device__ __forceinline__ bool ilu_take(const Dev& d, const typename PubBits<W>::U* pub, int col, W& x) {
  using U = typename PubBits<W>::U;
  U v = ld_relaxed_bits(pub + col);
  if (v != PubBits<W>::SENT) { x = *reinterpret_cast<W*>(&v); return true; }
  const unsigned long long t0 = globaltimer();
  for (int it = 0;; ++it) {
    v = ld_relaxed_bits(pub + col);
    if (v != PubBits<W>::SENT) { x = *reinterpret_cast<W*>(&v); return true; }
    if ((it & 63) == 63) {
      if (*(volatile int*)d.abort_flag) return false;
      if ((long long)(globaltimer() - t0) > d.timeout_ns) { atomicExch(d.abort_flag, 1); return false; }
    }
  }
}

template <class W, int T>
__device__ __forceinline__ bool ilu_solve_sf(const Dev& d, Shm& sh, const W* rhs_src, W* out) {
  using U = typename PubBits<W>::U;
  const W* __restrict__ f = (const W*)d.iluW;
  const int gt = sh.cta * NT + threadIdx.x, gs = d.G * NT, n = d.n;
  U* pub = reinterpret_cast<U*>(d.ilu_pub[T]);
  U* other = reinterpret_cast<U*>(d.ilu_pub[1 - T]);
  for (int i = gt; i < n; i += gs) other[i] = PubBits<W>::SENT;  // re-arm the other solve's buffer
  bool ok = true;
  for (int s = gt; s < n && ok; s += gs) {
    IluSlot<W> p;
    ilu_load<W, T>(d, rhs_src, s, n, p);
    // all inputs polled in one round (re-polling only those still unpublished)
    W acc = __ldcg(rhs_src + p.r.row);
    U v[ILU_KP];
#pragma unroll
    for (int k = 0; k < ILU_KP; ++k) v[k] = k < p.r.ne ? ld_relaxed_bits(pub + p.r.col[k]) : (U)0;
    {
      unsigned long long t0 = 0;
      for (int it = 0;; ++it) {
        bool pend = false;
#pragma unroll
        for (int k = 0; k < ILU_KP; ++k) pend |= v[k] == PubBits<W>::SENT;
        if (!pend) break;
#pragma unroll
        for (int k = 0; k < ILU_KP; ++k)
          if (v[k] == PubBits<W>::SENT) v[k] = ld_relaxed_bits(pub + p.r.col[k]);
        if ((it & 63) == 63) {
          const unsigned long long t = globaltimer();
          if (t0 == 0) t0 = t;
          if (*(volatile int*)d.abort_flag) { ok = false; break; }
          if ((long long)(t - t0) > d.timeout_ns) { atomicExch(d.abort_flag, 1); ok = false; break; }
        }
      }
    }
    W x[ILU_KP];
#pragma unroll
    for (int k = 0; k < ILU_KP; ++k) x[k] = *reinterpret_cast<const W*>(&v[k]);
#pragma unroll
    for (int k = 0; k < ILU_KP; ++k)
      if (k < p.r.ne) acc = subw(acc, mulw(p.r.val[k], x[k]));
    for (int k = ILU_KP; k < p.r.ne && ok; ++k) {
      W xk;
      ok = ilu_take<W>(d, pub, d.ilu_ecol[T][p.r.e0 + k], xk);
      acc = subw(acc, mulw(f[d.ilu_eidx[T][p.r.e0 + k]], xk));
    }
    if (!ok) break;
    const W res = T == 1 ? acc / p.r.diag : acc;
    out[p.r.row] = res;
    st_relaxed_bits(pub + p.r.row, *reinterpret_cast<const U*>(&res));
  }
  if (T == 1) fence_proxy_async_global();  // the next phase may stage the result with bulk copies
  return grid_sync(d, sh) && ok;
}

// seq: this apply's index within the launch (unused by the value-publishing solves)
template <class W>
__device__ __noinline__ bool ilu_apply_phase(const Dev& d, Shm& sh, const W* in, W* out, unsigned seq) {
  (void)seq;
  if (!(d.tune & 65536)) {  // sync-free (default)
    if (!ilu_solve_sf<W, 0>(d, sh, in, out)) return false;
    return ilu_solve_sf<W, 1>(d, sh, out, out);
  }
  if (!ilu_solve<W, 0>(d, sh, in, out)) return false;  // L y = in (unit lower), level-synchronous
  return ilu_solve<W, 1>(d, sh, out, out);              // U out = y
}

// fp32 ILU(0) inside the fp64 solver (the paper's single-precision
// ILU arm; oracle F_ILU32): out = (double) U32⁻¹ L32⁻¹ RN32(in), the fp32 solves
// on scratch vectors (in == out allowed).
static __device__ __noinline__ bool ilu_apply_f32(const Dev& d, Shm& sh, const double* in, double* out) {
  float* a = d.ilu_s32[0];
  float* b = d.ilu_s32[1];
  const int gt = sh.cta * NT + threadIdx.x, gs = d.G * NT;
  for (int i = gt; i < d.n; i += gs) a[i] = __double2float_rn(__ldcg(in + i));
  if (!grid_sync(d, sh)) return false;  // the solves read any row of the right-hand side
  if (!ilu_apply_phase<float>(d, sh, a, b, 0u)) return false;
  for (int i = gt; i < d.n; i += gs) out[i] = (double)__ldcg(b + i);
  fence_proxy_async_global();  // the next phase may stage `out` with bulk copies
  return grid_sync(d, sh);      // later phases read rows by CTA partition
}
template <class W>
__device__ __forceinline__ bool ilu_apply_any(const Dev& d, Shm& sh, const W* in, W* out, unsigned seq) {
  if constexpr (sizeof(W) == 8) {
    if (d.ilu32) return ilu_apply_f32(d, sh, in, out);
  }
  return ilu_apply_phase<W>(d, sh, in, out, seq);
}

// ------------------------------------------------------------------ a3
// One fused MGS sweep over the CTA's rows:
//   w ← RN_W(w − RN_W(RN_W(h_prev)·v_prev))  (line 155 of step i−1), then
//   the partial of h_i = w·v_next (line 154 of step i), or of ‖w‖² when
//   v_next == nullptr (line 104).  fp64 accumulation (reading R9).
template <class W>
__device__ __noinline__ double mgs_sweep(int r0, int r1, W* __restrict__ w, const W* __restrict__ vprev, W hprev,
                            const W* __restrict__ vnext) {
  using V4 = typename VecT<W>::T;
  constexpr int N = VecT<W>::N;
  constexpr int UB = 2;  // independent 16-byte loads in flight per array per thread (noinline: register budget)
  double acc = 0.0;
  const int q0 = r0 / N, q1 = r1 / N;
  for (int qb = q0 + threadIdx.x; qb < q1; qb += UB * NT) {
    V4 a[UB], b[UB], c[UB];
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const int q = qb + u * NT;
      if (q < q1) {
        a[u] = reinterpret_cast<V4*>(w)[q];
        if (vprev) b[u] = reinterpret_cast<const V4*>(vprev)[q];
        if (vnext) c[u] = reinterpret_cast<const V4*>(vnext)[q];
      }
    }
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const int q = qb + u * NT;
      if (q < q1) {
        if (vprev) {
          sub_scaled(a[u], b[u], hprev);
          reinterpret_cast<V4*>(w)[q] = a[u];
        }
        if (vnext) {
          acc += dotv(a[u], c[u]);
        } else {
          acc += dotv(a[u], a[u]);
        }
      }
    }
  }
  return acc;
}

// ------------------------------------------------------------------ a4/a8
// Row-tile passes over the CTA's rows with the V tile (and, for MODE 1–3, the
// w tile) staged in shared memory by TMA bulk copies, one per column segment,
// double buffered on mbar_t: a tile is T rows × ncols columns, T chosen so a
// buffer fills half the staging region; each pass reads V once from HBM.
//   MODE 1: acc_i += Σ_r V_ri w_r                          (CGS pass, line 161)
//   MODE 2: w ← RN_W(w − Σ_i V_i c_i), then acc_i += Vᵀw   (line 162 + the next line 161)
//   MODE 3: w ← RN_W(w − Σ_i V_i c_i), nn += ‖w‖²          (line 162 + line 104)
//   MODE 4: x_r += Σ_i (double)V_ri · y_i                   (lines 145–147, fp64)
// V·c is summed in W per row with i ascending (reading R2/R9).  Dots: warp w
// owns a fixed share of every tile's rows and lane l the columns l, l+32, …;
// each lane accumulates dotv partials in fp64 registers over all tiles, and
// the per-warp column partials (s_acc[warp][i]) are summed over the warps in
// order by combine_acc: deterministic, no per-tile shuffles.  Column segments
// sit TP = T + 16/w_B elements apart so that the lanes' 16-byte reads of one
// row group hit distinct banks.
constexpr int MAXSLOT = (MAX_M + 1 + 31) / 32;  // columns per lane
template <class W, int MODE>
__device__ __forceinline__ void rowtile_pass(const Dev& d, Shm& sh, int r0, int r1, const W* V, long long ldv,
                                             int ncols, W* w, const W* s_coefW, const double* s_y, double* s_acc,
                                             char* s_tiles, double& nn, int dir = 0, bool reuse = false) {
  using V4 = typename VecT<W>::T;
  constexpr int N = VecT<W>::N;
  constexpr int NTB = G200_NTB;  // ring depth
  constexpr int NWS = MODE == 4 ? 0 : 1;  // w tile staged (MODE 1-3)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nrows = r1 - r0;  // multiple of ROWALIGN
  double dacc[MAXSLOT];
#pragma unroll
  for (int t = 0; t < MAXSLOT; ++t) dacc[t] = 0.0;
  const int half = (d.tile_bytes / NTB) & ~127;
  constexpr int PADE = 16 / (int)sizeof(W);
  // tile geometry: element (tile row t, column i) at (t >> lg)·bsz + i·cs + (t & msk)
  int T, cs, lg, msk, bsz, woff;
  if (d.vtb) {  // row-blocked V: whole blocks per tile, one copy per block
    const int nbt = max(1, half / ((ncols * d.vtp + d.vtb) * (int)sizeof(W)));
    T = min(nbt * d.vtb, nrows);
    cs = d.vtp; lg = d.vtb_log; msk = d.vtb - 1; bsz = ncols * d.vtp;
    woff = nbt * bsz;
  } else {      // column-major V: one copy per column segment
    T = (half / ((ncols + 1) * (int)sizeof(W)) - PADE) & ~(ROWALIGN - 1);
    T = max(ROWALIGN, min(T, nrows));
    cs = T + PADE; lg = 30; msk = (1 << 30) - 1; bsz = 0;
    woff = ncols * cs;
  }
  auto el = [&](int t, int i) { return (size_t)(t >> lg) * bsz + (size_t)i * cs + (t & msk); };
  const int ntile = nrows > 0 ? (nrows + T - 1) / T : 0;
  unsigned ph = sh.tphase;
  auto buf = [&](int b) { return reinterpret_cast<W*>(s_tiles + (size_t)b * half); };
  // w rows of the tile are staged too (MODE 1-3); every generic store of w of
  // this CTA is followed by fence.proxy.async (csr_stream, this pass)
  auto issue = [&](int k) {  // warp 0
    const int rows = min(T, nrows - k * T);
    const long long row0 = r0 + (long long)k * T;
    const unsigned bytes = (unsigned)rows * (unsigned)sizeof(W);
    W* dst = buf(k % NTB);
    unsigned long long* bar = &sh.mbar_t[k % NTB];
    if (d.vtb) {
      const int nb = rows >> lg;  // CTA row ranges are block aligned
      const unsigned bb = (unsigned)(ncols * d.vtp) * (unsigned)sizeof(W);
      if (lane == 0) mbar_expect_tx(bar, bb * (unsigned)nb + (NWS ? bytes : 0u));
      __syncwarp();
      for (int b = lane; b < nb; b += 32) tma_load_1d(dst + (size_t)b * bsz, V + ((row0 >> lg) + b) * d.vbs, bb, bar);
      if (NWS && lane == 31) tma_load_1d(dst + woff, w + row0, bytes, bar);
    } else {
      if (lane == 0) mbar_expect_tx(bar, bytes * (unsigned)(ncols + NWS));
      __syncwarp();
      for (int i = lane; i < ncols + NWS; i += 32)
        tma_load_1d(i < ncols ? dst + (size_t)i * cs : dst + woff, (i < ncols ? V + (long long)i * ldv : w) + row0, bytes,
                    bar);
    }
  };
  // tiles in the pass's order: forward or reverse (dir); tile k always in buffer
  // k mod NTB.  reuse: the previous pass ran over the same tiles in the other
  // direction, so this pass's first min(NTB, ntile) tiles are still staged (its
  // last ones) — no copy, no wait — and the rest start where its reads ended
  // (the most recently streamed V rows, the ones left in L2).
  auto tile_of = [&](int kk) { return dir ? ntile - 1 - kk : kk; };
  auto staged = [&](int kk) { return reuse && kk < NTB; };
  if (warp == 0)
    for (int kk = 0; kk < NTB - 1 && kk < ntile; ++kk)
      if (!staged(kk)) issue(tile_of(kk));
  for (int kk = 0; kk < ntile; ++kk) {
    const int k = tile_of(kk);
    const int b = k % NTB;
    // the buffer of the tile before last is free (barrier at the end of its iteration)
    if (warp == 0 && kk + NTB - 1 < ntile && !staged(kk + NTB - 1)) issue(tile_of(kk + NTB - 1));
    if (!staged(kk)) {
      const unsigned par = (ph >> b) & 1u;
      ph ^= (1u << b);
      if (!mbar_try_wait(&sh.mbar_t[b], par)) {
        const unsigned long long t0 = globaltimer();
        while (!mbar_try_wait(&sh.mbar_t[b], par))
          if ((long long)(globaltimer() - t0) > d.timeout_ns) { atomicExch(d.abort_flag, 1); break; }
      }
    }
    const int rows = min(T, nrows - k * T);
    const int row0 = r0 + k * T;
    const W* VT = buf(b);
    W* s_w = buf(b) + woff;
    // step a: one thread per 16-byte row group (N rows: N independent chains,
    // one shared load per column)
    if (MODE != 1) {
      for (int g = threadIdx.x; g < rows / N; g += NT) {
        const int t = g * N;
        if (MODE == 4) {
          double u[N];
#pragma unroll
          for (int r = 0; r < N; ++r) u[r] = 0.0;
#pragma unroll 4
          for (int i = 0; i < ncols; ++i) {
            const double yi = s_y[i];
            const V4 v = *reinterpret_cast<const V4*>(VT + el(t, i));
            const W* pv = reinterpret_cast<const W*>(&v);
#pragma unroll
            for (int r = 0; r < N; ++r) u[r] = __dadd_rn(u[r], __dmul_rn((double)pv[r], yi));
          }
#pragma unroll
          for (int r = 0; r < N; ++r)
            if (row0 + t + r < d.n) d.x[row0 + t + r] = d.x[row0 + t + r] + u[r];
        } else {
          W acc[N];
#pragma unroll
          for (int r = 0; r < N; ++r) acc[r] = (W)0;
#pragma unroll 4
          for (int i = 0; i < ncols; ++i) {
            const W ci = s_coefW[i];
            const V4 v = *reinterpret_cast<const V4*>(VT + el(t, i));
            const W* pv = reinterpret_cast<const W*>(&v);
#pragma unroll
            for (int r = 0; r < N; ++r) acc[r] = addw(acc[r], mulw(pv[r], ci));
          }
          V4 wv = *reinterpret_cast<const V4*>(s_w + t);
          W* pw = reinterpret_cast<W*>(&wv);
#pragma unroll
          for (int r = 0; r < N; ++r) pw[r] = subw(pw[r], acc[r]);
          *reinterpret_cast<V4*>(w + row0 + t) = wv;
          if (MODE == 2) *reinterpret_cast<V4*>(s_w + t) = wv;
          if (MODE == 3) nn += dotv(wv, wv);
        }
      }
    }
    if (MODE == 1 || MODE == 2) {
      if (MODE == 2) __syncthreads();  // s_w complete
      const int nq = rows / N;
      const int qa = (warp * nq) / NW, qb = ((warp + 1) * nq) / NW;
      const V4* wq = reinterpret_cast<const V4*>(s_w);
#pragma unroll
      for (int sl = 0; sl < MAXSLOT; ++sl) {
        const int i = lane + 32 * sl;
        if (32 * sl < ncols && i < ncols) {
          // four independent accumulators (fixed structure: deterministic)
          double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
          int q = qa;
          for (; q + 3 < qb; q += 4) {
            p0 += dotv(*reinterpret_cast<const V4*>(VT + el(q * N, i)), wq[q]);
            p1 += dotv(*reinterpret_cast<const V4*>(VT + el((q + 1) * N, i)), wq[q + 1]);
            p2 += dotv(*reinterpret_cast<const V4*>(VT + el((q + 2) * N, i)), wq[q + 2]);
            p3 += dotv(*reinterpret_cast<const V4*>(VT + el((q + 3) * N, i)), wq[q + 3]);
          }
          for (; q < qb; ++q) p0 += dotv(*reinterpret_cast<const V4*>(VT + el(q * N, i)), wq[q]);
          dacc[sl] += (p0 + p1) + (p2 + p3);
        }
      }
    }
    __syncthreads();  // buffer b free
  }
  if (MODE == 1 || MODE == 2) {
#pragma unroll
    for (int sl = 0; sl < MAXSLOT; ++sl) {
      const int i = lane + 32 * sl;
      if (i < ncols) s_acc[warp * d.kmax + i] = dacc[sl];
    }
  }
  if (threadIdx.x == 0) sh.tphase = ph;  // every thread read it at entry, before the barriers above
  if (MODE == 2 || MODE == 3) fence_proxy_async_global();  // w is staged by TMA in the next pass
  __syncthreads();
}

// per-CTA column partials for the all-reduce: warps in order
__device__ __forceinline__ void combine_acc(const Dev& d, const double* s_acc, int ncols, double* s_part) {
  for (int i = threadIdx.x; i < ncols; i += NT) {
    double v = 0.0;
    for (int w = 0; w < NW; ++w) v += s_acc[w * d.kmax + i];
    s_part[i] = v;
  }
  __syncthreads();
}

// ------------------------------------------------------------------ a6
// Alg. 1 lines 108–140 for step j (1-based) on h[0..j] (fp64, reading R4/R7):
// apply rotations 1..j−1, form rotation j, rotate s.  Returns |s_{j+1}|.
// (the rotated h[i] is carried to the next rotation in a register: the chain no longer
// goes through a shared-memory store and load per rotation — same operations)
__device__ __forceinline__ double hess_step(int j, double* __restrict__ h, double* __restrict__ cs,
                                            double* __restrict__ sn, double* __restrict__ s) {
  double t1 = h[0];
  for (int i = 1; i <= j - 1; ++i) {
    const double t2 = h[i];
    const double c = cs[i - 1], sg = sn[i - 1];
    h[i - 1] = __dadd_rn(__dmul_rn(c, t1), __dmul_rn(sg, t2));
    t1 = __dadd_rn(__dmul_rn(-sg, t1), __dmul_rn(c, t2));
  }
  const double a = t1, b = h[j];
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
__device__ inline void backsolve_cta(int J, const double* R, int ldr, const double* s, double* s_rhs, double* y_out,
                              double* s_y) {
  for (int k = threadIdx.x; k < J; k += NT) s_rhs[k] = s[k];
  __syncthreads();
  for (int i = J - 1; i >= 0; --i) {
    if (threadIdx.x == 0) s_y[i] = s_rhs[i] / __ldcg(R + (size_t)i * ldr + i);
    __syncthreads();
    const double yi = s_y[i];
    for (int k = threadIdx.x; k < i; k += NT)
      s_rhs[k] = __dsub_rn(s_rhs[k], __dmul_rn(__ldcg(R + (size_t)i * ldr + k), yi));
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
    auto take = [&](size_t bytes) { size_t r = o; o += (bytes + 127) & ~size_t(127); return r; };
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

__host__ inline void set_smem_offsets(Dev& d) {
  const SmemLayout lay(d.kmax, d.tile_bytes);
  const size_t o[11] = {lay.off_part, lay.off_out, lay.off_tmp, lay.off_h, lay.off_cs, lay.off_sn,
                        lay.off_s, lay.off_y, lay.off_rhs, lay.off_coef, lay.off_tiles};
  for (int i = 0; i < 11; ++i) d.soff[i] = (int)o[i];
}

#define CTA_INDEX ((int)blockIdx.x)
#define G200_SMEM_CARVE(W)                                                  \
  extern __shared__ __align__(128) char dsm[];                              \
  __shared__ Shm sh;                                                        \
  const SmemLayout lay(d.kmax, d.tile_bytes);                               \
  double* s_part = reinterpret_cast<double*>(dsm + lay.off_part);           \
  double* s_out = reinterpret_cast<double*>(dsm + lay.off_out);             \
  double* s_tmp = reinterpret_cast<double*>(dsm + lay.off_tmp);             \
  double* s_h = reinterpret_cast<double*>(dsm + lay.off_h);                 \
  double* s_cs = reinterpret_cast<double*>(dsm + lay.off_cs);               \
  double* s_sn = reinterpret_cast<double*>(dsm + lay.off_sn);               \
  double* s_s = reinterpret_cast<double*>(dsm + lay.off_s);                 \
  double* s_y = reinterpret_cast<double*>(dsm + lay.off_y);                 \
  double* s_rhs = reinterpret_cast<double*>(dsm + lay.off_rhs);             \
  W* s_coefW = reinterpret_cast<W*>(dsm + lay.off_coef);                    \
  char* s_tiles = dsm + lay.off_tiles;                                      \
  (void)s_part; (void)s_out; (void)s_tmp; (void)s_h; (void)s_cs; (void)s_sn; \
  (void)s_s; (void)s_y; (void)s_rhs; (void)s_coefW; (void)s_tiles;          \
  init_shm(sh, CTA_INDEX);

// ------------------------------------------------------------------ a3 (resident)
// MGS with the CTA's rows of w in registers and the basis
// vectors streamed through a ring of NB shared-memory buffers by TMA bulk
// copies: step i forms w ← RN_W(w − RN_W(h_{i−1})·v_{i−1}) and the partial of
// h_i = w·v_i in one pass (v_{i−1}, v_i read from the ring); right after the
// CTA barrier of h_i's all-reduce the buffer of v_{i−1} is free and the copy
// of v_{i+NB−1} is issued into it, so the HBM reads of the next vectors overlap
// the all-reduce and no register holds an in-flight load across it.  Same
// operations and order per element as mgs_sweep.
constexpr int MGS_MV = 8;  // 16-byte vectors of w per thread in registers (both resident variants)
#ifndef G200_MGS_GRP
#define G200_MGS_GRP 4
#endif
constexpr int MGS_GRP = G200_MGS_GRP;  // vectors whose shared-memory loads are issued together (mgs_resident)
template <class W>
__device__ __forceinline__ bool mgs_resident(const Dev& d, Shm& sh, int r0, int r1, int j, const W* V, long long ldv,
                                             W* w, double* s_h, char* s_tiles, double& NN) {
  using V4 = typename VecT<W>::T;
  constexpr int N = VecT<W>::N;
  const int q0 = r0 / N, nq = r1 / N - q0;
  const int nqa = (nq + 7) & ~7;  // 128-byte aligned buffers
  const int NB = d.mgs_nbuf;
  V4* sv = reinterpret_cast<V4*>(s_tiles);
  const unsigned bytes = (unsigned)nq * 16u;
  unsigned ph = sh.vphase;
  // copies are issued by warp 0 (TMA_T): warp 1 performs the all-reduce's release
  constexpr int TMA_T = 0;
  auto issue_to = [&](int c, int b) {  // one thread: v_c (1-based) → buffer b = (c−1) mod NB
    char* dst = reinterpret_cast<char*>(sv + (size_t)b * nqa);
    const char* src = reinterpret_cast<const char*>(V + (long long)(c - 1) * ldv + r0);
    mbar_expect_tx(&sh.mbar_v[b], bytes);
    for (unsigned o = 0; o < bytes; o += 32768u)
      tma_load_1d(dst + o, src + o, min(32768u, bytes - o), &sh.mbar_v[b]);
  };
  auto issue = [&](int c) { issue_to(c, (c - 1) % NB); };
  auto wait = [&](int b) -> bool {
    const unsigned par = (ph >> b) & 1u;
    ph ^= (1u << b);
    if (mbar_try_wait(&sh.mbar_v[b], par)) return true;
    const unsigned long long t0 = globaltimer();
    for (;;) {
      if (mbar_try_wait(&sh.mbar_v[b], par)) return true;
      if ((long long)(globaltimer() - t0) > d.timeout_ns) { atomicExch(d.abort_flag, 1); return false; }
    }
  };
  if (threadIdx.x == TMA_T)
    for (int c = 1; c <= min(NB - 1, j); ++c) issue(c);
  V4 wr[MGS_MV];
  {
    const V4* wg = reinterpret_cast<const V4*>(w) + q0;
#pragma unroll
    for (int k = 0; k < MGS_MV; ++k) {
      const int t = threadIdx.x + k * NT;
      if (t < nq) wr[k] = wg[t];
    }
  }
  W hprev = (W)0;
  const int nk = (nq + NT - 1) / NT;  // vectors per thread that hold rows (of thread 0; ≤ MGS_MV)
  const bool lead = d.profile && sh.cta == 0 && threadIdx.x == 0;
  unsigned long long tp = lead ? globaltimer() : 0ull;
  auto tick = [&](int slot) {
    if (lead) { const unsigned long long t = globaltimer(); d.prof[slot] += t - tp; tp = t; }
  };
  // The ring copy of v_{i+NB−2} is issued at the start of step i, into the buffer step
  // i−1's update freed: its reads run under step i's shared-memory-only update + dot and
  // the CTA has no copy in flight when the all-reduce's round trips start, which a copy
  // issued in the all-reduce (the earlier r02 schedule) slowed.  C2 mixed MGS whole solve
  // (r02): 89.5 ms (copy in the all-reduce) → 82.7 (same + an L2 prefetch a step ahead)
  // → 79.4 (early copy; the prefetch on top: 79.2, not kept); the ortho phase 67.4 → 57.5 ms.
  // (a ring of two buffers has no free buffer at the start of a step: the copy of
  // v_{i+1} then goes in the all-reduce, into v_{i−1}'s buffer)
  const bool early = NB >= 3 && !(d.tune & 536870912);  // (bit 29, set by the host: copy in the all-reduce)
  // (b, bp: the ring buffers of v_i and v_{i−1}, stepped without the runtime modulo that sat on
  // every step's critical path — 5.6 % of the MGS launch's stall samples, ncu r02)
  int b = NB - 1, bp = NB - 2;
  for (int i = 1; i <= j; ++i) {
    bp = b;
    b = b + 1 == NB ? 0 : b + 1;
    if (early && threadIdx.x == TMA_T && i >= 2 && i + NB - 2 <= j) issue_to(i + NB - 2, b >= 2 ? b - 2 : b - 2 + NB);
    // (r02, measured and not kept: an L2 prefetch of the vector after it — no change, 55.9 vs
    // 55.3 ms; the copy inside the step's all-reduce instead, tune bit 28 — 57.4 ms)
    wait(b);
    tick(8);
    const V4* X = sv + (size_t)b * nqa;                       // v_i
    // v_{i−1}; at i = 1 there is no update: h = 0 against v_1 leaves w as it is
    // (RN_W(w − RN_W(0·v)) = w), so the loop below carries no branch on i
    const V4* Y = i > 1 ? sv + (size_t)bp * nqa : X;
    double acc = 0.0;
    // Pairs of this thread's vectors: the four shared-memory loads of a pair are issued
    // together from clamped indices (no branch between them — with `if (t < nq)` around
    // each vector the eight iterations ran strictly one after the other, two dependent
    // LDS latencies each: the step was latency-bound at 4 warps per scheduler), a thread
    // past the end of the row block just does not add its product.  Same operations on
    // every valid element and the same order of the fp64 adds as before.
#pragma unroll
    for (int k = 0; k < MGS_MV; k += MGS_GRP) {
      if (k < nk) {  // (CTA-uniform)
        V4 ys[MGS_GRP], xs[MGS_GRP];
#pragma unroll
        for (int u = 0; u < MGS_GRP; ++u) {
          const int c = min((int)threadIdx.x + (k + u) * NT, nq - 1);
          ys[u] = Y[c];
          xs[u] = X[c];
        }
#pragma unroll
        for (int u = 0; u < MGS_GRP; ++u) {  // (no branch on k + u < nk: the compiler sinks the loads under it)
          sub_scaled(wr[k + u], ys[u], hprev);
          const double p = dotv(wr[k + u], xs[u]);
          if ((int)threadIdx.x + (k + u) * NT < nq) acc += p;
        }
      }
    }
    tick(9);
    double h;
    auto mid = [&]() {
      if (!early && threadIdx.x == TMA_T && i + NB - 1 <= j) issue(i + NB - 1);  // into v_{i−1}'s buffer
    };
    if (!allreduce1<true>(d, sh, acc, false, h, mid)) return false;
    if (threadIdx.x == 0) s_h[i - 1] = h;
    hprev = RN<W>(h);
    tick(10);
  }
  // final update w ← w − h_j v_j, ‖w‖², w back to global for the next SpMV
  double nn = 0.0;
  {
    const V4* X = sv + (size_t)b * nqa;  // v_j (j ≥ 1)
    V4* wg = reinterpret_cast<V4*>(w) + q0;
#pragma unroll
    for (int k = 0; k < MGS_MV; ++k) {
      const int t = threadIdx.x + k * NT;
      if (t < nq) {
        sub_scaled(wr[k], X[t], hprev);
        nn += dotv(wr[k], wr[k]);
        wg[t] = wr[k];
      }
    }
  }
  if (threadIdx.x == 0) sh.vphase = ph;  // read by every thread at entry, before the syncs below
  NN = nn;  // this thread's share of ‖w‖²; the caller pushes the halo and all-reduces it
  return true;
}

// ------------------------------------------------------------------ a3 (chunk ring)
// MGS with the CTA's rows of w on chip and the basis
// streamed through a ring of d.mgs_nbuf chunk slots of MGS_CHUNK bytes in
// shared memory by TMA bulk copies.  Chunk k of a CTA's row block holds the
// 16-byte vector k·NT + t of thread t: w's chunks k < MGS_MV sit in thread
// registers, the rest (d.mgs_wsm of them) in shared memory after the ring,
// and a thread reads exactly its own vector of each basis chunk.  The chunks of
// v_1, v_2, … form one stream (counter sh.vg, persistent over the kernel: the
// parity of stream chunk g's barrier is (g / nslots) & 1) that runs as far
// ahead as the ring allows: the slots of v_i are refilled as soon as
// w ← RN_W(w − RN_W(h_i)·v_i) (line 155) has read them, so the reads of the
// next vectors overlap h_i's all-reduce.  Step i: partial of h_i = w·v_i
// (line 154), all-reduce, update with v_i.  Same operations and order per
// element as mgs_sweep.  (Used when two whole vectors do not fit on chip:
// the unfused update costs a pass and a barrier per step, mgs_resident.)
constexpr int MGS_CHUNK = NT * 16;    // bytes of one ring slot = one vector of every thread
constexpr int MGS_MAXSLOT = 32;       // ring slots (barriers in Shm)
constexpr int MGS_STREAM_SLOTS = 4;   // item slots of the streamed MGS (mgs_stream): 4 × 32 KB of operands in flight
template <class W>
__device__ __forceinline__ bool mgs_chunked(const Dev& d, Shm& sh, int r0, int r1, int j, const W* V, long long ldv,
                                             W* w, double* s_h, char* s_tiles, double& NN) {
  using V4 = typename VecT<W>::T;
  constexpr int N = VecT<W>::N;
  const int q0 = r0 / N, nq = r1 / N - q0;
  const int nch = (nq + NT - 1) / NT;  // chunks per basis vector
  const unsigned NS = (unsigned)d.mgs_nbuf;
  const unsigned g0 = sh.vg;           // stream index of v_1's first chunk
  const unsigned gend = g0 + (unsigned)(j * nch);
  V4* sv = reinterpret_cast<V4*>(s_tiles);
  V4* ws = sv + (size_t)NS * NT - (size_t)MGS_MV * NT;  // w's chunk k ≥ MGS_MV at ws + k·NT
  // lanes of warp 0 issue stream chunks [lo, hi), one chunk per lane and round
  // (warp 1 performs the all-reduce's release)
  auto issue = [&](unsigned lo, unsigned hi) {
    if (threadIdx.x < 32)
      for (unsigned g = lo + (threadIdx.x & 31); g < hi; g += 32) {
        const unsigned rel = g - g0;
        const int c = (int)(rel / (unsigned)nch), k = (int)(rel % (unsigned)nch);
        const unsigned bytes = (unsigned)min(NT, nq - k * NT) * 16u;
        const unsigned s = g % NS;
        mbar_expect_tx(&sh.mbar_v[s], bytes);
        tma_load_1d(sv + (size_t)s * NT, V + (long long)c * ldv + r0 + (long long)k * NT * N, bytes, &sh.mbar_v[s]);
      }
  };
  auto wait = [&](unsigned s, unsigned par) -> bool {  // slot and parity of a stream chunk
    if (mbar_try_wait(&sh.mbar_v[s], par)) return true;
    const unsigned long long t0 = globaltimer();
    for (;;) {
      if (mbar_try_wait(&sh.mbar_v[s], par)) return true;
      if ((long long)(globaltimer() - t0) > d.timeout_ns) { atomicExch(d.abort_flag, 1); return false; }
    }
  };
  unsigned issued = min(gend, g0 + NS);
  issue(g0, issued);
  V4 wr[MGS_MV];
  const V4* wg = reinterpret_cast<const V4*>(w) + q0;
#pragma unroll
  for (int k = 0; k < MGS_MV; ++k) {
    const int t = threadIdx.x + k * NT;
    if (t < nq) wr[k] = wg[t];
  }
  for (int t = threadIdx.x + MGS_MV * NT; t < nq; t += NT) ws[t] = wg[t];
  const bool lead = d.profile && sh.cta == 0 && threadIdx.x == 0;
  unsigned long long tp = lead ? globaltimer() : 0ull;
  auto tick = [&](int slot) {
    if (lead) { const unsigned long long t = globaltimer(); d.prof[slot] += t - tp; tp = t; }
  };
  // v_{i+2} is prefetched into L2 at the start of step i, so the ring refills issued in
  // the all-reduce are L2 hits (C2 fp64 MGS 160.8 → 154–159 ms; measured r02: refilling the
  // freed slots at the start of the step instead — the resident ring's schedule — 167 ms)
  const unsigned vbytes = (unsigned)nq * 16u;
  int sv0 = (int)(g0 % NS);
  unsigned qv0 = g0 / NS;
  for (int i = 1; i <= j; ++i) {
    const unsigned gi = g0 + (unsigned)((i - 1) * nch);  // v_i's first chunk
    // v_i's chunks sit in slots s0, s0+1, … (mod NS; NS ≥ nch); s0 = gi mod NS and qv = gi / NS
    // are stepped (no runtime division per chunk wait)
    const int s0 = sv0;
    const unsigned q0v = qv0;
    auto wait_k = [&](int k) -> bool {
      const int sk = s0 + k;
      return sk < (int)NS ? wait((unsigned)sk, q0v & 1u) : wait((unsigned)(sk - (int)NS), (q0v + 1u) & 1u);
    };
    sv0 += nch;
    if (sv0 >= (int)NS) { sv0 -= (int)NS; ++qv0; }
    if (threadIdx.x == 32 && i + 2 <= j)
      for (unsigned o = 0; o < vbytes; o += 32768u)
        prefetch_l2(reinterpret_cast<const char*>(V + (long long)(i + 1) * ldv + r0) + o, min(32768u, vbytes - o));
    auto slot = [&](int k) -> const V4* {
      const int s = s0 + k < (int)NS ? s0 + k : s0 + k - (int)NS;
      return sv + (size_t)s * NT + threadIdx.x;
    };
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < MGS_MV; ++k) {
      if (k < nch) {
        if (!wait_k(k)) return false;
        if (threadIdx.x + k * NT < nq) acc += dotv(wr[k], *slot(k));
      }
    }
    for (int k = MGS_MV; k < nch; ++k) {
      if (!wait_k(k)) return false;
      if (threadIdx.x + k * NT < nq) acc += dotv(ws[k * NT + threadIdx.x], *slot(k));
    }
    tick(9);
    double h;
    // refill the slots freed by step i−1's update while the reduction is in flight
    // (a warp that issues bulk copies stalls until the TMA unit takes them)
    auto mid = [&]() {
      const unsigned hi = min(gend, gi + NS);
      if (hi > issued) issue(issued, hi);
    };
    if (!allreduce1<true>(d, sh, acc, false, h, mid)) return false;
    issued = max(issued, min(gend, gi + NS));
    if (threadIdx.x == 0) s_h[i - 1] = h;
    const W hw = RN<W>(h);
    auto upd = [&](V4& a, const V4& x) { sub_scaled(a, x, hw); };
#pragma unroll
    for (int k = 0; k < MGS_MV; ++k)
      if (threadIdx.x + k * NT < nq) upd(wr[k], *slot(k));
    for (int k = MGS_MV; k < nch; ++k)
      if (threadIdx.x + k * NT < nq) upd(ws[k * NT + threadIdx.x], *slot(k));
    __syncthreads();  // v_i's slots are free
    // v_{i+1}'s chunks not in flight yet (a ring of < 2 vectors) go now, the rest in step i+1's mid()
    const unsigned need = min(gend, gi + 2u * (unsigned)nch);
    if (need > issued) { issue(issued, need); issued = need; }
    tick(10);
  }
  // ‖w‖², w back to global for the next SpMV
  double nn = 0.0;
  V4* wo = reinterpret_cast<V4*>(w) + q0;
#pragma unroll
  for (int k = 0; k < MGS_MV; ++k) {
    const int t = threadIdx.x + k * NT;
    if (t < nq) {
      nn += dotv(wr[k], wr[k]);
      wo[t] = wr[k];
    }
  }
  for (int t = threadIdx.x + MGS_MV * NT; t < nq; t += NT) {
    const V4 a = ws[t];
    nn += dotv(a, a);
    wo[t] = a;
  }
  if (threadIdx.x == 0) sh.vg = gend;  // read by every thread at entry, before the syncs below
  NN = nn;  // this thread's share of ‖w‖²; the caller pushes the halo and all-reduces it
  return true;
}

// ------------------------------------------------------------------ a3 (streamed, w off chip)
// MGS for row blocks whose w does not fit on chip (C4: 113 k
// rows per CTA).  Chunk k of the CTA's rows = the 16-byte vector k·NT + t of
// every thread t (MGS_CHUNK bytes); an item = MGS_IC consecutive chunks of one
// basis vector, one bulk copy (single-thread bulk copies below ~16 KB are paced
// at ~0.4 µs each, tools/tma_bench.cu r02).  w: the first d.mgs_wsm chunks in
// shared memory (after the ring), the rest in global memory (the w buffer
// itself: thread t alone reads and writes its vectors, so plain loads —
// prefetched one item ahead — and evict_last stores keep it in L2 with no
// cross-proxy ordering; w in registers spilled).  Step i = 1..j in two passes:
//   A: the partial of h_i = w·v_i (line 154), all-reduce;
//   B: w ← RN_W(w − RN_W(h_i)·v_i) (line 155), and at i = j the partial of ‖w‖²
//      (line 104).
// v_i streams through a ring of NS = d.mgs_nbuf item slots by TMA twice — from
// HBM in A (evict_normal), from L2 in B right after the reduction (evict_first:
// its last use).  (Measured on C4, r02: a fused update-then-dot pass re-reads
// v_{i−1} a whole step later and misses in L2 — 20 % hit rate, 1.3× slower.)
// One kernel-lifetime item sequence (sh.vg; per step: A's items, then B's),
// slot = item mod NS, full barrier mbar_v (transaction bytes), consumed barrier
// mbar_e (one arrival per warp).  Thread 0 issues items up to NS ahead of its
// own consumption, after the consumed barrier of the slot's previous item; in
// the all-reduce (A's items all consumed) it fills the ring with B's items.
// Same operations and order per element and per thread partial as mgs_sweep /
// mgs_resident (bit-identical solves).
constexpr int MGS_IC = 4;                       // chunks per streamed item (32 KB)
#ifndef G200_PS
#define G200_PS 2
#endif
constexpr int MGS_PS = G200_PS;                 // register sets of global w in flight (items ahead)
constexpr int MGS_ITEM = MGS_IC * MGS_CHUNK;
__device__ __forceinline__ float4 ld_hint(const float4* p, unsigned long long pol) {
  float4 v;
  asm volatile("ld.global.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double2 ld_hint(const double2* p, unsigned long long pol) {
  double2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}
template <class W>
__device__ __forceinline__ bool mgs_stream(const Dev& d, Shm& sh, int r0, int r1, int j, const W* V, long long ldv,
                                           W* w, double* s_h, char* s_tiles, double& NN) {
  using V4 = typename VecT<W>::T;
  constexpr int N = VecT<W>::N;
  const int lane = threadIdx.x & 31;
  const int q0 = r0 / N, nq = r1 / N - q0;
  const int nch = (nq + NT - 1) / NT;
  const int nit = (nch + MGS_IC - 1) / MGS_IC;  // items per pass
  const unsigned NS = (unsigned)d.mgs_nbuf;
  const int MG = min(nch, d.mgs_wsm);           // first global w chunk (a multiple of MGS_IC)
  V4* sv = reinterpret_cast<V4*>(s_tiles);
  V4* ws = sv + (size_t)NS * MGS_IC * NT;       // shared w chunk k < MG at ws + k·NT
  V4* wg = reinterpret_cast<V4*>(w) + q0;       // w chunk k at wg + k·NT
  const unsigned g0 = sh.vg;
  const unsigned gend = g0 + 2u * (unsigned)j * (unsigned)nit;
  const unsigned long long pol_last = policy_evict_last();
  const bool lead = d.profile && sh.cta == 0 && threadIdx.x == 0;
  // pass B runs over the items in reverse (tune bit 23: forward): it starts on the v_i
  // and w rows pass A touched last — the ones still in L2 — and ends where the next
  // pass A starts; the last step keeps the forward order (its ‖w‖² partial order).
  // C4 mixed MGS (r02): ortho 1512 → 1391 ms
  const bool rev = !((d.tune >> 23) & 1);
  // ---- producer (thread 0): cursor over (step ci, pass cp: 0 A / 1 B, item ck)
  unsigned issued = g0;
  int ci = 1, cp = 0, ck = 0;
  unsigned long long pol_first = 0, pol_norm = 0;
  if (threadIdx.x == 0) {
    pol_first = policy_evict_first();
    pol_norm = policy_evict_normal();
  }
  auto wait_bar = [&](unsigned long long* bar, unsigned par) -> bool {
    if (mbar_try_wait(bar, par)) return true;
    const unsigned long long t0 = globaltimer();
    for (;;) {
      if (mbar_try_wait(bar, par)) return true;
      if ((long long)(globaltimer() - t0) > d.timeout_ns) { atomicExch(d.abort_flag, 1); return false; }
    }
  };
  auto pump = [&](unsigned limit) {  // thread 0
    const unsigned long long tp0 = lead ? globaltimer() : 0ull;
    for (; issued < gend && issued < limit; ++issued) {
      const unsigned s = issued % NS;
      if (issued >= NS && !wait_bar(&sh.mbar_e[s], ((issued / NS) - 1u) & 1u)) return;
      const int cx = (cp && rev && ci < j) ? nit - 1 - ck : ck;  // B reversed (not the last step: ‖w‖² order)
      const unsigned bytes = (unsigned)min(MGS_IC * NT, nq - cx * MGS_IC * NT) * 16u;
      const V4* src = reinterpret_cast<const V4*>(V + (long long)(ci - 1) * ldv + r0) + (size_t)cx * MGS_IC * NT;
      mbar_expect_tx(&sh.mbar_v[s], bytes);
      tma_load_1d_hint(sv + (size_t)s * MGS_IC * NT, src, bytes, &sh.mbar_v[s], cp ? pol_first : pol_norm);
      if (++ck == nit) {
        ck = 0;
        if (++cp == 2) { cp = 0; ++ci; }
      }
    }
    if (lead) d.prof[11] += globaltimer() - tp0;  // profile: producer time
  };
  // ---- consumers (every thread; thread t owns vector t of every chunk)
  unsigned g = g0;  // next item to consume
  // the next item: wait for its bytes, return this thread's vectors in the slot (chunk c at [c·NT])
  auto acquire = [&]() -> const V4* {
    if (threadIdx.x == 0) pump(g + NS);
    const unsigned e = g;
    const unsigned long long tw0 = lead ? globaltimer() : 0ull;
    wait_bar(&sh.mbar_v[e % NS], (e / NS) & 1u);
    if (lead) d.prof[12] += globaltimer() - tw0;  // profile: waiting for ring data
    return sv + (size_t)(e % NS) * MGS_IC * NT + threadIdx.x;
  };
  auto release = [&]() {  // this warp is done with the item's slot
    const unsigned e = g++;
    __syncwarp();
    if (lane == 0) mbar_arrive(&sh.mbar_e[e % NS]);
  };
  if (threadIdx.x == 0) pump(g0 + NS);
  for (int k = 0; k < MG; ++k) {
    const int t = threadIdx.x + k * NT;
    if (t < nq) ws[t] = wg[t];
  }
  double nn = 0.0;
  for (int i = 1; i <= j; ++i) {
    // ---- pass A (B = 0): h_i = w·v_i; pass B (B = 1): w ← w − h_i v_i (and ‖w‖²
    // after the last step).  Global w is prefetched two items ahead in two register
    // sets (one item ahead left the loads' L2 latency exposed once per item).
    double acc = 0.0;
    W hw = (W)0;
    for (int B = 0; B < 2; ++B) {
      if (B) {
        double h;
        auto mid = [&]() {
          if (threadIdx.x == 0) pump(g + NS);  // A's items are all consumed: fill the ring with B's
        };
        const unsigned long long ta0 = lead ? globaltimer() : 0ull;
        if (!allreduce1<true>(d, sh, acc, false, h, mid)) return false;
        if (lead) d.prof[13] += globaltimer() - ta0;  // profile: all-reduce (incl. the refill)
        if (threadIdx.x == 0) s_h[i - 1] = h;
        hw = RN<W>(h);
      }
      const bool last = B && i == j;
      const bool rb = B && rev && i < j;
      V4 pfs[MGS_PS][MGS_IC];
#pragma unroll
      for (int o = 0; o < MGS_PS; ++o) {
        V4(&pf)[MGS_IC] = pfs[o];
        const int it = rb ? nit - 1 - o : o;
        if (o < nit && it * MGS_IC >= MG) {
#pragma unroll
          for (int c = 0; c < MGS_IC; ++c) {
            const int t = (it * MGS_IC + c) * NT + threadIdx.x;
            if (t < nq) pf[c] = ld_hint(wg + t, pol_last);
          }
        }
      }
      for (int i2 = 0; i2 < nit; i2 += MGS_PS) {
#pragma unroll
        for (int o = 0; o < MGS_PS; ++o) {
          if (i2 + o < nit) {
            V4(&pf)[MGS_IC] = pfs[o];
            const int it = rb ? nit - 1 - (i2 + o) : i2 + o;
            V4 wv[MGS_IC];
            const bool glob = it * MGS_IC >= MG;
            if (glob) {
#pragma unroll
              for (int c = 0; c < MGS_IC; ++c) wv[c] = pf[c];
            } else {
#pragma unroll
              for (int c = 0; c < MGS_IC; ++c)
                if ((it * MGS_IC + c) * NT + (int)threadIdx.x < nq) wv[c] = ws[(it * MGS_IC + c) * NT + threadIdx.x];
            }
            const int n2 = i2 + o + MGS_PS;  // the item MGS_PS ahead, into the set just read
            const int itn = rb ? nit - 1 - n2 : n2;
            if (n2 < nit && itn * MGS_IC >= MG) {
#pragma unroll
              for (int c = 0; c < MGS_IC; ++c) {
                const int t = (itn * MGS_IC + c) * NT + threadIdx.x;
                if (t < nq) pf[c] = ld_hint(wg + t, pol_last);
              }
            }
            const V4* x = acquire();
#pragma unroll
            for (int c = 0; c < MGS_IC; ++c) {
              const int t = (it * MGS_IC + c) * NT + threadIdx.x;
              if (t < nq) {
                if (!B) {
                  acc += dotv(wv[c], x[c * NT]);
                } else {
                  sub_scaled(wv[c], x[c * NT], hw);
                  if (last) nn += dotv(wv[c], wv[c]);
                  if (glob) st_hint(wg + t, wv[c], pol_last);
                  else ws[t] = wv[c];
                }
              }
            }
            release();
          }
        }
      }
    }
  }
  // shared chunks of w back to global for the next SpMV (global chunks were stored in the last pass)
  for (int k = 0; k < MG; ++k) {
    const int t = threadIdx.x + k * NT;
    if (t < nq) wg[t] = ws[t];
  }
  if (threadIdx.x == 0) sh.vg = gend;  // read by every thread at entry, before the syncs below
  NN = nn;  // this thread's share of ‖w‖²; the caller pushes the halo and all-reduces it
  return true;
}

// ‖w‖² all-reduce that ends the orthogonalisation.  With the orthogonality
// monitor (policy 3, reading R23) the dots V_jᵀw of the final w are formed in an
// extra pass over V_j and all-reduced TOGETHER with ‖w‖² (one reduction of j+1
// values); s_y[i] = (v_i·w)/‖w‖ = the new column of U (v_{j+1} = w/‖w‖).
// (MON: compiled only into the monitor's own kernel instantiation — the default
// kernel sits at the 128-register limit, tools/regcheck.sh)
template <class W, bool MON>
__device__ __forceinline__ bool final_norm(const Dev& d, Shm& sh, int r0, int r1, int j, const W* V, long long ldv,
                                           W* w, double nn, double* s_part, double* s_out, double* s_tmp,
                                           W* s_coefW, double* s_y, char* s_tiles, double& NN) {
  halo_push(d, sh, (const W*)w, wbuf_index(d, w));
  if (!MON || d.policy != 3) return allreduce1(d, sh, nn, true, NN);
  fence_proxy_async_global();  // w's generic stores are read by the pass's bulk copies
  __syncthreads();
  double dummy = 0.0;
  rowtile_pass<W, 1>(d, sh, r0, r1, V, ldv, j, w, s_coefW, s_y, s_tmp, s_tiles, dummy);
  combine_acc(d, s_tmp, j, s_part);
  double p[1] = {nn};
  block_sum<1>(p, sh, s_part + j);
  if (!grid_allreduce(d, sh, s_part, j + 1, s_out, s_tmp)) return false;
  NN = s_out[j];
  const double inv = NN > 0.0 ? 1.0 / sqrt(NN) : 0.0;
  for (int i = threadIdx.x; i < j; i += NT) s_y[i] = s_out[i] * inv;
  __syncthreads();
  return true;
}

// Orthogonalisation of w (own rows) against V[:, 0..j) and its norm: MGS
// or CGSR (two passes).  s_h[0..j) gets
// h_{1..j, j}; returns ‖w‖² through NN.
// CH: 1 the chunk-ring kernel instantiation (mgs_chunked, d.mgs_resident == 2),
// 2 the streamed one (mgs_stream, d.mgs_resident == 3); the default one (0) holds
// mgs_resident and mgs_sweep.  Each
// MGS variant lives in its own kernel: inlined together they raise the register
// pressure of every phase (tools/regcheck.sh).
template <class W, bool MON = false, int CH = 0, bool SW = true>
__device__ bool ortho_phase(const Dev& d, Shm& sh, int r0, int r1, int j, const W* V, long long ldv, W* w,
                            double* s_part, double* s_out, double* s_tmp, double* s_h, W* s_coefW, double* s_y,
                            char* s_tiles, double& NN) {
  if constexpr (CH == 1 || CH == 2) {
    if (d.ortho == 0) {
      double nn = 0.0;
      if constexpr (CH == 2) {
        if (!mgs_stream<W>(d, sh, r0, r1, j, V, ldv, w, s_h, s_tiles, nn)) return false;
      } else {
        if (!mgs_chunked<W>(d, sh, r0, r1, j, V, ldv, w, s_h, s_tiles, nn)) return false;
      }
      return final_norm<W, MON>(d, sh, r0, r1, j, V, ldv, w, nn, s_part, s_out, s_tmp, s_coefW, s_y, s_tiles, NN);
    }
  } else if (CH == 0 && d.ortho == 0 && (d.mgs_resident || !SW) && !(d.tune & 4)) {
    // (!SW: the headline kernels carry no sweep — the planner sends every other MGS
    // launch to the chunk-ring / streamed / sweep instantiations)
    double nn = 0.0;
    if (!mgs_resident<W>(d, sh, r0, r1, j, V, ldv, w, s_h, s_tiles, nn)) return false;
    return final_norm<W, MON>(d, sh, r0, r1, j, V, ldv, w, nn, s_part, s_out, s_tmp, s_coefW, s_y, s_tiles, NN);
  }
  if (SW && (CH == 0 || CH == 3) && d.ortho == 0) {
    W hprev = (W)0;
    const bool pf = !(d.tune & 1) && r1 > r0;
    const unsigned pf_bytes = (unsigned)((r1 - r0) * (int)sizeof(W));
    for (int i = 1; i <= j; ++i) {
      const double acc = mgs_sweep<W>(r0, r1, w, i > 1 ? V + (long long)(i - 2) * ldv : nullptr, hprev,
                                      V + (long long)(i - 1) * ldv);
      // while this step's reduction is in flight, pull the next basis
      // vector's rows (v_{i+1}) of this CTA into L2
      // (issued by warp 1: warp 0's release fence in the all-reduce must not wait on it)
      if (pf && i < j && threadIdx.x == 32) prefetch_l2(V + (long long)i * ldv + r0, pf_bytes);
      double h;
      if (!allreduce1<true>(d, sh, acc, false, h)) return false;
      if (threadIdx.x == 0) s_h[i - 1] = h;
      hprev = RN<W>(h);
    }
    const double acc = mgs_sweep<W>(r0, r1, w, V + (long long)(j - 1) * ldv, hprev, nullptr);
    return final_norm<W, MON>(d, sh, r0, r1, j, V, ldv, w, acc, s_part, s_out, s_tmp, s_coefW, s_y, s_tiles, NN);
  }
  double nn = 0.0;
  const bool lead = d.profile && sh.cta == 0 && threadIdx.x == 0;
  if (lead) sh.tsub = globaltimer();
  auto sub = [&](int slot) {
    if (d.profile) {
      grid_sync(d, sh);
      if (lead) { const unsigned long long t = globaltimer(); d.prof[8 + slot] += t - sh.tsub; sh.tsub = t; }
    }
  };
  // serpentine passes (rowtile_pass: reuse): 1 in direction D, 2 reversed, 3 in D;
  // D alternates between iterations, so every pass starts on the rows read last
  const int D = sh.cdir;
  rowtile_pass<W, 1>(d, sh, r0, r1, V, ldv, j, w, s_coefW, s_y, s_tmp, s_tiles, nn, D, false);
  combine_acc(d, s_tmp, j, s_part);
  sub(0);
  if (!grid_allreduce(d, sh, s_part, j, s_out, s_tmp, false)) return false;
  sub(1);
  for (int i = threadIdx.x; i < j; i += NT) {
    s_h[i] = s_out[i];
    s_coefW[i] = RN<W>(s_out[i]);
  }
  __syncthreads();
  rowtile_pass<W, 2>(d, sh, r0, r1, V, ldv, j, w, s_coefW, s_y, s_tmp, s_tiles, nn, 1 - D, true);
  combine_acc(d, s_tmp, j, s_part);
  sub(2);
  if (!grid_allreduce(d, sh, s_part, j, s_out, s_tmp, false)) return false;
  sub(3);
  for (int i = threadIdx.x; i < j; i += NT) {
    s_h[i] = s_h[i] + s_out[i];
    s_coefW[i] = RN<W>(s_out[i]);
  }
  __syncthreads();
  nn = 0.0;
  rowtile_pass<W, 3>(d, sh, r0, r1, V, ldv, j, w, s_coefW, s_y, s_tmp, s_tiles, nn, D, true);
  if (threadIdx.x == 0) sh.cdir = 1 - D;  // (every thread read D before the passes' barriers)
  sub(4);
  if (!final_norm<W, MON>(d, sh, r0, r1, j, V, ldv, w, nn, s_part, s_out, s_tmp, s_coefW, s_y, s_tiles, NN))
    return false;
  sub(5);
  return true;
}

// Orthogonality monitor (policy 3, reading R23): u = s_y[0..l) is the new
// column l of U (CTA 0 stores it); s = (I + U_l)⁻¹ u by column-oriented unit
// upper back-substitution with U's earlier columns from global memory; returns
// ‖s‖² (the new column's share of ‖S‖_F²), identical in every CTA.
__device__ __forceinline__ double orth_column(double* Umat, int ldu, int l, bool store, double* s_y, Shm& sh,
                                           double* s_part) {
  if (store)
    for (int i = threadIdx.x; i < l; i += NT) Umat[(size_t)l * ldu + i] = s_y[i];
  for (int q = l - 1; q >= 0; --q) {
    __syncthreads();
    const double sq = s_y[q];
    for (int i = threadIdx.x; i < q; i += NT) s_y[i] = __dsub_rn(s_y[i], __dmul_rn(__ldcg(Umat + (size_t)q * ldu + i), sq));
  }
  __syncthreads();
  double f[1] = {0.0};
  for (int i = threadIdx.x; i < l; i += NT) f[0] += s_y[i] * s_y[i];
  block_sum<1>(f, sh, s_part);
  return s_part[0];
}

// Spectral norm of S_k (policy 3, orth_norm 1, reading R23): 10
// power iterations on SᵀS from x = (1,…,1)/√k, k = l + 1, columns 0..l−1 of S
// from Smat (stored by CTA 0 in earlier inner steps, published by the
// all-reduces since), column l = s_col (this step's, in shared memory); then
// ‖S x‖ — the oracle's OrthMonitor::append step by step (each element's sum in
// the same order; the norms as block sums).  Identical in every CTA.  s_x, s_v:
// shared scratch of k doubles each.
static __device__ __noinline__ double spec_norm(const double* Smat, int ld, int l, const double* s_col, double* s_x,
                                         double* s_v, Shm& sh, double* s_part) {
  const int k = l + 1;
  auto S = [&](int i, int q) -> double { return q == l ? s_col[i] : __ldcg(Smat + (size_t)q * ld + i); };
  const double x0 = 1.0 / sqrt((double)k);
  for (int i = threadIdx.x; i < k; i += NT) s_x[i] = x0;
  __syncthreads();
  for (int it = 0; it < 10; ++it) {
    for (int i = threadIdx.x; i < k; i += NT) {  // y = S x (S strictly upper triangular)
      double t = 0.0;
      for (int q = i + 1; q < k; ++q) t += S(i, q) * s_x[q];
      s_v[i] = t;
    }
    __syncthreads();
    double f[1] = {0.0};
    for (int q = threadIdx.x; q < k; q += NT) {  // x = Sᵀ y
      double t = 0.0;
      for (int i = 0; i < q; ++i) t += S(i, q) * s_v[i];
      s_x[q] = t;
      f[0] += t * t;
    }
    block_sum<1>(f, sh, s_part);  // (its barriers also publish s_x)
    const double nx = sqrt(s_part[0]);
    if (nx == 0.0) return 0.0;
    for (int q = threadIdx.x; q < k; q += NT) s_x[q] /= nx;
    __syncthreads();
  }
  double f[1] = {0.0};
  for (int i = threadIdx.x; i < k; i += NT) {
    double t = 0.0;
    for (int q = i + 1; q < k; ++q) t += S(i, q) * s_x[q];
    f[0] += t * t;
  }
  block_sum<1>(f, sh, s_part);
  return sqrt(s_part[0]);
}

// ---------------------------------------------------------- the solve
// One launch runs the whole restarted solve of one rank (d = ds.d[0], G CTAs)
// or of ds.nv "virtual ranks" on one device (rank v = CTAs [v·G, (v+1)·G)):
// the same code, with peer buffers that are other allocations on the device —
// how the multi-rank path is exercised with one GPU (one cooperative launch:
// the ranks' CTAs wait on one another).
constexpr int MAXV = 4;
struct DevSet {
  Dev d[MAXV];
  int G;   // CTAs per rank
  int nv;  // ranks in this launch (1 = one rank per process/GPU)
};

template <class W, int L, bool VR, bool MON = false, int CH = 0, bool PC = false>
__global__ void __launch_bounds__(NT, 1) solve_kernel(const __grid_constant__ DevSet ds) {
  // (VR = false: a static index keeps every field of d a constant-bank operand)
  const int vr = VR ? (int)blockIdx.x / ds.G : 0;
  const Dev& d = ds.d[VR ? vr : 0];
  extern __shared__ __align__(128) char dsm[];
  __shared__ Shm sh;
  double* const s_part = reinterpret_cast<double*>(dsm + d.soff[0]);
  double* const s_out = reinterpret_cast<double*>(dsm + d.soff[1]);
  double* const s_tmp = reinterpret_cast<double*>(dsm + d.soff[2]);
  double* const s_h = reinterpret_cast<double*>(dsm + d.soff[3]);
  double* const s_cs = reinterpret_cast<double*>(dsm + d.soff[4]);
  double* const s_sn = reinterpret_cast<double*>(dsm + d.soff[5]);
  double* const s_s = reinterpret_cast<double*>(dsm + d.soff[6]);
  double* const s_y = reinterpret_cast<double*>(dsm + d.soff[7]);
  double* const s_rhs = reinterpret_cast<double*>(dsm + d.soff[8]);
  W* const s_coefW = reinterpret_cast<W*>(dsm + d.soff[9]);
  char* const s_tiles = dsm + d.soff[10];
  init_shm(sh, (int)blockIdx.x - vr * ds.G);
  if (threadIdx.x == 0) {
    sh.epoch = d.epoch0;
    sh.red_epoch = d.red0;
    sh.r0 = d.row_begin[sh.cta];
    sh.r1 = d.row_begin[sh.cta + 1];
  }
  __syncthreads();
  // (CTA index, row block and lead flag re-read from shared memory at each use:
  // kept in registers they lived across every phase and spilled)
#define cta_ (sh.cta)
#define r0_ (sh.r0)
#define r1_ (sh.r1)
#define lead (sh.cta == 0 && threadIdx.x == 0)
#define wb0 reinterpret_cast<W*>(d.w0)
  W* const V = reinterpret_cast<W*>(d.V);
  const long long ldv = d.ldv;
  // phase timers of CTA 0 (the previous timestamp lives in shared memory: no register
  // stays live across the phases for it)
  if (lead) sh.tprev = globaltimer();
  auto tick = [&](int ph) {
    if (lead) { const unsigned long long t = globaltimer(); d.prof[ph] += t - sh.tprev; sh.tprev = t; }
  };

  // loop state in shared memory (cycle count, inner total, 1/h): values live across
  // the phases otherwise spill (r02: the headline kernel's last local-memory ops)
  int status = ST_OK;
  if (threadIdx.x == 0) { sh.J1 = 0; sh.inner_len = 0; sh.kcyc = 0; sh.total_inner = 0; }
  unsigned ilu_seq = 0;  // ILU applies so far (sync-free solve sequence numbers)
  (void)ilu_seq;
  // (every rank reads its own flag: the cast overflow check is the same on all
  // ranks only if the caller built A32 on all of them; ranks agree on it via
  // the residual all-reduce below, which carries the error bits)
  if (d.halo) {  // x0's rows that peers gather
    halo_push(d, sh, (const double*)d.x, 2);
    if (!grid_sync(d, sh)) status = ST_ETIMEOUT;
  }
  for (; status == ST_OK;) {
    // ---------------- residual, stop test (Alg. 1 lines 86–92)
    // ‖z‖², ‖r‖², ‖b‖², ‖x‖² and (CTA 0 of each rank) this rank's ‖A‖_F²
    double v3[5] = {0.0, 0.0, 0.0, 0.0, cta_ == 0 && threadIdx.x == 0 ? d.normA2 : 0.0};
    int err = 0;
    resid_phase<W, L>(d, sh, s_tiles, wb0, v3[0], v3[1], v3[2], v3[3], err);
    if (err) atomicOr(d.err_flag, err);
    __syncthreads();
    // error indicators of every rank travel inside the sums, so all ranks stop
    // alike: non-finite → NaN in ‖z‖², fp32 overflow (this residual, or the A32
    // cast before the launch) → +Inf in ‖r‖² (a sum of fp32 squares is finite)
    if (threadIdx.x == 0) {
      const int f = *(volatile int*)d.err_flag;
      if (f & ERRF_NONFINITE) v3[0] = __longlong_as_double(0x7ff8000000000000ll);
      if (f & ERRF_RANGE) v3[1] = __longlong_as_double(0x7ff0000000000000ll);
    }
    halo_push(d, sh, (const W*)wb0, 0);
    block_sum<5>(v3, sh, s_part);
    if (!grid_allreduce(d, sh, s_part, 5, s_out, s_tmp)) { status = ST_ETIMEOUT; break; }
    const double ZZ = s_out[0], RR = s_out[1], nb = sqrt(s_out[2]);
    const int ef = *(volatile int*)d.err_flag;  // (other ranks' errors arrive as NaN/Inf in ZZ/RR)
    if (nb == 0.0) {  // b = 0 → x = 0, no cycle (reading R13)
      for (int i = r0_ + threadIdx.x; i < min(r1_, d.n); i += NT) d.x[i] = 0.0;
      if (lead) { if (d.hist_cap > 0) d.history[0] = 0.0; d.out_int[3] = 1; d.out_dbl[0] = 0.0; d.out_dbl[1] = 0.0; }
      status = ST_OK;
      break;
    }
    const double rho = sqrt(ZZ) / nb;
    if (lead) {
      if (sh.kcyc < d.hist_cap) d.history[sh.kcyc] = rho;
      d.out_int[3] = sh.kcyc + 1;
      d.out_dbl[0] = rho;
      // normwise backward error ‖b − Ax‖/(‖A‖_F‖x‖ + ‖b‖) of this iterate (report only)
      d.out_dbl[1] = sqrt(ZZ) / (sqrt(s_out[4]) * sqrt(s_out[3]) + nb);
    }
    tick(PH_RESID);
    if (ef & ERRF_NONFINITE || !isfinite(ZZ) || !isfinite(nb)) { status = ST_ENONFINITE; break; }
    if ((ef & ERRF_RANGE) || RR > DBL_MAX) { status = ST_EFP32RANGE; break; }
    if (rho <= d.tol) { status = ST_OK; break; }
    if (sh.kcyc >= d.max_cycles) { status = ST_NOT_CONVERGED; break; }
    double RRp = RR;
    if constexpr (PC) {  // line 90 with M = LU (reading R24): r = U⁻¹L⁻¹ RN_W(z), then ‖r‖²
      if (!ilu_apply_any<W>(d, sh, wb0, wb0, ilu_seq++)) { status = ST_ETIMEOUT; break; }
      double p = 0.0;
      for (int i = r0_ + threadIdx.x; i < min(r1_, d.n); i += NT) {
        const double v = (double)__ldcg(wb0 + i);
        p += v * v;
      }
      if (!allreduce1(d, sh, p, true, RRp)) { status = ST_ETIMEOUT; break; }
    }
    const double beta = sqrt(RRp);
    if (!(beta > 0.0) || !isfinite(beta)) { status = ST_ENONFINITE; break; }
    // restart threshold (readings R6, R22): the two-stage policy drops δ after
    // the first cycle and restarts at the first cycle's iteration count J1
    if (threadIdx.x == 0) {
      const bool repeat = d.policy == 1 && sh.kcyc > 0;
      sh.thr = beta * fmax(d.tol * nb / sqrt(ZZ), repeat ? 0.0 : d.delta);
      sh.jmax = repeat ? min(d.m, sh.J1) : d.m;
      sh.beta = beta;
      for (int i = 0; i <= d.m; ++i) s_s[i] = 0.0;
      s_s[0] = beta;
      s_rhs[0] = beta;  // |s| history of the cycle (stall policy; s_rhs is free until the back-solve)
      sh.inv = 1.0 / beta;
    }
    __syncthreads();
    // v_j's unnormalised source and w alternate between the work vectors (by the parity of j,
    // from the constant bank at each use: no pointer pair stays live in registers)
    auto src = [&](int jj) { return reinterpret_cast<W*>((jj & 1) ? d.w0 : d.w1); };
    auto dst = [&](int jj) { return reinterpret_cast<W*>((jj & 1) ? d.w1 : d.w0); };
    int J = 0;
    double mon_fro2 = 0.0;  // orthogonality monitor: ‖S‖_F² of this cycle (policy 3)
    bool fail = false;
    for (int j = 1; j <= d.m; ++j) {
      // ------------ w = M⁻¹ A v_j, v_j (own rows) → V   (lines 100, 105)
      if (d.profile && threadIdx.x == 0) sh.tsub = globaltimer();
      spmv_phase<W, L>(d, sh, s_tiles, src(j), sh.inv, dst(j), V, j - 1);
      if constexpr (PC) {  // w = U⁻¹L⁻¹(A_W v_j) (line 100 with M = LU)
        if (!grid_sync(d, sh) || !ilu_apply_any<W>(d, sh, dst(j), dst(j), ilu_seq++)) { fail = true; break; }
      }
      if (d.profile) {
        if (threadIdx.x == 0) d.prof_cta[cta_] += globaltimer() - sh.tsub;
        if (!grid_sync(d, sh)) { fail = true; break; }
      }
      tick(PH_SPMV);
      // ------------ orthogonalise (line 101) and ‖w‖ (line 104)
      double NN;
      // the headline instantiations (L ∈ {1, 4}, no monitor / ILU / virtual ranks) carry no
      // MGS sweep: its register budget spilled into the resident MGS (r02); CH = 3 is the sweep
      constexpr bool SW = !((L == 1 || L == 4) && !VR && !MON && !PC && CH == 0);
      if (!ortho_phase<W, MON, CH, SW>(d, sh, r0_, r1_, j, V, ldv, dst(j), s_part, s_out, s_tmp, s_h, s_coefW, s_y,
                                       s_tiles, NN)) {
        fail = true;
        break;
      }
      tick(PH_ORTHO);
      // ------------ orthogonality monitor (policy 3, reading R23): the new column
      // of S_k = (I+U_k)⁻¹U_k by unit upper back-substitution, ‖S‖_F² accumulated
      double mon_spec = 0.0;
      if (MON && d.policy == 3 && NN > 0.0) {
        mon_fro2 += orth_column(d.Umat, d.m + 1, j, cta_ == 0, s_y, sh, s_part);
        if (d.orth_spec) {  // S's new column j (rows 0..j−1, in s_y): store it (CTA 0), then ‖S‖₂
          mon_spec = spec_norm(d.Smat, d.m + 1, j, s_y, s_tmp, s_tmp + d.kmax + 1, sh, s_part);
          if (cta_ == 0)
            for (int i = threadIdx.x; i < j; i += NT) d.Smat[(size_t)j * (d.m + 1) + i] = s_y[i];
          __syncthreads();
        }
      }
      const bool orth = MON && d.policy == 3 && (d.orth_spec ? mon_spec : sqrt(mon_fro2)) >= d.orth_thresh;
      // ------------ h_{j+1,j}, Givens, exit test (lines 104, 108–140, 98)
      const double hn = sqrt(NN);
      if (threadIdx.x == 0) {
        s_h[j] = hn;
        const double sabs = hess_step(j, s_h, s_cs, s_sn, s_s);
        if (cta_ == 0 && sh.inner_len < d.inner_cap) d.inner_hist[sh.inner_len] = sabs / sh.beta;
        sh.inner_len++;
        s_rhs[j] = sabs;
        const bool stall = d.stall_w > 0 && j >= d.stall_w && sabs * d.stall_factor > s_rhs[j - d.stall_w];
        sh.flag = (j == sh.jmax) || (hn == 0.0) || (sabs <= sh.thr) || stall || orth || !isfinite(hn);
        sh.inv = 1.0 / hn;
      }
      __syncthreads();
      // R's column j (CTA 0, all threads; s_h is next written after the next SpMV's barrier)
      if (cta_ == 0)
        for (int i = threadIdx.x; i <= j; i += NT) d.R[(size_t)(j - 1) * (d.m + 1) + i] = s_h[i];
      tick(PH_GIVENS);
      J = j;
      if (!isfinite(hn)) { status = ST_ENONFINITE; fail = true; break; }
      if (sh.flag) break;
    }
    if (fail) { if (status == ST_OK) status = ST_ETIMEOUT; break; }
    if (threadIdx.x == 0) {
      if (sh.kcyc == 0) sh.J1 = J;
      sh.total_inner += J;
    }
    if (lead && sh.kcyc < d.hist_cap) d.cycle_J[sh.kcyc] = J;
    // ------------ y = R⁻¹ s, x ← x + V_J y  (lines 143–147)
    __syncthreads();  // (R's last column, stored by CTA 0's threads)
    if (cta_ == 0) backsolve_cta(J, d.R, d.m + 1, s_s, s_rhs, d.y, s_y);
    if (!grid_sync(d, sh)) { status = ST_ETIMEOUT; break; }
    for (int i = threadIdx.x; i < J; i += NT) s_y[i] = __ldcg(d.y + i);
    __syncthreads();
    double dummy = 0.0;
    rowtile_pass<W, 4>(d, sh, r0_, r1_, V, ldv, J, nullptr, s_coefW, s_y, s_tmp, s_tiles, dummy);
    halo_push(d, sh, (const double*)d.x, 2);
    if (!grid_sync(d, sh)) { status = ST_ETIMEOUT; break; }
    tick(PH_UPDATE);
    if (threadIdx.x == 0) sh.kcyc++;
    __syncthreads();
  }
  if (lead) {
    d.out_int[0] = status;
    d.out_int[1] = sh.kcyc;
    d.out_int[2] = sh.total_inner;
    d.out_int[4] = sh.inner_len;
    if (d.epoch_out) { d.epoch_out[0] = sh.epoch; d.epoch_out[1] = (unsigned long long)sh.red_epoch; }
  }
#undef wb0
#undef cta_
#undef r0_
#undef r1_
#undef lead
}

#ifdef G200_HOST_TU  // non-template kernels: defined once, in gmres_capi.cu
// ------------------------------------------------------ setup kernels
// a0: A32 = RN32(A64), overflow flagged.
__global__ void cast32_kernel(const double* __restrict__ a, float* __restrict__ o, long long cnt, int* err) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < cnt; e += (long long)gridDim.x * blockDim.x) {
    const double v = a[e];
    if (isfinite(v) && fabs(v) > (double)FLT_MAX) atomicOr(err, ERRF_RANGE);
    o[e] = __double2float_rn(v);
  }
}

#endif

// column-major V (ncols columns, leading dimension ldv, rows ≥ nvalid read
// as 0) → row-blocked layout (Dev::vtb); component entry points only
template <class W>
__global__ void pack_vblocked_kernel(const W* __restrict__ src, long long ldv, int ncols, long long nrows,
                                     long long nvalid, W* __restrict__ dst, int tb, int tp, long long bs) {
  const long long tot = nrows * ncols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e / nrows);
    const long long r = e - (long long)c * nrows;
    dst[(r / tb) * bs + (long long)c * tp + (r % tb)] = r < nvalid ? src[(long long)c * ldv + r] : (W)0;
  }
}

// basis columns (either layout) → caller's column-major buffer (instrumentation)
template <class W>
__global__ void unpack_basis_kernel(const W* __restrict__ V, long long ldv, int tb, int tb_log, int tp, long long bs,
                                    int col0, int ncols, long long n, W* __restrict__ dst, long long ld) {
  const long long tot = n * ncols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e / n);
    const long long r = e - (long long)c * n;
    const long long src = tb ? (r >> tb_log) * bs + (long long)(col0 + c) * tp + (r & (tb - 1)) : (long long)(col0 + c) * ldv + r;
    dst[(long long)c * ld + r] = V[src];
  }
}

#ifdef G200_HOST_TU
// ‖A‖_F² in a fixed order: block g sums its contiguous slice (warp trees, warps
// in order), then one block sums the partials in order (sumsq_final_kernel)
__global__ void sumsq_partial_kernel(const double* __restrict__ a, long long cnt, double* part) {
  const long long per = (cnt + gridDim.x - 1) / gridDim.x;
  const long long e0 = blockIdx.x * per, e1 = min(cnt, e0 + per);
  double s = 0.0;
  for (long long e = e0 + threadIdx.x; e < e1; e += blockDim.x) s += a[e] * a[e];
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}
__global__ void sumsq_final_kernel(const double* part, int np, double* out) {
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int g = 0; g < np; ++g) t += part[g];
    *out = t;
  }
}

// Jacobi M = diag(A) (reading R11): dinv64 = 1/a_ii (fp64), dinv32 = RN32(dinv64).
__global__ void dinv_kernel(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                            const double* __restrict__ a, double* dinv64, float* dinv32, int* bad_row,
                            long long row_base) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double dg = 0.0;
    for (int p = rp[i]; p < rp[i + 1]; ++p)
      if (ci[p] == i + row_base) dg = a[p];
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
#endif

// ------------------------------------------------- component kernels
// Each runs the same device functions as solve_kernel for one step.
template <class W, int L>
__global__ void __launch_bounds__(NT, 1) k_spmv_kernel(Dev d, const W* v, W* w) {
  G200_SMEM_CARVE(W)
  spmv_phase<W, L>(d, sh, s_tiles, v, 1.0, w, (W*)nullptr, 0);
}

template <class W>
__global__ void __launch_bounds__(NT, 1) k_ilu_apply_kernel(Dev d, const W* z, W* out) {
  G200_SMEM_CARVE(W)
  ilu_apply_phase<W>(d, sh, z, out, 0u);
}

template <class W, int L>
__global__ void __launch_bounds__(NT, 1) k_resid_kernel(Dev d, W* r, double* out2) {
  G200_SMEM_CARVE(W)
  double v3[3] = {0.0, 0.0, 0.0}, xx = 0.0;
  int err = 0;
  resid_phase<W, L>(d, sh, s_tiles, r, v3[0], v3[1], v3[2], xx, err);
  if (err) atomicOr(d.err_flag, err);
  block_sum<3>(v3, sh, s_part);
  if (!grid_allreduce(d, sh, s_part, 3, s_out, s_tmp)) return;
  if (blockIdx.x == 0 && threadIdx.x < 2) out2[threadIdx.x] = s_out[threadIdx.x];
}

template <class W, int CH = 0>
__global__ void __launch_bounds__(NT, 1) k_ortho_kernel(Dev d, int j, const W* V, long long ldv, W* w, double* hout) {
  G200_SMEM_CARVE(W)
  const int r0 = d.row_begin[blockIdx.x], r1 = d.row_begin[blockIdx.x + 1];
  double NN = 0.0;
  if (!ortho_phase<W, false, CH>(d, sh, r0, r1, j, V, ldv, w, s_part, s_out, s_tmp, s_h, s_coefW, s_y, s_tiles, NN))
    return;
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < j; i += NT) hout[i] = s_h[i];
    if (threadIdx.x == 0) hout[j] = sqrt(NN);
  }
}

template <class W>
__global__ void __launch_bounds__(NT, 1) k_xupdate_kernel(Dev d, int J, const W* V, long long ldv, const double* y) {
  G200_SMEM_CARVE(W)
  for (int i = threadIdx.x; i < J; i += NT) s_y[i] = y[i];
  __syncthreads();
  const int r0 = d.row_begin[blockIdx.x], r1 = d.row_begin[blockIdx.x + 1];
  double dummy = 0.0;
  rowtile_pass<W, 4>(d, sh, r0, r1, V, ldv, J, nullptr, s_coefW, s_y, s_tmp, s_tiles, dummy);
}

#ifdef G200_HOST_TU
// a6 + a7 on a given unrotated Hessenberg (tests): one CTA.
__global__ void __launch_bounds__(NT, 1) k_hess_kernel(int m, int J, const double* Hbar, double beta, double* R,
                                                     double* s, double* y) {
  extern __shared__ __align__(128) char dsm[];
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
#endif

}  // namespace g200
