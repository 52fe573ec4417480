// gmres_capi.cu — host side of libgmres.so: the C ABI of include/gmres.h.
//
// Owns the device copy of A (fp64 + lazily the fp32 copy), the
// Jacobi diagonal, the workspace (V, work vectors, reduction partials, R, y),
// the row partition over the persistent grid, and the cooperative launch of
// the fused solve kernel (gmres_kernels.cuh).  No compute happens here.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/gmres.h"
#define G200_HOST_TU
#include "gmres_kernels.cuh"
#include "ktab.h"

using namespace g200;

// V layout of a solve (gmres_kernels.cuh Dev): column-major (tb = 0) or row-blocked
struct VLayout { int tb = 0, tp = 0, lg = 0; long long bs = 0; };

struct gmres_ctx {
  int device = 0;
  int sms = 0;
  int64_t n = 0, nnz = 0;
  int64_t nvec = 0;  // n rounded up to VEC_ALIGN (padded length of every n-vector)
  int64_t ldv = 0;   // leading dimension of column-major V (= nvec)
  std::vector<int32_t> h_rp;  // host row_ptr (row partitioning)
  int32_t* d_rp = nullptr;
  int32_t* d_ci = nullptr;
  double* d_a64 = nullptr;
  float* d_a32 = nullptr;
  bool a32_ready = false;
  double* d_dinv64 = nullptr;
  float* d_dinv32 = nullptr;
  cudaStream_t stream = nullptr;
  // ILU(0) (§8 f2): level schedules (built once per context) and the factors per
  // precision (index = gmres_precision)
  bool ilu_plan = false;
  int ilu_nlev[2] = {0, 0};
  std::vector<int> ilu_hlev0;  // lower-solve level offsets (one factor launch per level)
  int* d_ilu_dpos = nullptr;
  int* d_ilu_lev[2] = {nullptr, nullptr};
  int* d_ilu_rows[2] = {nullptr, nullptr};
  int* d_ilu_eoff[2] = {nullptr, nullptr};
  int* d_ilu_ecol[2] = {nullptr, nullptr};
  int* d_ilu_eidx[2] = {nullptr, nullptr};
  void* d_ilu_f[2] = {nullptr, nullptr};
  void* d_ilu_rec[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [precision][solve]
  bool ilu_ready[2] = {false, false};
  void* d_ones[2] = {nullptr, nullptr};  // W ones (nvec): the Jacobi scale of ILU solves
  int* d_ilu_bad = nullptr;
  void* d_ilu_pub[2] = {nullptr, nullptr};  // [n] fp64-sized publish buffers of the sync-free solves
  float* d_ilu_s32[2] = {nullptr, nullptr}; // fp32 scratch vectors of the fp32-ILU-in-fp64 solver
  double* d_hb = nullptr;  // device staging of b / x for the host-array gmres_solve
  double* d_hx = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evk0 = nullptr, evk1 = nullptr;
  // workspace
  int ws_m = -1, ws_prec = -1, ws_G = 0;
  int ws_v_tb = -1;       // basis layout (block height, 0 = column-major) the workspace V last held
  size_t ws_v_bytes = 0;
  char* d_ws = nullptr;
  size_t ws_bytes = 0;
  void* d_V = nullptr;
  void* d_w0 = nullptr;
  void* d_w1 = nullptr;
  double* d_slots = nullptr;      // grid all-reduce partials [2][G][kst]
  unsigned long long* d_ctr = nullptr;  // arrival counter
  unsigned long long* d_fx = nullptr;   // fixed-point projection all-reduce words (reading R27), 1 KB
  int fx_exp = INT_MIN;                 // B = 2^fx_exp ≥ 2·√(‖D⁻¹A‖₁‖D⁻¹A‖∞) (single-rank contexts)
  size_t slots_count = 0;
  double* d_R = nullptr;
  double* d_umat = nullptr;  // orthogonality monitor U (policy 3)
  double* d_smat = nullptr;  // ... and S = (I+U)⁻¹U (spectral norm)
  double* d_y = nullptr;
  int* d_flags = nullptr;  // [0] abort [1] err [2] scratch
  int* d_out_int = nullptr;
  double* d_out_dbl = nullptr;
  unsigned long long* d_prof = nullptr;
  unsigned long long* d_prof_cta = nullptr;
  double* d_hist = nullptr;
  int* d_cycJ = nullptr;
  int hist_cap = 0;
  double* d_inner = nullptr;
  int inner_cap = 0;
  // current row partition over the grid (aliases of an entry of `parts`)
  int* d_row_begin = nullptr;
  int4* d_chunks = nullptr;
  int* d_chunk_off = nullptr;
  int part_G = 0, part_align = 0;
  struct Part {  // cached partitions: MGS (32-row) and CGSR (block-aligned) solves alternate
    int G, align, max_rows;
    int* d_row_begin;
    int4* d_chunks;
    int* d_chunk_off;
    int* d_send;
    int2* d_stages;
    int* d_stage_off;
    int4* d_mtiles;   // merge-path tiles, their CTA offsets, split rows and offsets, carries
    int* d_mt_off;
    int4* d_msplit;
    int* d_ms_off;
    double* d_mcarry;
  };
  std::vector<Part> parts;
  int2* d_stages = nullptr;      // block-stream stages of the current partition
  int* d_stage_off = nullptr;
  int4* d_mtiles = nullptr;      // merge-path stream of the current partition (irregular rows)
  int* d_mt_off = nullptr;
  int4* d_msplit = nullptr;
  int* d_ms_off = nullptr;
  double* d_mcarry = nullptr;
  bool merge_ok = false;         // not block_ok: use the merge-path CSR stream (G200_NO_MERGE_STREAM: chunk stream)
  bool block_ok = false;         // every row has ≤ BS_MAXROW nonzeros: use the block CSR stream
  int part_max_rows = 0;  // largest CTA row block of the partition
  // last solve
  std::vector<double> inner_host;
  std::vector<int32_t> cycJ_host;
  double phase_ns[PH_N] = {0};
  int32_t plan[GMRES_PLAN_N] = {0};  // launch plan of the last solve (gmres_get_plan)
  std::string err;
  // basis of the last solve (gmres_get_basis): layout, m, precision
  int last_m = 0, last_prec = -1;
  VLayout last_vl;
  // ---- row partition over ranks (gmres_create_dist)
  int nranks = 1, rank = 0;
  int64_t n_global = 0, row_begin = 0;  // this rank owns global rows [row_begin, row_begin + n)
  int64_t nvec_global = 0;
  std::vector<int32_t> ghosts;          // sorted global columns of the local rows outside them
  void* d_gw0 = nullptr;                // full-length (global) work vectors, 8 bytes per row
  void* d_gw1 = nullptr;
  double* d_gx = nullptr;               // full-length x
  double* d_dslots = nullptr;           // all-reduce partials [2][nranks·sms][KST_MAX]
  unsigned long long* d_dctr = nullptr; // arrival counter (monotonic across launches)
  unsigned long long* d_epoch = nullptr;  // [2] barrier epochs / all-reduces at the end of the last launch
  unsigned long long epoch_base = 0;
  int red_base = 0;
  bool linked = false, ipc = false;
  double normA2 = 0.0;                  // ‖A‖_F² of this context's rows (device-computed at create)
  unsigned halo_full = 0;               // peers that receive whole row blocks (bit q)
  void* peer_w0[MAXR] = {}, *peer_w1[MAXR] = {};
  double* peer_x[MAXR] = {};
  double* peer_slots[MAXR] = {};
  unsigned long long* peer_ctr[MAXR] = {};
  std::vector<std::vector<int32_t>> send_rows;  // per peer: local rows it gathers (sorted)
  int* d_send = nullptr;                // [G+1] offsets, rows, peers (rebuilt with the partition)
  bool dist() const { return nranks > 1; }
};

namespace {

thread_local std::string g_err;

int fail(gmres_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  g_err = msg;
  return code;
}

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) {                                                          \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? GMRES_ENOMEM : GMRES_ECUDA,  \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                \
    }                                                                                 \
  } while (0)

int64_t round_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }
constexpr int KST_MAX = (MAX_M + 1 + 8 + 3) & ~3;  // k stride bound of the all-reduce partials

// lanes per row in the CSR stream: one thread per row when a 512-row chunk of
// average rows fits the stage (stencils), else the power of two that keeps
// ~GT lanes (one warp) busy on a chunk of CHUNK_CAP non-zeros.
int auto_lanes(int64_t n, int64_t nnz) {
  const double mu = n > 0 ? (double)nnz / (double)n : 1.0;
  const double rows = std::min((double)CHUNK_RMAX, (double)CHUNK_CAP / std::max(mu, 1.0));
  int L = 1;
  while (L < 32 && rows * L < 0.75 * GT) L *= 2;
  return L;
}

// Row partition over G CTAs: boundaries on multiples of `align` rows (32, or
// the V block height of the row-blocked layout), balancing rows + nnz (the
// merge-path cost), last boundary = nvec.
void make_partition(const std::vector<int32_t>& rp, int64_t n, int64_t nvec, int G, int align, std::vector<int>& out) {
  out.assign(G + 1, 0);
  const double total = (double)nvec + (double)rp[n];
  auto cost = [&](int64_t r) { return (double)r + (double)rp[std::min(r, n)]; };
  const int64_t nblk = nvec / align;
  int64_t lo = 0;
  for (int g = 1; g < G; ++g) {
    const double target = total * g / G;
    int64_t a = lo, b = nblk;  // find smallest block boundary with cost ≥ target
    while (a < b) {
      int64_t mid = (a + b) / 2;
      if (cost(mid * align) < target) a = mid + 1; else b = mid;
    }
    lo = a;
    out[g] = (int)(a * align);
  }
  out[G] = (int)nvec;
}

// V layout of a solve (gmres_kernels.cuh Dev): CGSR → row-blocked with the
// largest power-of-two block height in [32, 256] whose (m+1)-column block fits
// half the staging region; MGS (and CGSR at very large m) → column-major.
VLayout vlayout_for(int ortho, int m, int wb, int tile_bytes) {
  VLayout L;
  if (ortho != GMRES_CGSR) return L;
  const int pade = 16 / wb;
  for (int tb = 256; tb >= 32; tb /= 2) {
    if ((long long)(m + 1) * (tb + pade) * wb <= tile_bytes / G200_NTB) {
      L.tb = tb;
      L.tp = tb + pade;
      L.lg = 0;
      while ((1 << L.lg) < tb) ++L.lg;
      L.bs = (long long)(m + 1) * L.tp;
      return L;
    }
  }
  return L;
}

constexpr bool kMgsCopyInAllreduce = false;

// fixed-point projection all-reduce (reading R27): B = 2^e and its exact scalings; the
// exponent range keeps 2^(42−e) and 2^(e−42) normal (else the fp64 all-reduce is used)
void set_fx(Dev& d, int e, unsigned long long* words) {
  if (e < -900 || e > 900) return;
  d.fx = 1;
  d.fx_exp = e;
  d.fx_bnd = std::ldexp(1.0, e);
  d.fx_up = std::ldexp(1.0, 42 - e);
  d.fx_dn = std::ldexp(1.0, e - 42);
  d.fx_words = words;
}

void set_vlayout(Dev& d, const VLayout& vl) {
  d.vtb = vl.tb;
  d.vtp = vl.tp;
  d.vtb_log = vl.lg;
  d.vbs = vl.bs;
}

// kernel pointers (ktab.h: one translation unit per group, compiled in parallel)
void* pick_solve(int prec, int L) {
  if (prec == GMRES_MIXED) return L <= 4 ? ktab_solve_f32_lo(L) : ktab_solve_f32_hi(L);
  return L <= 4 ? ktab_solve_f64_lo(L) : ktab_solve_f64_hi(L);
}
void* pick_solve_ext(int prec, int variant, int L) {
  return prec == GMRES_MIXED ? ktab_solve_f32_ext(variant, L) : ktab_solve_f64_ext(variant, L);
}
// orthogonality-monitor launches (restart policy 3): L ∈ {1, 4}
void* pick_solve_monitor(int prec, int L) { return pick_solve_ext(prec, 1, L); }
// chunk-ring MGS launches (d.mgs_resident == 2): L ∈ {1, 4}
void* pick_solve_chunked(int prec, int L) { return pick_solve_ext(prec, 2, L); }
// streamed MGS launches (d.mgs_resident == 3): L ∈ {1, 4}
void* pick_solve_stream(int prec, int L) { return pick_solve_ext(prec, 5, L); }
// MGS global-sweep launches (d.mgs_resident == 0) of the kernels without a sweep: L ∈ {1, 4}
void* pick_solve_sweep(int prec, int L) { return pick_solve_ext(prec, 6, L); }
// ILU(0)-preconditioned launches (§8 f2): L ∈ {1, 4}
void* pick_solve_ilu(int prec, int L) { return pick_solve_ext(prec, 3, L); }
// virtual-rank launches (several row blocks on one device): L ∈ {1, 4}
void* pick_solve_virtual(int prec, int L) { return pick_solve_ext(prec, 4, L); }

void* pick_kernel(int prec, int kind, int L) {
  return prec == GMRES_MIXED ? ktab_comp_f32(kind, L) : ktab_comp_f64(kind, L);
}

// stride of the per-CTA partial sums: m+1 Gram-Schmidt coefficients, and at
// least the 3 values of the residual reduction
int kmax_for(int m) { return std::max(m + 1, 8); }

// shared staging region: two CSR chunk stages, or two V tiles of ≥ 32 rows
constexpr size_t kMaxDynSmem = 227 * 1024;
// staging region: all the shared memory the fixed arrays (kmax-sized) and the
// static control block leave, at least the block stream's ring (TILE_BYTES)
int tile_bytes_for(int m) {
  const size_t fixed = SmemLayout(std::max(m + 1, 8), 0).total + 4096;  // + static Shm and slack
  const size_t avail = (kMaxDynSmem - fixed) & ~size_t(127);
  return (int)std::max<size_t>(TILE_BYTES, avail);
}
size_t smem_bytes(int m, int tile_bytes = 0) {
  return SmemLayout(kmax_for(m), tile_bytes ? tile_bytes : tile_bytes_for(m)).total;
}
struct OccKey { const void* k; size_t smem; };
thread_local std::vector<std::pair<OccKey, int>> g_occ;  // (kernel, smem) → blocks per SM

int grid_for(gmres_ctx* ctx, const void* kern, size_t smem, int ctas_per_sm, int* G) {
  int per_sm = -1;
  for (auto& e : g_occ)
    if (e.first.k == kern && e.first.smem == smem) per_sm = e.second;
  // the attribute is per kernel: set it to the largest smem used so far
  static thread_local std::vector<std::pair<const void*, size_t>> g_attr;
  size_t cur = 0;
  for (auto& a : g_attr)
    if (a.first == kern) cur = a.second;
  if (smem > cur) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    bool found = false;
    for (auto& a : g_attr)
      if (a.first == kern) { a.second = smem; found = true; }
    if (!found) g_attr.push_back({kern, smem});
  }
  if (per_sm < 0) {
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem));
    g_occ.push_back({OccKey{kern, smem}, per_sm});
  }
  if (per_sm < 1) return fail(ctx, GMRES_ECUDA, "solve kernel cannot be resident (occupancy 0)");
  if (ctas_per_sm > 0) per_sm = std::min(per_sm, ctas_per_sm);
  *G = per_sm * ctx->sms;
  return 0;
}

// CSR chunks of every CTA's rows for the TMA-staged stream (gmres_kernels.cuh
// csr_stream): ≤ CHUNK_RMAX rows and ≤ CHUNK_CAP non-zeros, boundaries at
// multiples of 4 rows; 4-row groups above CHUNK_CAP become "direct" chunks.
void make_chunks(const std::vector<int32_t>& rp, int64_t n, const std::vector<int>& rb, std::vector<int4>& ent,
                 std::vector<int>& off) {
  const int G = (int)rb.size() - 1;
  ent.clear();
  off.assign(G + 1, 0);
  for (int g = 0; g < G; ++g) {
    off[g] = (int)ent.size();
    const int64_t r0 = std::min<int64_t>(rb[g], n), r1 = std::min<int64_t>(rb[g + 1], n);
    int64_t r = r0;
    while (r < r1) {
      const int64_t g4 = std::min(r + 4, r1);
      if ((int64_t)rp[g4] - rp[r] > CHUNK_CAP) {  // direct chunk
        ent.push_back(make_int4((int)r, rp[r], 1, 0));
        r = g4;
        continue;
      }
      int64_t e = g4;
      while (e < r1) {
        const int64_t e4 = std::min(e + 4, r1);
        if (e4 - r > CHUNK_RMAX || (int64_t)rp[e4] - rp[r] > CHUNK_CAP) break;
        e = e4;
      }
      ent.push_back(make_int4((int)r, rp[r], 0, 0));
      r = e;
    }
    ent.push_back(make_int4((int)r1, rp[r1], 0, 0));  // sentinel
  }
  off[G] = (int)ent.size();
}

// block-stream stages of every CTA's rows (gmres_kernels.cuh csr_block_stream):
// ≤ BS_BYTES of row_ptr / per-row operand / col / val slices at the widest types
// (fp64 values and operand), boundaries at multiples of 4 rows
void make_stages(const std::vector<int32_t>& rp, int64_t n, const std::vector<int>& rb, std::vector<int2>& ent,
                 std::vector<int>& off) {
  const int G = (int)rb.size() - 1;
  auto bytes = [&](int64_t s, int64_t e) {
    const int64_t rows = e - s, ea = rp[s] & ~3LL, eb = (rp[e] + 3) & ~3LL;
    return ((rows + 1 + 3) & ~3LL) * 4 + ((rows * 8 + 15) & ~15LL) + (eb - ea) * 12;
  };
  ent.clear();
  off.assign(G + 1, 0);
  for (int g = 0; g < G; ++g) {
    off[g] = (int)ent.size();
    const int64_t r0 = std::min<int64_t>(rb[g], n), r1 = std::min<int64_t>(rb[g + 1], n);
    int64_t s = r0;
    while (s < r1) {
      int64_t e = std::min(s + 4, r1);
      while (e < r1) {
        const int64_t e2 = std::min(e + 4, r1);
        if (bytes(s, e2) > BS_BYTES) break;
        e = e2;
      }
      ent.push_back(make_int2((int)s, rp[s]));
      s = e;
    }
    ent.push_back(make_int2((int)r1, rp[r1]));  // sentinel
  }
  off[G] = (int)ent.size();
}

// merge-path tiles of every CTA's non-zeros (gmres_kernels.cuh csr_merge_stream):
// a tile starts at position s (its base A = s & ~7), ends at ne ≤ A + MT_CAP and
// touches ≤ MT_RMAX rows (else it ends with its MT_RMAX-th row); rows may span
// tiles.  Split rows: {local row, tile of its first position, tile of its last}.
// Rows are non-empty (every row holds its diagonal, validated at create).
void make_mtiles(const std::vector<int32_t>& rp, int64_t n, const std::vector<int>& rb, std::vector<int4>& ent,
                 std::vector<int>& off, std::vector<int4>& split, std::vector<int>& soff) {
  const int G = (int)rb.size() - 1;
  ent.clear();
  split.clear();
  off.assign(G + 1, 0);
  soff.assign(G + 1, 0);
  for (int g = 0; g < G; ++g) {
    off[g] = (int)ent.size();
    soff[g] = (int)split.size();
    const int64_t r0 = std::min<int64_t>(rb[g], n), r1 = std::min<int64_t>(rb[g + 1], n);
    int64_t s = rp[r0], r = r0, open_tile = -1;
    const int64_t E1 = rp[r1];
    while (s < E1) {
      const int64_t A = s & ~7LL;
      int64_t ne = std::min<int64_t>(A + MT_CAP, E1);
      int64_t rz = r;
      while (rp[rz + 1] < ne) ++rz;  // row holding position ne − 1
      if (rz - r + 1 > MT_RMAX) {
        rz = r + MT_RMAX - 1;
        ne = rp[rz + 1];
      }
      const int c = (int)ent.size();
      ent.push_back(make_int4((int)r, (int)s, (int)(rz - r + 1), 0));
      const bool open_l = rp[r] < s, open_r = rp[rz + 1] > ne;
      if (open_l && rp[r + 1] <= ne) split.push_back(make_int4((int)r, (int)open_tile, c, 0));
      if (open_r && !(open_l && rz == r)) open_tile = c;
      s = ne;
      r = rp[rz + 1] == ne ? rz + 1 : rz;
    }
    ent.push_back(make_int4((int)r1, (int)E1, 0, 0));  // sentinel (its y ends the last tile)
  }
  off[G] = (int)ent.size();
  soff[G] = (int)split.size();
}

void free_parts(gmres_ctx* ctx) {
  for (auto& p : ctx->parts) {
    cudaFree(p.d_row_begin);
    cudaFree(p.d_chunks);
    cudaFree(p.d_chunk_off);
    cudaFree(p.d_send);
    cudaFree(p.d_stages);
    cudaFree(p.d_stage_off);
    cudaFree(p.d_mtiles);
    cudaFree(p.d_mt_off);
    cudaFree(p.d_msplit);
    cudaFree(p.d_ms_off);
    cudaFree(p.d_mcarry);
  }
  ctx->d_stages = nullptr;
  ctx->d_stage_off = nullptr;
  ctx->d_mtiles = nullptr;
  ctx->d_mt_off = nullptr;
  ctx->d_msplit = nullptr;
  ctx->d_ms_off = nullptr;
  ctx->d_mcarry = nullptr;
  ctx->parts.clear();
  ctx->d_row_begin = nullptr;
  ctx->d_chunks = nullptr;
  ctx->d_chunk_off = nullptr;
  ctx->d_send = nullptr;
  ctx->part_G = 0;
}

int ensure_partition(gmres_ctx* ctx, int G, int align = ROWALIGN) {
  for (auto& p : ctx->parts) {
    if (p.G == G && p.align == align) {
      ctx->d_row_begin = p.d_row_begin;
      ctx->d_chunks = p.d_chunks;
      ctx->d_chunk_off = p.d_chunk_off;
      ctx->d_send = p.d_send;
      ctx->d_stages = p.d_stages;
      ctx->d_stage_off = p.d_stage_off;
      ctx->d_mtiles = p.d_mtiles;
      ctx->d_mt_off = p.d_mt_off;
      ctx->d_msplit = p.d_msplit;
      ctx->d_ms_off = p.d_ms_off;
      ctx->d_mcarry = p.d_mcarry;
      ctx->part_G = G;
      ctx->part_align = align;
      ctx->part_max_rows = p.max_rows;
      return 0;
    }
  }
  if (ctx->parts.size() >= 4) free_parts(ctx);
  std::vector<int> rb;
  make_partition(ctx->h_rp, ctx->n, ctx->nvec, G, align, rb);
  gmres_ctx::Part P{G, align, 0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                    nullptr, nullptr, nullptr, nullptr, nullptr};
  for (int g = 0; g < G; ++g) P.max_rows = std::max(P.max_rows, rb[g + 1] - rb[g]);
  std::vector<int4> ent;
  std::vector<int> off;
  make_chunks(ctx->h_rp, ctx->n, rb, ent, off);
  auto bail = [&](cudaError_t e) {
    cudaFree(P.d_row_begin); cudaFree(P.d_chunks); cudaFree(P.d_chunk_off); cudaFree(P.d_send);
    cudaFree(P.d_stages); cudaFree(P.d_stage_off);
    cudaFree(P.d_mtiles); cudaFree(P.d_mt_off); cudaFree(P.d_msplit); cudaFree(P.d_ms_off); cudaFree(P.d_mcarry);
    return fail(ctx, e == cudaErrorMemoryAllocation ? GMRES_ENOMEM : GMRES_ECUDA, cudaGetErrorString(e));
  };
  cudaError_t e = cudaMalloc(&P.d_row_begin, sizeof(int) * (G + 1));
  if (e == cudaSuccess) e = cudaMemcpy(P.d_row_begin, rb.data(), sizeof(int) * (G + 1), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&P.d_chunks, sizeof(int4) * ent.size());
  if (e == cudaSuccess) e = cudaMemcpy(P.d_chunks, ent.data(), sizeof(int4) * ent.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&P.d_chunk_off, sizeof(int) * (G + 1));
  if (e == cudaSuccess) e = cudaMemcpy(P.d_chunk_off, off.data(), sizeof(int) * (G + 1), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return bail(e);
  if (ctx->block_ok) {
    std::vector<int2> st;
    std::vector<int> soff;
    make_stages(ctx->h_rp, ctx->n, rb, st, soff);
    e = cudaMalloc(&P.d_stages, sizeof(int2) * st.size());
    if (e == cudaSuccess) e = cudaMemcpy(P.d_stages, st.data(), sizeof(int2) * st.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&P.d_stage_off, sizeof(int) * (G + 1));
    if (e == cudaSuccess) e = cudaMemcpy(P.d_stage_off, soff.data(), sizeof(int) * (G + 1), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return bail(e);
  }
  if (ctx->merge_ok) {
    std::vector<int4> mt, ms;
    std::vector<int> mto, mso;
    make_mtiles(ctx->h_rp, ctx->n, rb, mt, mto, ms, mso);
    auto up = [&](void** dst, const void* src, size_t bytes) {
      cudaError_t r = cudaMalloc(dst, std::max<size_t>(bytes, 16));
      if (r == cudaSuccess && bytes) r = cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
      return r;
    };
    e = up((void**)&P.d_mtiles, mt.data(), sizeof(int4) * mt.size());
    if (e == cudaSuccess) e = up((void**)&P.d_mt_off, mto.data(), sizeof(int) * mto.size());
    if (e == cudaSuccess) e = up((void**)&P.d_msplit, ms.data(), sizeof(int4) * ms.size());
    if (e == cudaSuccess) e = up((void**)&P.d_ms_off, mso.data(), sizeof(int) * mso.size());
    if (e == cudaSuccess) e = cudaMalloc(&P.d_mcarry, sizeof(double) * 2 * mt.size());
    if (e != cudaSuccess) return bail(e);
  }
  if (ctx->dist() && ctx->linked) {  // per-CTA send lists (halo push)
    // a peer that gathers at least half of this rank's rows (random-column matrices:
    // ghosts ≈ every remote row) receives whole contiguous row blocks
    // (an all-gather of the vector) instead of per-element pushes
    ctx->halo_full = 0;
    for (int q = 0; q < ctx->nranks; ++q)
      if (q != ctx->rank && 2 * (int64_t)ctx->send_rows[q].size() >= ctx->n) ctx->halo_full |= 1u << q;
    std::vector<std::pair<int, int>> se;  // (local row, peer)
    for (int q = 0; q < ctx->nranks; ++q)
      if (!((ctx->halo_full >> q) & 1u))
        for (int32_t r : ctx->send_rows[q]) se.push_back({r, q});
    std::sort(se.begin(), se.end());
    std::vector<int> buf(G + 1 + 2 * se.size());
    // offsets: CTA g pushes the entries with rb[g] <= row < rb[g+1]
    for (int g = 0; g <= G; ++g) {
      buf[g] = g == G ? (int)se.size()
                      : (int)(std::lower_bound(se.begin(), se.end(), std::make_pair(rb[g], -1)) - se.begin());
    }
    for (size_t i = 0; i < se.size(); ++i) {
      buf[G + 1 + i] = se[i].first;
      buf[G + 1 + se.size() + i] = se[i].second;
    }
    e = cudaMalloc(&P.d_send, sizeof(int) * std::max<size_t>(buf.size(), 1));
    if (e == cudaSuccess) e = cudaMemcpy(P.d_send, buf.data(), sizeof(int) * buf.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return bail(e);
  }
  ctx->parts.push_back(P);
  return ensure_partition(ctx, G, align);
}

// workspace for (m, prec, G); zero-filled so that padding rows stay 0
int ensure_ws(gmres_ctx* ctx, int m, int prec, int G, int hist_cap, int inner_cap) {
  if (ctx->ws_m == m && ctx->ws_prec == prec && ctx->ws_G >= G && ctx->hist_cap >= hist_cap &&
      ctx->inner_cap >= inner_cap)
    return 0;
  if (ctx->d_ws) cudaFree(ctx->d_ws);
  ctx->d_ws = nullptr;
  const size_t wb = prec == GMRES_MIXED ? 4 : 8;
  const size_t kmax = (size_t)kmax_for(m);
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t r = off; off += (bytes + 255) & ~size_t(255); return r; };
  // V: column-major ldv × (m+1), or row-blocked (nvec/32 blocks at most,
  // each (m+1) columns of 32 + 16/wb elements) — the larger of the two
  const size_t v_cm = (size_t)ctx->ldv * (m + 1);
  const size_t v_bl = (size_t)(ctx->nvec / 32) * (m + 1) * (32 + 16 / wb);
  const size_t oV = take(wb * std::max(v_cm, v_bl));
  const size_t ow0 = take(wb * ctx->ldv);
  const size_t ow1 = take(wb * ctx->ldv);
  const size_t kst = (kmax + 3) & ~size_t(3);
  const size_t oP = take(sizeof(double) * (2 * G * kst + 2 * G));  // + the one-value partials
  const size_t octr = take(sizeof(unsigned long long) * 4);
  const size_t oR = take(sizeof(double) * kmax * m);
  const size_t oy = take(sizeof(double) * kmax);
  const size_t oum = take(sizeof(double) * (m + 1) * (m + 1));
  const size_t osm = take(sizeof(double) * (m + 1) * (m + 1));
  const size_t ofl = take(sizeof(int) * 8);
  const size_t ooi = take(sizeof(int) * 8);
  const size_t ood = take(sizeof(double) * 4);
  const size_t opr = take(sizeof(unsigned long long) * PH_N);
  const size_t opc = take(sizeof(unsigned long long) * G);
  const size_t oh = take(sizeof(double) * hist_cap);
  const size_t ocj = take(sizeof(int) * hist_cap);
  const size_t oi = take(sizeof(double) * std::max(inner_cap, 1));
  CK(cudaMalloc(&ctx->d_ws, off));
  CK(cudaMemsetAsync(ctx->d_ws, 0, off, ctx->stream));
  ctx->ws_bytes = off;
  ctx->d_V = ctx->d_ws + oV;
  ctx->ws_v_bytes = ow0 - oV;
  ctx->ws_v_tb = -1;
  ctx->d_w0 = ctx->d_ws + ow0;
  ctx->d_w1 = ctx->d_ws + ow1;
  ctx->d_slots = (double*)(ctx->d_ws + oP);
  ctx->slots_count = 2 * G * kst;
  ctx->d_ctr = (unsigned long long*)(ctx->d_ws + octr);
  ctx->d_R = (double*)(ctx->d_ws + oR);
  ctx->d_y = (double*)(ctx->d_ws + oy);
  ctx->d_umat = (double*)(ctx->d_ws + oum);
  ctx->d_smat = (double*)(ctx->d_ws + osm);
  ctx->d_flags = (int*)(ctx->d_ws + ofl);
  ctx->d_out_int = (int*)(ctx->d_ws + ooi);
  ctx->d_out_dbl = (double*)(ctx->d_ws + ood);
  ctx->d_prof = (unsigned long long*)(ctx->d_ws + opr);
  ctx->d_prof_cta = (unsigned long long*)(ctx->d_ws + opc);
  ctx->d_hist = (double*)(ctx->d_ws + oh);
  ctx->d_cycJ = (int*)(ctx->d_ws + ocj);
  ctx->d_inner = (double*)(ctx->d_ws + oi);
  ctx->hist_cap = hist_cap;
  ctx->inner_cap = inner_cap;
  ctx->ws_m = m;
  ctx->ws_prec = prec;
  ctx->ws_G = G;
  return 0;
}

// A32 = RN32(A64) on the stream with the overflow flag in err (device int).
int launch_cast(gmres_ctx* ctx, cudaStream_t st, int* d_errflag) {
  if (!ctx->d_a32) {
    CK(cudaMalloc(&ctx->d_a32, sizeof(float) * (ctx->nnz + ARR_PAD)));
    CK(cudaMemset(ctx->d_a32, 0, sizeof(float) * (ctx->nnz + ARR_PAD)));
  }
  cast32_kernel<<<ctx->sms * 8, 256, 0, st>>>(ctx->d_a64, ctx->d_a32, ctx->nnz, d_errflag);
  CK(cudaGetLastError());
  return 0;
}

int ensure_a32(gmres_ctx* ctx, cudaStream_t st, bool force = false) {
  if (ctx->a32_ready && !force) return 0;
  if (!ctx->d_a32) {
    CK(cudaMalloc(&ctx->d_a32, sizeof(float) * (ctx->nnz + ARR_PAD)));
    CK(cudaMemset(ctx->d_a32, 0, sizeof(float) * (ctx->nnz + ARR_PAD)));
  }
  int* d_err = nullptr;
  CK(cudaMallocAsync(&d_err, sizeof(int), st));
  CK(cudaMemsetAsync(d_err, 0, sizeof(int), st));
  const int blocks = ctx->sms * 8;
  cast32_kernel<<<blocks, 256, 0, st>>>(ctx->d_a64, ctx->d_a32, ctx->nnz, d_err);
  CK(cudaGetLastError());
  int herr = 0;
  CK(cudaMemcpyAsync(&herr, d_err, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaFreeAsync(d_err, st));
  CK(cudaStreamSynchronize(st));
  if (herr) return fail(ctx, GMRES_EFP32RANGE, "matrix value outside the fp32 range (mixed mode)");
  ctx->a32_ready = true;
  return 0;
}

// ---------------------------------------------------------------- ILU(0) (§8 f2)
// Level schedules of the triangular solves (reading R24): lower level of row i =
// 1 + max over its columns k < i (0 if none), upper level = 1 + max over k > i;
// rows sorted by level, ascending row inside a level.  The factorisation follows
// the lower schedule.
int ensure_ilu_plan(gmres_ctx* ctx) {
  if (ctx->ilu_plan) return 0;
  if (ctx->dist()) return fail(ctx, GMRES_EINVAL, "ILU(0) needs a single-rank context");
  const int64_t n = ctx->n, nnz = ctx->nnz;
  const std::vector<int32_t>& rp = ctx->h_rp;
  std::vector<int32_t> ci(nnz);
  CK(cudaMemcpy(ci.data(), ctx->d_ci, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost));
  std::vector<int> dpos(n, -1), lev(n);
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e)
      if (ci[e] == i) dpos[i] = (int)e;
    if (dpos[i] < 0) return fail(ctx, GMRES_EZERODIAG, "ILU(0): row " + std::to_string(i) + " has no diagonal entry");
  }
  auto sched = [&](int t, bool lower) -> int {
    int nl = 0;
    for (int64_t s = 0; s < n; ++s) {
      const int64_t i = lower ? s : n - 1 - s;
      int l = 0;
      const int64_t e0 = lower ? rp[i] : dpos[i] + 1, e1 = lower ? dpos[i] : rp[i + 1];
      for (int64_t e = e0; e < e1; ++e) l = std::max(l, lev[ci[e]] + 1);
      lev[i] = l;
      nl = std::max(nl, l + 1);
    }
    std::vector<int> off(nl + 1, 0), rows(n);
    for (int64_t i = 0; i < n; ++i) off[lev[i] + 1]++;
    for (int l = 0; l < nl; ++l) off[l + 1] += off[l];
    std::vector<int> cur(off.begin(), off.end() - 1);
    for (int64_t i = 0; i < n; ++i) rows[cur[lev[i]]++] = (int)i;
    // entry lists per slot: the row's strictly lower (T = 0) or upper (T = 1) entries
    std::vector<int> eoff(n + 1, 0), ecol, eidx;
    for (int64_t s = 0; s < n; ++s) {
      const int i = rows[s];
      const int64_t e0 = lower ? rp[i] : dpos[i] + 1, e1 = lower ? dpos[i] : rp[i + 1];
      for (int64_t e = e0; e < e1; ++e) {
        ecol.push_back(ci[e]);
        eidx.push_back((int)e);
      }
      eoff[s + 1] = (int)ecol.size();
    }
    const size_t ne = std::max<size_t>(ecol.size(), 1);
    if (cudaMalloc(&ctx->d_ilu_lev[t], sizeof(int) * (nl + 2)) != cudaSuccess ||
        cudaMalloc(&ctx->d_ilu_rows[t], sizeof(int) * n) != cudaSuccess ||
        cudaMalloc(&ctx->d_ilu_eoff[t], sizeof(int) * (n + 1)) != cudaSuccess ||
        cudaMalloc(&ctx->d_ilu_ecol[t], sizeof(int) * ne) != cudaSuccess ||
        cudaMalloc(&ctx->d_ilu_eidx[t], sizeof(int) * ne) != cudaSuccess)
      return -1;
    off.push_back(off.back());  // lev[nl + 1]: the prefetch of "level nl" reads an empty range
    cudaMemcpy(ctx->d_ilu_lev[t], off.data(), sizeof(int) * (nl + 2), cudaMemcpyHostToDevice);
    off.pop_back();
    cudaMemcpy(ctx->d_ilu_rows[t], rows.data(), sizeof(int) * n, cudaMemcpyHostToDevice);
    cudaMemcpy(ctx->d_ilu_eoff[t], eoff.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice);
    if (!ecol.empty()) {
      cudaMemcpy(ctx->d_ilu_ecol[t], ecol.data(), sizeof(int) * ecol.size(), cudaMemcpyHostToDevice);
      cudaMemcpy(ctx->d_ilu_eidx[t], eidx.data(), sizeof(int) * eidx.size(), cudaMemcpyHostToDevice);
    }
    ctx->ilu_nlev[t] = nl;
    if (lower) ctx->ilu_hlev0 = off;
    return 0;
  };
  if (sched(0, true) || sched(1, false)) return fail(ctx, GMRES_ENOMEM, "ILU(0) level schedule allocation failed");
  CK(cudaMalloc(&ctx->d_ilu_dpos, sizeof(int) * n));
  CK(cudaMemcpy(ctx->d_ilu_dpos, dpos.data(), sizeof(int) * n, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&ctx->d_ilu_bad, sizeof(int)));
  CK(cudaMalloc(&ctx->d_ilu_pub[0], sizeof(double) * n));
  CK(cudaMalloc(&ctx->d_ilu_pub[1], sizeof(double) * n));
  ctx->ilu_plan = true;
  return 0;
}

// factorise A_W (mixed: the fp32 copy, already (re)built on st) into
// d_ilu_f[prec]: copy, then one launch per lower level; a zero pivot is reported
// unless the fp32 cast overflowed (the solve reports that)
int ilu_factor(gmres_ctx* ctx, int prec, cudaStream_t st) {
  if (int rc = ensure_ilu_plan(ctx)) return rc;
  const size_t wb = prec == GMRES_MIXED ? 4 : 8;
  if (!ctx->d_ilu_f[prec]) CK(cudaMalloc(&ctx->d_ilu_f[prec], wb * (ctx->nnz + ARR_PAD)));
  if (!ctx->d_ones[prec]) {
    CK(cudaMalloc(&ctx->d_ones[prec], wb * ctx->nvec));
    if (prec == GMRES_MIXED) {
      std::vector<float> one(ctx->nvec, 1.0f);
      CK(cudaMemcpy(ctx->d_ones[prec], one.data(), wb * ctx->nvec, cudaMemcpyHostToDevice));
    } else {
      std::vector<double> one(ctx->nvec, 1.0);
      CK(cudaMemcpy(ctx->d_ones[prec], one.data(), wb * ctx->nvec, cudaMemcpyHostToDevice));
    }
  }
  ctx->ilu_ready[prec] = false;
  const void* src = prec == GMRES_MIXED ? (const void*)ctx->d_a32 : (const void*)ctx->d_a64;
  CK(cudaMemcpyAsync(ctx->d_ilu_f[prec], src, wb * ctx->nnz, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemsetAsync(ctx->d_ilu_bad, 0x7f, sizeof(int), st));
  for (int t = 0; t < 2; ++t)  // arm the publish buffers (all-ones: the "not yet" NaN)
    CK(cudaMemsetAsync(ctx->d_ilu_pub[t], 0xff, sizeof(double) * ctx->n, st));
  const std::vector<int>& off = ctx->ilu_hlev0;
  for (int l = 0; l < ctx->ilu_nlev[0]; ++l) {
    const int cnt = off[l + 1] - off[l];
    const int blocks = (cnt + 255) / 256;
    if (prec == GMRES_MIXED)
      ilu_factor_level_kernel<float><<<blocks, 256, 0, st>>>(ctx->d_rp, ctx->d_ci, ctx->d_ilu_dpos,
                                                             ctx->d_ilu_rows[0] + off[l], cnt,
                                                             (float*)ctx->d_ilu_f[prec], ctx->d_ilu_bad);
    else
      ilu_factor_level_kernel<double><<<blocks, 256, 0, st>>>(ctx->d_rp, ctx->d_ci, ctx->d_ilu_dpos,
                                                              ctx->d_ilu_rows[0] + off[l], cnt,
                                                              (double*)ctx->d_ilu_f[prec], ctx->d_ilu_bad);
  }
  // packed per-slot records of both solves from the new factors
  const size_t recb = prec == GMRES_MIXED ? sizeof(IluRec<float>) : sizeof(IluRec<double>);
  for (int t = 0; t < 2; ++t) {
    if (!ctx->d_ilu_rec[prec][t]) CK(cudaMalloc(&ctx->d_ilu_rec[prec][t], recb * ctx->n));
    const int blocks = ctx->sms * 8;
    if (prec == GMRES_MIXED) {
      if (t == 0)
        ilu_records_kernel<float, 0><<<blocks, 256, 0, st>>>((int)ctx->n, ctx->d_ilu_rows[0], ctx->d_ilu_eoff[0],
            ctx->d_ilu_ecol[0], ctx->d_ilu_eidx[0], ctx->d_ilu_dpos, (const float*)ctx->d_ilu_f[prec],
            (IluRec<float>*)ctx->d_ilu_rec[prec][0]);
      else
        ilu_records_kernel<float, 1><<<blocks, 256, 0, st>>>((int)ctx->n, ctx->d_ilu_rows[1], ctx->d_ilu_eoff[1],
            ctx->d_ilu_ecol[1], ctx->d_ilu_eidx[1], ctx->d_ilu_dpos, (const float*)ctx->d_ilu_f[prec],
            (IluRec<float>*)ctx->d_ilu_rec[prec][1]);
    } else {
      if (t == 0)
        ilu_records_kernel<double, 0><<<blocks, 256, 0, st>>>((int)ctx->n, ctx->d_ilu_rows[0], ctx->d_ilu_eoff[0],
            ctx->d_ilu_ecol[0], ctx->d_ilu_eidx[0], ctx->d_ilu_dpos, (const double*)ctx->d_ilu_f[prec],
            (IluRec<double>*)ctx->d_ilu_rec[prec][0]);
      else
        ilu_records_kernel<double, 1><<<blocks, 256, 0, st>>>((int)ctx->n, ctx->d_ilu_rows[1], ctx->d_ilu_eoff[1],
            ctx->d_ilu_ecol[1], ctx->d_ilu_eidx[1], ctx->d_ilu_dpos, (const double*)ctx->d_ilu_f[prec],
            (IluRec<double>*)ctx->d_ilu_rec[prec][1]);
    }
  }
  CK(cudaGetLastError());
  int hb[2] = {0, 0};
  CK(cudaMemcpyAsync(&hb[0], ctx->d_ilu_bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  if (ctx->d_flags) CK(cudaMemcpyAsync(&hb[1], ctx->d_flags + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (hb[0] != 0x7f7f7f7f && !(prec == GMRES_MIXED && hb[1] != 0))
    return fail(ctx, GMRES_EZERODIAG, "ILU(0): zero or non-finite pivot at row " + std::to_string(hb[0]));
  ctx->ilu_ready[prec] = true;
  return 0;
}

void set_ilu_dev(gmres_ctx* ctx, Dev& d, int prec) {
  d.iluW = ctx->d_ilu_f[prec];
  d.ilu_dpos = ctx->d_ilu_dpos;
  for (int t = 0; t < 2; ++t) {
    d.ilu_lev[t] = ctx->d_ilu_lev[t];
    d.ilu_rows[t] = ctx->d_ilu_rows[t];
    d.ilu_nlev[t] = ctx->ilu_nlev[t];
    d.ilu_eoff[t] = ctx->d_ilu_eoff[t];
    d.ilu_ecol[t] = ctx->d_ilu_ecol[t];
    d.ilu_eidx[t] = ctx->d_ilu_eidx[t];
    d.ilu_rec[t] = ctx->d_ilu_rec[prec][t];
  }
  d.ilu_pub[0] = ctx->d_ilu_pub[0];
  d.ilu_pub[1] = ctx->d_ilu_pub[1];
}

Dev make_dev(gmres_ctx* ctx, int m, int prec, int ortho, int G) {
  Dev d{};
  d.n = (int)ctx->n;
  d.m = m;
  d.G = G;
  d.kmax = kmax_for(m);
  d.ortho = ortho;
  d.tile_bytes = tile_bytes_for(m);
  set_smem_offsets(d);
  d.normA2 = ctx->normA2;
  d.rp = ctx->d_rp;
  d.ci = ctx->d_ci;
  d.a64 = ctx->d_a64;
  d.aW = prec == GMRES_MIXED ? (const void*)ctx->d_a32 : (const void*)ctx->d_a64;
  d.dinvW = prec == GMRES_MIXED ? (const void*)ctx->d_dinv32 : (const void*)ctx->d_dinv64;
  d.V = ctx->d_V;
  d.ldv = ctx->ldv;
  d.w0 = ctx->d_w0;
  d.w1 = ctx->d_w1;
  d.slots = ctx->d_slots;
  d.s1off = (long long)ctx->slots_count;  // the one-value partials follow the K-value rows
  d.ctr = ctx->d_ctr;
  for (int q = 0; q < MAXR; ++q) { d.slot_peer[q] = ctx->d_slots; d.ctr_peer[q] = ctx->d_ctr; }
  d.kst = (d.kmax + 3) & ~3;
  d.GG = G;
  d.cta0 = 0;
  d.nranks = 1;
  d.rank = 0;
  d.sys_scope = 0;
  d.mgs_nbuf = 2;
  d.mgs_wsm = 0;
  d.R = ctx->d_R;
  d.y = ctx->d_y;
  d.abort_flag = ctx->d_flags;
  d.err_flag = ctx->d_flags + 1;
  d.row_begin = ctx->d_row_begin;
  d.chunks = ctx->d_chunks;
  d.chunk_off = ctx->d_chunk_off;
  d.stages = ctx->d_stages;
  d.stage_off = ctx->d_stage_off;
  d.block_stream = (ctx->block_ok && ctx->d_stages) ? 1 : 0;
  d.merge_stream = (!d.block_stream && ctx->merge_ok && ctx->d_mtiles) ? 1 : 0;
  d.mtiles = ctx->d_mtiles;
  d.mt_off = ctx->d_mt_off;
  d.msplit = ctx->d_msplit;
  d.ms_off = ctx->d_ms_off;
  d.mcarry = ctx->d_mcarry;
  d.history = ctx->d_hist;
  d.cycle_J = ctx->d_cycJ;
  d.hist_cap = ctx->hist_cap;
  d.inner_hist = ctx->d_inner;
  d.inner_cap = ctx->inner_cap;
  d.out_int = ctx->d_out_int;
  d.out_dbl = ctx->d_out_dbl;
  d.prof = ctx->d_prof;
  d.prof_cta = ctx->d_prof_cta;
  d.row_base = 0;
  d.halo = 0;
  for (int q = 0; q < MAXR; ++q) { d.vec_peer[0][q] = ctx->d_w0; d.vec_peer[1][q] = ctx->d_w1; d.vec_peer[2][q] = nullptr; }
  d.send_off = d.send_row = d.send_peer = nullptr;
  d.timeout_ns = 20ll * 1000 * 1000 * 1000;
  return d;
}

int reset_flags(gmres_ctx* ctx, cudaStream_t st) {
  CK(cudaMemsetAsync(ctx->d_ctr, 0, sizeof(unsigned long long) * 4, st));
  if (ctx->d_fx) CK(cudaMemsetAsync(ctx->d_fx, 0, 1024, st));
  CK(cudaMemsetAsync(ctx->d_flags, 0, sizeof(int) * 8, st));
  return 0;
}

int launch_coop(gmres_ctx* ctx, const void* kern, int G, size_t smem, void** args, cudaStream_t st) {
  CK(cudaLaunchCooperativeKernel(kern, dim3(G), dim3(NT), args, smem, st));
  return 0;
}

int check_prec(gmres_ctx* ctx, int prec) {
  if (prec != GMRES_FP64 && prec != GMRES_MIXED) return fail(ctx, GMRES_EINVAL, "precision must be 0 (fp64) or 1 (mixed)");
  return 0;
}

}  // namespace

extern "C" {

const char* gmres_last_error(const gmres_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

namespace {
// n rows of a (possibly row-partitioned) matrix: global rows [row_begin,
// row_begin + n) of an n_global × n_global matrix, CSR with global columns.
int create_impl(const int32_t* row_ptr, const int32_t* col, const double* val, int64_t n, int64_t nnz, int64_t n_global,
                int64_t row_begin, int nranks, int rank, gmres_ctx** out) {
  gmres_ctx* ctx = nullptr;
  if (!out) return fail(nullptr, GMRES_EINVAL, "out is NULL");
  *out = nullptr;
  if (!row_ptr || (!col && nnz > 0) || (!val && nnz > 0)) return fail(nullptr, GMRES_EINVAL, "null CSR array");
  if (n < 1 || nnz < 0 || n_global > 2000000000LL || nnz > 2147483647LL) return fail(nullptr, GMRES_EINVAL, "bad n/nnz");
  if (row_begin < 0 || row_begin + n > n_global) return fail(nullptr, GMRES_EINVAL, "rows outside [0, n_global)");
  // CSR invariants
  if (row_ptr[0] != 0 || row_ptr[n] != nnz) return fail(nullptr, GMRES_EBADCSR, "row_ptr[0] != 0 or row_ptr[n] != nnz");
  for (int64_t i = 0; i < n; ++i) {
    if (row_ptr[i + 1] < row_ptr[i])
      return fail(nullptr, GMRES_EBADCSR, "row_ptr decreases at row " + std::to_string(row_begin + i));
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
      if (col[e] < 0 || col[e] >= n_global)
        return fail(nullptr, GMRES_EBADCSR, "column out of range in row " + std::to_string(row_begin + i));
      if (e > row_ptr[i] && col[e] <= col[e - 1])
        return fail(nullptr, GMRES_EBADCSR, "columns not strictly increasing in row " + std::to_string(row_begin + i));
    }
  }
  ctx = new gmres_ctx();
  auto bail = [&](int rc) { gmres_destroy(ctx); return rc; };
  cudaError_t e = cudaGetDevice(&ctx->device);
  if (e != cudaSuccess) { g_err = cudaGetErrorString(e); return bail(GMRES_ECUDA); }
  e = cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, ctx->device);
  if (e != cudaSuccess) { g_err = cudaGetErrorString(e); return bail(GMRES_ECUDA); }
  ctx->n = n;
  ctx->nnz = nnz;
  ctx->nvec = round_up(n, VEC_ALIGN);
  ctx->ldv = ctx->nvec;
  ctx->h_rp.assign(row_ptr, row_ptr + n + 1);
  {
    int64_t mx = 0;
    for (int64_t i = 0; i < n; ++i) mx = std::max<int64_t>(mx, row_ptr[i + 1] - row_ptr[i]);
    ctx->block_ok = mx <= BS_MAXROW && !std::getenv("G200_NO_BLOCK_STREAM");
    int64_t mn = n > 0 ? INT64_MAX : 0;
    for (int64_t i = 0; i < n; ++i) mn = std::min<int64_t>(mn, row_ptr[i + 1] - row_ptr[i]);
    ctx->merge_ok = !ctx->block_ok && mn >= 1 && !std::getenv("G200_NO_MERGE_STREAM");
  }
  ctx->nranks = nranks;
  ctx->rank = rank;
  ctx->n_global = n_global;
  ctx->row_begin = row_begin;
  ctx->nvec_global = round_up(n_global, VEC_ALIGN);
  int rc;
  auto setup = [&]() -> int {
    CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&ctx->ev0));
    CK(cudaEventCreate(&ctx->ev1));
    CK(cudaEventCreate(&ctx->evk0));
    CK(cudaEventCreate(&ctx->evk1));
    // slack after the arrays: TMA bulk copies round sizes up to 16 bytes
    CK(cudaMalloc(&ctx->d_rp, sizeof(int32_t) * (n + 1 + ARR_PAD)));
    CK(cudaMalloc(&ctx->d_ci, sizeof(int32_t) * (nnz + ARR_PAD)));
    CK(cudaMalloc(&ctx->d_a64, sizeof(double) * (nnz + ARR_PAD)));
    CK(cudaMemset(ctx->d_rp, 0, sizeof(int32_t) * (n + 1 + ARR_PAD)));
    CK(cudaMemset(ctx->d_ci, 0, sizeof(int32_t) * (nnz + ARR_PAD)));
    CK(cudaMemset(ctx->d_a64, 0, sizeof(double) * (nnz + ARR_PAD)));
    CK(cudaMalloc(&ctx->d_dinv64, sizeof(double) * ctx->nvec));
    CK(cudaMalloc(&ctx->d_dinv32, sizeof(float) * ctx->nvec));
    CK(cudaMemset(ctx->d_dinv64, 0, sizeof(double) * ctx->nvec));
    CK(cudaMemset(ctx->d_dinv32, 0, sizeof(float) * ctx->nvec));
    CK(cudaMemcpy(ctx->d_rp, row_ptr, sizeof(int32_t) * (n + 1), cudaMemcpyHostToDevice));
    if (nnz > 0) {
      CK(cudaMemcpy(ctx->d_ci, col, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(ctx->d_a64, val, sizeof(double) * nnz, cudaMemcpyHostToDevice));
    }
    int* d_bad = nullptr;
    CK(cudaMalloc(&d_bad, sizeof(int)));
    const int big = 0x7fffffff;
    CK(cudaMemcpy(d_bad, &big, sizeof(int), cudaMemcpyHostToDevice));
    dinv_kernel<<<ctx->sms * 8, 256, 0, ctx->stream>>>((int)n, ctx->d_rp, ctx->d_ci, ctx->d_a64, ctx->d_dinv64,
                                                      ctx->d_dinv32, d_bad, (long long)row_begin);
    CK(cudaGetLastError());
    int bad = big;
    CK(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    cudaFree(d_bad);
    if (bad != big)
      return fail(ctx, GMRES_EZERODIAG, "zero or missing diagonal at row " + std::to_string(row_begin + bad));
    {  // ‖A‖_F² of these rows (the solves report the normwise backward error)
      const int np = ctx->sms * 4;
      double* d_part = nullptr;
      CK(cudaMalloc(&d_part, sizeof(double) * (np + 1)));
      sumsq_partial_kernel<<<np, 256, 0, ctx->stream>>>(ctx->d_a64, (long long)nnz, d_part);
      sumsq_final_kernel<<<1, 32, 0, ctx->stream>>>(d_part, np, d_part + np);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(&ctx->normA2, d_part + np, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      cudaFree(d_part);
    }
    if (nranks == 1 && n > 0) {
      // reading R27: a power-of-two bound B on every CTA partial of an MGS projection
      // h = w·v_i of the mixed Jacobi solve: |w_c·v_c| ≤ ‖w‖‖v_i‖ and w = D⁻¹A v_j, so
      // ‖w‖ ≤ ‖D⁻¹A‖₂ ≤ √(‖D⁻¹A‖₁‖D⁻¹A‖∞) (v normalised); ×2 covers the fp32 rounding
      std::vector<double> csum((size_t)n, 0.0);
      double rmax = 0.0;
      for (int64_t i = 0; i < n; ++i) {
        double di = 0.0, rs = 0.0;
        for (int32_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
          rs += std::fabs(val[k]);
          if (col[k] == i) di = val[k];
        }
        const double inv = 1.0 / std::fabs(di);
        rmax = std::max(rmax, rs * inv);
        for (int32_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) csum[(size_t)col[k]] += std::fabs(val[k]) * inv;
      }
      const double cmax = *std::max_element(csum.begin(), csum.end());
      const double bnd = 2.0 * std::sqrt(cmax * rmax);
      if (std::isfinite(bnd) && bnd > 0.0) {
        ctx->fx_exp = (int)std::ceil(std::log2(bnd));
        CK(cudaMalloc(&ctx->d_fx, 1024));
        CK(cudaMemset(ctx->d_fx, 0, 1024));
      }
    }
    if (nranks > 1) {
      // ghost columns (host) and the buffers peers push into / read from
      for (int64_t i = 0; i < nnz; ++i)
        if (col[i] < row_begin || col[i] >= row_begin + n) ctx->ghosts.push_back(col[i]);
      std::sort(ctx->ghosts.begin(), ctx->ghosts.end());
      ctx->ghosts.erase(std::unique(ctx->ghosts.begin(), ctx->ghosts.end()), ctx->ghosts.end());
      const size_t gb = sizeof(double) * ctx->nvec_global;
      CK(cudaMalloc(&ctx->d_gw0, gb));
      CK(cudaMalloc(&ctx->d_gw1, gb));
      CK(cudaMalloc(&ctx->d_gx, gb));
      CK(cudaMemset(ctx->d_gw0, 0, gb));
      CK(cudaMemset(ctx->d_gw1, 0, gb));
      CK(cudaMemset(ctx->d_gx, 0, gb));
      const size_t sb = sizeof(double) * (2 * (size_t)nranks * ctx->sms * KST_MAX + 2 * (size_t)nranks * ctx->sms);
      CK(cudaMalloc(&ctx->d_dslots, sb));
      CK(cudaMalloc(&ctx->d_dctr, 256));
      CK(cudaMemset(ctx->d_dctr, 0, 256));
      CK(cudaMalloc(&ctx->d_epoch, sizeof(unsigned long long) * 2));
      CK(cudaMemset(ctx->d_epoch, 0, sizeof(unsigned long long) * 2));
    }
    return 0;
  };
  rc = setup();
  if (rc != 0) { g_err = ctx->err; return bail(rc); }
  *out = ctx;
  return GMRES_OK;
}
}  // namespace

int gmres_create(const int32_t* row_ptr, const int32_t* col, const double* val, int64_t n, int64_t nnz,
                 gmres_ctx** out) {
  return create_impl(row_ptr, col, val, n, nnz, n, 0, 1, 0, out);
}

void gmres_destroy(gmres_ctx* ctx) {
  if (!ctx) return;
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  cudaFree(ctx->d_rp);
  cudaFree(ctx->d_fx);
  cudaFree(ctx->d_ci);
  cudaFree(ctx->d_a64);
  cudaFree(ctx->d_a32);
  cudaFree(ctx->d_dinv64);
  cudaFree(ctx->d_dinv32);
  cudaFree(ctx->d_ilu_dpos);
  cudaFree(ctx->d_ilu_bad);
  cudaFree(ctx->d_ilu_pub[0]);
  cudaFree(ctx->d_ilu_pub[1]);
  cudaFree(ctx->d_ilu_s32[0]);
  cudaFree(ctx->d_ilu_s32[1]);
  for (int t = 0; t < 2; ++t) {
    cudaFree(ctx->d_ilu_lev[t]);
    cudaFree(ctx->d_ilu_rows[t]);
    cudaFree(ctx->d_ilu_eoff[t]);
    cudaFree(ctx->d_ilu_ecol[t]);
    cudaFree(ctx->d_ilu_eidx[t]);
    cudaFree(ctx->d_ilu_f[t]);
    cudaFree(ctx->d_ilu_rec[t][0]);
    cudaFree(ctx->d_ilu_rec[t][1]);
    cudaFree(ctx->d_ones[t]);
  }
  cudaFree(ctx->d_ws);
  cudaFree(ctx->d_hb);
  cudaFree(ctx->d_hx);
  free_parts(ctx);
  if (ctx->ipc) {
    for (int q = 0; q < ctx->nranks; ++q) {
      if (q == ctx->rank) continue;
      if (ctx->peer_w0[q]) cudaIpcCloseMemHandle(ctx->peer_w0[q]);
      if (ctx->peer_w1[q]) cudaIpcCloseMemHandle(ctx->peer_w1[q]);
      if (ctx->peer_x[q]) cudaIpcCloseMemHandle(ctx->peer_x[q]);
      if (ctx->peer_slots[q]) cudaIpcCloseMemHandle(ctx->peer_slots[q]);
      if (ctx->peer_ctr[q]) cudaIpcCloseMemHandle(ctx->peer_ctr[q]);
    }
  }
  cudaFree(ctx->d_gw0);
  cudaFree(ctx->d_gw1);
  cudaFree(ctx->d_gx);
  cudaFree(ctx->d_dslots);
  cudaFree(ctx->d_dctr);
  cudaFree(ctx->d_epoch);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->evk0) cudaEventDestroy(ctx->evk0);
  if (ctx->evk1) cudaEventDestroy(ctx->evk1);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

namespace {
// MGS variant of a launch (gmres_kernels.cuh a3): 1 mgs_resident — w in ≤ MGS_MV
// 16-byte registers per thread and a ring of NB = 3 (else 2) whole basis-vector
// row blocks; 2 mgs_chunked — the rest of w in shared memory and a ring of ≥ one
// vector's worth of MGS_CHUNK slots; 3 mgs_stream — w off chip (shared + L2), a
// ring of MGS_ITEM slots; 0 mgs_sweep (fallback).  want = −1: the first that
// fits in that order; else exactly that variant (GMRES_EINVAL if it does not
// fit).  kern_for(v): the kernel a variant runs in (its static shared memory
// and occupancy decide "fits").  ext: the chunk-ring / streamed kernels exist
// for this launch.
extern "C++" {
struct MgsPlan { int variant = 0, nbuf = 2, wsm = 0, tile_bytes = 0; const void* kern = nullptr; };
template <class KernFor>
int plan_mgs(gmres_ctx* ctx, int precision, int m, int G, int tile_bytes, int want, int tune, bool ext,
             int ctas_per_sm, KernFor kern_for, MgsPlan& out) {
  const int wb = precision == GMRES_MIXED ? 4 : 8;
  const int nq = ctx->part_max_rows / (16 / wb);
  const int nch = (nq + NT - 1) / NT;
  const int buf_bytes = ((nq + 7) & ~7) * 16;
  out = MgsPlan{};
  out.tile_bytes = tile_bytes;
  out.kern = kern_for(0);
  // a candidate staging size fits when dynamic + the kernel's static shared memory stay within the
  // per-block opt-in limit and the grid stays co-resident; a failed probe leaves no latched error
  auto fits = [&](const void* k, int tb) {
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, k) != cudaSuccess) { cudaGetLastError(); return false; }
    int optin = 0;
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    if (smem_bytes(m, tb) + fa.sharedSizeBytes > (size_t)optin) return false;
    int G2 = 0;
    const bool ok = grid_for(ctx, k, smem_bytes(m, tb), ctas_per_sm, &G2) == 0 && G2 >= G;
    if (!ok) { cudaGetLastError(); ctx->err.clear(); }
    return ok;
  };
  const bool any = want < 0;
  if ((any || want == 1) && nq <= MGS_MV * NT && !(tune & 8192)) {
    for (int nb = (tune & 256) ? 2 : 3; nb >= 2; --nb) {
      const int tb = std::max(tile_bytes, nb * buf_bytes);
      if (fits(kern_for(1), tb)) {
        out = MgsPlan{1, nb, 0, tb, kern_for(1)};
        return 0;
      }
    }
  }
  if ((any || want == 2) && ext) {
    const int wsm = std::max(0, nch - MGS_MV);
    const int ns = std::min<int>(MGS_MAXSLOT, tile_bytes_for(m) / MGS_CHUNK - wsm);
    const int tb = std::max(tile_bytes, (ns + wsm) * MGS_CHUNK);
    if (ns >= nch && fits(kern_for(2), tb)) {
      out = MgsPlan{2, ns, wsm, tb, kern_for(2)};
      return 0;
    }
  }
  // streamed: a ring of item slots, as many whole items of w in shared memory as
  // the rest of the staging region holds (one item when forced, to exercise both tiers)
  if ((any || want == 3) && ext && !(tune & 16384) && (nch > MGS_MV || want == 3)) {
    const int slots = tile_bytes_for(m) / MGS_CHUNK;
    const int ns = std::min(MGS_STREAM_SLOTS, slots / MGS_IC);
    int wsm = std::max(0, std::min(want == 3 ? MGS_IC : slots - ns * MGS_IC, nch));
    wsm -= wsm % MGS_IC;
    const int tb = std::max(tile_bytes, ns * MGS_ITEM + wsm * MGS_CHUNK);
    if (ns >= 2 && fits(kern_for(3), tb)) {
      out = MgsPlan{3, ns, wsm, tb, kern_for(3)};
      return 0;
    }
  }
  if (any || want == 0) {  // mgs_sweep (its own instantiation for the headline kernels)
    if (!fits(out.kern, tile_bytes)) return fail(ctx, GMRES_ECUDA, "MGS sweep kernel cannot be resident");
    return 0;
  }
  return fail(ctx, GMRES_EINVAL, "the requested MGS variant does not fit this matrix / launch");
}
}  // extern "C++"

// Everything a launch of the fused solve needs for one rank: validation,
// grid, partition, basis layout, workspace, the a0 cast, x0 and the Dev.
struct Plan {
  const void* kern = nullptr;
  int G = 0;
  size_t smem = 0;
  Dev d{};
  cudaStream_t st = nullptr;
  int prec = 0;
  bool rec_inner = false;
  double* d_xuser = nullptr;  // caller's x (row-partitioned: copied from the internal full-length x)
};

int plan_solve(gmres_ctx* ctx, const double* d_b, const double* d_x0, double* d_x, int32_t m, double tol,
               int32_t ortho, int32_t precision, const gmres_opts* opts, void* stream, int G_force, bool virt,
               Plan& P) {
  if (!ctx) return fail(nullptr, GMRES_EINVAL, "ctx is NULL");
  ctx->err.clear();
  if (!d_b || !d_x) return fail(ctx, GMRES_EINVAL, "b/x is NULL");
  if (m < 1 || m > MAX_M) return fail(ctx, GMRES_EINVAL, "m must be in [1, 256]");
  if (!(tol > 0.0) || !std::isfinite(tol)) return fail(ctx, GMRES_EINVAL, "tol must be > 0");
  if (ortho != GMRES_MGS && ortho != GMRES_CGSR) return fail(ctx, GMRES_EINVAL, "ortho must be 0 (MGS) or 1 (CGSR)");
  if (int rc = check_prec(ctx, precision)) return rc;
  if (ctx->dist() && !ctx->linked) return fail(ctx, GMRES_EINVAL, "row-partitioned context not linked to its peers");
  const int policy = opts ? opts->restart_policy : 0;
  if (policy < 0 || policy > 3) return fail(ctx, GMRES_EINVAL, "restart_policy must be 0, 1, 2 or 3");
  const double orth_thresh = (opts && opts->orth_thresh > 0.0) ? opts->orth_thresh : 1.0;
  const int orth_norm = opts ? opts->orth_norm : 0;
  if (orth_norm != 0 && orth_norm != 1) return fail(ctx, GMRES_EINVAL, "orth_norm must be 0 (Frobenius) or 1 (spectral)");
  double delta = (opts && opts->delta >= 0.0) ? opts->delta
                                              : (precision == GMRES_MIXED && policy != 2 ? 1e-6 : 0.0);
  if (!std::isfinite(delta)) return fail(ctx, GMRES_EINVAL, "delta must be finite");
  const double stall_factor = (opts && opts->stall_factor > 0.0) ? opts->stall_factor : 1.001;
  const double stall_frac = (opts && opts->stall_frac > 0.0) ? opts->stall_frac : 0.05;
  // f > 1: with f = 1 the stall test |s_{j+1}|·f > |s_{j+1−w}| can never fire (the Arnoldi
  // residual does not increase) — StallDetect's factor
  if (!(stall_factor > 1.0) || !std::isfinite(stall_factor) || !(stall_frac <= 1.0))
    return fail(ctx, GMRES_EINVAL, "stall_factor must be > 1 and stall_frac in (0, 1]");
  const int max_cycles = (opts && opts->max_cycles > 0) ? opts->max_cycles : 10000;
  P.rec_inner = opts && opts->record_inner;
  int L = (opts && opts->lanes_per_row) ? opts->lanes_per_row : auto_lanes(ctx->n, ctx->nnz);
  if (L != 1 && L != 2 && L != 4 && L != 8 && L != 16 && L != 32)
    return fail(ctx, GMRES_EINVAL, "lanes_per_row must be 1/2/4/8/16/32");
  const int precond = opts ? opts->precond : GMRES_PRECOND_JACOBI;
  if (precond != GMRES_PRECOND_JACOBI && precond != GMRES_PRECOND_ILU0 && precond != GMRES_PRECOND_ILU0_FP32)
    return fail(ctx, GMRES_EINVAL, "precond must be 0 (Jacobi), 1 (ILU(0)) or 2 (fp32 ILU(0), fp64 solver)");
  if (precond == GMRES_PRECOND_ILU0_FP32 && precision != GMRES_FP64)
    return fail(ctx, GMRES_EINVAL, "precond 2 (fp32 ILU(0)) needs precision GMRES_FP64");
  const bool ilu = precond != GMRES_PRECOND_JACOBI;
  const bool ilu32 = precond == GMRES_PRECOND_ILU0_FP32;
  if (ilu && (virt || ctx->dist())) return fail(ctx, GMRES_EINVAL, "ILU(0) needs a single-rank context");
  if (ilu && policy == 3) return fail(ctx, GMRES_EINVAL, "restart_policy 3 is not available with ILU(0)");
  // virtual ranks, the monitor and ILU kernels exist for 1 and 4 lanes per row only
  if ((virt || policy == 3 || ilu) && L != 1 && L != 4) {
    if (opts && opts->lanes_per_row)
      return fail(ctx, GMRES_EINVAL, "lanes_per_row must be 1 or 4 with virtual ranks, restart_policy 3 or ILU(0)");
    L = 4;
  }
  P.st = stream ? (cudaStream_t)stream : ctx->stream;
  P.prec = precision;
  const cudaStream_t st = P.st;

  const void* kern = virt ? pick_solve_virtual(precision, L)
                    : policy == 3 ? pick_solve_monitor(precision, L)
                    : ilu ? pick_solve_ilu(precision, L) : pick_solve(precision, L);
  if (virt && policy == 3) return fail(ctx, GMRES_EINVAL, "restart_policy 3 is not available for virtual ranks");
  // CGSR's row tiles take all the shared memory left; MGS needs only the CSR
  // stream's ring (more L1 for the non-resident sweep's loads)
  int tile_bytes = ortho == GMRES_CGSR ? tile_bytes_for(m) : TILE_BYTES;
  size_t smem = smem_bytes(m, tile_bytes);
  int G = 0;
  if (int rc = grid_for(ctx, kern, smem, opts ? opts->ctas_per_sm : 0, &G)) return rc;
  if (G_force) G = G_force;
  const VLayout vl = (opts && (opts->tune & 4096)) ? VLayout{} :
                     vlayout_for(ortho, m, precision == GMRES_MIXED ? 4 : 8, tile_bytes);
  if (int rc = ensure_partition(ctx, G, vl.tb ? vl.tb : ROWALIGN)) return rc;
  int mgs_resident = 0, mgs_nbuf = 2, mgs_wsm = 0;
  if (ortho == GMRES_MGS) {
    const int tune = opts ? opts->tune : 0;
    const bool ext = !virt && policy != 3 && !ilu && (L == 1 || L == 4);  // chunk-ring / streamed kernels exist
    const int want = (tune & 4) ? 0 : (tune & 524288) ? 3 : -1;
    MgsPlan mp;
    if (int rc = plan_mgs(ctx, precision, m, G, tile_bytes, want, tune, ext, opts ? opts->ctas_per_sm : 0,
                          [&](int v) -> const void* {
                            return v == 2 ? pick_solve_chunked(precision, L)
                                 : v == 3 ? pick_solve_stream(precision, L)
                                 : v == 0 && ext ? pick_solve_sweep(precision, L) : kern;
                          }, mp))
      return rc;
    mgs_resident = mp.variant;
    mgs_nbuf = mp.nbuf;
    mgs_wsm = mp.wsm;
    tile_bytes = mp.tile_bytes;
    kern = mp.kern;
    smem = smem_bytes(m, tile_bytes);
  }
  const int hist_cap_dev = max_cycles + 2;
  const int inner_cap_dev = P.rec_inner ? (int)std::min<int64_t>((int64_t)max_cycles * m, 1 << 22) : 0;
  if (int rc = ensure_ws(ctx, m, precision, G, hist_cap_dev, inner_cap_dev)) return rc;

  CK(cudaEventRecord(ctx->ev0, st));
  // The padding rows (n ≤ row < nvec) of V must read as zero (the passes run over
  // whole row blocks; zero padding keeps w's padding zero).  MGS (column-major)
  // and CGSR (row-blocked) solves share the workspace, and one layout's padding
  // aliases the other's data: clear V whenever the layout changes.
  if (ctx->ws_v_tb != vl.tb) {
    CK(cudaMemsetAsync(ctx->d_V, 0, ctx->ws_v_bytes, st));
    ctx->ws_v_tb = vl.tb;
  }
  if (ctx->dist()) {  // the arrival counter stays monotonic (epoch base): only the flags reset
    CK(cudaMemsetAsync(ctx->d_flags, 0, sizeof(int) * 8, st));
  } else if (int rc = reset_flags(ctx, st)) {
    return rc;
  }
  // a0, preconditioner construction inside the timed solve: the Jacobi
  // diagonal (validated at create; rebuilt here — ~30 µs on C2)
  dinv_kernel<<<ctx->sms * 8, 256, 0, st>>>((int)ctx->n, ctx->d_rp, ctx->d_ci, ctx->d_a64, ctx->d_dinv64,
                                            ctx->d_dinv32, ctx->d_flags + 2, (long long)ctx->row_begin);
  CK(cudaGetLastError());
  if (precision == GMRES_MIXED) {  // a0: rebuilt inside every timed solve;
    // overflow is flagged on the device and reported by the solve kernel
    if (int rc = launch_cast(ctx, st, ctx->d_flags + 1)) return rc;
    ctx->a32_ready = false;  // validated only by a completed solve
  }
  if (ilu32) {  // fp32 factors of RN32(A) for the fp64 solver: the A32 copy first (its range check included)
    if (int rc = launch_cast(ctx, st, ctx->d_flags + 1)) return rc;
    ctx->a32_ready = false;
    for (int t = 0; t < 2; ++t)
      if (!ctx->d_ilu_s32[t]) CK(cudaMalloc(&ctx->d_ilu_s32[t], sizeof(float) * ctx->nvec));
  }
  if (ilu)  // ILU(0) factorisation, inside the timed solve
    if (int rc = ilu_factor(ctx, ilu32 ? GMRES_MIXED : precision, st)) return rc;
  if (ilu32 && !ctx->d_ones[GMRES_FP64]) {  // the fp64 epilogues' unit Jacobi scale
    CK(cudaMalloc(&ctx->d_ones[GMRES_FP64], sizeof(double) * ctx->nvec));
    std::vector<double> one(ctx->nvec, 1.0);
    CK(cudaMemcpy(ctx->d_ones[GMRES_FP64], one.data(), sizeof(double) * ctx->nvec, cudaMemcpyHostToDevice));
  }
  double* xin = ctx->dist() ? ctx->d_gx + ctx->row_begin : d_x;  // the kernel's x (local view)
  if (d_x0 && d_x0 != xin) CK(cudaMemcpyAsync(xin, d_x0, sizeof(double) * ctx->n, cudaMemcpyDeviceToDevice, st));
  if (!d_x0) CK(cudaMemsetAsync(xin, 0, sizeof(double) * ctx->n, st));
  P.d_xuser = d_x;
  CK(cudaMemsetAsync(ctx->d_prof, 0, sizeof(unsigned long long) * PH_N, st));
  CK(cudaMemsetAsync(ctx->d_prof_cta, 0, sizeof(unsigned long long) * G, st));
  CK(cudaMemsetAsync(ctx->d_out_int, 0, sizeof(int) * 8, st));

  Dev d = make_dev(ctx, m, precision, ortho, G);
  d.b = d_b;
  d.x = xin;
  d.tol = tol;
  d.delta = delta;
  d.max_cycles = max_cycles;
  d.policy = policy;
  d.stall_w = policy == 2 ? std::max(1, (int)std::ceil(stall_frac * m)) : 0;
  d.stall_factor = stall_factor;
  d.orth_thresh = orth_thresh;
  d.Umat = ctx->d_umat;
  d.Smat = ctx->d_smat;
  d.orth_spec = orth_norm;
  d.inner_cap = inner_cap_dev;
  d.profile = (opts && opts->profile) ? 1 : 0;
  d.tile_bytes = tile_bytes;
  set_smem_offsets(d);
  d.mgs_resident = mgs_resident;
  d.mgs_nbuf = mgs_nbuf;
  d.mgs_wsm = mgs_wsm;
  if (ilu) {  // M = LU: the SpMV/residual epilogues scale by one, the kernel applies U⁻¹L⁻¹
    set_ilu_dev(ctx, d, ilu32 ? GMRES_MIXED : precision);
    d.dinvW = ctx->d_ones[precision];
    d.ilu32 = ilu32 ? 1 : 0;
    d.ilu_s32[0] = ctx->d_ilu_s32[0];
    d.ilu_s32[1] = ctx->d_ilu_s32[1];
  }
  set_vlayout(d, vl);
  d.tune = opts ? opts->tune : 0;
  // resident MGS ring: the copy of the next vector at the start of the step (default) or inside the
  // step's all-reduce (tune bit 28 flips the default; the kernel reads bit 29)
  d.tune &= ~536870912;
  if (kMgsCopyInAllreduce != bool(d.tune & 268435456)) d.tune |= 536870912;
  if (d.tune & 4194304) d.merge_stream = 0;  // dev A/B: chunk stream instead of the merge-path stream
  // reading R27: exact fixed-point MGS projections in the mixed Jacobi solve on one rank
  // (tune bit 25: the fp64 partial all-reduce instead, dev A/B)
  if (precision == GMRES_MIXED && !ilu && !virt && !ctx->dist() && ctx->d_fx && G <= 600 && !(d.tune & 33554432)) {
    set_fx(d, ctx->fx_exp, ctx->d_fx);
  }
  if (ctx->dist()) {
    const size_t wb = precision == GMRES_MIXED ? 4 : 8;
    d.nranks = ctx->nranks;
    d.rank = ctx->rank;
    d.cta0 = ctx->rank * G;
    d.GG = ctx->nranks * G;
    d.kst = (d.kmax + 3) & ~3;
    d.slots = ctx->d_dslots;
    d.s1off = 2ll * ctx->nranks * ctx->sms * KST_MAX;
    d.ctr = ctx->d_dctr;
    for (int q = 0; q < MAXR; ++q) {
      d.slot_peer[q] = q < ctx->nranks ? ctx->peer_slots[q] : nullptr;
      d.ctr_peer[q] = q < ctx->nranks ? ctx->peer_ctr[q] : nullptr;
      d.vec_peer[0][q] = q < ctx->nranks ? ctx->peer_w0[q] : nullptr;
      d.vec_peer[1][q] = q < ctx->nranks ? ctx->peer_w1[q] : nullptr;
      d.vec_peer[2][q] = q < ctx->nranks ? (void*)ctx->peer_x[q] : nullptr;
    }
    // system-scope release/acquire between GPUs; tune bit 21 forces it for in-process
    // (virtual) ranks so the single-GPU tests execute the multi-GPU memory-order path
    d.sys_scope = (ctx->ipc || (opts && (opts->tune & 2097152))) ? 1 : 0;
    d.halo_full = ctx->halo_full;
    d.row_base = ctx->row_begin;
    d.halo = 1;
    d.w0 = (char*)ctx->d_gw0 + wb * ctx->row_begin;
    d.w1 = (char*)ctx->d_gw1 + wb * ctx->row_begin;
    d.send_off = ctx->d_send;
    d.send_row = ctx->d_send + G + 1;
    d.send_peer = ctx->d_send + G + 1 + (ctx->send_rows.empty() ? 0 : [&] {
      size_t t = 0;
      for (auto& v : ctx->send_rows) t += v.size();
      return t;
    }());
    d.epoch0 = ctx->epoch_base;
    d.red0 = ctx->red_base;
    d.epoch_out = ctx->d_epoch;
  }
  P.kern = kern;
  P.G = G;
  P.smem = smem;
  P.d = d;
  {
    const int32_t pl[GMRES_PLAN_N] = {G, L, d.mgs_resident, d.mgs_nbuf, d.mgs_wsm, tile_bytes, (int32_t)smem,
                                      d.block_stream ? 1 : d.merge_stream ? 2 : 0, vl.tb};
    std::copy(pl, pl + GMRES_PLAN_N, ctx->plan);
  }
  ctx->last_m = m;
  ctx->last_prec = precision;
  ctx->last_vl = vl;
  return 0;
}

// results of a finished launch (stream synchronised by the caller)
int finish_solve(gmres_ctx* ctx, const Plan& P, float ms, float kms, gmres_result* res, double* history,
                 int32_t history_cap, int32_t* history_len) {
  const cudaStream_t st = P.st;
  gmres_result r{};
  int oi[8];
  double od[4];
  unsigned long long prof[PH_N];
  CK(cudaMemcpyAsync(oi, ctx->d_out_int, sizeof(oi), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(od, ctx->d_out_dbl, sizeof(od), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(prof, ctx->d_prof, sizeof(prof), cudaMemcpyDeviceToHost, st));
  if (ctx->dist()) {
    unsigned long long ep[2];
    CK(cudaMemcpyAsync(ep, ctx->d_epoch, sizeof(ep), cudaMemcpyDeviceToHost, st));
    if (P.d_xuser != P.d.x)
      CK(cudaMemcpyAsync(P.d_xuser, P.d.x, sizeof(double) * ctx->n, cudaMemcpyDeviceToDevice, st));
    CK(cudaStreamSynchronize(st));
    ctx->epoch_base = ep[0];
    ctx->red_base = (int)ep[1];
  }
  CK(cudaStreamSynchronize(st));
  r.kernel_ms = kms;
  r.status = oi[0];
  r.cycles = oi[1];
  r.inner_iters = oi[2];
  r.history_len = oi[3];
  r.final_relres = od[0];
  r.final_backward_err = od[1];
  r.device_ms = ms;
  for (int i = 0; i < PH_N; ++i) ctx->phase_ns[i] = (double)prof[i];
  if (P.d.profile) {  // per-CTA own SpMV time: [5] max, [6] mean
    std::vector<unsigned long long> pc(P.G);
    CK(cudaMemcpy(pc.data(), ctx->d_prof_cta, sizeof(unsigned long long) * P.G, cudaMemcpyDeviceToHost));
    double mx = 0, sm = 0;
    for (auto v : pc) { mx = std::max(mx, (double)v); sm += (double)v; }
    ctx->phase_ns[5] = mx;
    ctx->phase_ns[6] = sm / P.G;
    ctx->phase_ns[7] = 0;
  }
  const int hl = std::min(r.history_len, std::min(history_cap, ctx->hist_cap));
  if (history && hl > 0) CK(cudaMemcpy(history, ctx->d_hist, sizeof(double) * hl, cudaMemcpyDeviceToHost));
  if (history_len) *history_len = r.history_len;
  ctx->inner_host.clear();
  ctx->cycJ_host.assign(std::max(0, std::min(r.cycles, ctx->hist_cap)), 0);
  if (!ctx->cycJ_host.empty())
    CK(cudaMemcpy(ctx->cycJ_host.data(), ctx->d_cycJ, sizeof(int) * ctx->cycJ_host.size(), cudaMemcpyDeviceToHost));
  if (P.rec_inner && oi[4] > 0) {
    const int il = std::min(oi[4], ctx->inner_cap);
    ctx->inner_host.resize(il);
    CK(cudaMemcpy(ctx->inner_host.data(), ctx->d_inner, sizeof(double) * il, cudaMemcpyDeviceToHost));
  }
  if (res) *res = r;
  if (r.status == ST_ETIMEOUT) return fail(ctx, GMRES_ETIMEOUT, "device watchdog fired in a grid barrier");
  if (P.prec == GMRES_MIXED && r.status != ST_EFP32RANGE) ctx->a32_ready = true;
  if (r.status == ST_EFP32RANGE) return fail(ctx, GMRES_EFP32RANGE, "matrix or residual entry outside the fp32 range");
  if (r.status == ST_ENONFINITE) return fail(ctx, GMRES_ENONFINITE, "non-finite value in the residual or Arnoldi process");
  return r.status;
}
}  // namespace

int gmres_solve_device(gmres_ctx* ctx, const double* d_b, const double* d_x0, double* d_x, int32_t m, double tol,
                       int32_t ortho, int32_t precision, const gmres_opts* opts, gmres_result* res,
                       double* history, int32_t history_cap, int32_t* history_len, void* stream) {
  if (history_cap < 0) return fail(ctx, GMRES_EINVAL, "history_cap < 0");
  if (ctx && ctx->dist() && !ctx->ipc)
    return fail(ctx, GMRES_EINVAL, "in-process (virtual) ranks are solved together by gmres_solve_virtual");
  Plan P;
  if (int rc = plan_solve(ctx, d_b, d_x0, d_x, m, tol, ortho, precision, opts, stream, 0, false, P)) return rc;
  DevSet ds{};
  ds.d[0] = P.d;
  ds.G = P.G;
  ds.nv = 1;
  void* args[] = {&ds};
  CK(cudaEventRecord(ctx->evk0, P.st));
  if (int rc = launch_coop(ctx, P.kern, P.G, P.smem, args, P.st)) return rc;
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->evk1, P.st));
  CK(cudaEventRecord(ctx->ev1, P.st));
  CK(cudaStreamSynchronize(P.st));
  float ms = 0.f, kms = 0.f;
  CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  CK(cudaEventElapsedTime(&kms, ctx->evk0, ctx->evk1));
  return finish_solve(ctx, P, ms, kms, res, history, history_cap, history_len);
}

// ------------------------------------------------ row partition over ranks (§8 e)
namespace {
// sorted unique global columns of local rows [0, n) (global rows
// [row_begin, row_begin + n)) that lie outside them
void ghosts_of(const int32_t* row_ptr, const int32_t* col, int64_t n, int64_t row_begin, std::vector<int32_t>& g) {
  g.clear();
  for (int64_t e = 0; e < row_ptr[n]; ++e)
    if (col[e] < row_begin || col[e] >= row_begin + n) g.push_back(col[e]);
  std::sort(g.begin(), g.end());
  g.erase(std::unique(g.begin(), g.end()), g.end());
}
// local rows of [row_begin, row_begin + n) that appear in a peer's ghost list
void sends_to(int64_t row_begin, int64_t n, const int32_t* pg, int64_t np, std::vector<int32_t>& rows) {
  rows.clear();
  const int32_t* lo = std::lower_bound(pg, pg + np, (int32_t)row_begin);
  for (const int32_t* p = lo; p < pg + np && *p < row_begin + n; ++p) rows.push_back((int32_t)(*p - row_begin));
}
int copy_out(const std::vector<int32_t>& v, int32_t* out, int64_t cap, int64_t* count) {
  if (count) *count = (int64_t)v.size();
  if (out) std::memcpy(out, v.data(), sizeof(int32_t) * std::min<int64_t>(cap, (int64_t)v.size()));
  return 0;
}
constexpr uint32_t BLOB_MAGIC = 0x47324230u;  // "G2B0"
struct BlobHdr {
  uint32_t magic;
  int32_t rank, nranks, pad;
  int64_t row_begin, n_local, n_global, n_ghost;
  cudaIpcMemHandle_t h[5];  // w0, w1, x, all-reduce partials, arrival counter
};
void relink(gmres_ctx* c) { free_parts(c); c->linked = true; }
}  // namespace

int gmres_dist_ghosts(const int32_t* row_ptr, const int32_t* col, int64_t n_local, int64_t row_begin, int32_t* ghosts,
                      int64_t cap, int64_t* count) {
  if (!row_ptr || (!col && row_ptr[n_local] > 0) || n_local < 0) return fail(nullptr, GMRES_EINVAL, "bad arguments");
  std::vector<int32_t> g;
  ghosts_of(row_ptr, col, n_local, row_begin, g);
  return copy_out(g, ghosts, cap, count);
}

int gmres_dist_sends(int64_t row_begin, int64_t n_local, const int32_t* peer_ghosts, int64_t n_peer_ghosts,
                     int32_t* rows, int64_t cap, int64_t* count) {
  if ((!peer_ghosts && n_peer_ghosts > 0) || n_local < 0) return fail(nullptr, GMRES_EINVAL, "bad arguments");
  std::vector<int32_t> r;
  sends_to(row_begin, n_local, peer_ghosts, n_peer_ghosts, r);
  return copy_out(r, rows, cap, count);
}

int gmres_dist_partition(const int32_t* row_ptr, int64_t n, int32_t nranks, int64_t align, int64_t* bounds) {
  if (!row_ptr || !bounds || n < 1 || nranks < 1 || nranks > MAXR || align < 1) return fail(nullptr, GMRES_EINVAL, "bad arguments");
  // balance rows + nnz (the per-rank cost of a restart cycle: vectors and A),
  // boundaries at multiples of align, last = n
  const double total = (double)n + (double)row_ptr[n];
  bounds[0] = 0;
  for (int q = 1; q < nranks; ++q) {
    const double target = total * q / nranks;
    int64_t lo = bounds[q - 1] / align, hi = n / align;
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if ((double)(mid * align) + (double)row_ptr[mid * align] < target) lo = mid + 1; else hi = mid;
    }
    bounds[q] = lo * align;
  }
  bounds[nranks] = n;
  for (int q = 0; q < nranks; ++q)
    if (bounds[q + 1] <= bounds[q]) return fail(nullptr, GMRES_EINVAL, "too many ranks for this matrix");
  return 0;
}

int gmres_plan_mtiles(const int32_t* row_ptr, int64_t n, const int32_t* cta_rows, int32_t G, int32_t* tiles,
                      int64_t tiles_cap, int64_t* n_tiles, int32_t* tile_off, int32_t* splits, int64_t splits_cap,
                      int64_t* n_splits, int32_t* split_off) {
  if (!row_ptr || !cta_rows || !n_tiles || !n_splits || n < 1 || G < 1) return fail(nullptr, GMRES_EINVAL, "bad arguments");
  for (int64_t i = 0; i < n; ++i)
    if (row_ptr[i + 1] <= row_ptr[i]) return fail(nullptr, GMRES_EINVAL, "merge-path tiles need non-empty rows");
  for (int g = 0; g < G; ++g)
    if (cta_rows[g] < 0 || cta_rows[g + 1] < cta_rows[g]) return fail(nullptr, GMRES_EINVAL, "bad CTA row boundaries");
  std::vector<int32_t> rp(row_ptr, row_ptr + n + 1);
  std::vector<int> rb(cta_rows, cta_rows + G + 1), off, soff;
  std::vector<int4> ent, sp;
  make_mtiles(rp, n, rb, ent, off, sp, soff);
  *n_tiles = (int64_t)ent.size();
  *n_splits = (int64_t)sp.size();
  for (int64_t i = 0; i < std::min<int64_t>(tiles_cap, (int64_t)ent.size()); ++i) {
    tiles[4 * i] = ent[i].x; tiles[4 * i + 1] = ent[i].y; tiles[4 * i + 2] = ent[i].z; tiles[4 * i + 3] = ent[i].w;
  }
  for (int64_t i = 0; i < std::min<int64_t>(splits_cap, (int64_t)sp.size()); ++i) {
    splits[4 * i] = sp[i].x; splits[4 * i + 1] = sp[i].y; splits[4 * i + 2] = sp[i].z; splits[4 * i + 3] = sp[i].w;
  }
  if (tile_off) std::copy(off.begin(), off.end(), tile_off);
  if (split_off) std::copy(soff.begin(), soff.end(), split_off);
  return 0;
}

int gmres_create_dist(const int32_t* row_ptr, const int32_t* col, const double* val, int64_t n_global,
                      int64_t row_begin, int64_t n_local, int32_t nranks, int32_t rank, gmres_ctx** out) {
  if (nranks < 2 || nranks > MAXR || rank < 0 || rank >= nranks) return fail(nullptr, GMRES_EINVAL, "bad nranks/rank");
  if (row_begin % VEC_ALIGN || (n_local % VEC_ALIGN && row_begin + n_local != n_global))
    return fail(nullptr, GMRES_EINVAL, "rank row blocks must start and end at multiples of 256 rows (except the last end)");
  if (!row_ptr) return fail(nullptr, GMRES_EINVAL, "null CSR array");
  return create_impl(row_ptr, col, val, n_local, row_ptr[n_local], n_global, row_begin, nranks, rank, out);
}

int gmres_dist_link_local(gmres_ctx* const* ctxs, int32_t nranks) {
  if (!ctxs || nranks < 2 || nranks > MAXV) return fail(nullptr, GMRES_EINVAL, "need 2..4 in-process ranks");
  for (int i = 0; i < nranks; ++i) {
    gmres_ctx* c = ctxs[i];
    if (!c || c->nranks != nranks || c->rank != i || c->n_global != ctxs[0]->n_global || c->device != ctxs[0]->device)
      return fail(c, GMRES_EINVAL, "contexts must be ranks 0..P-1 of one matrix on one device, in order");
  }
  for (int i = 0; i < nranks; ++i) {
    gmres_ctx* c = ctxs[i];
    c->send_rows.assign(nranks, {});
    for (int q = 0; q < nranks; ++q) {
      c->peer_w0[q] = ctxs[q]->d_gw0;
      c->peer_w1[q] = ctxs[q]->d_gw1;
      c->peer_x[q] = ctxs[q]->d_gx;
      c->peer_slots[q] = ctxs[q]->d_dslots;
      c->peer_ctr[q] = ctxs[q]->d_dctr;
      if (q != i) sends_to(c->row_begin, c->n, ctxs[q]->ghosts.data(), (int64_t)ctxs[q]->ghosts.size(), c->send_rows[q]);
    }
    c->ipc = false;
    relink(c);
  }
  return 0;
}

int gmres_dist_export(gmres_ctx* ctx, void* blob, int64_t cap, int64_t* len) {
  if (!ctx || !ctx->dist() || !len) return fail(ctx, GMRES_EINVAL, "not a row-partitioned context");
  const int64_t need = (int64_t)sizeof(BlobHdr) + (int64_t)sizeof(int32_t) * (int64_t)ctx->ghosts.size();
  *len = need;
  if (!blob) return 0;
  if (cap < need) return fail(ctx, GMRES_EINVAL, "blob buffer too small");
  BlobHdr h{};
  h.magic = BLOB_MAGIC;
  h.rank = ctx->rank;
  h.nranks = ctx->nranks;
  h.row_begin = ctx->row_begin;
  h.n_local = ctx->n;
  h.n_global = ctx->n_global;
  h.n_ghost = (int64_t)ctx->ghosts.size();
  void* bufs[5] = {ctx->d_gw0, ctx->d_gw1, ctx->d_gx, ctx->d_dslots, ctx->d_dctr};
  for (int i = 0; i < 5; ++i) CK(cudaIpcGetMemHandle(&h.h[i], bufs[i]));
  std::memcpy(blob, &h, sizeof(h));
  if (!ctx->ghosts.empty())
    std::memcpy((char*)blob + sizeof(h), ctx->ghosts.data(), sizeof(int32_t) * ctx->ghosts.size());
  return 0;
}

int gmres_dist_import(gmres_ctx* ctx, const void* blobs, const int64_t* offsets) {
  if (!ctx || !ctx->dist() || !blobs || !offsets) return fail(ctx, GMRES_EINVAL, "bad arguments");
  ctx->send_rows.assign(ctx->nranks, {});
  for (int q = 0; q < ctx->nranks; ++q) {
    const char* b = (const char*)blobs + offsets[q];
    BlobHdr h;
    std::memcpy(&h, b, sizeof(h));
    if (h.magic != BLOB_MAGIC || h.rank != q || h.nranks != ctx->nranks || h.n_global != ctx->n_global ||
        offsets[q + 1] - offsets[q] != (int64_t)sizeof(h) + (int64_t)sizeof(int32_t) * h.n_ghost)
      return fail(ctx, GMRES_EINVAL, "malformed blob of rank " + std::to_string(q));
    if (q == ctx->rank) {
      ctx->peer_w0[q] = ctx->d_gw0;
      ctx->peer_w1[q] = ctx->d_gw1;
      ctx->peer_x[q] = ctx->d_gx;
      ctx->peer_slots[q] = ctx->d_dslots;
      ctx->peer_ctr[q] = ctx->d_dctr;
      continue;
    }
    void* p[5];
    for (int i = 0; i < 5; ++i) CK(cudaIpcOpenMemHandle(&p[i], h.h[i], cudaIpcMemLazyEnablePeerAccess));
    ctx->peer_w0[q] = p[0];
    ctx->peer_w1[q] = p[1];
    ctx->peer_x[q] = (double*)p[2];
    ctx->peer_slots[q] = (double*)p[3];
    ctx->peer_ctr[q] = (unsigned long long*)p[4];
    sends_to(ctx->row_begin, ctx->n, (const int32_t*)(b + sizeof(h)), h.n_ghost, ctx->send_rows[q]);
  }
  ctx->ipc = true;
  relink(ctx);
  return 0;
}

int gmres_solve_virtual(gmres_ctx* const* ctxs, int32_t nranks, const double* const* d_b, const double* const* d_x0,
                        double* const* d_x, int32_t m, double tol, int32_t ortho, int32_t precision,
                        const gmres_opts* opts, gmres_result* res) {
  if (!ctxs || nranks < 2 || nranks > MAXV || !d_b || !d_x) return fail(nullptr, GMRES_EINVAL, "bad arguments");
  for (int i = 0; i < nranks; ++i)
    if (!ctxs[i] || !ctxs[i]->linked || ctxs[i]->ipc || ctxs[i]->nranks != nranks || ctxs[i]->rank != i)
      return fail(ctxs[i], GMRES_EINVAL, "contexts must be linked in-process ranks 0..P-1");
  gmres_ctx* c0 = ctxs[0];
  gmres_ctx* ctx = c0;  // (error reporting)
  const int G = c0->sms / nranks;  // every rank gets an equal share of the device
  Plan P[MAXV];
  for (int i = 0; i < nranks; ++i)
    if (int rc = plan_solve(ctxs[i], d_b[i], d_x0 ? d_x0[i] : nullptr, d_x[i], m, tol, ortho, precision, opts, nullptr,
                            G, true, P[i]))
      return rc;
  for (int i = 0; i < nranks; ++i) {
    cudaError_t e = cudaStreamSynchronize(ctxs[i]->stream);
    if (e != cudaSuccess) return fail(ctxs[i], GMRES_ECUDA, cudaGetErrorString(e));
  }
  size_t smem = 0;
  for (int i = 0; i < nranks; ++i) {
    if (P[i].kern != P[0].kern) return fail(c0, GMRES_EINVAL, "ranks need the same kernel (lanes per row)");
    smem = std::max(smem, P[i].smem);
  }
  int per_sm = 0;
  CK(cudaFuncSetAttribute(P[0].kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, P[0].kern, NT, smem));
  if (per_sm < 1) return fail(c0, GMRES_ECUDA, "solve kernel cannot be resident");
  DevSet ds{};
  for (int i = 0; i < nranks; ++i) ds.d[i] = P[i].d;
  ds.G = G;
  ds.nv = nranks;
  void* args[] = {&ds};
  CK(cudaEventRecord(c0->evk0, c0->stream));
  if (int rc = launch_coop(c0, P[0].kern, G * nranks, smem, args, c0->stream)) return rc;
  CK(cudaGetLastError());
  CK(cudaEventRecord(c0->evk1, c0->stream));
  CK(cudaStreamSynchronize(c0->stream));
  float kms = 0.f;
  CK(cudaEventElapsedTime(&kms, c0->evk0, c0->evk1));
  int rc_all = 0;
  for (int i = 0; i < nranks; ++i) {
    const int rc = finish_solve(ctxs[i], P[i], kms, kms, res ? &res[i] : nullptr, nullptr, 0, nullptr);
    if (i == 0 || rc < 0) rc_all = rc;
  }
  return rc_all;
}

int gmres_solve(gmres_ctx* ctx, const double* b, const double* x0, double* x_out, int32_t m, double tol,
                int32_t ortho, int32_t precision, const gmres_opts* opts, gmres_result* res, double* history,
                int32_t history_cap, int32_t* history_len) {
  if (!ctx) return fail(nullptr, GMRES_EINVAL, "ctx is NULL");
  if (!b || !x_out) return fail(ctx, GMRES_EINVAL, "b/x_out is NULL");
  const size_t bytes = sizeof(double) * ctx->n;
  if (!ctx->d_hb) CK(cudaMalloc(&ctx->d_hb, bytes));
  if (!ctx->d_hx) CK(cudaMalloc(&ctx->d_hx, bytes));
  CK(cudaMemcpyAsync(ctx->d_hb, b, bytes, cudaMemcpyHostToDevice, ctx->stream));
  if (x0) CK(cudaMemcpyAsync(ctx->d_hx, x0, bytes, cudaMemcpyHostToDevice, ctx->stream));
  int rc = gmres_solve_device(ctx, ctx->d_hb, x0 ? ctx->d_hx : nullptr, ctx->d_hx, m, tol, ortho, precision, opts, res,
                              history, history_cap, history_len, nullptr);
  if (rc >= 0) {
    cudaError_t e = cudaMemcpyAsync(x_out, ctx->d_hx, bytes, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = fail(ctx, GMRES_ECUDA, cudaGetErrorString(e));
  }
  return rc;
}

int gmres_get_inner_history(gmres_ctx* ctx, double* buf, int32_t cap, int32_t* len) {
  if (!ctx) return fail(nullptr, GMRES_EINVAL, "ctx is NULL");
  const int n = (int)ctx->inner_host.size();
  if (buf) std::memcpy(buf, ctx->inner_host.data(), sizeof(double) * std::min(n, std::max(cap, 0)));
  if (len) *len = n;
  return 0;
}

int gmres_get_cycle_iters(gmres_ctx* ctx, int32_t* buf, int32_t cap, int32_t* len) {
  if (!ctx) return fail(nullptr, GMRES_EINVAL, "ctx is NULL");
  const int n = (int)ctx->cycJ_host.size();
  if (buf) std::memcpy(buf, ctx->cycJ_host.data(), sizeof(int32_t) * std::min(n, std::max(cap, 0)));
  if (len) *len = n;
  return 0;
}

int gmres_get_basis(gmres_ctx* ctx, int32_t col0, int32_t ncols, void* d_dst, int64_t ld) {
  if (!ctx || !d_dst || ctx->last_prec < 0) return fail(ctx, GMRES_EINVAL, "no solve yet / null argument");
  if (col0 < 0 || ncols < 1 || col0 + ncols > ctx->last_m + 1 || ld < ctx->n)
    return fail(ctx, GMRES_EINVAL, "columns outside [0, m] or ld < n");
  const VLayout& vl = ctx->last_vl;
  if (ctx->last_prec == GMRES_MIXED)
    unpack_basis_kernel<float><<<ctx->sms * 4, 256, 0, ctx->stream>>>((const float*)ctx->d_V, ctx->ldv, vl.tb, vl.lg,
                                                                     vl.tp, vl.bs, col0, ncols, ctx->n, (float*)d_dst, ld);
  else
    unpack_basis_kernel<double><<<ctx->sms * 4, 256, 0, ctx->stream>>>((const double*)ctx->d_V, ctx->ldv, vl.tb, vl.lg,
                                                                      vl.tp, vl.bs, col0, ncols, ctx->n, (double*)d_dst,
                                                                      ld);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int gmres_get_plan(gmres_ctx* ctx, int32_t* buf, int32_t cap) {
  if (!ctx || !buf) return fail(ctx, GMRES_EINVAL, "null argument");
  const int k = std::min(cap, (int32_t)GMRES_PLAN_N);
  std::copy(ctx->plan, ctx->plan + k, buf);
  return k;
}

int gmres_get_phase_ns(gmres_ctx* ctx, double* buf, int32_t cap) {
  if (!ctx || !buf) return fail(ctx, GMRES_EINVAL, "null argument");
  const int k = std::min(cap, (int)PH_N);
  for (int i = 0; i < k; ++i) buf[i] = ctx->phase_ns[i];
  return k;
}

// ------------------------------------------------------------ components
int gmres_k_cast32(gmres_ctx* ctx) {
  if (!ctx) return fail(nullptr, GMRES_EINVAL, "ctx is NULL");
  return ensure_a32(ctx, ctx->stream);
}

namespace {
// common prologue of the component entry points: kernels, grid, partition, workspace
int comp_setup(gmres_ctx* ctx, int prec, int m_req, int kind, int L, const void** kern, int* G, size_t* smem,
               int* m_ws, int align = ROWALIGN) {
  if (int rc = check_prec(ctx, prec)) return rc;
  if (ctx->dist()) return fail(ctx, GMRES_EINVAL, "component entry points take a single-rank context");
  if (prec == GMRES_MIXED)
    if (int rc = ensure_a32(ctx, ctx->stream)) return rc;
  const int m = (ctx->ws_m > 0 && ctx->ws_prec == prec) ? std::max(m_req, ctx->ws_m) : m_req;
  *m_ws = m;
  *smem = smem_bytes(m);
  const void* sk = pick_solve(prec, L);
  if (int rc = grid_for(ctx, sk, *smem, 0, G)) return rc;  // same grid as the solve
  *kern = pick_kernel(prec, kind, L);
  int Gk = 0;
  if (int rc = grid_for(ctx, *kern, *smem, 0, &Gk)) return rc;
  if (Gk < *G) *G = Gk;
  if (int rc = ensure_partition(ctx, *G, align)) return rc;
  if (int rc = ensure_ws(ctx, m, prec, std::max(*G, ctx->ws_G), std::max(ctx->hist_cap, 4), ctx->inner_cap))
    return rc;
  return reset_flags(ctx, ctx->stream);
}
// pack the caller's column-major V into the workspace V in row-blocked layout
int pack_blocked(gmres_ctx* ctx, int prec, const void* d_V, int64_t ldv, int ncols, const VLayout& vl) {
  ctx->ws_v_tb = -1;  // the workspace V now holds packed data: clear it before the next solve
  const long long nvalid = std::min<long long>(ldv, ctx->n);
  if (prec == GMRES_MIXED)
    pack_vblocked_kernel<float><<<ctx->sms * 4, 256, 0, ctx->stream>>>((const float*)d_V, ldv, ncols, ctx->nvec, nvalid,
                                                                     (float*)ctx->d_V, vl.tb, vl.tp, vl.bs);
  else
    pack_vblocked_kernel<double><<<ctx->sms * 4, 256, 0, ctx->stream>>>((const double*)d_V, ldv, ncols, ctx->nvec,
                                                                      nvalid, (double*)ctx->d_V, vl.tb, vl.tp, vl.bs);
  CK(cudaGetLastError());
  return 0;
}

}  // namespace

int gmres_k_spmv(gmres_ctx* ctx, int32_t precision, const void* d_v, void* d_w) {
  if (!ctx || !d_v || !d_w) return fail(ctx, GMRES_EINVAL, "null argument");
  const int L = auto_lanes(ctx->n, ctx->nnz);
  const void* kern;
  int G;
  size_t smem;
  int mws;
  if (int rc = comp_setup(ctx, precision, 1, 0, L, &kern, &G, &smem, &mws)) return rc;
  Dev d = make_dev(ctx, mws, precision, 0, G);
  void* args[] = {&d, (void*)&d_v, &d_w};
  if (int rc = launch_coop(ctx, kern, G, smem, args, ctx->stream)) return rc;
  CK(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int gmres_k_resid(gmres_ctx* ctx, int32_t precision, const double* d_b, const double* d_x, void* d_r, double* out2) {
  if (!ctx || !d_b || !d_x || !d_r || !out2) return fail(ctx, GMRES_EINVAL, "null argument");
  const int L = auto_lanes(ctx->n, ctx->nnz);
  const void* kern;
  int G;
  size_t smem;
  int mws;
  if (int rc = comp_setup(ctx, precision, 1, 1, L, &kern, &G, &smem, &mws)) return rc;
  Dev d = make_dev(ctx, mws, precision, 0, G);
  d.b = d_b;
  d.x = const_cast<double*>(d_x);
  double* d_out2 = nullptr;
  CK(cudaMalloc(&d_out2, sizeof(double) * 2));
  void* args[] = {&d, &d_r, &d_out2};
  int rc = launch_coop(ctx, kern, G, smem, args, ctx->stream);
  if (rc == 0) {
    cudaError_t e = cudaMemcpyAsync(out2, d_out2, sizeof(double) * 2, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = fail(ctx, GMRES_ECUDA, cudaGetErrorString(e));
  }
  int fl[2] = {0, 0};
  cudaMemcpy(fl, ctx->d_flags, sizeof(fl), cudaMemcpyDeviceToHost);
  cudaFree(d_out2);
  if (rc == 0 && fl[0]) rc = fail(ctx, GMRES_ETIMEOUT, "device watchdog fired");
  if (rc == 0 && (fl[1] & ERRF_NONFINITE)) rc = fail(ctx, GMRES_ENONFINITE, "non-finite residual");
  if (rc == 0 && (fl[1] & ERRF_RANGE)) rc = fail(ctx, GMRES_EFP32RANGE, "residual entry outside the fp32 range");
  return rc;
}

int gmres_k_ortho_ex(gmres_ctx* ctx, int32_t precision, int32_t ortho, int32_t j, const void* d_V, int64_t ldv,
                     void* d_w, double* h_out, int32_t mgs_variant, int32_t* variant_used) {
  if (!ctx || !d_V || !d_w || !h_out) return fail(ctx, GMRES_EINVAL, "null argument");
  if (j < 1 || ldv < ctx->ldv || ldv % LDALIGN) return fail(ctx, GMRES_EINVAL, "need j >= 1, ldv >= round_up(n,256), ldv % 64 == 0");
  if (ortho != GMRES_MGS && ortho != GMRES_CGSR) return fail(ctx, GMRES_EINVAL, "bad ortho");
  if (mgs_variant < -1 || mgs_variant > 3) return fail(ctx, GMRES_EINVAL, "mgs_variant must be -1, 0, 1, 2 or 3");
  const int L = auto_lanes(ctx->n, ctx->nnz);
  const void* kern;
  int G;
  size_t smem;
  int m;
  if (int rc = comp_setup(ctx, precision, j, 2, L, &kern, &G, &smem, &m)) return rc;
  const size_t wb = precision == GMRES_MIXED ? 4 : 8;
  // CGSR runs on the row-blocked V of a CGSR solve: pack the caller's V
  const VLayout vl = vlayout_for(ortho, m, (int)wb, tile_bytes_for(m));
  if (vl.tb) {
    if (int rc = ensure_partition(ctx, G, vl.tb)) return rc;
    if (int rc = pack_blocked(ctx, precision, d_V, ldv, j, vl)) return rc;
  }
  // the work vector lives in the padded workspace buffer (zero padding rows)
  CK(cudaMemsetAsync(ctx->d_w0, 0, wb * ctx->ldv, ctx->stream));
  CK(cudaMemcpyAsync(ctx->d_w0, d_w, wb * ctx->n, cudaMemcpyDeviceToDevice, ctx->stream));
  Dev d = make_dev(ctx, m, precision, ortho, G);
  set_vlayout(d, vl);
  if (vl.tb) d_V = ctx->d_V;
  if (precision == GMRES_MIXED && ortho == GMRES_MGS && ctx->d_fx) {
    // the mixed solve's fixed-point projections (reading R27), with the bound taken from
    // this call's w (the callers pass orthonormal bases, ‖v_i‖ ≤ 1): B = 2^⌈log2(2‖w‖)⌉
    std::vector<float> hw((size_t)ctx->n);
    CK(cudaMemcpy(hw.data(), d_w, sizeof(float) * ctx->n, cudaMemcpyDeviceToHost));
    double ss = 0.0;
    for (float v : hw) ss += (double)v * (double)v;
    const double bnd = 2.0 * std::sqrt(ss);
    if (bnd > 0.0 && std::isfinite(bnd)) {
      set_fx(d, (int)std::ceil(std::log2(bnd)), ctx->d_fx);
      CK(cudaMemsetAsync(ctx->d_fx, 0, 1024, ctx->stream));
    }
  }
  int used = -1;
  if (ortho == GMRES_MGS) {  // the MGS variant the solve would run (or the one requested)
    MgsPlan mp;
    if (int rc = plan_mgs(ctx, precision, m, G, TILE_BYTES, mgs_variant, 0, true, 0,
                          [&](int v) -> const void* { return pick_kernel(precision, v == 2 ? 6 : v == 3 ? 7 : 2, L); },
                          mp))
      return rc;
    kern = mp.kern;
    d.mgs_resident = mp.variant;
    d.mgs_nbuf = mp.nbuf;
    d.mgs_wsm = mp.wsm;
    d.tile_bytes = mp.tile_bytes;
    set_smem_offsets(d);
    smem = smem_bytes(m, mp.tile_bytes);
    used = mp.variant;
  }
  if (variant_used) *variant_used = used;
  double* d_h = nullptr;
  CK(cudaMalloc(&d_h, sizeof(double) * (j + 1)));
  long long ld = ldv;
  void* wp = ctx->d_w0;
  void* args[] = {&d, &j, (void*)&d_V, &ld, &wp, &d_h};
  int rc = launch_coop(ctx, kern, G, smem, args, ctx->stream);
  if (rc == 0) {
    cudaError_t e = cudaMemcpyAsync(d_w, ctx->d_w0, wb * ctx->n, cudaMemcpyDeviceToDevice, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_out, d_h, sizeof(double) * (j + 1), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = fail(ctx, GMRES_ECUDA, cudaGetErrorString(e));
  }
  cudaFree(d_h);
  int fl[2] = {0, 0};
  cudaMemcpy(fl, ctx->d_flags, sizeof(int) * 2, cudaMemcpyDeviceToHost);
  if (rc == 0 && fl[0]) rc = fail(ctx, GMRES_ETIMEOUT, "device watchdog fired");
  if (rc == 0 && fl[1]) rc = fail(ctx, GMRES_ENONFINITE, "a projection partial exceeded its fixed-point bound (non-finite data)");
  return rc;
}

int gmres_k_ortho(gmres_ctx* ctx, int32_t precision, int32_t ortho, int32_t j, const void* d_V, int64_t ldv,
                  void* d_w, double* h_out) {
  return gmres_k_ortho_ex(ctx, precision, ortho, j, d_V, ldv, d_w, h_out, -1, nullptr);
}

int gmres_k_xupdate(gmres_ctx* ctx, int32_t precision, int32_t J, const void* d_V, int64_t ldv, const double* y,
                    double* d_x, int32_t blocked) {
  if (!ctx || !d_V || !y || !d_x) return fail(ctx, GMRES_EINVAL, "null argument");
  if (J < 1 || ldv < ctx->ldv || ldv % LDALIGN) return fail(ctx, GMRES_EINVAL, "need J >= 1, ldv >= round_up(n,256), ldv % 64 == 0");
  const int L = auto_lanes(ctx->n, ctx->nnz);
  const void* kern;
  int G;
  size_t smem;
  int mws;
  if (int rc = comp_setup(ctx, precision, J, 3, L, &kern, &G, &smem, &mws)) return rc;
  const VLayout vl = blocked ? vlayout_for(GMRES_CGSR, mws, precision == GMRES_MIXED ? 4 : 8, tile_bytes_for(mws))
                             : VLayout{};
  if (vl.tb) {
    if (int rc = ensure_partition(ctx, G, vl.tb)) return rc;
    if (int rc = pack_blocked(ctx, precision, d_V, ldv, J, vl)) return rc;
    d_V = ctx->d_V;
  }
  Dev d = make_dev(ctx, mws, precision, 0, G);
  set_vlayout(d, vl);
  d.x = d_x;
  double* d_y = nullptr;
  CK(cudaMalloc(&d_y, sizeof(double) * J));
  CK(cudaMemcpy(d_y, y, sizeof(double) * J, cudaMemcpyHostToDevice));
  long long ld = ldv;
  void* args[] = {&d, &J, (void*)&d_V, &ld, &d_y};
  cudaError_t e = cudaLaunchCooperativeKernel(kern, dim3(G), dim3(NT), args, smem, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  cudaFree(d_y);
  if (e != cudaSuccess) return fail(ctx, GMRES_ECUDA, cudaGetErrorString(e));
  return 0;
}

int gmres_k_hessenberg(gmres_ctx* ctx, int32_t m, int32_t J, const double* Hbar, double beta, double* R, double* s,
                       double* y) {
  if (!Hbar || !R || !s || !y) return fail(ctx, GMRES_EINVAL, "null argument");
  if (m < 1 || J < 1 || J > m) return fail(ctx, GMRES_EINVAL, "need 1 <= J <= m");
  double *dH, *dR, *ds, *dy;
  const size_t hb = sizeof(double) * (m + 1) * m;
  CK(cudaMalloc(&dH, hb));
  CK(cudaMalloc(&dR, hb));
  CK(cudaMalloc(&ds, sizeof(double) * (m + 1)));
  CK(cudaMalloc(&dy, sizeof(double) * m));
  CK(cudaMemcpy(dH, Hbar, hb, cudaMemcpyHostToDevice));
  CK(cudaMemset(dR, 0, hb));
  const size_t smem = sizeof(double) * (6 * (m + 2));
  k_hess_kernel<<<1, NT, smem>>>(m, J, dH, beta, dR, ds, dy);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(R, dR, hb, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(s, ds, sizeof(double) * (J + 1), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(y, dy, sizeof(double) * J, cudaMemcpyDeviceToHost);
  cudaFree(dH); cudaFree(dR); cudaFree(ds); cudaFree(dy);
  if (e != cudaSuccess) return fail(ctx, GMRES_ECUDA, cudaGetErrorString(e));
  return 0;
}

}  // extern "C"

int gmres_ilu0_factor(gmres_ctx* ctx, int32_t precision, void* d_f) {
  if (!ctx) return fail(nullptr, GMRES_EINVAL, "ctx is NULL");
  if (int rc = check_prec(ctx, precision)) return rc;
  if (ctx->dist()) return fail(ctx, GMRES_EINVAL, "ILU(0) needs a single-rank context");
  if (precision == GMRES_MIXED)
    if (int rc = ensure_a32(ctx, ctx->stream)) return rc;
  if (int rc = ilu_factor(ctx, precision, ctx->stream)) return rc;
  if (d_f)
    CK(cudaMemcpyAsync(d_f, ctx->d_ilu_f[precision], (precision == GMRES_MIXED ? 4 : 8) * ctx->nnz,
                       cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int gmres_k_ilu_apply(gmres_ctx* ctx, int32_t precision, const void* d_z, void* d_out, int32_t schedule) {
  if (!ctx || !d_z || !d_out) return fail(ctx, GMRES_EINVAL, "null argument");
  if (int rc = check_prec(ctx, precision)) return rc;
  if (!ctx->ilu_ready[precision]) return fail(ctx, GMRES_EINVAL, "no ILU(0) factors of this precision: call gmres_ilu0_factor");
  const void* kern;
  int G;
  size_t smem;
  int mws;
  if (int rc = comp_setup(ctx, precision, 1, 4, 1, &kern, &G, &smem, &mws)) return rc;
  Dev d = make_dev(ctx, mws, precision, 0, G);
  set_ilu_dev(ctx, d, precision);
  for (int t = 0; t < 2; ++t)
    CK(cudaMemsetAsync(ctx->d_ilu_pub[t], 0xff, sizeof(double) * ctx->n, ctx->stream));
  d.tune = schedule & 65536;
  void* args[] = {&d, (void*)&d_z, &d_out};
  if (int rc = launch_coop(ctx, kern, G, smem, args, ctx->stream)) return rc;
  CK(cudaStreamSynchronize(ctx->stream));
  int flags[2] = {0, 0};
  CK(cudaMemcpy(flags, ctx->d_flags, sizeof(int) * 2, cudaMemcpyDeviceToHost));
  if (flags[0]) return fail(ctx, GMRES_ETIMEOUT, "grid barrier watchdog fired");
  return 0;
}

int gmres_ilu0_levels(gmres_ctx* ctx, int32_t* nlev_lower, int32_t* nlev_upper) {
  if (!ctx || !nlev_lower || !nlev_upper) return fail(ctx, GMRES_EINVAL, "null argument");
  if (int rc = ensure_ilu_plan(ctx)) return rc;
  *nlev_lower = ctx->ilu_nlev[0];
  *nlev_upper = ctx->ilu_nlev[1];
  return 0;
}
