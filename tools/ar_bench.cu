// Dev microbenchmark: grid all-reduce variants on a 148 x 512 cooperative grid.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ar_bench tools/ar_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>

constexpr int NT = 512, NW = 16;
constexpr unsigned long long SENT = 0x7ff4dead0badf00dull;

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t;
}
__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) {
  unsigned long long v; asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ unsigned long long ld_rlx(const void* p) {
  unsigned long long v; asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ unsigned long long ld_vol(const void* p) {
  unsigned long long v; asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void st_rel(void* p, double v) {
  asm volatile("st.release.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void st_rlx(void* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_rel(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_rlx(unsigned long long* p, unsigned long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

struct Args {
  int variant, iters, G, stride;  // stride: doubles between CTA slots (variant-dependent)
  unsigned long long* ctr;
  double* slots;  // [3][G*stride]
  double* parts;  // [2][G]
  unsigned long long* out;
};

__global__ void __launch_bounds__(NT, 1) kern(Args a) {
  __shared__ double red[NW], red2[NW];
  __shared__ unsigned long long epoch;
  __shared__ double cred[8], cres;
  __shared__ unsigned long long fxprev[2];
  __shared__ int stuckf;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = blockIdx.x, G = a.G;
  if (threadIdx.x == 0) { epoch = 0; fxprev[0] = fxprev[1] = 0; stuckf = 0; }
  __syncthreads();
  double acc_all = 0.0;
  int e3 = 0;
  const unsigned long long t0 = gtime();
  for (int it = 0; it < a.iters; ++it) {
    double v = (double)(g + 1) * 1e-3 + (it & 3);  // CTA sums < 2^12: inside the fixed-point variants' bound
    if (a.variant <= 2) {
      // counter barrier + load partials (old design); 0: red.release+ld.acquire, 1: relaxed red + fence, 2: barrier only
      v = warp_sum(v);
      if (lane == 0) red[warp] = v;
      __syncthreads();
      double* P = a.parts + (size_t)(it & 1) * G;
      if (threadIdx.x == 0) {
        double s = 0; for (int w = 0; w < NW; ++w) s += red[w];
        P[g] = s;
        const unsigned long long target = (epoch += 1) * (unsigned long long)G;
        if (a.variant == 1) { __threadfence(); red_rlx(a.ctr, 1); while (ld_vol(a.ctr) < target) {} __threadfence(); }
        else { red_rel(a.ctr, 1); while (ld_acq(a.ctr) < target) {} }
      }
      __syncthreads();
      if (a.variant != 2) {
        double x = 0.0;
        if (threadIdx.x < G) x = __ldcg(P + threadIdx.x);
        if (warp < (G + 31) / 32) { x = warp_sum(x); if (lane == 0) red2[warp] = x; }
        __syncthreads();
        double s = 0; for (int w = 0; w < (G + 31) / 32; ++w) s += red2[w];
        acc_all += s;
      }
    } else if (a.variant == 8 || a.variant == 9) {
      // as 7 but the arrival carries its data: red.relaxed (8: CTA 0 alone releases, for
      // its zeroing of the word two epochs ahead; 9: all release), relaxed polling and
      // one acquire fence after the poll succeeds
      v = warp_sum(v);
      if (lane == 0) red[warp] = v;
      __syncthreads();
      if (warp == 1) {
        double s = lane < NW ? red[lane] : 0.0;
        for (int o = NW / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) {
          unsigned long long* w = a.ctr + (size_t)(e3 & 3) * 32;
          long long q = llrint(ldexp(s, 43 - 12));
          const unsigned long long add = (1ull << 53) + (unsigned long long)(q + (1ll << 44));
          if (a.variant == 9 || g == 0) red_rel(w, add); else red_rlx(w, add);
          unsigned long long x;
          while (((x = ld_rlx(w)) >> 53) < (unsigned long long)G) {}
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          const long long sum = (long long)(x & ((1ull << 53) - 1)) - (long long)G * (1ll << 44);
          red2[0] = ldexp((double)sum, 12 - 43);
          if (g == 0) st_rlx(a.ctr + (size_t)((e3 + 2) & 3) * 32, 0ull);
        }
      }
      __syncthreads();
      acc_all += red2[0];
      e3 = e3 + 1;
    } else if (a.variant >= 60 && a.variant <= 62) {
      // as 8 without the zeroing: two alternating words that only ever grow (mod 2^64);
      // each CTA keeps the word's previous full value and reads count and sum from the
      // difference — no store, no release and (60, 61) no fence: the next add of a CTA
      // depends on its poll's result.  61/62: power-of-two multiplies instead of ldexp.
      v = warp_sum(v);
      if (lane == 0) red[warp] = v;
      __syncthreads();
      if (warp == 1) {
        double s = lane < NW ? red[lane] : 0.0;
        for (int o = NW / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) {
          unsigned long long* w = a.ctr + (size_t)(e3 & 1) * 32;
          const unsigned long long prev = fxprev[e3 & 1];
          long long q = a.variant == 60 ? llrint(ldexp(s, 43 - 12)) : __double2ll_rn(s * 2147483648.0);
          const unsigned long long add = (1ull << 53) + (unsigned long long)(q + (1ll << 44));
          red_rlx(w, add);
          unsigned long long x;
          unsigned spin = 0;
          while ((((x = ld_rlx(w)) - prev) >> 53) < (unsigned long long)G) {
            if ((++spin & 0xfffffu) == 0u) {  // stuck (≈ 1 s): report and release everybody
              if (spin >= 0x1000000u || ld_rlx(a.ctr + 512)) {
                if (!atomicExch(a.ctr + 512, 1ull))
                  printf("stuck: cta %d it %d word %d x %llx prev %llx other %llx\n", g, it, e3 & 1, x, prev,
                         ld_rlx(a.ctr + (size_t)((e3 + 1) & 1) * 32));
                stuckf = 1;
                break;
              }
            }
          }
          if (a.variant == 62) asm volatile("fence.acq_rel.gpu;" ::: "memory");
          fxprev[e3 & 1] = x;
          const long long sum = (long long)((x - prev) & ((1ull << 53) - 1)) - (long long)G * (1ll << 44);
          red2[0] = a.variant == 60 ? ldexp((double)sum, 12 - 43) : (double)sum * (1.0 / 2147483648.0);
        }
      }
      __syncthreads();
      if (stuckf) break;
      acc_all += red2[0];
      e3 = e3 + 1;
    } else if (a.variant == 7) {
      // single-word fixed-point all-reduce: count in bits 53..63, offset-binary 43-bit
      // quantised partials below (sum exact, order-independent); 4 rotating words,
      // CTA 0 zeroes the word two epochs ahead; one round trip after the last arrival
      v = warp_sum(v);
      if (lane == 0) red[warp] = v;
      __syncthreads();
      if (warp == 1) {
        double s = lane < NW ? red[lane] : 0.0;
        for (int o = NW / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) {
          unsigned long long* w = a.ctr + (size_t)(e3 & 3) * 32;
          long long q = llrint(ldexp(s, 43 - 12));
          const unsigned long long add = (1ull << 53) + (unsigned long long)(q + (1ll << 44));
          red_rel(w, add);
          unsigned long long x;
          while (((x = ld_acq(w)) >> 53) < (unsigned long long)G) {}
          const long long sum = (long long)(x & ((1ull << 53) - 1)) - (long long)G * (1ll << 44);
          red2[0] = ldexp((double)sum, 12 - 43);
          if (g == 0) st_rlx(a.ctr + (size_t)((e3 + 2) & 3) * 32, 0ull);
        }
      }
      __syncthreads();
      acc_all += red2[0];
      e3 = e3 + 1;
    } else if (a.variant >= 40) {
      // cluster pre-reduction (C = variant mod 10 CTAs per cluster): CTA sums → DSMEM
      // store into the leader's shared slot → cluster barrier → the leader pushes the
      // cluster partial and arrives (G/C arrivals).  40+C: every CTA polls the counter
      // and loads the G/C partials; 50+C: only the leaders do, then broadcast the
      // result over DSMEM (second cluster barrier)
      const int C = a.variant % 10;
      const bool bcast = a.variant >= 50;
      unsigned crank, cid;
      asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
      asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
      v = warp_sum(v);
      if (lane == 0) red[warp] = v;
      __syncthreads();
      if (threadIdx.x == 0) {
        double s = 0; for (int w = 0; w < NW; ++w) s += red[w];
        const unsigned loc = (unsigned)__cvta_generic_to_shared(&cred[crank]);
        unsigned rem;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rem) : "r"(loc), "r"(0));
        asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(rem), "d"(s) : "memory");
      }
      asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
      const int GC = G / C;
      double* P = a.parts + (size_t)(it & 1) * G;
      const bool poll = !bcast || crank == 0;
      if (warp == 0 && lane == 0) {
        if (crank == 0) {
          double s = 0; for (int r = 0; r < C; ++r) s += cred[r];
          P[cid] = s;
          red_rel(a.ctr, 1);
        }
        epoch += 1;
        if (poll) { const unsigned long long target = epoch * (unsigned long long)GC; while (ld_acq(a.ctr) < target) {} }
      }
      __syncthreads();
      double s = 0.0;
      if (poll) {
        double x = threadIdx.x < GC ? __ldcg(P + threadIdx.x) : 0.0;
        if (warp < (GC + 31) / 32) { x = warp_sum(x); if (lane == 0) red2[warp] = x; }
        __syncthreads();
        for (int w = 0; w < (GC + 31) / 32; ++w) s += red2[w];
      }
      if (bcast) {
        if (crank == 0 && threadIdx.x < C) {
          const unsigned loc = (unsigned)__cvta_generic_to_shared(&cres);
          unsigned rem;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rem) : "r"(loc), "r"(threadIdx.x));
          asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(rem), "d"(s) : "memory");
        }
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        s = cres;
      }
      acc_all += s;
    } else if (a.variant >= 10) {
      // counter + partial load with the arrivals spread over NC = variant-10 counters
      // (256 B apart: different L2 slices); warp 0 lane c polls counter c
      const int NC = a.variant - 10;
      v = warp_sum(v);
      if (lane == 0) red[warp] = v;
      __syncthreads();
      double* P = a.parts + (size_t)(it & 1) * G;
      if (warp == 0) {
        if (lane == 0) {
          double s = 0; for (int w = 0; w < NW; ++w) s += red[w];
          P[g] = s;
          red_rel(a.ctr + (size_t)(g % NC) * 32, 1);
        }
        epoch += (lane == 0);
        const unsigned long long ep = __shfl_sync(0xffffffffu, epoch, 0);
        // counter c receives the arrivals of CTAs g ≡ c (mod NC)
        const unsigned long long want = lane < NC ? ep * (unsigned long long)((G - lane + NC - 1) / NC) : 0ull;
        bool done = false;
        while (!done) {
          const unsigned long long cv = lane < NC ? ld_acq(a.ctr + (size_t)lane * 32) : 0ull;
          done = __all_sync(0xffffffffu, cv >= want);
        }
      }
      __syncthreads();
      double x = 0.0;
      if (threadIdx.x < G) x = __ldcg(P + threadIdx.x);
      if (warp < (G + 31) / 32) { x = warp_sum(x); if (lane == 0) red2[warp] = x; }
      __syncthreads();
      double s = 0; for (int w = 0; w < (G + 31) / 32; ++w) s += red2[w];
      acc_all += s;
    } else {
      // sentinel slots: 3: st.release push, relaxed poll, slot stride a.stride (doubles)
      //                 4: st.relaxed push
      //                 5: like 3 + acquire fence per polling warp
      //                 6: like 3 but only warp 0 polls with each lane covering G/32 slots
      v = warp_sum(v);
      if (lane == 0) red[warp] = v;
      __syncthreads();
      double* S = a.slots + (size_t)e3 * G * a.stride;
      if (threadIdx.x == 0) {
        double s = 0; for (int w = 0; w < NW; ++w) s += red[w];
        if (a.variant == 4) st_rlx(S + (size_t)g * a.stride, __double_as_longlong(s));
        else st_rel(S + (size_t)g * a.stride, s);
      }
      double x = 0.0;
      if (a.variant == 6) {
        if (warp == 0) {
          for (int t = lane; t < G; t += 32) {
            unsigned long long u;
            while ((u = ld_rlx(S + (size_t)t * a.stride)) == SENT) {}
            x += __longlong_as_double(u);
          }
        }
      } else if (threadIdx.x < G) {
        unsigned long long u;
        while ((u = ld_rlx(S + (size_t)threadIdx.x * a.stride)) == SENT) {}
        x = __longlong_as_double(u);
      }
      if (a.variant == 5 && threadIdx.x < G) __threadfence();
      const int nwp = a.variant == 6 ? 1 : (G + 31) / 32;
      if (warp < nwp) { x = warp_sum(x); if (lane == 0) red2[warp] = x; }
      __syncthreads();
      double s = 0; for (int w = 0; w < nwp; ++w) s += red2[w];
      acc_all += s;
      // reset own slot of buffer (e3+2)%3 (written at the previous epoch)
      if (threadIdx.x == 0) st_rlx(a.slots + ((size_t)((e3 + 2) % 3) * G + g) * a.stride, SENT);
      e3 = (e3 + 1) % 3;
    }
  }
  const unsigned long long t1 = gtime();
  if (g == 0 && threadIdx.x == 0) { a.out[0] = t1 - t0; a.out[1] = __double_as_longlong(acc_all); }
}

__global__ void fill(unsigned long long* p, size_t n, unsigned long long v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;  // run one variant only
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int G = sms, iters = 2000;
  unsigned long long *ctr, *out; double *slots, *parts;
  cudaMalloc(&ctr, 8 * 32 * 32); cudaMalloc(&out, 16);
  const int maxstride = 32;
  cudaMalloc(&slots, sizeof(double) * 3 * G * maxstride);
  cudaMalloc(&parts, sizeof(double) * 2 * G);
  struct V { int v, stride; const char* name; } vs[] = {
    {0, 1, "counter red.release/ld.acquire + partial load"},
    {1, 1, "counter fence+red.relaxed/volatile + partial load"},
    {2, 1, "counter barrier only"},
    {3, 1, "slots release push, relaxed poll, stride 8B"},
    {3, 4, "slots release push, relaxed poll, stride 32B"},
    {3, 32, "slots release push, relaxed poll, stride 256B"},
    {4, 1, "slots relaxed push, stride 8B"},
    {4, 32, "slots relaxed push, stride 256B"},
    {5, 1, "slots release push + acquire fence, stride 8B"},
    {6, 1, "slots release push, warp-0 poll, stride 8B"},
    {6, 32, "slots release push, warp-0 poll, stride 256B"},
    {7, 1, "fixed-point single word (count + sum), one round trip"},
    {8, 1, "fixed-point word, relaxed arrivals (CTA 0 releases), relaxed poll + fence"},
    {9, 1, "fixed-point word, release arrivals, relaxed poll + fence"},
    {60, 1, "fixed-point 2 growing words, all relaxed, no fence"},
    {61, 1, "same, power-of-two multiplies instead of ldexp"},
    {62, 1, "same as 61 + acquire fence after the poll"},
    {11, 1, "counter x1 (warp-0 poll) + partial load"},
    {12, 1, "counters x2 + partial load"},
    {14, 1, "counters x4 + partial load"},
    {18, 1, "counters x8 + partial load"},
    {26, 1, "counters x16 + partial load"},
    {42, 1, "cluster 2 pre-reduction, all CTAs poll + load"},
    {44, 1, "cluster 4 pre-reduction, all CTAs poll + load"},
    {52, 1, "cluster 2 pre-reduction, leader polls, DSMEM broadcast"},
    {54, 1, "cluster 4 pre-reduction, leader polls, DSMEM broadcast"},
  };
  for (auto& v : vs) {
    if (only >= 0 && v.v != only) continue;
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(ctr, 0, 8 * 32 * 32);
      fill<<<64, 256>>>((unsigned long long*)slots, (size_t)3 * G * maxstride, SENT);
      Args a{v.v, iters, G, v.stride, ctr, slots, parts, out};
      void* args[] = {&a};
      cudaError_t e;
      if (v.v >= 40 && v.v < 60) {  // cooperative launch in clusters of C
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(G); cfg.blockDim = dim3(NT);
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = v.v % 10; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeCooperative; at[1].val.cooperative = 1;
        cfg.attrs = at; cfg.numAttrs = 2;
        int ncl = 0;
        cudaOccupancyMaxActiveClusters(&ncl, (void*)kern, &cfg);
        if (rep == 0) printf("  (max active clusters of %d: %d, need %d)\n", v.v % 10, ncl, G / (v.v % 10));
        if (ncl * (v.v % 10) < G) { printf("%-55s cannot co-schedule %d CTAs\n", v.name, G); break; }
        e = cudaLaunchKernelEx(&cfg, kern, a);
      } else {
        e = cudaLaunchCooperativeKernel((void*)kern, dim3(G), dim3(NT), args, 0, 0);
      }
      if (e != cudaSuccess) { printf("launch: %s\n", cudaGetErrorString(e)); return 1; }
      e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("run: %s\n", cudaGetErrorString(e)); return 1; }
      unsigned long long h[2]; cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
      if (rep == 1) { printf("%-55s %7.3f us/op  (check %.6e)\n", v.name, h[0] / 1e3 / iters, __builtin_bit_cast(double, h[1])); fflush(stdout); }
    }
  }
  return 0;
}
