// Dev microbenchmark: per-SM streaming bandwidth of cp.async.bulk (TMA bulk copies)
// global→shared vs plain 16-byte loads, 148 CTAs x 512 threads, each CTA streams
// its own contiguous 64 MB / 148 slice.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_bench tools/tma_bench.cu
#include <cuda_runtime.h>
#include <cstdio>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void expect_tx(unsigned long long* b, unsigned n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, unsigned n, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
               "l"(src), "r"(n), "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ bool try_wait(unsigned long long* b, unsigned par) {
  unsigned ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
               : "=r"(ok) : "r"(smem_u32(b)), "r"(par) : "memory");
  return ok;
}

// mode 0: TMA, stage = S bytes split into `pieces` copies issued by `issuers` lanes of warp 0; R stages
// mode 1: plain LDG.128 by all threads, 8 in flight each
__global__ void __launch_bounds__(512, 1) kern(const char* src, size_t per_cta, int mode, int S, int pieces, int R,
                                               float* sink) {
  extern __shared__ __align__(128) char sm[];
  __shared__ unsigned long long bar[8];
  const char* base = src + per_cta * blockIdx.x;
  float acc = 0.f;
  if (mode == 0) {
    if (threadIdx.x == 0) { for (int r = 0; r < R; ++r) mbar_init(&bar[r], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    const int nst = (int)(per_cta / S);
    const unsigned piece = S / pieces;
    auto issue = [&](int k) {
      const int r = k % R;
      if ((threadIdx.x & 31) == 0) expect_tx(&bar[r], S);
      __syncwarp();
      for (int p = threadIdx.x; p < pieces; p += 32) bulk(sm + (size_t)r * S + p * piece, base + (size_t)k * S + p * piece, piece, &bar[r]);
    };
    if (threadIdx.x < 32) for (int k = 0; k < R - 1 && k < nst; ++k) issue(k);
    unsigned ph = 0;
    for (int k = 0; k < nst; ++k) {
      const int r = k % R;
      if (threadIdx.x < 32 && k + R - 1 < nst) issue(k + R - 1);
      while (!try_wait(&bar[r], (ph >> r) & 1)) {}
      ph ^= 1u << r;
      acc += reinterpret_cast<const float*>(sm + (size_t)r * S)[threadIdx.x];
      __syncthreads();
    }
  } else {
    const float4* p = reinterpret_cast<const float4*>(base);
    const size_t nv = per_cta / 16;
    for (size_t i = threadIdx.x; i < nv; i += 512 * 8) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = i + u * 512 < nv ? __ldcs(p + i + u * 512) : make_float4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u].x;
    }
  }
  if (acc == 1234.5f) sink[0] = acc;
}

int main() {
  int G; cudaDeviceGetAttribute(&G, cudaDevAttrMultiProcessorCount, 0);
  const size_t total = (size_t)1 << 31;  // 2 GB
  const size_t per = (total / G) & ~(size_t)65535;
  char* src; float* sink;
  cudaMalloc(&src, per * G); cudaMalloc(&sink, 4);
  cudaMemset(src, 1, per * G);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct C { int mode, S, pieces, R; } cs[] = {
    {1, 0, 0, 0},
    {0, 16384, 1, 2}, {0, 16384, 1, 4}, {0, 32768, 1, 2}, {0, 32768, 1, 4}, {0, 49152, 1, 3},
    {0, 32768, 8, 4}, {0, 32768, 16, 4}, {0, 32768, 32, 4}, {0, 65536, 32, 3}, {0, 65536, 16, 2},
    {0, 4096, 1, 8}, {0, 8192, 1, 8}, {0, 8192, 1, 16}, {0, 8192, 1, 24}, {0, 16384, 1, 8}, {0, 86016, 21, 2},
  };
  for (auto& c : cs) {
    float best = 1e9;
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(e0);
      kern<<<G, 512, c.mode == 0 ? (size_t)c.S * c.R : 0>>>(src, per, c.mode, c.S, c.pieces, c.R, sink);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    cudaError_t e = cudaGetLastError();
    printf("mode=%d stage=%6d pieces=%2d ring=%d : %7.0f GB/s %s\n", c.mode, c.S, c.pieces, c.R, per * G / best / 1e6,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
