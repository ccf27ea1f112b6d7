// tcgen05.mma issue/execute rate: CTA-pair (cta_group::2, M = 256) against single-CTA shapes
// (diagnostics for the K3 design; not product code).  A cluster of two CTAs per SM pair; the
// leader's thread 0 issues `iters` MMAs of one shape back to back on resident smem tiles (each CTA
// holds its 128 rows of A and half of B at the same smem offsets), commits to both CTAs' barriers
// and reports cycles per MMA and flop/clk per SM.  Variants:
//   0: cg1 SS M128 N128 K16 (reference: K3's S = Q K^T today)
//   1: cg1 SS M128 N256 K16
//   2: cg1 TS M128 N256 K16  (A in TMEM)
//   3: cg2 SS M256 N128 K16  (B: 64 rows per CTA)
//   4: cg2 SS M256 N256 K16  (B: 128 rows per CTA)
//   5: cg2 TS M256 N128 K16, B MN-major (PV: A = P in TMEM of both CTAs, V split by dims)
//   6: cg2 TS M256 N256 K16, B K-major
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate_cg2 mma_rate_cg2.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)(lbo & 0x3FFF) << 16) | ((uint64_t)(sbo & 0x3FFF) << 32) |
         (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc(int m, int n, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (b_mn ? (1u << 16) : 0u) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <bool kCg2>
__global__ void __launch_bounds__(128, 1) bench(int variant, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tm;
  uint8_t* s = (uint8_t*)(((uintptr_t)smem + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) ((uint32_t*)s)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    if (kCg2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(&tm)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(&tm)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (kCg2) cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = tm;
  const bool leader = !kCg2 || cta_rank() == 0;
  if (threadIdx.x == 0 && leader) {
    const uint32_t a = smem_addr(s), b = smem_addr(s + 32768);
    int m = 128, n = 128;
    bool bmn = false, ts = false;
    switch (variant) {
      case 0: break;
      case 1: n = 256; break;
      case 2: n = 256; ts = true; break;
      case 3: m = 256; break;
      case 4: m = 256; n = 256; break;
      case 5: m = 256; ts = true; bmn = true; break;
      case 6: m = 256; n = 256; ts = true; break;
    }
    const uint32_t id = idesc(m, n, bmn);
    uint64_t AD[8], BD[8];
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      AD[ks] = sdesc(a + (ks >> 2) * 16384 + (ks & 3) * 32, 1, 64);
      BD[ks] = bmn ? sdesc(b + ks * 2048, 16384 >> 4, 64) : sdesc(b + (ks >> 2) * 16384 + (ks & 3) * 32, 1, 64);
    }
    const uint32_t d = t + 256;  // accumulator columns [256, 256 + n)
    const uint32_t dd = n == 256 ? t + 256 : d;
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 8) {
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const uint32_t dst = n == 256 ? (ts ? t + 256 : t) : dd;
        if (kCg2) {
          if (ts)
            asm volatile("tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, 1;\n" ::"r"(dst), "r"(t + ks * 8),
                         "l"(BD[ks]), "r"(id) : "memory");
          else
            asm volatile("tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, 1;\n" ::"r"(dst), "l"(AD[ks]),
                         "l"(BD[ks]), "r"(id) : "memory");
        } else {
          if (ts)
            asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n" ::"r"(dst), "r"(t + ks * 8),
                         "l"(BD[ks]), "r"(id) : "memory");
          else
            asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n" ::"r"(dst), "l"(AD[ks]),
                         "l"(BD[ks]), "r"(id) : "memory");
        }
      }
    }
    long long t1 = clock64();
    if (kCg2)
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              smem_addr(&bar)),
          "h"((uint16_t)3)
          : "memory");
    else
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(&bar))
                   : "memory");
    uint32_t ok = 0;
    while (!ok) {
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(ok)
                   : "r"(smem_addr(&bar))
                   : "memory");
    }
    long long t2 = clock64();
    out[blockIdx.x * 2 + 0] = t1 - t0;
    out[blockIdx.x * 2 + 1] = t2 - t0;
  } else if (threadIdx.x == 0) {
    // follower: wait for the leader's multicast commit before the TMEM is released
    uint32_t ok = 0;
    while (!ok) {
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(ok)
                   : "r"(smem_addr(&bar))
                   : "memory");
    }
    out[blockIdx.x * 2 + 0] = -1;
    out[blockIdx.x * 2 + 1] = -1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (kCg2) cluster_sync();
  if (threadIdx.x < 32) {
    if (kCg2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(t));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
  }
}

int main() {
  const int grid = 148;
  long long* d;
  cudaMalloc(&d, grid * 2 * sizeof(long long));
  long long h[2 * grid];
  const char* names[] = {"cg1 SS M128N128K16", "cg1 SS M128N256K16", "cg1 TS M128N256K16",
                         "cg2 SS M256N128K16", "cg2 SS M256N256K16", "cg2 TS M256N128K16 B MN (PV)",
                         "cg2 TS M256N256K16"};
  const int M[] = {128, 128, 128, 256, 256, 256, 256}, N[] = {128, 256, 256, 128, 256, 128, 256};
  cudaFuncSetAttribute(bench<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(bench<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int v = 0; v < 7; ++v) {
    const bool cg2 = v >= 3;
    const int iters = 4096;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = 100 * 1024;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cg2 ? 2 : 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cg2 ? cudaLaunchKernelEx(&cfg, bench<true>, v, iters, d)
                        : cudaLaunchKernelEx(&cfg, bench<false>, v, iters, d);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("variant %d (%s): %s\n", v, names[v], cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(h, d, grid * 2 * sizeof(long long), cudaMemcpyDeviceToHost);
    double issue = 0, total = 0;
    int nl = 0;
    for (int b = 0; b < grid; ++b)
      if (h[2 * b] >= 0) {
        issue += h[2 * b];
        total += h[2 * b + 1];
        ++nl;
      }
    issue /= nl;
    total /= nl;
    // flops per SM: an M256 MMA runs on two SMs
    const double flop_sm = 2.0 * M[v] * N[v] * 16 / (cg2 ? 2 : 1);
    printf("%-30s grid %3d: issue %6.1f cyc/MMA, complete %6.1f cyc/MMA -> %6.0f flop/clk/SM (peak 8192)\n",
           names[v], grid, issue / iters, total / iters, flop_sm * iters / total);
  }
  return 0;
}
