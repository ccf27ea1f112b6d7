// tcgen05.mma issue/execute rate microbenchmark (diagnostics for K3 design; not product code).
// One CTA per SM; thread 0 issues `iters` MMAs of one shape back to back on resident smem tiles,
// commits, waits, and reports cycles per MMA.  Variants:
//   0: SS  M128 N128 K16, A,B K-major SW128        (K3's S = Q K^T)
//   1: TS  M128 N128 K16, A in TMEM, B MN-major     (K3's O += P V)
//   2: SS  M128 N256 K16
//   3: SS  M128 N64  K16
//   4: TS  M128 N64  K16, A in TMEM, B K-major      (S = Q K^T with Q in TMEM, 64-key tiles)
//   5: SS  M128 N128 K16, B MN-major
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)(lbo & 0x3FFF) << 16) | ((uint64_t)(sbo & 0x3FFF) << 32) |
         (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc(int n, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (b_mn ? (1u << 16) : 0u) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__global__ void __launch_bounds__(128, 1) bench(int variant, int iters, long long* out, int n_acc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tm;
  uint8_t* s = (uint8_t*)(((uintptr_t)smem + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) ((uint32_t*)s)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(&tm)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = tm;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_addr(s), b = smem_addr(s + 32768);
    const int n = (variant == 2) ? 256 : (variant == 3 || variant == 4) ? 64 : 128;
    const bool bmn = variant == 1 || variant == 5;
    const uint32_t id = idesc(n, bmn);
    uint64_t AD[8], BD[8];
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      AD[ks] = sdesc(a + (ks >> 2) * 16384 + (ks & 3) * 32, 1, 64);
      BD[ks] = bmn ? sdesc(b + ks * 2048, 16384 >> 4, 64) : sdesc(b + (ks >> 2) * 16384 + (ks & 3) * 32, 1, 64);
    }
    const uint32_t d0 = t + 256, d1 = (n == 256) ? t + 256 : t + 384;
    const bool ts = variant == 1 || variant == 4;
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 8) {
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const uint32_t d = (n_acc > 1 && (ks & 1)) ? d1 : d0;
        const uint32_t dd = (variant == 2) ? t : d;
        if (ts) {
          asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n"
                       ::"r"(dd), "r"(t + ks * 8), "l"(BD[ks]), "r"(id) : "memory");
        } else {
          asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n"
                       ::"r"(dd), "l"(AD[ks]), "l"(BD[ks]), "r"(id) : "memory");
        }
      }
    }
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(&bar)) : "memory");
    uint32_t ok = 0;
    while (!ok) {
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(smem_addr(&bar)) : "memory");
    }
    long long t2 = clock64();
    out[blockIdx.x * 2 + 0] = t1 - t0;
    out[blockIdx.x * 2 + 1] = t2 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 2 * sizeof(long long));
  long long h[296];
  const char* names[] = {"SS M128N128K16 Kmaj (S=QK^T)", "TS M128N128K16 B MN (PV)", "SS M128N256K16",
                         "SS M128N64K16", "TS M128N64K16 B Kmaj (Q in TMEM)", "SS M128N128K16 B MN"};
  const double flop[] = {2.0 * 128 * 128 * 16, 2.0 * 128 * 128 * 16, 2.0 * 128 * 256 * 16, 2.0 * 128 * 64 * 16,
                         2.0 * 128 * 64 * 16, 2.0 * 128 * 128 * 16};
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int v = 0; v < 6; ++v) {
   for (int n_acc : {1, 2}) {
    for (int grid : {148}) {
      const int iters = 4096;
      bench<<<grid, 128, 100 * 1024>>>(v, iters, d, n_acc);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("variant %d: %s\n", v, cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, d, grid * 2 * sizeof(long long), cudaMemcpyDeviceToHost);
      double issue = 0, total = 0;
      for (int b = 0; b < grid; ++b) { issue += h[2 * b]; total += h[2 * b + 1]; }
      issue /= grid; total /= grid;
      printf("acc %d %-36s grid %3d: issue %6.1f cyc/MMA, complete %6.1f cyc/MMA -> %6.0f flop/clk/SM (peak 8192)\n",
             n_acc, names[v], grid, issue / iters, total / iters, flop[v] * iters / total);
    }
   }
  }
  return 0;
}
