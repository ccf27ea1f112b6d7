// Decode GEMMs on tcgen05: Y[n][N] (+)= X[n][K] . W[N][K]^T for n <= 64 token rows (the decode
// steps of the prefill/decode engine).  With a handful of rows the product is a weight stream:
// 2 bytes of W per 2 x n flops, HBM-bound.  cuBLAS picks tile shapes that stream W at 3.5-5.5
// TB/s for n = 64; this kernel swaps the operands so the weight rows fill the 128-row MMA tile:
//   D[128 out rows][64 tokens] (fp32, TMEM) += W_tile[128][64 k] . X_tile[64 tokens][64 k]^T
// per 64-wide K block, both operands TMA-loaded as 128-byte swizzled K-major tiles into a
// kStages-deep ring (warp 0), one elected thread issuing 4 MMAs per block (warp 1), 4 epilogue
// warps reading TMEM (thread = output feature, 64 token columns).  Grid (N / 128, splits): narrow
// matrices (QKV, O, down) split K so ~1-2 waves of CTAs stream at once; the partial tiles
// (fp32, L2-resident) are summed by the last-arriving CTA of each output tile (self-resetting
// per-tile counter), so there is no extra launch.  Output modes: bf16 store, fp32 store (logits),
// fp32 accumulate into the residual stream.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <atomic>

#include "common.cuh"
#include "gemv_tc.cuh"
#include "tc_ptx.cuh"

namespace glmx {

using namespace tcx;

namespace {

constexpr int kBM = 128;  // output features per tile (MMA M)
constexpr int kBN = 64;   // token rows (MMA N)
constexpr int kBK = 64;   // K per stage: 128-byte rows, 128B swizzle
constexpr int kStages = 4;
constexpr int kStageA = kBM * kBK * 2;  // 16 KB
constexpr int kStageB = kBN * kBK * 2;  // 8 KB
constexpr int kThreads = 192;           // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue
constexpr int kOffB = kStages * kStageA;
constexpr int kOffBar = kOffB + kStages * kStageB;
constexpr int kSmem = kOffBar + 256 + 1024;

// kind::f16 instruction descriptor: D f32, A/B bf16 K-major, M = 128, N = 64
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(kBN >> 3) << 17) |
                            (static_cast<uint32_t>(kBM >> 4) << 24);

struct GemvParams {
  int N, K, n;
  int kb_per_split, splits;
  int mode;  // 0 bf16 store, 1 fp32 store, 2 fp32 accumulate
  void* y;
  float* part;    // [splits][64][N]
  int* counters;  // [N / 128]
};

__device__ __forceinline__ void store_out(const GemvParams& p, int t, int o, float v) {
  if (p.mode == 0) {
    static_cast<__nv_bfloat16*>(p.y)[static_cast<int64_t>(t) * p.N + o] = __float2bfloat16_rn(v);
  } else if (p.mode == 1) {
    static_cast<float*>(p.y)[static_cast<int64_t>(t) * p.N + o] = v;
  } else {
    static_cast<float*>(p.y)[static_cast<int64_t>(t) * p.N + o] += v;
  }
}

__global__ void __launch_bounds__(kThreads, 2)
gemv_tc_kernel(const __grid_constant__ CUtensorMap w_map, const __grid_constant__ CUtensorMap x_map,
               GemvParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_addr(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  const uint32_t b_full = smem_addr(bars), b_empty = smem_addr(bars + kStages);
  const uint32_t b_done = smem_addr(bars + 2 * kStages);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 1);
  int* s_last = reinterpret_cast<int*>(bars + 2 * kStages + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x, split = blockIdx.y;
  const int kb0 = split * p.kb_per_split;
  const int nkb = min(p.K / kBK, kb0 + p.kb_per_split) - kb0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(b_full + 8 * s, 1);
      mbar_init(b_empty + 8 * s, 1);
    }
    mbar_init(b_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(
        smem_addr(tmem_holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int slot = i % kStages;
        if (i >= kStages) mbar_wait(b_empty + 8 * slot, ((i / kStages) - 1) & 1, 1);
        const uint32_t full = b_full + 8 * slot;
        mbar_expect_tx(full, kStageA + kStageB);
        const int kc = (kb0 + i) * kBK;
        tma_load_2d(sbase + slot * kStageA, &w_map, kc, tile * kBM, full);
        tma_load_2d(sbase + kOffB + slot * kStageB, &x_map, kc, 0, full);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int slot = i % kStages;
        mbar_wait(b_full + 8 * slot, (i / kStages) & 1, 2);
        tc_fence_after();
        const uint32_t a_addr = sbase + slot * kStageA, b_addr = sbase + kOffB + slot * kStageB;
#pragma unroll
        for (int ks = 0; ks < kBK / 16; ++ks) {
          const uint64_t a = smem_desc(a_addr + ks * 32, 1, 64);
          const uint64_t b = smem_desc(b_addr + ks * 32, 1, 64);
          tc_mma(tmem, a, b, kIdesc, (i > 0 || ks > 0) ? 1u : 0u);
        }
        tc_commit(b_empty + 8 * slot);
      }
      tc_commit(b_done);
    }
    __syncwarp();
  } else {
    // epilogue: TMEM lane quarter of this warp (warps 2..5 -> quarters 2, 3, 0, 1)
    const int q = warp & 3;
    const int o = tile * kBM + q * 32 + lane;  // output feature of this thread
    mbar_wait(b_done, 0, 3);
    tc_fence_after();
    uint32_t acc[64];
    const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16);
    TC_LD32(taddr, acc);
    TC_LD32(taddr + 32, (acc + 32));
    tc_wait_ld();
    // token loops fully unrolled (acc stays in registers), predicated on the live rows
    if (p.splits == 1) {
#pragma unroll
      for (int t = 0; t < kBN; ++t)
        if (t < p.n) store_out(p, t, o, __uint_as_float(acc[t]));
    } else {
      float* part = p.part + static_cast<int64_t>(split) * kBN * p.N;
#pragma unroll
      for (int t = 0; t < kBN; ++t)
        if (t < p.n) part[static_cast<int64_t>(t) * p.N + o] = __uint_as_float(acc[t]);
      __threadfence();
      asm volatile("bar.sync 1, 128;" ::: "memory");  // the 4 epilogue warps
      if (warp == 2 && lane == 0) {
        const int prev = atomicAdd(p.counters + tile, 1);
        *s_last = prev == p.splits - 1;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (*s_last) {
        // last CTA of this tile: sum the split partials (other CTAs' writes are visible after
        // their fence + counter increment), write the output, reset the counter
        __threadfence();
        // 16 token rows at a time: all splits' loads of a chunk issued before any store
#pragma unroll
        for (int t0 = 0; t0 < kBN; t0 += 16) {
          if (t0 >= p.n) break;
          float v[16];
#pragma unroll
          for (int tt = 0; tt < 16; ++tt) v[tt] = 0.f;
          for (int s = 0; s < p.splits; ++s) {
            const float* src = p.part + (static_cast<int64_t>(s) * kBN + t0) * p.N + o;
#pragma unroll
            for (int tt = 0; tt < 16; ++tt)
              if (t0 + tt < p.n) v[tt] += __ldcg(src + static_cast<int64_t>(tt) * p.N);
          }
#pragma unroll
          for (int tt = 0; tt < 16; ++tt)
            if (t0 + tt < p.n) store_out(p, t0 + tt, o, v[tt]);
        }
        if (warp == 2 && lane == 0) p.counters[tile] = 0;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    GLMX_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (!f || q != cudaDriverEntryPointSuccess) throw Error(GLMX_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

}  // namespace

// [rows][cols] bf16 row-major, box [box_rows][64 cols], 128B swizzle
void make_gemv_map(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows, void* out_map) {
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(reinterpret_cast<CUtensorMap*>(out_map), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                           const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(GLMX_ERR_CUDA, "cuTensorMapEncodeTiled (gemv) failed: " + std::to_string(r));
}

bool gemv_tc_supported(int n, int K, int N) {
  return n >= 1 && n <= kBN && K % kBK == 0 && N % kBM == 0;
}

int gemv_tc_splits(int K, int N) {
  const int tiles = N / kBM, kb = K / kBK;
  // ~1.3 waves of single-CTA SMs for narrow matrices, no split for wide ones
  int s = std::max(1, (2 * kNumSMs) / std::max(1, tiles));
  s = std::min(s, std::max(1, kb / 4));  // >= 4 K blocks per split
  const int per = (kb + s - 1) / s;
  return (kb + per - 1) / per;
}

void gemv_tc(const void* w_map, const void* x_map, int n, int K, int N, int mode, void* y,
             float* part, int* counters, cudaStream_t s) {
  if (n <= 0) return;
  if (!gemv_tc_supported(n, K, N)) throw Error(GLMX_ERR_ARG, "gemv_tc: unsupported shape");
  static std::atomic<bool> attr[64];
  int dev = 0;
  GLMX_CUDA(cudaGetDevice(&dev));
  if (!attr[dev & 63].load(std::memory_order_acquire)) {
    GLMX_CUDA(cudaFuncSetAttribute(gemv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    attr[dev & 63].store(true, std::memory_order_release);
  }
  const int kb = K / kBK;
  const int splits = gemv_tc_splits(K, N);
  GemvParams p{N, K, n, (kb + splits - 1) / splits, splits, mode, y, part, counters};
  gemv_tc_kernel<<<dim3(N / kBM, splits), kThreads, kSmem, s>>>(
      *reinterpret_cast<const CUtensorMap*>(w_map), *reinterpret_cast<const CUtensorMap*>(x_map), p);
  GLMX_CHECK_LAUNCH();
}

size_t gemv_tc_part_floats(int K, int N) { return static_cast<size_t>(gemv_tc_splits(K, N)) * kBN * N; }

}  // namespace glmx
