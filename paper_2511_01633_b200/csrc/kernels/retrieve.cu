// K5 — RetrieveNode's exact nearest scan (index.cpp:41-56) over the device-resident index.
//
// Scores are bit-identical to the reference's dot kernels (dot.hpp:9-13, dot_scalar.cpp): eight
// lanes, lane j accumulating a[i+j]*b[i+j] over i = 0, 8, 16, ... with separately rounded
// products (-ffp-contract=off there, __fmul_rn/__fadd_rn here), then the fixed tree
// ((l0+l4)+(l2+l6)) + ((l1+l5)+(l3+l7)).  One thread scores one index row against a block of
// queries held in shared memory; the top-1 per query is a 64-bit key (orderable score, ~row)
// reduced by two warp REDUX steps and one atomicMax per warp, so ties go to the lowest row
// (= ascending id, the reference's tie-break) whatever the launch order.  HBM-bound: the index
// (n x 64 fp32) is streamed once per block of up to 32 queries.
#include "common.cuh"
#include "retrieve.cuh"

namespace glmx {

namespace {

constexpr int kQB = 32;  // queries per pass

__device__ __forceinline__ uint32_t orderable(float f) {
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ uint64_t pack2(float lo, float hi) {
  return static_cast<uint64_t>(__float_as_uint(lo)) | (static_cast<uint64_t>(__float_as_uint(hi)) << 32);
}

template <int DPAD, bool kPacked>
__global__ void __launch_bounds__(256)
nearest_kernel(const float* __restrict__ emb, int n_rows, const float* __restrict__ queries, int n_q,
               unsigned long long* __restrict__ best) {
  __shared__ float sq[kQB * DPAD];
  const int q0 = blockIdx.y * kQB;
  const int nq = min(kQB, n_q - q0);
  for (int i = threadIdx.x; i < nq * DPAD; i += blockDim.x) sq[i] = queries[q0 * DPAD + i];
  __syncthreads();
  unsigned long long bk[kQB];
#pragma unroll
  for (int q = 0; q < kQB; ++q) bk[q] = 0ull;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += gridDim.x * blockDim.x) {
    float row[DPAD];
    const float4* src = reinterpret_cast<const float4*>(emb + static_cast<int64_t>(r) * DPAD);
#pragma unroll
    for (int i = 0; i < DPAD / 4; ++i) {
      const float4 v = __ldg(src + i);
      row[4 * i] = v.x;
      row[4 * i + 1] = v.y;
      row[4 * i + 2] = v.z;
      row[4 * i + 3] = v.w;
    }
#pragma unroll
    for (int q = 0; q < kQB; ++q) {
      if (q >= nq) break;
      float l[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if constexpr (kPacked) {
        // the 8 lanes of dot.hpp as 4 packed fp32 pairs: mul.rn.f32x2 / add.rn.f32x2 round every
        // element exactly like __fmul_rn / __fadd_rn (no FMA contraction), two per instruction
        const float2* b2 = reinterpret_cast<const float2*>(sq + q * DPAD);
        uint64_t l2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
        for (int i = 0; i < DPAD; i += 8)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 bb = b2[i / 2 + j];
            const uint64_t x = pack2(row[i + 2 * j], row[i + 2 * j + 1]);
            const uint64_t y = pack2(bb.x, bb.y);
            uint64_t m;
            asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(m) : "l"(x), "l"(y));
            asm("add.rn.f32x2 %0, %1, %2;" : "=l"(l2[j]) : "l"(l2[j]), "l"(m));
          }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          l[2 * j] = __uint_as_float(static_cast<uint32_t>(l2[j]));
          l[2 * j + 1] = __uint_as_float(static_cast<uint32_t>(l2[j] >> 32));
        }
      } else {
        const float* b = sq + q * DPAD;
#pragma unroll
        for (int i = 0; i < DPAD; i += 8)
#pragma unroll
          for (int j = 0; j < 8; ++j) l[j] = __fadd_rn(l[j], __fmul_rn(row[i + j], b[i + j]));
      }
      const float even = __fadd_rn(__fadd_rn(l[0], l[4]), __fadd_rn(l[2], l[6]));
      const float odd = __fadd_rn(__fadd_rn(l[1], l[5]), __fadd_rn(l[3], l[7]));
      const float score = __fadd_rn(even, odd);
      const unsigned long long key =
          (static_cast<unsigned long long>(orderable(score)) << 32) | (0xFFFFFFFFu - static_cast<uint32_t>(r));
      bk[q] = key > bk[q] ? key : bk[q];
    }
  }
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < kQB; ++q) {
    if (q >= nq) break;
    const uint32_t hi = __reduce_max_sync(0xffffffffu, static_cast<uint32_t>(bk[q] >> 32));
    const uint32_t lo = __reduce_max_sync(
        0xffffffffu, static_cast<uint32_t>(bk[q] >> 32) == hi ? static_cast<uint32_t>(bk[q]) : 0u);
    if (lane == 0 && (hi | lo))
      atomicMax(best + q0 + q, (static_cast<unsigned long long>(hi) << 32) | lo);
  }
}

}  // namespace

void nearest_top1(const float* emb, int n_rows, int dpad, const float* queries, int n_q,
                  unsigned long long* best, cudaStream_t s, bool packed) {
  if (n_q <= 0 || n_rows <= 0) return;
  const int blocks_x = static_cast<int>(std::min<uint64_t>(ceil_div(n_rows, 256), kNumSMs * 2));
  dim3 grid(blocks_x, static_cast<unsigned>(ceil_div(n_q, kQB)));
  switch (dpad) {
    case 64:
      if (packed) nearest_kernel<64, true><<<grid, 256, 0, s>>>(emb, n_rows, queries, n_q, best);
      else nearest_kernel<64, false><<<grid, 256, 0, s>>>(emb, n_rows, queries, n_q, best);
      break;
    case 32:
      if (packed) nearest_kernel<32, true><<<grid, 256, 0, s>>>(emb, n_rows, queries, n_q, best);
      else nearest_kernel<32, false><<<grid, 256, 0, s>>>(emb, n_rows, queries, n_q, best);
      break;
    case 128:
      if (packed) nearest_kernel<128, true><<<grid, 256, 0, s>>>(emb, n_rows, queries, n_q, best);
      else nearest_kernel<128, false><<<grid, 256, 0, s>>>(emb, n_rows, queries, n_q, best);
      break;
    default: throw Error(GLMX_ERR_ARG, "embedding dim must pad to 32, 64 or 128");
  }
  GLMX_CHECK_LAUNCH();
}

}  // namespace glmx
