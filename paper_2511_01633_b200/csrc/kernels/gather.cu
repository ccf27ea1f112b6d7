// K2 gather — block-table-driven, TMA-staged KV gather out of the paged pool:
//   out[(i * B + tok) * Hkv * hd + h * hd + d] = pool[pages[i]][layer][kv][h][tok][d]
// i.e. one layer's K (or V) of a request's pages into a dense token-major [tokens][Hkv][hd] buffer
// (the layout torch / the fp32 oracle use).  Every (page, head) tile is a contiguous 4 KB
// [16 tok][128 dims] box: a 1-D bulk copy (cp.async.bulk) brings it into shared memory and a 2-D
// TMA store writes it as 16 rows of 256 B at stride Hkv * hd into the output; no thread touches
// the data.  One elected thread per CTA runs a kStages-deep ring with the stores kLag tiles
// behind the loads.  HBM-bound: 2 x 4 KB per tile (read + write).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "ops.cuh"

namespace glmx {

namespace {

constexpr int kStages = 8, kLag = 4;
constexpr int kTileBytes = 16 * 128 * 2;

__device__ __forceinline__ uint32_t saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(32)
kv_gather_tma_kernel(const __grid_constant__ CUtensorMap out_map, PoolGeom pool, uint32_t layer,
                     uint32_t kv, const int32_t* __restrict__ pages, int n_tiles) {
  __shared__ alignas(128) uint8_t buf[kStages][kTileBytes];
  __shared__ alignas(8) uint64_t bar[kStages];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kStages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int Hkv = static_cast<int>(pool.n_kv_heads);
  const int K = n_tiles > static_cast<int>(blockIdx.x) ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  for (int k = 0; k < K + kLag; ++k) {
    if (k < K) {
      const int t = blockIdx.x + k * gridDim.x;  // tile = (page index i, head h)
      const int i = t / Hkv, h = t % Hkv;
      const int s = k % kStages;
      if (k >= kStages)  // the store that last used this slot has finished reading it
        asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kStages - kLag - 1) : "memory");
      const __nv_bfloat16* src = pool.base + pool.tile_off(pages[i], layer, kv, h);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(&bar[s])), "n"(kTileBytes)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              saddr(buf[s])),
          "l"(src), "n"(kTileBytes), "r"(saddr(&bar[s]))
          : "memory");
    }
    if (k >= kLag) {
      const int kk = k - kLag;
      const int t = blockIdx.x + kk * gridDim.x;
      const int i = t / Hkv, h = t % Hkv;
      const int s = kk % kStages;
      const uint32_t parity = (kk / kStages) & 1;
      uint32_t ok = 0;
      while (!ok)
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(saddr(&bar[s])), "r"(parity)
            : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
              reinterpret_cast<uint64_t>(&out_map)),
          "r"(h * static_cast<int>(pool.head_dim)), "r"(i * static_cast<int>(pool.block_tokens)), "r"(saddr(buf[s]))
          : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

PFN_cuTensorMapEncodeTiled_v12000 encode_tiled() {
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

void kv_gather_tma(const PoolGeom& pool, uint32_t layer, uint32_t kv, const int32_t* pages, int n,
                   __nv_bfloat16* out, cudaStream_t s) {
  if (n <= 0) return;
  if (pool.head_dim != 128 || pool.block_tokens != 16)
    throw Error(GLMX_ERR_ARG, "the TMA gather is built for 16-token pages of head_dim 128");
  alignas(64) CUtensorMap map;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(pool.n_kv_heads) * pool.head_dim,
                        static_cast<cuuint64_t>(n) * pool.block_tokens};
  cuuint64_t strides[1] = {dims[0] * sizeof(__nv_bfloat16)};
  cuuint32_t box[2] = {pool.head_dim, pool.block_tokens};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_tiled()(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, out, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(GLMX_ERR_CUDA, "cuTensorMapEncodeTiled (gather) failed: " + std::to_string(r));
  const int tiles = n * static_cast<int>(pool.n_kv_heads);
  const int grid = std::min(tiles, kNumSMs * 16);
  kv_gather_tma_kernel<<<grid, 32, 0, s>>>(map, pool, layer, kv, pages, tiles);
  GLMX_CHECK_LAUNCH();
}

}  // namespace glmx
