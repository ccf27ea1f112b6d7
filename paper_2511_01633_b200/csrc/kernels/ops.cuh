// Elementwise / memory-bound kernels of the decoder + the paged KV pool (K2, K4).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace glmx {

// Page geometry of the device KV pool: page = [layer][K|V][kv_head][B][head_dim] bf16.
struct PoolGeom {
  __nv_bfloat16* base;
  uint32_t n_layers, n_kv_heads, block_tokens, head_dim;
  __host__ __device__ uint64_t page_elems() const {
    return static_cast<uint64_t>(n_layers) * 2 * n_kv_heads * block_tokens * head_dim;
  }
  // first element of the (page, layer, kv, head) 2D tile [B][head_dim]
  __host__ __device__ uint64_t tile_off(int64_t page, uint32_t layer, uint32_t kv,
                                        uint32_t head) const {
    return static_cast<uint64_t>(page) * page_elems() +
           ((static_cast<uint64_t>(layer) * 2 + kv) * n_kv_heads + head) *
               static_cast<uint64_t>(block_tokens) * head_dim;
  }
};

void init_normal_bf16(__nv_bfloat16* p, uint64_t n, uint64_t seed, float std, cudaStream_t s);
void init_const_bf16(__nv_bfloat16* p, uint64_t n, float v, cudaStream_t s);

void embed_gather(const int32_t* tokens, int T, const __nv_bfloat16* embed, int d, float* x,
                  cudaStream_t s);
// out[t] = bf16(x[t] * rsqrt(mean(x^2) + eps) * w)   (x fp32 residual stream)
void rmsnorm(const float* x, const int32_t* rows, int T, int d, const __nv_bfloat16* w,
             float eps, __nv_bfloat16* out, cudaStream_t s);
// RoPE table of a forward: out[t][i] = (cos, sin)(float(pos[t]) * inv_freq[i]), i < half; shared
// by every layer's K2 append and the fused decode attention.
void rope_table(const int32_t* pos, int T, int half, const float* inv_freq, float2* out,
                cudaStream_t s);
// K2 append fused with RoPE: qkv [T][(H+2Hkv)*hd] -> q_out [T][H][hd] (roped), K (roped) and V
// into the pool pages given by slot[t] = page * B + offset.  head_dim 128 reads the angles from
// rope_cs (rope_table); other head dims compute them from pos / inv_freq.
void rope_kv_append(const __nv_bfloat16* qkv, const int32_t* pos, const int64_t* slot, int T,
                    int H, int Hkv, int hd, const float* inv_freq, const float2* rope_cs,
                    const PoolGeom& pool, uint32_t layer, __nv_bfloat16* q_out, cudaStream_t s);
void swiglu(const __nv_bfloat16* gu, int T, int ff, __nv_bfloat16* out, cudaStream_t s);
// dst[i] = src[idx[i]] (decode: first tokens into decode row order)
void gather_i32(const int32_t* src, const int32_t* idx, int n, int32_t* dst, cudaStream_t s);
// dst[i] = idx[i] < na ? a[idx[i]] : b[idx[i] - na] (a merged decode's two first-token sets)
void gather2_i32(const int32_t* a, int na, const int32_t* b, const int32_t* idx, int n, int32_t* dst,
                 cudaStream_t s);
// keys: n x 8 bytes of device scratch (split over CTAs), or nullptr (one CTA per row)
void argmax_rows(const float* logits, int n, int V, int32_t* out, void* keys, cudaStream_t s);
// K4: copy whole pages (all layers) pool_src[src[i]] -> pool_dst[dst[i]]; peer pointers allowed.
void pool_copy_pages(const __nv_bfloat16* src_base, __nv_bfloat16* dst_base, uint64_t page_elems,
                     const int32_t* src_pages, const int32_t* dst_pages, int n, cudaStream_t s);
// K2 gather (kernels/gather.cu): one layer's K or V of a page list into a dense
// [n*B][Hkv][hd] buffer, TMA-staged (bulk load of each 4 KB (page, head) tile, 2-D TMA store)
void kv_gather_tma(const PoolGeom& pool, uint32_t layer, uint32_t kv, const int32_t* pages, int n,
                   __nv_bfloat16* out, cudaStream_t s);
// scalar reference version (kept for A/B)
void kv_gather(const PoolGeom& pool, uint32_t layer, uint32_t kv, const int32_t* pages, int n,
               __nv_bfloat16* out, cudaStream_t s);

}  // namespace glmx
