// K3 paged prefill attention (and 1-token decode through the same path).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "ops.cuh"

namespace glmx {

struct AttnParams {
  const __nv_bfloat16* q;  // [T][H][hd], RoPE applied
  __nv_bfloat16* o;        // [T][H][hd]
  PoolGeom pool;
  uint32_t layer;
  const int32_t* q_start;      // [n_req] first row of the request in q / o
  const int32_t* q_len;        // [n_req] computed tokens (suffix) of the request
  const int32_t* ctx_len;      // [n_req] keys visible to the last query (cached + q_len)
  const int32_t* block_table;  // [n_req][bt_stride] pages, key j lives in page j / B
  int bt_stride;
  const int2* work;  // (request, first query token) per CTA tile, longest first
  int n_work;
  int H, Hkv;
  float scale_log2;  // softmax scale * log2(e)
};

// tcgen05 / TMEM / TMA version (attn_tc.cu): 128 query rows per CTA.
int attn_tc_tokens_per_tile(int H, int Hkv);
void make_pool_tensor_map(const PoolGeom& g, uint64_t pages, void* out_map, uint32_t* rows_total);
void make_q_tensor_map(const void* q, uint64_t T, int H, int Hkv, void* out_map);
// Stream-K schedule on the device (host/attn_sched.hpp packed by the caller) + the partial
// workspace: part_o [2 * 148][256][128] fp32, part_ml [2 * 148][256] float2.
struct AttnTcSched {
  const int4* pieces;
  const int* cta_off;
  const int4* combine;
  int grid, n_combine;
  float* part_o;
  float2* part_ml;
  const int4* partners;  // nullptr: no paired pieces
};
int attn_tc_partial_rows();  // rows per partial slot (256)
// trace build only (-DGLMX_ATTN_TRACE): copy + clear CTA 0's pipeline stamps; -1 otherwise
int attn_trace_read(long long* out, int n);
// Persistent launch: sc.grid CTAs walk their pieces; then the combine pass for split items.
void paged_attention_tc(const AttnParams& p, const void* kv_map, uint32_t rows_total,
                        const void* q_map, const AttnTcSched& sc, cudaStream_t s);
}  // namespace glmx

namespace glmx {
// Decode rows (q_len == 1 for every request) on CUDA cores (attn_decode.cu): flash-decoding over
// the block table, n_split CTAs per (request, kv head); partials (n_split > 1) in part_o /
// part_ml ([item * n_split + split][4 heads] rows), merged by a combine kernel.
bool decode_attention_supported(const AttnParams& p);
int decode_attention_splits(int n_items, int max_ctx, int max_rows);
void paged_attention_decode(const AttnParams& p, int n_req, int n_split, float* part_o,
                            float2* part_ml, cudaStream_t s);
// Same, fused with K2 for the decode rows: q, k are RoPE'd from the qkv rows inside the kernel
// (k and v appended to the pool page at slot[row] by the CTA that owns the last key), so no
// separate rope_kv_append launch and no q buffer round trip.
struct DecodeRope {
  const __nv_bfloat16* qkv;  // [rows][(H + 2 Hkv) * hd]
  const int32_t* pos;        // [rows]
  const int64_t* slot;       // [rows] pool slot (page * B + offset) of the new key
  const float2* rope_cs;     // [rows][hd / 2] (cos, sin) of the forward (rope_table)
};
void paged_attention_decode_rope(const AttnParams& p, const DecodeRope& r, int n_req, int n_split,
                                 float* part_o, float2* part_ml, cudaStream_t s);
}  // namespace glmx
