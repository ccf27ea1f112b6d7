// K1 vertex-chunk assembly: device graph view + launch wrappers (see chunk.cu).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace glmx {

struct DevGraph {
  const char* entry_bytes;
  const uint32_t* entry_off;
  const uint32_t* und_off;
  const int32_t* und_idx;
  const uint32_t* dir_off;
  const int32_t* dir_idx;
  const int32_t* w_total;
  const int32_t* w_by_type;
  const uint32_t* ent_stat;  // per entry: whitespace token count + edge flags (entry_stats)
  uint32_t n;
};

struct ChunkParams {
  int k;            // max(k, 0)
  int k_stride;     // row stride of the selection buffer (>= k)
  int weight_mode;  // 0 TotalDegree, 1 ByEdgeType
  int directed;
};

// select: warp path + CTA path for rows queued in big_list (n_req entries) / big_count (1 int);
// per chunk: the k selected neighbours, byte length and whitespace token count
void chunk_select(const DevGraph& g, const ChunkParams& p, const int32_t* node_idx, int n_req,
                  int32_t* sel, int32_t* sel_count, uint64_t* byte_len, uint32_t* tok_count,
                  int32_t* big_list, int32_t* big_count, cudaStream_t s);
// render + tokenize: chunk bytes at byte_off[r], token spans (relative to the chunk) + fnv1a ids
// at tok_off[r] (exclusive scans of the select outputs)
void chunk_render_emit(const DevGraph& g, const ChunkParams& p, const int32_t* node_idx, int n_req,
                       const int32_t* sel, const int32_t* sel_count, const uint64_t* byte_off,
                       const uint32_t* tok_off, uint32_t vocab, char* out, int32_t* tok_id,
                       uint64_t* tok_begin, uint64_t* tok_end, cudaStream_t s);
// per-entry whitespace stats (DevGraph::ent_stat), once at graph upload
void entry_stats(const char* bytes, const uint32_t* off, uint32_t n, uint32_t* st, cudaStream_t s);
size_t scan_u64_temp_bytes(int n);
size_t scan_u32_temp_bytes(uint64_t n);
void scan_u64(void* temp, size_t temp_bytes, const uint64_t* in, uint64_t* out, int n,
              cudaStream_t s);
void scan_u32(void* temp, size_t temp_bytes, const uint32_t* in, uint32_t* out, uint64_t n,
              cudaStream_t s);

}  // namespace glmx
