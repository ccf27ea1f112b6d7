// K1 vertex-chunk assembly: device graph view + launch wrappers (see chunk.cu).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace glmx {

// Per-entry record for the per-piece loads of the tokenizer / render (one 32-byte line):
// entry bytes [off, off + len), first-token length (0 = irregular), last-token offset, interior
// tokens [ioff, ioff + ni), fnv1a state after the last token.
struct __align__(32) EntryRec {
  uint32_t off, len, head, tail, ioff, ni;
  uint64_t tstate;
};

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
  // Per-entry token tables (entry_tokens, at upload) for the fast tokenizer of regular entries
  // (non-empty, first and last byte non-space, >= 2 whitespace tokens): the interior tokens (all
  // but the first and the last) never touch a chunk junction, so their spans and fnv1a hashes are
  // precomputed; only the junction tokens (separator + the entry's first token, its last token +
  // separator) are hashed per chunk, the last token continuing from its precomputed fnv1a state.
  const uint32_t* ent_head;   // bytes of the first token; 0 = irregular entry (slow path)
  const uint32_t* ent_tail;   // offset of the last token
  const uint64_t* ent_tstate; // fnv1a state after the last token's bytes
  const uint32_t* ent_ioff;   // interior tokens of entry u: [ent_ioff[u], ent_ioff[u+1])
  const uint2* itok_span;     // {begin, end} relative to the entry
  const uint64_t* itok_hash;  // fnv1a of the token bytes
  const uint32_t* itok_id;    // hash mod the vocab of the batch (chunk_token_ids), or null
  const EntryRec* ent;        // packed per-entry view of the above (entry_records)
  uint32_t n;
};

// Neighbours of every node ranked by (weight desc, node index asc) for one (weight mode,
// directed) variant -- Retriever::node_info's order (retriever.cpp:97-113) -- plus exclusive
// prefix sums along the CSR order (rows are contiguous: a row's sums are differences):
//   pbytes: entry_len(u) + 3 ("(" E ")" and the "," before every piece but the first)
//   ptoks : piece_tokens(ent_stat[u]) (whitespace tokens the piece adds to a chunk)
//   pirr  : irregular entries (the byte-level tokenizer handles their chunks)
struct RankedAdj {
  const uint32_t* off;  // CSR row offsets (und_off or dir_off)
  const int32_t* idx;
  const EntryRec* recs;  // ent[idx[e]]: the ranked neighbours' records, contiguous per row
  const uint4* lens;     // per node for the batch's k: {bytes, tokens, k' | irregular << 31, row}
                         // (chunk_len_table), or null
  const uint64_t* pbytes;
  const uint32_t* ptoks;
  const uint32_t* pirr;
};

// The per-node chunk lengths for one k (chunk_len_scan reads them with one load per chunk)
void chunk_len_table(const DevGraph& g, const RankedAdj& ra, int k, uint4* out, cudaStream_t s);
// Decoupled look-back state of chunk_lengths_scan: per tile aggregate + inclusive prefix + a
// status word (epoch << 2 | 1 aggregate / 2 inclusive); sized chunk_scan_tiles(n)
struct ScanState {
  uint64_t* bytes;
  uint64_t* ibytes;
  uint32_t* toks;
  uint32_t* itoks;
  uint32_t* flag;
};
int chunk_scan_tiles(int n_req);
// per chunk: k' = min(k, deg) | irregular << 31, and the exclusive scans of byte lengths and
// whitespace token counts (byte_off / tok_off [0..n], [n] = totals) in one single-pass kernel;
// epoch: distinct per call on the same state (starts at 1; the state is zeroed once); the
// irregular chunks' indices are appended to irr_list (*irr_count zeroed by the caller); vrow[r] =
// (node, first entry of its ranked row) for the render kernels
void chunk_lengths_scan(const DevGraph& g, const RankedAdj& ra, int k, const int32_t* node_idx,
                        int n_req, int32_t* sel_count, uint64_t* byte_off, uint32_t* tok_off,
                        const ScanState& st, uint32_t epoch, int32_t* irr_list, int32_t* irr_count,
                        int2* vrow, cudaStream_t s);
// render + tokenize: chunk bytes at byte_off[r], token spans (relative to the chunk) + fnv1a ids
// at tok_off[r] (chunk_lengths_scan's outputs).  Output capacities (bytes, tokens)
// are checked on the device: a chunk that does not fit sets *overflow and is skipped, and the
// host grows the buffers and launches the render again (no host round trip before the render).
// Regular chunks: one kernel whose CTAs pair 4 text warps with 4 token warps (table-driven
// tokenizer); irregular chunks: a small grid over the list chunk_lengths_scan compacted (not
// launched when irr_list is null: the caller knows the graph has no irregular entries).
void chunk_render_emit(const DevGraph& g, const RankedAdj& ra, const int32_t* node_idx, int n_req,
                       const int32_t* sel_count, const uint64_t* byte_off, const uint32_t* tok_off,
                       uint32_t vocab, char* out, int32_t* tok_id, uint64_t* tok_begin,
                       uint64_t* tok_end, uint64_t bytes_cap, uint64_t tok_cap, int32_t* overflow,
                       const int32_t* irr_list, const int32_t* irr_count, const int2* vrow,
                       cudaStream_t s);
// ranked adjacency of one CSR (off[0..n], idx) under weights w: keys/sorted scratch of e_count
// u64, tmp32 of e_count + 1; outputs ridx[e_count], pbytes/ptoks/pirr[e_count + 1], recs[e_count]
// (g.ent must be built)
size_t rank_sort_temp_bytes(uint64_t e_count, uint32_t n);
void rank_adjacency(const DevGraph& g, const uint32_t* off, const int32_t* idx, const int32_t* w,
                    uint64_t e_count, uint32_t n, void* temp, size_t temp_bytes, uint64_t* keys,
                    uint64_t* sorted, int32_t* ridx, uint64_t* pbytes, uint32_t* ptoks,
                    uint32_t* pirr, uint32_t* tmp32, EntryRec* recs, cudaStream_t s);
// per-entry whitespace stats (DevGraph::ent_stat), once at graph upload
void entry_stats(const char* bytes, const uint32_t* off, uint32_t n, uint32_t* st, cudaStream_t s);
// per-entry interior-token counts (-> ent_ioff by an exclusive scan), then the token tables
void entry_interior_counts(const uint32_t* st, uint32_t n, uint32_t* cnt, cudaStream_t s);
void entry_tokens(const char* bytes, const uint32_t* off, const uint32_t* st, uint32_t n,
                  const uint32_t* ioff, uint32_t* head, uint32_t* tail, uint64_t* tstate,
                  uint2* itok_span, uint64_t* itok_hash, cudaStream_t s);
// the packed per-entry records (after entry_tokens)
void entry_records(const uint32_t* off, const uint32_t* head, const uint32_t* tail,
                   const uint64_t* tstate, const uint32_t* ioff, uint32_t n, EntryRec* rec,
                   cudaStream_t s);
// the interior tokens' ids for one vocab (fnv1a mod vocab), recomputed when the vocab changes
void chunk_token_ids(const uint64_t* hash, uint32_t n, uint32_t vocab, uint32_t* ids, cudaStream_t s);
size_t scan_u64_temp_bytes(int n);
size_t scan_u32_temp_bytes(uint64_t n);
void scan_u64(void* temp, size_t temp_bytes, const uint64_t* in, uint64_t* out, int n,
              cudaStream_t s);
void scan_u32(void* temp, size_t temp_bytes, const uint32_t* in, uint32_t* out, uint64_t n,
              cudaStream_t s);

}  // namespace glmx
