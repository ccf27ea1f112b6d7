/* glmx — B200-native prefill over a paged KV pool with vertex-chunk prefix reuse.
 *
 * C-ABI drop-in boundary for the hot path of the GLM reference (/root/reference/proj).  The
 * reference exposes C++ classes in a static library (no C ABI, no plugin registry); each entry
 * point below replaces one reference interface, cited as file:line.  Conventions:
 *   - plain pointers + sizes, caller-allocated outputs, no torch / STL types;
 *   - int status codes map 1:1 onto the reference's exception classes (error.hpp:29-137);
 *     glmx_last_error() returns the message (thread-local);
 *   - handles are NOT thread-safe: callers serialise calls on one handle exactly as the
 *     reference serialises KvCacheState under Orchestrator::kv_mutex_ (orchestrator.cpp:95,152);
 *   - one kv / model / engine handle per GPU.
 * Everything that computes runs on the GPU (sm_100a); there is no CPU fallback: compute entry
 * points on a handle created without a device return GLMX_ERR_NO_DEVICE.
 */
#ifndef GLMX_H
#define GLMX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status codes */
#define GLMX_OK 0
#define GLMX_ERR_GLM 1             /* GlmError, e.g. bad TierMap (cache.cpp:57-63)            */
#define GLMX_ERR_CACHE_EXHAUSTED 2 /* CacheExhausted (cache.cpp:122-124); partial state stays  */
#define GLMX_ERR_CONFIG 3          /* ConfigError (cache.cpp:28)                               */
#define GLMX_ERR_RETRIEVAL 4       /* RetrievalError wrapping UnknownNode (retriever.cpp:123)  */
#define GLMX_ERR_CUDA 5            /* CUDA / cuBLAS failure                                    */
#define GLMX_ERR_ARG 6             /* bad argument or caller buffer too small                  */
#define GLMX_ERR_NO_DEVICE 7       /* compute requested on a bookkeeping-only handle           */
#define GLMX_ERR_MALFORMED 8       /* MalformedRecord / DanglingEdge / DuplicateNode (graph)   */
#define GLMX_ERR_POOL 9            /* physical page pool (headroom) exhausted                  */

#define GLMX_POLICY_PRIORITY 0 /* CachePolicy::Priority (config.hpp:10) */
#define GLMX_POLICY_LRU 1      /* CachePolicy::PlainLru */
#define GLMX_TIER_I 0          /* Tier (tier.hpp:10) */
#define GLMX_TIER_II 1
#define GLMX_TIER_III 2
#define GLMX_TIER_IV 3

const char* glmx_last_error(void);
const char* glmx_version(void);
int glmx_device_count(void);

/* ================================================================== KV cache
 * KvCacheState (cache.hpp:56-99) semantics, bit-exact, over a device page pool.  One page per
 * cached block holds all layers: [layer][K|V][kv_head][block_tokens][head_dim] bf16. */
typedef struct glmx_kv glmx_kv;

typedef struct {
  uint64_t capacity_blocks; /* logical capacity == the reference's kv.capacity_blocks     */
  uint32_t block_tokens;    /* B (config.hpp:30); 0 -> GLMX_ERR_CONFIG as cache.cpp:28     */
  int32_t policy;           /* GLMX_POLICY_*                                               */
  int32_t device;           /* CUDA ordinal, or -1 for bookkeeping only (no pool)          */
  uint32_t n_layers;        /* pool page geometry; ignored when device < 0                 */
  uint32_t n_kv_heads;
  uint32_t head_dim;
  uint64_t headroom_pages; /* physical pages beyond capacity: tails, decode, deferred frees */
} glmx_kv_config;

typedef struct {
  uint64_t begin, end; /* token positions, end exclusive (cache.hpp:25-31) */
  int32_t tier;
  int32_t reserved;
} glmx_tier_range;

typedef struct {             /* PrefillReport (cache.hpp:33-39) */
  uint64_t cached_tokens;    /* reused along the maximal resident chain prefix */
  uint64_t computed_tokens;  /* full blocks computed by this call */
  uint64_t tail_tokens;      /* trailing partial block, never cached */
  uint64_t n_evicted;        /* ids written to `evicted` (in eviction order) */
  uint64_t n_blocks;         /* full blocks == entries written to `block_table` */
} glmx_prefill_report;

/* replaces KvCacheState::KvCacheState (cache.cpp:25-29) */
int glmx_kv_create(const glmx_kv_config* cfg, glmx_kv** out);
void glmx_kv_destroy(glmx_kv* kv);

/* replaces KvCacheState::prefill (cache.cpp:54-107).  Tokens cross as bytes because block ids
 * hash token bytes (cache.cpp:13-21): token i = tok_bytes[tok_offsets[i] .. tok_offsets[i+1]).
 * block_table[b] = physical page of full block b (hit, newly inserted, or orphan).  When the
 * evicted buffer is too small the true count is still reported and glmx_kv_last_evicted returns
 * the whole list. */
int glmx_kv_prefill(glmx_kv* kv, const char* tok_bytes, const uint64_t* tok_offsets,
                    uint64_t n_tok, const glmx_tier_range* tiers, uint64_t n_tiers,
                    const char* session, glmx_prefill_report* report, int32_t* block_table,
                    uint64_t block_table_cap, uint64_t* evicted, uint64_t evicted_cap);

/* replaces Orchestrator::kv_prefill (orchestrator.cpp:81-97): segments are tokenised separately
 * (tokenizer.hpp:14-25; tokens never fuse across segments), empty ones skipped, adjacent
 * same-tier ranges merged, then glmx_kv_prefill. */
int glmx_kv_prefill_segments(glmx_kv* kv, uint64_t n_seg, const char* const* seg_text,
                             const uint64_t* seg_len, const int32_t* seg_tier,
                             const char* session, glmx_prefill_report* report,
                             int32_t* block_table, uint64_t block_table_cap, uint64_t* evicted,
                             uint64_t evicted_cap);

uint64_t glmx_kv_last_evicted(const glmx_kv* kv, uint64_t* out, uint64_t cap);
/* replaces KvCacheState::evict (cache.cpp:109-148); *n_out = ids written */
int glmx_kv_evict(glmx_kv* kv, uint64_t n, uint64_t* out, uint64_t cap, uint64_t* n_out);
/* replaces KvCacheState::set_tier (cache.cpp:150-153) <- Orchestrator::finish (:147-154) */
int glmx_kv_set_tier(glmx_kv* kv, const char* session, int32_t from_tier, int32_t to_tier);
/* replaces KvCacheState::force_insert (cache.cpp:167-176) — test / trace-replay hook */
int glmx_kv_force_insert(glmx_kv* kv, uint64_t id, int32_t tier, uint64_t last_used,
                         const char* session);
/* CacheCounters (cache.hpp:41-49): hits, misses, evictions_by_tier[4] */
int glmx_kv_counters(const glmx_kv* kv, int64_t out6[6]);
/* resident_snapshot (cache.cpp:160-165), sorted by id; returns the resident count.  pages[i] is
 * the block's page in the device pool, or -1 (device pools) when the page holds no KV for it (stale: inserted
 * by a bookkeeping-only prefill, force_insert, or a batch that failed before its forward). */
uint64_t glmx_kv_resident(const glmx_kv* kv, uint64_t* ids, int32_t* tiers, uint64_t* last_used,
                          int32_t* pages, uint64_t cap);
/* CacheBlock::session of a resident block (cache.hpp:17-23); -1 when not resident */
/* KvCacheState::block (cache.hpp:80): 1 and the block's CacheBlock fields (cache.hpp:17-23) when
 * `id` is resident, else 0 (all out-params nullable) */
int32_t glmx_kv_block(const glmx_kv* kv, uint64_t id, int32_t* tier, uint64_t* last_used,
                      uint64_t* parent, int32_t* has_parent);
int64_t glmx_kv_block_session(const glmx_kv* kv, uint64_t id, char* buf, uint64_t cap);
/* snapshot_json (cache.cpp:178-189); returns the full length */
int64_t glmx_kv_snapshot_json(const glmx_kv* kv, char* buf, uint64_t cap);
/* KvCacheState::chain_ids (cache.cpp:31-40), static; returns the number of full blocks */
uint64_t glmx_kv_chain_ids(const char* tok_bytes, const uint64_t* tok_offsets, uint64_t n_tok,
                           uint32_t block_tokens, uint64_t* out);
/* Pages of blocks evicted since the last call become reusable.  Only safe once no enqueued
 * device work reads them (the engine calls this itself, stream-ordered). */
int glmx_kv_release_deferred(glmx_kv* kv);
/* Pipelined epochs (host work of rotation r+1 overlaps the forward of r): deferred pages are
 * numbered in eviction order; glmx_kv_defer_mark = how many were deferred so far, and
 * glmx_kv_release_deferred_before(mark) frees only those deferred before the mark. */
uint64_t glmx_kv_defer_mark(const glmx_kv* kv);
int glmx_kv_release_deferred_before(glmx_kv* kv, uint64_t mark);
uint64_t glmx_kv_pool_pages(const glmx_kv* kv);
uint64_t glmx_kv_free_pages(const glmx_kv* kv);
/* Device address of the pool (for tests / peer mapping); bytes per page. */
void* glmx_kv_pool_ptr(const glmx_kv* kv);
uint64_t glmx_kv_page_bytes(const glmx_kv* kv);

/* ---- cross-GPU prefix hits (one process and one pool per GPU) ----------------
 * Each rank exports its pool once (CUDA IPC) and, at every epoch (a rotation of the workload),
 * publishes the (block id, page) pairs of its residents; a rank's engine prefill then serves the
 * run of missed blocks that directly extends its local hit prefix from peer pools by K4 page
 * copies instead of recomputing them.  Bookkeeping is unchanged (those blocks are misses,
 * inserted locally with their tier/owner, exactly as G independent KvCacheStates would count
 * them); only the compute differs.  Epoch mode keeps evicted pages deferred until the caller's
 * epoch-end barrier (glmx_kv_release_deferred), so a page named in a directory stays intact for
 * the whole epoch. */
int glmx_kv_ipc_handle(const glmx_kv* kv, uint8_t out[64]);
int glmx_kv_attach_peer(glmx_kv* kv, int32_t peer, const uint8_t handle[64]);
/* same-process variant: another pool (possibly on another device) as peer `peer` */
int glmx_kv_attach_peer_local(glmx_kv* kv, int32_t peer, const glmx_kv* other);
/* (entries with page < 0 are skipped) */
int glmx_kv_set_peer_directory(glmx_kv* kv, uint64_t n, const uint64_t* block_ids,
                               const int32_t* peers, const int32_t* pages);
int glmx_kv_set_epoch_mode(glmx_kv* kv, int32_t on);
/* blocks served by peer copies since creation */
int64_t glmx_kv_peer_hits(const glmx_kv* kv);

/* whitespace tokenizer (tokenizer.hpp:14-25): writes begin/end byte spans, returns count */
uint64_t glmx_tokenize(const char* text, uint64_t len, uint64_t* begins, uint64_t* ends,
                       uint64_t cap);
/* builder-defined token id map: fnv1a(token bytes) mod vocab */
int32_t glmx_token_id(const char* tok, uint64_t len, uint32_t vocab);

/* ================================================================== graph + vertex chunks
 * PropertyGraph (graph_store.hpp:27-75) loaded into a device CSR; Retriever::node_info +
 * render_chunk (retriever.cpp:9-30, 74-129) as a batched GPU kernel (K1). */
typedef struct glmx_graph glmx_graph;

/* replaces PropertyGraph::load (graph_store.cpp:38-90) + build_indexes (:108-124) */
int glmx_graph_load_jsonl(const char* path, int32_t device, glmx_graph** out);
/* seeded power-law property graph (builder-defined synthetic input for C2/C5):
 * n_nodes items/users, ~edges_per_node out-edges per node, dst ~ u^3 skew, 2 edge types */
int glmx_graph_synth_powerlaw(uint64_t n_nodes, uint32_t edges_per_node, uint64_t seed,
                              int32_t device, glmx_graph** out);
int glmx_graph_save_jsonl(const glmx_graph* g, const char* path);
void glmx_graph_destroy(glmx_graph* g);
uint64_t glmx_graph_node_count(const glmx_graph* g);
uint64_t glmx_graph_edge_count(const glmx_graph* g);
/* node index in ascending-id order (graph_store.hpp:63 node_ids()), -1 if unknown */
int64_t glmx_graph_node_index(const glmx_graph* g, const char* id);
int64_t glmx_graph_node_id(const glmx_graph* g, uint64_t idx, char* buf, uint64_t cap);
int64_t glmx_graph_degree(const glmx_graph* g, uint64_t idx); /* total_degree (:209-213) */
/* Bytes the graph's K1 chunk builds and K5 RetrieveNode scans moved since load: out2[0]
 * host->device (node ids, query embeddings), out2[1] device->host (chunk bytes, offsets, token
 * ids / spans, nearest winners). */
int glmx_graph_io_bytes(const glmx_graph* g, uint64_t out2[2]);
/* PropertyGraph::node(id).attributes[key] (graph_store.hpp:27-75) in its canonical rendering
 * (render_attr_value, attr.hpp:38-48); kind (nullable): 0 string, 1 int, 2 double, 3 bool,
 * 4 list.  Returns the value's byte length, or -1 when the node has no such attribute. */
int64_t glmx_graph_node_attr(const glmx_graph* g, uint64_t idx, const char* key, char* buf,
                             uint64_t cap, int32_t* kind);

typedef struct {
  int32_t k;           /* chunk.k (config.hpp:20); negative -> 0 like max(k,0) */
  int32_t weight_mode; /* 0 TotalDegree, 1 ByEdgeType (config.hpp:21) */
  int32_t directed;    /* chunk.directed (config.hpp:22) */
  uint32_t vocab;      /* token-id space for out_tok_ids (0 -> ids not produced) */
} glmx_chunk_config;

/* K1: batched vertex-chunk assembly.  For each requested node: render_chunk(node_info(id)) bytes
 * into out_bytes[out_byte_offsets[i] ..), its whitespace tokens (spans relative to the chunk,
 * tokens fuse across entry boundaries exactly as text) and token ids.  Sizes: call once with
 * out_bytes == NULL to get *total_bytes / *total_tokens. */
int glmx_chunk_build(glmx_graph* g, const glmx_chunk_config* cfg, const int32_t* node_idx,
                     uint64_t n, char* out_bytes, uint64_t bytes_cap, uint64_t* out_byte_offsets,
                     int32_t* out_tok_ids, uint64_t* out_tok_begin, uint64_t* out_tok_end,
                     uint64_t tok_cap, uint64_t* out_tok_offsets, uint64_t* total_bytes,
                     uint64_t* total_tokens);
/* replaces Retriever::node_info_rendered (retriever.cpp:123-129); runs K1 for one node.
 * Returns the length, or -GLMX_ERR_RETRIEVAL for an unknown id. */
int64_t glmx_node_info_rendered(glmx_graph* g, const glmx_chunk_config* cfg, const char* id,
                                char* buf, uint64_t cap);
/* device time (ms) of the last K1 launch, measured with CUDA events on its stream */
/* RetrieveNode (Retriever::retrieve_node_traced, retriever.cpp:49-66 over VectorIndex,
 * index.hpp:22-41).  glmx_index_build embeds (embedder.cpp:19-36) the index text of every node —
 * its string "title", else string "name" (index.cpp:12-25, default Config) — into a device
 * resident [rows][dim] fp32 table and sizes the retrieval LRU (Config::retrieval_cache_capacity,
 * 1024 by default).  glmx_retrieve_nodes resolves n texts (bytes + n+1 offsets) in order: an LRU
 * hit returns the cached node, a miss runs the exact GPU nearest scan (K5: scores bit-identical to
 * dot.hpp's 8-lane tree, ties to the lowest id) and caches the result.  Out: graph node indices
 * and hit flags.  Empty index -> GLMX_ERR_RETRIEVAL (EmptyIndex). */
int glmx_index_build(glmx_graph* g, int32_t dim, uint64_t cache_capacity);
uint64_t glmx_index_size(const glmx_graph* g);
int glmx_retrieve_nodes(glmx_graph* g, const char* text_bytes, const uint64_t* text_offsets,
                        uint64_t n, int32_t* out_node_idx, uint8_t* out_cache_hit);
/* generate_workload(seed, n, nondet_ratio, graph, default Config) (workload.cpp:158-255) at
 * scale: the per-candidate "title retrieves its own node" validation runs as one batched K5 scan;
 * pools, mt19937_64 draws and the JSONL (Workload::serialize_jsonl) are the reference's.  Returns
 * the JSONL length (write up to cap bytes to buf), or -status (GLMX_ERR_GLM = GraphTooSmall,
 * GLMX_ERR_CONFIG = bad ratio).  out_scan_ms: device time of the validation scan. */
int64_t glmx_workload_generate(glmx_graph* g, uint64_t seed, int32_t n, double nondet_ratio,
                               char* buf, uint64_t cap, float* out_scan_ms);
/* {cache_hits, cache_misses, index_probes} since glmx_index_build (RetrievalStats) */
void glmx_retriever_stats(const glmx_graph* g, int64_t out3[3]);
float glmx_retrieve_last_kernel_ms(const glmx_graph* g);
/* embed(text, dim) on the host (embedder.cpp:19-36): writes (dim + 7) / 8 * 8 floats */
int glmx_embed_text(const char* text, uint64_t len, int32_t dim, float* out);
float glmx_chunk_last_kernel_ms(const glmx_graph* g);

/* ================================================================== model (random-init Llama) */
typedef struct glmx_model glmx_model;
typedef struct {
  uint32_t n_layers, d_model, n_heads, n_kv_heads, head_dim, d_ff, vocab;
  float rope_theta; /* 500000 for Llama-3 */
  float norm_eps;   /* 1e-5 */
  float init_std;   /* N(0, init_std) weights, seeded, bf16 */
  uint64_t seed;
} glmx_model_config;

int glmx_model_create(const glmx_model_config* cfg, int32_t device, glmx_model** out);
/* frees the weights; with engines still alive the release is deferred to the last engine's destroy */
void glmx_model_destroy(glmx_model* m);
/* test hook: copy one bf16 weight tensor to host (raw uint16 bits).  which: 0 embed [V,d],
 * 1 attn_norm [d], 2 wqkv [(H+2Hkv)*hd, d], 3 wo [d, H*hd], 4 mlp_norm [d], 5 w_gate_up
 * [2*ff, d], 6 w_down [d, ff], 7 final_norm [d], 8 lm_head [V, d] */
int glmx_model_export_weight(const glmx_model* m, int32_t which, int32_t layer, uint16_t* out,
                             uint64_t n);

/* Times cuBLAS's algorithm candidates for the four per-layer projections (QKV, O, gate/up,
 * down) at every M bucket up to max_tokens (128-row buckets to 2048, 256-row to 16384, 2048-row above) against the
 * default cublasGemmEx choice, on layer 0's weights, and records the winners; later forwards of
 * every engine on this model launch them.  Takes seconds and synchronises the device: call it
 * once at start-up, before any engine work is in flight.  No reference counterpart (the
 * reference's model step is a cost model, orchestrator.cpp:131-132); untuned models keep
 * cublasGemmEx.  *out_entries (nullable) = buckets with a recorded winner. */
int glmx_model_tune_gemms(glmx_model* m, int32_t max_tokens, int32_t* out_entries);

/* ================================================================== engine: prefill / decode step
 * The seam at orchestrator.cpp:131-132 (span = c_prefill*computed + c_decode*tokens_out) becomes
 * a real forward: bookkeeping prefill per request in caller order (sequential semantics, exactly
 * the reference's), then ONE batched, layer-synchronous forward (append-before-attention) of all
 * computed+tail tokens against the paged pool, greedy first token per request. */
typedef struct glmx_engine glmx_engine;
typedef struct {
  uint32_t max_requests;     /* per batch */
  uint32_t max_batch_tokens; /* computed+tail tokens per batch */
  uint32_t max_decode;       /* decode steps reserved per request */
  uint32_t max_context;      /* tokens per request (prompt + decode) */
} glmx_engine_config;

typedef struct {
  const char* tok_bytes;
  const uint64_t* tok_offsets; /* n_tok + 1 */
  uint64_t n_tok;
  const glmx_tier_range* tiers;
  uint64_t n_tiers;
  const char* session;
  /* nonzero: this call's reply is a Finish (known ahead for scripted replies), so the session's
   * Orchestrator::finish -- KvCacheState::set_tier(session, II, III), orchestrator.cpp:147-154 --
   * is applied right after this request's bookkeeping, before the next request's: the batch then
   * reproduces run_bench's exact round-robin call order (bench.cpp:65-83). */
  int32_t finish;
} glmx_request;

int glmx_engine_create(glmx_model* m, glmx_kv* kv, const glmx_engine_config* cfg,
                       glmx_engine** out);
void glmx_engine_destroy(glmx_engine* e);
/* One prefill step over n_req requests (host buffers).  reports[i] as glmx_kv_prefill;
 * first_token[i] = greedy argmax (first max index) of the last prompt position's logits.
 * logits (optional, host [n_req][vocab] fp32) for parity tests.  Returns the first bookkeeping
 * error (earlier requests' bookkeeping stays applied, like the reference; no forward runs). */
int glmx_engine_prefill(glmx_engine* e, uint64_t n_req, const glmx_request* reqs,
                        glmx_prefill_report* reports, int32_t* first_token, float* logits);
/* Same step with prompts given as (text, tier) segments — the Orchestrator::call_llm ->
 * kv_prefill path (orchestrator.cpp:81-97, 116-135): per-segment whitespace tokenisation,
 * same-tier range merge, then the prefill step above. */
typedef struct {
  const char* const* seg_text;
  const uint64_t* seg_len;
  const int32_t* seg_tier;
  uint64_t n_seg;
  const char* session;
  int32_t finish; /* as glmx_request::finish */
} glmx_segment_request;
int glmx_engine_prefill_segments(glmx_engine* e, uint64_t n_req,
                                 const glmx_segment_request* reqs, glmx_prefill_report* reports,
                                 int32_t* first_token, float* logits);
/* Asynchronous step: bookkeeping (reports, exactly as the synchronous call) and staging happen
 * now, the forward is enqueued on the engine stream, and the call returns without waiting, so a
 * caller can stage batch r+1 while batch r runs (at most two batches in flight).
 * glmx_engine_wait completes the OLDEST in-flight batch: writes its greedy first tokens
 * (first_token[cap], -1 for empty prompts) and publishes its timings/work; returns its request
 * count, or -status.  The synchronous entry points and decode wait for in-flight batches
 * first. */
int glmx_engine_prefill_segments_async(glmx_engine* e, uint64_t n_req,
                                       const glmx_segment_request* reqs,
                                       glmx_prefill_report* reports);
int glmx_engine_wait(glmx_engine* e, int32_t* first_token, uint64_t cap);
int32_t glmx_engine_in_flight(const glmx_engine* e);
/* Greedy decode continuing the last prefill batch: steps[i] tokens for request i (<= max_decode);
 * out_tokens host [n_req][max_steps], -1 past a request's count. */
int glmx_engine_decode(glmx_engine* e, const uint32_t* steps, int32_t* out_tokens,
                       float* last_logits);
/* The same decode split in two: _async stages and launches every step of the last staged batch
 * without waiting for the GPU (a prefill may still be in flight; the next prefill may be staged
 * before the collect), _collect waits and writes out_tokens [n_req][max_steps] as above.
 * Continuous batching across rotations: _defer(steps) sets the staged batch's decode aside (its
 * pages are kept); the next batch's _async then runs both sets of rows in one decode (one weight
 * stream per step) and _collect also writes out_prev [deferred n_req][max_steps]. */
int glmx_engine_decode_async(glmx_engine* e, const uint32_t* steps);
int glmx_engine_decode_defer(glmx_engine* e, const uint32_t* steps);
int glmx_engine_decode_collect(glmx_engine* e, int32_t* out_tokens, int32_t* out_prev);
/* Per-phase device times of the last forward (CUDA events on the compute stream), ms:
 * [0] whole forward, [1] attention kernels (sum), [2] KV append (sum), [3] GEMMs (sum),
 * [4] other elementwise, [5] H2D, [6] D2H */
int glmx_engine_last_timings(const glmx_engine* e, float out7[7]);
/* algorithmic work of the last completed forward: [0] attention FLOPs, [1] attention bytes (KV read +
 * Q in + O out), [2] K2 bytes (qkv read + q write + K/V page writes), [3] linear FLOPs, [4] computed tokens, [5] context tokens */
int glmx_engine_last_work(const glmx_engine* e, double out6[6]);
void glmx_engine_set_profiling(glmx_engine* e, int32_t on);
/* KV reuse switch for the reuse on/off A/B: 0 -> every prompt token is computed,
 * cache hits included (their KV is recomputed into scratch pages; the cached pages are not
 * touched); bookkeeping and reports are unchanged.  Default 1. */
void glmx_engine_set_reuse(glmx_engine* e, int32_t on);
/* Bytes the engine moved between host and device since it was created: out2[0] host->device
 * (batch and decode-step metadata: token ids, positions, slots, block tables, the attention
 * schedule, peer-copy lists — the used part of each section only), out2[1] device->host
 * (greedy tokens, requested logits). */
int glmx_engine_io_bytes(const glmx_engine* e, uint64_t out2[2]);

/* ================================================================== kernel-level test hooks */
/* K4: copy pages (all layers) src_pages[i] -> dst_pages[i] between two pools (same or peer
 * device).  Stream-ordered on `stream` (of dst's device). */
int glmx_pool_copy(glmx_kv* src, glmx_kv* dst, const int32_t* src_pages,
                   const int32_t* dst_pages, uint64_t n, void* stream);
float glmx_pool_last_copy_ms(const glmx_kv* dst);
/* K2 on caller-owned DEVICE buffers: qkv [n_tokens][(H + 2 Hkv) * head_dim] bf16 (the QKV
 * projection), pos/slot (device int32 / int64: absolute position, page * block_tokens + offset)
 * -> q_out [n_tokens][H][head_dim] (RoPE'd) and K (RoPE'd), V written into the pool pages of
 * `layer`.  The KV write replaces the reference's block insert (cache.cpp:95-105 inserts the ids;
 * the GPU fills their pages).  Launches `reps` times; out_ms = mean device ms per launch. */
int glmx_rope_kv_append_run(const void* qkv, const int32_t* pos, const int64_t* slot,
                            uint64_t n_tokens, int32_t n_heads, int32_t n_kv_heads,
                            int32_t head_dim, float rope_theta, void* pool, uint32_t n_layers,
                            uint32_t layer, uint32_t block_tokens, void* q_out, int32_t reps,
                            void* stream, float* out_ms);
/* K3's persistent-CTA schedule (host only, no device): items w = i * n_kv_heads + h of work entries
 * work_xy[i] = (request, first token) are flattened into 128-key tiles and cut into <= n_sm
 * equal CTA ranges.  out_pieces [(n_work*n_kv_heads + n_sm) x 4] = (item, j0, j1, partial slot or
 * -1), out_cta_off [n_sm + 1], out_combine [n_sm x 4] = (item, first slot, n slots, 0);
 * out_partners (nullable; same shape as out_pieces) = the single-query-tile item paired with
 * piece i on the CTA's second softmax warpgroup (item -1: none; nullptr disables pairing);
 * out_counts = {pieces, grid, combines, partial slots, total tiles}. */
int glmx_attn_schedule(const int32_t* work_xy, int32_t n_work, int32_t n_kv_heads,
                       const int32_t* q_len, const int32_t* ctx_len, int32_t tokens_per_item,
                       int32_t n_sm, int32_t* out_pieces, int32_t* out_cta_off,
                       int32_t* out_combine, int32_t* out_partners, int64_t out_counts[5]);
/* K2 gather on caller-owned DEVICE buffers: one layer's K (kv = 0) or V (kv = 1) of the pages
 * pages[0..n) (host array, a request's block table) into out [n * block_tokens][n_kv_heads]
 * [head_dim] bf16 — the dense view the attention core reads through TMA; used to export a
 * request's KV.  impl 0 = TMA-staged (bulk load + 2-D TMA store per 4 KB tile), 1 = scalar. */
int glmx_kv_gather_run(void* pool, uint64_t n_pages, uint32_t n_layers, uint32_t n_kv_heads,
                       uint32_t block_tokens, uint32_t head_dim, uint32_t layer, uint32_t kv,
                       const int32_t* pages, uint64_t n, void* out, int32_t impl, int32_t reps,
                       void* stream, float* out_ms);
/* Diagnostics: in the trace build (libglmx_trace.so, `make -C paper_2511_01633_b200/csrc trace`)
 * copies CTA 0's K3 pipeline clock64 stamps (16 events x 1024 key tiles) and clears them;
 * returns the count, or -1 in the product build. */
int32_t glmx_attn_trace_read(int64_t* out, int32_t n);
/* K3 on caller-owned DEVICE buffers — the attention core of the prefill step that replaces the
 * c_prefill cost term (orchestrator.cpp:131-132); no reference counterpart (tensor
 * math is builder-defined).  q/o [n_q_rows][n_heads][head_dim] bf16 (q RoPE'd), pool = pages x
 * [n_layers][K|V][n_kv_heads][block_tokens][head_dim] bf16.  Host arrays per request: q_start,
 * q_len (suffix rows), ctx_len (cached + suffix keys), block_table [n_req][bt_stride] pages.
 * Causal over absolute positions (query t of request r sits at ctx_len - q_len + t).
 * impl 0 = the tcgen05/TMEM/TMA prefill kernel, 2 = the CUDA-core decode kernel (every q_len == 1;
 * the engine uses it for decode steps); any other value is GLMX_ERR_ARG.  Launches `reps` times on `stream`;
 * out_ms = mean device time per launch (CUDA events). */
int glmx_attention_run(int32_t impl, const void* q, void* o, uint64_t n_q_rows, int32_t n_heads,
                       int32_t n_kv_heads, int32_t head_dim, void* pool, uint64_t n_pages,
                       uint32_t n_layers, uint32_t layer, uint32_t block_tokens, uint64_t n_req,
                       const int32_t* q_start, const int32_t* q_len, const int32_t* ctx_len,
                       const int32_t* block_table, int32_t bt_stride, int32_t reps, void* stream,
                       float* out_ms);

#ifdef __cplusplus
}
#endif
#endif /* GLMX_H */
