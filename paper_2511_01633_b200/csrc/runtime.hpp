// Runtime objects behind the C-ABI handles: KV (block engine + device page pool), graph
// (host ingest + device CSR for K1), model (random-init Llama weights), engine (batched
// prefill / decode step).
#pragma once

#include <cublas_v2.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "host/attn_sched.hpp"
#include "host/block_engine.hpp"
#include "host/gemm_tune.hpp"
#include "host/vindex.hpp"
#include "host/graph.hpp"
#include "kernels/attn.cuh"
#include "kernels/chunk.cuh"
#include "kernels/ops.cuh"

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev);
  ~DeviceGuard();
};

// Growable device buffer.
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void reserve(size_t n);
  ~DBuf();
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

struct glmx_kv {
  glmx_kv_config cfg{};
  std::unique_ptr<glmx::BlockEngine> bk;
  glmx::PoolGeom geom{};
  uint64_t page_bytes = 0;
  bool has_pool() const { return geom.base != nullptr; }
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  float last_copy_ms = 0.f;
  DBuf scratch;  // page lists for copies
  // cross-GPU prefix hits
  struct Peer {
    __nv_bfloat16* base = nullptr;
    bool ipc = false;  // opened with cudaIpcOpenMemHandle (closed on destroy)
  };
  std::vector<Peer> peers;
  std::unordered_map<uint64_t, std::pair<int32_t, int32_t>> peer_dir;  // block -> (peer, page)
  bool epoch_mode = false;
  int64_t peer_hits = 0;
  ~glmx_kv();
};

struct glmx_graph {
  glmx::HostGraph host;
  int device = -1;
  glmx::DevGraph dev{};
  uint32_t max_entry = 0;  // longest pre-rendered entry (K1 output bound)
  std::vector<void*> allocs;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  float last_ms = 0.f;
  // K1 scratch
  DBuf d_nodes, d_cnt, d_off, d_bytes, d_tid, d_tbeg, d_tend, d_toff, d_scan, d_irr, d_vrow;
  uint32_t scan_epoch = 0;  // chunk_lengths_scan look-back state (d_scan) epoch
  uint32_t n_irregular = 0;  // irregular entries (0: K1 skips its byte-level chunk kernel)
  uint32_t n_interior = 0;  // interior tokens of the regular entries (DevGraph::itok_*)
  DBuf d_lens;               // per-node chunk lengths for lens_key (chunk_len_table)
  int64_t lens_key = -1;     // (k, weight mode, directed) the table was built for
  DBuf d_itok_id;           // their ids for itok_vocab
  uint32_t itok_vocab = 0;
  // ranked adjacency per (weight mode, directed) variant, built on first use (kernels/chunk.cuh)
  struct Ranked {
    bool ready = false;
    DBuf ridx, pbytes, ptoks, pirr, recs;
  } ranked[4];
  glmx::RankedAdj ranked_adj(int weight_mode, int directed);
  // the last batch built (nodes + config) and its totals: the fill call of the two-call protocol
  // (size query, then the same request with buffers) copies that result out instead of
  // rebuilding it
  std::vector<int32_t> k1_nodes;
  glmx_chunk_config k1_cfg{};
  bool k1_valid = false;
  uint64_t k1_total = 0, k1_ntok = 0;
  // K5 RetrieveNode: device index (rows = nodes with an index text, ascending id), LRU, stats
  int idx_dim = 0, idx_pad = 0;
  std::vector<int32_t> idx_node;  // row -> node index
  DBuf d_emb, d_qemb, d_best;
  glmx::TextLru lru{1024};
  int64_t stats[3] = {0, 0, 0};  // cache_hits, cache_misses, index_probes
  float last_retrieve_ms = 0.f;
  uint64_t h2d_bytes = 0, d2h_bytes = 0;  // K1 / K5 host<->device copies (glmx_graph_io_bytes)
  void upload();
  ~glmx_graph();
};

struct LayerW {
  __nv_bfloat16 *attn_norm, *wqkv, *wo, *mlp_norm, *wgu, *wdown;
};

struct glmx_model {
  glmx_model_config cfg{};
  int device = -1;
  void* arena = nullptr;
  uint64_t arena_bytes = 0;
  __nv_bfloat16 *embed = nullptr, *final_norm = nullptr, *lm_head = nullptr;
  std::vector<LayerW> layers;
  float* inv_freq = nullptr;
  cublasHandle_t blas = nullptr;
  void* blas_ws = nullptr;
  glmx::GemmTuner tuner;  // per-(projection, M bucket) cuBLASLt algorithms; empty = cublasGemmEx
  int n_engines = 0;      // live engines: the algorithm table is immutable while any exists
  bool destroy_pending = false;  // glmx_model_destroy with live engines: freed with the last one
  ~glmx_model();
};

struct glmx_engine {
  glmx_model* m = nullptr;
  glmx_kv* kv = nullptr;
  glmx_engine_config cfg{};
  cudaStream_t stream = nullptr;
  int bt_stride = 0;
  int tpt = 0;  // attention tokens per tile
  alignas(64) uint8_t kv_map[128];  // CUtensorMap over the KV pool (TMA)
  alignas(64) uint8_t q_map[128];   // CUtensorMap over the q activation buffer
  uint32_t kv_rows = 0;

  // activations
  DBuf x, h, qkv, q, attn, gu, act, hl, logits, next_tok, amax_keys, dec_in;
  DBuf rope_cs;  // [T][hd / 2] (cos, sin) of the forward's positions (one table for all layers)
  // batch metadata (device) + pinned host staging (single H2D)
  DBuf meta;
  void* h_meta = nullptr;  // the staging slot in use (one of h_ring)
  // pinned staging ring: the host stages batch / decode-step metadata up to kMetaRing copies
  // ahead of the GPU (slot reuse waits on the event of that slot's previous upload)
  static constexpr int kMetaRing = 8;
  void* h_ring[kMetaRing] = {};
  cudaEvent_t ring_ev[kMetaRing] = {};
  int ring_slot = 0;
  // asynchronous decode: enqueued steps of the staged batch, collected by engine_decode_collect
  bool dec_pending = false;
  std::vector<int> dec_order;
  std::vector<uint32_t> dec_steps;
  uint32_t dec_max = 0;
  int dec_R = 0;
  int32_t* h_dec = nullptr;
  cudaEvent_t dec_done = nullptr;
  size_t o_perm = 0;  // meta: decode row order (first-token gather)
  uint64_t prof_tag = 0;       // != 0: profiling spans tagged with this instead of batch_seq
  uint64_t dec_tag_batch = 0;  // batch_seq when the pending decode was enqueued
  size_t meta_bytes = 0;
  int32_t* h_out = nullptr;  // pinned: tokens out
  cudaEvent_t h2d_done = nullptr, fwd_done = nullptr;

  // last batch (for decode / replay)
  struct Req {
    int32_t ctx_len = 0;
    std::vector<int32_t> pages;  // full blocks + scratch
    std::vector<int32_t> scratch;
  };
  std::vector<Req> reqs;
  // a batch whose decode is deferred to run merged with the next batch's decode (continuous
  // batching of decode rows across rotations): its requests (pages kept), steps, first tokens
  std::vector<Req> def_reqs;
  std::vector<uint32_t> def_steps;
  DBuf def_first;
  int def_R = 0;            // rows of the deferred batch (0: none)
  int dec_R_def = 0;        // rows of the deferred batch merged into the pending decode
  std::vector<Req> dec_free;  // requests whose scratch pages are freed at the next collect
  int last_T = 0, last_R = 0, last_work = 0;
  bool has_batch = false;
  // offsets into meta
  struct Copy {
    int32_t peer, src_page, dst_page;
  };
  std::vector<Copy> copies;  // peer page copies of the current batch
  size_t max_copies = 0, o_copy = 0;
  size_t o_tok = 0, o_pos = 0, o_slot = 0, o_qs = 0, o_ql = 0, o_ctx = 0, o_bt = 0, o_work = 0,
         o_last = 0;
  // The host stages a batch at the fixed capacity offsets above; meta_commit packs the used part
  // of every section (block-table rows at the batch's own stride) in place and uploads only
  // those bytes.  ml = the packed layout of the last upload (what the kernels read).
  struct MetaLayout {
    size_t tok, pos, slot, qs, ql, ctx, bt, work, last, perm, pieces, partners, cta, comb, copy;
    size_t bytes;
    int bt_stride;
  };
  MetaLayout ml{};
  int sc_npieces = 0;
  uint64_t h2d_bytes = 0, d2h_bytes = 0;  // cumulative host<->device bytes moved by the engine
  DBuf blas_ws;                           // this engine's cuBLAS / cuBLASLt workspace
  // deferred (evicted) pages: released at the next prefill's start (rel_mark = the pool's defer
  // mark after the last batch), or, for a batch whose decode is deferred, only once that merged
  // decode is enqueued (def_mark)
  uint64_t rel_mark = 0, def_mark = 0;
  std::vector<uint64_t> batch_written;  // stale blocks this batch recomputes (rollback on error)
  // K3 stream-K schedule (packed in meta) + partial workspace
  size_t o_sched = 0, o_sc_pieces = 0, o_sc_cta = 0, o_sc_comb = 0, o_sc_part = 0;
  int sc_grid = 0, sc_ncomb = 0;
  int dec_split = 0;      // > 0: the staged batch is all one-token rows -> K3d with this many splits
  DBuf part_o, part_ml;

  int reuse = 1;          // 0: hits recomputed into scratch pages (reuse on/off A/B)
  // profiling
  int profiling = 0;
  struct Span {
    cudaEvent_t a, b;
    int cat;
    uint64_t batch;
  };
  std::vector<cudaEvent_t> ev_free;  // recycled timing events
  std::vector<Span> spans;
  float timings[7] = {0};
  double work[6] = {0};       // algorithmic work of the batch being staged
  double work_done[6] = {0};  // ... of the last completed (waited) batch
  // asynchronous prefill: up to two batches in flight on the engine stream (the host stages and
  // does the bookkeeping of batch r+1 while batch r runs); results are collected in order
  struct Pending {
    std::vector<int> req_row;
    uint64_t batch;
    int slot;
    double work[6];
  };
  std::vector<Pending> pending;  // FIFO (front = oldest)
  uint64_t batch_seq = 0;        // batch being staged / enqueued
  cudaEvent_t done_ev[2] = {nullptr, nullptr};
  size_t h_out_stride = 0;       // int32 entries per h_out slot

  ~glmx_engine();
};
