// extern "C" surface (include/glmx.h).  Every entry point converts C++ exceptions into the
// status codes that mirror the reference's exception classes (error.hpp:29-137).
#include <cstring>
#include <string>

#include "runtime.hpp"

using namespace glmx;

#define GLMX_CUDA(call)                                                                       \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      throw ::glmx::Error(GLMX_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

int chunk_build_impl(glmx_graph*, const glmx_chunk_config*, const int32_t*, uint64_t, char*,
                     uint64_t, uint64_t*, int32_t*, uint64_t*, uint64_t*, uint64_t, uint64_t*,
                     uint64_t*, uint64_t*);
glmx_kv* kv_create_impl(const glmx_kv_config*);
void pool_copy_impl(glmx_kv*, glmx_kv*, const int32_t*, const int32_t*, uint64_t, cudaStream_t);
glmx_model* model_create_impl(const glmx_model_config*, int);
int model_export_impl(const glmx_model*, int, int, uint16_t*, uint64_t);
int model_tune_gemms_impl(glmx_model*, int);
glmx_engine* engine_create_impl(glmx_model*, glmx_kv*, const glmx_engine_config*);
int engine_prefill_impl(glmx_engine*, uint64_t, const glmx_request*, glmx_prefill_report*,
                        int32_t*, float*, bool);
int engine_wait_impl(glmx_engine*, int32_t*, uint64_t);
int engine_decode_impl(glmx_engine*, const uint32_t*, int32_t*, float*);
int engine_decode_enqueue(glmx_engine*, const uint32_t*);
int engine_decode_collect(glmx_engine*, int32_t*, int32_t*, float*);
int engine_decode_defer(glmx_engine*, const uint32_t*);
int index_build_impl(glmx_graph*, int, uint64_t);
int kv_gather_run_impl(void*, uint64_t, uint32_t, uint32_t, uint32_t, uint32_t, uint32_t, uint32_t,
                       const int32_t*, uint64_t, void*, int, int, cudaStream_t, float*);
int workload_generate_impl(glmx_graph*, uint64_t, int, double, std::string*, float*);
int retrieve_impl(glmx_graph*, const char*, const uint64_t*, uint64_t, int32_t*, uint8_t*);
int rope_append_run_impl(const void*, const int32_t*, const int64_t*, uint64_t, int, int, int,
                         float, void*, uint32_t, uint32_t, uint32_t, void*, int, cudaStream_t,
                         float*);
int attention_run_impl(int, const void*, void*, uint64_t, int, int, int, void*, uint64_t, uint32_t,
                       uint32_t, uint32_t, uint64_t, const int32_t*, const int32_t*,
                       const int32_t*, const int32_t*, int, int, cudaStream_t, float*);

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    g_err.clear();
    return f();
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return GLMX_ERR_ARG;
  } catch (const std::exception& e) {
    g_err = e.what();
    return GLMX_ERR_ARG;
  }
}

int64_t copy_str(const std::string& s, char* buf, uint64_t cap) {
  if (buf && cap) std::memcpy(buf, s.data(), std::min<uint64_t>(cap, s.size()));
  return static_cast<int64_t>(s.size());
}

void fill_report(const PrefillResult& r, glmx_prefill_report* rep, int32_t* bt, uint64_t bt_cap,
                 uint64_t* ev, uint64_t ev_cap) {
  if (rep) {
    rep->cached_tokens = r.cached;
    rep->computed_tokens = r.computed;
    rep->tail_tokens = r.tail;
    rep->n_evicted = r.evicted.size();
    rep->n_blocks = r.pages.size();
  }
  if (bt)
    for (uint64_t i = 0; i < r.pages.size() && i < bt_cap; ++i) bt[i] = r.pages[i];
  if (ev)
    for (uint64_t i = 0; i < r.evicted.size() && i < ev_cap; ++i) ev[i] = r.evicted[i];
}
}  // namespace

extern "C" {

const char* glmx_last_error(void) { return g_err.c_str(); }
const char* glmx_version(void) { return "glmx 0.1 (sm_100a)"; }
int glmx_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

// ------------------------------------------------------------------ KV
int glmx_kv_create(const glmx_kv_config* cfg, glmx_kv** out) {
  return guarded([&] {
    if (!cfg || !out) throw Error(GLMX_ERR_ARG, "null argument");
    *out = kv_create_impl(cfg);
    return GLMX_OK;
  });
}
void glmx_kv_destroy(glmx_kv* kv) {
  if (!kv) return;
  DeviceGuard g(kv->cfg.device);
  delete kv;
}

int glmx_kv_prefill(glmx_kv* kv, const char* tok_bytes, const uint64_t* tok_offsets,
                    uint64_t n_tok, const glmx_tier_range* tiers, uint64_t n_tiers,
                    const char* session, glmx_prefill_report* report, int32_t* block_table,
                    uint64_t block_table_cap, uint64_t* evicted, uint64_t evicted_cap) {
  return guarded([&] {
    if (!kv->has_pool()) kv->bk->pool().release_deferred();
    PrefillResult r;
    TokenSpans ts{tok_bytes, tok_offsets, n_tok};
    kv->bk->prefill(ts, tiers, n_tiers, session ? session : "", r);
    fill_report(r, report, block_table, block_table_cap, evicted, evicted_cap);
    return GLMX_OK;
  });
}

int glmx_kv_prefill_segments(glmx_kv* kv, uint64_t n_seg, const char* const* seg_text,
                             const uint64_t* seg_len, const int32_t* seg_tier,
                             const char* session, glmx_prefill_report* report,
                             int32_t* block_table, uint64_t block_table_cap, uint64_t* evicted,
                             uint64_t evicted_cap) {
  return guarded([&] {
    // Orchestrator::kv_prefill (orchestrator.cpp:81-97)
    std::string bytes;
    std::vector<uint64_t> offs{0};
    std::vector<glmx_tier_range> tiers;
    std::vector<uint64_t> b, e;
    for (uint64_t i = 0; i < n_seg; ++i) {
      b.clear();
      e.clear();
      tokenize_spans(seg_text[i], seg_len[i], b, e);
      if (b.empty()) continue;
      const uint64_t begin = offs.size() - 1;
      for (size_t j = 0; j < b.size(); ++j) {
        bytes.append(seg_text[i] + b[j], e[j] - b[j]);
        offs.push_back(bytes.size());
      }
      const uint64_t end = offs.size() - 1;
      if (!tiers.empty() && tiers.back().tier == seg_tier[i])
        tiers.back().end = end;
      else
        tiers.push_back({begin, end, seg_tier[i], 0});
    }
    if (!kv->has_pool()) kv->bk->pool().release_deferred();
    PrefillResult r;
    TokenSpans ts{bytes.data(), offs.data(), offs.size() - 1};
    kv->bk->prefill(ts, tiers.data(), tiers.size(), session ? session : "", r);
    fill_report(r, report, block_table, block_table_cap, evicted, evicted_cap);
    return GLMX_OK;
  });
}

uint64_t glmx_kv_last_evicted(const glmx_kv* kv, uint64_t* out, uint64_t cap) {
  const auto& v = kv->bk->last_evicted();
  for (uint64_t i = 0; i < v.size() && i < cap; ++i) out[i] = v[i];
  return v.size();
}

int glmx_kv_evict(glmx_kv* kv, uint64_t n, uint64_t* out, uint64_t cap, uint64_t* n_out) {
  return guarded([&] {
    if (n_out) *n_out = 0;
    auto ids = kv->bk->evict(n);
    for (uint64_t i = 0; i < ids.size() && i < cap; ++i) out[i] = ids[i];
    if (n_out) *n_out = std::min<uint64_t>(ids.size(), cap);
    if (!kv->has_pool()) kv->bk->pool().release_deferred();
    return GLMX_OK;
  });
}

int glmx_kv_set_tier(glmx_kv* kv, const char* session, int32_t from_tier, int32_t to_tier) {
  return guarded([&] {
    kv->bk->set_tier(session ? session : "", from_tier, to_tier);
    return GLMX_OK;
  });
}

int glmx_kv_force_insert(glmx_kv* kv, uint64_t id, int32_t tier, uint64_t last_used,
                         const char* session) {
  return guarded([&] {
    if (tier < 0 || tier > 3) throw Error(GLMX_ERR_ARG, "tier out of range");
    kv->bk->force_insert(id, tier, last_used, session ? session : "");
    return GLMX_OK;
  });
}

int glmx_kv_counters(const glmx_kv* kv, int64_t out6[6]) {
  out6[0] = kv->bk->hits();
  out6[1] = kv->bk->misses();
  for (int t = 0; t < 4; ++t) out6[2 + t] = kv->bk->evictions_by_tier()[t];
  return GLMX_OK;
}

uint64_t glmx_kv_resident(const glmx_kv* kv, uint64_t* ids, int32_t* tiers, uint64_t* last_used,
                          int32_t* pages, uint64_t cap) {
  if (cap == 0) return kv->bk->resident();
  auto v = kv->bk->resident_sorted();
  for (uint64_t i = 0; i < v.size() && i < cap; ++i) {
    if (ids) ids[i] = v[i]->id;
    if (tiers) tiers[i] = v[i]->tier;
    if (last_used) last_used[i] = v[i]->last_used;
    if (pages) pages[i] = (kv->has_pool() && v[i]->stale) ? -1 : v[i]->page;  // -1: no KV (yet)
  }
  return v.size();
}

int32_t glmx_kv_block(const glmx_kv* kv, uint64_t id, int32_t* tier, uint64_t* last_used,
                      uint64_t* parent, int32_t* has_parent) {
  const Block* b = kv->bk->block(id);
  if (!b) return 0;
  if (tier) *tier = b->tier;
  if (last_used) *last_used = b->last_used;
  if (parent) *parent = b->parent;
  if (has_parent) *has_parent = b->has_parent ? 1 : 0;
  return 1;
}

int64_t glmx_kv_block_session(const glmx_kv* kv, uint64_t id, char* buf, uint64_t cap) {
  const Block* b = kv->bk->block(id);
  if (!b) return -1;
  return copy_str(kv->bk->session_name(b->session), buf, cap);
}

int64_t glmx_kv_snapshot_json(const glmx_kv* kv, char* buf, uint64_t cap) {
  return copy_str(kv->bk->snapshot_json(), buf, cap);
}

uint64_t glmx_kv_chain_ids(const char* tok_bytes, const uint64_t* tok_offsets, uint64_t n_tok,
                           uint32_t block_tokens, uint64_t* out) {
  if (block_tokens == 0) return 0;
  std::vector<uint64_t> ids;
  BlockEngine::chain_ids(TokenSpans{tok_bytes, tok_offsets, n_tok}, block_tokens, ids);
  if (out) std::memcpy(out, ids.data(), ids.size() * 8);
  return ids.size();
}

int glmx_kv_release_deferred(glmx_kv* kv) {
  kv->bk->pool().release_deferred();
  return GLMX_OK;
}
uint64_t glmx_kv_defer_mark(const glmx_kv* kv) { return kv->bk->pool().mark(); }
int glmx_kv_release_deferred_before(glmx_kv* kv, uint64_t mark) {
  kv->bk->pool().release_before(mark);
  return GLMX_OK;
}
uint64_t glmx_kv_pool_pages(const glmx_kv* kv) { return kv->bk->pool().total(); }
uint64_t glmx_kv_free_pages(const glmx_kv* kv) { return kv->bk->pool().free_count(); }
void* glmx_kv_pool_ptr(const glmx_kv* kv) { return kv->geom.base; }
uint64_t glmx_kv_page_bytes(const glmx_kv* kv) { return kv->page_bytes; }

// ------------------------------------------------------------------ cross-GPU prefix hits
int glmx_kv_ipc_handle(const glmx_kv* kv, uint8_t out[64]) {
  return guarded([&] {
    if (!kv->has_pool()) throw Error(GLMX_ERR_NO_DEVICE, "no device pool");
    DeviceGuard g(kv->cfg.device);
    cudaIpcMemHandle_t h;
    GLMX_CUDA(cudaIpcGetMemHandle(&h, kv->geom.base));
    static_assert(sizeof(h) == 64, "ipc handle size");
    std::memcpy(out, &h, 64);
    return GLMX_OK;
  });
}

static void set_peer(glmx_kv* kv, int32_t peer, __nv_bfloat16* base, bool ipc) {
  if (peer < 0 || peer > 1024) throw Error(GLMX_ERR_ARG, "peer index out of range");
  if (kv->peers.size() <= static_cast<size_t>(peer)) kv->peers.resize(peer + 1);
  kv->peers[peer] = {base, ipc};
}

int glmx_kv_attach_peer(glmx_kv* kv, int32_t peer, const uint8_t handle[64]) {
  return guarded([&] {
    if (!kv->has_pool()) throw Error(GLMX_ERR_NO_DEVICE, "no device pool");
    DeviceGuard g(kv->cfg.device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    void* p = nullptr;
    GLMX_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    set_peer(kv, peer, static_cast<__nv_bfloat16*>(p), true);
    return GLMX_OK;
  });
}

int glmx_kv_attach_peer_local(glmx_kv* kv, int32_t peer, const glmx_kv* other) {
  return guarded([&] {
    if (!kv->has_pool() || !other->has_pool()) throw Error(GLMX_ERR_NO_DEVICE, "no device pool");
    if (other->page_bytes != kv->page_bytes) throw Error(GLMX_ERR_ARG, "pool geometries differ");
    if (other->cfg.device != kv->cfg.device) {
      DeviceGuard g(kv->cfg.device);
      cudaError_t e = cudaDeviceEnablePeerAccess(other->cfg.device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        throw Error(GLMX_ERR_CUDA, std::string("peer access: ") + cudaGetErrorString(e));
      cudaGetLastError();
    }
    set_peer(kv, peer, other->geom.base, false);
    return GLMX_OK;
  });
}

int glmx_kv_set_peer_directory(glmx_kv* kv, uint64_t n, const uint64_t* block_ids,
                               const int32_t* peers, const int32_t* pages) {
  return guarded([&] {
    kv->peer_dir.clear();
    kv->peer_dir.reserve(n);
    const uint64_t total = kv->bk->pool().total();
    for (uint64_t i = 0; i < n; ++i) {
      if (pages[i] < 0) continue;  // a stale block (no KV in its page): not servable
      if (static_cast<uint64_t>(pages[i]) >= total) throw Error(GLMX_ERR_ARG, "directory page out of range");
      kv->peer_dir.emplace(block_ids[i], std::make_pair(peers[i], pages[i]));  // first wins
    }
    return GLMX_OK;
  });
}

int glmx_kv_set_epoch_mode(glmx_kv* kv, int32_t on) {
  kv->epoch_mode = on != 0;
  return GLMX_OK;
}

int64_t glmx_kv_peer_hits(const glmx_kv* kv) { return kv->peer_hits; }

uint64_t glmx_tokenize(const char* text, uint64_t len, uint64_t* begins, uint64_t* ends,
                       uint64_t cap) {
  std::vector<uint64_t> b, e;
  tokenize_spans(text, len, b, e);
  for (uint64_t i = 0; i < b.size() && i < cap; ++i) {
    if (begins) begins[i] = b[i];
    if (ends) ends[i] = e[i];
  }
  return b.size();
}

int32_t glmx_token_id(const char* tok, uint64_t len, uint32_t vocab) {
  return vocab ? token_id(tok, len, vocab) : -1;
}

// ------------------------------------------------------------------ graph
static glmx_graph* finish_graph(HostGraph&& h, int device) {
  auto g = std::make_unique<glmx_graph>();
  g->host = std::move(h);
  g->device = device;
  if (device >= 0) g->upload();
  return g.release();
}

int glmx_graph_load_jsonl(const char* path, int32_t device, glmx_graph** out) {
  return guarded([&] {
    *out = finish_graph(load_graph_jsonl(path, device < 0), device);
    return GLMX_OK;
  });
}

int glmx_graph_synth_powerlaw(uint64_t n_nodes, uint32_t edges_per_node, uint64_t seed,
                              int32_t device, glmx_graph** out) {
  return guarded([&] {
    *out = finish_graph(synth_powerlaw(n_nodes, edges_per_node, seed, device < 0), device);
    return GLMX_OK;
  });
}

int glmx_graph_save_jsonl(const glmx_graph* g, const char* path) {
  return guarded([&] {
    FILE* f = std::fopen(path, "wb");
    if (!f) throw Error(GLMX_ERR_GLM, std::string("cannot write graph file: ") + path);
    std::string s = g->host.serialize_jsonl();
    std::fwrite(s.data(), 1, s.size(), f);
    std::fclose(f);
    return GLMX_OK;
  });
}

void glmx_graph_destroy(glmx_graph* g) {
  if (!g) return;
  DeviceGuard dg(g->device);
  delete g;
}
uint64_t glmx_graph_node_count(const glmx_graph* g) { return g->host.n(); }
uint64_t glmx_graph_edge_count(const glmx_graph* g) { return g->host.src.size(); }
int64_t glmx_graph_node_index(const glmx_graph* g, const char* id) {
  auto it = g->host.index.find(id);
  return it == g->host.index.end() ? -1 : it->second;
}
int64_t glmx_graph_node_id(const glmx_graph* g, uint64_t idx, char* buf, uint64_t cap) {
  if (idx >= g->host.n()) return -1;
  return copy_str(g->host.ids[idx], buf, cap);
}
int64_t glmx_graph_node_attr(const glmx_graph* g, uint64_t idx, const char* key, char* buf,
                             uint64_t cap, int32_t* kind) {
  if (idx >= g->host.n() || !key) return -1;
  const auto& a = g->host.attrs[idx];
  for (size_t i = 0; i < a.size(); ++i)
    if (a[i].first == key) {
      if (kind) *kind = g->host.attr_kind.empty() ? 0 : g->host.attr_kind[idx][i];
      return copy_str(a[i].second, buf, cap);
    }
  return -1;
}
int glmx_graph_io_bytes(const glmx_graph* g, uint64_t out2[2]) {
  out2[0] = g->h2d_bytes;
  out2[1] = g->d2h_bytes;
  return GLMX_OK;
}
int64_t glmx_graph_degree(const glmx_graph* g, uint64_t idx) {
  if (idx >= g->host.n()) return -1;
  return g->host.w_total[idx];
}

int glmx_chunk_build(glmx_graph* g, const glmx_chunk_config* cfg, const int32_t* node_idx,
                     uint64_t n, char* out_bytes, uint64_t bytes_cap, uint64_t* out_byte_offsets,
                     int32_t* out_tok_ids, uint64_t* out_tok_begin, uint64_t* out_tok_end,
                     uint64_t tok_cap, uint64_t* out_tok_offsets, uint64_t* total_bytes,
                     uint64_t* total_tokens) {
  return guarded([&] {
    return chunk_build_impl(g, cfg, node_idx, n, out_bytes, bytes_cap, out_byte_offsets,
                            out_tok_ids, out_tok_begin, out_tok_end, tok_cap, out_tok_offsets,
                            total_bytes, total_tokens);
  });
}

int64_t glmx_node_info_rendered(glmx_graph* g, const glmx_chunk_config* cfg, const char* id,
                                char* buf, uint64_t cap) {
  int64_t len = -GLMX_ERR_ARG;
  int st = guarded([&] {
    auto it = g->host.index.find(id);
    if (it == g->host.index.end()) throw Error(GLMX_ERR_RETRIEVAL, std::string("unknown node id: ") + id);
    int32_t idx = it->second;
    uint64_t tb = 0, tt = 0;
    chunk_build_impl(g, cfg, &idx, 1, nullptr, 0, nullptr, nullptr, nullptr, nullptr, 0, nullptr,
                     &tb, &tt);
    std::string out(tb, '\0');
    uint64_t offs[2];
    chunk_build_impl(g, cfg, &idx, 1, out.data(), tb, offs, nullptr, nullptr, nullptr, 0,
                     nullptr, &tb, &tt);
    len = copy_str(out, buf, cap);
    return GLMX_OK;
  });
  return st == GLMX_OK ? len : -st;
}

float glmx_chunk_last_kernel_ms(const glmx_graph* g) { return g->last_ms; }

int glmx_index_build(glmx_graph* g, int32_t dim, uint64_t cache_capacity) {
  return guarded([&] { return index_build_impl(g, dim, cache_capacity); });
}
uint64_t glmx_index_size(const glmx_graph* g) { return g->idx_node.size(); }
int64_t glmx_workload_generate(glmx_graph* g, uint64_t seed, int32_t n, double nondet_ratio,
                               char* buf, uint64_t cap, float* out_scan_ms) {
  std::string out;
  const int st = guarded([&] { return workload_generate_impl(g, seed, n, nondet_ratio, &out, out_scan_ms); });
  if (st != GLMX_OK) return -st;
  return copy_str(out, buf, cap);
}
int glmx_retrieve_nodes(glmx_graph* g, const char* text_bytes, const uint64_t* text_offsets,
                        uint64_t n, int32_t* out_node_idx, uint8_t* out_cache_hit) {
  return guarded([&] { return retrieve_impl(g, text_bytes, text_offsets, n, out_node_idx, out_cache_hit); });
}
void glmx_retriever_stats(const glmx_graph* g, int64_t out3[3]) {
  for (int i = 0; i < 3; ++i) out3[i] = g->stats[i];
}
float glmx_retrieve_last_kernel_ms(const glmx_graph* g) { return g->last_retrieve_ms; }
int glmx_embed_text(const char* text, uint64_t len, int32_t dim, float* out) {
  return guarded([&] {
    if (dim < 1) throw Error(GLMX_ERR_ARG, "dim must be >= 1");
    glmx::embed(text, len, dim, out);
    return GLMX_OK;
  });
}

// ------------------------------------------------------------------ model / engine
int glmx_model_create(const glmx_model_config* cfg, int32_t device, glmx_model** out) {
  return guarded([&] {
    *out = model_create_impl(cfg, device);
    return GLMX_OK;
  });
}
void glmx_model_destroy(glmx_model* m) {
  if (!m) return;
  if (m->n_engines > 0) {  // engines still run on its weights: freed when the last one goes
    m->destroy_pending = true;
    return;
  }
  DeviceGuard g(m->device);
  delete m;
}
int glmx_model_export_weight(const glmx_model* m, int32_t which, int32_t layer, uint16_t* out,
                             uint64_t n) {
  return guarded([&] { return model_export_impl(m, which, layer, out, n); });
}

int glmx_model_tune_gemms(glmx_model* m, int32_t max_tokens, int32_t* out_entries) {
  return guarded([&] {
    const int n = model_tune_gemms_impl(m, max_tokens);
    if (out_entries) *out_entries = n;
    return GLMX_OK;
  });
}

int glmx_engine_create(glmx_model* m, glmx_kv* kv, const glmx_engine_config* cfg,
                       glmx_engine** out) {
  return guarded([&] {
    *out = engine_create_impl(m, kv, cfg);
    return GLMX_OK;
  });
}
void glmx_engine_destroy(glmx_engine* e) {
  if (!e) return;
  DeviceGuard g(e->m->device);
  delete e;
}
int glmx_engine_prefill(glmx_engine* e, uint64_t n_req, const glmx_request* reqs,
                        glmx_prefill_report* reports, int32_t* first_token, float* logits) {
  return guarded([&] { return engine_prefill_impl(e, n_req, reqs, reports, first_token, logits, false); });
}
}  // extern "C"

namespace {
int prefill_segments(glmx_engine* e, uint64_t n_req, const glmx_segment_request* reqs,
                     glmx_prefill_report* reports, int32_t* first_token, float* logits, bool async) {
  return guarded([&] {
    // Orchestrator::kv_prefill (orchestrator.cpp:81-97) per request, then one batched step.
    struct Tok {
      std::string bytes;
      std::vector<uint64_t> offs{0};
      std::vector<glmx_tier_range> tiers;
    };
    std::vector<Tok> toks(n_req);
    std::vector<glmx_request> rq(n_req);
    std::vector<uint64_t> b, en;
    for (uint64_t r = 0; r < n_req; ++r) {
      Tok& t = toks[r];
      const glmx_segment_request& s = reqs[r];
      for (uint64_t i = 0; i < s.n_seg; ++i) {
        b.clear();
        en.clear();
        tokenize_spans(s.seg_text[i], s.seg_len[i], b, en);
        if (b.empty()) continue;
        const uint64_t begin = t.offs.size() - 1;
        for (size_t j = 0; j < b.size(); ++j) {
          t.bytes.append(s.seg_text[i] + b[j], en[j] - b[j]);
          t.offs.push_back(t.bytes.size());
        }
        const uint64_t end = t.offs.size() - 1;
        if (!t.tiers.empty() && t.tiers.back().tier == s.seg_tier[i])
          t.tiers.back().end = end;
        else
          t.tiers.push_back({begin, end, s.seg_tier[i], 0});
      }
      rq[r] = {t.bytes.data(), t.offs.data(), t.offs.size() - 1, t.tiers.data(), t.tiers.size(),
               s.session, s.finish};
    }
    return engine_prefill_impl(e, n_req, rq.data(), reports, first_token, logits, async);
  });
}
}  // namespace

extern "C" {
int glmx_engine_prefill_segments(glmx_engine* e, uint64_t n_req,
                                 const glmx_segment_request* reqs, glmx_prefill_report* reports,
                                 int32_t* first_token, float* logits) {
  return prefill_segments(e, n_req, reqs, reports, first_token, logits, false);
}
int glmx_engine_prefill_segments_async(glmx_engine* e, uint64_t n_req,
                                       const glmx_segment_request* reqs,
                                       glmx_prefill_report* reports) {
  return prefill_segments(e, n_req, reqs, reports, nullptr, nullptr, true);
}
int glmx_engine_wait(glmx_engine* e, int32_t* first_token, uint64_t cap) {
  int n = 0;
  const int st = guarded([&] {
    n = engine_wait_impl(e, first_token, cap);
    return GLMX_OK;
  });
  return st == GLMX_OK ? n : -st;
}
int32_t glmx_engine_in_flight(const glmx_engine* e) { return static_cast<int32_t>(e->pending.size()); }
int glmx_engine_decode(glmx_engine* e, const uint32_t* steps, int32_t* out_tokens,
                       float* last_logits) {
  return guarded([&] { return engine_decode_impl(e, steps, out_tokens, last_logits); });
}
int glmx_engine_decode_async(glmx_engine* e, const uint32_t* steps) {
  return guarded([&] { return engine_decode_enqueue(e, steps); });
}
int glmx_engine_decode_collect(glmx_engine* e, int32_t* out_tokens, int32_t* out_prev) {
  return guarded([&] { return engine_decode_collect(e, out_tokens, out_prev, nullptr); });
}
int glmx_engine_decode_defer(glmx_engine* e, const uint32_t* steps) {
  return guarded([&] { return engine_decode_defer(e, steps); });
}
int glmx_engine_last_timings(const glmx_engine* e, float out7[7]) {
  std::memcpy(out7, e->timings, sizeof(e->timings));
  return GLMX_OK;
}
int glmx_engine_last_work(const glmx_engine* e, double out6[6]) {  // of the last completed batch
  std::memcpy(out6, e->work_done, sizeof(e->work_done));
  return GLMX_OK;
}
void glmx_engine_set_profiling(glmx_engine* e, int32_t level) { e->profiling = level; }
void glmx_engine_set_reuse(glmx_engine* e, int32_t on) { e->reuse = on ? 1 : 0; }
int glmx_engine_io_bytes(const glmx_engine* e, uint64_t out2[2]) {
  out2[0] = e->h2d_bytes;
  out2[1] = e->d2h_bytes;
  return GLMX_OK;
}

// ------------------------------------------------------------------ kernel test hooks
int glmx_pool_copy(glmx_kv* src, glmx_kv* dst, const int32_t* src_pages,
                   const int32_t* dst_pages, uint64_t n, void* stream) {
  return guarded([&] {
    pool_copy_impl(src, dst, src_pages, dst_pages, n, static_cast<cudaStream_t>(stream));
    return GLMX_OK;
  });
}
float glmx_pool_last_copy_ms(const glmx_kv* dst) { return dst->last_copy_ms; }

int glmx_rope_kv_append_run(const void* qkv, const int32_t* pos, const int64_t* slot,
                            uint64_t n_tokens, int32_t n_heads, int32_t n_kv_heads,
                            int32_t head_dim, float rope_theta, void* pool, uint32_t n_layers,
                            uint32_t layer, uint32_t block_tokens, void* q_out, int32_t reps,
                            void* stream, float* out_ms) {
  return guarded([&] {
    return rope_append_run_impl(qkv, pos, slot, n_tokens, n_heads, n_kv_heads, head_dim,
                                rope_theta, pool, n_layers, layer, block_tokens, q_out, reps,
                                static_cast<cudaStream_t>(stream), out_ms);
  });
}

int32_t glmx_attn_trace_read(int64_t* out, int32_t n) {
  int32_t r = -1;
  guarded([&] {
    r = attn_trace_read(reinterpret_cast<long long*>(out), n);
    return GLMX_OK;
  });
  return r;
}

int glmx_kv_gather_run(void* pool, uint64_t n_pages, uint32_t n_layers, uint32_t n_kv_heads,
                       uint32_t block_tokens, uint32_t head_dim, uint32_t layer, uint32_t kv,
                       const int32_t* pages, uint64_t n, void* out, int32_t impl, int32_t reps,
                       void* stream, float* out_ms) {
  return guarded([&] {
    return kv_gather_run_impl(pool, n_pages, n_layers, n_kv_heads, block_tokens, head_dim, layer, kv,
                              pages, n, out, impl, reps, static_cast<cudaStream_t>(stream), out_ms);
  });
}

int glmx_attn_schedule(const int32_t* work_xy, int32_t n_work, int32_t n_kv_heads,
                       const int32_t* q_len, const int32_t* ctx_len, int32_t tokens_per_item,
                       int32_t n_sm, int32_t* out_pieces, int32_t* out_cta_off,
                       int32_t* out_combine, int32_t* out_partners, int64_t out_counts[5]) {
  return guarded([&] {
    if (n_work < 0 || n_kv_heads < 1 || tokens_per_item < 1 || n_sm < 1)
      throw Error(GLMX_ERR_ARG, "bad schedule arguments");
    AttnSchedule sc;
    sc.pieces = reinterpret_cast<AttnPiece*>(out_pieces);
    sc.cta_off = out_cta_off;
    sc.combine = reinterpret_cast<AttnCombine*>(out_combine);
    sc.partners = reinterpret_cast<AttnPiece*>(out_partners);
    build_attn_schedule(work_xy, n_work, n_kv_heads, q_len, ctx_len, tokens_per_item, 128, n_sm, sc);
    out_counts[0] = sc.n_pieces;
    out_counts[1] = sc.grid;
    out_counts[2] = sc.n_combine;
    out_counts[3] = sc.n_partials;
    out_counts[4] = sc.total_tiles;
    return GLMX_OK;
  });
}

int glmx_attention_run(int32_t impl, const void* q, void* o, uint64_t n_q_rows, int32_t n_heads,
                       int32_t n_kv_heads, int32_t head_dim, void* pool, uint64_t n_pages,
                       uint32_t n_layers, uint32_t layer, uint32_t block_tokens, uint64_t n_req,
                       const int32_t* q_start, const int32_t* q_len, const int32_t* ctx_len,
                       const int32_t* block_table, int32_t bt_stride, int32_t reps, void* stream,
                       float* out_ms) {
  return guarded([&] {
    return attention_run_impl(impl, q, o, n_q_rows, n_heads, n_kv_heads, head_dim, pool, n_pages,
                              n_layers, layer, block_tokens, n_req, q_start, q_len, ctx_len,
                              block_table, bt_stride, reps, static_cast<cudaStream_t>(stream),
                              out_ms);
  });
}

}  // extern "C"
