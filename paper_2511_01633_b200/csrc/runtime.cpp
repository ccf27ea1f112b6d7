#include "runtime.hpp"

#include <nvtx3/nvToolsExt.h>

namespace {
// NVTX range over a host-side phase (bookkeeping, staging, K1/K5 batches, decode, page copies)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

#include <algorithm>
#include <cmath>
#include <cstring>

#include "kernels/common.cuh"
#include "kernels/retrieve.cuh"
#include "kernels/ingest.cuh"
#include "host/workload_gen.hpp"

using namespace glmx;

namespace {

// Non-blocking stream at the device's greatest (high) or least (low) priority.
cudaStream_t make_stream(bool high) {
  int least = 0, greatest = 0;
  GLMX_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  cudaStream_t s = nullptr;
  GLMX_CUDA(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, high ? greatest : least));
  return s;
}
constexpr size_t kBlasWsBytes = 64ull << 20;  // cuBLAS / cuBLASLt workspace per model
}

#define GLMX_BLAS(call)                                                                   \
  do {                                                                                    \
    cublasStatus_t s_ = (call);                                                           \
    if (s_ != CUBLAS_STATUS_SUCCESS)                                                      \
      throw Error(GLMX_ERR_CUDA, std::string(#call) + ": cublas status " + std::to_string(s_)); \
  } while (0)

DeviceGuard::DeviceGuard(int dev) {
  if (dev >= 0) {
    cudaGetDevice(&prev);
    if (prev != dev) GLMX_CUDA(cudaSetDevice(dev));
  }
}
DeviceGuard::~DeviceGuard() {
  int cur = -1;
  if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
}

void DBuf::reserve(size_t n) {
  if (n <= bytes) return;
  // cudaFree synchronises the whole device (it would stall the retrieval thread behind the
  // engine's forward): grow geometrically so steady-state batches never reallocate
  if (p) cudaFree(p);
  p = nullptr;
  n = std::max<size_t>(std::max<size_t>(n, 256), bytes + bytes / 2);
  bytes = 0;
  GLMX_CUDA(cudaMalloc(&p, n));
  bytes = n;
}
DBuf::~DBuf() {
  if (p) cudaFree(p);
}

glmx_kv::~glmx_kv() {
  for (auto& p : peers)
    if (p.ipc && p.base) cudaIpcCloseMemHandle(p.base);
  if (geom.base) cudaFree(geom.base);
  if (stream) cudaStreamDestroy(stream);
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
}

glmx_graph::~glmx_graph() {
  for (void* p : allocs) cudaFree(p);
  if (stream) cudaStreamDestroy(stream);
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
}

glmx_model::~glmx_model() {
  if (arena) cudaFree(arena);
  if (inv_freq) cudaFree(inv_freq);
  if (blas_ws) cudaFree(blas_ws);
  if (blas) cublasDestroy(blas);
}

glmx_engine::~glmx_engine() {
  for (auto& hp : h_ring)
    if (hp) cudaFreeHost(hp);
  for (auto& ev : ring_ev)
    if (ev) cudaEventDestroy(ev);
  if (h_dec) cudaFreeHost(h_dec);
  if (dec_done) cudaEventDestroy(dec_done);
  if (h_out) cudaFreeHost(h_out);
  if (h2d_done) cudaEventDestroy(h2d_done);
  if (fwd_done) cudaEventDestroy(fwd_done);
  for (auto e : ev_free) cudaEventDestroy(e);
  for (auto& sp : spans) {
    cudaEventDestroy(sp.a);
    cudaEventDestroy(sp.b);
  }
  for (auto e : done_ev)
    if (e) cudaEventDestroy(e);
  if (stream) cudaStreamDestroy(stream);
  if (m && --m->n_engines == 0 && m->destroy_pending) delete m;  // the model outlived its handle
}

// ======================================================================== graph upload
void glmx_graph::upload() {
  DeviceGuard g(device);
  auto put = [&](const void* src, size_t bytes) -> void* {
    void* p = nullptr;
    GLMX_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
    if (bytes && src) GLMX_CUDA(cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice));
    allocs.push_back(p);
    return p;
  };
  {
    // K1 reads entries as 16-byte words: pad the allocation past the last word
    std::vector<char> eb(host.entry_bytes.size() + 32, 0);
    std::memcpy(eb.data(), host.entry_bytes.data(), host.entry_bytes.size());
    dev.entry_bytes = static_cast<const char*>(put(eb.data(), eb.size()));
  }
  dev.entry_off = static_cast<const uint32_t*>(put(host.entry_off.data(), host.entry_off.size() * 4));
  for (size_t i = 0; i + 1 < host.entry_off.size(); ++i)
    max_entry = std::max(max_entry, host.entry_off[i + 1] - host.entry_off[i]);
  // the graph stream (K1 chunks, K5 RetrieveNode) runs beside the prefill at the lowest priority:
  // the forward's CTAs are dispatched first whenever an SM frees up
  stream = make_stream(false);
  {
    uint32_t* st = static_cast<uint32_t*>(put(nullptr, host.n() * 4));
    entry_stats(dev.entry_bytes, dev.entry_off, static_cast<uint32_t>(host.n()), st, stream);
    dev.ent_stat = st;
    // interior-token tables of the regular entries (K1 fast tokenizer)
    const uint32_t n = static_cast<uint32_t>(host.n());
    uint32_t* cnt = static_cast<uint32_t*>(put(nullptr, (n + 1) * 4));
    uint32_t* ioff = static_cast<uint32_t*>(put(nullptr, (n + 1) * 4));
    entry_interior_counts(st, n, cnt, stream);
    DBuf tmp;
    size_t tb = scan_u32_temp_bytes(n + 1);
    tmp.reserve(tb);
    scan_u32(tmp.p, tb, cnt, ioff, n + 1, stream);
    uint32_t n_int = 0;
    GLMX_CUDA(cudaMemcpyAsync(&n_int, ioff + n, 4, cudaMemcpyDeviceToHost, stream));
    GLMX_CUDA(cudaStreamSynchronize(stream));
    uint32_t* head = static_cast<uint32_t*>(put(nullptr, n * 4));
    uint32_t* tail = static_cast<uint32_t*>(put(nullptr, n * 4));
    uint64_t* tstate = static_cast<uint64_t*>(put(nullptr, n * 8));
    uint2* itok_span = static_cast<uint2*>(put(nullptr, static_cast<size_t>(n_int) * 8));
    uint64_t* itok_hash = static_cast<uint64_t*>(put(nullptr, static_cast<size_t>(n_int) * 8));
    entry_tokens(dev.entry_bytes, dev.entry_off, st, n, ioff, head, tail, tstate, itok_span,
                 itok_hash, stream);
    n_interior = n_int;
    // irregular entries (entry_regular in chunk.cu: >= 2 tokens, first and last byte non-space):
    // a graph without any never launches the byte-level chunk kernel
    std::vector<uint32_t> hst(n);
    GLMX_CUDA(cudaMemcpyAsync(hst.data(), st, static_cast<size_t>(n) * 4, cudaMemcpyDeviceToHost, stream));
    GLMX_CUDA(cudaStreamSynchronize(stream));  // before tmp (scan scratch) is released
    n_irregular = 0;
    for (uint32_t v : hst) n_irregular += ((v >> 29) == 7u && (v & 0x1FFFFFFFu) >= 2) ? 0u : 1u;
    dev.ent_head = head;
    dev.ent_tail = tail;
    dev.ent_tstate = tstate;
    dev.ent_ioff = ioff;
    dev.itok_span = itok_span;
    dev.itok_hash = itok_hash;
    dev.itok_id = nullptr;
    EntryRec* rec = static_cast<EntryRec*>(put(nullptr, static_cast<size_t>(n) * sizeof(EntryRec)));
    entry_records(dev.entry_off, head, tail, tstate, ioff, n, rec, stream);
    GLMX_CUDA(cudaStreamSynchronize(stream));
    dev.ent = rec;
  }
  if (host.und_off.empty()) {
    // GPU ingest (kernels/ingest.cu): CSRs and weights built on the device from the edge list
    DeviceCsr dc;
    build_graph_device(host.src.data(), host.dst.data(), host.etype.data(), host.src.size(),
                       static_cast<uint32_t>(host.n()), dc, host.w_total, stream);
    for (void* p : dc.allocs) allocs.push_back(p);
    dev.und_off = dc.und_off;
    dev.und_idx = dc.und_idx;
    dev.dir_off = dc.dir_off;
    dev.dir_idx = dc.dir_idx;
    dev.w_total = dc.w_total;
    dev.w_by_type = dc.w_by_type;
  } else {
    dev.und_off = static_cast<const uint32_t*>(put(host.und_off.data(), host.und_off.size() * 4));
    dev.und_idx = static_cast<const int32_t*>(put(host.und_idx.data(), host.und_idx.size() * 4));
    dev.dir_off = static_cast<const uint32_t*>(put(host.dir_off.data(), host.dir_off.size() * 4));
    dev.dir_idx = static_cast<const int32_t*>(put(host.dir_idx.data(), host.dir_idx.size() * 4));
    dev.w_total = static_cast<const int32_t*>(put(host.w_total.data(), host.w_total.size() * 4));
    dev.w_by_type = static_cast<const int32_t*>(put(host.w_by_type.data(), host.w_by_type.size() * 4));
  }
  dev.n = static_cast<uint32_t>(host.n());
  GLMX_CUDA(cudaEventCreate(&ev0));
  GLMX_CUDA(cudaEventCreate(&ev1));
  // K1 / K5 scratch for batches of up to 512 chunks of k <= 64 (~8 KB each) without reallocation
  constexpr size_t kChunks = 512, kBytes = kChunks * 8192, kTok = kBytes / 2 + kChunks + 1;
  d_nodes.reserve(kChunks * 4);
  d_cnt.reserve(kChunks * 4);
  d_off.reserve((kChunks + 1) * 8);
  d_toff.reserve((kChunks + 2) * 4);
  d_bytes.reserve(kBytes + 16);
  d_tid.reserve(kTok * 4);
  d_tbeg.reserve(kTok * 8);
  d_tend.reserve(kTok * 8);
  d_qemb.reserve(kChunks * 128 * 4);
  d_best.reserve(kChunks * 8);
}

// Ranked adjacency of one (weight mode, directed) variant: sorted once per graph on first use
// (a segmented sort of the CSR + three prefix scans; the graph is immutable).
glmx::RankedAdj glmx_graph::ranked_adj(int weight_mode, int directed) {
  Ranked& rk = ranked[(weight_mode ? 2 : 0) + (directed ? 1 : 0)];
  const uint32_t* off = directed ? dev.dir_off : dev.und_off;
  if (!rk.ready) {
    const uint32_t n = dev.n;
    uint32_t e32 = 0;
    GLMX_CUDA(cudaMemcpyAsync(&e32, off + n, 4, cudaMemcpyDeviceToHost, stream));
    GLMX_CUDA(cudaStreamSynchronize(stream));
    const uint64_t E = e32;
    DBuf keys, sorted, tmp32, temp;
    keys.reserve((E + 1) * 8);
    sorted.reserve(std::max<uint64_t>(E, 1) * 8);
    tmp32.reserve((E + 1) * 4);
    const size_t tb = rank_sort_temp_bytes(E, n);
    temp.reserve(std::max<size_t>(tb, 16));
    rk.ridx.reserve(std::max<uint64_t>(E, 1) * 4);
    rk.pbytes.reserve((E + 1) * 8);
    rk.ptoks.reserve((E + 1) * 4);
    rk.pirr.reserve((E + 1) * 4);
    rk.recs.reserve(std::max<uint64_t>(E, 1) * sizeof(glmx::EntryRec));
    rank_adjacency(dev, off, directed ? dev.dir_idx : dev.und_idx,
                   weight_mode ? dev.w_by_type : dev.w_total, E, n, temp.p, temp.bytes,
                   keys.as<uint64_t>(), sorted.as<uint64_t>(), rk.ridx.as<int32_t>(),
                   rk.pbytes.as<uint64_t>(), rk.ptoks.as<uint32_t>(), rk.pirr.as<uint32_t>(),
                   tmp32.as<uint32_t>(), rk.recs.as<glmx::EntryRec>(), stream);
    GLMX_CUDA(cudaStreamSynchronize(stream));  // before the scratch buffers are released
    rk.ready = true;
  }
  return glmx::RankedAdj{off, rk.ridx.as<int32_t>(), rk.recs.as<glmx::EntryRec>(), nullptr,
                         rk.pbytes.as<uint64_t>(), rk.ptoks.as<uint32_t>(), rk.pirr.as<uint32_t>()};
}

// K1 driver: lengths -> scans -> render + tokenize.  Returns GLMX_ERR_ARG (with totals) when the
// caller's buffers are too small.
int chunk_build_impl(glmx_graph* g, const glmx_chunk_config* cfg, const int32_t* node_idx,
                     uint64_t n, char* out_bytes, uint64_t bytes_cap, uint64_t* out_byte_offsets,
                     int32_t* out_tok_ids, uint64_t* out_tok_begin, uint64_t* out_tok_end,
                     uint64_t tok_cap, uint64_t* out_tok_offsets, uint64_t* total_bytes,
                     uint64_t* total_tokens) {
  NvtxRange nvtx_range("glmx.k1.chunk_build");
  if (g->device < 0) throw Error(GLMX_ERR_NO_DEVICE, "graph has no device");
  if (n == 0) {
    if (total_bytes) *total_bytes = 0;
    if (total_tokens) *total_tokens = 0;
    if (out_byte_offsets) out_byte_offsets[0] = 0;
    if (out_tok_offsets) out_tok_offsets[0] = 0;
    return GLMX_OK;
  }
  for (uint64_t i = 0; i < n; ++i)
    if (node_idx[i] < 0 || static_cast<uint64_t>(node_idx[i]) >= g->host.n())
      throw Error(GLMX_ERR_RETRIEVAL, "unknown node index " + std::to_string(node_idx[i]));
  const int k = std::max(cfg->k, 0);
  DeviceGuard dg(g->device);
  cudaStream_t s = g->stream;
  const bool same = g->k1_valid && out_bytes && g->k1_nodes.size() == n &&
                    g->k1_cfg.k == cfg->k && g->k1_cfg.weight_mode == cfg->weight_mode &&
                    g->k1_cfg.directed == cfg->directed && g->k1_cfg.vocab == cfg->vocab &&
                    std::memcmp(g->k1_nodes.data(), node_idx, n * 4) == 0;
  uint64_t total = 0, ntok = 0;
  if (same) {
    total = g->k1_total;
    ntok = g->k1_ntok;
  } else {
    g->k1_valid = false;
    glmx::RankedAdj ra = g->ranked_adj(cfg->weight_mode, cfg->directed);
    // per-node lengths for this k (one kernel over the nodes when k or the variant changes)
    const int64_t key = (static_cast<int64_t>(k) << 2) | (cfg->weight_mode ? 2 : 0) | (cfg->directed ? 1 : 0);
    if (g->lens_key != key) {
      g->d_lens.reserve(std::max<size_t>(g->dev.n, 1) * sizeof(uint4));
      chunk_len_table(g->dev, ra, k, g->d_lens.as<uint4>(), s);
      g->lens_key = key;
    }
    ra.lens = g->d_lens.as<uint4>();
    if (cfg->vocab && cfg->vocab != g->itok_vocab) {  // interior-token ids for this vocab
      g->d_itok_id.reserve(std::max<size_t>(g->n_interior, 1) * 4);
      chunk_token_ids(g->dev.itok_hash, g->n_interior, cfg->vocab, g->d_itok_id.as<uint32_t>(), s);
      g->dev.itok_id = g->d_itok_id.as<uint32_t>();
      g->itok_vocab = cfg->vocab;
    }
    g->d_nodes.reserve(n * 4);
    g->d_cnt.reserve(n * 4);
    g->d_off.reserve((n + 1) * 8);
    g->d_toff.reserve((n + 3) * 4);   // token offsets ([n] = total) + overflow flag + irregular count
    g->d_irr.reserve(n * 4);          // irregular chunks (byte-level tokenizer)
    g->d_vrow.reserve(n * 8);         // (node, ranked-row start) per chunk
    const int tiles = chunk_scan_tiles(static_cast<int>(n));
    if (g->d_scan.bytes < static_cast<size_t>(tiles) * 32) {
      g->d_scan.reserve(static_cast<size_t>(tiles) * 32);
      GLMX_CUDA(cudaMemsetAsync(g->d_scan.p, 0, g->d_scan.bytes, s));
      g->scan_epoch = 0;
    }
    const size_t cap_tiles = g->d_scan.bytes / 32;
    uint8_t* sb = g->d_scan.as<uint8_t>();
    const glmx::ScanState st{reinterpret_cast<uint64_t*>(sb), reinterpret_cast<uint64_t*>(sb + cap_tiles * 8),
                             reinterpret_cast<uint32_t*>(sb + cap_tiles * 16),
                             reinterpret_cast<uint32_t*>(sb + cap_tiles * 20),
                             reinterpret_cast<uint32_t*>(sb + cap_tiles * 24)};
    int32_t* overflow = reinterpret_cast<int32_t*>(g->d_toff.as<uint32_t>() + n + 1);
    int32_t* irr_count = overflow + 1;
    GLMX_CUDA(cudaMemcpyAsync(g->d_nodes.p, node_idx, n * 4, cudaMemcpyHostToDevice, s));
    g->h2d_bytes += n * 4;
    GLMX_CUDA(cudaMemsetAsync(overflow, 0, 8, s));
    GLMX_CUDA(cudaEventRecord(g->ev0, s));
    chunk_lengths_scan(g->dev, ra, k, g->d_nodes.as<int32_t>(), static_cast<int>(n),
                       g->d_cnt.as<int32_t>(), g->d_off.as<uint64_t>(), g->d_toff.as<uint32_t>(), st,
                       ++g->scan_epoch, g->d_irr.as<int32_t>(), irr_count, g->d_vrow.as<int2>(), s);
    // The render goes straight on with the output buffers as they are (no host round trip): a
    // batch that does not fit raises the device overflow flag, and is rendered again below into
    // buffers grown to its totals.  Small batches are sized from a bound up front.
    const uint64_t bound = n * (21 + static_cast<uint64_t>(k + 1) * (g->max_entry + 3));
    if (bound <= (64ull << 20)) {
      // a token has >= 1 byte and is followed by a space or the chunk end: <= total/2 + n tokens
      g->d_bytes.reserve(bound + 16);
      g->d_tid.reserve((bound / 2 + n + 1) * 4);
      g->d_tbeg.reserve((bound / 2 + n + 1) * 8);
      g->d_tend.reserve((bound / 2 + n + 1) * 8);
    }
    auto render = [&] {
      const uint64_t tok_cap = std::min(g->d_tid.bytes / 4, std::min(g->d_tbeg.bytes, g->d_tend.bytes) / 8);
      chunk_render_emit(g->dev, ra, g->d_nodes.as<int32_t>(), static_cast<int>(n),
                        g->d_cnt.as<int32_t>(), g->d_off.as<uint64_t>(), g->d_toff.as<uint32_t>(),
                        cfg->vocab, g->d_bytes.as<char>(), g->d_tid.as<int32_t>(),
                        g->d_tbeg.as<uint64_t>(), g->d_tend.as<uint64_t>(),
                        g->d_bytes.bytes >= 16 ? g->d_bytes.bytes - 16 : 0, tok_cap, overflow,
                        g->n_irregular ? g->d_irr.as<int32_t>() : nullptr, irr_count,
                        g->d_vrow.as<int2>(), s);
    };
    render();
    GLMX_CUDA(cudaEventRecord(g->ev1, s));
    uint64_t total32 = 0;
    uint32_t ntok32 = 0;
    int32_t ovf = 0;
    GLMX_CUDA(cudaMemcpyAsync(&total32, g->d_off.as<uint64_t>() + n, 8, cudaMemcpyDeviceToHost, s));
    GLMX_CUDA(cudaMemcpyAsync(&ntok32, g->d_toff.as<uint32_t>() + n, 4, cudaMemcpyDeviceToHost, s));
    GLMX_CUDA(cudaMemcpyAsync(&ovf, overflow, 4, cudaMemcpyDeviceToHost, s));
    GLMX_CUDA(cudaStreamSynchronize(s));
    g->d2h_bytes += 16;
    if (ovf) {
      g->d_bytes.reserve(total32 + total32 / 4 + 16);
      g->d_tid.reserve((ntok32 + ntok32 / 4 + 1) * 4ull);
      g->d_tbeg.reserve((ntok32 + ntok32 / 4 + 1) * 8ull);
      g->d_tend.reserve((ntok32 + ntok32 / 4 + 1) * 8ull);
      render();  // the timed span (ev0 .. ev1) then covers the first attempt and this one
      GLMX_CUDA(cudaEventRecord(g->ev1, s));
      GLMX_CUDA(cudaStreamSynchronize(s));
    }
    GLMX_CUDA(cudaEventElapsedTime(&g->last_ms, g->ev0, g->ev1));
    total = total32;
    ntok = ntok32;
    g->k1_nodes.assign(node_idx, node_idx + n);
    g->k1_cfg = *cfg;
    g->k1_total = total;
    g->k1_ntok = ntok;
    g->k1_valid = true;
  }
  if (total_bytes) *total_bytes = total;
  if (total_tokens) *total_tokens = ntok;
  if (!out_bytes) return GLMX_OK;
  if (bytes_cap < total || (tok_cap < ntok && (out_tok_ids || out_tok_begin || out_tok_end)))
    throw Error(GLMX_ERR_ARG, "chunk output buffers too small");
  GLMX_CUDA(cudaMemcpyAsync(out_bytes, g->d_bytes.p, total, cudaMemcpyDeviceToHost, s));
  g->d2h_bytes += total;
  if (out_byte_offsets) {
    GLMX_CUDA(cudaMemcpyAsync(out_byte_offsets, g->d_off.p, (n + 1) * 8, cudaMemcpyDeviceToHost, s));
    g->d2h_bytes += (n + 1) * 8;
  }
  if (out_tok_ids && cfg->vocab) {
    GLMX_CUDA(cudaMemcpyAsync(out_tok_ids, g->d_tid.p, ntok * 4, cudaMemcpyDeviceToHost, s));
    g->d2h_bytes += ntok * 4;
  }
  if (out_tok_begin) {
    GLMX_CUDA(cudaMemcpyAsync(out_tok_begin, g->d_tbeg.p, ntok * 8, cudaMemcpyDeviceToHost, s));
    g->d2h_bytes += ntok * 8;
  }
  if (out_tok_end) {
    GLMX_CUDA(cudaMemcpyAsync(out_tok_end, g->d_tend.p, ntok * 8, cudaMemcpyDeviceToHost, s));
    g->d2h_bytes += ntok * 8;
  }
  std::vector<uint32_t> toff32(out_tok_offsets ? n + 1 : 0);
  if (out_tok_offsets) {
    GLMX_CUDA(cudaMemcpyAsync(toff32.data(), g->d_toff.p, (n + 1) * 4, cudaMemcpyDeviceToHost, s));
    g->d2h_bytes += (n + 1) * 4;
  }
  GLMX_CUDA(cudaStreamSynchronize(s));
  if (out_tok_offsets)
    for (uint64_t i = 0; i <= n; ++i) out_tok_offsets[i] = toff32[i];
  return GLMX_OK;
}

// ======================================================================== KV
glmx_kv* kv_create_impl(const glmx_kv_config* cfg) {
  auto kv = std::make_unique<glmx_kv>();
  kv->cfg = *cfg;
  uint64_t pages = cfg->capacity_blocks + cfg->headroom_pages;
  if (cfg->device < 0) {
    // bookkeeping only: pages are logical handles; deferred pages recycle on every call
    pages = std::max<uint64_t>(pages, cfg->capacity_blocks + 1024);
  }
  if (pages > 0x7FFFFFFFULL) throw Error(GLMX_ERR_ARG, "too many pages");
  kv->bk = std::make_unique<BlockEngine>(cfg->capacity_blocks, cfg->block_tokens, cfg->policy, pages);
  if (cfg->device >= 0) {
    if (cfg->n_layers == 0 || cfg->n_kv_heads == 0 || cfg->head_dim == 0)
      throw Error(GLMX_ERR_ARG, "device pool needs n_layers, n_kv_heads, head_dim");
    DeviceGuard g(cfg->device);
    kv->geom.n_layers = cfg->n_layers;
    kv->geom.n_kv_heads = cfg->n_kv_heads;
    kv->geom.block_tokens = cfg->block_tokens;
    kv->geom.head_dim = cfg->head_dim;
    kv->page_bytes = kv->geom.page_elems() * sizeof(__nv_bfloat16);
    void* base = nullptr;
    GLMX_CUDA(cudaMalloc(&base, pages * kv->page_bytes));
    GLMX_CUDA(cudaMemset(base, 0, pages * kv->page_bytes));
    kv->geom.base = static_cast<__nv_bfloat16*>(base);
    GLMX_CUDA(cudaStreamCreateWithFlags(&kv->stream, cudaStreamNonBlocking));
    GLMX_CUDA(cudaEventCreate(&kv->ev0));
    GLMX_CUDA(cudaEventCreate(&kv->ev1));
  }
  return kv.release();
}

void pool_copy_impl(glmx_kv* src, glmx_kv* dst, const int32_t* sp, const int32_t* dp, uint64_t n,
                    cudaStream_t s) {
  NvtxRange nvtx_range("glmx.k4.pool_copy");
  if (!src->has_pool() || !dst->has_pool()) throw Error(GLMX_ERR_NO_DEVICE, "pool copy needs device pools");
  if (src->page_bytes != dst->page_bytes) throw Error(GLMX_ERR_ARG, "pool geometries differ");
  for (uint64_t i = 0; i < n; ++i)
    if (sp[i] < 0 || static_cast<uint64_t>(sp[i]) >= src->bk->pool().total() || dp[i] < 0 ||
        static_cast<uint64_t>(dp[i]) >= dst->bk->pool().total())
      throw Error(GLMX_ERR_ARG, "page index out of range");
  DeviceGuard g(dst->cfg.device);
  if (src->cfg.device != dst->cfg.device) {
    cudaError_t e = cudaDeviceEnablePeerAccess(src->cfg.device, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
      throw Error(GLMX_ERR_CUDA, std::string("peer access: ") + cudaGetErrorString(e));
    cudaGetLastError();
  }
  if (!s) s = dst->stream;
  dst->scratch.reserve(n * 8);
  GLMX_CUDA(cudaMemcpyAsync(dst->scratch.p, sp, n * 4, cudaMemcpyHostToDevice, s));
  GLMX_CUDA(cudaMemcpyAsync(dst->scratch.as<int32_t>() + n, dp, n * 4, cudaMemcpyHostToDevice, s));
  GLMX_CUDA(cudaEventRecord(dst->ev0, s));
  for (uint64_t o = 0; o < n; o += 65535)
    pool_copy_pages(src->geom.base, dst->geom.base, dst->geom.page_elems(),
                    dst->scratch.as<int32_t>() + o, dst->scratch.as<int32_t>() + n + o,
                    static_cast<int>(std::min<uint64_t>(65535, n - o)), s);
  GLMX_CUDA(cudaEventRecord(dst->ev1, s));
  GLMX_CUDA(cudaEventSynchronize(dst->ev1));
  GLMX_CUDA(cudaEventElapsedTime(&dst->last_copy_ms, dst->ev0, dst->ev1));
}

// ======================================================================== model
glmx_model* model_create_impl(const glmx_model_config* c, int device) {
  if (device < 0) throw Error(GLMX_ERR_NO_DEVICE, "model needs a CUDA device");
  if (c->n_heads % c->n_kv_heads || c->d_model % 8 || c->head_dim != 128)
    throw Error(GLMX_ERR_ARG, "unsupported model shape");
  auto m = std::make_unique<glmx_model>();
  m->cfg = *c;
  m->device = device;
  DeviceGuard g(device);
  const uint64_t d = c->d_model, hd = c->head_dim, H = c->n_heads, Hkv = c->n_kv_heads,
                 ff = c->d_ff, V = c->vocab, L = c->n_layers;
  const uint64_t qkv = (H + 2 * Hkv) * hd;
  const uint64_t per_layer = d + qkv * d + d * H * hd + d + 2 * ff * d + d * ff;
  const uint64_t total = V * d + L * per_layer + d + V * d;
  m->arena_bytes = total * sizeof(__nv_bfloat16);
  GLMX_CUDA(cudaMalloc(&m->arena, m->arena_bytes + 256));
  __nv_bfloat16* p = static_cast<__nv_bfloat16*>(m->arena);
  auto take = [&](uint64_t n) {
    __nv_bfloat16* r = p;
    p += n;
    return r;
  };
  uint64_t tid = 0;
  auto seed_of = [&](uint64_t t) { return mix64(c->seed * 0x100000001b3ULL + t); };
  m->embed = take(V * d);
  init_normal_bf16(m->embed, V * d, seed_of(tid++), c->init_std, 0);
  m->layers.resize(L);
  for (uint64_t l = 0; l < L; ++l) {
    LayerW& w = m->layers[l];
    w.attn_norm = take(d);
    init_const_bf16(w.attn_norm, d, 1.0f, 0);
    w.wqkv = take(qkv * d);
    init_normal_bf16(w.wqkv, qkv * d, seed_of(tid++), c->init_std, 0);
    w.wo = take(d * H * hd);
    init_normal_bf16(w.wo, d * H * hd, seed_of(tid++), c->init_std, 0);
    w.mlp_norm = take(d);
    init_const_bf16(w.mlp_norm, d, 1.0f, 0);
    w.wgu = take(2 * ff * d);
    init_normal_bf16(w.wgu, 2 * ff * d, seed_of(tid++), c->init_std, 0);
    w.wdown = take(d * ff);
    init_normal_bf16(w.wdown, d * ff, seed_of(tid++), c->init_std, 0);
  }
  m->final_norm = take(d);
  init_const_bf16(m->final_norm, d, 1.0f, 0);
  m->lm_head = take(V * d);
  init_normal_bf16(m->lm_head, V * d, seed_of(tid++), c->init_std, 0);
  // RoPE inverse frequencies in double, rounded once (the oracle uses the same table).
  std::vector<float> inv(hd / 2);
  for (uint64_t i = 0; i < hd / 2; ++i)
    inv[i] = static_cast<float>(1.0 / std::pow(static_cast<double>(c->rope_theta),
                                               static_cast<double>(2 * i) / static_cast<double>(hd)));
  GLMX_CUDA(cudaMalloc(&m->inv_freq, inv.size() * 4));
  GLMX_CUDA(cudaMemcpy(m->inv_freq, inv.data(), inv.size() * 4, cudaMemcpyHostToDevice));
  GLMX_BLAS(cublasCreate(&m->blas));
  GLMX_CUDA(cudaMalloc(&m->blas_ws, kBlasWsBytes));
  GLMX_BLAS(cublasSetWorkspace(m->blas, m->blas_ws, kBlasWsBytes));
  GLMX_CUDA(cudaDeviceSynchronize());
  return m.release();
}

int model_export_impl(const glmx_model* m, int which, int layer, uint16_t* out, uint64_t n) {
  const auto& c = m->cfg;
  const uint64_t d = c.d_model, hd = c.head_dim, H = c.n_heads, Hkv = c.n_kv_heads, ff = c.d_ff,
                 V = c.vocab;
  const __nv_bfloat16* src = nullptr;
  uint64_t cnt = 0;
  if (which != 0 && which != 7 && which != 8 && (layer < 0 || layer >= static_cast<int>(c.n_layers)))
    throw Error(GLMX_ERR_ARG, "layer out of range");
  switch (which) {
    case 0: src = m->embed; cnt = V * d; break;
    case 1: src = m->layers[layer].attn_norm; cnt = d; break;
    case 2: src = m->layers[layer].wqkv; cnt = (H + 2 * Hkv) * hd * d; break;
    case 3: src = m->layers[layer].wo; cnt = d * H * hd; break;
    case 4: src = m->layers[layer].mlp_norm; cnt = d; break;
    case 5: src = m->layers[layer].wgu; cnt = 2 * ff * d; break;
    case 6: src = m->layers[layer].wdown; cnt = d * ff; break;
    case 7: src = m->final_norm; cnt = d; break;
    case 8: src = m->lm_head; cnt = V * d; break;
    default: throw Error(GLMX_ERR_ARG, "unknown weight");
  }
  if (n < cnt) throw Error(GLMX_ERR_ARG, "export buffer too small");
  DeviceGuard g(m->device);
  GLMX_CUDA(cudaMemcpy(out, src, cnt * 2, cudaMemcpyDeviceToHost));
  return GLMX_OK;
}

// Times the projection GEMMs' algorithm candidates per M bucket (host/gemm_tune.hpp) on layer
// 0's weights and random activations; T <= 128 (decode rows) stays with cublasGemmEx.
int model_tune_gemms_impl(glmx_model* m, int max_tokens) {
  if (m->n_engines > 0)
    throw Error(GLMX_ERR_ARG, "tune the GEMMs before creating engines (the table is read by every forward)");
  if (max_tokens <= 128) return 0;
  DeviceGuard g(m->device);
  const auto& c = m->cfg;
  const uint64_t d = c.d_model, hd = c.head_dim, H = c.n_heads, Hkv = c.n_kv_heads, ff = c.d_ff;
  struct P {
    int shape;
    const __nv_bfloat16* w;
    int in, out;
    bool fp32, acc;
  };
  const LayerW& w = m->layers.at(0);
  const P ps[kGemmShapes] = {
      {kGemmQKV, w.wqkv, int(d), int((H + 2 * Hkv) * hd), false, false},
      {kGemmO, w.wo, int(H * hd), int(d), true, true},
      {kGemmGU, w.wgu, int(d), int(2 * ff), false, false},
      {kGemmDown, w.wdown, int(ff), int(d), true, true}};
  const int nb = GemmTuner::bucket(max_tokens) + 1;
  const uint64_t T = static_cast<uint64_t>(GemmTuner::bucket_hi(nb - 1));
  uint64_t x_elems = 0, y_bytes = 0;
  for (const P& p : ps) {
    x_elems = std::max<uint64_t>(x_elems, T * p.in);
    y_bytes = std::max<uint64_t>(y_bytes, T * p.out * (p.fp32 ? 4 : 2));
  }
  __nv_bfloat16* X = nullptr;
  void* Y = nullptr;
  GLMX_CUDA(cudaMalloc(&X, x_elems * 2));
  cudaError_t ye = cudaMalloc(&Y, y_bytes);
  if (ye != cudaSuccess) {
    cudaFree(X);
    GLMX_CUDA(ye);
  }
  int n = 0;
  try {
    // random operands: all-zero inputs draw less power and would favour the wrong candidates
    init_normal_bf16(X, x_elems, 0x7e57u, 1.0f, 0);
    GLMX_CUDA(cudaMemset(Y, 0, y_bytes));
    for (int b = 1; b < nb; ++b)
      for (const P& p : ps)
        n += m->tuner.tune(p.shape, b, m->blas, 0, X, p.w, Y, p.fp32, p.acc, p.in, p.out,
                           m->blas_ws, kBlasWsBytes);
    GLMX_CUDA(cudaDeviceSynchronize());
  } catch (...) {
    cudaFree(X);
    cudaFree(Y);
    throw;
  }
  cudaFree(X);
  cudaFree(Y);
  return n;
}

// ======================================================================== engine
namespace {

// Y[T][out] (+)= X[T][in] * W[out][in]^T  (column-major: C(out x T) = W^T' * X); `shape` names
// the projection for the tuned algorithm table (host/gemm_tune.hpp), -1 = always cublasGemmEx
// (the workspace is the calling engine's: engines sharing a model run on their own streams)
void gemm(glmx_engine* e, int shape, const __nv_bfloat16* X, const __nv_bfloat16* W, void* Y,
          bool y_fp32, bool accumulate, int T, int in, int out) {
  if (T <= 0) return;
  glmx_model* m = e->m;
  cudaStream_t s = e->stream;
  if (shape >= 0 && m->tuner.run(shape, s, X, W, Y, y_fp32, accumulate, T, in, out, e->blas_ws.p,
                                 kBlasWsBytes))
    return;
  cublasHandle_t h = m->blas;
  GLMX_BLAS(cublasSetStream(h, s));
  GLMX_BLAS(cublasSetWorkspace(h, e->blas_ws.p, kBlasWsBytes));
  const float alpha = 1.f, beta = accumulate ? 1.f : 0.f;
  GLMX_BLAS(cublasGemmEx(h, CUBLAS_OP_T, CUBLAS_OP_N, out, T, in, &alpha, W, CUDA_R_16BF, in, X,
                         CUDA_R_16BF, in, &beta, Y, y_fp32 ? CUDA_R_32F : CUDA_R_16BF, out,
                         CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT));
}

cudaEvent_t next_event(glmx_engine* e) {
  if (e->ev_free.empty()) {
    cudaEvent_t ev;
    GLMX_CUDA(cudaEventCreate(&ev));
    return ev;
  }
  cudaEvent_t ev = e->ev_free.back();
  e->ev_free.pop_back();
  return ev;
}

// A kernel group of the forward: an NVTX range (host-side enqueue; an NVTX-aware profiler maps
// the group's kernels to it) and, when profiling, a CUDA event pair on the engine stream.
struct Prof {
  glmx_engine* e;
  int cat;
  cudaEvent_t a = nullptr;
  // profiling 1: whole forward + copies only; 2: every kernel category
  Prof(glmx_engine* e_, int c) : e(e_), cat(c) {
    static const char* const kNames[] = {"glmx.forward", "glmx.attention", "glmx.kv_append",
                                         "glmx.gemm", "glmx.elementwise", "glmx.h2d", "glmx.d2h"};
    nvtxRangePushA(kNames[c]);
    if (e->profiling >= 2 || (e->profiling == 1 && (c == 0 || c >= 5))) {
      a = next_event(e);
      GLMX_CUDA(cudaEventRecord(a, e->stream));
    }
  }
  ~Prof() {
    if (a) {
      cudaEvent_t b = next_event(e);
      cudaEventRecord(b, e->stream);
      e->spans.push_back({a, b, cat, e->prof_tag ? e->prof_tag : e->batch_seq});
    }
    nvtxRangePop();
  }
};

enum { kCatAll = 0, kCatAttn = 1, kCatAppend = 2, kCatGemm = 3, kCatOther = 4, kCatH2D = 5, kCatD2H = 6 };

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

}  // namespace

glmx_engine* engine_create_impl(glmx_model* m, glmx_kv* kv, const glmx_engine_config* cfg) {
  if (!kv->has_pool()) throw Error(GLMX_ERR_NO_DEVICE, "engine needs a device KV pool");
  if (kv->cfg.device != m->device) throw Error(GLMX_ERR_ARG, "model and kv on different devices");
  const auto& c = m->cfg;
  if (kv->cfg.n_layers != c.n_layers || kv->cfg.n_kv_heads != c.n_kv_heads ||
      kv->cfg.head_dim != c.head_dim)
    throw Error(GLMX_ERR_ARG, "kv pool geometry does not match the model");
  auto e = std::make_unique<glmx_engine>();
  e->m = m;
  ++m->n_engines;  // (the destructor undoes it)
  e->kv = kv;
  e->cfg = *cfg;
  DeviceGuard g(m->device);
  e->stream = make_stream(true);  // the forward outranks the graph stream
  e->blas_ws.reserve(kBlasWsBytes);
  GLMX_CUDA(cudaEventCreateWithFlags(&e->h2d_done, cudaEventDisableTiming));
  GLMX_CUDA(cudaEventCreateWithFlags(&e->fwd_done, cudaEventDisableTiming));
  // decode steps may merge two batches' rows (deferred decode): row buffers hold 2 x max_requests
  const uint64_t T = std::max<uint32_t>(cfg->max_batch_tokens, 2 * cfg->max_requests);
  const uint64_t R = 2ull * cfg->max_requests;
  const uint64_t d = c.d_model, hd = c.head_dim, H = c.n_heads, Hkv = c.n_kv_heads, ff = c.d_ff;
  const uint32_t B = kv->cfg.block_tokens;
  // block-table rows padded to a multiple of 8 pages: K3 reads a key tile's 8 entries with two
  // 16-byte loads
  e->bt_stride = static_cast<int>(align_up((cfg->max_context + B - 1) / B + 1, 8));
  e->tpt = attn_tc_tokens_per_tile(static_cast<int>(H), static_cast<int>(Hkv));
  make_pool_tensor_map(kv->geom, kv->bk->pool().total(), e->kv_map, &e->kv_rows);
  e->x.reserve(T * d * 4);
  e->h.reserve(T * d * 2);
  e->qkv.reserve(T * (H + 2 * Hkv) * hd * 2);
  e->q.reserve(T * H * hd * 2);
  e->rope_cs.reserve(T * (hd / 2) * sizeof(float2));
  make_q_tensor_map(e->q.p, T, static_cast<int>(H), static_cast<int>(Hkv), e->q_map);
  e->attn.reserve(T * H * hd * 2);
  e->gu.reserve(T * 2 * ff * 2);
  e->act.reserve(T * ff * 2);
  e->hl.reserve(R * d * 2);
  e->logits.reserve(R * c.vocab * 4);
  e->next_tok.reserve((R * (cfg->max_decode + 1) + 16) * 4);
  e->amax_keys.reserve(R * 8 + 64);
  // metadata layout (one pinned block, one H2D)
  const uint64_t max_work = T / e->tpt + R;  // attention work items: sum of ceil(q_len / tpt)
  size_t o = 0;
  e->o_tok = o; o = align_up(o + T * 4, 256);
  e->o_pos = o; o = align_up(o + T * 4, 256);
  e->o_slot = o; o = align_up(o + T * 8, 256);
  e->o_qs = o; o = align_up(o + R * 4, 256);
  e->o_ql = o; o = align_up(o + R * 4, 256);
  e->o_ctx = o; o = align_up(o + R * 4, 256);
  e->o_bt = o; o = align_up(o + R * e->bt_stride * 4, 256);
  e->o_work = o; o = align_up(o + max_work * 8, 256);
  e->o_last = o; o = align_up(o + R * 4, 256);
  e->o_perm = o; o = align_up(o + R * 4, 256);
  e->o_sched = o;
  o = align_up(o + attn_sched_bytes(static_cast<int>(max_work * Hkv), kNumSMs, &e->o_sc_pieces,
                                    &e->o_sc_cta, &e->o_sc_comb, &e->o_sc_part), 256);
  e->part_o.reserve(static_cast<size_t>(2 * kNumSMs) * attn_tc_partial_rows() * hd * 4);
  e->part_ml.reserve(static_cast<size_t>(2 * kNumSMs) * attn_tc_partial_rows() * 8);
  e->max_copies = T / B + R + 16;  // peer page copies per batch (src, dst int32 each)
  e->o_copy = o; o = align_up(o + e->max_copies * 8, 256);
  e->meta_bytes = o;
  e->meta.reserve(o);
  for (int i = 0; i < glmx_engine::kMetaRing; ++i) {
    GLMX_CUDA(cudaMallocHost(&e->h_ring[i], o));
    GLMX_CUDA(cudaEventCreateWithFlags(&e->ring_ev[i], cudaEventDisableTiming));
  }
  e->h_meta = e->h_ring[0];
  GLMX_CUDA(cudaMallocHost(reinterpret_cast<void**>(&e->h_dec), (R * (cfg->max_decode + 1) + 16) * 4));
  GLMX_CUDA(cudaEventCreateWithFlags(&e->dec_done, cudaEventDisableTiming));
  e->dec_in.reserve(R * 4 + 64);
  e->def_first.reserve(R * 4 + 64);
  e->h_out_stride = R * (cfg->max_decode + 1) + 16;
  GLMX_CUDA(cudaMallocHost(reinterpret_cast<void**>(&e->h_out), 2 * e->h_out_stride * 4));
  for (auto& ev : e->done_ev) GLMX_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  return e.release();
}

namespace {

// One-token batches (decode steps) take the CUDA-core decode kernel: returns its split count, or
// 0 when the batch has a longer row (prefill) or the geometry is not the kernel's (G != 4).
int choose_decode_split(glmx_engine* e, int R, int T, const int32_t* ctx_len) {
  if (R <= 0 || T != R) return 0;
  const auto& c = e->m->cfg;
  if (c.n_heads != 4 * c.n_kv_heads || c.head_dim != 128 || e->kv->cfg.block_tokens != 16) return 0;
  int max_ctx = 0;
  for (int r = 0; r < R; ++r) max_ctx = std::max(max_ctx, ctx_len[r]);
  return decode_attention_splits(R * static_cast<int>(c.n_kv_heads), max_ctx,
                                 2 * kNumSMs * attn_tc_partial_rows());
}

// Next pinned staging slot (waits until that slot's previous upload has been consumed).
uint8_t* meta_acquire(glmx_engine* e) {
  e->ring_slot = (e->ring_slot + 1) % glmx_engine::kMetaRing;
  GLMX_CUDA(cudaEventSynchronize(e->ring_ev[e->ring_slot]));
  e->h_meta = e->h_ring[e->ring_slot];
  return static_cast<uint8_t*>(e->h_meta);
}
// Used sizes of the staged sections (rows, requests, work items, schedule, peer copies) and the
// batch's block-table stride (a multiple of 8 entries: K3 reads a key tile's 8 pages as 2 x 16 B).
struct MetaCounts {
  int n_tok = 0;  // token ids (prefill; decode steps read their input tokens on the device)
  int T = 0, R = 0, n_work = 0, n_perm = 0, n_copy = 0, bt_stride = 8;
  bool sched = false;  // the K3 schedule was staged (prefill-shaped batch)
};

// Packs the used part of every section of the current slot in place (sections keep their
// order, so a section's packed offset never exceeds its staging offset and forward memmoves are
// safe; block-table rows move from the capacity stride to the batch stride) and uploads exactly
// those bytes to the device metadata buffer, stream-ordered after the previous batch's kernels.
void meta_commit(glmx_engine* e, cudaStream_t s, const MetaCounts& n) {
  uint8_t* hm = static_cast<uint8_t*>(e->h_meta);
  glmx_engine::MetaLayout L{};
  size_t o = 0;
  auto put = [&](size_t src, size_t bytes) {
    const size_t dst = o;
    if (bytes && dst != src) std::memmove(hm + dst, hm + src, bytes);
    o = align_up(o + bytes, 16);
    return dst;
  };
  L.tok = put(e->o_tok, static_cast<size_t>(n.n_tok) * 4);
  L.pos = put(e->o_pos, static_cast<size_t>(n.T) * 4);
  L.slot = put(e->o_slot, static_cast<size_t>(n.T) * 8);
  L.qs = put(e->o_qs, static_cast<size_t>(n.R) * 4);
  L.ql = put(e->o_ql, static_cast<size_t>(n.R) * 4);
  L.ctx = put(e->o_ctx, static_cast<size_t>(n.R) * 4);
  L.bt = o;
  L.bt_stride = n.bt_stride;
  const size_t row = static_cast<size_t>(n.bt_stride) * 4;
  for (int r = 0; r < n.R; ++r) {
    const size_t src = e->o_bt + static_cast<size_t>(r) * e->bt_stride * 4;
    if (L.bt + r * row != src) std::memmove(hm + L.bt + r * row, hm + src, row);
  }
  o = align_up(o + n.R * row, 16);
  L.work = put(e->o_work, static_cast<size_t>(n.n_work) * 8);
  L.last = put(e->o_last, static_cast<size_t>(n.R) * 4);
  L.perm = put(e->o_perm, static_cast<size_t>(n.n_perm) * 4);
  const size_t sp = n.sched ? static_cast<size_t>(e->sc_npieces) * sizeof(AttnPiece) : 0;
  L.pieces = put(e->o_sched + e->o_sc_pieces, sp);
  L.partners = put(e->o_sched + e->o_sc_part, sp);
  L.cta = put(e->o_sched + e->o_sc_cta, n.sched ? static_cast<size_t>(e->sc_grid + 1) * 4 : 0);
  L.comb = put(e->o_sched + e->o_sc_comb, n.sched ? static_cast<size_t>(e->sc_ncomb) * sizeof(AttnCombine) : 0);
  L.copy = put(e->o_copy, static_cast<size_t>(n.n_copy) * 8);
  L.bytes = o;
  e->ml = L;
  GLMX_CUDA(cudaMemcpyAsync(e->meta.p, hm, o, cudaMemcpyHostToDevice, s));
  e->h2d_bytes += o;
  GLMX_CUDA(cudaEventRecord(e->ring_ev[e->ring_slot], s));
  GLMX_CUDA(cudaEventRecord(e->h2d_done, s));
}

// Packs the K3 stream-K schedule of the staged work list into the host metadata block.
void stage_attn_schedule(glmx_engine* e, uint8_t* hm, const int2* work, int n_work,
                         const int32_t* q_len, const int32_t* ctx_len) {
  AttnSchedule sc;
  sc.pieces = reinterpret_cast<AttnPiece*>(hm + e->o_sched + e->o_sc_pieces);
  sc.cta_off = reinterpret_cast<int32_t*>(hm + e->o_sched + e->o_sc_cta);
  sc.combine = reinterpret_cast<AttnCombine*>(hm + e->o_sched + e->o_sc_comb);
  sc.partners = reinterpret_cast<AttnPiece*>(hm + e->o_sched + e->o_sc_part);
  build_attn_schedule(reinterpret_cast<const int32_t*>(work), n_work,
                      static_cast<int>(e->m->cfg.n_kv_heads), q_len, ctx_len, e->tpt, 128,
                      kNumSMs, sc);
  e->sc_grid = sc.grid;
  e->sc_ncomb = sc.n_combine;
  e->sc_npieces = sc.n_pieces;
}

// Runs the decoder over the staged batch: T rows (tokens/pos/slot), R requests (attention
// metadata), n_last rows whose final hidden states produce logits + greedy tokens.
void forward(glmx_engine* e, int T, int R, int n_work, int n_last, const int32_t* d_tokens) {
  glmx_model* m = e->m;
  const auto& c = m->cfg;
  const int d = c.d_model, hd = c.head_dim, H = c.n_heads, Hkv = c.n_kv_heads, ff = c.d_ff;
  const int QKV = (H + 2 * Hkv) * hd;
  cudaStream_t s = e->stream;
  uint8_t* meta = e->meta.as<uint8_t>();
  const glmx_engine::MetaLayout& ml = e->ml;
  const int32_t* pos = reinterpret_cast<const int32_t*>(meta + ml.pos);
  const int64_t* slot = reinterpret_cast<const int64_t*>(meta + ml.slot);
  AttnParams ap{};
  ap.q = e->q.as<__nv_bfloat16>();
  ap.o = e->attn.as<__nv_bfloat16>();
  ap.pool = e->kv->geom;
  ap.q_start = reinterpret_cast<const int32_t*>(meta + ml.qs);
  ap.q_len = reinterpret_cast<const int32_t*>(meta + ml.ql);
  ap.ctx_len = reinterpret_cast<const int32_t*>(meta + ml.ctx);
  ap.block_table = reinterpret_cast<const int32_t*>(meta + ml.bt);
  ap.bt_stride = ml.bt_stride;
  ap.work = reinterpret_cast<const int2*>(meta + ml.work);
  ap.n_work = n_work;
  ap.H = H;
  ap.Hkv = Hkv;
  ap.scale_log2 = static_cast<float>(1.0 / std::sqrt(static_cast<double>(hd)) * 1.4426950408889634);
  (void)R;
  AttnTcSched sc{reinterpret_cast<const int4*>(meta + ml.pieces),
                 reinterpret_cast<const int*>(meta + ml.cta),
                 reinterpret_cast<const int4*>(meta + ml.comb),
                 e->sc_grid, e->sc_ncomb, e->part_o.as<float>(), e->part_ml.as<float2>(),
                 reinterpret_cast<const int4*>(meta + ml.partners)};
  Prof all(e, kCatAll);
  {
    Prof p(e, kCatOther);
    embed_gather(d_tokens, T, m->embed, d, e->x.as<float>(), s);
    rope_table(pos, T, static_cast<int>(hd / 2), m->inv_freq, e->rope_cs.as<float2>(), s);
  }
  for (uint32_t l = 0; l < c.n_layers; ++l) {
    const LayerW& w = m->layers[l];
    {
      Prof p(e, kCatOther);
      rmsnorm(e->x.as<float>(), nullptr, T, d, w.attn_norm, c.norm_eps, e->h.as<__nv_bfloat16>(), s);
    }
    {
      Prof p(e, kCatGemm);
      gemm(e, kGemmQKV, e->h.as<__nv_bfloat16>(), w.wqkv, e->qkv.p, false, false, T, d, QKV);
    }
    // decode rows with the fused kernel: RoPE + K/V append happen inside the decode attention
    const bool fuse = e->dec_split > 0;
    if (!fuse) {
      Prof p(e, kCatAppend);
      rope_kv_append(e->qkv.as<__nv_bfloat16>(), pos, slot, T, H, Hkv, hd, m->inv_freq,
                     e->rope_cs.as<float2>(), e->kv->geom, l, e->q.as<__nv_bfloat16>(), s);
    }
    {
      Prof p(e, kCatAttn);
      ap.layer = l;
      if (fuse)
        paged_attention_decode_rope(ap, DecodeRope{e->qkv.as<__nv_bfloat16>(), pos, slot, e->rope_cs.as<float2>()},
                                    R, e->dec_split, e->part_o.as<float>(), e->part_ml.as<float2>(), s);
      else
        paged_attention_tc(ap, e->kv_map, e->kv_rows, e->q_map, sc, s);
    }
    {
      Prof p(e, kCatGemm);
      gemm(e, kGemmO, e->attn.as<__nv_bfloat16>(), w.wo, e->x.p, true, true, T, H * hd, d);
    }
    {
      Prof p(e, kCatOther);
      rmsnorm(e->x.as<float>(), nullptr, T, d, w.mlp_norm, c.norm_eps, e->h.as<__nv_bfloat16>(), s);
    }
    {
      Prof p(e, kCatGemm);
      gemm(e, kGemmGU, e->h.as<__nv_bfloat16>(), w.wgu, e->gu.p, false, false, T, d, 2 * ff);
    }
    {
      Prof p(e, kCatOther);
      swiglu(e->gu.as<__nv_bfloat16>(), T, ff, e->act.as<__nv_bfloat16>(), s);
    }
    {
      Prof p(e, kCatGemm);
      gemm(e, kGemmDown, e->act.as<__nv_bfloat16>(), w.wdown, e->x.p, true, true, T, ff, d);
    }
  }
  {
    Prof p(e, kCatOther);
    rmsnorm(e->x.as<float>(), reinterpret_cast<const int32_t*>(meta + ml.last), n_last, d,
            m->final_norm, c.norm_eps, e->hl.as<__nv_bfloat16>(), s);
  }
  {
    Prof p(e, kCatGemm);
    gemm(e, -1, e->hl.as<__nv_bfloat16>(), m->lm_head, e->logits.p, true, false, n_last, d,
         c.vocab);
  }
}

// Per-category device times of batch `batch` (its events have completed: the caller waited for
// the batch); spans of later batches stay queued.
void collect_profile(glmx_engine* e, uint64_t batch) {
  for (float& t : e->timings) t = 0.f;
  std::vector<glmx_engine::Span> keep;
  for (const auto& sp : e->spans) {
    if (sp.batch != batch) {
      keep.push_back(sp);
      continue;
    }
    float ms = 0.f;
    GLMX_CUDA(cudaEventSynchronize(sp.b));
    GLMX_CUDA(cudaEventElapsedTime(&ms, sp.a, sp.b));
    e->timings[sp.cat] += ms;
    e->ev_free.push_back(sp.a);
    e->ev_free.push_back(sp.b);
  }
  e->spans.swap(keep);
}
void collect_profile(glmx_engine* e) {
  GLMX_CUDA(cudaStreamSynchronize(e->stream));
  collect_profile(e, e->batch_seq);
}

}  // namespace

int engine_wait_impl(glmx_engine* e, int32_t* first_token, uint64_t cap);

int engine_prefill_impl(glmx_engine* e, uint64_t n_req, const glmx_request* reqs,
                        glmx_prefill_report* reports, int32_t* first_token, float* logits_out,
                        bool async) {
  NvtxRange nvtx_range("glmx.prefill");
  if (e->pending.size() >= 2) throw Error(GLMX_ERR_ARG, "two batches in flight: wait for one first");
  if (async && logits_out) throw Error(GLMX_ERR_ARG, "logits are only returned by the synchronous step");
  if (!async)
    while (!e->pending.empty()) engine_wait_impl(e, nullptr, 0);
  glmx_model* m = e->m;
  glmx_kv* kv = e->kv;
  BlockEngine& bk = *kv->bk;
  const auto& c = m->cfg;
  const uint32_t B = kv->cfg.block_tokens;
  if (n_req > e->cfg.max_requests) throw Error(GLMX_ERR_ARG, "too many requests in batch");
  // engine limits that do not depend on cache state are checked before any bookkeeping
  for (uint64_t i = 0; i < n_req; ++i)
    if (reqs[i].n_tok > 0 && reqs[i].n_tok + e->cfg.max_decode > e->cfg.max_context)
      throw Error(GLMX_ERR_ARG, "request exceeds max_context");
  DeviceGuard dg(m->device);
  // The previous batch's scratch pages become free (device reuse is stream-ordered after its
  // forward and decode steps); its staging slot stays untouched until its upload was consumed.
  for (auto& r : e->reqs)
    for (int32_t p : r.scratch) bk.pool().free_now(p);
  e->reqs.clear();
  e->has_batch = false;
  // Pages evicted by earlier batches: every batch that may read them is enqueued by now, unless
  // the last batch's decode is deferred (it still reads that batch's self-evicted pages).
  if (!kv->epoch_mode && !e->def_R) bk.pool().release_before(e->rel_mark);

  uint8_t* hm = meta_acquire(e);
  int32_t* h_tok = reinterpret_cast<int32_t*>(hm + e->o_tok);
  int32_t* h_pos = reinterpret_cast<int32_t*>(hm + e->o_pos);
  int64_t* h_slot = reinterpret_cast<int64_t*>(hm + e->o_slot);
  int32_t* h_qs = reinterpret_cast<int32_t*>(hm + e->o_qs);
  int32_t* h_ql = reinterpret_cast<int32_t*>(hm + e->o_ql);
  int32_t* h_ctx = reinterpret_cast<int32_t*>(hm + e->o_ctx);
  int32_t* h_bt = reinterpret_cast<int32_t*>(hm + e->o_bt);
  int2* h_work = reinterpret_cast<int2*>(hm + e->o_work);
  int32_t* h_last = reinterpret_cast<int32_t*>(hm + e->o_last);

  PrefillResult pr;
  int T = 0, R = 0, n_work = 0;
  size_t max_pages = 0;
  std::vector<int> req_row(n_req, -1);
  e->copies.clear();
  e->batch_written.clear();
  double attn_flops = 0, attn_bytes = 0, ctx_tokens = 0;
  const double kv_tok_bytes = 2.0 * c.n_kv_heads * c.head_dim * 2;  // per layer
  try {
    for (uint64_t i = 0; i < n_req; ++i) {
      const glmx_request& rq = reqs[i];
      TokenSpans ts{rq.tok_bytes, rq.tok_offsets, rq.n_tok};
      // may throw with partial state, exactly like the reference; the blocks it inserted stay
      // stale, so their KV is recomputed on first use
      bk.prefill(ts, rq.tiers, rq.n_tiers, rq.session ? rq.session : "", pr);
      if (rq.finish) bk.set_tier(rq.session ? rq.session : "", GLMX_TIER_II, GLMX_TIER_III);
      glmx_prefill_report& rep = reports[i];
      rep.cached_tokens = pr.cached;
      rep.computed_tokens = pr.computed;
      rep.tail_tokens = pr.tail;
      rep.n_evicted = pr.evicted.size();
      rep.n_blocks = pr.pages.size();
      if (first_token) first_token[i] = -1;
      if (rq.n_tok == 0) continue;
      e->reqs.emplace_back();
      glmx_engine::Req& st = e->reqs.back();
      st.pages = pr.pages;
      const uint64_t full = pr.pages.size();
      const uint64_t need = rq.n_tok + e->cfg.max_decode;
      for (uint64_t t = full * B; t < need; t += B) {
        int32_t p = bk.pool().alloc();
        st.scratch.push_back(p);
        st.pages.push_back(p);
      }
      // KV reuse = the leading cached blocks whose pages hold their KV; a stale cached block
      // (its batch failed, or it was inserted without the engine) is recomputed from there on
      uint64_t reuse_blocks = 0;
      while (reuse_blocks < pr.hit_blocks && !pr.stale[reuse_blocks]) ++reuse_blocks;
      // Cross-GPU prefix hit: the run of freshly inserted blocks that directly extends the local
      // hit prefix and is resident on a peer is copied instead of computed (bookkeeping already
      // counted them as misses, like independent per-GPU caches).
      uint64_t first_written = std::min(pr.hit_blocks, reuse_blocks);
      if (!e->reuse) {
        // reuse off (A/B): the hit blocks' KV is recomputed into scratch pages; their cached
        // pages stay as they are
        for (uint64_t b = 0; b < pr.hit_blocks; ++b) {
          st.pages[b] = bk.pool().alloc();
          st.scratch.push_back(st.pages[b]);
        }
        reuse_blocks = 0;
        first_written = pr.hit_blocks;
      } else if (reuse_blocks == pr.hit_blocks && !kv->peer_dir.empty()) {
        for (uint64_t b = pr.hit_blocks; b < full && pr.fresh[b]; ++b) {
          auto it = kv->peer_dir.find(pr.ids[b]);
          if (it == kv->peer_dir.end()) break;
          e->copies.push_back({it->second.first, it->second.second, pr.pages[b]});
          ++reuse_blocks;
        }
      }
      const uint64_t q0 = std::min<uint64_t>(reuse_blocks * B, rq.n_tok - 1);  // always >= 1 row
      const int ql = static_cast<int>(rq.n_tok - q0);
      if (T + ql > static_cast<int>(e->cfg.max_batch_tokens))
        throw Error(GLMX_ERR_ARG, "batch exceeds max_batch_tokens");
      // every block from reuse_blocks on is written by this batch (peer copy or K2 append):
      // no longer stale for the requests staged after this one (the append of a layer precedes
      // its attention); re-marked if the batch fails before its forward is enqueued
      for (uint64_t b = first_written; b < full; ++b) {
        if (st.pages[b] < 0) {  // a force_insert'ed block without a page
          if (bk.block(pr.ids[b])) {
            st.pages[b] = bk.ensure_page(pr.ids[b]);
          } else {  // ... already evicted again by this request: a scratch page serves it
            st.pages[b] = bk.pool().alloc();
            st.scratch.push_back(st.pages[b]);
          }
        }
        const Block* blk = bk.block(pr.ids[b]);
        if (blk && blk->stale) {
          bk.set_stale(pr.ids[b], false);
          e->batch_written.push_back(pr.ids[b]);
        }
      }
      h_qs[R] = T;
      h_ql[R] = ql;
      h_ctx[R] = static_cast<int32_t>(rq.n_tok);
      std::memcpy(h_bt + static_cast<size_t>(R) * e->bt_stride, st.pages.data(), st.pages.size() * 4);
      max_pages = std::max(max_pages, st.pages.size());
      for (uint64_t t = q0; t < rq.n_tok; ++t, ++T) {
        h_tok[T] = token_id(rq.tok_bytes + rq.tok_offsets[t], rq.tok_offsets[t + 1] - rq.tok_offsets[t], c.vocab);
        h_pos[T] = static_cast<int32_t>(t);
        h_slot[T] = static_cast<int64_t>(st.pages[t / B]) * B + (t % B);
      }
      for (int t0 = 0; t0 < ql; t0 += e->tpt) h_work[n_work++] = make_int2(R, t0);
      h_last[R] = T - 1;
      req_row[i] = R;
      for (uint64_t qi = q0; qi < rq.n_tok; ++qi) attn_flops += 4.0 * c.n_heads * c.head_dim * (qi + 1);
      attn_bytes += kv_tok_bytes * rq.n_tok + 2.0 * ql * c.n_heads * c.head_dim * 2;
      ctx_tokens += rq.n_tok;
      st.ctx_len = static_cast<int32_t>(rq.n_tok);
      ++R;
    }
    if (e->copies.size() > e->max_copies) throw Error(GLMX_ERR_ARG, "too many peer copies in batch");
  } catch (...) {
    // No forward will write this batch's blocks: they become stale again (recomputed on their
    // next use), and its scratch pages go back to the pool.
    for (uint64_t id : e->batch_written) bk.set_stale(id, true);
    e->batch_written.clear();
    for (auto& r : e->reqs)
      for (int32_t p : r.scratch) bk.pool().free_now(p);
    e->reqs.clear();
    e->copies.clear();
    throw;
  }
  // longest tiles first (LPT over the 148 SMs)
  std::sort(h_work, h_work + n_work, [&](const int2& a, const int2& b) {
    int ka = h_ctx[a.x] - h_ql[a.x] + a.y, kb = h_ctx[b.x] - h_ql[b.x] + b.y;
    return ka > kb;
  });
  e->dec_split = choose_decode_split(e, R, T, h_ctx);
  if (!e->dec_split) stage_attn_schedule(e, hm, h_work, n_work, h_ql, h_ctx);
  e->last_T = T;
  e->last_R = R;
  e->last_work = n_work;
  e->work[0] = attn_flops * c.n_layers;
  e->work[1] = attn_bytes * c.n_layers;
  // K2 (fused RoPE + append) algorithmic bytes: read the qkv row, write q and the K/V rows
  e->work[2] = static_cast<double>(T) * c.n_layers *
               (2.0 * (c.n_heads + 2 * c.n_kv_heads) * c.head_dim + 2.0 * c.n_heads * c.head_dim +
                kv_tok_bytes);
  const double lin = 2.0 * (static_cast<double>(c.d_model) * (c.n_heads + 2 * c.n_kv_heads) * c.head_dim +
                            static_cast<double>(c.d_model) * c.n_heads * c.head_dim +
                            3.0 * c.d_model * c.d_ff);
  e->work[3] = lin * T * c.n_layers + 2.0 * c.d_model * c.vocab * R;
  e->work[4] = T;
  e->work[5] = ctx_tokens;
  e->rel_mark = bk.pool().mark();
  if (R == 0) {  // nothing to compute (empty prompts): a completed pseudo-batch keeps wait() in order
    glmx_engine::Pending pd;
    pd.req_row.assign(n_req, -1);
    pd.batch = e->batch_seq++;
    pd.slot = -1;
    std::memcpy(pd.work, e->work, sizeof(pd.work));
    e->pending.push_back(std::move(pd));
    if (!async) engine_wait_impl(e, nullptr, 0);
    return GLMX_OK;
  }
  // peer copies, grouped by source pool: src pages then dst pages per group in the copy section
  std::stable_sort(e->copies.begin(), e->copies.end(),
                   [](const glmx_engine::Copy& a, const glmx_engine::Copy& b) { return a.peer < b.peer; });
  {
    int32_t* h_cp = reinterpret_cast<int32_t*>(hm + e->o_copy);
    const size_t nc = e->copies.size();
    for (size_t i = 0; i < nc; ++i) {
      h_cp[i] = e->copies[i].src_page;
      h_cp[nc + i] = e->copies[i].dst_page;
    }
    kv->peer_hits += static_cast<int64_t>(nc);
  }
  cudaStream_t s = e->stream;
  {
    Prof p(e, kCatH2D);
    MetaCounts mc;
    mc.n_tok = T;
    mc.T = T;
    mc.R = R;
    mc.n_work = n_work;
    mc.n_copy = static_cast<int>(e->copies.size());
    mc.bt_stride = static_cast<int>(align_up(std::max<size_t>(max_pages, 1), 8));
    mc.sched = !e->dec_split;
    meta_commit(e, s, mc);
  }
  if (!e->copies.empty()) {
    Prof p(e, kCatOther);
    const int32_t* d_cp = reinterpret_cast<const int32_t*>(e->meta.as<uint8_t>() + e->ml.copy);
    const size_t nc = e->copies.size();
    for (size_t a = 0; a < nc;) {
      size_t b = a;
      while (b < nc && e->copies[b].peer == e->copies[a].peer) ++b;
      const int32_t peer = e->copies[a].peer;
      if (peer < 0 || static_cast<size_t>(peer) >= kv->peers.size() || !kv->peers[peer].base)
        throw Error(GLMX_ERR_ARG, "peer " + std::to_string(peer) + " is not attached");
      for (size_t o = a; o < b; o += 65535)
        pool_copy_pages(kv->peers[peer].base, kv->geom.base, kv->geom.page_elems(), d_cp + o,
                        d_cp + nc + o, static_cast<int>(std::min<size_t>(65535, b - o)), s);
      a = b;
    }
  }
  forward(e, T, R, n_work, R, reinterpret_cast<const int32_t*>(e->meta.as<uint8_t>() + e->ml.tok));
  argmax_rows(e->logits.as<float>(), R, c.vocab, e->next_tok.as<int32_t>(), e->amax_keys.p, s);
  const int slot = static_cast<int>(e->batch_seq & 1);
  {
    Prof p(e, kCatD2H);
    GLMX_CUDA(cudaMemcpyAsync(e->h_out + slot * e->h_out_stride, e->next_tok.p, R * 4,
                              cudaMemcpyDeviceToHost, s));
    e->d2h_bytes += static_cast<uint64_t>(R) * 4;
  }
  GLMX_CUDA(cudaEventRecord(e->fwd_done, s));
  GLMX_CUDA(cudaEventRecord(e->done_ev[slot], s));
  glmx_engine::Pending pd;
  pd.req_row = std::move(req_row);
  pd.batch = e->batch_seq;
  pd.slot = slot;
  std::memcpy(pd.work, e->work, sizeof(pd.work));
  e->pending.push_back(std::move(pd));
  ++e->batch_seq;
  // decode continues from the last prompt token's greedy successor
  e->has_batch = true;
  if (async) return GLMX_OK;
  // synchronous step: collect this batch now (logits stay valid: nothing else was enqueued)
  const int32_t* h = e->h_out + slot * e->h_out_stride;
  const std::vector<int> rows = e->pending.back().req_row;
  engine_wait_impl(e, nullptr, 0);
  for (uint64_t i = 0; i < n_req; ++i) {
    if (rows[i] < 0) continue;
    if (first_token) first_token[i] = h[rows[i]];
    if (logits_out) {
      GLMX_CUDA(cudaMemcpy(logits_out + i * c.vocab, e->logits.as<float>() + static_cast<size_t>(rows[i]) * c.vocab,
                           c.vocab * 4, cudaMemcpyDeviceToHost));
      e->d2h_bytes += static_cast<uint64_t>(c.vocab) * 4;
    }
  }
  return GLMX_OK;
}

// Completes the oldest in-flight prefill batch: waits for it, publishes its timings and work,
// writes its greedy first tokens (-1 for empty prompts).  Returns the batch's request count.
int engine_wait_impl(glmx_engine* e, int32_t* first_token, uint64_t cap) {
  NvtxRange nvtx_range("glmx.wait");
  if (e->pending.empty()) throw Error(GLMX_ERR_ARG, "no prefill batch in flight");
  DeviceGuard dg(e->m->device);
  glmx_engine::Pending pd = std::move(e->pending.front());
  e->pending.erase(e->pending.begin());
  if (pd.slot >= 0) GLMX_CUDA(cudaEventSynchronize(e->done_ev[pd.slot]));
  collect_profile(e, pd.batch);
  std::memcpy(e->work_done, pd.work, sizeof(pd.work));
  const int32_t* h = e->h_out + std::max(pd.slot, 0) * e->h_out_stride;
  if (first_token) {
    if (cap < pd.req_row.size()) throw Error(GLMX_ERR_ARG, "first_token buffer too small");
    for (size_t i = 0; i < pd.req_row.size(); ++i) first_token[i] = pd.req_row[i] < 0 ? -1 : h[pd.req_row[i]];
  }
  return static_cast<int>(pd.req_row.size());
}

// Greedy decode.  Requests are re-ordered by step count (descending) so the active set of every
// step is a row prefix and step s+1 consumes step s's argmax rows in place on the device.
// engine_decode_enqueue stages and launches all steps of the staged batch without waiting for
// the GPU (the prefill that produced the first tokens may still be in flight: the first-token
// row order is a device gather); engine_decode_collect waits and returns the tokens.  The next
// prefill may be staged in between (its staging uses the next pinned slots; the decode's pages
// and device buffers are stream-ordered before it).
// Defers the decode of the staged batch so it runs merged with the next batch's decode (one
// weight stream per step for both sets of rows): the batch's requests keep their pages (the next
// prefill's staging will not free them) and its first tokens are copied aside on the stream.
int engine_decode_defer(glmx_engine* e, const uint32_t* steps) {
  if (!e->has_batch) throw Error(GLMX_ERR_ARG, "decode needs a prefill batch");
  if (e->def_R) throw Error(GLMX_ERR_ARG, "a decode is already deferred");
  if (e->dec_pending) throw Error(GLMX_ERR_ARG, "a decode is already enqueued: collect it first");
  const int R = e->last_R;
  for (int i = 0; i < R; ++i)
    if (steps[i] > e->cfg.max_decode) throw Error(GLMX_ERR_ARG, "steps exceed max_decode");
  DeviceGuard dg(e->m->device);
  e->def_reqs = std::move(e->reqs);
  e->reqs.clear();
  e->def_steps.assign(steps, steps + R);
  e->def_R = R;
  e->def_mark = e->rel_mark;  // pages this batch evicted stay deferred until its decode is enqueued
  e->has_batch = false;
  GLMX_CUDA(cudaMemcpyAsync(e->def_first.p, e->next_tok.p, static_cast<size_t>(R) * 4,
                            cudaMemcpyDeviceToDevice, e->stream));
  return GLMX_OK;
}

// Greedy decode.  Rows (the deferred batch's first, then the staged batch's) are re-ordered by
// step count (descending) so the active set of every step is a row prefix and step s+1 consumes
// step s's argmax rows in place on the device.  engine_decode_enqueue stages and launches all
// steps without waiting for the GPU (the prefill that produced the first tokens may still be in
// flight: the first-token row order is a device gather); engine_decode_collect waits and returns
// the tokens.  The next prefill may be staged in between (its staging uses the next pinned
// slots; the decode's pages and device buffers are stream-ordered before it).
int engine_decode_enqueue(glmx_engine* e, const uint32_t* steps) {
  NvtxRange nvtx_range("glmx.decode");
  if (!e->has_batch) throw Error(GLMX_ERR_ARG, "decode needs a prefill batch");
  if (e->dec_pending) throw Error(GLMX_ERR_ARG, "a decode is already enqueued: collect it first");
  glmx_model* m = e->m;
  const auto& c = m->cfg;
  const uint32_t B = e->kv->cfg.block_tokens;
  const int Rc = e->last_R, Rd = e->def_R, R = Rc + Rd;
  uint32_t max_steps = 0;
  e->dec_steps.assign(e->def_steps.begin(), e->def_steps.begin() + Rd);
  for (int i = 0; i < Rc; ++i) {
    if (steps[i] > e->cfg.max_decode) throw Error(GLMX_ERR_ARG, "steps exceed max_decode");
    // the request's pages cover its prompt + max_decode positions (scratch allocated at prefill)
    if (static_cast<uint64_t>(e->reqs[i].ctx_len) + steps[i] > e->reqs[i].pages.size() * B)
      throw Error(GLMX_ERR_ARG, "decode steps exceed the request's pages");
    e->dec_steps.push_back(steps[i]);
  }
  e->has_batch = false;  // one decode per prefill batch
  for (uint32_t st : e->dec_steps) max_steps = std::max(max_steps, st);
  e->dec_max = max_steps;
  e->dec_R = R;
  e->dec_R_def = Rd;
  e->dec_order.resize(R);
  for (int i = 0; i < R; ++i) e->dec_order[i] = i;
  const std::vector<uint32_t>& all_steps = e->dec_steps;
  std::stable_sort(e->dec_order.begin(), e->dec_order.end(),
                   [&](int a, int b) { return all_steps[a] > all_steps[b]; });
  e->dec_pending = true;
  // the deferred requests' scratch pages are freed at the collect (after their last step)
  e->dec_free = std::move(e->def_reqs);
  std::vector<glmx_engine::Req>& dreqs = e->dec_free;
  // row i < Rd: deferred request i; else staged request i - Rd
  auto row_req = [&](int i) -> glmx_engine::Req& { return i < Rd ? dreqs[i] : e->reqs[i - Rd]; };
  e->def_R = 0;
  e->def_reqs.clear();
  e->def_steps.clear();
  // the deferred batch's self-evicted pages are released once the merged decode that reads them
  // is enqueued (any later writer, the next prefill, is stream-ordered after it)
  const bool release_def = Rd > 0 && !e->kv->epoch_mode;
  if (max_steps == 0) {
    if (release_def) e->kv->bk->pool().release_before(e->def_mark);
    return GLMX_OK;
  }
  DeviceGuard dg(m->device);
  cudaStream_t s = e->stream;
  const std::vector<int>& order = e->dec_order;
  int32_t* d_seq = e->next_tok.as<int32_t>() + R;  // [max_steps][R] generated tokens
  int32_t* d_in = e->dec_in.as<int32_t>();         // step 0 input, decode row order
  static constexpr uint64_t kDecTag = 1ull << 63;
  e->dec_tag_batch = e->batch_seq;
  e->prof_tag = kDecTag | e->batch_seq;
  for (uint32_t st = 0; st < max_steps; ++st) {
    int n = 0;
    while (n < R && all_steps[order[n]] > st) ++n;
    uint8_t* hm = meta_acquire(e);
    int32_t* h_pos = reinterpret_cast<int32_t*>(hm + e->o_pos);
    int64_t* h_slot = reinterpret_cast<int64_t*>(hm + e->o_slot);
    int32_t* h_qs = reinterpret_cast<int32_t*>(hm + e->o_qs);
    int32_t* h_ql = reinterpret_cast<int32_t*>(hm + e->o_ql);
    int32_t* h_ctx = reinterpret_cast<int32_t*>(hm + e->o_ctx);
    int32_t* h_bt = reinterpret_cast<int32_t*>(hm + e->o_bt);
    int2* h_work = reinterpret_cast<int2*>(hm + e->o_work);
    int32_t* h_last = reinterpret_cast<int32_t*>(hm + e->o_last);
    int32_t* h_perm = reinterpret_cast<int32_t*>(hm + e->o_perm);
    size_t max_pages = 1;
    for (int j = 0; j < n; ++j) {
      glmx_engine::Req& rq = row_req(order[j]);
      const int32_t p = rq.ctx_len;  // position of the token being fed
      h_pos[j] = p;
      h_slot[j] = static_cast<int64_t>(rq.pages[p / B]) * B + (p % B);
      h_qs[j] = j;
      h_ql[j] = 1;
      h_ctx[j] = p + 1;
      std::memcpy(h_bt + static_cast<size_t>(j) * e->bt_stride, rq.pages.data(), rq.pages.size() * 4);
      max_pages = std::max(max_pages, rq.pages.size());
      h_work[j] = make_int2(j, 0);
      h_last[j] = j;
      rq.ctx_len = p + 1;
    }
    if (st == 0)  // first-token gather: every decode row (rows with 0 steps are never fed)
      for (int j = 0; j < R; ++j) h_perm[j] = order[j];
    e->dec_split = choose_decode_split(e, n, n, h_ctx);
    if (!e->dec_split) stage_attn_schedule(e, hm, h_work, n, h_ql, h_ctx);
    MetaCounts mc;
    mc.T = n;
    mc.R = n;
    mc.n_work = n;
    mc.n_perm = st == 0 ? R : 0;
    mc.bt_stride = static_cast<int>(align_up(max_pages, 8));
    mc.sched = !e->dec_split;
    meta_commit(e, s, mc);
    if (st == 0)
      gather2_i32(e->def_first.as<int32_t>(), Rd, e->next_tok.as<int32_t>(),
                  reinterpret_cast<const int32_t*>(e->meta.as<uint8_t>() + e->ml.perm), R, d_in, s);
    const int32_t* in_tok = st == 0 ? d_in : d_seq + static_cast<size_t>(st - 1) * R;
    forward(e, n, n, n, n, in_tok);
    argmax_rows(e->logits.as<float>(), n, c.vocab, d_seq + static_cast<size_t>(st) * R,
                e->amax_keys.p, s);
  }
  e->prof_tag = 0;
  GLMX_CUDA(cudaMemcpyAsync(e->h_dec, d_seq, static_cast<size_t>(max_steps) * R * 4,
                            cudaMemcpyDeviceToHost, s));
  e->d2h_bytes += static_cast<uint64_t>(max_steps) * R * 4;
  GLMX_CUDA(cudaEventRecord(e->dec_done, s));
  if (release_def) e->kv->bk->pool().release_before(e->def_mark);
  return GLMX_OK;
}

// out_tokens [staged rows][max_steps]; out_prev (nullable) [deferred rows][max_steps] for the
// rows of a batch whose decode was deferred into this one.
int engine_decode_collect(glmx_engine* e, int32_t* out_tokens, int32_t* out_prev, float* last_logits) {
  NvtxRange nvtx_range("glmx.decode_collect");
  if (!e->dec_pending) throw Error(GLMX_ERR_ARG, "no decode enqueued");
  e->dec_pending = false;
  const int R = e->dec_R, Rd = e->dec_R_def;
  const uint32_t max_steps = e->dec_max;
  DeviceGuard dg(e->m->device);
  if (max_steps > 0) {
    GLMX_CUDA(cudaEventSynchronize(e->dec_done));
    collect_profile(e, (1ull << 63) | e->dec_tag_batch);
  }
  for (auto& rq : e->dec_free)
    for (int32_t pg : rq.scratch) e->kv->bk->pool().free_now(pg);
  e->dec_free.clear();
  for (int i = 0; i < R; ++i) {
    int32_t* dst = i < Rd ? out_prev : out_tokens;
    if (!dst) continue;
    const int row = i < Rd ? i : i - Rd;
    for (uint32_t st = 0; st < max_steps; ++st) dst[static_cast<size_t>(row) * max_steps + st] = -1;
  }
  if (max_steps == 0) return GLMX_OK;
  const std::vector<int>& order = e->dec_order;
  for (int j = 0; j < R; ++j) {
    const int i = order[j];
    int32_t* dst = i < Rd ? out_prev : out_tokens;
    if (!dst) continue;
    const int row = i < Rd ? i : i - Rd;
    for (uint32_t st = 0; st < e->dec_steps[i]; ++st)
      dst[static_cast<size_t>(row) * max_steps + st] = e->h_dec[static_cast<size_t>(st) * R + j];
  }
  if (last_logits) {
    // logits of the final step for the staged requests still active in it (synchronous path)
    const int V = static_cast<int>(e->m->cfg.vocab);
    int n = 0;
    while (n < R && e->dec_steps[order[n]] >= max_steps) ++n;
    for (int j = 0; j < n; ++j) {
      if (order[j] < Rd) continue;
      GLMX_CUDA(cudaMemcpy(last_logits + static_cast<size_t>(order[j] - Rd) * V,
                           e->logits.as<float>() + static_cast<size_t>(j) * V, V * 4,
                           cudaMemcpyDeviceToHost));
    }
  }
  return GLMX_OK;
}

int engine_decode_impl(glmx_engine* e, const uint32_t* steps, int32_t* out_tokens, float* last_logits) {
  while (!e->pending.empty()) engine_wait_impl(e, nullptr, 0);
  if (e->def_R) throw Error(GLMX_ERR_ARG, "a decode is deferred: use the async decode to merge it");
  engine_decode_enqueue(e, steps);
  return engine_decode_collect(e, out_tokens, nullptr, last_logits);
}

// ======================================================================== K3 kernel-level hook
// Runs the paged attention kernel on caller-owned device buffers (tests + attention sweeps):
// uploads the request metadata, builds the same longest-first work list as the engine, launches
// `reps` times on `stream` and reports the mean kernel time (CUDA events on that stream).
int attention_run_impl(int impl, const void* q, void* o, uint64_t T, int H, int Hkv, int hd,
                       void* pool_base, uint64_t n_pages, uint32_t n_layers, uint32_t layer,
                       uint32_t block_tokens, uint64_t n_req, const int32_t* q_start,
                       const int32_t* q_len, const int32_t* ctx_len, const int32_t* block_table,
                       int bt_stride, int reps, cudaStream_t s, float* out_ms) {
  if (n_req == 0) return GLMX_OK;
  if (H % Hkv != 0 || reps < 1) throw Error(GLMX_ERR_ARG, "bad attention arguments");
  // impl 0: the tcgen05 kernel; impl 2: the CUDA-core decode kernel (every request one token)
  if (impl != 0 && impl != 2) throw Error(GLMX_ERR_ARG, "attention impl must be 0 (tcgen05) or 2 (decode)");
  const bool dec = impl == 2;
  if (dec)
    for (uint64_t r = 0; r < n_req; ++r)
      if (q_len[r] != 1) throw Error(GLMX_ERR_ARG, "decode attention needs q_len == 1");
  PoolGeom geom{static_cast<__nv_bfloat16*>(pool_base), n_layers, static_cast<uint32_t>(Hkv),
                block_tokens, static_cast<uint32_t>(hd)};
  const int tpt = attn_tc_tokens_per_tile(H, Hkv);
  std::vector<int2> work;
  for (uint64_t r = 0; r < n_req; ++r) {
    if (q_len[r] < 1 || ctx_len[r] < q_len[r] ||
        static_cast<uint64_t>(q_start[r]) + q_len[r] > T ||
        (ctx_len[r] + static_cast<int>(block_tokens) - 1) / static_cast<int>(block_tokens) > bt_stride)
      throw Error(GLMX_ERR_ARG, "bad request geometry");
    for (int t0 = 0; t0 < q_len[r]; t0 += tpt) work.push_back(make_int2(static_cast<int>(r), t0));
  }
  std::stable_sort(work.begin(), work.end(), [&](const int2& a, const int2& b) {
    return ctx_len[a.x] - q_len[a.x] + a.y > ctx_len[b.x] - q_len[b.x] + b.y;
  });
  // repack the caller's block table into rows of a multiple of 8 entries (K3's 16-byte reads)
  const int bt_pad = static_cast<int>(align_up(static_cast<size_t>(bt_stride), 8));
  std::vector<int32_t> bt_packed(n_req * static_cast<size_t>(bt_pad), 0);
  for (uint64_t r = 0; r < n_req; ++r)
    std::memcpy(bt_packed.data() + r * bt_pad, block_table + r * bt_stride, bt_stride * 4);
  block_table = bt_packed.data();
  bt_stride = bt_pad;
  const size_t nr = n_req * 4, nbt = n_req * static_cast<size_t>(bt_stride) * 4;
  auto a16 = [](size_t x) { return (x + 15) & ~size_t(15); };
  const size_t o_ql = a16(nr), o_ctx = o_ql + a16(nr), o_bt = o_ctx + a16(nr);
  const size_t o_wk = o_bt + a16(nbt);
  size_t o_pc = 0, o_cta = 0, o_cb = 0, o_pp = 0;
  const size_t sched_bytes =
      attn_sched_bytes(static_cast<int>(work.size()) * Hkv, kNumSMs, &o_pc, &o_cta, &o_cb, &o_pp);
  const size_t o_sched = (o_wk + work.size() * 8 + 255) & ~size_t(255);
  const size_t bytes = o_sched + sched_bytes;
  std::vector<uint8_t> h(bytes);
  std::memcpy(h.data(), q_start, nr);
  std::memcpy(h.data() + o_ql, q_len, nr);
  std::memcpy(h.data() + o_ctx, ctx_len, nr);
  std::memcpy(h.data() + o_bt, block_table, nbt);
  std::memcpy(h.data() + o_wk, work.data(), work.size() * 8);
  AttnSchedule hs;
  hs.pieces = reinterpret_cast<AttnPiece*>(h.data() + o_sched + o_pc);
  hs.cta_off = reinterpret_cast<int32_t*>(h.data() + o_sched + o_cta);
  hs.combine = reinterpret_cast<AttnCombine*>(h.data() + o_sched + o_cb);
  hs.partners = reinterpret_cast<AttnPiece*>(h.data() + o_sched + o_pp);
  if (!dec)
    build_attn_schedule(reinterpret_cast<const int32_t*>(work.data()), static_cast<int>(work.size()),
                        Hkv, q_len, ctx_len, tpt, 128, kNumSMs, hs);
  DBuf meta, part_o, part_ml;
  meta.reserve(bytes);
  GLMX_CUDA(cudaMemcpyAsync(meta.p, h.data(), bytes, cudaMemcpyHostToDevice, s));
  if (!dec && hs.n_combine > 0) {
    part_o.reserve(static_cast<size_t>(hs.n_partials) * attn_tc_partial_rows() * hd * 4);
    part_ml.reserve(static_cast<size_t>(hs.n_partials) * attn_tc_partial_rows() * 8);
  }
  const uint8_t* dm = meta.as<uint8_t>();
  AttnTcSched sc{reinterpret_cast<const int4*>(dm + o_sched + o_pc),
                 reinterpret_cast<const int*>(dm + o_sched + o_cta),
                 reinterpret_cast<const int4*>(dm + o_sched + o_cb), hs.grid, hs.n_combine,
                 part_o.as<float>(), part_ml.as<float2>(),
                 reinterpret_cast<const int4*>(dm + o_sched + o_pp)};
  AttnParams ap{};
  ap.q = static_cast<const __nv_bfloat16*>(q);
  ap.o = static_cast<__nv_bfloat16*>(o);
  ap.pool = geom;
  ap.layer = layer;
  ap.q_start = reinterpret_cast<const int32_t*>(dm);
  ap.q_len = reinterpret_cast<const int32_t*>(dm + o_ql);
  ap.ctx_len = reinterpret_cast<const int32_t*>(dm + o_ctx);
  ap.block_table = reinterpret_cast<const int32_t*>(dm + o_bt);
  ap.bt_stride = bt_stride;
  ap.work = reinterpret_cast<const int2*>(dm + o_wk);
  ap.n_work = static_cast<int>(work.size());
  ap.H = H;
  ap.Hkv = Hkv;
  ap.scale_log2 = static_cast<float>(1.0 / std::sqrt(static_cast<double>(hd)) * 1.4426950408889634);
  alignas(64) uint8_t kv_map[128], q_map[128];
  uint32_t rows = 0;
  if (!dec) {
    make_pool_tensor_map(geom, n_pages, kv_map, &rows);
    make_q_tensor_map(q, T, H, Hkv, q_map);
  }
  int dec_split = 0;
  if (dec) {
    if (!decode_attention_supported(ap)) throw Error(GLMX_ERR_ARG, "decode attention: unsupported geometry");
    int max_ctx = 0;
    for (uint64_t r = 0; r < n_req; ++r) max_ctx = std::max(max_ctx, ctx_len[r]);
    dec_split = decode_attention_splits(static_cast<int>(n_req) * Hkv, max_ctx, 1 << 20);
    part_o.reserve(static_cast<size_t>(n_req) * Hkv * dec_split * 4 * hd * 4);
    part_ml.reserve(static_cast<size_t>(n_req) * Hkv * dec_split * 4 * 8);
  }
  cudaEvent_t e0, e1;
  GLMX_CUDA(cudaEventCreate(&e0));
  GLMX_CUDA(cudaEventCreate(&e1));
  float ms = 0.f;
  try {
    GLMX_CUDA(cudaEventRecord(e0, s));
    for (int i = 0; i < reps; ++i) {
      if (dec)
        paged_attention_decode(ap, static_cast<int>(n_req), dec_split, part_o.as<float>(),
                               part_ml.as<float2>(), s);
      else
        paged_attention_tc(ap, kv_map, rows, q_map, sc, s);
    }
    GLMX_CUDA(cudaEventRecord(e1, s));
    GLMX_CUDA(cudaEventSynchronize(e1));
    GLMX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  } catch (...) {
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    throw;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (out_ms) *out_ms = ms / static_cast<float>(reps);
  return GLMX_OK;
}

// ======================================================================== K2 kernel-level hook
int rope_append_run_impl(const void* qkv, const int32_t* pos, const int64_t* slot, uint64_t T,
                         int H, int Hkv, int hd, float rope_theta, void* pool_base,
                         uint32_t n_layers, uint32_t layer, uint32_t block_tokens, void* q_out,
                         int reps, cudaStream_t s, float* out_ms) {
  if (T == 0) return GLMX_OK;
  if (reps < 1 || hd % 16 || hd > 256) throw Error(GLMX_ERR_ARG, "bad append arguments");
  std::vector<float> inv(hd / 2);
  for (int i = 0; i < hd / 2; ++i)
    inv[i] = static_cast<float>(1.0 / std::pow(static_cast<double>(rope_theta), 2.0 * i / hd));
  DBuf d_inv;
  d_inv.reserve(inv.size() * 4);
  GLMX_CUDA(cudaMemcpyAsync(d_inv.p, inv.data(), inv.size() * 4, cudaMemcpyHostToDevice, s));
  // the engine builds this table once per forward (rope_table) and shares it across the layers:
  // outside the timed launches here too
  DBuf d_cs;
  d_cs.reserve(T * (hd / 2) * sizeof(float2));
  rope_table(pos, static_cast<int>(T), hd / 2, d_inv.as<float>(), d_cs.as<float2>(), s);
  PoolGeom geom{static_cast<__nv_bfloat16*>(pool_base), n_layers, static_cast<uint32_t>(Hkv),
                block_tokens, static_cast<uint32_t>(hd)};
  cudaEvent_t e0, e1;
  GLMX_CUDA(cudaEventCreate(&e0));
  GLMX_CUDA(cudaEventCreate(&e1));
  float ms = 0.f;
  try {
    GLMX_CUDA(cudaEventRecord(e0, s));
    for (int i = 0; i < reps; ++i)
      rope_kv_append(static_cast<const __nv_bfloat16*>(qkv), pos, slot, static_cast<int>(T), H, Hkv,
                     hd, d_inv.as<float>(), d_cs.as<float2>(), geom, layer,
                     static_cast<__nv_bfloat16*>(q_out), s);
    GLMX_CUDA(cudaEventRecord(e1, s));
    GLMX_CUDA(cudaEventSynchronize(e1));
    GLMX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  } catch (...) {
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    throw;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (out_ms) *out_ms = ms / static_cast<float>(reps);
  return GLMX_OK;
}

// ======================================================================== K5 RetrieveNode
// VectorIndex::build (index.cpp:27-39) with the default Config: every node with a string "title"
// (else "name") attribute, ascending id, embed(text, dim) computed on the host exactly as
// embedder.cpp does, rows uploaded once.
int index_build_impl(glmx_graph* g, int dim, uint64_t lru_capacity) {
  if (dim < 1 || glmx::embed_padded(dim) > 128) throw Error(GLMX_ERR_ARG, "embedding dim must be in [1, 128]");
  if (g->device < 0) throw Error(GLMX_ERR_NO_DEVICE, "graph has no device");
  const int pad = glmx::embed_padded(dim);
  const int dpad = pad <= 32 ? 32 : pad <= 64 ? 64 : 128;  // kernel row widths (zero-filled)
  std::vector<float> rows;
  g->idx_node.clear();
  std::vector<float> e(pad);
  for (uint64_t v = 0; v < g->host.n(); ++v) {
    if (!g->host.has_itext[v]) continue;
    const std::string& t = g->host.itext[v];
    glmx::embed(t.data(), t.size(), dim, e.data());
    rows.insert(rows.end(), e.begin(), e.end());
    rows.insert(rows.end(), dpad - pad, 0.f);
    g->idx_node.push_back(static_cast<int32_t>(v));
  }
  g->idx_dim = dim;
  g->idx_pad = dpad;
  DeviceGuard dg(g->device);
  g->d_emb.reserve(std::max<size_t>(rows.size(), 1) * 4);
  if (!rows.empty())
    GLMX_CUDA(cudaMemcpy(g->d_emb.p, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice));
  g->lru.set_capacity(lru_capacity);
  g->stats[0] = g->stats[1] = g->stats[2] = 0;
  return GLMX_OK;
}

// Batched Retriever::retrieve_node_traced (retriever.cpp:49-66) in request order: LRU get ->
// hit; else a probe, whose result is put into the LRU at that point of the sequence (value
// resolved after the one GPU scan that serves every probe of the batch).
int retrieve_impl(glmx_graph* g, const char* bytes, const uint64_t* offs, uint64_t n,
                  int32_t* out_node, uint8_t* out_hit) {
  NvtxRange nvtx_range("glmx.k5.retrieve");
  if (g->idx_pad == 0) throw Error(GLMX_ERR_ARG, "no index: call glmx_index_build first");
  if (g->idx_node.empty() && n) throw Error(GLMX_ERR_RETRIEVAL, "EmptyIndex: the index has no entries");
  std::vector<int64_t> val(n);
  std::vector<std::string> probe_text;
  std::unordered_map<std::string, int64_t> probe_of;  // text -> probe slot of this batch
  for (uint64_t i = 0; i < n; ++i) {
    std::string t(bytes + offs[i], offs[i + 1] - offs[i]);
    int64_t v;
    if (g->lru.get(t, &v)) {
      ++g->stats[0];
      if (out_hit) out_hit[i] = 1;
      val[i] = v;
      continue;
    }
    ++g->stats[1];
    ++g->stats[2];
    if (out_hit) out_hit[i] = 0;
    auto it = probe_of.find(t);
    int64_t slot;
    if (it == probe_of.end()) {
      slot = static_cast<int64_t>(probe_text.size());
      probe_of.emplace(t, slot);
      probe_text.push_back(std::move(t));
      t = probe_text.back();
    } else {
      slot = it->second;
    }
    const int64_t ph = -(slot + 1);  // placeholder until the scan resolves it
    g->lru.put(t, ph);
    val[i] = ph;
  }
  std::vector<int32_t> probe_node(probe_text.size(), -1);
  if (!probe_text.empty()) {
    const int pad = glmx::embed_padded(g->idx_dim), dpad = g->idx_pad;
    const int nq = static_cast<int>(probe_text.size());
    std::vector<float> q(static_cast<size_t>(nq) * dpad, 0.f);
    for (int k = 0; k < nq; ++k)
      glmx::embed(probe_text[k].data(), probe_text[k].size(), g->idx_dim, q.data() + static_cast<size_t>(k) * dpad);
    (void)pad;
    DeviceGuard dg(g->device);
    cudaStream_t s = g->stream;
    g->d_qemb.reserve(q.size() * 4);
    g->d_best.reserve(static_cast<size_t>(nq) * 8);
    GLMX_CUDA(cudaMemcpyAsync(g->d_qemb.p, q.data(), q.size() * 4, cudaMemcpyHostToDevice, s));
    g->h2d_bytes += q.size() * 4;
    g->d2h_bytes += static_cast<uint64_t>(nq) * 8;
    GLMX_CUDA(cudaMemsetAsync(g->d_best.p, 0, static_cast<size_t>(nq) * 8, s));
    GLMX_CUDA(cudaEventRecord(g->ev0, s));
    nearest_top1(g->d_emb.as<float>(), static_cast<int>(g->idx_node.size()), dpad, g->d_qemb.as<float>(), nq,
                 g->d_best.as<unsigned long long>(), s);
    GLMX_CUDA(cudaEventRecord(g->ev1, s));
    std::vector<unsigned long long> best(nq);
    GLMX_CUDA(cudaMemcpyAsync(best.data(), g->d_best.p, nq * 8, cudaMemcpyDeviceToHost, s));
    GLMX_CUDA(cudaStreamSynchronize(s));
    GLMX_CUDA(cudaEventElapsedTime(&g->last_retrieve_ms, g->ev0, g->ev1));
    for (int k = 0; k < nq; ++k) {
      const uint32_t row = 0xFFFFFFFFu - static_cast<uint32_t>(best[k] & 0xFFFFFFFFu);
      if (best[k] == 0 || row >= g->idx_node.size()) throw Error(GLMX_ERR_CUDA, "nearest scan returned no row");
      probe_node[k] = g->idx_node[row];
      g->lru.resolve(-(k + 1), probe_node[k]);
    }
  }
  for (uint64_t i = 0; i < n; ++i) {
    int64_t v = val[i];
    if (v < 0) v = probe_node[-v - 1];
    if (out_node) out_node[i] = static_cast<int32_t>(v);
  }
  return GLMX_OK;
}

// ======================================================================== scalable generate_workload
// The validation "every title retrieves its own node" (workload.cpp:166-171), one full-scan
// nearest per candidate in the reference (O(N^2), >10 min at 100k nodes), is one batched K5 scan
// of all titles against the device index; the pools and draws then follow the reference exactly.
int workload_generate_impl(glmx_graph* g, uint64_t seed, int n, double ratio, std::string* out,
                           float* scan_ms) {
  if (g->device < 0) throw Error(GLMX_ERR_NO_DEVICE, "graph has no device");
  if (g->idx_pad == 0 || g->idx_dim != 64) index_build_impl(g, 64, 1024);  // Config::embed_dim
  const uint64_t N = g->host.n();
  std::vector<uint8_t> unique(N, 0);
  std::vector<int32_t> qnode;
  for (uint64_t v = 0; v < N; ++v)
    if (g->host.has_itext[v] && g->host.itext_is_title[v]) qnode.push_back(static_cast<int32_t>(v));
  DeviceGuard dg(g->device);
  cudaStream_t s = g->stream;
  const int dpad = g->idx_pad, chunk = 32768;
  float total_ms = 0.f;
  std::vector<float> q;
  std::vector<unsigned long long> best;
  for (size_t c0 = 0; c0 < qnode.size(); c0 += chunk) {
    const int nq = static_cast<int>(std::min<size_t>(chunk, qnode.size() - c0));
    q.assign(static_cast<size_t>(nq) * dpad, 0.f);
    for (int k = 0; k < nq; ++k) {
      const std::string& t = g->host.itext[qnode[c0 + k]];
      glmx::embed(t.data(), t.size(), g->idx_dim, q.data() + static_cast<size_t>(k) * dpad);
    }
    g->d_qemb.reserve(q.size() * 4);
    g->d_best.reserve(static_cast<size_t>(nq) * 8);
    GLMX_CUDA(cudaMemcpyAsync(g->d_qemb.p, q.data(), q.size() * 4, cudaMemcpyHostToDevice, s));
    GLMX_CUDA(cudaMemsetAsync(g->d_best.p, 0, static_cast<size_t>(nq) * 8, s));
    GLMX_CUDA(cudaEventRecord(g->ev0, s));
    nearest_top1(g->d_emb.as<float>(), static_cast<int>(g->idx_node.size()), dpad,
                 g->d_qemb.as<float>(), nq, g->d_best.as<unsigned long long>(), s, /*packed=*/true);
    GLMX_CUDA(cudaEventRecord(g->ev1, s));
    best.resize(nq);
    GLMX_CUDA(cudaMemcpyAsync(best.data(), g->d_best.p, nq * 8, cudaMemcpyDeviceToHost, s));
    GLMX_CUDA(cudaStreamSynchronize(s));
    float ms = 0.f;
    GLMX_CUDA(cudaEventElapsedTime(&ms, g->ev0, g->ev1));
    total_ms += ms;
    for (int k = 0; k < nq; ++k) {
      const uint32_t row = 0xFFFFFFFFu - static_cast<uint32_t>(best[k] & 0xFFFFFFFFu);
      if (best[k] != 0 && row < g->idx_node.size() && g->idx_node[row] == qnode[c0 + k])
        unique[qnode[c0 + k]] = 1;
    }
  }
  if (scan_ms) *scan_ms = total_ms;
  *out = glmx::generate_workload_jsonl(g->host, unique, seed, n, ratio);
  return GLMX_OK;
}

// ======================================================================== K2 gather hook
int kv_gather_run_impl(void* pool_base, uint64_t n_pages_pool, uint32_t n_layers, uint32_t Hkv,
                       uint32_t block_tokens, uint32_t hd, uint32_t layer, uint32_t kv,
                       const int32_t* pages, uint64_t n, void* out, int impl, int reps,
                       cudaStream_t s, float* out_ms) {
  if (n == 0) return GLMX_OK;
  if (layer >= n_layers || kv > 1 || reps < 1) throw Error(GLMX_ERR_ARG, "bad gather arguments");
  for (uint64_t i = 0; i < n; ++i)
    if (pages[i] < 0 || static_cast<uint64_t>(pages[i]) >= n_pages_pool) throw Error(GLMX_ERR_ARG, "page out of range");
  PoolGeom geom{static_cast<__nv_bfloat16*>(pool_base), n_layers, Hkv, block_tokens, hd};
  DBuf d_pages;
  d_pages.reserve(n * 4);
  GLMX_CUDA(cudaMemcpyAsync(d_pages.p, pages, n * 4, cudaMemcpyHostToDevice, s));
  cudaEvent_t e0, e1;
  GLMX_CUDA(cudaEventCreate(&e0));
  GLMX_CUDA(cudaEventCreate(&e1));
  float ms = 0.f;
  try {
    GLMX_CUDA(cudaEventRecord(e0, s));
    for (int r = 0; r < reps; ++r) {
      if (impl == 0)
        kv_gather_tma(geom, layer, kv, d_pages.as<int32_t>(), static_cast<int>(n), static_cast<__nv_bfloat16*>(out), s);
      else
        kv_gather(geom, layer, kv, d_pages.as<int32_t>(), static_cast<int>(n), static_cast<__nv_bfloat16*>(out), s);
    }
    GLMX_CUDA(cudaEventRecord(e1, s));
    GLMX_CUDA(cudaEventSynchronize(e1));
    GLMX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  } catch (...) {
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    throw;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (out_ms) *out_ms = ms / static_cast<float>(reps);
  return GLMX_OK;
}

