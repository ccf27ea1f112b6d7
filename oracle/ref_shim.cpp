// TEST INFRASTRUCTURE ONLY (oracle/_ref/libglmref.so).
//
// extern "C" shim over the UNMODIFIED reference classes so tests (ctypes) and the bench's
// reference arm can drive the reference itself:
//   * KvCacheState (cache.hpp:56-99)            -> ref_kv_*
//   * KvCacheState::chain_ids (cache.cpp:31-40) -> ref_chain_ids
//   * Retriever::node_info_rendered (retriever.cpp:123-129) over PropertyGraph::load /
//     synth_graph (graph_store.cpp:38, workload.cpp:36)   -> ref_graph_*, ref_node_info_rendered
//   * TemplateSet::render_* (templates.cpp:189-223)        -> ref_render
//   * run_bench (bench.cpp:45-161), and a ScriptedProvider round-robin identical to
//     bench.cpp:65-83, with the orchestrator's prefill/set_tier call sequence recorded
//     (ref_shim_rec.cpp)                                  -> ref_run_bench, ref_run_scripted
// Product code never links this.
#include <cstdint>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "glm/agents/templates.hpp"
#include "glm/bench/bench.hpp"
#include "glm/bench/workload.hpp"
#include "glm/embed/index.hpp"
#include "glm/error.hpp"
#include "glm/graph/graph_store.hpp"
#include "glm/kvcache/cache.hpp"
#include "glm/kvcache/tokenizer.hpp"
#include "glm/llm/scripted.hpp"
#include "glm/orchestrator/orchestrator.hpp"
#include "glm/retrieve/retriever.hpp"
#include "glm/embed/embedder.hpp"
#include "json.hpp"

using nlohmann::json;

namespace {
thread_local std::string g_err;
std::vector<std::string> g_trace;  // JSONL lines
bool g_recording = false;

glm::TokenSeq tokens_from(const char* bytes, const std::uint64_t* offs, std::uint64_t n) {
  glm::TokenSeq t;
  t.reserve(n);
  for (std::uint64_t i = 0; i < n; ++i) t.emplace_back(bytes + offs[i], offs[i + 1] - offs[i]);
  return t;
}

int64_t copy_out(const std::string& s, char* buf, std::uint64_t cap) {
  if (buf && cap > 0) {
    std::size_t n = std::min<std::size_t>(s.size(), cap);
    std::memcpy(buf, s.data(), n);
  }
  return static_cast<int64_t>(s.size());
}

int status_of(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const glm::CacheExhausted*>(&e)) return 2;
  if (dynamic_cast<const glm::ConfigError*>(&e)) return 3;
  if (dynamic_cast<const glm::RetrievalError*>(&e)) return 4;
  if (dynamic_cast<const glm::UnknownNode*>(&e)) return 4;
  if (dynamic_cast<const glm::GlmError*>(&e)) return 1;
  return 9;
}

json tiers_json(const glm::TierMap& t) {
  json a = json::array();
  for (const auto& r : t) a.push_back({r.begin, r.end, static_cast<int>(r.tier)});
  return a;
}
}  // namespace

namespace glm {
PrefillReport glmref_real_prefill(KvCacheState* kv, const TokenSeq& p, const TierMap& t,
                                  const std::string& s) {
  return kv->prefill(p, t, s);
}
void glmref_real_set_tier(KvCacheState* kv, const std::string& s, Tier from, Tier to) {
  kv->set_tier(s, from, to);
}
// segment texts kv_prefill tokenized since the last recorded prefill (rec_tokenize.hpp)
thread_local std::vector<std::string> g_seg_texts;
void glmref_record_segment_text(std::string_view text) {
  if (g_recording) g_seg_texts.emplace_back(text);
}
void glmref_record_prefill(const TokenSeq& p, const TierMap& t, const std::string& s,
                           const PrefillReport* rep, const char* error) {
  if (!g_recording) return;
  json j;
  j["op"] = "prefill";
  j["session"] = s;
  j["tokens"] = p;
  j["tiers"] = tiers_json(t);
  // the PromptSegments behind this call: (text, tier) per part.  A part's tier is the TierMap
  // tier at its first token (kv_prefill gave all its tokens that tier); empty parts (skipped by
  // kv_prefill) carry the previous part's tier.
  json segs = json::array();
  std::size_t at = 0;
  int last_tier = 0;
  for (const auto& text : g_seg_texts) {
    const std::size_t n = glm::tokenize(text).size();
    int tier = last_tier;
    if (n > 0)
      for (const auto& r : t)
        if (r.begin <= at && at < r.end) tier = static_cast<int>(r.tier);
    segs.push_back(json::array({text, tier}));
    at += n;
    last_tier = tier;
  }
  g_seg_texts.clear();
  if (at == p.size()) j["segments"] = segs;
  if (rep) {
    j["cached"] = rep->cached_tokens;
    j["computed"] = rep->computed_tokens;
    j["tail"] = rep->tail_tokens;
    j["evicted"] = rep->evicted;
  } else {
    j["error"] = error;
  }
  g_trace.push_back(j.dump());
}
void glmref_record_set_tier(const std::string& s, Tier from, Tier to) {
  if (!g_recording) return;
  json j;
  j["op"] = "set_tier";
  j["session"] = s;
  j["from"] = static_cast<int>(from);
  j["to"] = static_cast<int>(to);
  g_trace.push_back(j.dump());
}
}  // namespace glm

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- KvCacheState
void* ref_kv_create(std::uint64_t cap, std::uint64_t block_tokens, int policy) {
  try {
    return new glm::KvCacheState(cap, block_tokens,
                                 policy == 0 ? glm::CachePolicy::Priority
                                             : glm::CachePolicy::PlainLru);
  } catch (const std::exception& e) {
    status_of(e);
    return nullptr;
  }
}
void ref_kv_destroy(void* h) { delete static_cast<glm::KvCacheState*>(h); }

int ref_kv_prefill(void* h, const char* bytes, const std::uint64_t* offs, std::uint64_t n_tok,
                   const std::uint64_t* tiers, std::uint64_t n_tiers, const char* session,
                   std::uint64_t* rep3, std::uint64_t* evicted, std::uint64_t ev_cap,
                   std::uint64_t* n_ev) {
  auto* kv = static_cast<glm::KvCacheState*>(h);
  glm::TokenSeq toks = tokens_from(bytes, offs, n_tok);
  glm::TierMap tm;
  for (std::uint64_t i = 0; i < n_tiers; ++i)
    tm.push_back({tiers[3 * i], tiers[3 * i + 1], static_cast<glm::Tier>(tiers[3 * i + 2])});
  try {
    glm::PrefillReport r = kv->prefill(toks, tm, session);
    rep3[0] = r.cached_tokens;
    rep3[1] = r.computed_tokens;
    rep3[2] = r.tail_tokens;
    *n_ev = r.evicted.size();
    for (std::size_t i = 0; i < r.evicted.size() && i < ev_cap; ++i) evicted[i] = r.evicted[i];
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

int ref_kv_evict(void* h, std::uint64_t n, std::uint64_t* out, std::uint64_t cap,
                 std::uint64_t* n_out) {
  try {
    auto ids = static_cast<glm::KvCacheState*>(h)->evict(n);
    *n_out = ids.size();
    for (std::size_t i = 0; i < ids.size() && i < cap; ++i) out[i] = ids[i];
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

void ref_kv_set_tier(void* h, const char* session, int from, int to) {
  static_cast<glm::KvCacheState*>(h)->set_tier(session, static_cast<glm::Tier>(from),
                                               static_cast<glm::Tier>(to));
}

void ref_kv_force_insert(void* h, std::uint64_t id, int tier, std::uint64_t last_used,
                         const char* session) {
  static_cast<glm::KvCacheState*>(h)->force_insert(id, static_cast<glm::Tier>(tier), last_used,
                                                   session);
}

void ref_kv_counters(void* h, std::int64_t* out6) {
  const auto& c = static_cast<glm::KvCacheState*>(h)->counters();
  out6[0] = c.hits;
  out6[1] = c.misses;
  for (int t = 0; t < 4; ++t) out6[2 + t] = c.evictions_by_tier[t];
}

// Resident blocks sorted by id: ids, tiers, last_used and parent (0 = none).
std::uint64_t ref_kv_resident(void* h, std::uint64_t* ids, std::int32_t* tiers,
                              std::uint64_t* last_used, std::uint64_t* parents,
                              std::uint64_t cap) {
  auto snap = static_cast<glm::KvCacheState*>(h)->resident_snapshot();
  for (std::size_t i = 0; i < snap.size() && i < cap; ++i) {
    ids[i] = snap[i].id;
    tiers[i] = static_cast<std::int32_t>(snap[i].tier);
    last_used[i] = snap[i].last_used;
    parents[i] = snap[i].parent ? *snap[i].parent : 0;
  }
  return snap.size();
}

int64_t ref_kv_block_session(void* h, std::uint64_t id, char* buf, std::uint64_t cap) {
  const glm::CacheBlock* b = static_cast<glm::KvCacheState*>(h)->block(id);
  if (!b) return -1;
  return copy_out(b->session, buf, cap);
}

int64_t ref_kv_snapshot_json(void* h, char* buf, std::uint64_t cap) {
  return copy_out(static_cast<glm::KvCacheState*>(h)->snapshot_json(), buf, cap);
}

std::uint64_t ref_chain_ids(const char* bytes, const std::uint64_t* offs, std::uint64_t n_tok,
                            std::uint64_t block_tokens, std::uint64_t* out) {
  auto ids = glm::KvCacheState::chain_ids(tokens_from(bytes, offs, n_tok), block_tokens);
  for (std::size_t i = 0; i < ids.size(); ++i) out[i] = ids[i];
  return ids.size();
}

// Whitespace tokenizer (tokenizer.hpp:14-25): writes n+1 byte offsets pairs (begin,end) per token.
std::uint64_t ref_tokenize(const char* text, std::uint64_t len, std::uint64_t* begins,
                           std::uint64_t* ends, std::uint64_t cap) {
  std::string_view sv(text, len);
  glm::TokenSeq t = glm::tokenize(sv);
  // Recover spans by re-scanning (tokenize returns copies).
  std::uint64_t i = 0, k = 0;
  for (const auto& tok : t) {
    std::size_t at = sv.find(tok, i);
    if (k < cap) {
      begins[k] = at;
      ends[k] = at + tok.size();
    }
    i = at + tok.size();
    ++k;
  }
  return k;
}

// ---------------------------------------------------------------- graph + retriever
struct RefGraph {
  glm::PropertyGraph g;
};

void* ref_graph_load(const char* path) {
  try {
    return new RefGraph{glm::PropertyGraph::load(path)};
  } catch (const std::exception& e) {
    status_of(e);
    return nullptr;
  }
}

void* ref_synth_graph(std::uint64_t seed, int nodes) {
  try {
    glm::SynthGraphOptions o;
    o.seed = seed;
    o.nodes = nodes;
    return new RefGraph{glm::synth_graph(o)};
  } catch (const std::exception& e) {
    status_of(e);
    return nullptr;
  }
}

int ref_graph_save(void* g, const char* path) {
  try {
    static_cast<RefGraph*>(g)->g.save(path);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

void ref_graph_free(void* g) { delete static_cast<RefGraph*>(g); }

std::uint64_t ref_graph_node_count(void* g) { return static_cast<RefGraph*>(g)->g.node_count(); }

int64_t ref_graph_node_id(void* g, std::uint64_t i, char* buf, std::uint64_t cap) {
  const auto& ids = static_cast<RefGraph*>(g)->g.node_ids();
  if (i >= ids.size()) return -1;
  return copy_out(ids[i], buf, cap);
}

// Returns the rendered length (>=0), or -status on error (-4 = RetrievalError).
int64_t ref_node_info_rendered(void* g, const char* id, int k, int weight_mode, int directed,
                               char* buf, std::uint64_t cap) {
  auto* rg = static_cast<RefGraph*>(g);
  glm::Config cfg;
  cfg.chunk_k = k;
  cfg.chunk_weight_mode =
      weight_mode == 0 ? glm::ChunkWeightMode::TotalDegree : glm::ChunkWeightMode::ByEdgeType;
  cfg.chunk_directed = directed != 0;
  glm::VectorIndex index;  // node_info never touches the index
  glm::Retriever r(rg->g, index, cfg);
  try {
    return copy_out(r.node_info_rendered(id), buf, cap);
  } catch (const std::exception& e) {
    return -status_of(e);
  }
}

int64_t ref_retrieve_node(void* g, const char* text, char* buf, std::uint64_t cap) {
  auto* rg = static_cast<RefGraph*>(g);
  glm::Config cfg;
  glm::VectorIndex index = glm::VectorIndex::build(rg->g, cfg);
  glm::Retriever r(rg->g, index, cfg);
  try {
    return copy_out(r.retrieve_node(text), buf, cap);
  } catch (const std::exception& e) {
    return -status_of(e);
  }
}

// embed(text, dim) of the reference (embedder.cpp:19-36); writes padded_size floats
int64_t ref_embed(const char* text, int dim, float* out, std::uint64_t cap) {
  glm::Embedding e = glm::embed(text, dim);
  const std::uint64_t n = e.padded_size();
  for (std::uint64_t i = 0; i < n && i < cap; ++i) out[i] = e.data()[i];
  return static_cast<int64_t>(n);
}

// VectorIndex::nearest(text, k) ids (index.cpp:41-56), '\n'-joined; -status on error
int64_t ref_nearest(void* g, const char* text, int k, char* buf, std::uint64_t cap) {
  auto* rg = static_cast<RefGraph*>(g);
  try {
    glm::Config cfg;
    glm::VectorIndex index = glm::VectorIndex::build(rg->g, cfg);
    std::string out;
    for (const auto& s : index.nearest(text, k)) {
      if (!out.empty()) out += '\n';
      out += s.id;
    }
    return copy_out(out, buf, cap);
  } catch (const std::exception& e) {
    return -status_of(e);
  }
}

// generate_workload(seed, n, ratio, graph, default Config).serialize_jsonl(); -status on error
int64_t ref_generate_workload(void* g, std::uint64_t seed, int n, double ratio, char* buf,
                              std::uint64_t cap) {
  auto* rg = static_cast<RefGraph*>(g);
  try {
    glm::Config cfg;
    return copy_out(glm::generate_workload(seed, n, ratio, rg->g, cfg).serialize_jsonl(), buf, cap);
  } catch (const std::exception& e) {
    return -status_of(e);
  }
}

// ---------------------------------------------------------------- templates
// Renders a builtin template into (text, tier) segments, serialised as JSON [[tier, text], ...].
int64_t ref_render(const char* name, const char* a0, const char* a1, const char* a2, char* buf,
                   std::uint64_t cap) {
  try {
    glm::TemplateSet ts = glm::TemplateSet::builtin();
    std::string n = name;
    glm::PromptSegments seg;
    if (n == "classification") {
      seg = ts.render_classification(a0);
    } else if (n == "reasoning") {
      glm::Notebook nb;
      if (a1 && *a1) nb.append({"round1", a1});
      seg = ts.render_reasoning(a0, nb);
    } else if (n == "action") {
      seg = ts.render_action(a0);
    } else if (n == "action_repair") {
      seg = ts.render_action_repair(a0, a1, a2);
    } else if (n == "baseline_thought") {
      seg = ts.render_baseline_thought(a0, a1);
    } else if (n == "baseline_action") {
      seg = ts.render_baseline_action(a0, a1);
    } else {
      g_err = "unknown template";
      return -1;
    }
    json a = json::array();
    for (const auto& [t, tier] : seg.parts) a.push_back({static_cast<int>(tier), t});
    return copy_out(a.dump(), buf, cap);
  } catch (const std::exception& e) {
    return -status_of(e);
  }
}

// ---------------------------------------------------------------- trace recording
void ref_trace_clear() { g_trace.clear(); }
std::uint64_t ref_trace_len() { return g_trace.size(); }
int64_t ref_trace_line(std::uint64_t i, char* buf, std::uint64_t cap) {
  if (i >= g_trace.size()) return -1;
  return copy_out(g_trace[i], buf, cap);
}

// ---------------------------------------------------------------- bench drivers
// run_bench (bench.cpp:45) over synth_graph(seed_graph, nodes) and
// generate_workload(seed_wl, n, ratio). Records the bookkeeping trace when record != 0.
int64_t ref_run_bench(void* g, std::uint64_t seed_wl, int n, double ratio, int concurrency,
                      std::uint64_t cap_blocks, int policy, int glm_mode, int record, char* buf,
                      std::uint64_t cap) {
  auto* rg = static_cast<RefGraph*>(g);
  try {
    glm::BenchOptions opt;
    opt.glm_mode = glm_mode != 0;
    opt.policy = policy == 0 ? glm::CachePolicy::Priority : glm::CachePolicy::PlainLru;
    opt.concurrency = concurrency;
    opt.config.kv_capacity_blocks = cap_blocks;
    glm::Workload wl = glm::generate_workload(seed_wl, n, ratio, rg->g, opt.config);
    g_recording = record != 0;
    glm::BenchReport rep = glm::run_bench(wl, rg->g, opt);
    g_recording = false;
    return copy_out(rep.to_json(), buf, cap);
  } catch (const std::exception& e) {
    g_recording = false;
    return -status_of(e);
  }
}

// Scripted (ScriptedProvider, scripted.hpp:21-30) Graph-CoT run with the run_bench round-robin
// (bench.cpp:65-83). questions_jsonl lines: {"id","text","baseline":bool}. Output JSON:
// {"sessions":[{"id","answer","state","records":[[actor,in,out,cached,computed,span,outcome]]}],
//  "kv": snapshot_json}
int64_t ref_run_scripted(void* g, const char* trace_path, const char* questions_jsonl,
                         int concurrency, std::uint64_t cap_blocks, int policy, int chunk_k,
                         int record, char* buf, std::uint64_t cap) {
  auto* rg = static_cast<RefGraph*>(g);
  try {
    glm::Config cfg;
    cfg.kv_capacity_blocks = cap_blocks;
    cfg.kv_policy = policy == 0 ? glm::CachePolicy::Priority : glm::CachePolicy::PlainLru;
    cfg.chunk_k = chunk_k;
    cfg.timing_mode = glm::TimingMode::Simulated;
    glm::VectorIndex index = glm::VectorIndex::build(rg->g, cfg);
    glm::Retriever retriever(rg->g, index, cfg);
    glm::KvCacheState kv(cfg.kv_capacity_blocks, cfg.kv_block_tokens, cfg.kv_policy);
    glm::TemplateSet templates = glm::TemplateSet::builtin();
    glm::ScriptedProvider provider = glm::ScriptedProvider::load_jsonl(trace_path);
    glm::Orchestrator orch(retriever, templates, provider, kv, cfg);

    std::vector<glm::Session> sessions;
    std::istringstream qs(questions_jsonl);
    std::string line;
    while (std::getline(qs, line)) {
      if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
      json j = json::parse(line);
      sessions.push_back(orch.make_session(j.at("id").get<std::string>(),
                                           j.at("text").get<std::string>(),
                                           j.value("baseline", false)));
    }
    g_recording = record != 0;
    std::size_t admitted = 0;
    std::vector<std::size_t> active;
    std::size_t lanes = static_cast<std::size_t>(std::max(1, concurrency));
    while (admitted < sessions.size() || !active.empty()) {
      while (active.size() < lanes && admitted < sessions.size()) active.push_back(admitted++);
      for (std::size_t i = 0; i < active.size();) {
        glm::Session& s = sessions[active[i]];
        orch.run_step(s);
        if (s.state == glm::SessionState::Interrupted) orch.resume(s);
        if (s.terminal())
          active.erase(active.begin() + static_cast<std::ptrdiff_t>(i));
        else
          ++i;
      }
    }
    g_recording = false;
    json out;
    out["sessions"] = json::array();
    for (const auto& s : sessions) {
      json js;
      js["id"] = s.id;
      js["answer"] = s.answer;
      js["state"] = static_cast<int>(s.state);
      js["error"] = s.error ? glm::to_string(*s.error) : "";
      js["records"] = json::array();
      for (const auto& r : s.trace.records)
        js["records"].push_back({std::string(1, r.actor), r.tokens_in, r.tokens_out,
                                 r.cached_tokens, r.computed_tokens, r.span, r.outcome});
      out["sessions"].push_back(js);
    }
    out["kv"] = json::parse(kv.snapshot_json());
    return copy_out(out.dump(), buf, cap);
  } catch (const std::exception& e) {
    g_recording = false;
    return -status_of(e);
  }
}

// ---------------------------------------------------------------- rotation-granular scripted run
// The same round-robin as ref_run_scripted, one rotation per call, so a caller can time the
// reference's CPU path rotation by rotation (bench.py --impl reference).
struct RefScripted {
  glm::Config cfg;
  std::unique_ptr<glm::VectorIndex> index;
  std::unique_ptr<glm::Retriever> retriever;
  std::unique_ptr<glm::KvCacheState> kv;
  glm::TemplateSet templates = glm::TemplateSet::builtin();
  std::unique_ptr<glm::ScriptedProvider> provider;
  std::unique_ptr<glm::Orchestrator> orch;
  std::vector<glm::Session> sessions;
  std::size_t admitted = 0, lanes = 1;
  std::vector<std::size_t> active;
};

void* ref_scripted_open(void* g, const char* trace_path, const char* questions_jsonl,
                        int concurrency, std::uint64_t cap_blocks, int policy, int chunk_k) {
  auto* rg = static_cast<RefGraph*>(g);
  try {
    auto r = std::make_unique<RefScripted>();
    r->cfg.kv_capacity_blocks = cap_blocks;
    r->cfg.kv_policy = policy == 0 ? glm::CachePolicy::Priority : glm::CachePolicy::PlainLru;
    r->cfg.chunk_k = chunk_k;
    r->cfg.timing_mode = glm::TimingMode::Simulated;
    r->index = std::make_unique<glm::VectorIndex>(glm::VectorIndex::build(rg->g, r->cfg));
    r->retriever = std::make_unique<glm::Retriever>(rg->g, *r->index, r->cfg);
    r->kv = std::make_unique<glm::KvCacheState>(r->cfg.kv_capacity_blocks, r->cfg.kv_block_tokens,
                                                r->cfg.kv_policy);
    r->provider = std::make_unique<glm::ScriptedProvider>(glm::ScriptedProvider::load_jsonl(trace_path));
    r->orch = std::make_unique<glm::Orchestrator>(*r->retriever, r->templates, *r->provider, *r->kv,
                                                  r->cfg);
    std::istringstream qs(questions_jsonl);
    std::string line;
    while (std::getline(qs, line)) {
      if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
      json j = json::parse(line);
      r->sessions.push_back(r->orch->make_session(j.at("id").get<std::string>(),
                                                  j.at("text").get<std::string>(), false));
    }
    r->lanes = static_cast<std::size_t>(std::max(1, concurrency));
    return r.release();
  } catch (const std::exception& e) {
    status_of(e);
    return nullptr;
  }
}

// One rotation (bench.cpp:71-83).  Writes {"calls": [[session, actor, cached, computed], ...],
// "done": bool}: the C / R / A records the rotation's run_steps appended, in call order.
int64_t ref_scripted_rotation(void* h, char* buf, std::uint64_t cap) {
  auto* r = static_cast<RefScripted*>(h);
  try {
    while (r->active.size() < r->lanes && r->admitted < r->sessions.size())
      r->active.push_back(r->admitted++);
    json calls = json::array();
    for (std::size_t i = 0; i < r->active.size();) {
      glm::Session& s = r->sessions[r->active[i]];
      const std::size_t before = s.trace.records.size();
      r->orch->run_step(s);
      if (s.state == glm::SessionState::Interrupted) r->orch->resume(s);
      for (std::size_t k = before; k < s.trace.records.size(); ++k) {
        const auto& rec = s.trace.records[k];
        if (rec.actor == 'C' || rec.actor == 'R' || rec.actor == 'A')
          calls.push_back({s.id, std::string(1, rec.actor), rec.cached_tokens, rec.computed_tokens});
      }
      if (s.terminal())
        r->active.erase(r->active.begin() + static_cast<std::ptrdiff_t>(i));
      else
        ++i;
    }
    json out;
    out["calls"] = calls;
    out["done"] = r->admitted >= r->sessions.size() && r->active.empty();
    return copy_out(out.dump(), buf, cap);
  } catch (const std::exception& e) {
    return -status_of(e);
  }
}

int64_t ref_scripted_snapshot(void* h, char* buf, std::uint64_t cap) {
  return copy_out(static_cast<RefScripted*>(h)->kv->snapshot_json(), buf, cap);
}

void ref_scripted_close(void* h) { delete static_cast<RefScripted*>(h); }

}  // extern "C"
