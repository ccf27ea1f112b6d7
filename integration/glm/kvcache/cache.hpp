// Drop-in replacement for the reference's glm/kvcache/cache.hpp (cache.hpp:1-99): the same types
// and the same KvCacheState interface, implemented over libglmx's C ABI (include/glmx.h).
// A maintainer puts this directory ahead of the reference's include/ and links libglmx.so
// instead of compiling src/kvcache/cache.cpp; Orchestrator (orchestrator.cpp:81-97, 147-154) and
// run_bench (bench.cpp:55, 138) compile unchanged.  oracle/Makefile's `dropin` target does exactly
// that and tests/test_dropin.py checks run_bench's report is identical to the stock build's.
//
// The handle is bookkeeping-only (device -1), like the reference's simulator; the GPU path adds a
// device pool and a glmx_engine on top.  Errors come back as the reference's
// exception classes (error.hpp:29-137), with the same partial-state semantics.
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "glm/config.hpp"
#include "glm/error.hpp"
#include "glm/kvcache/tier.hpp"
#include "glm/kvcache/tokenizer.hpp"
#include "glmx.h"

namespace glm {

using BlockId = std::uint64_t;

struct CacheBlock {
  BlockId id = 0;
  std::optional<BlockId> parent;
  Tier tier = Tier::IV;
  std::uint64_t last_used = 0;
  std::string session;
};

struct TierRange {
  std::size_t begin = 0;
  std::size_t end = 0;
  Tier tier = Tier::IV;
};
using TierMap = std::vector<TierRange>;

struct PrefillReport {
  std::size_t cached_tokens = 0;
  std::size_t computed_tokens = 0;
  std::size_t tail_tokens = 0;
  std::vector<BlockId> evicted;
  std::size_t total_computed() const { return computed_tokens + tail_tokens; }
};

struct CacheCounters {
  std::int64_t hits = 0;
  std::int64_t misses = 0;
  std::int64_t evictions_by_tier[4] = {0, 0, 0, 0};
  double hit_rate() const {
    std::int64_t total = hits + misses;
    return total == 0 ? 0.0 : static_cast<double>(hits) / static_cast<double>(total);
  }
};

class KvCacheState {
 public:
  KvCacheState(std::size_t capacity_blocks, std::size_t block_tokens,
               CachePolicy policy = CachePolicy::Priority)
      : capacity_(capacity_blocks), block_tokens_(block_tokens), policy_(policy) {
    glmx_kv_config c{};
    c.capacity_blocks = capacity_blocks;
    c.block_tokens = static_cast<uint32_t>(block_tokens);
    c.policy = policy == CachePolicy::Priority ? GLMX_POLICY_PRIORITY : GLMX_POLICY_LRU;
    c.device = -1;
    check(glmx_kv_create(&c, &h_));
  }
  ~KvCacheState() { glmx_kv_destroy(h_); }
  KvCacheState(const KvCacheState&) = delete;
  KvCacheState& operator=(const KvCacheState&) = delete;

  PrefillReport prefill(const TokenSeq& prompt, const TierMap& tiers, const std::string& session) {
    std::string bytes;
    std::vector<uint64_t> offs{0};
    offs.reserve(prompt.size() + 1);
    for (const auto& t : prompt) {
      bytes += t;
      offs.push_back(bytes.size());
    }
    std::vector<glmx_tier_range> tr;
    tr.reserve(tiers.size());
    for (const auto& r : tiers) tr.push_back({r.begin, r.end, static_cast<int32_t>(r.tier), 0});
    glmx_prefill_report rep{};
    std::vector<uint64_t> ev(prompt.size() / (block_tokens_ ? block_tokens_ : 1) + 8);
    check(glmx_kv_prefill(h_, bytes.data(), offs.data(), prompt.size(), tr.data(), tr.size(),
                          session.c_str(), &rep, nullptr, 0, ev.data(), ev.size()));
    if (rep.n_evicted > ev.size()) {
      ev.resize(rep.n_evicted);
      glmx_kv_last_evicted(h_, ev.data(), ev.size());
    }
    PrefillReport out;
    out.cached_tokens = rep.cached_tokens;
    out.computed_tokens = rep.computed_tokens;
    out.tail_tokens = rep.tail_tokens;
    out.evicted.assign(ev.begin(), ev.begin() + static_cast<std::ptrdiff_t>(rep.n_evicted));
    return out;
  }

  std::vector<BlockId> evict(std::size_t n) {
    std::vector<uint64_t> out(n > 0 ? n : 1);
    uint64_t got = 0;
    check(glmx_kv_evict(h_, n, out.data(), out.size(), &got));
    out.resize(got);
    return out;
  }

  void set_tier(const std::string& session, Tier from_tier, Tier to_tier) {
    check(glmx_kv_set_tier(h_, session.c_str(), static_cast<int32_t>(from_tier),
                           static_cast<int32_t>(to_tier)));
  }

  std::size_t resident_blocks() const { return glmx_kv_resident(h_, nullptr, nullptr, nullptr, nullptr, 0); }
  std::size_t capacity_blocks() const { return capacity_; }
  std::size_t block_tokens() const { return block_tokens_; }
  CachePolicy policy() const { return policy_; }
  const CacheCounters& counters() const {
    int64_t c[6];
    glmx_kv_counters(h_, c);
    counters_.hits = c[0];
    counters_.misses = c[1];
    for (int t = 0; t < 4; ++t) counters_.evictions_by_tier[t] = c[2 + t];
    return counters_;
  }

  bool is_resident(BlockId id) const { return glmx_kv_block(h_, id, nullptr, nullptr, nullptr, nullptr) == 1; }
  const CacheBlock* block(BlockId id) const {
    CacheBlock b;
    if (!fetch(id, b)) return nullptr;
    return &(blocks_[id] = std::move(b));
  }
  std::vector<CacheBlock> resident_snapshot() const {
    const uint64_t n = resident_blocks();
    std::vector<uint64_t> ids(n ? n : 1);
    glmx_kv_resident(h_, ids.data(), nullptr, nullptr, nullptr, n);
    std::vector<CacheBlock> out(n);
    for (uint64_t i = 0; i < n; ++i) fetch(ids[i], out[i]);
    return out;
  }

  std::string snapshot_json() const {
    std::string s(512, '\0');
    int64_t n = glmx_kv_snapshot_json(h_, s.data(), s.size());
    if (n > static_cast<int64_t>(s.size())) {
      s.resize(static_cast<std::size_t>(n));
      n = glmx_kv_snapshot_json(h_, s.data(), s.size());
    }
    s.resize(static_cast<std::size_t>(n));
    return s;
  }

  void force_insert(BlockId id, Tier tier, std::uint64_t last_used, const std::string& session) {
    check(glmx_kv_force_insert(h_, id, static_cast<int32_t>(tier), last_used, session.c_str()));
  }

  static std::vector<BlockId> chain_ids(const TokenSeq& prompt, std::size_t block_tokens) {
    std::string bytes;
    std::vector<uint64_t> offs{0};
    for (const auto& t : prompt) {
      bytes += t;
      offs.push_back(bytes.size());
    }
    std::vector<BlockId> out(block_tokens ? prompt.size() / block_tokens + 1 : 1);
    out.resize(glmx_kv_chain_ids(bytes.data(), offs.data(), prompt.size(),
                                 static_cast<uint32_t>(block_tokens), out.data()));
    return out;
  }

 private:
  bool fetch(BlockId id, CacheBlock& b) const {
    int32_t tier = 0, has_parent = 0;
    uint64_t lu = 0, parent = 0;
    if (glmx_kv_block(h_, id, &tier, &lu, &parent, &has_parent) != 1) return false;
    b.id = id;
    b.tier = static_cast<Tier>(tier);
    b.last_used = lu;
    if (has_parent) b.parent = parent;
    char buf[4096];
    const int64_t n = glmx_kv_block_session(h_, id, buf, sizeof buf);
    b.session.assign(buf, static_cast<std::size_t>(n < 0 ? 0 : std::min<int64_t>(n, sizeof buf)));
    return true;
  }
  static void check(int st) {  // status -> the reference's exception classes
    if (st == GLMX_OK) return;
    const char* m = glmx_last_error();
    if (st == GLMX_ERR_CACHE_EXHAUSTED) throw CacheExhausted(m);
    if (st == GLMX_ERR_CONFIG) throw ConfigError(m);
    throw GlmError(m);
  }

  glmx_kv* h_ = nullptr;
  std::size_t capacity_, block_tokens_;
  CachePolicy policy_;
  mutable CacheCounters counters_;
  mutable std::map<BlockId, CacheBlock> blocks_;
};

}  // namespace glm
