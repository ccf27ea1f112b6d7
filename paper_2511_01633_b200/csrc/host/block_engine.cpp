#include "block_engine.hpp"

#include <algorithm>
#include <cstdio>

namespace glmx {

void PagePool::reset(uint64_t n) {
  total_ = n;
  free_.clear();
  deferred_.clear();
  deferred_base_ = 0;
  free_.reserve(n);
  // LIFO: page 0 is handed out first.
  for (uint64_t i = n; i-- > 0;) free_.push_back(static_cast<int32_t>(i));
}

bool PagePool::try_alloc(int32_t& p) {
  if (free_.empty()) return false;
  p = free_.back();
  free_.pop_back();
  return true;
}

int32_t PagePool::alloc() {
  int32_t p;
  if (!try_alloc(p))
    throw Error(GLMX_ERR_POOL, "kv page pool exhausted (" + std::to_string(total_) +
                                   " pages, " + std::to_string(deferred_.size()) +
                                   " deferred); raise headroom_pages");
  return p;
}

void PagePool::release_deferred() {
  free_.insert(free_.end(), deferred_.rbegin(), deferred_.rend());
  deferred_base_ += deferred_.size();
  deferred_.clear();
}

void PagePool::release_before(uint64_t m) {
  if (m <= deferred_base_) return;
  const size_t n = static_cast<size_t>(std::min<uint64_t>(m - deferred_base_, deferred_.size()));
  free_.insert(free_.end(), std::make_reverse_iterator(deferred_.begin() + n),
               std::make_reverse_iterator(deferred_.begin()));
  deferred_.erase(deferred_.begin(), deferred_.begin() + n);
  deferred_base_ += n;
}

BlockEngine::BlockEngine(uint64_t capacity, uint32_t block_tokens, int policy,
                         uint64_t pool_pages)
    : cap_(capacity), B_(block_tokens), policy_(policy), pool_(pool_pages) {
  if (B_ == 0) throw Error(GLMX_ERR_CONFIG, "kv block size must be positive");  // cache.cpp:28
  if (policy_ != GLMX_POLICY_PRIORITY && policy_ != GLMX_POLICY_LRU)
    throw Error(GLMX_ERR_ARG, "unknown cache policy");
  sessions_.push_back(std::string());
  session_ids_[std::string()] = 0;
}

int32_t BlockEngine::intern(const std::string& s) {
  auto it = session_ids_.find(s);
  if (it != session_ids_.end()) return it->second;
  int32_t id = static_cast<int32_t>(sessions_.size());
  sessions_.push_back(s);
  session_ids_.emplace(s, id);
  return id;
}

// cache.cpp:13-21: seed 1469598103934665603 (NOT the FNV offset basis), root "parent"
// 0xb10c0000c0ffee, and the 8-byte separator fnv1a_u64(0x1f) after every token.
void BlockEngine::chain_ids(const TokenSpans& t, uint32_t B, std::vector<uint64_t>& out) {
  out.clear();
  uint64_t parent = 0xb10c0000c0ffeeULL;
  for (uint64_t b = 0; (b + 1) * B <= t.n; ++b) {
    uint64_t h = fnv1a_u64(parent, 1469598103934665603ULL);
    for (uint64_t i = b * B; i < (b + 1) * B; ++i) {
      h = fnv1a(t.bytes + t.offsets[i], t.offsets[i + 1] - t.offsets[i], h);
      h = fnv1a_u64(0x1f, h);
    }
    out.push_back(h);
    parent = h;
  }
}

// cache.cpp:42-52: a block straddling a tier boundary keeps the strongest (lowest) tier.
int BlockEngine::strongest_tier_over(const glmx_tier_range* t, uint64_t n, uint64_t b,
                                     uint64_t e) {
  int best = GLMX_TIER_IV;
  for (uint64_t i = 0; i < n; ++i) {
    if (t[i].end <= b || t[i].begin >= e) continue;
    if (t[i].tier < best) best = t[i].tier;
  }
  return best;
}

void BlockEngine::touch(Block& b, uint64_t stamp, int want_tier) {
  order_erase(b);
  b.last_used = stamp;
  if (want_tier < b.tier) b.tier = want_tier;  // upgrade only; owner unchanged (cache.cpp:80)
  order_insert(b);
}

void BlockEngine::erase_block(uint64_t id) {
  auto it = resident_.find(id);
  Block& b = it->second;
  order_erase(b);
  auto o = owned_.find(b.session);
  if (o != owned_.end()) o->second.erase(id);
  pool_.defer(b.page);
  resident_.erase(it);
}

void BlockEngine::prefill(const TokenSpans& toks, const glmx_tier_range* tiers,
                          uint64_t n_tiers, const std::string& session, PrefillResult& out) {
  // TierMap must cover [0, len) with disjoint ordered ranges (cache.cpp:56-63).
  uint64_t expect = 0;
  for (uint64_t i = 0; i < n_tiers; ++i) {
    if (tiers[i].begin != expect || tiers[i].end < tiers[i].begin)
      throw Error(GLMX_ERR_GLM, "tier map must cover the prompt with ordered disjoint ranges");
    if (tiers[i].tier < GLMX_TIER_I || tiers[i].tier > GLMX_TIER_IV)
      throw Error(GLMX_ERR_ARG, "tier out of range");
    expect = tiers[i].end;
  }
  if (expect != toks.n) throw Error(GLMX_ERR_GLM, "tier map does not cover the prompt");

  out.cached = out.computed = 0;
  out.evicted.clear();
  out.pages.clear();
  last_evicted_.clear();
  chain_ids(toks, B_, out.ids);
  const uint64_t full = out.ids.size();
  out.tail = toks.n - full * B_;
  out.pages.resize(full, -1);
  out.fresh.assign(full, 0);
  out.stale.assign(full, 0);

  // Maximal resident chain prefix counts as cached (cache.cpp:70-81).
  uint64_t hit = 0;
  while (hit < full) {
    auto it = resident_.find(out.ids[hit]);
    if (it == resident_.end()) break;
    out.pages[hit] = it->second.page;
    out.stale[hit] = it->second.stale;
    ++hit;
  }
  out.hit_blocks = hit;
  out.cached = hit * B_;
  hits_ += static_cast<int64_t>(hit);
  for (uint64_t b = 0; b < hit; ++b)
    touch(resident_.find(out.ids[b])->second, ++clock_,
          strongest_tier_over(tiers, n_tiers, b * B_, (b + 1) * B_));

  const int32_t sess = intern(session);
  for (uint64_t b = hit; b < full; ++b) {  // cache.cpp:83-105
    out.computed += B_;
    ++misses_;
    int tier = strongest_tier_over(tiers, n_tiers, b * B_, (b + 1) * B_);
    auto it = resident_.find(out.ids[b]);
    if (it != resident_.end()) {
      // Orphaned descendant of an evicted block: recomputed, stamp refreshed, tier upgraded.
      touch(it->second, ++clock_, tier);
      out.pages[b] = it->second.page;
      out.stale[b] = it->second.stale;
      continue;
    }
    if (resident_.size() >= cap_) {
      auto ev = evict(resident_.size() - cap_ + 1);  // may throw CacheExhausted: partial state
      out.evicted.insert(out.evicted.end(), ev.begin(), ev.end());
      last_evicted_ = out.evicted;
    }
    Block blk;
    blk.id = out.ids[b];
    blk.has_parent = b > 0;
    blk.parent = b > 0 ? out.ids[b - 1] : 0;
    blk.tier = tier;
    blk.last_used = ++clock_;
    blk.session = tier == GLMX_TIER_I ? 0 : sess;
    blk.page = pool_.alloc();
    out.pages[b] = blk.page;
    out.fresh[b] = 1;
    out.stale[b] = 1;
    order_insert(blk);
    owned_[blk.session].insert(blk.id);
    resident_.emplace(blk.id, blk);
  }
  last_evicted_ = out.evicted;
}

std::vector<uint64_t> BlockEngine::evict(uint64_t n) {
  if (n == 0) return {};
  const bool prio = policy_ == GLMX_POLICY_PRIORITY;
  uint64_t candidates = 0;
  for (int t = prio ? 1 : 0; t < 4; ++t) candidates += order_[t].size();
  if (candidates < n)
    throw Error(GLMX_ERR_CACHE_EXHAUSTED, "need " + std::to_string(n) +
                                              " evictable blocks, have " +
                                              std::to_string(candidates));
  std::vector<uint64_t> out;
  out.reserve(n);
  for (uint64_t i = 0; i < n; ++i) {
    int pick = -1;
    if (prio) {
      // Weakest tier first (IV, III, II), LRU then id within a tier (cache.cpp:126-132).
      for (int t = 3; t >= 1; --t)
        if (!order_[t].empty()) {
          pick = t;
          break;
        }
    } else {
      // Tier-blind (last_used, id) order (cache.cpp:133-137).
      for (int t = 0; t < 4; ++t)
        if (!order_[t].empty() && (pick < 0 || *order_[t].begin() < *order_[pick].begin()))
          pick = t;
    }
    uint64_t id = order_[pick].begin()->second;
    out.push_back(id);
    ++ev_[pick];
    erase_block(id);
  }
  return out;
}

void BlockEngine::set_tier(const std::string& session, int from, int to) {
  auto s = session_ids_.find(session);
  if (s == session_ids_.end()) return;
  auto o = owned_.find(s->second);
  if (o == owned_.end()) return;
  for (uint64_t id : o->second) {
    Block& b = resident_.find(id)->second;
    if (b.tier != from) continue;
    order_erase(b);
    b.tier = to;
    order_insert(b);
  }
}

void BlockEngine::force_insert(uint64_t id, int tier, uint64_t last_used,
                               const std::string& session) {
  int32_t page = -1;
  bool stale = true;  // a new block's page holds no KV
  auto it = resident_.find(id);
  if (it != resident_.end()) {
    page = it->second.page;
    stale = it->second.stale;
    order_erase(it->second);
    auto o = owned_.find(it->second.session);
    if (o != owned_.end()) o->second.erase(id);
    resident_.erase(it);
  } else if (!pool_.try_alloc(page)) {
    page = -1;
  }
  Block b;
  b.id = id;
  b.tier = tier;
  b.last_used = last_used;
  b.session = intern(session);
  b.page = page;
  b.stale = stale;
  order_insert(b);
  owned_[b.session].insert(id);
  resident_.emplace(id, b);
  clock_ = std::max(clock_, last_used);
}

void BlockEngine::set_stale(uint64_t id, bool stale) {
  auto it = resident_.find(id);
  if (it != resident_.end()) it->second.stale = stale;
}

int32_t BlockEngine::ensure_page(uint64_t id) {
  Block& b = resident_.at(id);
  if (b.page < 0) b.page = pool_.alloc();
  return b.page;
}

const Block* BlockEngine::block(uint64_t id) const {
  auto it = resident_.find(id);
  return it == resident_.end() ? nullptr : &it->second;
}

std::vector<const Block*> BlockEngine::resident_sorted() const {
  std::vector<const Block*> v;
  v.reserve(resident_.size());
  for (const auto& kv : resident_) v.push_back(&kv.second);
  std::sort(v.begin(), v.end(), [](const Block* a, const Block* b) { return a->id < b->id; });
  return v;
}

// cache.cpp:178-189 (nlohmann dump: keys sorted, doubles shortest round-trip).
std::string BlockEngine::snapshot_json() const {
  int64_t total = hits_ + misses_;
  double rate = total == 0 ? 0.0 : static_cast<double>(hits_) / static_cast<double>(total);
  char rate_buf[64];
  // %.17g round-trips; trim to the shortest representation that still round-trips.
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(rate_buf, sizeof(rate_buf), "%.*g", prec, rate);
    if (std::strtod(rate_buf, nullptr) == rate) break;
  }
  std::string r = rate_buf;
  if (r.find_first_of(".e") == std::string::npos) r += ".0";
  char buf[512];
  std::snprintf(buf, sizeof(buf),
                "{\"evictions_by_tier\":{\"I\":%lld,\"II\":%lld,\"III\":%lld,\"IV\":%lld},"
                "\"hit_rate\":%s,\"hits\":%lld,\"misses\":%lld,\"resident_blocks\":%llu}",
                static_cast<long long>(ev_[0]), static_cast<long long>(ev_[1]),
                static_cast<long long>(ev_[2]), static_cast<long long>(ev_[3]), r.c_str(),
                static_cast<long long>(hits_), static_cast<long long>(misses_),
                static_cast<unsigned long long>(resident_.size()));
  return buf;
}

}  // namespace glmx
