// Host block engine: the reference's KvCacheState (cache.hpp:56-99, cache.cpp) re-designed for
// a device page pool.  Bookkeeping semantics are bit-exact with the reference (same hits,
// misses, tiers, owners, clock stamps, eviction order, exceptions and partial state); the data
// structures are not: O(1) residency lookups and O(log R) per-tier LRU order instead of the
// reference's std::map + full sort per evict (cache.cpp:116-138).  Each resident block also owns
// one physical page of the device pool; evicted blocks' pages are deferred-freed so a batch that
// is still in flight can read them (SURVEY.md §7 "hard parts" 2).
#pragma once

#include <cstdint>
#include <set>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <utility>
#include <vector>

#include "common.hpp"

namespace glmx {

struct Block {                // CacheBlock (cache.hpp:17-23) + physical page
  uint64_t id = 0;
  uint64_t parent = 0;
  bool has_parent = false;
  int tier = GLMX_TIER_IV;
  uint64_t last_used = 0;
  int32_t session = 0;        // interned owner; 0 == "" (shared)
  int32_t page = -1;          // physical page in the device pool, -1 = none (force_insert)
  // the page does not hold this block's KV yet: inserted by a prefill whose forward has not been
  // enqueued (or never was: a failed batch, a bookkeeping-only prefill, force_insert).  The
  // engine recomputes a stale block on its next use instead of attending over the page.
  bool stale = true;
};

// Deterministic physical-page allocator (LIFO free list).
class PagePool {
 public:
  explicit PagePool(uint64_t n = 0) { reset(n); }
  void reset(uint64_t n);
  int32_t alloc();            // throws Error(GLMX_ERR_POOL)
  bool try_alloc(int32_t& p);
  void defer(int32_t p) { if (p >= 0) deferred_.push_back(p); }
  void free_now(int32_t p) { if (p >= 0) free_.push_back(p); }
  void release_deferred();
  // deferred pages are numbered in order; mark() = number deferred so far.  release_before(m)
  // frees the ones deferred before mark m (pipelined epochs release with a lag)
  uint64_t mark() const { return deferred_base_ + deferred_.size(); }
  void release_before(uint64_t m);
  uint64_t total() const { return total_; }
  uint64_t free_count() const { return free_.size(); }
  uint64_t deferred_count() const { return deferred_.size(); }

 private:
  uint64_t total_ = 0;
  std::vector<int32_t> free_;
  std::vector<int32_t> deferred_;
  uint64_t deferred_base_ = 0;  // number of deferred pages released so far
};

struct PrefillResult {        // PrefillReport (cache.hpp:33-39) + block table
  uint64_t cached = 0, computed = 0, tail = 0;
  std::vector<uint64_t> evicted;
  std::vector<uint64_t> ids;     // chain ids of the full blocks
  std::vector<int32_t> pages;    // physical page per full block
  std::vector<uint8_t> fresh;    // 1 = inserted by this call (new page, KV not yet present)
  std::vector<uint8_t> stale;    // per full block: Block::stale at the end of the call
  uint64_t hit_blocks = 0;
};

class BlockEngine {
 public:
  BlockEngine(uint64_t capacity, uint32_t block_tokens, int policy, uint64_t pool_pages);

  // KvCacheState::prefill (cache.cpp:54-107).  Throws Error(GLMX_ERR_GLM) on a bad TierMap and
  // Error(GLMX_ERR_CACHE_EXHAUSTED) with partial state, exactly like the reference.
  void prefill(const TokenSpans& toks, const glmx_tier_range* tiers, uint64_t n_tiers,
               const std::string& session, PrefillResult& out);
  // KvCacheState::evict (cache.cpp:109-148)
  std::vector<uint64_t> evict(uint64_t n);
  // KvCacheState::set_tier (cache.cpp:150-153)
  void set_tier(const std::string& session, int from, int to);
  // KvCacheState::force_insert (cache.cpp:167-176)
  void force_insert(uint64_t id, int tier, uint64_t last_used, const std::string& session);
  // KvCacheState::chain_ids (cache.cpp:31-40)
  static void chain_ids(const TokenSpans& toks, uint32_t B, std::vector<uint64_t>& out);

  const Block* block(uint64_t id) const;
  // KV-presence flag of a resident block (no-op for absent ids); ensure_page gives a resident
  // block without a page (force_insert on a full pool) one, returning it
  void set_stale(uint64_t id, bool stale);
  int32_t ensure_page(uint64_t id);
  std::vector<const Block*> resident_sorted() const;
  uint64_t resident() const { return resident_.size(); }
  uint64_t capacity() const { return cap_; }
  uint32_t block_tokens() const { return B_; }
  int policy() const { return policy_; }
  int64_t hits() const { return hits_; }
  int64_t misses() const { return misses_; }
  const int64_t* evictions_by_tier() const { return ev_; }
  const std::string& session_name(int32_t s) const { return sessions_[s]; }
  std::string snapshot_json() const;
  PagePool& pool() { return pool_; }
  const PagePool& pool() const { return pool_; }
  const std::vector<uint64_t>& last_evicted() const { return last_evicted_; }

 private:
  int32_t intern(const std::string& s);
  void order_insert(const Block& b) { order_[b.tier].insert({b.last_used, b.id}); }
  void order_erase(const Block& b) { order_[b.tier].erase({b.last_used, b.id}); }
  void touch(Block& b, uint64_t stamp, int want_tier);
  void erase_block(uint64_t id);
  static int strongest_tier_over(const glmx_tier_range* t, uint64_t n, uint64_t b, uint64_t e);

  uint64_t cap_;
  uint32_t B_;
  int policy_;
  std::unordered_map<uint64_t, Block> resident_;
  std::set<std::pair<uint64_t, uint64_t>> order_[4];  // per tier: (last_used, id) ascending
  std::unordered_map<int32_t, std::unordered_set<uint64_t>> owned_;
  std::unordered_map<std::string, int32_t> session_ids_;
  std::vector<std::string> sessions_;
  uint64_t clock_ = 0;
  int64_t hits_ = 0, misses_ = 0, ev_[4] = {0, 0, 0, 0};
  PagePool pool_;
  std::vector<uint64_t> last_evicted_;
};

}  // namespace glmx
