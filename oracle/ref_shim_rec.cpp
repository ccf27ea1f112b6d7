// TEST INFRASTRUCTURE ONLY (oracle/_ref). Compiled with -Dprefill=prefill_recorded
// -Dset_tier=set_tier_recorded, exactly like the reference's orchestrator.cpp in this build, so
// the orchestrator's calls to KvCacheState::prefill / ::set_tier (orchestrator.cpp:96, :153) land
// here; they are recorded and forwarded to the real reference methods (cache.cpp:54, :150).
#include "glm/kvcache/cache.hpp"

namespace glm {
PrefillReport glmref_real_prefill(KvCacheState* kv, const TokenSeq& p, const TierMap& t,
                                  const std::string& s);
void glmref_real_set_tier(KvCacheState* kv, const std::string& s, Tier from, Tier to);
void glmref_record_prefill(const TokenSeq& p, const TierMap& t, const std::string& s,
                           const PrefillReport* rep, const char* error);
void glmref_record_set_tier(const std::string& s, Tier from, Tier to);

PrefillReport KvCacheState::prefill_recorded(const TokenSeq& p, const TierMap& t,
                                             const std::string& s) {
  try {
    PrefillReport rep = glmref_real_prefill(this, p, t, s);
    glmref_record_prefill(p, t, s, &rep, nullptr);
    return rep;
  } catch (const std::exception& e) {
    glmref_record_prefill(p, t, s, nullptr, e.what());
    throw;
  }
}

void KvCacheState::set_tier_recorded(const std::string& s, Tier from, Tier to) {
  glmref_real_set_tier(this, s, from, to);
  glmref_record_set_tier(s, from, to);
}
}  // namespace glm
