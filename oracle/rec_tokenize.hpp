// TEST INFRASTRUCTURE ONLY (oracle/_ref).  Forced include (-include) for the reference's
// orchestrator.cpp in this build: Orchestrator::kv_prefill (orchestrator.cpp:81-97) tokenizes
// each PromptSegments part with glm::tokenize (its only call of it); routing that call through a
// recorder lets the trace keep the exact segment texts the reference prefilled.  tokenizer.hpp is
// included first under its real name (it is #pragma once), so the recorder forwards to it.
#pragma once
#include <string_view>

#include "glm/kvcache/tokenizer.hpp"

namespace glm {
void glmref_record_segment_text(std::string_view text);
inline TokenSeq tokenize_rec(std::string_view text) {
  glmref_record_segment_text(text);
  return tokenize(text);
}
}  // namespace glm
#define tokenize tokenize_rec
