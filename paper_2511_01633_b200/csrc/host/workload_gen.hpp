// Scalable re-implementation of the reference's question generator (generate_workload,
// workload.cpp:158-255) — same candidate pools, same std::mt19937_64 draw sequence, same JSONL
// (Workload::serialize_jsonl, workload.cpp:122-133) — whose O(N^2) part, the "title retrieves its
// own node" validation (one full-scan VectorIndex::nearest per candidate, workload.cpp:166-171),
// is ONE batched exact GPU scan (K5).  The caller supplies that validation as `unique[v]`.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "graph.hpp"

namespace glmx {

// unique[v] = 1 iff node v has a string title and nearest(title, 1) is v.  Throws Error with
// GLMX_ERR_GLM and the reference's GraphTooSmall / ConfigError messages.
std::string generate_workload_jsonl(const HostGraph& g, const std::vector<uint8_t>& unique,
                                    uint64_t seed, int n, double nondet_ratio,
                                    const std::string& link = "linked");

}  // namespace glmx
