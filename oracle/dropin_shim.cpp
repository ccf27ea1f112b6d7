// TEST INFRASTRUCTURE ONLY.  The reference's run_bench (bench.cpp:45-161) with its Orchestrator,
// RuleProvider, Retriever and workload generator compiled UNMODIFIED against the drop-in
// glm/kvcache/cache.hpp of integration/ (KvCacheState over libglmx's C ABI) instead of
// src/kvcache/cache.cpp: the compiled proof that the boundary is a drop-in (tests/test_dropin.py
// compares the report with the stock build's, oracle/_ref).
#include <cstdint>
#include <cstring>
#include <string>

#include "glm/bench/bench.hpp"
#include "glm/bench/workload.hpp"
#include "glm/graph/graph_store.hpp"

extern "C" {
// synth_graph(seed, nodes) + generate_workload(seed_wl, n, ratio) + run_bench -> report JSON.
int64_t dropin_run_bench(std::uint64_t graph_seed, int nodes, std::uint64_t seed_wl, int n,
                         double ratio, int concurrency, std::uint64_t cap_blocks, int policy,
                         int glm_mode, char* buf, std::uint64_t cap) {
  try {
    glm::SynthGraphOptions o;
    o.seed = graph_seed;
    o.nodes = nodes;
    glm::PropertyGraph g = glm::synth_graph(o);
    glm::BenchOptions opt;
    opt.glm_mode = glm_mode != 0;
    opt.policy = policy == 0 ? glm::CachePolicy::Priority : glm::CachePolicy::PlainLru;
    opt.concurrency = concurrency;
    opt.config.kv_capacity_blocks = cap_blocks;
    glm::Workload wl = glm::generate_workload(seed_wl, n, ratio, g, opt.config);
    const std::string out = glm::run_bench(wl, g, opt).to_json();
    if (buf && cap) std::memcpy(buf, out.data(), std::min<std::uint64_t>(cap, out.size()));
    return static_cast<int64_t>(out.size());
  } catch (const std::exception& e) {
    const std::string msg = std::string("error: ") + e.what();
    if (buf && cap) std::memcpy(buf, msg.data(), std::min<std::uint64_t>(cap, msg.size()));
    return -static_cast<int64_t>(msg.size());
  }
}
}
