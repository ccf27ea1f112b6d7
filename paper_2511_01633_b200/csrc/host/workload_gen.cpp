#include "workload_gen.hpp"

#include <algorithm>
#include <cstdio>
#include <random>
#include <set>

namespace glmx {

namespace {

uint64_t pick(std::mt19937_64& rng, uint64_t n) { return rng() % n; }  // workload.cpp:27

std::string pad4(int i) {
  char buf[16];
  std::snprintf(buf, sizeof(buf), "%04d", i);
  return buf;
}

// nlohmann::json::dump() string escaping (ensure_ascii = false)
void json_str(std::string& out, const std::string& s) {
  out += '"';
  for (unsigned char c : s) {
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\b': out += "\\b"; break;
      case '\f': out += "\\f"; break;
      case '\n': out += "\\n"; break;
      case '\r': out += "\\r"; break;
      case '\t': out += "\\t"; break;
      default:
        if (c < 0x20) {
          char b[8];
          std::snprintf(b, sizeof(b), "\\u%04x", c);
          out += b;
        } else {
          out += static_cast<char>(c);
        }
    }
  }
  out += '"';
}

struct Question {
  std::string text, answer;
  bool det = true;
  int facts = 1;
};

}  // namespace

std::string generate_workload_jsonl(const HostGraph& g, const std::vector<uint8_t>& unique,
                                    uint64_t seed, int n, double nondet_ratio,
                                    const std::string& link) {
  if (nondet_ratio < 0.0 || nondet_ratio > 1.0)
    throw Error(GLMX_ERR_CONFIG, "nondet_ratio must be in [0, 1]");
  std::mt19937_64 rng(seed ^ 0x9e3779b97f4a7c15ULL);
  const int64_t N = static_cast<int64_t>(g.n());
  bool any_indexed = false;
  for (int64_t v = 0; v < N; ++v) any_indexed = any_indexed || g.has_itext[v];
  if (!any_indexed) throw Error(GLMX_ERR_GLM, "graph has no indexable nodes");
  int32_t link_t = -1;
  for (size_t t = 0; t < g.etypes.size(); ++t)
    if (g.etypes[t] == link) link_t = static_cast<int32_t>(t);
  // link adjacency, sorted by node (= id) order, duplicates kept (graph_store.cpp:108-124)
  std::vector<std::vector<int32_t>> out_l(N), in_l(N);
  if (link_t >= 0)
    for (size_t e = 0; e < g.src.size(); ++e)
      if (g.etype[e] == link_t) {
        out_l[g.src[e]].push_back(g.dst[e]);
        in_l[g.dst[e]].push_back(g.src[e]);
      }
  for (auto& v : out_l) std::sort(v.begin(), v.end());
  for (auto& v : in_l) std::sort(v.begin(), v.end());
  auto titled = [&](int64_t v) { return g.has_itext[v] && g.itext_is_title[v]; };

  // candidate pools (workload.cpp:173-210)
  std::vector<int32_t> det_pool;
  struct Cluster {
    int32_t target;
    std::vector<int32_t> sources;
  };
  std::vector<Cluster> nondet_pool;
  for (int64_t v = 0; v < N; ++v) {
    if (!titled(v) || !unique[v]) continue;
    det_pool.push_back(static_cast<int32_t>(v));
    const auto& sources = in_l[v];
    if (sources.size() < 2 || sources.size() > 4) continue;
    bool ok = true;
    std::set<int32_t> common;
    for (size_t i = 0; i < sources.size() && ok; ++i) {
      const int32_t sv = sources[i];
      if (!titled(sv) || !unique[sv]) {
        ok = false;
        break;
      }
      std::set<int32_t> s(out_l[sv].begin(), out_l[sv].end());
      if (i == 0) {
        common = std::move(s);
      } else {
        std::set<int32_t> next;
        std::set_intersection(common.begin(), common.end(), s.begin(), s.end(),
                              std::inserter(next, next.end()));
        common = std::move(next);
      }
    }
    if (ok && common.size() == 1 && *common.begin() == v)
      nondet_pool.push_back({static_cast<int32_t>(v), sources});
  }
  if (det_pool.empty()) throw Error(GLMX_ERR_GLM, "no deterministic question candidates");

  // question draws (workload.cpp:212-247)
  static const char* det_attrs[] = {"price", "brand", "category"};
  auto attr_of = [&](int32_t v, const std::string& k) -> const std::string* {
    for (const auto& kv : g.attrs[v])
      if (kv.first == k) return &kv.second;
    return nullptr;
  };
  std::vector<Question> qs;
  const int want_nondet = static_cast<int>(nondet_ratio * n + 0.5);
  int attempts = 0;
  for (int i = 0; i < n; ++i) {
    if (++attempts > 10 * n + 100) throw Error(GLMX_ERR_GLM, "could not instantiate enough valid questions");
    const bool make_nondet = i < want_nondet;
    if (make_nondet && nondet_pool.empty())
      throw Error(GLMX_ERR_GLM, "not enough link clusters for non-deterministic questions");
    Question q;
    if (make_nondet) {
      const Cluster& c = nondet_pool[pick(rng, nondet_pool.size())];
      std::string text = "Which item is linked from all of: ";
      for (size_t j = 0; j < c.sources.size(); ++j) {
        if (j) text += "; ";
        text += g.itext[c.sources[j]];
      }
      q.text = text + "?";
      q.det = false;
      q.facts = static_cast<int>(c.sources.size());
      q.answer = g.itext[c.target];
    } else {
      const int32_t id = det_pool[pick(rng, det_pool.size())];
      std::vector<std::string> usable;
      for (const char* a : det_attrs)
        if (attr_of(id, a)) usable.push_back(a);
      if (usable.empty()) {
        --i;  // try another node
        continue;
      }
      const std::string attr = usable[pick(rng, usable.size())];
      q.text = "What is the " + attr + " of " + g.itext[id] + "?";
      q.det = true;
      q.facts = 1;
      q.answer = "[" + *attr_of(id, attr) + "]";
    }
    qs.push_back(std::move(q));
  }
  // deterministic Fisher-Yates (workload.cpp:250-251)
  for (size_t i = qs.size(); i > 1; --i) std::swap(qs[i - 1], qs[pick(rng, i)]);
  std::string out;
  for (size_t i = 0; i < qs.size(); ++i) {
    // nlohmann::json objects are key-sorted
    out += "{\"expected_answer\":";
    json_str(out, qs[i].answer);
    out += ",\"id\":";
    json_str(out, "q" + pad4(static_cast<int>(i)));
    out += ",\"kind\":";
    json_str(out, qs[i].det ? "deterministic" : "non_deterministic");
    out += ",\"required_facts\":" + std::to_string(qs[i].facts) + ",\"text\":";
    json_str(out, qs[i].text);
    out += "}\n";
  }
  return out;
}

}  // namespace glmx
