// Property graph ingest (graph_store.cpp:38-124) into the flat, device-friendly form that the
// vertex-chunk kernel K1 consumes:
//   * nodes ordered by id bytes (== the reference's std::map / node_ids() order, so "ties break
//     by id ascending" becomes "ties break by node index ascending");
//   * per node the pre-rendered entry text  "<id> {k:v, ...}"  (retriever.cpp:34-41 +
//     attr.hpp:19-48), which is query-independent;
//   * the undirected and the out-only de-duplicated neighbour CSRs (retriever.cpp:79-89);
//   * both weight columns: total_degree (graph_store.cpp:209-213) and the by-edge-type maximum
//     (retriever.cpp:100-105).
#pragma once

#include <cstdint>
#include <string>
#include <unordered_map>
#include <vector>

#include "common.hpp"

namespace glmx {

// attribute value kinds (attr.hpp:13-16): Scalar string / int64 / double / bool, or a list
constexpr uint8_t kAttrString = 0, kAttrInt = 1, kAttrDouble = 2, kAttrBool = 3, kAttrList = 4;

struct HostGraph {
  std::vector<std::string> ids;            // ascending
  std::vector<std::string> types;
  std::vector<std::vector<std::pair<std::string, std::string>>> attrs;  // rendered, key order
  std::vector<std::vector<uint8_t>> attr_kind;  // per attrs entry: kAttr*
  // VectorIndex text per node (index.cpp:12-25, default Config): the "title" attribute when it is
  // a string, else "name" when it is a string; has_itext[v] = 0 for nodes without one
  std::vector<std::string> itext;
  std::vector<uint8_t> has_itext;
  std::vector<uint8_t> itext_is_title;  // the index text is the string "title" (title_of)
  std::unordered_map<std::string, int32_t> index;
  std::vector<std::string> etypes;
  std::vector<int32_t> src, dst, etype;    // edges in file order

  // derived (finalize())
  std::vector<char> entry_bytes;           // concatenated "<id> {k:v, ...}"
  std::vector<uint32_t> entry_off;         // n+1
  std::vector<uint32_t> und_off, dir_off;  // n+1
  std::vector<int32_t> und_idx, dir_idx;
  std::vector<int32_t> w_total, w_by_type;

  uint64_t n() const { return ids.size(); }
  // entries always; CSRs and weights on the host unless host_csr = false (GPU ingest)
  void finalize(bool host_csr = true);
  std::string serialize_jsonl() const;
};

HostGraph load_graph_jsonl(const std::string& path, bool host_csr = true);
HostGraph synth_powerlaw(uint64_t n_nodes, uint32_t edges_per_node, uint64_t seed,
                         bool host_csr = true);

// attr.hpp:19-24 shortest round-trip double rendering (std::to_chars).
std::string format_double(double d);

}  // namespace glmx
