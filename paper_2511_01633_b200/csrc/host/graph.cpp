#include "graph.hpp"

#include <algorithm>
#include <iterator>
#include <exception>
#include <thread>
#include <charconv>
#include <cmath>
#include <cstring>
#include <fstream>
#include <map>
#include <set>
#include <numeric>

namespace glmx {

std::string format_double(double d) {
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof(buf), d);
  return std::string(buf, r.ptr);
}

namespace {

// ------------------------------------------------------------------ minimal JSON reader
// Enough of RFC 8259 for the graph records (graph_store.cpp:46-88): objects, arrays, strings
// with escapes, numbers classified like nlohmann (integer iff no '.', 'e', 'E'), bools, null.
struct JVal {
  enum Kind { Null, Bool, Int, UInt, Double, Str, Arr, Obj } kind = Null;
  bool b = false;
  int64_t i = 0;
  uint64_t u = 0;
  double d = 0;
  std::string s;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;  // later duplicates override earlier
  const JVal* get(const char* key) const {
    const JVal* r = nullptr;
    for (const auto& kv : obj)
      if (kv.first == key) r = &kv.second;
    return r;
  }
};

struct JParser {
  const char* p;
  const char* e;
  size_t line;
  [[noreturn]] void fail(const std::string& why) {
    throw Error(GLMX_ERR_MALFORMED, "malformed record at line " + std::to_string(line) + ": " + why);
  }
  void ws() {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
  }
  static void put_utf8(std::string& out, uint32_t cp) {
    if (cp < 0x80) {
      out += static_cast<char>(cp);
    } else if (cp < 0x800) {
      out += static_cast<char>(0xC0 | (cp >> 6));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      out += static_cast<char>(0xE0 | (cp >> 12));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else {
      out += static_cast<char>(0xF0 | (cp >> 18));
      out += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    }
  }
  uint32_t hex4() {
    if (e - p < 4) fail("bad \\u escape");
    uint32_t v = 0;
    for (int k = 0; k < 4; ++k) {
      char c = *p++;
      v <<= 4;
      if (c >= '0' && c <= '9') v |= c - '0';
      else if (c >= 'a' && c <= 'f') v |= c - 'a' + 10;
      else if (c >= 'A' && c <= 'F') v |= c - 'A' + 10;
      else fail("bad \\u escape");
    }
    return v;
  }
  std::string str() {
    if (p >= e || *p != '"') fail("expected string");
    ++p;
    std::string out;
    while (true) {
      if (p >= e) fail("unterminated string");
      char c = *p++;
      if (c == '"') break;
      if (static_cast<unsigned char>(c) < 0x20) fail("control character in string");
      if (c != '\\') {
        out += c;
        continue;
      }
      if (p >= e) fail("bad escape");
      char x = *p++;
      switch (x) {
        case '"': out += '"'; break;
        case '\\': out += '\\'; break;
        case '/': out += '/'; break;
        case 'b': out += '\b'; break;
        case 'f': out += '\f'; break;
        case 'n': out += '\n'; break;
        case 'r': out += '\r'; break;
        case 't': out += '\t'; break;
        case 'u': {
          uint32_t cp = hex4();
          if (cp >= 0xD800 && cp <= 0xDBFF) {
            if (e - p < 6 || p[0] != '\\' || p[1] != 'u') fail("lone surrogate");
            p += 2;
            uint32_t lo = hex4();
            if (lo < 0xDC00 || lo > 0xDFFF) fail("bad surrogate pair");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          }
          put_utf8(out, cp);
          break;
        }
        default: fail("bad escape");
      }
    }
    return out;
  }
  JVal value() {
    ws();
    if (p >= e) fail("unexpected end");
    JVal v;
    char c = *p;
    if (c == '{') {
      v.kind = JVal::Obj;
      ++p;
      ws();
      if (p < e && *p == '}') {
        ++p;
        return v;
      }
      while (true) {
        ws();
        std::string k = str();
        ws();
        if (p >= e || *p != ':') fail("expected ':'");
        ++p;
        v.obj.emplace_back(std::move(k), value());
        ws();
        if (p < e && *p == ',') {
          ++p;
          continue;
        }
        if (p < e && *p == '}') {
          ++p;
          break;
        }
        fail("expected ',' or '}'");
      }
    } else if (c == '[') {
      v.kind = JVal::Arr;
      ++p;
      ws();
      if (p < e && *p == ']') {
        ++p;
        return v;
      }
      while (true) {
        v.arr.push_back(value());
        ws();
        if (p < e && *p == ',') {
          ++p;
          continue;
        }
        if (p < e && *p == ']') {
          ++p;
          break;
        }
        fail("expected ',' or ']'");
      }
    } else if (c == '"') {
      v.kind = JVal::Str;
      v.s = str();
    } else if (e - p >= 4 && std::strncmp(p, "true", 4) == 0) {
      v.kind = JVal::Bool;
      v.b = true;
      p += 4;
    } else if (e - p >= 5 && std::strncmp(p, "false", 5) == 0) {
      v.kind = JVal::Bool;
      p += 5;
    } else if (e - p >= 4 && std::strncmp(p, "null", 4) == 0) {
      p += 4;
    } else {
      const char* s = p;
      bool is_float = false;
      if (p < e && *p == '-') ++p;
      if (p >= e || !(*p >= '0' && *p <= '9')) fail("bad literal");
      while (p < e && ((*p >= '0' && *p <= '9') || *p == '.' || *p == 'e' || *p == 'E' ||
                       *p == '+' || *p == '-')) {
        if (*p == '.' || *p == 'e' || *p == 'E') is_float = true;
        ++p;
      }
      std::string num(s, p);
      if (!is_float) {
        if (num[0] == '-') {
          auto r = std::from_chars(num.data(), num.data() + num.size(), v.i);
          if (r.ec == std::errc()) {
            v.kind = JVal::Int;
            return v;
          }
        } else {
          auto r = std::from_chars(num.data(), num.data() + num.size(), v.u);
          if (r.ec == std::errc()) {
            v.kind = JVal::UInt;
            return v;
          }
        }
      }
      v.kind = JVal::Double;
      v.d = std::strtod(num.c_str(), nullptr);
    }
    return v;
  }
};

struct RawNode {
  std::string id, type;
  std::map<std::string, std::string> attrs;  // key -> rendered value (std::map like NodeRecord)
  std::set<std::string> str_attrs;           // keys whose value is a JSON string scalar
  std::map<std::string, uint8_t> kinds;      // key -> AttrKind (strings: str_attrs)
};
struct RawEdge {
  std::string src, dst, etype;
};

// attr.hpp:28-36
std::string render_scalar(const JVal& v, JParser& jp) {
  switch (v.kind) {
    case JVal::Str: return v.s;
    case JVal::Int: return std::to_string(v.i);
    case JVal::UInt: return std::to_string(static_cast<int64_t>(v.u));
    case JVal::Double: return format_double(v.d);
    case JVal::Bool: return v.b ? "true" : "false";
    default: jp.fail("attribute values must be scalars or lists of scalars");
  }
}

HostGraph build(std::vector<RawNode> nodes, std::vector<RawEdge> edges, bool host_csr) {
  HostGraph g;
  std::sort(nodes.begin(), nodes.end(),
            [](const RawNode& a, const RawNode& b) { return a.id < b.id; });
  for (size_t i = 0; i < nodes.size(); ++i) {
    if (nodes[i].id.empty()) throw Error(GLMX_ERR_MALFORMED, "node id must be non-empty");
    if (i && nodes[i].id == nodes[i - 1].id)
      throw Error(GLMX_ERR_MALFORMED, "duplicate node id: " + nodes[i].id);
  }
  g.ids.reserve(nodes.size());
  for (size_t i = 0; i < nodes.size(); ++i) {
    g.index.emplace(nodes[i].id, static_cast<int32_t>(i));
    g.ids.push_back(std::move(nodes[i].id));
    g.types.push_back(std::move(nodes[i].type));
    g.attrs.emplace_back(nodes[i].attrs.begin(), nodes[i].attrs.end());
    std::vector<uint8_t> kinds;
    kinds.reserve(nodes[i].attrs.size());
    for (const auto& kv : nodes[i].attrs) {
      auto k = nodes[i].kinds.find(kv.first);
      kinds.push_back(nodes[i].str_attrs.count(kv.first) ? kAttrString
                      : k != nodes[i].kinds.end()         ? k->second
                                                          : kAttrInt);
    }
    g.attr_kind.push_back(std::move(kinds));
    std::string text;
    uint8_t has = 0, is_title = 0;
    for (const char* f : {"title", "name"}) {
      auto it = nodes[i].attrs.find(f);
      if (it != nodes[i].attrs.end() && nodes[i].str_attrs.count(f)) {
        text = it->second;
        has = 1;
        is_title = f[0] == 't';
        break;
      }
    }
    g.itext.push_back(std::move(text));
    g.has_itext.push_back(has);
    g.itext_is_title.push_back(is_title);
  }
  std::unordered_map<std::string, int32_t> et;
  for (const auto& e : edges) {
    auto s = g.index.find(e.src), d = g.index.find(e.dst);
    if (s == g.index.end() || d == g.index.end())
      throw Error(GLMX_ERR_MALFORMED, "edge references unknown node: " + e.src + " -> " + e.dst);
    auto t = et.find(e.etype);
    int32_t ti;
    if (t == et.end()) {
      ti = static_cast<int32_t>(g.etypes.size());
      et.emplace(e.etype, ti);
      g.etypes.push_back(e.etype);
    } else {
      ti = t->second;
    }
    g.src.push_back(s->second);
    g.dst.push_back(d->second);
    g.etype.push_back(ti);
  }
  g.finalize(host_csr);
  return g;
}

uint64_t splitmix(uint64_t& s) {
  uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

void json_escape(std::string& out, const std::string& s) {
  out += '"';
  for (unsigned char c : s) {
    if (c == '"') out += "\\\"";
    else if (c == '\\') out += "\\\\";
    else if (c == '\n') out += "\\n";
    else if (c == '\t') out += "\\t";
    else if (c == '\r') out += "\\r";
    else if (c < 0x20) {
      char b[8];
      std::snprintf(b, sizeof(b), "\\u%04x", c);
      out += b;
    } else {
      out += static_cast<char>(c);
    }
  }
  out += '"';
}

}  // namespace

void HostGraph::finalize(bool host_csr) {
  const uint64_t N = n();
  // Entries: "<id> {k:v, ...}" with ("type", node_type) added and pairs sorted by (key, value)
  // (retriever.cpp:34-41, render_chunk retriever.cpp:10-20); rendered on up to 16 threads.
  std::vector<std::string> ent(N);
  {
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const uint64_t n_thr = std::max<uint64_t>(1, std::min<uint64_t>(hw, N / 8192 + 1));
    std::vector<std::thread> th;
    for (uint64_t t = 0; t < n_thr; ++t)
      th.emplace_back([&, t] {
        for (uint64_t v = N * t / n_thr; v < N * (t + 1) / n_thr; ++v) {
          std::vector<std::pair<std::string, std::string>> pairs = attrs[v];
          pairs.emplace_back("type", types[v]);
          std::sort(pairs.begin(), pairs.end());
          std::string s = ids[v] + " {";
          for (size_t i = 0; i < pairs.size(); ++i) {
            if (i) s += ", ";
            s += pairs[i].first;
            s += ':';
            s += pairs[i].second;
          }
          s += '}';
          ent[v] = std::move(s);
        }
      });
    for (auto& x : th) x.join();
  }
  entry_off.assign(N + 1, 0);
  entry_bytes.clear();
  for (uint64_t v = 0; v < N; ++v) {
    entry_off[v] = static_cast<uint32_t>(entry_bytes.size());
    entry_bytes.insert(entry_bytes.end(), ent[v].begin(), ent[v].end());
    if (entry_bytes.size() > 0xFFFFFFF0ULL) throw Error(GLMX_ERR_ARG, "graph text exceeds 4 GiB");
  }
  entry_off[N] = static_cast<uint32_t>(entry_bytes.size());
  // the neighbour CSRs and weights are built on the GPU (kernels/ingest.cu) for device graphs
  if (!host_csr) return;

  // total_degree (graph_store.cpp:116-121): every edge counts once at each endpoint.
  w_total.assign(N, 0);
  for (size_t e = 0; e < src.size(); ++e) {
    ++w_total[src[e]];
    ++w_total[dst[e]];
  }
  // ByEdgeType: max over incident types of out+in count of that type (retriever.cpp:100-105).
  w_by_type.assign(N, 0);
  {
    std::vector<uint64_t> key;
    key.reserve(2 * src.size());
    for (size_t e = 0; e < src.size(); ++e) {
      key.push_back((static_cast<uint64_t>(src[e]) << 24) | static_cast<uint64_t>(etype[e]));
      key.push_back((static_cast<uint64_t>(dst[e]) << 24) | static_cast<uint64_t>(etype[e]));
    }
    std::sort(key.begin(), key.end());
    for (size_t i = 0; i < key.size();) {
      size_t j = i;
      while (j < key.size() && key[j] == key[i]) ++j;
      int32_t v = static_cast<int32_t>(key[i] >> 24);
      w_by_type[v] = std::max<int32_t>(w_by_type[v], static_cast<int32_t>(j - i));
      i = j;
    }
  }
  // Neighbour CSRs, de-duplicated and ascending (retriever.cpp:79-89).
  auto csr = [&](bool undirected, std::vector<uint32_t>& off, std::vector<int32_t>& idx) {
    std::vector<uint64_t> pr;
    pr.reserve((undirected ? 2 : 1) * src.size());
    for (size_t e = 0; e < src.size(); ++e) {
      pr.push_back((static_cast<uint64_t>(src[e]) << 32) | static_cast<uint32_t>(dst[e]));
      if (undirected)
        pr.push_back((static_cast<uint64_t>(dst[e]) << 32) | static_cast<uint32_t>(src[e]));
    }
    std::sort(pr.begin(), pr.end());
    pr.erase(std::unique(pr.begin(), pr.end()), pr.end());
    off.assign(N + 1, 0);
    idx.resize(pr.size());
    for (size_t i = 0; i < pr.size(); ++i) {
      ++off[(pr[i] >> 32) + 1];
      idx[i] = static_cast<int32_t>(pr[i] & 0xFFFFFFFFu);
    }
    for (uint64_t v = 0; v < N; ++v) off[v + 1] += off[v];
  };
  csr(true, und_off, und_idx);
  csr(false, dir_off, dir_idx);
}

std::string HostGraph::serialize_jsonl() const {
  std::string out;
  for (uint64_t v = 0; v < n(); ++v) {
    out += "{\"kind\":\"node\",\"id\":";
    json_escape(out, ids[v]);
    out += ",\"type\":";
    json_escape(out, types[v]);
    out += ",\"attrs\":{";
    for (size_t i = 0; i < attrs[v].size(); ++i) {
      if (i) out += ',';
      json_escape(out, attrs[v][i].first);
      out += ':';
      // scalars round-trip (the canonical renders of ints, doubles and bools are JSON numbers /
      // literals); a list is written as its rendered string
      const std::string& val = attrs[v][i].second;
      const uint8_t kind = attr_kind.empty() ? kAttrString : attr_kind[v][i];
      if (kind == kAttrInt || kind == kAttrDouble || kind == kAttrBool) out += val;
      else json_escape(out, val);
    }
    out += "}}\n";
  }
  for (size_t e = 0; e < src.size(); ++e) {
    out += "{\"kind\":\"edge\",\"src\":";
    json_escape(out, ids[src[e]]);
    out += ",\"dst\":";
    json_escape(out, ids[dst[e]]);
    out += ",\"etype\":";
    json_escape(out, etypes[etype[e]]);
    out += "}\n";
  }
  return out;
}

namespace {

// Parses lines [first, last) of the file (line_no = first + 1, ...) into nodes/edges.
void parse_lines(const std::vector<std::pair<const char*, const char*>>& lines, size_t first,
                 size_t last, std::vector<RawNode>& nodes, std::vector<RawEdge>& edges) {
  for (size_t li = first; li < last; ++li) {
    const char* lb = lines[li].first;
    const char* le = lines[li].second;
    const size_t line_no = li + 1;
    bool blank = true;
    for (const char* c = lb; c < le && blank; ++c) blank = *c == ' ' || *c == '\t' || *c == '\r';
    if (blank) continue;
    JParser jp{lb, le, line_no};
    JVal j = jp.value();
    if (j.kind != JVal::Obj || !j.get("kind")) jp.fail("expected object with \"kind\"");
    const JVal* kind = j.get("kind");
    if (kind->kind != JVal::Str) jp.fail("kind must be a string");
    if (kind->s == "node") {
      const JVal* id = j.get("id");
      const JVal* ty = j.get("type");
      if (!id || !ty) jp.fail("node requires id and type");
      if (id->kind != JVal::Str || ty->kind != JVal::Str) jp.fail("id and type must be strings");
      RawNode n;
      n.id = id->s;
      n.type = ty->s;
      if (n.id.empty()) jp.fail("node id must be non-empty");
      if (const JVal* at = j.get("attrs")) {
        if (at->kind != JVal::Obj) jp.fail("attrs must be an object");
        for (const auto& [k, v] : at->obj) {
          if (k.empty()) jp.fail("attribute names must be non-empty");
          if (v.kind == JVal::Arr) {
            std::string s = "[";
            for (size_t i = 0; i < v.arr.size(); ++i) {
              if (i) s += ", ";
              s += render_scalar(v.arr[i], jp);
            }
            n.attrs[k] = s + "]";
            n.kinds[k] = kAttrList;
          } else {
            n.attrs[k] = render_scalar(v, jp);
            if (v.kind == JVal::Str) n.str_attrs.insert(k);
            n.kinds[k] = v.kind == JVal::Str    ? kAttrString
                         : v.kind == JVal::Bool ? kAttrBool
                         : v.kind == JVal::Double ? kAttrDouble
                                                  : kAttrInt;
          }
        }
      }
      nodes.push_back(std::move(n));
    } else if (kind->s == "edge") {
      const JVal* s = j.get("src");
      const JVal* d = j.get("dst");
      const JVal* t = j.get("etype");
      if (!s || !d || !t) jp.fail("edge requires src, dst and etype");
      if (s->kind != JVal::Str || d->kind != JVal::Str || t->kind != JVal::Str)
        jp.fail("edge fields must be strings");
      edges.push_back({s->s, d->s, t->s});
    } else {
      jp.fail("kind must be node or edge");
    }
  }
}

}  // namespace

// Reads the whole file, then parses it on up to 16 host threads (line ranges of ~equal bytes);
// nodes and edges are merged in file order, and the first malformed line (lowest line number)
// is the one reported, as with a sequential parse.
HostGraph load_graph_jsonl(const std::string& path, bool host_csr) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Error(GLMX_ERR_GLM, "cannot open graph file: " + path);
  std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  std::vector<std::pair<const char*, const char*>> lines;
  const char* p = text.data();
  const char* end = p + text.size();
  while (p < end) {
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', end - p));
    const char* le = nl ? nl : end;
    lines.emplace_back(p, le);
    p = nl ? nl + 1 : end;
  }
  const size_t n_lines = lines.size();
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  const size_t n_thr = std::max<size_t>(1, std::min<size_t>(hw, n_lines / 4096 + 1));
  std::vector<std::vector<RawNode>> tn(n_thr);
  std::vector<std::vector<RawEdge>> te(n_thr);
  std::vector<std::exception_ptr> err(n_thr);
  std::vector<std::thread> th;
  for (size_t t = 0; t < n_thr; ++t)
    th.emplace_back([&, t] {
      try {
        parse_lines(lines, n_lines * t / n_thr, n_lines * (t + 1) / n_thr, tn[t], te[t]);
      } catch (...) {
        err[t] = std::current_exception();
      }
    });
  for (auto& x : th) x.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);  // earliest range first = lowest line number
  std::vector<RawNode> nodes;
  std::vector<RawEdge> edges;
  for (size_t t = 0; t < n_thr; ++t) {
    for (auto& n : tn[t]) nodes.push_back(std::move(n));
    for (auto& e : te[t]) edges.push_back(std::move(e));
  }
  return build(std::move(nodes), std::move(edges), host_csr);
}


// Seeded power-law property graph: out-edge targets dst = floor(n*u^3) concentrate in-degree on
// low indices (hub degree ~ n^(2/3)), ids zero-padded so byte order == numeric order.
HostGraph synth_powerlaw(uint64_t n_nodes, uint32_t edges_per_node, uint64_t seed, bool host_csr) {
  static const char* adj[] = {"umber", "cobalt", "ivory", "sable", "viridian", "amber",
                              "russet", "pewter", "indigo", "maroon", "ochre", "teal",
                              "slate", "coral", "fawn", "lilac"};
  static const char* noun[] = {"lattice", "widget", "gasket", "spindle", "crucible", "bobbin",
                               "ratchet", "gimbal", "flange", "tumbler", "sprocket", "mandrel",
                               "ferrule", "plinth", "luggage", "brazier"};
  static const char* brand[] = {"acme", "orion", "zephyr", "halcyon", "vertex", "quanta"};
  static const char* cat[] = {"tools", "kitchen", "garden", "office", "sport", "audio"};
  if (n_nodes < 2) throw Error(GLMX_ERR_ARG, "synthetic graph needs at least 2 nodes");
  uint64_t s = seed;
  std::vector<RawNode> nodes(n_nodes);
  char idb[32];
  for (uint64_t i = 0; i < n_nodes; ++i) {
    std::snprintf(idb, sizeof(idb), "v%07llu", static_cast<unsigned long long>(i));
    RawNode& r = nodes[i];
    r.id = idb;
    if (i % 10 == 9) {
      r.type = "user";
      r.attrs["name"] = std::string("user ") + idb;
      r.str_attrs.insert("name");
    } else {
      r.type = "item";
      uint64_t x = splitmix(s);
      r.attrs["title"] = std::string(adj[x % 16]) + " " + noun[(x >> 8) % 16] + " " + idb;
      r.attrs["price"] = std::to_string(1 + (x >> 16) % 999);
      r.attrs["brand"] = brand[(x >> 32) % 6];
      r.attrs["category"] = cat[(x >> 40) % 6];
      r.str_attrs = {"title", "brand", "category"};
    }
  }
  std::vector<RawEdge> edges;
  edges.reserve(n_nodes * edges_per_node);
  for (uint64_t i = 0; i < n_nodes; ++i) {
    for (uint32_t k = 0; k < edges_per_node; ++k) {
      uint64_t x = splitmix(s);
      double u = static_cast<double>(x >> 11) * (1.0 / 9007199254740992.0);
      uint64_t d = static_cast<uint64_t>(static_cast<double>(n_nodes) * u * u * u);
      if (d >= n_nodes) d = n_nodes - 1;
      if (d == i) d = (d + 1) % n_nodes;
      edges.push_back({nodes[i].id, nodes[d].id, (x & 3) == 3 ? "viewed" : "linked"});
    }
  }
  return build(std::move(nodes), std::move(edges), host_csr);
}

}  // namespace glmx
