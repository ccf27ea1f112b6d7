// RetrieveNode support (host side): the reference's trigram embedding and retrieval LRU.
//   embed()        — embedder.cpp:19-36: character-trigram feature hashing (fnv1a of every
//                    3-byte window, bucket h % dim), L2 norm accumulated in double, scaled by
//                    float(1 / sqrt(sumsq)); storage zero-padded to a multiple of 8 floats;
//                    texts with no trigram map to the first basis vector.
//   TextLru        — lru_cache.hpp:13-48 (get refreshes recency, put at capacity evicts the least
//                    recently used entry, capacity 0 stores nothing), text -> node index.
// The exact nearest scan itself runs on the GPU (kernels/retrieve.cu).
#pragma once

#include <cstdint>
#include <list>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

namespace glmx {

int embed_padded(int dim);
// Writes embed_padded(dim) floats.
void embed(const char* text, size_t len, int dim, float* out);

class TextLru {
 public:
  explicit TextLru(size_t capacity = 1024) : cap_(capacity) {}
  bool get(const std::string& k, int64_t* v);
  void put(const std::string& k, int64_t v);
  void set_capacity(size_t c) {
    cap_ = c;
    map_.clear();
    order_.clear();
  }
  size_t size() const { return map_.size(); }
  // replace every value equal to `from` (placeholders of probes resolved after the GPU scan)
  void resolve(int64_t from, int64_t to);

 private:
  size_t cap_;
  std::list<std::pair<std::string, int64_t>> order_;  // front = most recent
  std::unordered_map<std::string, std::list<std::pair<std::string, int64_t>>::iterator> map_;
};

}  // namespace glmx
