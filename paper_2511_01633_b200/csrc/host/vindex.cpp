#include "vindex.hpp"

#include <cmath>

namespace glmx {

namespace {
uint64_t fnv1a3(const char* p) {
  uint64_t h = 14695981039346656037ULL;
  for (int i = 0; i < 3; ++i) {
    h ^= static_cast<unsigned char>(p[i]);
    h *= 1099511628211ULL;
  }
  return h;
}
}  // namespace

int embed_padded(int dim) { return (dim + 7) / 8 * 8; }

void embed(const char* text, size_t len, int dim, float* out) {
  const int pad = embed_padded(dim);
  for (int i = 0; i < pad; ++i) out[i] = 0.f;
  if (len >= 3)
    for (size_t i = 0; i + 3 <= len; ++i) out[fnv1a3(text + i) % static_cast<uint64_t>(dim)] += 1.0f;
  double sumsq = 0.0;
  for (int i = 0; i < pad; ++i) sumsq += static_cast<double>(out[i]) * out[i];
  if (sumsq == 0.0) {
    out[0] = 1.0f;
    return;
  }
  const float inv = static_cast<float>(1.0 / std::sqrt(sumsq));
  for (int i = 0; i < pad; ++i) out[i] *= inv;
}

bool TextLru::get(const std::string& k, int64_t* v) {
  auto it = map_.find(k);
  if (it == map_.end()) return false;
  order_.splice(order_.begin(), order_, it->second);
  *v = it->second->second;
  return true;
}

void TextLru::put(const std::string& k, int64_t v) {
  if (cap_ == 0) return;
  auto it = map_.find(k);
  if (it != map_.end()) {
    it->second->second = v;
    order_.splice(order_.begin(), order_, it->second);
    return;
  }
  if (map_.size() == cap_) {
    map_.erase(order_.back().first);
    order_.pop_back();
  }
  order_.emplace_front(k, v);
  map_[k] = order_.begin();
}

void TextLru::resolve(int64_t from, int64_t to) {
  for (auto& e : order_)
    if (e.second == from) e.second = to;
}

}  // namespace glmx
