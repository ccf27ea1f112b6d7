// Shared host-side helpers: error type, FNV-1a, whitespace tokenizer.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "glmx.h"

namespace glmx {

// Carries a GLMX_ERR_* code across the C++ layers; capi.cpp turns it into a status.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& msg) : std::runtime_error(msg), code(c) {}
};

// 64-bit FNV-1a over bytes (fnv.hpp:9-16).
inline uint64_t fnv1a(const char* p, size_t n, uint64_t h = 14695981039346656037ULL) {
  for (size_t i = 0; i < n; ++i) {
    h ^= static_cast<unsigned char>(p[i]);
    h *= 1099511628211ULL;
  }
  return h;
}

// FNV-1a over the eight little-endian bytes of a u64 (fnv.hpp:18-25).
inline uint64_t fnv1a_u64(uint64_t v, uint64_t h) {
  for (int i = 0; i < 8; ++i) {
    h ^= (v >> (i * 8)) & 0xff;
    h *= 1099511628211ULL;
  }
  return h;
}

// std::isspace in the "C" locale.
inline bool is_space(unsigned char c) { return c == ' ' || (c >= '\t' && c <= '\r'); }

// A token sequence as byte spans into one contiguous buffer.
struct TokenSpans {
  const char* bytes = nullptr;
  const uint64_t* offsets = nullptr;  // n+1
  uint64_t n = 0;
  std::string_view tok(uint64_t i) const {
    return std::string_view(bytes + offsets[i], offsets[i + 1] - offsets[i]);
  }
};

// Whitespace tokenizer (tokenizer.hpp:14-25) producing [begin,end) spans.
inline void tokenize_spans(const char* text, uint64_t len, std::vector<uint64_t>& begins,
                           std::vector<uint64_t>& ends) {
  uint64_t i = 0;
  while (i < len) {
    while (i < len && is_space(static_cast<unsigned char>(text[i]))) ++i;
    uint64_t s = i;
    while (i < len && !is_space(static_cast<unsigned char>(text[i]))) ++i;
    if (i > s) {
      begins.push_back(s);
      ends.push_back(i);
    }
  }
}

inline int32_t token_id(const char* p, uint64_t n, uint32_t vocab) {
  return static_cast<int32_t>(fnv1a(p, n) % vocab);
}

}  // namespace glmx
