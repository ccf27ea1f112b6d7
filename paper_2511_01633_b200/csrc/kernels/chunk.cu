// K1 — batched vertex-chunk assembly (Retriever::node_info + render_chunk, retriever.cpp:9-30,
// 74-121; tokenize, tokenizer.hpp:14-25).
//
//   select  : one CTA per request.  CSR row gather of the de-duplicated neighbour set, top-k by
//             (weight desc, node index asc) with a 64-bit key  w<<32 | ~idx  sorted in shared
//             memory (bitonic, 1024-key window; rows longer than the window stream through it
//             keeping the running top-k), byte length of the rendered chunk.
//   scan    : exclusive sums of chunk lengths (cub).
//   render  : one CTA per request, one warp per entry: scatter of the pre-rendered per-node
//             entries "<id> {k:v,...}" between the literal separators.
//   tokenize: per byte token-start flags -> scan -> per token span + fnv1a id.  Tokens fuse
//             across entry boundaries exactly as in the text ("[neighbours:(n3", "type:item}),(u1").
// All of it is integer/byte work: HBM/latency bound, no tensor cores.
#include <cub/cub.cuh>

#include "chunk.cuh"
#include "common.cuh"

namespace glmx {

namespace {

constexpr int kSelThreads = 256;
constexpr int kWindow = 1024;

__device__ __forceinline__ void bitonic_sort_desc(uint64_t* s, int n) {
  // n is a power of two <= kWindow; all threads of the CTA participate.
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < n / 2; i += blockDim.x) {
        int lo = 2 * i - (i & (stride - 1));
        int hi = lo + stride;
        bool desc = ((lo & size) == 0);
        uint64_t a = s[lo], b = s[hi];
        if ((a < b) == desc) {
          s[lo] = b;
          s[hi] = a;
        }
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(kSelThreads)
chunk_select_kernel(DevGraph g, ChunkParams p, const int32_t* __restrict__ node_idx, int n_req,
                    int32_t* __restrict__ sel, int32_t* __restrict__ sel_count,
                    uint64_t* __restrict__ byte_len) {
  __shared__ uint64_t keys[kWindow];
  const int r = blockIdx.x;
  if (r >= n_req) return;
  const int32_t v = node_idx[r];
  const uint32_t* off = p.directed ? g.dir_off : g.und_off;
  const int32_t* idx = p.directed ? g.dir_idx : g.und_idx;
  const int32_t* w = p.weight_mode ? g.w_by_type : g.w_total;
  const uint32_t beg = off[v], end = off[v + 1];
  const int deg = static_cast<int>(end - beg);
  const int k = min(p.k, deg);

  int have = 0;  // sorted survivors at keys[0, have)
  uint32_t next = beg;
  if (k > 0) {
    while (next < end) {
      const int room = kWindow - have;
      const int take = min(static_cast<int>(end - next), room);
      int total = have + take;
      int pw = 32;
      while (pw < total) pw <<= 1;
      for (int i = threadIdx.x; i < pw - have; i += blockDim.x) {
        uint64_t key = 0;  // below every real key: real neighbours have weight >= 1
        if (i < take) {
          int32_t u = idx[next + i];
          key = (static_cast<uint64_t>(static_cast<uint32_t>(w[u])) << 32) |
                (0xFFFFFFFFu - static_cast<uint32_t>(u));
        }
        keys[have + i] = key;
      }
      __syncthreads();
      bitonic_sort_desc(keys, pw);
      next += take;
      have = k;
    }
  }
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    int32_t u = static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(keys[j] & 0xFFFFFFFFu));
    sel[static_cast<int64_t>(r) * p.k_stride + j] = u;
  }
  // byte length: "[Node:" E "]\n[neighbours:" {","}"(" E ")" "]"
  __shared__ unsigned long long acc;
  if (threadIdx.x == 0) acc = 0;
  __syncthreads();
  unsigned long long part = 0;
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    int32_t u = static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(keys[j] & 0xFFFFFFFFu));
    part += (g.entry_off[u + 1] - g.entry_off[u]) + 2 + (j > 0 ? 1 : 0);
  }
  atomicAdd(&acc, part);
  __syncthreads();
  if (threadIdx.x == 0) {
    sel_count[r] = k;
    byte_len[r] = acc + 6 + (g.entry_off[v + 1] - g.entry_off[v]) + 14 + 1;
  }
}

__device__ __forceinline__ void warp_copy(char* dst, const char* src, uint32_t n, int lane) {
  for (uint32_t i = lane; i < n; i += 32) dst[i] = src[i];
}

__global__ void __launch_bounds__(256)
chunk_render_kernel(DevGraph g, ChunkParams p, const int32_t* __restrict__ node_idx, int n_req,
                    const int32_t* __restrict__ sel, const int32_t* __restrict__ sel_count,
                    const uint64_t* __restrict__ byte_off, char* __restrict__ out) {
  extern __shared__ uint32_t piece_off[];  // k + 1
  const int r = blockIdx.x;
  if (r >= n_req) return;
  const int32_t v = node_idx[r];
  const int k = sel_count[r];
  const int32_t* mine = sel + static_cast<int64_t>(r) * p.k_stride;
  const uint32_t ec = g.entry_off[v + 1] - g.entry_off[v];
  const uint32_t head = 6 + ec + 14;
  if (threadIdx.x == 0) {
    uint32_t o = head;
    for (int j = 0; j < k; ++j) {
      piece_off[j] = o;
      int32_t u = mine[j];
      o += (g.entry_off[u + 1] - g.entry_off[u]) + 2 + (j > 0 ? 1 : 0);
    }
    piece_off[k] = o;
  }
  __syncthreads();
  char* dst = out + byte_off[r];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  if (warp == 0) {
    const char* hdr = "[Node:";
    if (lane < 6) dst[lane] = hdr[lane];
    warp_copy(dst + 6, g.entry_bytes + g.entry_off[v], ec, lane);
    const char* mid = "]\n[neighbours:";
    if (lane < 14) dst[6 + ec + lane] = mid[lane];
    if (lane == 0) dst[piece_off[k]] = ']';
  }
  for (int j = warp; j < k; j += nwarps) {
    int32_t u = mine[j];
    char* d = dst + piece_off[j];
    if (j > 0) {
      if (lane == 0) d[0] = ',';
      ++d;
    }
    const uint32_t eu = g.entry_off[u + 1] - g.entry_off[u];
    if (lane == 0) {
      d[0] = '(';
      d[1 + eu] = ')';
    }
    warp_copy(d + 1, g.entry_bytes + g.entry_off[u], eu, lane);
  }
}

// Locates the request that owns byte b (byte_off is exclusive-scanned, n_req+1 entries).
__device__ __forceinline__ int owner_of(const uint64_t* byte_off, int n_req, uint64_t b) {
  int lo = 0, hi = n_req - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (byte_off[mid] <= b) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void token_flag_kernel(const char* __restrict__ bytes, const uint64_t* __restrict__ byte_off,
                                  int n_req, uint64_t total, uint32_t* __restrict__ flag) {
  for (uint64_t b = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; b < total;
       b += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    unsigned char c = bytes[b];
    uint32_t f = 0;
    if (!dev_is_space(c)) {
      int r = owner_of(byte_off, n_req, b);
      f = (b == byte_off[r] || dev_is_space(static_cast<unsigned char>(bytes[b - 1]))) ? 1u : 0u;
    }
    flag[b] = f;
  }
}

__global__ void token_emit_kernel(const char* __restrict__ bytes, const uint64_t* __restrict__ byte_off,
                                  int n_req, uint64_t total, const uint32_t* __restrict__ flag,
                                  const uint32_t* __restrict__ tok_index, uint32_t vocab,
                                  int32_t* __restrict__ tok_id, uint64_t* __restrict__ tok_begin,
                                  uint64_t* __restrict__ tok_end, uint64_t* __restrict__ tok_off) {
  for (uint64_t b = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; b < total;
       b += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (!flag[b]) continue;
    // every chunk starts with "[Node:", so its first byte is always a token start
    const int r = owner_of(byte_off, n_req, b);
    if (b == byte_off[r]) tok_off[r] = tok_index[b];
    const uint64_t lim = byte_off[r + 1];
    uint64_t e = b + 1;
    while (e < lim && !dev_is_space(static_cast<unsigned char>(bytes[e]))) ++e;
    const uint32_t t = tok_index[b];
    tok_begin[t] = b - byte_off[r];
    tok_end[t] = e - byte_off[r];
    if (vocab) tok_id[t] = static_cast<int32_t>(dev_fnv1a(bytes + b, static_cast<uint32_t>(e - b)) % vocab);
  }
}

}  // namespace

void chunk_select(const DevGraph& g, const ChunkParams& p, const int32_t* node_idx, int n_req,
                  int32_t* sel, int32_t* sel_count, uint64_t* byte_len, cudaStream_t s) {
  chunk_select_kernel<<<n_req, kSelThreads, 0, s>>>(g, p, node_idx, n_req, sel, sel_count,
                                                    byte_len);
  GLMX_CHECK_LAUNCH();
}

void chunk_render(const DevGraph& g, const ChunkParams& p, const int32_t* node_idx, int n_req,
                  const int32_t* sel, const int32_t* sel_count, const uint64_t* byte_off,
                  char* out, cudaStream_t s) {
  chunk_render_kernel<<<n_req, 256, (p.k_stride + 1) * sizeof(uint32_t), s>>>(
      g, p, node_idx, n_req, sel, sel_count, byte_off, out);
  GLMX_CHECK_LAUNCH();
}

size_t scan_u64_temp_bytes(int n) {
  size_t t = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t, static_cast<uint64_t*>(nullptr),
                                static_cast<uint64_t*>(nullptr), n);
  return t;
}
size_t scan_u32_temp_bytes(uint64_t n) {
  size_t t = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t, static_cast<uint32_t*>(nullptr),
                                static_cast<uint32_t*>(nullptr), static_cast<int64_t>(n));
  return t;
}

void scan_u64(void* temp, size_t temp_bytes, const uint64_t* in, uint64_t* out, int n,
              cudaStream_t s) {
  GLMX_CUDA(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, in, out, n, s));
}

void scan_u32(void* temp, size_t temp_bytes, const uint32_t* in, uint32_t* out, uint64_t n,
              cudaStream_t s) {
  GLMX_CUDA(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, in, out, static_cast<int64_t>(n), s));
}

void chunk_tokenize(const char* bytes, const uint64_t* byte_off, int n_req, uint64_t total,
                    uint32_t* flag, uint32_t* tok_index, void* temp, size_t temp_bytes,
                    uint32_t vocab, int32_t* tok_id, uint64_t* tok_begin, uint64_t* tok_end,
                    uint64_t* tok_off, cudaStream_t s) {
  const int blocks = static_cast<int>(std::min<uint64_t>(ceil_div(total, 256), 148 * 16));
  token_flag_kernel<<<blocks, 256, 0, s>>>(bytes, byte_off, n_req, total, flag);
  GLMX_CHECK_LAUNCH();
  // flag has total+1 entries (last = 0) so tok_index[total] = token count
  scan_u32(temp, temp_bytes, flag, tok_index, total + 1, s);
  token_emit_kernel<<<blocks, 256, 0, s>>>(bytes, byte_off, n_req, total, flag, tok_index, vocab,
                                           tok_id, tok_begin, tok_end, tok_off);
  GLMX_CHECK_LAUNCH();
}

}  // namespace glmx
