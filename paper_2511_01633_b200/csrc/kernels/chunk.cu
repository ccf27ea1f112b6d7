// K1 — batched vertex-chunk assembly (Retriever::node_info + render_chunk, retriever.cpp:9-30,
// 74-121; tokenize, tokenizer.hpp:14-25).  One WARP per chunk end to end:
//
//   select  : CSR row gather of the de-duplicated neighbour set into registers (<= 4 keys per
//             lane, rows up to 128), then a warp-level top-k by repeated selection: the 64-bit key
//             w<<32 | ~idx (weight desc, node index asc) is reduced with two REDUX max steps
//             (weight word, then index word among the lanes holding the top weight) per pick.
//             Rows longer than 128 (hubs) or k > 64 are queued for the CTA path: bitonic sort in
//             shared memory over a 1024-key window that the row streams through.
//             The chunk's byte length is a warp sum of the selected entries' lengths.
//   scan    : exclusive sums of chunk lengths (cub) -> byte offsets.
//   render  : the warp scatters the pre-rendered per-node entries "<id> {k:v,...}" between the
//             literal separators (warp exclusive scan of entry lengths for the piece offsets), then
//             counts the chunk's whitespace tokens with ballots over its own bytes.
//   scan    : exclusive sums of token counts -> token offsets.
//   emit    : per 32-byte window a ballot marks token starts; each start lane walks to its token
//             end and hashes the bytes (fnv1a -> id); spans are written at the token offset.
//             Tokens fuse across entry boundaries exactly as in the text ("[neighbours:(n3",
//             "type:item}),(u1").
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
                    const int32_t* __restrict__ big_list, const int32_t* __restrict__ big_count,
                    int32_t* __restrict__ sel, int32_t* __restrict__ sel_count,
                    uint64_t* __restrict__ byte_len) {
  __shared__ uint64_t keys[kWindow];
  const int n_big = *big_count;
  for (int bi = blockIdx.x; bi < n_big; bi += gridDim.x) {
  __syncthreads();  // keys / acc reuse across iterations
  const int r = big_list[bi];
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

constexpr int kWarpKeys = 4;                 // keys per lane on the warp path
constexpr int kWarpMaxDeg = 32 * kWarpKeys;  // longer rows take the CTA path
constexpr int kWarpMaxK = 64;

__device__ __forceinline__ uint32_t entry_len(const DevGraph& g, int32_t u) {
  return g.entry_off[u + 1] - g.entry_off[u];
}

// Warp path of select (8 warps per CTA, one chunk each).  Rows that do not fit are appended to
// big_list for chunk_select_kernel.
__global__ void __launch_bounds__(256)
chunk_select_warp_kernel(DevGraph g, ChunkParams p, const int32_t* __restrict__ node_idx,
                         int n_req, int32_t* __restrict__ sel, int32_t* __restrict__ sel_count,
                         uint64_t* __restrict__ byte_len, int32_t* __restrict__ big_list,
                         int32_t* __restrict__ big_count) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= n_req) return;
  const int32_t v = node_idx[r];
  const uint32_t* off = p.directed ? g.dir_off : g.und_off;
  const int32_t* idx = p.directed ? g.dir_idx : g.und_idx;
  const int32_t* w = p.weight_mode ? g.w_by_type : g.w_total;
  const uint32_t beg = off[v], end = off[v + 1];
  const int deg = static_cast<int>(end - beg);
  const int k = min(p.k, deg);
  if (deg > kWarpMaxDeg || k > kWarpMaxK) {
    if (lane == 0) big_list[atomicAdd(big_count, 1)] = r;
    return;
  }
  // lane holds neighbours lane, lane+32, ... ; key 0 = empty (real weights are >= 1)
  uint64_t key[kWarpKeys];
#pragma unroll
  for (int i = 0; i < kWarpKeys; ++i) {
    const int e = lane + 32 * i;
    key[i] = 0;
    if (e < deg) {
      const int32_t u = idx[beg + e];
      key[i] = (static_cast<uint64_t>(static_cast<uint32_t>(w[u])) << 32) |
               (0xFFFFFFFFu - static_cast<uint32_t>(u));
    }
  }
  uint64_t best = key[0];
#pragma unroll
  for (int i = 1; i < kWarpKeys; ++i) best = key[i] > best ? key[i] : best;
  int32_t* out = sel + static_cast<int64_t>(r) * p.k_stride;
  uint32_t bytes = 0;  // this lane's share of the neighbour pieces
  for (int j = 0; j < k; ++j) {
    const uint32_t hi = __reduce_max_sync(0xffffffffu, static_cast<uint32_t>(best >> 32));
    const bool cand = static_cast<uint32_t>(best >> 32) == hi;
    const uint32_t lo = __reduce_max_sync(0xffffffffu, cand ? static_cast<uint32_t>(best) : 0u);
    const bool mine = cand && static_cast<uint32_t>(best) == lo;  // unique: indices differ
    const int32_t u = static_cast<int32_t>(0xFFFFFFFFu - lo);
    if (lane == (j & 31)) {
      out[j] = u;
      bytes += entry_len(g, u) + 2 + (j > 0 ? 1 : 0);  // "(" E ")" and the "," separator
    }
    if (mine) {  // drop the winner, recompute this lane's best
      uint64_t nb = 0;
#pragma unroll
      for (int i = 0; i < kWarpKeys; ++i) {
        if (key[i] == best) key[i] = 0;
        nb = key[i] > nb ? key[i] : nb;
      }
      best = nb;
    }
  }
  bytes = __reduce_add_sync(0xffffffffu, bytes);
  if (lane == 0) {
    sel_count[r] = k;
    byte_len[r] = bytes + 6 + entry_len(g, v) + 14 + 1;
  }
}

__device__ __forceinline__ void warp_copy_bytes(char* dst, const char* src, uint32_t n, int lane) {
  for (uint32_t i = lane; i < n; i += 32) dst[i] = src[i];
}

// Render one chunk per warp, then count its whitespace tokens (ballot over the chunk's bytes).
__global__ void __launch_bounds__(256)
chunk_render_warp_kernel(DevGraph g, ChunkParams p, const int32_t* __restrict__ node_idx,
                         int n_req, const int32_t* __restrict__ sel,
                         const int32_t* __restrict__ sel_count, const uint64_t* __restrict__ byte_off,
                         char* __restrict__ out, uint32_t* __restrict__ tok_count) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= n_req) return;
  const int32_t v = node_idx[r];
  const int k = sel_count[r];
  const int32_t* mine = sel + static_cast<int64_t>(r) * p.k_stride;
  char* dst = out + byte_off[r];
  const uint32_t ec = entry_len(g, v);
  if (lane < 6) dst[lane] = "[Node:"[lane];
  warp_copy_bytes(dst + 6, g.entry_bytes + g.entry_off[v], ec, lane);
  if (lane < 14) dst[6 + ec + lane] = "]\n[neighbours:"[lane];
  uint32_t o = 6 + ec + 14;  // offset of the next piece, uniform across the warp
  for (int j0 = 0; j0 < k; j0 += 32) {
    const int j = j0 + lane;
    const int32_t u = j < k ? mine[j] : 0;
    const uint32_t len = j < k ? entry_len(g, u) + 2 + (j > 0 ? 1 : 0) : 0;
    uint32_t incl = len;  // warp inclusive scan of piece lengths
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += t;
    }
    const uint32_t my_off = o + incl - len;
    const int n_here = min(32, k - j0);
    for (int q = 0; q < n_here; ++q) {
      const uint32_t po = __shfl_sync(0xffffffffu, my_off, q);
      const int32_t uq = __shfl_sync(0xffffffffu, u, q);
      char* d = dst + po;
      if (j0 + q > 0) {
        if (lane == 0) d[0] = ',';
        ++d;
      }
      const uint32_t eu = entry_len(g, uq);
      if (lane == 0) d[0] = '(';
      if (lane == 1) d[1 + eu] = ')';
      warp_copy_bytes(d + 1, g.entry_bytes + g.entry_off[uq], eu, lane);
    }
    o += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) dst[o] = ']';
  const uint32_t n = o + 1;
  __syncwarp();
  // token starts: non-space byte at position 0 or after a space
  uint32_t cnt = 0;
  for (uint32_t b = lane; b < n; b += 32) {
    const bool start = !dev_is_space(static_cast<unsigned char>(dst[b])) &&
                       (b == 0 || dev_is_space(static_cast<unsigned char>(dst[b - 1])));
    cnt += start ? 1u : 0u;
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if (lane == 0) tok_count[r] = cnt;
}

// Token spans + ids of one chunk per warp; tok_off = exclusive scan of the per-chunk counts.
// The chunk is staged in a per-warp shared-memory buffer together with its whitespace bitmask
// (one ballot per 32 bytes).  Then, per 1 KB segment, the token starts are compacted into a
// shared list (ballot + popc ranks) and the warp processes the list one TOKEN per lane: end by
// bit scans over the mask, fnv1a over the staged bytes, and coalesced span/id stores.  Chunks
// longer than the buffer (k in the hundreds) take the same steps reading global memory.
constexpr int kEmitWarps = 4;
constexpr int kEmitBuf = 8192;
constexpr int kEmitSeg = 1024;

__device__ __forceinline__ uint32_t token_end_from_mask(const uint32_t* sp, uint32_t b, uint32_t n) {
  // first whitespace position > b, or n
  uint32_t w = (b + 1) >> 5;
  uint32_t m = (b + 1) & 31 ? sp[w] & (0xFFFFFFFFu << ((b + 1) & 31)) : sp[w];
  const uint32_t nw = (n + 31) >> 5;
  while (m == 0) {
    if (++w >= nw) return n;
    m = sp[w];
  }
  return min(n, (w << 5) + __ffs(m) - 1);
}

__global__ void __launch_bounds__(kEmitWarps * 32)
chunk_emit_warp_kernel(const char* __restrict__ bytes, const uint64_t* __restrict__ byte_off,
                       int n_req, const uint32_t* __restrict__ tok_off, uint32_t vocab,
                       int32_t* __restrict__ tok_id, uint64_t* __restrict__ tok_begin,
                       uint64_t* __restrict__ tok_end) {
  __shared__ char sbuf[kEmitWarps][kEmitBuf];
  __shared__ uint32_t smask[kEmitWarps][kEmitBuf / 32 + 1];
  __shared__ uint32_t slist[kEmitWarps][kEmitSeg / 2 + 1];
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  const int r = blockIdx.x * kEmitWarps + wi;
  if (r >= n_req) return;
  const char* c = bytes + byte_off[r];
  const uint32_t n = static_cast<uint32_t>(byte_off[r + 1] - byte_off[r]);
  uint32_t t = tok_off[r];
  const bool staged = n <= kEmitBuf;
  const char* src = staged ? sbuf[wi] : c;
  uint32_t* sp = smask[wi];
  uint32_t* list = slist[wi];
  if (staged) {
    char* buf = sbuf[wi];
    for (uint32_t b0 = 0; b0 < n; b0 += 32) {
      const uint32_t b = b0 + lane;
      const char ch = b < n ? c[b] : ' ';
      buf[b] = ch;  // b < roundup(n, 32) <= kEmitBuf
      const uint32_t m = __ballot_sync(0xffffffffu, dev_is_space(static_cast<unsigned char>(ch)));
      if (lane == 0) sp[b0 >> 5] = m;
    }
    __syncwarp();
  }
  for (uint32_t s0 = 0; s0 < n; s0 += kEmitSeg) {
    // compact the token starts of this segment
    uint32_t cnt = 0;
    const uint32_t s1 = min(n, s0 + kEmitSeg);
    for (uint32_t b0 = s0; b0 < s1; b0 += 32) {
      const uint32_t b = b0 + lane;
      bool start = false;
      if (b < s1) {
        if (staged) {
          const uint32_t m = sp[b0 >> 5];
          const bool sp_prev = lane ? (m >> (lane - 1)) & 1u : (b == 0 || ((sp[(b0 >> 5) - 1] >> 31) & 1u));
          start = !((m >> lane) & 1u) && sp_prev;
        } else {
          start = !dev_is_space(static_cast<unsigned char>(c[b])) &&
                  (b == 0 || dev_is_space(static_cast<unsigned char>(c[b - 1])));
        }
      }
      const uint32_t mask = __ballot_sync(0xffffffffu, start);
      if (start) list[cnt + __popc(mask & ((1u << lane) - 1u))] = b;
      cnt += __popc(mask);
    }
    __syncwarp();
    // one token per lane
    for (uint32_t i = lane; i < cnt; i += 32) {
      const uint32_t b = list[i];
      uint32_t e;
      if (staged) {
        e = token_end_from_mask(sp, b, n);
      } else {
        e = b + 1;
        while (e < n && !dev_is_space(static_cast<unsigned char>(c[e]))) ++e;
      }
      uint64_t h = 14695981039346656037ULL;
      for (uint32_t q = b; q < e; ++q) h = (h ^ static_cast<unsigned char>(src[q])) * 1099511628211ULL;
      tok_begin[t + i] = b;
      tok_end[t + i] = e;
      if (vocab) tok_id[t + i] = static_cast<int32_t>(h % vocab);
    }
    t += cnt;
    __syncwarp();
  }
}

}  // namespace

void chunk_select(const DevGraph& g, const ChunkParams& p, const int32_t* node_idx, int n_req,
                  int32_t* sel, int32_t* sel_count, uint64_t* byte_len, int32_t* big_list,
                  int32_t* big_count, cudaStream_t s) {
  GLMX_CUDA(cudaMemsetAsync(big_count, 0, 4, s));
  chunk_select_warp_kernel<<<static_cast<int>(ceil_div(n_req, 8)), 256, 0, s>>>(
      g, p, node_idx, n_req, sel, sel_count, byte_len, big_list, big_count);
  GLMX_CHECK_LAUNCH();
  // CTA path for hub rows / large k: a fixed grid walks the queued requests
  chunk_select_kernel<<<std::min(n_req, kNumSMs * 4), kSelThreads, 0, s>>>(
      g, p, node_idx, n_req, big_list, big_count, sel, sel_count, byte_len);
  GLMX_CHECK_LAUNCH();
}

void chunk_render(const DevGraph& g, const ChunkParams& p, const int32_t* node_idx, int n_req,
                  const int32_t* sel, const int32_t* sel_count, const uint64_t* byte_off,
                  char* out, uint32_t* tok_count, cudaStream_t s) {
  chunk_render_warp_kernel<<<static_cast<int>(ceil_div(n_req, 8)), 256, 0, s>>>(
      g, p, node_idx, n_req, sel, sel_count, byte_off, out, tok_count);
  GLMX_CHECK_LAUNCH();
}

void chunk_emit(const char* bytes, const uint64_t* byte_off, int n_req, const uint32_t* tok_off,
                uint32_t vocab, int32_t* tok_id, uint64_t* tok_begin, uint64_t* tok_end,
                cudaStream_t s) {
  chunk_emit_warp_kernel<<<static_cast<int>(ceil_div(n_req, kEmitWarps)), kEmitWarps * 32, 0, s>>>(
      bytes, byte_off, n_req, tok_off, vocab, tok_id, tok_begin, tok_end);
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

}  // namespace glmx
