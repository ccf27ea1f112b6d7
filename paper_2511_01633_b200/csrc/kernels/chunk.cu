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

// Whitespace tokens a neighbour piece [","] "(" E ")" adds to the chunk, from the entry's stats
// (kernels entry_stats_kernel): the piece is T(E) + 2 tokens, minus one where "(" fuses with E's
// first token and one where E's last token fuses with ")" (an empty E gives the one token "()"),
// minus one more because the piece's first byte ("," or "(") fuses with the byte before it (a ")"
// or the ":" of "[neighbours:").  The header "[Node:" E "]\n[neighbours:" is that + 2 and the
// closing "]" always fuses.
__device__ __forceinline__ uint32_t piece_tokens(uint32_t st) {
  const uint32_t T = st & 0x1FFFFFFFu, L = (st >> 29) & 1u;
  const uint32_t R = (st >> 31) ? (st >> 30) & 1u : 1u;
  return 1u + T - L - R;
}

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
                    uint64_t* __restrict__ byte_len, uint32_t* __restrict__ tok_count) {
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
  __shared__ unsigned int tacc;
  if (threadIdx.x == 0) {
    acc = 0;
    tacc = 0;
  }
  __syncthreads();
  unsigned long long part = 0;
  unsigned int tpart = 0;
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    int32_t u = static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(keys[j] & 0xFFFFFFFFu));
    part += (g.entry_off[u + 1] - g.entry_off[u]) + 2 + (j > 0 ? 1 : 0);
    tpart += piece_tokens(g.ent_stat[u]);
  }
  atomicAdd(&acc, part);
  atomicAdd(&tacc, tpart);
  __syncthreads();
  if (threadIdx.x == 0) {
    sel_count[r] = k;
    byte_len[r] = acc + 6 + (g.entry_off[v + 1] - g.entry_off[v]) + 14 + 1;
    tok_count[r] = tacc + piece_tokens(g.ent_stat[v]) + 2;
  }
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
                         uint64_t* __restrict__ byte_len, uint32_t* __restrict__ tok_count,
                         int32_t* __restrict__ big_list, int32_t* __restrict__ big_count) {
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
  if (deg <= 32) {
    // one key per lane: a 15-stage warp bitonic sort (descending) leaves the j-th pick in lane j
    uint64_t kk = 0;
    if (lane < deg) {
      const int32_t u = idx[beg + lane];
      kk = (static_cast<uint64_t>(static_cast<uint32_t>(w[u])) << 32) |
           (0xFFFFFFFFu - static_cast<uint32_t>(u));
    }
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        const uint64_t o = __shfl_xor_sync(0xffffffffu, kk, stride);
        const bool keep_max = ((lane & stride) == 0) == ((lane & size) == 0);
        kk = keep_max ? (o > kk ? o : kk) : (o < kk ? o : kk);
      }
    }
    uint32_t bytes = 0, toks = 0;
    if (lane < k) {
      const int32_t u = static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(kk));
      sel[static_cast<int64_t>(r) * p.k_stride + lane] = u;
      bytes = entry_len(g, u) + 2 + (lane > 0 ? 1 : 0);
      toks = piece_tokens(g.ent_stat[u]);
    }
    if (lane == 0) {
      bytes += 6 + entry_len(g, v) + 14 + 1;
      toks += piece_tokens(g.ent_stat[v]) + 2;
    }
    bytes = __reduce_add_sync(0xffffffffu, bytes);
    toks = __reduce_add_sync(0xffffffffu, toks);
    if (lane == 0) {
      sel_count[r] = k;
      byte_len[r] = bytes;
      tok_count[r] = toks;
    }
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
  int32_t pick[kWarpMaxK / 32] = {-1, -1};  // picks j with j % 32 == lane
  for (int j = 0; j < k; ++j) {
    const uint32_t hi = __reduce_max_sync(0xffffffffu, static_cast<uint32_t>(best >> 32));
    const bool cand = static_cast<uint32_t>(best >> 32) == hi;
    const uint32_t lo = __reduce_max_sync(0xffffffffu, cand ? static_cast<uint32_t>(best) : 0u);
    const bool mine = cand && static_cast<uint32_t>(best) == lo;  // unique: indices differ
    const int32_t u = static_cast<int32_t>(0xFFFFFFFFu - lo);
    if (lane == (j & 31)) {
      out[j] = u;
      pick[j >> 5] = u;
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
  // byte and token lengths of this lane's pieces: the entry loads of all picks issue together
  uint32_t bytes = 0, toks = 0;
#pragma unroll
  for (int i = 0; i < kWarpMaxK / 32; ++i) {
    const int32_t u = pick[i];
    if (u >= 0) {
      bytes += entry_len(g, u) + 2 + (lane + 32 * i > 0 ? 1 : 0);  // [","] "(" E ")"
      toks += piece_tokens(g.ent_stat[u]);
    }
  }
  if (lane == 0) {
    bytes += 6 + entry_len(g, v) + 14 + 1;
    toks += piece_tokens(g.ent_stat[v]) + 2;
  }
  bytes = __reduce_add_sync(0xffffffffu, bytes);
  toks = __reduce_add_sync(0xffffffffu, toks);
  if (lane == 0) {
    sel_count[r] = k;
    byte_len[r] = bytes;
    tok_count[r] = toks;
  }
}



// CTA path for hub rows (degree > 128) with k <= 64: each of the 8 warps streams its share of
// the row in 128-key slabs (4 keys per lane, loads of two slabs in flight) and keeps a running
// top-k in registers (slots j = lane, lane + 32); a slab whose keys are all below the current
// k-th best is skipped after one ballot.  The 8 partial top-k lists meet in shared memory and
// warp 0 selects the final k with the same REDUX picks as the warp path.
template <int kPer>
__device__ __forceinline__ int warp_pick_topk(uint64_t (&pool)[kPer], int k, uint64_t (&held)[2],
                                              int lane) {
  uint64_t best = 0;
#pragma unroll
  for (int i = 0; i < kPer; ++i) best = pool[i] > best ? pool[i] : best;
  held[0] = held[1] = 0;
  int got = 0;
  for (int j = 0; j < k; ++j) {
    const uint32_t hi = __reduce_max_sync(0xffffffffu, static_cast<uint32_t>(best >> 32));
    const bool cand = static_cast<uint32_t>(best >> 32) == hi;
    const uint32_t lo = __reduce_max_sync(0xffffffffu, cand ? static_cast<uint32_t>(best) : 0u);
    if (hi == 0 && lo == 0) break;  // fewer than k keys so far
    const uint64_t win = (static_cast<uint64_t>(hi) << 32) | lo;
    if (lane == (j & 31)) {
      if (j < 32) held[0] = win;
      else held[1] = win;
    }
    if (cand && static_cast<uint32_t>(best) == lo) {
      uint64_t nb = 0;
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        if (pool[i] == win) pool[i] = 0;
        nb = pool[i] > nb ? pool[i] : nb;
      }
      best = nb;
    }
    ++got;
  }
  return got;
}

__global__ void __launch_bounds__(256)
chunk_select_hub_kernel(DevGraph g, ChunkParams p, const int32_t* __restrict__ node_idx, int n_req,
                        const int32_t* __restrict__ big_list, const int32_t* __restrict__ big_count,
                        int32_t* __restrict__ sel, int32_t* __restrict__ sel_count,
                        uint64_t* __restrict__ byte_len, uint32_t* __restrict__ tok_count) {
  __shared__ uint64_t wtop[8][kWarpMaxK];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n_big = *big_count;
  const uint32_t* off = p.directed ? g.dir_off : g.und_off;
  const int32_t* idx = p.directed ? g.dir_idx : g.und_idx;
  const int32_t* w = p.weight_mode ? g.w_by_type : g.w_total;
  for (int bi = blockIdx.x; bi < n_big; bi += gridDim.x) {
    const int r = big_list[bi];
    const int32_t v = node_idx[r];
    const uint32_t beg = off[v], end = off[v + 1];
    const int deg = static_cast<int>(end - beg);
    const int k = min(p.k, deg);
    uint64_t held[2] = {0, 0};
    uint64_t thr = 0;  // k-th best key of this warp once it holds k keys
    for (int c0 = warp * 256; c0 < deg; c0 += 8 * 256) {
      // two 128-key slabs: 8 independent idx loads, then 8 weight gathers
      int32_t u[8];
      uint64_t key[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int e = c0 + lane + 32 * i;
        u[i] = e < deg ? idx[beg + e] : -1;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        key[i] = 0;
        if (u[i] >= 0) {
          const uint64_t kk = (static_cast<uint64_t>(static_cast<uint32_t>(w[u[i]])) << 32) |
                              (0xFFFFFFFFu - static_cast<uint32_t>(u[i]));
          key[i] = kk > thr ? kk : 0;
        }
      }
      bool any = false;
#pragma unroll
      for (int i = 0; i < 8; ++i) any |= key[i] != 0;
      if (!__any_sync(0xffffffffu, any)) continue;
      uint64_t pool[10] = {held[0], held[1], key[0], key[1], key[2], key[3],
                           key[4], key[5], key[6], key[7]};
      const int got = warp_pick_topk<10>(pool, k, held, lane);
      const uint64_t hk = __shfl_sync(0xffffffffu, k > 32 ? held[1] : held[0], (k - 1) & 31);
      thr = got == k ? hk : 0;
    }
    wtop[warp][lane] = held[0];
    if (lane + 32 < kWarpMaxK) wtop[warp][lane + 32] = held[1];
    __syncthreads();
    if (warp == 0) {
      // 8 x k candidates (k <= 64): 16 per lane
      uint64_t pool[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int e = lane + 32 * i;  // candidate e = warp e / 64, slot e % 64
        pool[i] = wtop[e >> 6][e & 63];
      }
      uint64_t fin[2];
      warp_pick_topk<16>(pool, k, fin, lane);
      int32_t* out = sel + static_cast<int64_t>(r) * p.k_stride;
      uint32_t bytes = 0, toks = 0;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int j = lane + 32 * i;
        if (j < k) {
          const int32_t uu = static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(fin[i]));
          out[j] = uu;
          bytes += entry_len(g, uu) + 2 + (j > 0 ? 1 : 0);
          toks += piece_tokens(g.ent_stat[uu]);
        }
      }
      if (lane == 0) {
        bytes += 6 + entry_len(g, v) + 14 + 1;
        toks += piece_tokens(g.ent_stat[v]) + 2;
      }
      bytes = __reduce_add_sync(0xffffffffu, bytes);
      toks = __reduce_add_sync(0xffffffffu, toks);
      if (lane == 0) {
        sel_count[r] = k;
        byte_len[r] = bytes;
        tok_count[r] = toks;
      }
    }
    __syncthreads();  // wtop reuse
  }
}

// ---------------------------------------------------------------------------------- render+emit
// One warp per chunk: the chunk is assembled in a per-warp shared-memory buffer placed at the
// same 16-byte phase as its global destination, written out with 16-byte stores, and tokenised
// from shared memory — the text is never read back from HBM.  Entry bytes are fetched as 16-byte
// aligned words: the words of all pieces of a round (the centre entry + up to 31 neighbours) are
// numbered by a warp scan, each lane finds its piece by a shuffle binary search, and four loads
// per lane are in flight before any byte is scattered.  Chunks longer than the buffer are built
// in place in global memory by the same code.
constexpr int kRW = 4;         // warps (chunks) per CTA
constexpr int kBuf = 6144;     // staged chunk bytes per warp
constexpr int kSeg = 1024;     // bytes per token-start compaction segment
constexpr int kWordsU = 4;     // 16-byte loads in flight per lane

// h % vocab for a 64-bit h by Barrett reduction with m = floor((2^64 - 1) / vocab): the estimate
// q = hi64(h * m) is at most 2 below the true quotient.
__device__ __forceinline__ uint32_t mod_vocab(uint64_t h, uint32_t vocab, uint64_t m) {
  const uint64_t q = __umul64hi(h, m);
  uint64_t r = h - q * vocab;
  if (r >= vocab) r -= vocab;
  if (r >= vocab) r -= vocab;
  return static_cast<uint32_t>(r);
}

__device__ __forceinline__ uint32_t first_space_after(const uint32_t* sp, uint32_t b, uint32_t n) {
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

// whitespace bits of the 4 bytes of x (bit j: byte j is ' ' or '\t'..'\r'), byte-SIMD
__device__ __forceinline__ uint32_t space_bits4(uint32_t x) {
  const uint32_t eq = __vcmpeq4(x, 0x20202020u);
  const uint32_t lt = __vcmpltu4(__vsub4(x, 0x09090909u), 0x05050505u);
  return ((((eq | lt) >> 7) & 0x01010101u) * 0x10204080u) >> 28;
}

// token-start bits of mask word w: a non-space byte after a space (position 0 counts as after one)
__device__ __forceinline__ uint32_t start_bits(const uint32_t* sp, uint32_t w) {
  const uint32_t m = sp[w];
  return ~m & ((m << 1) | (w ? sp[w - 1] >> 31 : 1u));
}

// first token start at a position >= q, or Q
__device__ __forceinline__ uint32_t next_start(const uint32_t* sp, uint32_t q, uint32_t nwm,
                                               uint32_t Q) {
  uint32_t w = q >> 5;
  if (w >= nwm) return Q;
  uint32_t st = start_bits(sp, w) & (~0u << (q & 31));
  while (st == 0) {
    if (++w >= nwm) return Q;
    st = start_bits(sp, w);
  }
  return min(Q, (w << 5) + __ffs(st) - 1);
}

// Assemble chunk bytes [0, n) at buf (shared or global).  Returns nothing; buf[n-1] = ']'.
__device__ __forceinline__ void build_chunk(const DevGraph& g, int32_t v, int k,
                                            const int32_t* __restrict__ mine, char* buf, int lane) {
  const uint32_t ev = g.entry_off[v];
  const uint32_t ec = g.entry_off[v + 1] - ev;
  if (lane < 6) buf[lane] = "[Node:"[lane];
  if (lane < 14) buf[6 + ec + lane] = "]\n[neighbours:"[lane];
  uint32_t o = 6 + ec + 14;  // offset of the next neighbour piece
  const uint4* words = reinterpret_cast<const uint4*>(g.entry_bytes);
  for (int s0 = 0; s0 <= k; s0 += 32) {
    // segment s = s0 + lane: s == 0 is the centre entry, s >= 1 neighbour piece j = s - 1
    const int s = s0 + lane;
    uint32_t src = 0, len = 0, dst = 0, plen = 0;
    if (s == 0) {
      src = ev;
      len = ec;
      dst = 6;
    } else if (s <= k) {
      const int j = s - 1;
      const int32_t u = mine[j];
      src = g.entry_off[u];
      len = g.entry_off[u + 1] - src;
      plen = len + 2 + (j > 0 ? 1u : 0u);
    }
    uint32_t pincl = plen;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, pincl, d);
      if (lane >= d) pincl += t;
    }
    if (s >= 1 && s <= k) {
      const uint32_t pst = o + pincl - plen;
      const uint32_t c = s > 1 ? 1u : 0u;
      if (c) buf[pst] = ',';
      buf[pst + c] = '(';
      buf[pst + c + 1 + len] = ')';
      dst = pst + c + 1;
    }
    o += __shfl_sync(0xffffffffu, pincl, 31);
    // 16-byte words covering [src, src + len), numbered across the round's segments
    const uint32_t wc = len ? ((src + len - 1) >> 4) - (src >> 4) + 1 : 0;
    uint32_t wincl = wc;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, wincl, d);
      if (lane >= d) wincl += t;
    }
    const uint32_t W = __shfl_sync(0xffffffffu, wincl, 31);
    const uint32_t wexcl = wincl - wc;
    for (uint32_t w0 = 0; w0 < W; w0 += 32 * kWordsU) {
      uint4 x[kWordsU];
      uint32_t qsrc[kWordsU], qlen[kWordsU], qdst[kWordsU], qword[kWordsU];
#pragma unroll
      for (int t = 0; t < kWordsU; ++t) {
        const uint32_t wi = w0 + t * 32 + lane;
        int q = 0;  // last segment whose first word is <= wi
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
          const uint32_t e = __shfl_sync(0xffffffffu, wexcl, q + step);
          if (e <= wi) q += step;
        }
        const uint32_t qe = __shfl_sync(0xffffffffu, wexcl, q);
        qsrc[t] = __shfl_sync(0xffffffffu, src, q);
        qlen[t] = __shfl_sync(0xffffffffu, len, q);
        qdst[t] = __shfl_sync(0xffffffffu, dst, q);
        qword[t] = (qsrc[t] >> 4) + (wi - qe);
        x[t] = wi < W ? __ldg(words + qword[t]) : make_uint4(0, 0, 0, 0);
        if (wi >= W) qlen[t] = 0;
      }
#pragma unroll
      for (int t = 0; t < kWordsU; ++t) {
        const uint32_t base = qword[t] << 4;
        const uint32_t xs[4] = {x[t].x, x[t].y, x[t].z, x[t].w};
        if (qlen[t] && base >= qsrc[t] && base + 16 <= qsrc[t] + qlen[t]) {
          // interior word: realign the 16 bytes to the destination's 4-byte phase s and store
          // 3 aligned words (funnel shifts) plus 4 edge bytes (4 words when s == 0)
          char* d = buf + qdst[t] + (base - qsrc[t]);
          const uint32_t s = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(d)) & 3u;
          if (s == 0) {
            uint32_t* d4 = reinterpret_cast<uint32_t*>(d);
            d4[0] = xs[0];
            d4[1] = xs[1];
            d4[2] = xs[2];
            d4[3] = xs[3];
          } else {
            const uint32_t sh = 8 * (4 - s);
            uint32_t* a4 = reinterpret_cast<uint32_t*>(d + (4 - s));
            a4[0] = __funnelshift_r(xs[0], xs[1], sh);
            a4[1] = __funnelshift_r(xs[1], xs[2], sh);
            a4[2] = __funnelshift_r(xs[2], xs[3], sh);
#pragma unroll
            for (uint32_t j = 0; j < 3; ++j) {
              if (j < 4 - s) d[j] = static_cast<char>(xs[0] >> (8 * j));
              if (j < s) d[16 - s + j] = static_cast<char>(xs[3] >> (8 * (4 - s + j)));
            }
          }
        } else {
#pragma unroll
          for (int b = 0; b < 16; ++b) {
            const uint32_t gp = base + b;
            if (gp >= qsrc[t] && gp < qsrc[t] + qlen[t])
              buf[qdst[t] + (gp - qsrc[t])] = static_cast<char>(xs[b >> 2] >> ((b & 3) * 8));
          }
        }
      }
    }
  }
  if (lane == 0) buf[o] = ']';
  __syncwarp();
}

__global__ void __launch_bounds__(kRW * 32, 7)
chunk_render_emit_kernel(DevGraph g, ChunkParams p, const int32_t* __restrict__ node_idx,
                         int n_req, const int32_t* __restrict__ sel,
                         const int32_t* __restrict__ sel_count,
                         const uint64_t* __restrict__ byte_off, const uint32_t* __restrict__ tok_off,
                         uint32_t vocab, uint64_t vmagic, char* __restrict__ out,
                         int32_t* __restrict__ tok_id, uint64_t* __restrict__ tok_begin,
                         uint64_t* __restrict__ tok_end) {
  __shared__ __align__(16) char sbuf[kRW][kBuf + 16];
  __shared__ uint32_t smask[kRW][kBuf / 32 + 1];
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  const int r = blockIdx.x * kRW + wi;
  if (r >= n_req) return;
  const int32_t v = node_idx[r];
  const int k = sel_count[r];
  const int32_t* mine = sel + static_cast<int64_t>(r) * p.k_stride;
  const uint64_t goff = byte_off[r];
  const uint32_t n = static_cast<uint32_t>(byte_off[r + 1] - goff);
  const bool staged = n <= kBuf;
  char* gdst = out + goff;
  uint32_t* sp = smask[wi];
  // token-start list of the unstaged path (chunks > kBuf), which leaves the staging buffer free
  uint32_t* list = reinterpret_cast<uint32_t*>(sbuf[wi]);
  uint32_t t = tok_off[r];
  if (staged) {
    // staged span: smem bytes [pad, Q) hold the chunk at the 16-byte phase of its destination
    char* sb = sbuf[wi];
    const uint32_t pad = static_cast<uint32_t>(goff & 15), Q = pad + n;
    build_chunk(g, v, k, mine, sb + pad, lane);
    // per 16-byte word (one per lane): text out (aligned words as one 16-byte store, the two edge
    // words byte by byte) and 16 whitespace bits; bytes outside [pad, Q) count as spaces
    char* gbase = out + (goff - pad);
    const uint32_t nw16 = (Q + 15) >> 4;
    for (uint32_t i0 = 0; i0 < nw16; i0 += 32) {
      const uint32_t i = i0 + lane;
      uint32_t bits = 0xFFFFu;
      if (i < nw16) {
        const uint4 x = *reinterpret_cast<const uint4*>(sb + 16 * i);
        const uint32_t lo = 16 * i, hi = lo + 16;
        if (lo >= pad && hi <= Q) {
          *reinterpret_cast<uint4*>(gbase + lo) = x;
        } else {
          for (uint32_t q = max(lo, pad); q < min(hi, Q); ++q) gbase[q] = sb[q];
        }
        bits = space_bits4(x.x) | (space_bits4(x.y) << 4) | (space_bits4(x.z) << 8) |
               (space_bits4(x.w) << 12);
        if (lo < pad) bits |= (1u << (pad - lo)) - 1u;
        if (hi > Q) bits |= 0xFFFFu & ~((1u << (Q - lo)) - 1u);
      }
      const uint32_t up = __shfl_down_sync(0xffffffffu, bits, 1);
      if ((lane & 1) == 0 && i < nw16) sp[i >> 1] = bits | (up << 16);
    }
    __syncwarp();
    // tokens: lane L owns the token STARTS in its contiguous byte range [qs, qe); the output
    // index is a warp scan of the per-lane start counts.  Balanced by bytes, not by tokens.
    const uint32_t nwm = (Q + 31) >> 5;
    const uint32_t per = (((Q + 31) >> 5) + 3) & ~3u;
    const uint32_t qs = min(Q, lane * per), qe = min(Q, qs + per);
    uint32_t c = 0;
    for (uint32_t w = qs >> 5; (w << 5) < qe; ++w) {
      uint32_t st = start_bits(sp, w);
      const uint32_t wlo = w << 5;
      if (qs > wlo) st &= ~0u << (qs - wlo);
      if (qe < wlo + 32) st &= (1u << (qe - wlo)) - 1u;
      c += __popc(st);
    }
    uint32_t incl = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t x = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += x;
    }
    uint32_t o = t + incl - c;
    for (uint32_t b = next_start(sp, qs, nwm, Q); b < qe;) {
      const uint32_t e = first_space_after(sp, b, Q);
      uint64_t h = 14695981039346656037ULL;
#pragma unroll 4
      for (uint32_t q = b; q < e; ++q) h = (h ^ static_cast<unsigned char>(sb[q])) * 1099511628211ULL;
      tok_begin[o] = b - pad;
      tok_end[o] = e - pad;
      if (vocab) tok_id[o] = static_cast<int32_t>(mod_vocab(h, vocab, vmagic));
      ++o;
      b = next_start(sp, e, nwm, Q);
    }
    return;
  }
  // longer than the buffer: built in place in global memory, tokenised from there
  build_chunk(g, v, k, mine, gdst, lane);
  const char* src = gdst;
  for (uint32_t s0 = 0; s0 < n; s0 += kSeg) {
    uint32_t cnt = 0;
    const uint32_t s1 = min(n, s0 + kSeg);
    for (uint32_t b0 = s0; b0 < s1; b0 += 32) {
      const uint32_t b = b0 + lane;
      const bool start = b < s1 && !dev_is_space(static_cast<unsigned char>(src[b])) &&
                         (b == 0 || dev_is_space(static_cast<unsigned char>(src[b - 1])));
      const uint32_t mask = __ballot_sync(0xffffffffu, start);
      if (start) list[cnt + __popc(mask & ((1u << lane) - 1u))] = b;
      cnt += __popc(mask);
    }
    __syncwarp();
    for (uint32_t i = lane; i < cnt; i += 32) {
      const uint32_t b = list[i];
      uint32_t e = b + 1;
      while (e < n && !dev_is_space(static_cast<unsigned char>(src[e]))) ++e;
      uint64_t h = 14695981039346656037ULL;
      for (uint32_t q = b; q < e; ++q) h = (h ^ static_cast<unsigned char>(src[q])) * 1099511628211ULL;
      tok_begin[t + i] = b;
      tok_end[t + i] = e;
      if (vocab) tok_id[t + i] = static_cast<int32_t>(mod_vocab(h, vocab, vmagic));
    }
    t += cnt;
    __syncwarp();
  }
}

// Per-entry whitespace stats for the token count of a chunk: bits 0-28 number of whitespace
// tokens, 29 first byte is not a space, 30 last byte is not a space, 31 non-empty.
__global__ void entry_stats_kernel(const char* __restrict__ bytes, const uint32_t* __restrict__ off,
                                   uint32_t n, uint32_t* __restrict__ st) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t b = off[i], e = off[i + 1];
  uint32_t T = 0;
  bool prev_space = true;
  for (uint32_t q = b; q < e; ++q) {
    const bool sp = dev_is_space(static_cast<unsigned char>(bytes[q]));
    T += (!sp && prev_space) ? 1u : 0u;
    prev_space = sp;
  }
  uint32_t w = T & 0x1FFFFFFFu;
  if (e > b) {
    w |= 1u << 31;
    if (!dev_is_space(static_cast<unsigned char>(bytes[b]))) w |= 1u << 29;
    if (!dev_is_space(static_cast<unsigned char>(bytes[e - 1]))) w |= 1u << 30;
  }
  st[i] = w;
}
}  // namespace

void chunk_select(const DevGraph& g, const ChunkParams& p, const int32_t* node_idx, int n_req,
                  int32_t* sel, int32_t* sel_count, uint64_t* byte_len, uint32_t* tok_count,
                  int32_t* big_list, int32_t* big_count, cudaStream_t s) {
  GLMX_CUDA(cudaMemsetAsync(big_count, 0, 4, s));
  chunk_select_warp_kernel<<<static_cast<int>(ceil_div(n_req, 8)), 256, 0, s>>>(
      g, p, node_idx, n_req, sel, sel_count, byte_len, tok_count, big_list, big_count);
  GLMX_CHECK_LAUNCH();
  // CTA path for hub rows / large k: a fixed grid walks the queued requests (warp-merge top-k for
  // k <= 64, the bitonic window for larger k)
  if (p.k <= kWarpMaxK)
    chunk_select_hub_kernel<<<std::min(n_req, kNumSMs * 4), 256, 0, s>>>(
        g, p, node_idx, n_req, big_list, big_count, sel, sel_count, byte_len, tok_count);
  else
    chunk_select_kernel<<<std::min(n_req, kNumSMs * 4), kSelThreads, 0, s>>>(
        g, p, node_idx, n_req, big_list, big_count, sel, sel_count, byte_len, tok_count);
  GLMX_CHECK_LAUNCH();
}

void chunk_render_emit(const DevGraph& g, const ChunkParams& p, const int32_t* node_idx, int n_req,
                       const int32_t* sel, const int32_t* sel_count, const uint64_t* byte_off,
                       const uint32_t* tok_off, uint32_t vocab, char* out, int32_t* tok_id,
                       uint64_t* tok_begin, uint64_t* tok_end, cudaStream_t s) {
  const uint64_t vmagic = vocab ? ~uint64_t(0) / vocab : 0;
  chunk_render_emit_kernel<<<static_cast<int>(ceil_div(n_req, kRW)), kRW * 32, 0, s>>>(
      g, p, node_idx, n_req, sel, sel_count, byte_off, tok_off, vocab, vmagic, out, tok_id,
      tok_begin, tok_end);
  GLMX_CHECK_LAUNCH();
}

void entry_stats(const char* bytes, const uint32_t* off, uint32_t n, uint32_t* st, cudaStream_t s) {
  if (n == 0) return;
  entry_stats_kernel<<<static_cast<int>(ceil_div(n, 256)), 256, 0, s>>>(bytes, off, n, st);
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
