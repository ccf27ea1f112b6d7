// K1 — batched vertex-chunk assembly (Retriever::node_info + render_chunk, retriever.cpp:9-30,
// 74-121; tokenize, tokenizer.hpp:14-25).
//
// Ingest-time tables (the graph is immutable):
//   ranked adjacency : per (weight mode, directed) variant, every CSR row sorted by (weight desc,
//                      node index asc) -- node_info's stable_sort order (retriever.cpp:97-113) --
//                      plus exclusive prefix sums along the rows of the piece bytes (entry + 3),
//                      piece tokens and irregular entries: top-k of a row is its first k entries,
//                      and a chunk's byte length / token count are two differences of prefixes
//   entry tokens     : per regular entry (first and last byte non-space, >= 2 tokens) the spans
//                      and fnv1a hashes of its interior tokens, its first-token length and its
//                      last token's offset + fnv1a state
// Per batch (chunk_build):
//   chunk_len_scan : one thread per chunk computes (k', byte length, token count, regular flag)
//                    from the prefixes; both exclusive scans in the same single-pass kernel
//                    (warp-cooperative decoupled look-back); irregular chunks compacted to a list
//   chunk_regular  : CTA = a text warp + a token warp for one chunk.  Text: per round of 32
//                    pieces the 16-byte source words are numbered by a warp scan, each lane finds
//                    its piece by a shuffle binary search, realigns the words to the destination
//                    with funnel shifts and stores them whole (the separator bytes framing each
//                    entry are merged into its edge words), into a per-warp smem buffer at the
//                    destination's 16-byte phase, then 16-byte stores.  Tokens (emit_fast): the
//                    k + 3 junction tokens hashed from the neighbouring entries' precomputed
//                    states over the separator and first-token bytes; interior tokens copied from
//                    the tables (ids precomputed per vocab).
//   chunk_irregular: a small grid over the irregular list: byte-level tokenizer over a whitespace
//                    mask (per-token fnv1a).
// Tokens fuse across entry boundaries exactly as in the text ("[neighbours:(n3", "type:item}),(u1").
// All of it is integer/byte work: HBM/latency bound, no tensor cores.
#include <cub/cub.cuh>

#include "chunk.cuh"
#include "common.cuh"

namespace glmx {

namespace {

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


// regular entry: non-empty, first and last byte non-space, >= 2 tokens (head != tail)
__device__ __forceinline__ bool entry_regular(uint32_t st) {
  return (st >> 29) == 7u && (st & 0x1FFFFFFFu) >= 2;
}

// Per chunk r: k' = min(k, deg), byte length, whitespace token count and the regular flag (bit 31
// of sel_count), from the ranked-adjacency prefixes.
struct ChunkLen {
  uint64_t bytes;
  uint32_t toks;
  uint32_t sel;
  uint32_t row;
};
__device__ __forceinline__ ChunkLen chunk_len(const DevGraph& g, const RankedAdj& ra, int k,
                                              int32_t v) {
  const uint32_t row = ra.off[v], deg = ra.off[v + 1] - row;
  const uint32_t kk = min(static_cast<uint32_t>(k), deg);
  const uint32_t sv = g.ent_stat[v];
  const uint64_t pb = ra.pbytes[row + kk] - ra.pbytes[row];
  ChunkLen c;
  // "[Node:" E_v "]\n[neighbours:" {(","), "(" E ")"} "]"
  c.bytes = 6 + (g.entry_off[v + 1] - g.entry_off[v]) + 14 + (kk ? pb - 1 : 0) + 1;
  c.toks = piece_tokens(sv) + 2 + (ra.ptoks[row + kk] - ra.ptoks[row]);
  const bool irregular = !entry_regular(sv) || ra.pirr[row + kk] != ra.pirr[row];
  c.sel = kk | (irregular ? 0x80000000u : 0u);
  c.row = row;
  return c;
}

// Lengths + both exclusive scans in one single-pass kernel (decoupled look-back): tile t (kLenTile
// chunks, blockIdx order) publishes its aggregate, sums its predecessors' aggregates / inclusive
// prefixes back to the first inclusive one, then publishes its own inclusive prefix.  Status words
// carry the call's epoch, so the state needs no reset between calls.  Outputs byte_off[0..n] and
// tok_off[0..n] ([n] = totals) and sel_count.
constexpr int kLenThreads = 256, kLenItems = 1, kLenTile = kLenThreads * kLenItems;

__global__ void __launch_bounds__(kLenThreads)
chunk_len_scan_kernel(DevGraph g, RankedAdj ra, int k, const int32_t* __restrict__ node_idx,
                      int n_req, int32_t* __restrict__ sel_count, uint64_t* __restrict__ byte_off,
                      uint32_t* __restrict__ tok_off, ScanState st, uint32_t epoch,
                      int32_t* __restrict__ irr_list, int32_t* __restrict__ irr_count,
                      int2* __restrict__ vrow) {
  using BS64 = cub::BlockScan<uint64_t, kLenThreads>;
  using BS32 = cub::BlockScan<uint32_t, kLenThreads>;
  __shared__ typename BS64::TempStorage t64;
  __shared__ typename BS32::TempStorage t32;
  __shared__ uint64_t pre_b;
  __shared__ uint32_t pre_t;
  const int tile = blockIdx.x;
  const int r0 = tile * kLenTile + threadIdx.x * kLenItems;
  ChunkLen c[kLenItems];
  int32_t vv[kLenItems];
  uint64_t sb = 0;
  uint32_t stk = 0;
#pragma unroll
  for (int i = 0; i < kLenItems; ++i) {
    c[i] = ChunkLen{0, 0, 0, 0};
    vv[i] = 0;
    if (r0 + i < n_req) {
      vv[i] = node_idx[r0 + i];
      if (ra.lens) {
        const uint4 l = __ldg(ra.lens + vv[i]);
        c[i] = ChunkLen{l.x, l.y, l.z, l.w};
      } else {
        c[i] = chunk_len(g, ra, k, vv[i]);
      }
    }
    sb += c[i].bytes;
    stk += c[i].toks;
  }
  uint64_t xb, agg_b;
  uint32_t xt, agg_t;
  BS64(t64).ExclusiveSum(sb, xb, agg_b);
  BS32(t32).ExclusiveSum(stk, xt, agg_t);
  if (threadIdx.x < 32) {
    // warp 0: publish the aggregate, then look back over windows of 32 predecessors at once
    const int lane = threadIdx.x;
    uint64_t pb = 0;
    uint32_t pt = 0;
    if (tile > 0) {
      if (lane == 0) {
        st.bytes[tile] = agg_b;
        st.toks[tile] = agg_t;
        __threadfence();
        atomicExch(st.flag + tile, (epoch << 2) | 1u);  // aggregate available
      }
      for (int w = tile - 1; w >= 0; w -= 32) {
        const int p = w - lane;  // lane 0 = nearest predecessor
        uint32_t f = (epoch << 2) | 1u;
        if (p >= 0) {
          do {
            f = *reinterpret_cast<volatile uint32_t*>(st.flag + p);
          } while ((f >> 2) != epoch);
        }
        __threadfence();
        const uint32_t incl = __ballot_sync(0xffffffffu, p >= 0 && (f & 3u) == 2u);
        const int stop = incl ? __ffs(incl) - 1 : 32;  // nearest predecessor with a prefix
        uint64_t vb = 0;
        uint32_t vt = 0;
        if (p >= 0 && lane <= stop) {
          if (lane == stop) {
            vb = *reinterpret_cast<volatile uint64_t*>(st.ibytes + p);
            vt = *reinterpret_cast<volatile uint32_t*>(st.itoks + p);
          } else {
            vb = *reinterpret_cast<volatile uint64_t*>(st.bytes + p);
            vt = *reinterpret_cast<volatile uint32_t*>(st.toks + p);
          }
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
          vb += __shfl_xor_sync(0xffffffffu, vb, d);
          vt += __shfl_xor_sync(0xffffffffu, vt, d);
        }
        pb += vb;
        pt += vt;
        if (incl) break;
      }
    }
    if (lane == 0) {
      st.ibytes[tile] = pb + agg_b;
      st.itoks[tile] = pt + agg_t;
      __threadfence();
      atomicExch(st.flag + tile, (epoch << 2) | 2u);  // inclusive prefix available
      pre_b = pb;
      pre_t = pt;
    }
  }
  __syncthreads();
  uint64_t ob = pre_b + xb;
  uint32_t ot = pre_t + xt;
#pragma unroll
  for (int i = 0; i < kLenItems; ++i) {
    const int r = r0 + i;
    if (r < n_req) {
      byte_off[r] = ob;
      tok_off[r] = ot;
      sel_count[r] = static_cast<int32_t>(c[i].sel);
      vrow[r] = make_int2(vv[i], static_cast<int32_t>(c[i].row));
      if (c[i].sel >> 31) irr_list[atomicAdd(irr_count, 1)] = r;
    }
    ob += c[i].bytes;
    ot += c[i].toks;
    if (r == n_req - 1) {
      byte_off[n_req] = ob;
      tok_off[n_req] = ot;
    }
  }
  asm volatile("griddepcontrol.launch_dependents;");
}

__global__ void chunk_len_table_kernel(DevGraph g, RankedAdj ra, int k, uint4* __restrict__ out) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= g.n) return;
  const ChunkLen c = chunk_len(g, ra, k, static_cast<int32_t>(v));
  out[v] = make_uint4(static_cast<uint32_t>(c.bytes), c.toks, c.sel, c.row);
}

// ranked adjacency: sort keys w << 32 | ~u (descending == weight desc, index asc)
__global__ void rank_keys_kernel(const int32_t* __restrict__ idx, const int32_t* __restrict__ w,
                                 uint64_t e_count, uint64_t* __restrict__ keys) {
  const uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= e_count) return;
  const int32_t u = idx[e];
  keys[e] = (static_cast<uint64_t>(static_cast<uint32_t>(w[u])) << 32) |
            (0xFFFFFFFFu - static_cast<uint32_t>(u));
}

// sorted keys -> neighbour indices + per-entry values of the three prefixes (the value arrays
// have e_count + 1 slots; the last is 0 so the exclusive scans also yield the totals)
__global__ void rank_fill_kernel(DevGraph g, const uint64_t* __restrict__ sorted, uint64_t e_count,
                                 int32_t* __restrict__ ridx, uint64_t* __restrict__ vb,
                                 uint32_t* __restrict__ vt, uint32_t* __restrict__ vi) {
  const uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e > e_count) return;
  if (e == e_count) {
    vb[e] = 0;
    vt[e] = 0;
    vi[e] = 0;
    return;
  }
  const int32_t u = static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(sorted[e]));
  ridx[e] = u;
  const uint32_t st = g.ent_stat[u];
  vb[e] = (g.entry_off[u + 1] - g.entry_off[u]) + 3;
  vt[e] = piece_tokens(st);
  vi[e] = entry_regular(st) ? 0u : 1u;
}

// ---------------------------------------------------------------------------------- render+emit
// One warp per chunk: the chunk is assembled in a per-warp shared-memory buffer placed at the
// same 16-byte phase as its global destination, written out with 16-byte stores, and tokenised
// without reading the text back from HBM.  Lane s copies piece s (entry bytes as aligned 4-byte
// words, realigned to the destination by funnel shifts, ragged ends byte by byte).  Chunks longer
// than the buffer are built in place in global memory by the same code.
constexpr int kRW = 4;         // warps (chunks) per CTA of the irregular-chunk kernel
// chunks per CTA of chunk_regular (one text + one token warp each): one, so a CTA's slot frees as
// soon as its own two warps finish (one-box A/B: 155 us vs 155-157 with 4 chunks per CTA, and a
// tighter spread)
constexpr int kRegW = 1;
constexpr int kRegBlocks = 48 / (2 * kRegW);  // CTAs per SM at 40 registers (48 warps)
constexpr int kBuf = 4096;     // staged chunk bytes per warp
constexpr int kSeg = 1024;     // bytes per token-start compaction segment
constexpr int kWordsU = 2;     // 16-byte loads in flight per lane

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

// One 16-byte source word x (entry bytes [base, base + 16)) of a segment [src, end) whose byte p
// goes to dstp + p: the destination-aligned 4-byte words that lie wholly inside the entry, each a
// funnel shift of two source words (nx = the next source word), predicated stores.  The <= 3
// ragged bytes at each end of the entry are stored by the segment's own lane (build_chunk), so
// every byte has exactly one writer.
__device__ __forceinline__ void put_block(char* dstp, uint4 x, uint32_t nx, uint32_t base,
                                          uint32_t src, uint32_t end) {
  const uint32_t q = (0u - static_cast<uint32_t>(reinterpret_cast<uintptr_t>(dstp))) & 3u;
  const uint32_t w[5] = {x.x, x.y, x.z, x.w, nx};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t p0 = base + q + 4 * j;  // source position of the word's first byte
    const uint32_t v = q ? __funnelshift_r(w[j], w[j + 1], 8 * q) : w[j];
    if (p0 >= src && p0 + 4 <= end) *reinterpret_cast<uint32_t*>(dstp + p0) = v;
  }
}

// The bytes [max(lo, pad), min(lo + 16, Q)) of a staged 16-byte word: 4-byte stores where a
// quarter is whole, byte stores for the rest.
__device__ __forceinline__ void put_edge16(char* gbase, const char* sb, uint32_t lo, uint32_t pad,
                                           uint32_t Q) {
#pragma unroll
  for (uint32_t c = 0; c < 16; c += 4) {
    const uint32_t a = lo + c;
    if (a >= pad && a + 4 <= Q) {
      *reinterpret_cast<uint32_t*>(gbase + a) = *reinterpret_cast<const uint32_t*>(sb + a);
    } else if (a + 4 > pad && a < Q) {
      for (uint32_t b = max(a, pad); b < min(a + 4, Q); ++b) gbase[b] = sb[b];
    }
  }
}

// Assemble chunk bytes [0, n) at buf (shared or global): "[Node:" E_v "]\n[neighbours:"
// {(","), "(" E_j ")"} "]".  Per round of 32 segments (the centre entry + up to 31 neighbour
// pieces) the 16-byte source words of all segments are numbered by a warp scan; each lane finds
// its segment by a shuffle binary search and keeps kWordsU loads in flight before it stores.
__device__ __forceinline__ void build_chunk(const DevGraph& g, int32_t v, int k,
                                            const EntryRec* __restrict__ mine, char* buf, int lane) {
  const uint32_t ev = g.entry_off[v];
  const uint32_t ec = g.entry_off[v + 1] - ev;
  if (lane < 6) buf[lane] = "[Node:"[lane];
  if (lane < 14) buf[6 + ec + lane] = "]\n[neighbours:"[lane];
  uint32_t o = 6 + ec + 14;  // offset of the next round's first neighbour piece
  const uint4* words = reinterpret_cast<const uint4*>(g.entry_bytes);
  const uint32_t* words4 = reinterpret_cast<const uint32_t*>(g.entry_bytes);
  for (int s0 = 0; s0 <= k; s0 += 32) {
    const int s = s0 + lane;
    uint32_t src = 0, len = 0, dst = 0, plen = 0;
    if (s == 0) {
      src = ev;
      len = ec;
      dst = 6;
    } else if (s <= k) {
      const uint2 ol = __ldg(reinterpret_cast<const uint2*>(mine + (s - 1)));  // (off, len)
      src = ol.x;
      len = ol.y;
      plen = len + 2 + (s > 1 ? 1u : 0u);
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
    // the entry's ragged ends (bytes outside its destination-aligned whole words): <= 3 + 3 bytes
    if (s <= k && len) {
      const char* sp = g.entry_bytes + src;
      char* dp = buf + dst;
      const uint32_t ph = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(dp)) & 3u;
      const uint32_t head = min(len, (4u - ph) & 3u);
      const uint32_t tail = max(head, len - ((ph + len) & 3u));
      for (uint32_t i = 0; i < head; ++i) dp[i] = sp[i];
      for (uint32_t i = tail; i < len; ++i) dp[i] = sp[i];
    }
    // 16-byte source words covering [src, src + len), numbered across the round's segments
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
      uint32_t nx[kWordsU], qsrc[kWordsU], qlen[kWordsU], qdst[kWordsU], qword[kWordsU];
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
        const bool in = wi < W;
        x[t] = in ? __ldg(words + qword[t]) : make_uint4(0, 0, 0, 0);
        nx[t] = in ? __ldg(words4 + 4 * (qword[t] + 1)) : 0u;
        if (!in) qlen[t] = 0;
      }
#pragma unroll
      for (int t = 0; t < kWordsU; ++t)
        put_block(buf + qdst[t] - qsrc[t], x[t], nx[t], qword[t] << 4, qsrc[t], qsrc[t] + qlen[t]);
    }
  }
  if (lane == 0) buf[o] = ']';
  __syncwarp();
}

constexpr uint64_t kFnvBasis = 14695981039346656037ULL, kFnvPrime = 1099511628211ULL;
__host__ __device__ constexpr uint64_t fnv_lit(const char* c, uint64_t h = kFnvBasis) {
  return *c ? fnv_lit(c + 1, (h ^ static_cast<unsigned char>(*c)) * kFnvPrime) : h;
}
constexpr uint64_t kNodeState = fnv_lit("[Node:");         // first token of every chunk
constexpr uint64_t kNbrState = fnv_lit("[neighbours:(");   // first neighbour junction
constexpr uint64_t kNbrEmpty = fnv_lit("[neighbours:]");   // k = 0: the whole last token

__device__ __forceinline__ uint64_t fnv_byte(uint64_t h, unsigned char c) {
  return (h ^ c) * kFnvPrime;
}

__device__ __forceinline__ void put_token(uint32_t o, uint32_t b, uint32_t e, uint64_t h,
                                          uint32_t vocab, uint64_t vmagic, int32_t* tok_id,
                                          uint64_t* tok_begin, uint64_t* tok_end) {
  tok_begin[o] = b;
  tok_end[o] = e;
  if (vocab) tok_id[o] = static_cast<int32_t>(mod_vocab(h, vocab, vmagic));
}

// Fast tokenizer of a chunk whose pieces are all regular entries (DevGraph::ent_head != 0).  The
// chunk's tokens, in order:
//   J_0 = "[Node:" + head(E_v), interior(E_v), T_v = tail(E_v) + "]"            (centre piece 0)
//   J_s = sep + head(E_s), interior(E_s)    (neighbour piece s >= 1; sep = "[neighbours:(" for
//         s = 1, else tail(E_{s-1}) + "),(")
//   last = tail(E_k) + ")]"   (k = 0: "[neighbours:]")
// Lane s of a round computes J_s (its hash continues from E_{s-1}'s precomputed tail state over
// the separator and E_s's first-token bytes); the interior tokens are copied from the tables,
// lanes striding over the round's interior tokens.
__device__ __forceinline__ void emit_fast(const DevGraph& g, int32_t v, int k,
                                          const EntryRec* __restrict__ mine, uint32_t n, uint32_t t,
                                          uint32_t vocab, uint64_t vmagic, int32_t* tok_id,
                                          uint64_t* tok_begin, uint64_t* tok_end, int lane) {
  const uint32_t lv = g.entry_off[v + 1] - g.entry_off[v];
  uint32_t prev_dst = 0, prev_tail = 0;
  uint64_t prev_ts = 0;
  uint32_t o = 6 + lv + 14;  // byte offset of the next neighbour piece
  uint32_t tb = t;           // first token of the round
  for (int s0 = 0; s0 <= k; s0 += 32) {
    const int s = s0 + lane;
    const bool act = s <= k;
    // the piece's entry record: two 16-byte loads of one 32-byte line
    uint4 ra4 = make_uint4(0, 0, 0, 0), rb4 = make_uint4(0, 0, 0, 0);
    if (act) {
      const uint4* rp = reinterpret_cast<const uint4*>(s > 0 ? mine + (s - 1) : g.ent + v);
      ra4 = __ldg(rp);
      rb4 = __ldg(rp + 1);
    }
    const uint32_t eo = ra4.x, len = ra4.y;
    uint32_t dst = 6, plen = 0;
    if (act && s > 0) plen = len + 2 + (s > 1 ? 1u : 0u);
    uint32_t pincl = plen;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t x = __shfl_up_sync(0xffffffffu, pincl, d);
      if (lane >= d) pincl += x;
    }
    if (s > 0) dst = o + (pincl - plen) + (s > 1 ? 2u : 1u);
    o += __shfl_sync(0xffffffffu, pincl, 31);
    const uint32_t hl = ra4.z, tl = ra4.w, io = rb4.x, ni = rb4.y;
    const uint64_t ts = (static_cast<uint64_t>(rb4.w) << 32) | rb4.z;
    const uint32_t grp = act ? ni + (s == 0 ? 2u : 1u) : 0u;
    uint32_t gin = grp, iin = ni;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t x = __shfl_up_sync(0xffffffffu, gin, d);
      const uint32_t y = __shfl_up_sync(0xffffffffu, iin, d);
      if (lane >= d) {
        gin += x;
        iin += y;
      }
    }
    const uint32_t gex = gin - grp, iex = iin - ni;
    const uint32_t gtot = __shfl_sync(0xffffffffu, gin, 31);
    const uint32_t itot = __shfl_sync(0xffffffffu, iin, 31);
    uint32_t pd = __shfl_up_sync(0xffffffffu, dst, 1), pt = __shfl_up_sync(0xffffffffu, tl, 1);
    uint64_t pts = __shfl_up_sync(0xffffffffu, ts, 1);
    if (lane == 0) {
      pd = prev_dst;
      pt = prev_tail;
      pts = prev_ts;
    }
    if (act) {
      uint64_t h;
      uint32_t b;
      if (s == 0) {
        h = kNodeState;
        b = 0;
      } else if (s == 1) {
        h = kNbrState;
        b = 6 + lv + 2;
      } else {
        h = fnv_byte(fnv_byte(fnv_byte(pts, ')'), ','), '(');
        b = pd + pt;
      }
      const unsigned char* hb = reinterpret_cast<const unsigned char*>(g.entry_bytes) + eo;
      for (uint32_t q = 0; q < hl; ++q) h = fnv_byte(h, hb[q]);
      put_token(tb + gex, b, dst + hl, h, vocab, vmagic, tok_id, tok_begin, tok_end);
      if (s == 0)
        put_token(tb + gex + 1 + ni, dst + tl, dst + len + 1, fnv_byte(ts, ']'), vocab, vmagic,
                  tok_id, tok_begin, tok_end);
      if (s == k) {
        if (k == 0)
          put_token(tb + gex + grp, 6 + lv + 2, n, kNbrEmpty, vocab, vmagic, tok_id, tok_begin,
                    tok_end);
        else
          put_token(tb + gex + grp, dst + tl, n, fnv_byte(fnv_byte(ts, ')'), ']'), vocab, vmagic,
                    tok_id, tok_begin, tok_end);
      }
    }
    // interior tokens of the round's pieces, lanes striding over them (two per lane per
    // iteration: both record loads are in flight before the stores)
    for (uint32_t i0 = 0; i0 < itot; i0 += 64) {
      uint32_t jj[2], qg[2], qd[2], id[2];
      uint2 sp[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t i = i0 + 32 * h + lane;
        int q = 0;  // last piece whose first interior token is <= i
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
          const uint32_t e = __shfl_sync(0xffffffffu, iex, q + step);
          if (e <= i) q += step;
        }
        const uint32_t qiex = __shfl_sync(0xffffffffu, iex, q);
        const uint32_t qio = __shfl_sync(0xffffffffu, io, q);
        qg[h] = __shfl_sync(0xffffffffu, gex, q);
        qd[h] = __shfl_sync(0xffffffffu, dst, q);
        jj[h] = i - qiex;
        const bool in = i < itot;
        sp[h] = in ? __ldg(g.itok_span + qio + jj[h]) : make_uint2(0, 0);
        id[h] = in && vocab ? __ldg(g.itok_id + qio + jj[h]) : 0u;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t o = tb + qg[h] + 1 + jj[h];
        if (i0 + 32 * h + lane < itot) {
          tok_begin[o] = qd[h] + sp[h].x;
          tok_end[o] = qd[h] + sp[h].y;
          if (vocab) tok_id[o] = static_cast<int32_t>(id[h]);
        }
      }
    }
    tb += gtot;
    prev_dst = __shfl_sync(0xffffffffu, dst, 31);
    prev_tail = __shfl_sync(0xffffffffu, tl, 31);
    prev_ts = __shfl_sync(0xffffffffu, ts, 31);
  }
}

// Text of a regular chunk (its tokens come from emit_fast in the same CTA's token warps).
__device__ __forceinline__ void render_text(const DevGraph& g, int32_t v, int k,
                                            const EntryRec* __restrict__ mine, uint64_t goff,
                                            uint32_t n, char* __restrict__ out, char* sb, int lane) {
  if (n <= kBuf) {
    const uint32_t pad = static_cast<uint32_t>(goff & 15), Q = pad + n;
    build_chunk(g, v, k, mine, sb + pad, lane);
    char* gbase = out + (goff - pad);
    // whole 16-byte words [a16, z16) as 16-byte stores; the < 16 ragged bytes at each end as one
    // byte per lane (lanes 0-15 the head, 16-31 the tail)
    const uint32_t a16 = (pad + 15) & ~15u, z16 = Q & ~15u;
    for (uint32_t lo = a16 + 16 * lane; lo < z16; lo += 512)
      *reinterpret_cast<uint4*>(gbase + lo) = *reinterpret_cast<const uint4*>(sb + lo);
    const uint32_t b = lane < 16 ? pad + lane : max(z16, a16) + (lane - 16);
    if (lane < 16 ? b < min(a16, Q) : b < Q) gbase[b] = sb[b];
  } else {
    build_chunk(g, v, k, mine, out + goff, lane);
  }
}

// Text and tokens of an irregular chunk (the byte-level tokenizer over a whitespace mask).
__device__ __forceinline__ void render_slow(const DevGraph& g, int32_t v, int k,
                                            const EntryRec* __restrict__ mine, uint64_t goff,
                                            uint32_t n, uint32_t t, uint32_t vocab, uint64_t vmagic,
                                            char* __restrict__ out, int32_t* __restrict__ tok_id,
                                            uint64_t* __restrict__ tok_begin,
                                            uint64_t* __restrict__ tok_end, char* sbw,
                                            uint32_t* sp, int lane) {
  const bool staged = n <= kBuf;
  char* gdst = out + goff;
  // token-start list of the unstaged path (chunks > kBuf), which leaves the staging buffer free
  uint32_t* list = reinterpret_cast<uint32_t*>(sbw);
  if (staged) {
    // staged span: smem bytes [pad, Q) hold the chunk at the 16-byte phase of its destination
    char* sb = sbw;
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
          put_edge16(gbase, sb, lo, pad, Q);
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

// Irregular chunks: a small grid walks the list chunk_len_scan compacted and runs the
// byte-level path (text + tokens over a whitespace mask).  Output capacity overflow: see
// chunk_render_emit.
__global__ void __launch_bounds__(kRW * 32)
chunk_irregular_kernel(DevGraph g, RankedAdj ra, const uint64_t* __restrict__ byte_off,
                       const uint32_t* __restrict__ tok_off, const int32_t* __restrict__ sel_count,
                       uint32_t vocab, uint64_t vmagic, char* __restrict__ out,
                       int32_t* __restrict__ tok_id, uint64_t* __restrict__ tok_begin,
                       uint64_t* __restrict__ tok_end, uint64_t bytes_cap, uint64_t tok_cap,
                       int32_t* __restrict__ overflow, const int32_t* __restrict__ irr_list,
                       const int32_t* __restrict__ irr_count, const int2* __restrict__ vrow) {
  __shared__ __align__(16) char sbuf[kRW][kBuf + 16];
  __shared__ uint32_t smask[kRW][kBuf / 32 + 1];
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  const int n_items = *irr_count;
  for (int i = blockIdx.x * kRW + wi; i < n_items; i += gridDim.x * kRW) {
    const int r = irr_list[i];
    const uint64_t goff = byte_off[r], gend = byte_off[r + 1];
    if (gend > bytes_cap || tok_off[r + 1] > tok_cap) {  // the host grows the buffers and reruns
      if (lane == 0) *overflow = 1;
      continue;
    }
    const int2 vr = vrow[r];  // node, first entry of its ranked row (chunk_len_scan)
    const int k = static_cast<int>(static_cast<uint32_t>(sel_count[r]) & 0x7FFFFFFFu);
    render_slow(g, vr.x, k, ra.recs + vr.y, goff, static_cast<uint32_t>(gend - goff), tok_off[r],
                vocab, vmagic, out, tok_id, tok_begin, tok_end, sbuf[wi], smask[wi], lane);
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

__global__ void entry_interior_counts_kernel(const uint32_t* __restrict__ st, uint32_t n,
                                             uint32_t* __restrict__ cnt) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) cnt[i] = entry_regular(st[i]) ? (st[i] & 0x1FFFFFFFu) - 2 : 0u;
  if (i == n) cnt[i] = 0;
}

// one thread per entry (ingest time): spans + fnv1a hashes of the interior tokens, the first
// token's length, the last token's offset and its fnv1a state
__global__ void entry_tokens_kernel(const char* __restrict__ bytes, const uint32_t* __restrict__ off,
                                    const uint32_t* __restrict__ st, uint32_t n,
                                    const uint32_t* __restrict__ ioff, uint32_t* __restrict__ head,
                                    uint32_t* __restrict__ tail, uint64_t* __restrict__ tstate,
                                    uint2* __restrict__ itok_span, uint64_t* __restrict__ itok_hash) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (!entry_regular(st[i])) {
    head[i] = 0;
    tail[i] = 0;
    tstate[i] = 0;
    return;
  }
  const uint32_t b = off[i], e = off[i + 1], T = st[i] & 0x1FFFFFFFu;
  uint32_t tok = 0, o = ioff[i];
  uint32_t q = b;
  while (q < e) {
    while (q < e && dev_is_space(static_cast<unsigned char>(bytes[q]))) ++q;
    if (q >= e) break;
    const uint32_t t0 = q;
    uint64_t h = 14695981039346656037ULL;
    while (q < e && !dev_is_space(static_cast<unsigned char>(bytes[q]))) {
      h = (h ^ static_cast<unsigned char>(bytes[q])) * 1099511628211ULL;
      ++q;
    }
    if (tok == 0) {
      head[i] = q - b;
    } else if (tok == T - 1) {
      tail[i] = t0 - b;
      tstate[i] = h;
    } else {
      itok_span[o] = make_uint2(t0 - b, q - b);
      itok_hash[o++] = h;
    }
    ++tok;
  }
}
__global__ void entry_records_kernel(const uint32_t* __restrict__ off, const uint32_t* __restrict__ head,
                                     const uint32_t* __restrict__ tail, const uint64_t* __restrict__ tstate,
                                     const uint32_t* __restrict__ ioff, uint32_t n,
                                     EntryRec* __restrict__ rec) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  EntryRec r;
  r.off = off[i];
  r.len = off[i + 1] - r.off;
  r.head = head[i];
  r.tail = tail[i];
  r.ioff = ioff[i];
  r.ni = ioff[i + 1] - r.ioff;
  r.tstate = tstate[i];
  rec[i] = r;
}

__global__ void token_ids_kernel(const uint64_t* __restrict__ hash, uint32_t n, uint32_t vocab,
                                 uint64_t vmagic, uint32_t* __restrict__ ids) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) ids[i] = mod_vocab(hash[i], vocab, vmagic);
}

// Regular chunks, text and tokens in one launch: warp w < kRegW of a CTA renders the text of chunk
// kRegW * b + w (render_text), warp kRegW + w emits its tokens (emit_fast), so the two halves of a
// chunk run side by side on every SM.
__global__ void __launch_bounds__(2 * kRegW * 32, kRegBlocks)
chunk_regular_kernel(DevGraph g, RankedAdj ra, int n_req, const int32_t* __restrict__ sel_count,
                     const uint64_t* __restrict__ byte_off, const uint32_t* __restrict__ tok_off,
                     uint32_t vocab, uint64_t vmagic, char* __restrict__ out,
                     int32_t* __restrict__ tok_id, uint64_t* __restrict__ tok_begin,
                     uint64_t* __restrict__ tok_end, uint64_t bytes_cap, uint64_t tok_cap,
                     int32_t* __restrict__ overflow, const int2* __restrict__ vrow) {
  __shared__ __align__(16) char sbuf[kRegW][kBuf + 16];
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  const bool text = wi < kRegW;
  const int r = blockIdx.x * kRegW + (text ? wi : wi - kRegW);
  // launched as a programmatic dependent of chunk_len_scan: the CTAs are resident while the scan
  // finishes and wait here for its outputs
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (r >= n_req) return;
  const uint64_t goff = byte_off[r], gend = byte_off[r + 1];
  if (gend > bytes_cap || tok_off[r + 1] > tok_cap) {  // the host grows the buffers and reruns
    if (lane == 0) *overflow = 1;
    return;
  }
  const uint32_t kr = static_cast<uint32_t>(sel_count[r]);
  if (kr >> 31) return;  // irregular: chunk_irregular_kernel
  const int2 vr = vrow[r];
  const int k = static_cast<int>(kr);
  const uint32_t n = static_cast<uint32_t>(gend - goff);
  if (text)
    render_text(g, vr.x, k, ra.recs + vr.y, goff, n, out, sbuf[wi], lane);
  else
    emit_fast(g, vr.x, k, ra.recs + vr.y, n, tok_off[r], vocab, vmagic, tok_id, tok_begin, tok_end,
              lane);
}

// the ranked neighbours' entry records, in rank order (the chunk kernels read a row's pieces as
// one contiguous run instead of idx -> ent gathers)
__global__ void rank_recs_kernel(DevGraph g, const int32_t* __restrict__ ridx, uint64_t e_count,
                                 EntryRec* __restrict__ recs) {
  const uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e < e_count) recs[e] = g.ent[ridx[e]];
}

}  // namespace

void entry_records(const uint32_t* off, const uint32_t* head, const uint32_t* tail,
                   const uint64_t* tstate, const uint32_t* ioff, uint32_t n, EntryRec* rec,
                   cudaStream_t s) {
  if (n == 0) return;
  entry_records_kernel<<<static_cast<int>(ceil_div(n, 256)), 256, 0, s>>>(off, head, tail, tstate,
                                                                          ioff, n, rec);
  GLMX_CHECK_LAUNCH();
}

void chunk_token_ids(const uint64_t* hash, uint32_t n, uint32_t vocab, uint32_t* ids,
                     cudaStream_t s) {
  if (n == 0 || vocab == 0) return;
  token_ids_kernel<<<static_cast<int>(ceil_div(n, 256)), 256, 0, s>>>(hash, n, vocab,
                                                                      ~uint64_t(0) / vocab, ids);
  GLMX_CHECK_LAUNCH();
}

void chunk_len_table(const DevGraph& g, const RankedAdj& ra, int k, uint4* out, cudaStream_t s) {
  if (g.n == 0) return;
  RankedAdj r = ra;
  r.lens = nullptr;
  chunk_len_table_kernel<<<static_cast<int>(ceil_div(g.n, 256)), 256, 0, s>>>(g, r, k, out);
  GLMX_CHECK_LAUNCH();
}

int chunk_scan_tiles(int n_req) { return static_cast<int>(ceil_div(n_req, kLenTile)); }

void chunk_lengths_scan(const DevGraph& g, const RankedAdj& ra, int k, const int32_t* node_idx,
                        int n_req, int32_t* sel_count, uint64_t* byte_off, uint32_t* tok_off,
                        const ScanState& st, uint32_t epoch, int32_t* irr_list, int32_t* irr_count,
                        int2* vrow, cudaStream_t s) {
  chunk_len_scan_kernel<<<chunk_scan_tiles(n_req), kLenThreads, 0, s>>>(
      g, ra, k, node_idx, n_req, sel_count, byte_off, tok_off, st, epoch, irr_list, irr_count, vrow);
  GLMX_CHECK_LAUNCH();
}

void chunk_render_emit(const DevGraph& g, const RankedAdj& ra, const int32_t* node_idx, int n_req,
                       const int32_t* sel_count, const uint64_t* byte_off, const uint32_t* tok_off,
                       uint32_t vocab, char* out, int32_t* tok_id, uint64_t* tok_begin,
                       uint64_t* tok_end, uint64_t bytes_cap, uint64_t tok_cap, int32_t* overflow,
                       const int32_t* irr_list, const int32_t* irr_count, const int2* vrow,
                       cudaStream_t s) {
  const uint64_t vmagic = vocab ? ~uint64_t(0) / vocab : 0;
  // programmatic dependent launch: the regular-chunk CTAs start while the length+scan kernel
  // drains (griddepcontrol.wait in the kernel orders them after its writes)
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(static_cast<unsigned>(ceil_div(n_req, kRegW)));
  lc.blockDim = dim3(2 * kRegW * 32);
  lc.dynamicSmemBytes = 0;
  lc.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  GLMX_CUDA(cudaLaunchKernelEx(&lc, chunk_regular_kernel, g, ra, n_req, sel_count, byte_off,
                               tok_off, vocab, vmagic, out, tok_id, tok_begin, tok_end, bytes_cap,
                               tok_cap, overflow, vrow));
  GLMX_CHECK_LAUNCH();
  if (!irr_list) return;  // the graph has no irregular entries, so no irregular chunks
  chunk_irregular_kernel<<<2 * kNumSMs, kRW * 32, 0, s>>>(
      g, ra, byte_off, tok_off, sel_count, vocab, vmagic, out, tok_id, tok_begin, tok_end,
      bytes_cap, tok_cap, overflow, irr_list, irr_count, vrow);
  GLMX_CHECK_LAUNCH();
}

size_t rank_sort_temp_bytes(uint64_t e_count, uint32_t n) {
  size_t t = 0;
  cub::DeviceSegmentedSort::SortKeysDescending(nullptr, t, static_cast<const uint64_t*>(nullptr),
                                               static_cast<uint64_t*>(nullptr),
                                               static_cast<int64_t>(e_count), static_cast<int64_t>(n),
                                               static_cast<const uint32_t*>(nullptr),
                                               static_cast<const uint32_t*>(nullptr));
  size_t t1 = 0, t2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t1, static_cast<uint64_t*>(nullptr),
                                static_cast<uint64_t*>(nullptr), static_cast<int64_t>(e_count + 1));
  cub::DeviceScan::ExclusiveSum(nullptr, t2, static_cast<uint32_t*>(nullptr),
                                static_cast<uint32_t*>(nullptr), static_cast<int64_t>(e_count + 1));
  return std::max(t, std::max(t1, t2));
}

void rank_adjacency(const DevGraph& g, const uint32_t* off, const int32_t* idx, const int32_t* w,
                    uint64_t e_count, uint32_t n, void* temp, size_t temp_bytes, uint64_t* keys,
                    uint64_t* sorted, int32_t* ridx, uint64_t* pbytes, uint32_t* ptoks,
                    uint32_t* pirr, uint32_t* tmp32, EntryRec* recs, cudaStream_t s) {
  if (e_count) {
    rank_keys_kernel<<<static_cast<int>(ceil_div(e_count, 256)), 256, 0, s>>>(idx, w, e_count, keys);
    GLMX_CHECK_LAUNCH();
    GLMX_CUDA(cub::DeviceSegmentedSort::SortKeysDescending(
        temp, temp_bytes, keys, sorted, static_cast<int64_t>(e_count), static_cast<int64_t>(n),
        off, off + 1, s));
  }
  // values into keys (bytes, u64) / tmp32 (tokens) / pirr's own slot via ptoks scratch
  rank_fill_kernel<<<static_cast<int>(ceil_div(e_count + 1, 256)), 256, 0, s>>>(
      g, sorted, e_count, ridx, keys, tmp32, pirr);
  GLMX_CHECK_LAUNCH();
  GLMX_CUDA(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, keys, pbytes,
                                          static_cast<int64_t>(e_count + 1), s));
  GLMX_CUDA(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, tmp32, ptoks,
                                          static_cast<int64_t>(e_count + 1), s));
  // irregular flags -> prefix, through tmp32 as the scan output (then copied back)
  GLMX_CUDA(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, pirr, tmp32,
                                          static_cast<int64_t>(e_count + 1), s));
  GLMX_CUDA(cudaMemcpyAsync(pirr, tmp32, (e_count + 1) * 4, cudaMemcpyDeviceToDevice, s));
  if (e_count) {
    rank_recs_kernel<<<static_cast<int>(ceil_div(e_count, 256)), 256, 0, s>>>(g, ridx, e_count, recs);
    GLMX_CHECK_LAUNCH();
  }
}

void entry_stats(const char* bytes, const uint32_t* off, uint32_t n, uint32_t* st, cudaStream_t s) {
  if (n == 0) return;
  entry_stats_kernel<<<static_cast<int>(ceil_div(n, 256)), 256, 0, s>>>(bytes, off, n, st);
  GLMX_CHECK_LAUNCH();
}

void entry_interior_counts(const uint32_t* st, uint32_t n, uint32_t* cnt, cudaStream_t s) {
  entry_interior_counts_kernel<<<static_cast<int>(ceil_div(n + 1, 256)), 256, 0, s>>>(st, n, cnt);
  GLMX_CHECK_LAUNCH();
}

void entry_tokens(const char* bytes, const uint32_t* off, const uint32_t* st, uint32_t n,
                  const uint32_t* ioff, uint32_t* head, uint32_t* tail, uint64_t* tstate,
                  uint2* itok_span, uint64_t* itok_hash, cudaStream_t s) {
  if (n == 0) return;
  entry_tokens_kernel<<<static_cast<int>(ceil_div(n, 128)), 128, 0, s>>>(bytes, off, st, n, ioff,
                                                                        head, tail, tstate, itok_span,
                                                                        itok_hash);
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
