// K3 — paged causal GQA prefill attention on 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// Persistent kernel: one CTA per SM walks a static slice of the work items (request, 64-token
// query block, kv head), sorted longest-first on the host.  An item holds TWO 128-row query tiles
// (Q0 = tokens [t0, t0+32) x the G=4 query heads of one kv head, Q1 = the next 32 tokens), so
// every K/V page is fetched once per GQA group and used for 256 query rows: per 128-key tile the
// CTA moves 64 KB from L2 for 8.4 MFLOP of tensor work (half the single-tile design's L2 load,
// which at 148 SMs exceeded the chip's L2 throughput).
//   warps 0-3  softmax WG0: thread i owns row i of Q0 == TMEM lane i (S0 / P0 / O0)
//   warps 4-7  softmax WG1: same for Q1 (S1 / P1 / O1)
//   warp 8     TMA producer: K_0, Q0+Q1, V_0, K_1, V_1, ... through a 4-slot ring of 32 KB
//              [128 keys][128 dims] SW128 tiles (16 page boxes per tile; pages past the context
//              are out of bounds -> zero fill), in exactly the order the MMA warp consumes them
//   warp 9     MMA issuer (one thread), per key tile j:
//                PV0(j-1) S0(j) PV1(j-1) S1(j)  ... i.e. S_i(j+1) is issued right behind PV_i(j),
//              so while WG0 runs the softmax of tile j the tensor pipe executes PV1(j-1), S1(j),
//              and vice versa (ping-pong of the two query tiles)
// TMEM (512 cols): S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512).  P_i (bf16) overwrites the
// first 64 columns of S_i and is the TMEM A operand of PV_i.  Online softmax in base 2 with a
// lazily updated reference max (O rescaled only when a row max grows by > 2^8, decided
// warp-uniformly because tcgen05.ld/st are .sync.aligned); 1/l normalisation in the epilogue.
// Every mbarrier wait is bounded (%globaltimer): a protocol error prints its location and traps.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cfloat>

#include "attn.cuh"
#include "common.cuh"
#include "tc_ptx.cuh"

namespace glmx {

namespace {

constexpr int kHD = 128;
constexpr int kB = 16;
constexpr int kM = 128;       // query rows per tile (TMEM lanes)
constexpr int kQT = 2;        // query tiles per item
constexpr int kN = 128;       // keys per tile
constexpr int kHalf = 16384;  // bytes of one [128][64] bf16 SW128 half tile
constexpr int kTile = 2 * kHalf;
constexpr int kKSlots = 3;    // K ring depth (32 KB [128 keys][128 dims] tiles)
constexpr int kVSlots = 2;    // V ring depth
constexpr int kSoftmaxThreads = 128 * kQT;
constexpr int kThreads = kSoftmaxThreads + 96;  // + K producer, MMA, V producer warps
// registers: up to 3 warps per SM sub-partition (16K regs each) -> <= 168 per thread
// smem map (1024-aligned): Q0 Q1 | K ring | V ring | barriers
constexpr int kOffQ = 0;
constexpr int kOffK = kOffQ + kQT * kTile;
constexpr int kOffV = kOffK + kKSlots * kTile;
constexpr int kOffBar = kOffV + kVSlots * kTile;
constexpr int kSmem = kOffBar + 256 + 1024;  // + alignment slack
static_assert(kSmem <= 232448, "shared memory budget");

using namespace tcx;  // PTX wrappers (kernels/tc_ptx.cuh)

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// kind::f16 instruction descriptor: D f32, A/B bf16, M=128.
__host__ __device__ constexpr uint32_t idesc_bf16(int n, bool b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (b_mn_major ? (1u << 16) : 0u) |
         (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(kM >> 4) << 24);
}
// byte offset of 16-byte chunk c16 (0..15 over 128 elements) of row r in a two-half SW128 tile
__device__ __forceinline__ uint32_t sw128(int r, int c16) {
  return static_cast<uint32_t>((c16 >> 3) * kHalf + r * 128 + (((c16 & 7) ^ (r & 7)) << 4));
}

// Debug trace (build with -DGLMX_ATTN_TRACE, `make trace` -> libglmx_trace.so): CTA 0 records
// clock64 stamps of the pipeline events per key tile into a global buffer (kTraceEv x kTraceN).
#ifdef GLMX_ATTN_TRACE
__device__ long long g_attn_trace[16 * 1024];
void* g_attn_trace_ptr() {
  void* p = nullptr;
  cudaGetSymbolAddress(&p, g_attn_trace);
  return p;
}
#define ATTN_TRACE(ev, j)                                                       \
  do {                                                                          \
    if (blockIdx.x == 0 && (j) < 1024) g_attn_trace[(ev) * 1024 + (j)] = clock64(); \
  } while (0)
// CTA-level stamps of CTA 0 (kernel entry, setup done, teardown) in the last slots of event 15
#define ATTN_TRACE_CTA(k)                                                          \
  do {                                                                             \
    if (blockIdx.x == 0 && threadIdx.x == 0) g_attn_trace[15 * 1024 + 1023 - (k)] = clock64(); \
  } while (0)
#else
#define ATTN_TRACE_CTA(k) \
  do {                    \
  } while (0)
#define ATTN_TRACE(ev, j) \
  do {                    \
  } while (0)
#endif

struct TcParams {
  AttnParams a;
  uint32_t rows_total;  // rows of the pool tensor map (OOB row -> zero fill)
  const int4* pieces;   // AttnPiece {item, j0, j1, part} (host/attn_sched.hpp)
  const int* cta_off;   // pieces of CTA c: [cta_off[c], cta_off[c+1])
  float* part_o;        // [part][256 rows][128] unnormalised O of split items
  float2* part_ml;      // [part][256 rows] (reference max, row sum)
  const int4* partners; // per piece: the paired single-tile item for warpgroup 1 (x = -1: none)
};

struct Item {
  int req, tok0, kvh, qlen, ctx, qs, n_kt;
  int nqt;  // query tiles in use: 1 when the item's block holds <= 128/G tokens
};

__device__ __forceinline__ Item item_of(const AttnParams& p, int w) {
  Item it;
  const int2 wk = p.work[w / p.Hkv];
  it.req = wk.x;
  it.tok0 = wk.y;
  it.kvh = w % p.Hkv;
  it.qlen = p.q_len[it.req];
  it.ctx = p.ctx_len[it.req];
  it.qs = p.q_start[it.req];
  const int G = p.H / p.Hkv;
  const int max_pos = it.ctx - it.qlen + min(it.tok0 + kQT * kM / G, it.qlen) - 1;
  it.n_kt = max_pos / kN + 1;
  it.nqt = it.qlen - it.tok0 > kM / G ? 2 : 1;
  return it;
}

__global__ void __launch_bounds__(kThreads, 1)
paged_attn_tc_kernel(const __grid_constant__ CUtensorMap kv_map,
                     const __grid_constant__ CUtensorMap q_map, TcParams tp) {
  const AttnParams& p = tp.a;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_addr(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  // barriers (8 B each): kfull[kKSlots] kempty[kKSlots] vfull[kVSlots] vempty[kVSlots]
  //                      sfull[2] pfull[2] ofull[2] qfull qempty
  constexpr int kB0 = 2 * (kKSlots + kVSlots);
  const uint32_t b_kfull = smem_addr(bars + 0), b_kempty = smem_addr(bars + kKSlots);
  const uint32_t b_vfull = smem_addr(bars + 2 * kKSlots), b_vempty = smem_addr(bars + 2 * kKSlots + kVSlots);
  const uint32_t b_sfull = smem_addr(bars + kB0), b_pfull = smem_addr(bars + kB0 + 2);
  const uint32_t b_ofull = smem_addr(bars + kB0 + 4);
  const uint32_t b_qfull = smem_addr(bars + kB0 + 6), b_qempty = smem_addr(bars + kB0 + 7);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + kB0 + 8);

  ATTN_TRACE_CTA(0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = p.H / p.Hkv;
  constexpr int kWarpProducer = kSoftmaxThreads / 32, kWarpMma = kWarpProducer + 1;
  constexpr int kWarpVProducer = kWarpMma + 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kKSlots; ++s) {
      mbar_init(b_kfull + 8 * s, 1);
      mbar_init(b_kempty + 8 * s, 1);
    }
    for (int s = 0; s < kVSlots; ++s) {
      mbar_init(b_vfull + 8 * s, 1);
      mbar_init(b_vempty + 8 * s, 1);
    }
    for (int i = 0; i < kQT; ++i) {
      mbar_init(b_sfull + 8 * i, 1);
      mbar_init(b_pfull + 8 * i, 128);
      mbar_init(b_ofull + 8 * i, 1);
    }
    mbar_init(b_qfull, 1);
    mbar_init(b_qempty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kWarpMma) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_addr(tmem_holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // barriers and TMEM are set up while the K2 append before us drains (programmatic dependent
  // launch); nothing global is read before this point
  pdl_wait();
  const uint32_t tmem = *tmem_holder;
  const uint32_t t_s0 = tmem, t_o0 = tmem + kQT * kN;
  ATTN_TRACE_CTA(1);

  if (warp == kWarpProducer || warp == kWarpVProducer) {
    // ---------------------------------------------------------------- TMA producers
    // warp 8 loads Q and the K tiles through the K ring, warp 10 the V tiles through the V ring:
    // a V slot still in use never holds back the next K load (and vice versa)
    if (lane == 0) {
      const int kv = warp == kWarpVProducer ? 1 : 0;
      const uint32_t L = p.pool.n_layers, Hkv = p.pool.n_kv_heads;
      const int n_slots = kv ? kVSlots : kKSlots;
      const uint32_t ring = sbase + (kv ? kOffV : kOffK);
      const uint32_t b_full = kv ? b_vfull : b_kfull, b_empty = kv ? b_vempty : b_kempty;
      int c = 0, it_local = 0;
      // one ring load of key tile j (global tile count c), whose 8 pages are pg[0..7]
      auto load_tile = [&](const Item& it, const int32_t* pg, int j) {
        const int slot = c % n_slots;
        const uint32_t use = static_cast<uint32_t>(c / n_slots);
        if (use > 0) mbar_wait(b_empty + 8 * slot, (use - 1) & 1, 2 + kv);
        const uint32_t full = b_full + 8 * slot;
        ATTN_TRACE(14 + kv, c);
        mbar_expect_tx(full, kTile);
        const uint32_t dst = ring + slot * kTile;
#pragma unroll
        for (int q = 0; q < kN / kB; ++q) {
          const int key0 = j * kN + q * kB;
          uint32_t row = tp.rows_total;  // out of bounds -> zeros
          if (key0 < it.ctx) row = (((static_cast<uint32_t>(pg[q]) * L + p.layer) * 2 + kv) * Hkv + it.kvh) * kB;
          for (int hf = 0; hf < 2; ++hf)
            tma_load_2d(dst + hf * kHalf + q * kB * 128, &kv_map, hf * 64, static_cast<int>(row), full);
        }
        ++c;
      };
      // the 8 block-table entries of key tile j: two 16-byte loads (rows are padded to a
      // multiple of 8 entries), issued one tile ahead so their latency hides behind the previous
      // tile's slot wait and TMA issue
      auto fetch = [&](const int32_t* bt, int j, int32_t* pg) {
        const int4 x = reinterpret_cast<const int4*>(bt + j * 8)[0];
        const int4 y = reinterpret_cast<const int4*>(bt + j * 8)[1];
        pg[0] = x.x; pg[1] = x.y; pg[2] = x.z; pg[3] = x.w;
        pg[4] = y.x; pg[5] = y.y; pg[6] = y.z; pg[7] = y.w;
      };
      for (int pc = tp.cta_off[blockIdx.x]; pc < tp.cta_off[blockIdx.x + 1]; ++pc, ++it_local) {
        const int4 pz = tp.pieces[pc];
        const Item it = item_of(p, pz.x);
        const int32_t* bt = p.block_table + static_cast<int64_t>(it.req) * p.bt_stride;
        const int4 pb = tp.partners ? tp.partners[pc] : make_int4(-1, 0, 0, -1);
        if (pb.x >= 0) {
          // paired single-tile items A (warpgroup 0) and B (warpgroup 1): their key tiles are
          // interleaved A(0) B(0) A(1) B(1) ..., the shorter one dropping out when it ends
          const Item ib = item_of(p, pb.x);
          const int32_t* btb = p.block_table + static_cast<int64_t>(ib.req) * p.bt_stride;
          const int na = pz.z - pz.y, nb = pb.z - pb.y;
          int32_t ca[8], cb[8], xa[8], xb[8];
          fetch(bt, pz.y, ca);
          fetch(btb, pb.y, cb);
          for (int j = 0; j < max(na, nb); ++j) {
            if (j + 1 < na) fetch(bt, pz.y + j + 1, xa);
            if (j + 1 < nb) fetch(btb, pb.y + j + 1, xb);
            if (j < na) load_tile(it, ca, pz.y + j);
            if (kv == 0 && j == 0) {
              if (it_local > 0) mbar_wait(b_qempty, (it_local - 1) & 1, 1);
              mbar_expect_tx(b_qfull, 2 * kTile);
              for (int hf = 0; hf < 2; ++hf) {
                tma_load_3d(sbase + kOffQ + hf * kHalf, &q_map, hf * 64, it.kvh * G, it.qs + it.tok0, b_qfull);
                tma_load_3d(sbase + kOffQ + kTile + hf * kHalf, &q_map, hf * 64, ib.kvh * G,
                            ib.qs + ib.tok0, b_qfull);
              }
            }
            if (j < nb) load_tile(ib, cb, pb.y + j);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              ca[q] = xa[q];
              cb[q] = xb[q];
            }
          }
          continue;
        }
        int32_t cur[8], nxt[8];
        fetch(bt, pz.y, cur);
        for (int j = pz.y; j < pz.z; ++j) {
          if (j + 1 < pz.z) fetch(bt, j + 1, nxt);
          load_tile(it, cur, j);
          if (kv == 0 && j == pz.y) {
            if (it_local > 0) mbar_wait(b_qempty, (it_local - 1) & 1, 1);  // prev piece's last S done
            mbar_expect_tx(b_qfull, it.nqt * kTile);
            for (int i = 0; i < it.nqt; ++i)
              for (int hf = 0; hf < 2; ++hf)
                tma_load_3d(sbase + kOffQ + i * kTile + hf * kHalf, &q_map, hf * 64, it.kvh * G,
                            it.qs + it.tok0 + i * (kM / G), b_qfull);
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) cur[q] = nxt[q];
        }
      }
    }
    __syncwarp();  // reconverge before the CTA barrier (bar.sync is .aligned)
  } else if (warp == kWarpMma) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idS = idesc_bf16(kN, false), idO = idesc_bf16(kHD, true);
      int g = 0, it_local = 0;
      // S_i = Q_i K_g^T into S buffer i
      auto issue_s = [&](int i, int gk) {
        const uint32_t q_addr = sbase + kOffQ + i * kTile;
        const uint32_t k_addr = sbase + kOffK + (gk % kKSlots) * kTile;
#pragma unroll
        for (int ks = 0; ks < kHD / 16; ++ks) {
          const uint64_t a = smem_desc(q_addr + (ks >> 2) * kHalf + (ks & 3) * 32, 1, 64);
          const uint64_t b = smem_desc(k_addr + (ks >> 2) * kHalf + (ks & 3) * 32, 1, 64);
          tc_mma(t_s0 + i * kN, a, b, idS, ks > 0 ? 1u : 0u);
        }
        tc_commit(b_sfull + 8 * i);
      };
      // O_i += P_i V_g (P from the first 64 TMEM columns of S_i, V MN-major)
      auto issue_pv = [&](int i, int gv, bool first) {
        const uint32_t v_addr = sbase + kOffV + (gv % kVSlots) * kTile;
#pragma unroll
        for (int ks = 0; ks < kN / 16; ++ks) {
          const uint64_t b = smem_desc(v_addr + ks * 2048, kHalf >> 4, 64);
          tc_mma_ts(t_o0 + i * kHD, t_s0 + i * kN + ks * 8, b, idO, (!first || ks > 0) ? 1u : 0u);
        }
      };
      auto wait_k = [&](int gk, int tag) {
        mbar_wait(b_kfull + 8 * (gk % kKSlots), (gk / kKSlots) & 1, tag);
        tc_fence_after();
      };
      auto wait_v = [&](int gv, int tag) {
        mbar_wait(b_vfull + 8 * (gv % kVSlots), (gv / kVSlots) & 1, tag);
        tc_fence_after();
      };
      int c0 = 0, c1 = 0;  // tiles consumed by softmax warpgroup 0 / 1 (pfull phases)
      for (int pc = tp.cta_off[blockIdx.x]; pc < tp.cta_off[blockIdx.x + 1]; ++pc, ++it_local) {
        const int4 pz = tp.pieces[pc];
        const int4 pb = tp.partners ? tp.partners[pc] : make_int4(-1, 0, 0, -1);
        if (pb.x >= 0) {
          // paired items: side 0 = A on S0/O0 (K/V loads gA(j)), side 1 = B on S1/O1 (gB(j));
          // the producers interleave A(j) B(j), so with n_x = tiles of side x
          //   gA(j) = g + min(j, na) + min(j, nb),  gB(j) = gA(j) + (j < na)
          const int na = pz.z - pz.y, nb = pb.z - pb.y, n = max(na, nb);
          auto ga = [&](int j) { return g + min(j, na) + min(j, nb); };
          auto gb = [&](int j) { return g + min(j, na) + min(j, nb) + (j < na ? 1 : 0); };
          mbar_wait(b_qfull, it_local & 1, 12);
          wait_k(ga(0), 13);
          issue_s(0, ga(0));
          tc_commit(b_kempty + 8 * (ga(0) % kKSlots));
          wait_k(gb(0), 13);
          issue_s(1, gb(0));
          tc_commit(b_kempty + 8 * (gb(0) % kKSlots));
          if (n == 1) tc_commit(b_qempty);
          for (int j = 0; j < n; ++j) {
            if (j < na) {
              mbar_wait(b_pfull, c0 & 1, 10);
              ++c0;
              wait_v(ga(j), 11);
              issue_pv(0, ga(j), j == 0);
              tc_commit(b_vempty + 8 * (ga(j) % kVSlots));
              if (j == na - 1) tc_commit(b_ofull);
              if (j + 1 < na) {
                wait_k(ga(j + 1), 13);
                issue_s(0, ga(j + 1));
                tc_commit(b_kempty + 8 * (ga(j + 1) % kKSlots));
              }
            }
            if (j < nb) {
              mbar_wait(b_pfull + 8, c1 & 1, 15);
              ++c1;
              wait_v(gb(j), 11);
              issue_pv(1, gb(j), j == 0);
              tc_commit(b_vempty + 8 * (gb(j) % kVSlots));
              if (j == nb - 1) tc_commit(b_ofull + 8);
              if (j + 1 < nb) {
                wait_k(gb(j + 1), 13);
                issue_s(1, gb(j + 1));
                tc_commit(b_kempty + 8 * (gb(j + 1) % kKSlots));
              }
            }
            if (j + 2 == n) tc_commit(b_qempty);  // the last S of the pair was issued above
          }
          g += na + nb;
          continue;
        }
        const int n = pz.z - pz.y;
        const bool two = item_of(p, pz.x).nqt == 2;  // single-tile items leave WG1 out
        const int g0 = g;  // global tile count of this piece's first key tile
        wait_k(g0, 13);
        mbar_wait(b_qfull, it_local & 1, 12);
        tc_fence_after();
        issue_s(0, g0);
        if (two) issue_s(1, g0);
        tc_commit(b_kempty + 8 * (g0 % kKSlots));
        if (n == 1) tc_commit(b_qempty);
        for (int j = 0; j < n; ++j, ++g) {
          // ---- query tile 0: PV0(j), then S0(j+1) behind it (P0 is consumed in order)
          ATTN_TRACE(0, g);
          mbar_wait(b_pfull, c0 & 1, 10);
          ++c0;
          ATTN_TRACE(1, g);
          wait_v(g, 11);
          ATTN_TRACE(11, g);
          issue_pv(0, g, j == 0);
          if (j == n - 1) tc_commit(b_ofull);
          if (j + 1 < n) {
            ATTN_TRACE(12, g);
            wait_k(g + 1, 13);
            ATTN_TRACE(13, g);
            issue_s(0, g + 1);
          }
          ATTN_TRACE(2, g);
          // ---- query tile 1
          if (two) {
            mbar_wait(b_pfull + 8, c1 & 1, 15);
            ++c1;
            ATTN_TRACE(3, g);
            tc_fence_after();
            issue_pv(1, g, j == 0);
          }
          tc_commit(b_vempty + 8 * (g % kVSlots));
          if (two && j == n - 1) tc_commit(b_ofull + 8);
          if (j + 1 < n) {
            if (two) issue_s(1, g + 1);
            tc_commit(b_kempty + 8 * ((g + 1) % kKSlots));
            ATTN_TRACE(4, g);
            if (j + 2 == n) tc_commit(b_qempty);
          }
        }
      }
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- softmax warpgroups
    const int qt = warp >> 2;                  // query tile of this warpgroup
    const int r = threadIdx.x & 127;           // row == TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t ts = t_s0 + qt * kN + lane_off;
    const uint32_t t_o = t_o0 + qt * kHD + lane_off;
    const uint32_t b_s = b_sfull + 8 * qt, b_p = b_pfull + 8 * qt, b_o = b_ofull + 8 * qt;
    const float scale = p.scale_log2;
    uint32_t v[kN];
    int g = 0, it_local = 0;
    for (int pc = tp.cta_off[blockIdx.x]; pc < tp.cta_off[blockIdx.x + 1]; ++pc) {
      int4 pz = tp.pieces[pc];
      int qi = qt;  // query tile of the item this warpgroup works on
      if (qt == 1 && tp.partners) {
        const int4 pb = tp.partners[pc];
        if (pb.x >= 0) {  // paired piece: warpgroup 1 runs the partner's (single) query tile
          pz = pb;
          qi = 0;
        }
      }
      const Item it = item_of(p, pz.x);
      if (qi >= it.nqt) continue;  // single-tile item: this warpgroup has no rows in it
      const int t_row = it.tok0 + qi * (kM / G) + r / G;  // query token of this row
      const int tq = min(t_row, it.qlen - 1);
      const int pos = it.ctx - it.qlen + tq;
      const int pos_lo = it.ctx - it.qlen + it.tok0 + qi * (kM / G);  // smallest in the tile
      float m_used = -INFINITY, l = 0.f;
      for (int j = pz.y; j < pz.z; ++j, ++g) {
        if ((threadIdx.x & 127) == 0) ATTN_TRACE(5 + 3 * qt, g);
        mbar_wait(b_s, g & 1, 20 + qt);
        if ((threadIdx.x & 127) == 0) ATTN_TRACE(6 + 3 * qt, g);
        tc_fence_after();
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) TC_LD32(ts + cc * 32, (v + cc * 32));
        tc_wait_ld();
        const int kbase = j * kN;
        // row max of the raw scores (scale > 0 commutes with max); 8 independent chains
        float mx8[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) mx8[a] = -INFINITY;
        if (kbase + kN - 1 <= pos_lo) {  // tile fully visible to every row of the tile
#pragma unroll
          for (int i = 0; i < kN; ++i) mx8[i & 7] = fmaxf(mx8[i & 7], __uint_as_float(v[i]));
        } else {
#pragma unroll
          for (int i = 0; i < kN; ++i) {
            if (kbase + i > pos) v[i] = __float_as_uint(-INFINITY);
            mx8[i & 7] = fmaxf(mx8[i & 7], __uint_as_float(v[i]));
          }
        }
        const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                               fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * scale;
        const bool grow = mx > m_used + 8.f;
        const bool any_grow = __any_sync(0xffffffffu, grow);
        float alpha = 1.f;
        if (grow) {
          alpha = ex2(m_used - mx);
          m_used = mx;
        }
        // P = 2^(s*scale - m_used) as bf16 pairs into the first 64 columns of S_i (the S values
        // are already in registers); masked keys are -inf -> 0.  The first 32 packed columns
        // are stored while the second half is computed.  (Packed fp32x2 FFMA2/FADD2 and a
        // polynomial exp2 for a quarter of the pairs were measured slower here: the softmax
        // phase went from ~1650 to ~2000 cycles per tile, scripts/attn_trace.py.)
        // a row with no visible key so far (a split piece that starts past its position) keeps
        // m_used = -inf: use 0 so 2^(-inf - m) is 0, not 2^(-inf + inf) = NaN
        const float neg_m = m_used == -INFINITY ? 0.f : -m_used;
        float ls[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < kN; i += 2) {
          const float p0 = ex2(fmaf(__uint_as_float(v[i]), scale, neg_m));
          const float p1 = ex2(fmaf(__uint_as_float(v[i + 1]), scale, neg_m));
          ls[(i >> 1) & 3] += p0 + p1;
          __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
          v[i >> 1] = *reinterpret_cast<uint32_t*>(&b2);
          if (i == kN / 2 - 2) TC_ST32(ts, v);
        }
        l = l * alpha + ((ls[0] + ls[1]) + (ls[2] + ls[3]));
        TC_ST32(ts + 32, (v + 32));
        // O_i holds PV_i(0..j-1), all complete (S_i(j), which we waited for, was committed
        // after PV_i(j-1)); PV_i(j) is not issued before our pfull arrival.
        if (any_grow && j > pz.y) {
#pragma unroll 1
          for (int cc = 0; cc < 4; ++cc) {
            uint32_t o[32];
            TC_LD32(t_o + cc * 32, o);
            tc_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            TC_ST32(t_o + cc * 32, o);
          }
        }
        tc_wait_st();
        tc_fence_before();
        if ((threadIdx.x & 127) == 0) ATTN_TRACE(7 + 3 * qt, g);
        mbar_arrive(b_p);
      }
      // epilogue of this item: wait for its last PV_i (one ofull phase per item)
      mbar_wait(b_o, it_local & 1, 22 + qt);
      tc_fence_after();
      if (pz.w >= 0) {
        // split item: unnormalised O + (reference max, row sum) for the combine pass
        const int64_t prow = static_cast<int64_t>(pz.w) * (kQT * kM) + qi * kM + r;
        float4* dst = reinterpret_cast<float4*>(tp.part_o + prow * kHD);
        for (int cc = 0; cc < 4; ++cc) {
          uint32_t o[32];
          TC_LD32(t_o + cc * 32, o);
          tc_wait_ld();
          if (t_row < it.qlen) {
#pragma unroll
            for (int q4 = 0; q4 < 8; ++q4)
              dst[cc * 8 + q4] = make_float4(__uint_as_float(o[4 * q4]), __uint_as_float(o[4 * q4 + 1]),
                                             __uint_as_float(o[4 * q4 + 2]), __uint_as_float(o[4 * q4 + 3]));
          }
        }
        if (t_row < it.qlen) tp.part_ml[prow] = make_float2(m_used, l);
      } else {
        const float inv = 1.f / l;
        __nv_bfloat16* dst = p.o + (static_cast<int64_t>(it.qs + tq) * p.H + it.kvh * G + r % G) * kHD;
        for (int cc = 0; cc < 4; ++cc) {
          uint32_t o[32];
          TC_LD32(t_o + cc * 32, o);
          tc_wait_ld();
          if (t_row < it.qlen) {
            uint4* d4 = reinterpret_cast<uint4*>(dst + cc * 32);
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              uint32_t pk[4];
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const int i = q4 * 8 + 2 * k;
                __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(o[i]) * inv, __uint_as_float(o[i + 1]) * inv);
                pk[k] = *reinterpret_cast<uint32_t*>(&b2);
              }
              d4[q4] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            }
          }
        }
      }
      // the next item's PV_i(0) (accumulate = 0) is issued only after our next pfull arrival,
      // which program order puts after these TMEM reads
      tc_fence_before();
      ++it_local;  // ofull phases of this warpgroup count only its own items
    }
  }
  tc_fence_before();
  __syncthreads();
  ATTN_TRACE_CTA(2);
  if (warp == kWarpMma) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// Merge the partials of split items: one warp per query row, 4 dims per lane.
__global__ void __launch_bounds__(256)
attn_combine_kernel(AttnParams p, const int4* __restrict__ combine, const float* __restrict__ part_o,
                    const float2* __restrict__ part_ml) {
  const int4 cb = combine[blockIdx.x];
  const int rr = blockIdx.y * 8 + (threadIdx.x >> 5);  // row of the item, [0, 256)
  const int lane = threadIdx.x & 31;
  const Item it = item_of(p, cb.x);
  const int G = p.H / p.Hkv;
  const int qt = rr / kM, r = rr % kM;
  const int t_row = it.tok0 + qt * (kM / G) + r / G;
  if (t_row >= it.qlen) return;
  float m = -INFINITY;
  for (int k = 0; k < cb.z; ++k) m = fmaxf(m, part_ml[static_cast<int64_t>(cb.y + k) * (kQT * kM) + rr].x);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  float l = 0.f;
  for (int k = 0; k < cb.z; ++k) {
    const int64_t prow = static_cast<int64_t>(cb.y + k) * (kQT * kM) + rr;
    const float2 ml = part_ml[prow];
    if (ml.x == -INFINITY || ml.y == 0.f) continue;  // piece with no visible key for this row
    const float wgt = ex2(ml.x - m);
    const float4 o = reinterpret_cast<const float4*>(part_o + prow * kHD)[lane];
    acc.x += wgt * o.x;
    acc.y += wgt * o.y;
    acc.z += wgt * o.z;
    acc.w += wgt * o.w;
    l += wgt * ml.y;
  }
  const float inv = 1.f / l;
  __nv_bfloat16* dst = p.o + (static_cast<int64_t>(it.qs + t_row) * p.H + it.kvh * G + r % G) * kHD + lane * 4;
  __nv_bfloat162 a = __floats2bfloat162_rn(acc.x * inv, acc.y * inv);
  __nv_bfloat162 b = __floats2bfloat162_rn(acc.z * inv, acc.w * inv);
  uint2 pk = make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
  *reinterpret_cast<uint2*>(dst) = pk;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    GLMX_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (!f || q != cudaDriverEntryPointSuccess) throw Error(GLMX_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

}  // namespace

// Tensor map over the whole pool viewed as [rows][128] bf16 (row = one token of one
// (page, layer, K|V, kv head) tile); box [16 rows][64 dims], 128B swizzle.
void make_pool_tensor_map(const PoolGeom& g, uint64_t pages, void* out_map, uint32_t* rows_total) {
  const uint64_t rows = pages * g.n_layers * 2 * g.n_kv_heads * g.block_tokens;
  if (rows >= 0x7FFFFFFFull) throw Error(GLMX_ERR_ARG, "pool too large for one tensor map");
  cuuint64_t dims[2] = {g.head_dim, rows};
  cuuint64_t strides[1] = {g.head_dim * sizeof(__nv_bfloat16)};
  cuuint32_t box[2] = {64, g.block_tokens};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(reinterpret_cast<CUtensorMap*>(out_map), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                           g.base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(GLMX_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  *rows_total = static_cast<uint32_t>(rows);
}

// Tensor map over the query buffer q [T][H][hd]: box [128/G tokens][G heads][64 dims] lands as
// the item's 128 rows (row = token * G + head-in-group), 128B swizzle; tokens >= T read zeros.
void make_q_tensor_map(const void* q, uint64_t T, int H, int Hkv, void* out_map) {
  const int G = H / Hkv;
  cuuint64_t dims[3] = {kHD, static_cast<cuuint64_t>(H), T};
  cuuint64_t strides[2] = {kHD * sizeof(__nv_bfloat16), static_cast<cuuint64_t>(H) * kHD * sizeof(__nv_bfloat16)};
  cuuint32_t box[3] = {64, static_cast<cuuint32_t>(G), static_cast<cuuint32_t>(kM / G)};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(reinterpret_cast<CUtensorMap*>(out_map), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                           const_cast<void*>(q), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(GLMX_ERR_CUDA, "cuTensorMapEncodeTiled (q) failed: " + std::to_string(r));
}

void paged_attention_tc(const AttnParams& p, const void* kv_map, uint32_t rows_total,
                        const void* q_map, const AttnTcSched& sc, cudaStream_t s) {
  if (p.n_work <= 0 || sc.grid <= 0) return;
  if (p.pool.head_dim != kHD || p.pool.block_tokens != kB)
    throw Error(GLMX_ERR_ARG, "paged attention is built for head_dim 128 and 16-token pages");
  const int G = p.H / p.Hkv;
  if (G * p.Hkv != p.H || kM % G != 0) throw Error(GLMX_ERR_ARG, "unsupported GQA ratio");
  if (p.bt_stride % 8 != 0 || (reinterpret_cast<uintptr_t>(p.block_table) & 15) != 0)
    throw Error(GLMX_ERR_ARG, "block-table rows must be 16-byte aligned multiples of 8 entries");
  // the attribute is per device: one flag per device ordinal (atomic, launches may race)
  static std::atomic<bool> attr[64];
  int dev = 0;
  GLMX_CUDA(cudaGetDevice(&dev));
  if (!attr[dev & 63].load(std::memory_order_acquire)) {
    GLMX_CUDA(cudaFuncSetAttribute(paged_attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    attr[dev & 63].store(true, std::memory_order_release);
  }
  TcParams tp{p, rows_total, sc.pieces, sc.cta_off, sc.part_o, sc.part_ml, sc.partners};
  launch_pdl(paged_attn_tc_kernel, dim3(sc.grid), dim3(kThreads), kSmem, s,
             *reinterpret_cast<const CUtensorMap*>(kv_map), *reinterpret_cast<const CUtensorMap*>(q_map), tp);
  GLMX_CHECK_LAUNCH();
  if (sc.n_combine > 0) {
    attn_combine_kernel<<<dim3(sc.n_combine, kQT * kM / 8), 256, 0, s>>>(p, sc.combine, sc.part_o, sc.part_ml);
    GLMX_CHECK_LAUNCH();
  }
}

int attn_tc_partial_rows() { return kQT * kM; }

int attn_trace_read(long long* out, int n) {
#ifdef GLMX_ATTN_TRACE
  const int m = std::min(n, 16 * 1024);
  GLMX_CUDA(cudaMemcpyFromSymbol(out, g_attn_trace, m * sizeof(long long)));
  GLMX_CUDA(cudaMemset(g_attn_trace_ptr(), 0, sizeof(long long) * 16 * 1024));
  return m;
#else
  (void)out;
  (void)n;
  return -1;
#endif
}

// Query tokens per work item: two 128-row tiles of 128/G tokens x G heads.
int attn_tc_tokens_per_tile(int H, int Hkv) { return kQT * kM / (H / Hkv); }

}  // namespace glmx
