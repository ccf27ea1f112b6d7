// K3 — paged causal GQA prefill attention on 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// CTA = one kv head x 128 query rows (128/G tokens x the G query heads sharing that kv head, so
// every K/V page is fetched once per GQA group).  Warp roles (192 threads):
//   warps 0-3  softmax / correction / epilogue: thread i owns query row i == TMEM lane i
//   warp 4     TMA producer: K and V pages of 128-key tiles -> 2-stage smem ring (16 boxes of
//              [16 tokens][64 dims] per operand per tile, 128B-swizzled, OOB pages zero-filled)
//   warp 5     MMA issuer (one elected thread):  S_j = Q K_j^T  (M128 N128 K128, fp32 in TMEM,
//              double-buffered)  and  O += P_{j-1} V_{j-1}  (P from smem, V MN-major)
// Online softmax in base 2 with a lazily updated running max (O in TMEM is only rescaled when
// the row max grows by more than 2^8), final 1/l normalisation in the epilogue.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cfloat>

#include "attn.cuh"
#include "common.cuh"

namespace glmx {

namespace {

constexpr int kHD = 128;
constexpr int kB = 16;
constexpr int kM = 128;        // query rows per CTA
constexpr int kN = 128;        // keys per tile
constexpr int kHalf = 16384;   // bytes of one [128][64] bf16 SW128 half tile
constexpr int kTile = 2 * kHalf;
constexpr int kThreads = 192;
// smem map (1024-aligned): Q | K0 K1 | V0 V1 | P | barriers
constexpr int kOffQ = 0;
constexpr int kOffK = kOffQ + kTile;
constexpr int kOffV = kOffK + 2 * kTile;
constexpr int kOffP = kOffV + 2 * kTile;
constexpr int kOffBar = kOffP + kTile;
constexpr int kSmem = kOffBar + 256 + 1024;  // + alignment slack

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// Bounded wait: a protocol bug traps with a location instead of hanging the GPU.  Roles record
// their progress in shared memory (g_prog) so a stuck thread reports every role's state.
__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __noinline__ void mbar_stuck(uint32_t bar, uint32_t parity, int tag, const volatile int* prog) {
  printf("paged_attn_tc: wait timeout block (%d,%d) thread %d bar 0x%x parity %u tag %d | prod %d mma %d sm0 %d sm127 %d sm64 %d\n",
         blockIdx.x, blockIdx.y, threadIdx.x, bar, parity, tag, prog[0], prog[1], prog[2], prog[3], prog[4]);
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity, int tag = 0,
                                          const volatile int* prog = nullptr) {
  if (mbar_try(bar, parity)) return;
  const uint64_t t0 = gtime();
  bool told = false;
  while (!mbar_try(bar, parity)) {
    const uint64_t dt = gtime() - t0;
    if (!told && dt > 2000000000ull) {
      if (prog) mbar_stuck(bar, parity, tag, prog);
      told = true;
    }
    if (dt > 4000000000ull) __trap();
  }
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
#define TC_LD32(taddr, r)                                                                      \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12," \
               "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, " \
               "[%32];"                                                                        \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),      \
                 "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),    \
                 "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), \
                 "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), \
                 "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), \
                 "=r"(r[30]), "=r"(r[31])                                                      \
               : "r"(taddr))
#define TC_ST32(taddr, r)                                                                      \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11," \
               "%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31," \
               "%32};" ::"r"(taddr),                                                           \
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),   \
               "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), \
               "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]),         \
               "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]),         \
               "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]))
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// UMMA shared-memory descriptor, SWIZZLE_128B, sm100 version 1.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFF) |
         (static_cast<uint64_t>(lbo & 0x3FFF) << 16) |
         (static_cast<uint64_t>(sbo & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
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

struct TcParams {
  AttnParams a;
  uint32_t rows_total;  // rows of the pool tensor map (OOB row -> zero fill)
};

__global__ void __launch_bounds__(kThreads, 1)
paged_attn_tc_kernel(const __grid_constant__ CUtensorMap kv_map, TcParams tp) {
  const AttnParams& p = tp.a;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_addr(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  // barriers: kfull[2] vfull[2] kempty[2] vempty[2] sfull[2] pfull ofull
  const uint32_t b_kfull = smem_addr(bars + 0), b_vfull = smem_addr(bars + 2);
  const uint32_t b_kempty = smem_addr(bars + 4), b_vempty = smem_addr(bars + 6);
  const uint32_t b_sfull = smem_addr(bars + 8), b_pfull = smem_addr(bars + 10);
  const uint32_t b_ofull = smem_addr(bars + 11);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 16);
  volatile int* prog = reinterpret_cast<volatile int*>(bars + 20);  // debug progress

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kvh = blockIdx.y;
  const int2 wk = p.work[blockIdx.x];
  const int req = wk.x, tok0 = wk.y;
  const int G = p.H / p.Hkv;
  const int TPT = kM / G;
  const int qlen = p.q_len[req], ctx = p.ctx_len[req], qs = p.q_start[req];
  const int base_pos = ctx - qlen;
  const int max_pos = base_pos + min(tok0 + TPT, qlen) - 1;
  const int n_kt = max_pos / kN + 1;
  const int32_t* bt = p.block_table + static_cast<int64_t>(req) * p.bt_stride;

  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(b_kfull + 8 * s, 1);
      mbar_init(b_vfull + 8 * s, 1);
      mbar_init(b_kempty + 8 * s, 1);
      mbar_init(b_vempty + 8 * s, 1);
      mbar_init(b_sfull + 8 * s, 1);
    }
    mbar_init(b_pfull, 128);
    mbar_init(b_ofull, 1);
    for (int i = 0; i < 5; ++i) prog[i] = -1;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 5) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_addr(tmem_holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // Q tile -> smem (rows m: token m/G, head kvh*G + m%G), 128B swizzle, by the softmax warps
  if (warp < 4) {
    for (int i = threadIdx.x; i < kM * 16; i += 128) {
      const int m = i >> 4, c = i & 15;
      const int t = min(tok0 + m / G, qlen - 1);
      const int h = kvh * G + m % G;
      const uint4 v = *reinterpret_cast<const uint4*>(p.q + (static_cast<int64_t>(qs + t) * p.H + h) * kHD + c * 8);
      *reinterpret_cast<uint4*>(smem + kOffQ + sw128(m, c)) = v;
    }
    fence_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const uint32_t t_s0 = tmem, t_o = tmem + 256;

  if (warp == 4) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      const uint32_t L = p.pool.n_layers, Hkv = p.pool.n_kv_heads;
      for (int j = 0; j < n_kt; ++j) {
        const int s = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        for (int kv = 0; kv < 2; ++kv) {
          const uint32_t full = (kv ? b_vfull : b_kfull) + 8 * s;
          if (j >= 2) mbar_wait((kv ? b_vempty : b_kempty) + 8 * s, ph ^ 1, 100 + j * 10 + kv, prog);
          mbar_expect_tx(full, kTile);
          const uint32_t dst = sbase + (kv ? kOffV : kOffK) + s * kTile;
          for (int pg = 0; pg < kN / kB; ++pg) {
            const int key0 = j * kN + pg * kB;
            uint32_t row = tp.rows_total;  // out of bounds -> zeros
            if (key0 < ctx) {
              const uint32_t page = static_cast<uint32_t>(bt[key0 / kB]);
              row = (((page * L + p.layer) * 2 + kv) * Hkv + kvh) * kB;
            }
            for (int hf = 0; hf < 2; ++hf)
              tma_load_2d(dst + hf * kHalf + pg * kB * 128, &kv_map, hf * 64, static_cast<int>(row), full);
          }
          prog[0] = j * 10 + kv;
        }
      }
    }
    __syncwarp();  // reconverge before the CTA barrier (bar.sync is .aligned)
  } else if (warp == 5) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idS = idesc_bf16(kN, false), idO = idesc_bf16(kHD, true);
      const uint32_t q_addr = sbase + kOffQ, p_addr = sbase + kOffP;
      auto issue_pv = [&](int j) {
        const int s = j & 1;
        mbar_wait(b_pfull, j & 1, 3000 + j * 10 + threadIdx.x % 10, prog);  // P_j in smem, O rescaled
        mbar_wait(b_vfull + 8 * s, (j >> 1) & 1, 400 + j, prog);
        tc_fence_after();
        const uint32_t v_addr = sbase + kOffV + s * kTile;
        for (int ks = 0; ks < kN / 16; ++ks) {
          const uint64_t a = smem_desc(p_addr + (ks >> 2) * kHalf + (ks & 3) * 32, 1, 64);
          const uint64_t b = smem_desc(v_addr + ks * 2048, kHalf >> 4, 64);
          tc_mma(t_o, a, b, idO, (j > 0 || ks > 0) ? 1u : 0u);
        }
        tc_commit(b_vempty + 8 * s);
        tc_commit(b_ofull);
        prog[1] = j * 10 + 2;
      };
      for (int j = 0; j < n_kt; ++j) {
        const int s = j & 1;
        // S buffer s is free: softmax(j-2) arrived on pfull before issue_pv(j-2) (iteration
        // j-1) could proceed.  (Re-waiting pfull here could alias a later phase.)
        mbar_wait(b_kfull + 8 * s, (j >> 1) & 1, 200 + j, prog);
        tc_fence_after();
        const uint32_t k_addr = sbase + kOffK + s * kTile;
        for (int ks = 0; ks < kHD / 16; ++ks) {
          const uint64_t a = smem_desc(q_addr + (ks >> 2) * kHalf + (ks & 3) * 32, 1, 64);
          const uint64_t b = smem_desc(k_addr + (ks >> 2) * kHalf + (ks & 3) * 32, 1, 64);
          tc_mma(t_s0 + s * kN, a, b, idS, ks > 0 ? 1u : 0u);
        }
        tc_commit(b_kempty + 8 * s);
        tc_commit(b_sfull + 8 * s);
        prog[1] = j * 10 + 1;
        if (j >= 1) issue_pv(j - 1);
      }
      issue_pv(n_kt - 1);
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- softmax warps
    const int r = threadIdx.x;  // query row == TMEM lane
    const int tq = min(tok0 + r / G, qlen - 1);
    const int pos = base_pos + tq;
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    float m_used = -FLT_MAX, l = 0.f;
    uint32_t v[32];
    for (int j = 0; j < n_kt; ++j) {
      const int s = j & 1;
      mbar_wait(b_sfull + 8 * s, (j >> 1) & 1, 500 + j * 1000 + n_kt, prog);
      tc_fence_after();
      const uint32_t ts = t_s0 + s * kN + lane_off;
      // pass 1: masked row max
      float mx = -FLT_MAX;
      for (int c = 0; c < 4; ++c) {
        TC_LD32(ts + c * 32, v);
        tc_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int key = j * kN + c * 32 + i;
          if (key <= pos) mx = fmaxf(mx, __uint_as_float(v[i]) * p.scale_log2);
        }
      }
      // PV_{j-1} must be complete before O is rescaled or P is overwritten
      if (j >= 1) {
        mbar_wait(b_ofull, (j - 1) & 1, 600 + j, prog);
        tc_fence_after();
      }
      // Lazy rescale: a row only moves its reference max when it grew by > 2^8.  The decision
      // is made warp-uniform because tcgen05.ld/st are .sync.aligned (rows that do not need it
      // scale by 1).
      const bool grow = mx > m_used + 8.f;
      if (__any_sync(0xffffffffu, grow)) {
        const float alpha = grow ? exp2f(m_used - mx) : 1.f;
        if (j >= 1) {
          for (int c = 0; c < 4; ++c) {
            TC_LD32(t_o + lane_off + c * 32, v);
            tc_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
            TC_ST32(t_o + lane_off + c * 32, v);
          }
          tc_wait_st();
        }
        l *= alpha;
        if (grow) m_used = mx;
      }
      // pass 2: p = exp2(s - m_used) -> bf16 P tile (row r, 128 keys), row sum
      for (int c = 0; c < 4; ++c) {
        TC_LD32(ts + c * 32, v);
        tc_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const int key = j * kN + c * 32 + i;
          const float p0 = key <= pos ? exp2f(__uint_as_float(v[i]) * p.scale_log2 - m_used) : 0.f;
          const float p1 = key + 1 <= pos ? exp2f(__uint_as_float(v[i + 1]) * p.scale_log2 - m_used) : 0.f;
          l += p0 + p1;
          __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
          pk[i >> 1] = *reinterpret_cast<uint32_t*>(&b2);
        }
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const int c16 = c * 4 + q4;
          *reinterpret_cast<uint4*>(smem + kOffP + sw128(r, c16)) =
              make_uint4(pk[4 * q4], pk[4 * q4 + 1], pk[4 * q4 + 2], pk[4 * q4 + 3]);
        }
      }
      fence_async_smem();
      tc_fence_before();
      mbar_arrive(b_pfull);
      if (r == 0) prog[2] = j;
      if (r == 127) prog[3] = j;
      if (r == 64) prog[4] = j;
    }
    // epilogue
    mbar_wait(b_ofull, (n_kt - 1) & 1, 700 + n_kt, prog);
    tc_fence_after();
    const int t = tok0 + r / G;
    const float inv = 1.f / l;
    __nv_bfloat16* dst = p.o + (static_cast<int64_t>(qs + tq) * p.H + kvh * G + r % G) * kHD;
    for (int c = 0; c < 4; ++c) {
      TC_LD32(t_o + lane_off + c * 32, v);
      tc_wait_ld();
      if (t < qlen) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(v[i]) * inv, __uint_as_float(v[i + 1]) * inv);
          pk[i >> 1] = *reinterpret_cast<uint32_t*>(&b2);
        }
        uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) d4[q4] = make_uint4(pk[4 * q4], pk[4 * q4 + 1], pk[4 * q4 + 2], pk[4 * q4 + 3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
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

void paged_attention_tc(const AttnParams& p, const void* kv_map, uint32_t rows_total, cudaStream_t s) {
  if (p.n_work <= 0) return;
  if (p.pool.head_dim != kHD || p.pool.block_tokens != kB)
    throw Error(GLMX_ERR_ARG, "paged attention is built for head_dim 128 and 16-token pages");
  const int G = p.H / p.Hkv;
  if (G * p.Hkv != p.H || kM % G != 0) throw Error(GLMX_ERR_ARG, "unsupported GQA ratio");
  static bool attr = false;
  if (!attr) {
    GLMX_CUDA(cudaFuncSetAttribute(paged_attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    attr = true;
  }
  TcParams tp{p, rows_total};
  dim3 grid(p.n_work, p.Hkv);
  paged_attn_tc_kernel<<<grid, kThreads, kSmem, s>>>(*reinterpret_cast<const CUtensorMap*>(kv_map), tp);
  GLMX_CHECK_LAUNCH();
}

int attn_tc_tokens_per_tile(int H, int Hkv) { return kM / (H / Hkv); }

}  // namespace glmx
