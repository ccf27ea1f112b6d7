// K3 v0: paged causal GQA attention, FA2-style on mma.sync (HMMA) — the correctness baseline
// for the tcgen05 kernel.  One CTA = one kv head x 64 query rows (64/G tokens x G query heads of
// that kv head, so each K/V page is read once for the whole GQA group); 4 warps x 16 rows.
// K/V tiles of 64 keys = 4 pages of 16 tokens, cp.async double-buffered into XOR-swizzled smem.
#include <atomic>
#include <cfloat>

#include "attn.cuh"
#include "common.cuh"

namespace glmx {

namespace {

constexpr int kHD = 128;
constexpr int kB = 16;
constexpr int kRows = 64;
constexpr int kKeys = 64;
constexpr int kThreads = 128;
constexpr int kTileBytes = kRows * kHD * 2;  // 16 KiB

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// byte offset of 16-byte chunk c of row r in a [rows][128] bf16 tile, XOR swizzled
__device__ __forceinline__ uint32_t swz(int r, int c) {
  return static_cast<uint32_t>(r * 256 + ((c ^ (r & 7)) << 4));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& a, uint32_t& b, uint32_t& c,
                                        uint32_t& d) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& a, uint32_t& b, uint32_t& c,
                                          uint32_t& d) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

__global__ void __launch_bounds__(kThreads)
paged_attn_mma_kernel(AttnParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQ = smem;
  uint8_t* sK = smem + kTileBytes;           // 2 buffers
  uint8_t* sV = smem + 3 * kTileBytes;       // 2 buffers

  const int kvh = blockIdx.y;
  const int2 wk = p.work[blockIdx.x];
  const int req = wk.x, tok0 = wk.y;
  const int G = p.H / p.Hkv;
  const int TPT = kRows / G;
  const int qlen = p.q_len[req], ctx = p.ctx_len[req], qs = p.q_start[req];
  const int base_pos = ctx - qlen;
  const int last_tok = min(tok0 + TPT, qlen) - 1;
  const int max_pos = base_pos + last_tok;
  const int n_kt = max_pos / kKeys + 1;
  const int32_t* bt = p.block_table + static_cast<int64_t>(req) * p.bt_stride;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- Q tile -> smem (rows m: token m/G, head kvh*G + m%G)
  for (int i = tid; i < kRows * 16; i += kThreads) {
    const int m = i >> 4, c = i & 15;
    const int t = tok0 + m / G;
    const int h = kvh * G + m % G;
    const bool valid = t < qlen;
    const __nv_bfloat16* src = p.q + (static_cast<int64_t>(qs + (valid ? t : 0)) * p.H + h) * kHD + c * 8;
    cp_async16(smem_u32(sQ + swz(m, c)), src, valid);
  }
  auto load_kv = [&](int kt, int buf) {
    uint8_t* dK = sK + buf * kTileBytes;
    uint8_t* dV = sV + buf * kTileBytes;
    for (int i = tid; i < kKeys * 16; i += kThreads) {
      const int key = i >> 4, c = i & 15;
      const int j = kt * kKeys + key;
      const bool valid = j < ctx;
      const int page = valid ? bt[j / kB] : 0;
      const int slot = j % kB;
      const __nv_bfloat16* k = p.pool.base + p.pool.tile_off(page, p.layer, 0, kvh) + slot * kHD + c * 8;
      const __nv_bfloat16* v = p.pool.base + p.pool.tile_off(page, p.layer, 1, kvh) + slot * kHD + c * 8;
      cp_async16(smem_u32(dK + swz(key, c)), k, valid);
      cp_async16(smem_u32(dV + swz(key, c)), v, valid);
    }
  };
  load_kv(0, 0);
  cp_commit();

  // per-thread rows (within the warp's 16): r0 = lane/4, r1 = r0 + 8
  int pos_r[2];
  for (int i = 0; i < 2; ++i) {
    const int m = warp * 16 + (lane >> 2) + i * 8;
    const int t = min(tok0 + m / G, qlen - 1);
    pos_r[i] = base_pos + t;
  }
  float m_r[2] = {-FLT_MAX, -FLT_MAX}, l_r[2] = {0.f, 0.f};
  float o[16][4];
#pragma unroll
  for (int n = 0; n < 16; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  uint32_t qf[8][4];

  for (int kt = 0; kt < n_kt; ++kt) {
    if (kt + 1 < n_kt) {
      load_kv(kt + 1, (kt + 1) & 1);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    if (kt == 0) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int r = warp * 16 + (lane & 15);
        const int c = kk * 2 + (lane >> 4);
        ldsm_x4(smem_u32(sQ + swz(r, c)), qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
      }
    }
    const uint8_t* cK = sK + (kt & 1) * kTileBytes;
    const uint8_t* cV = sV + (kt & 1) * kTileBytes;

    // ---- S = Q K^T : 16 rows x 64 keys per warp
    float s[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {  // pairs of 8-key n tiles
        uint32_t b0, b1, b2, b3;
        const int key = np * 16 + ((lane >> 4) << 3) + (lane & 7);
        const int c = kk * 2 + ((lane >> 3) & 1);
        ldsm_x4(smem_u32(cK + swz(key, c)), b0, b1, b2, b3);
        mma16816(s[2 * np], qf[kk], b0, b1);
        mma16816(s[2 * np + 1], qf[kk], b2, b3);
      }
    }
    // ---- mask + online softmax (base-2)
    float mx[2] = {-FLT_MAX, -FLT_MAX};
#pragma unroll
    for (int n = 0; n < 8; ++n) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = kt * kKeys + n * 8 + 2 * (lane & 3) + (e & 1);
        const int ri = e >> 1;
        float v = s[n][e] * p.scale_log2;
        v = key <= pos_r[ri] ? v : -FLT_MAX;
        s[n][e] = v;
        mx[ri] = fmaxf(mx[ri], v);
      }
    }
    float alpha[2];
#pragma unroll
    for (int ri = 0; ri < 2; ++ri) {
      mx[ri] = fmaxf(mx[ri], __shfl_xor_sync(0xffffffffu, mx[ri], 1));
      mx[ri] = fmaxf(mx[ri], __shfl_xor_sync(0xffffffffu, mx[ri], 2));
      const float mn = fmaxf(m_r[ri], mx[ri]);
      alpha[ri] = exp2f(m_r[ri] - mn);
      m_r[ri] = mn;
    }
    float rs[2] = {0.f, 0.f};
#pragma unroll
    for (int n = 0; n < 8; ++n) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int ri = e >> 1;
        const float pv = s[n][e] == -FLT_MAX ? 0.f : exp2f(s[n][e] - m_r[ri]);
        s[n][e] = pv;
        rs[ri] += pv;
      }
    }
#pragma unroll
    for (int ri = 0; ri < 2; ++ri) l_r[ri] = l_r[ri] * alpha[ri] + rs[ri];
#pragma unroll
    for (int n = 0; n < 16; ++n) {
      o[n][0] *= alpha[0];
      o[n][1] *= alpha[0];
      o[n][2] *= alpha[1];
      o[n][3] *= alpha[1];
    }
    // ---- O += P V
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {  // 16 keys per k-step
      uint32_t a[4];
      a[0] = pack_bf16(s[2 * kk][0], s[2 * kk][1]);
      a[1] = pack_bf16(s[2 * kk][2], s[2 * kk][3]);
      a[2] = pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      a[3] = pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int dp = 0; dp < 8; ++dp) {  // pairs of 8-wide d tiles
        uint32_t b0, b1, b2, b3;
        const int key = kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
        const int c = dp * 2 + (lane >> 4);
        ldsm_x4_t(smem_u32(cV + swz(key, c)), b0, b1, b2, b3);
        mma16816(o[2 * dp], a, b0, b1);
        mma16816(o[2 * dp + 1], a, b2, b3);
      }
    }
    __syncthreads();
  }
  // ---- finalize rows: full quad sum of l, normalise, store
#pragma unroll
  for (int ri = 0; ri < 2; ++ri) {
    l_r[ri] += __shfl_xor_sync(0xffffffffu, l_r[ri], 1);
    l_r[ri] += __shfl_xor_sync(0xffffffffu, l_r[ri], 2);
  }
#pragma unroll
  for (int ri = 0; ri < 2; ++ri) {
    const int m = warp * 16 + (lane >> 2) + ri * 8;
    const int t = tok0 + m / G;
    if (t >= qlen) continue;
    const int h = kvh * G + m % G;
    const float inv = 1.f / l_r[ri];
    __nv_bfloat16* dst = p.o + (static_cast<int64_t>(qs + t) * p.H + h) * kHD;
#pragma unroll
    for (int n = 0; n < 16; ++n) {
      const int col = n * 8 + 2 * (lane & 3);
      *reinterpret_cast<uint32_t*>(dst + col) = pack_bf16(o[n][2 * ri] * inv, o[n][2 * ri + 1] * inv);
    }
  }
}

}  // namespace

int attn_tokens_per_tile(int H, int Hkv) { return kRows / (H / Hkv); }

void paged_attention(const AttnParams& p, cudaStream_t s) {
  if (p.n_work <= 0) return;
  if (p.pool.head_dim != kHD || p.pool.block_tokens != kB)
    throw Error(GLMX_ERR_ARG, "paged attention is built for head_dim 128 and 16-token pages");
  const int G = p.H / p.Hkv;
  if (G * p.Hkv != p.H || kRows % G != 0) throw Error(GLMX_ERR_ARG, "unsupported GQA ratio");
  const int smem = 5 * kTileBytes;
  // the attribute is per device: one flag per device ordinal (atomic, launches may race)
  static std::atomic<bool> attr[64];
  int dev = 0;
  GLMX_CUDA(cudaGetDevice(&dev));
  if (!attr[dev & 63].load(std::memory_order_acquire)) {
    GLMX_CUDA(cudaFuncSetAttribute(paged_attn_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr[dev & 63].store(true, std::memory_order_release);
  }
  dim3 grid(p.n_work, p.Hkv);
  paged_attn_mma_kernel<<<grid, kThreads, smem, s>>>(p);
  GLMX_CHECK_LAUNCH();
}

}  // namespace glmx
