// K3d — paged attention for decode rows (one query token per request, q_len == 1) on CUDA cores.
//
// A decode row of a GQA group is 4 query heads x 128 dims against the request's cached keys: a
// GEMV-shaped, HBM-bound read of the K and V pages (4 KB per page per kv head each).  The tcgen05
// kernel (attn_tc.cu) would fill 4 of its 128 MMA rows and serialise softmax -> PV -> S per key
// tile, so decode batches take this path instead (flash-decoding):
//   grid (request x kv head, split): a CTA walks pages [pg0, pg1) of its item's block table, its
//   4 warps taking half pages (8 keys) round robin.  Lane (half = lane / 16, slice = lane % 16)
//   loads 16 bytes (8 dims) of 4 key rows of K and of V (all 8 loads issued together), computes
//   partial dot products for the 4 heads, and a 4-step butterfly reduce-scatter over the 16
//   lanes of its half leaves every lane one full score (key, head).  Online softmax in base 2
//   per head (running max / sum in lanes 0-3, probabilities through shared memory), PV
//   accumulated in fp32 registers (4 heads x 8 dims per lane); the halves and the 4 warps merge
//   at the end.  Splits > 1 write unnormalised partials (O, m, l) that decode_combine_kernel
//   merges.
#include <cfloat>

#include "attn.cuh"
#include "common.cuh"

namespace glmx {

namespace {

constexpr int kG = 4;     // query heads per kv head
constexpr int kHd = 128;  // head dim
constexpr int kB = 16;    // tokens per page
constexpr int kWarps = 4;
constexpr int kStage = 2;  // half pages in flight per warp (cp.async ring, 32 KB per CTA)

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// packed fp32 pairs (FFMA2 / FMUL2 on sm_100): two lanes of the 8-dim slice per instruction
__device__ __forceinline__ uint64_t f2(float lo, float hi) {
  return static_cast<uint64_t>(__float_as_uint(lo)) | (static_cast<uint64_t>(__float_as_uint(hi)) << 32);
}
__device__ __forceinline__ float f2lo(uint64_t x) { return __uint_as_float(static_cast<uint32_t>(x)); }
__device__ __forceinline__ float f2hi(uint64_t x) { return __uint_as_float(static_cast<uint32_t>(x >> 32)); }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// 8 bf16 -> 4 packed fp32 pairs
__device__ __forceinline__ void bf8x2(const uint4& u, uint64_t (&f)[4]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) f[i] = f2(__uint_as_float(w[i] << 16), __uint_as_float(w[i] & 0xFFFF0000u));
}

__device__ __forceinline__ void bf8(const uint4& u, float (&f)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}

template <bool kFused>
__global__ void __launch_bounds__(kWarps * 32)
decode_attn_kernel(AttnParams p, DecodeRope rp, int n_split, float* __restrict__ part_o,
                   float2* __restrict__ part_ml) {
  __shared__ float4 s_p[kWarps][8];  // probabilities of the current half page: [key][head]
  __shared__ float s_mx[kWarps][kG], s_alpha[kWarps][kG];
  __shared__ float s_m[kWarps][kG], s_l[kWarps][kG];
  __shared__ float s_acc[kWarps][kG][kHd];
  // cp.async staging of the next half page: [warp][slot][K|V][row i][lane] 16-byte chunks (each
  // lane reads back exactly the chunks it copied)
  __shared__ uint4 s_kv[kWarps][kStage][2][4][32];
  const int item = blockIdx.x, split = blockIdx.y;
  const int req = item / p.Hkv, kvh = item % p.Hkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = lane >> 4, sl = lane & 15;
  const int ctx = p.ctx_len[req];
  const int n_units = (ctx + 7) / 8;  // half pages
  const int per = (n_units + n_split - 1) / n_split;
  const int u0 = split * per, u1 = min(n_units, u0 + per);
  const int qrow = p.q_start[req] + p.q_len[req] - 1;
  const float scale = p.scale_log2;
  float q[kG][8];
  if constexpr (kFused) {
    // RoPE of this lane's 8 dims (rotation partner dims are in lane sl ^ 8 of the same half),
    // rounded to bf16 like the separate K2 kernel's q / pool writes
    const int heads = p.H + 2 * p.Hkv;
    const __nv_bfloat16* row = rp.qkv + static_cast<int64_t>(qrow) * heads * kHd + sl * 8;
    float cs[8], sn[8];
    {
      const float4* tab = reinterpret_cast<const float4*>(rp.rope_cs + static_cast<int64_t>(qrow) * (kHd / 2) +
                                                          (sl & 7) * 8);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float4 v = __ldg(tab + j);
        cs[2 * j] = v.x;
        sn[2 * j] = v.y;
        cs[2 * j + 1] = v.z;
        sn[2 * j + 1] = v.w;
      }
    }
    auto rope8 = [&](const uint4& u, float (&out)[8]) {
      float f[8], o[8];
      bf8(u, f);
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = __shfl_xor_sync(0xffffffffu, f[j], 8);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        // first half: x1 c - x2 s; second half: x2 c + x1 s (own = x2, partner = x1)
        const float v = sl < 8 ? f[j] * cs[j] - o[j] * sn[j] : f[j] * cs[j] + o[j] * sn[j];
        out[j] = __bfloat162float(__float2bfloat16_rn(v));
      }
    };
#pragma unroll
    for (int h = 0; h < kG; ++h) {
      const uint4 u = *reinterpret_cast<const uint4*>(row + (kvh * kG + h) * kHd);
      float f[8];
      rope8(u, f);
#pragma unroll
      for (int j = 0; j < 8; ++j) q[h][j] = f[j] * scale;
    }
    // the new key / value: appended by the CTA whose range holds the last key, before its loop
    const uint4 ku = *reinterpret_cast<const uint4*>(row + (p.H + kvh) * kHd);
    const uint4 vu = *reinterpret_cast<const uint4*>(row + (p.H + p.Hkv + kvh) * kHd);
    float kf[8];
    rope8(ku, kf);
    if (u1 == n_units && half == 0 && warp == 0) {
      const int64_t slt = rp.slot[qrow];
      __nv_bfloat16* kd = p.pool.base + p.pool.tile_off(slt / p.pool.block_tokens, p.layer, 0, kvh) +
                          static_cast<int64_t>(slt % p.pool.block_tokens) * kHd + sl * 8;
      __nv_bfloat16* vd = p.pool.base + p.pool.tile_off(slt / p.pool.block_tokens, p.layer, 1, kvh) +
                          static_cast<int64_t>(slt % p.pool.block_tokens) * kHd + sl * 8;
      uint4 kb;
      __nv_bfloat162* k2 = reinterpret_cast<__nv_bfloat162*>(&kb);
#pragma unroll
      for (int j = 0; j < 4; ++j) k2[j] = __floats2bfloat162_rn(kf[2 * j], kf[2 * j + 1]);
      *reinterpret_cast<uint4*>(kd) = kb;
      *reinterpret_cast<uint4*>(vd) = vu;
      __threadfence();
    }
    __syncthreads();  // the appended key is read through L2 by the cp.async loads below
  } else {
#pragma unroll
    for (int h = 0; h < kG; ++h) {
      const uint4 u = *reinterpret_cast<const uint4*>(
          p.q + (static_cast<int64_t>(qrow) * p.H + kvh * kG + h) * kHd + sl * 8);
      float f[8];
      bf8(u, f);
#pragma unroll
      for (int j = 0; j < 8; ++j) q[h][j] = f[j] * scale;
    }
  }
  uint64_t q2[kG][4];
#pragma unroll
  for (int h = 0; h < kG; ++h)
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) q2[h][jj] = f2(q[h][2 * jj], q[h][2 * jj + 1]);
  uint64_t acc2[kG][4];
#pragma unroll
  for (int h = 0; h < kG; ++h)
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) acc2[h][jj] = 0ull;
  float m_run = -INFINITY, l_run = 0.f;  // head = lane, lanes 0-3
  const int32_t* bt = p.block_table + static_cast<int64_t>(req) * p.bt_stride;
  const uint64_t kv_stride = p.pool.tile_off(0, p.layer, 1, kvh) - p.pool.tile_off(0, p.layer, 0, kvh);
  // half pages u0 + warp, u0 + warp + kWarps, ...; the next one is staged in shared memory by
  // cp.async while this one is processed (a register double buffer was slower: 188 registers
  // halve the resident warps)
  auto process = [&](int u, const uint4 (&kr)[4], const uint4 (&vr)[4]) {
    // partial dots of this lane's 8 dims: v[i * 4 + h]
    float v[16];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint64_t kf[4];
      bf8x2(kr[i], kf);
#pragma unroll
      for (int h = 0; h < kG; ++h) {
        uint64_t s2 = 0ull;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) s2 = ffma2(q2[h][jj], kf[jj], s2);
        v[i * 4 + h] = f2lo(s2) + f2hi(s2);
      }
    }
    // reduce-scatter over the 16 lanes of this half: lane bit b keeps the half of the values
    // whose index bit matches; afterwards lane sl holds value index sl (i = sl >> 2, h = sl & 3)
#pragma unroll
    for (int step = 0; step < 4; ++step) {
      const int m = 8 >> step, c = 16 >> step;  // partner mask, values still held
      const bool up = sl & m;
#pragma unroll
      for (int j = 0; j < c / 2; ++j) {
        const float send = up ? v[j] : v[j + c / 2];
        const float keep = up ? v[j + c / 2] : v[j];
        v[j] = keep + __shfl_xor_sync(0xffffffffu, send, m);
      }
    }
    const int my_i = sl >> 2, my_h = sl & 3;
    const int key_abs = u * 8 + 2 * my_i + half;
    const float sc = key_abs < ctx ? v[0] : -INFINITY;
    // per-head max over the 8 keys: lanes with the same my_h (xor over bits 2, 3 and 4)
    float mx = sc;
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
    if (lane < kG) {  // lane == my_h here
      const float m_new = fmaxf(m_run, mx);
      s_alpha[warp][lane] = ex2f(m_run - m_new);  // m_run = -inf -> 0
      s_mx[warp][lane] = m_new;
      m_run = m_new;
    }
    __syncwarp();
    const float pr = ex2f(sc - s_mx[warp][my_h]);
    reinterpret_cast<float*>(&s_p[warp][2 * my_i + half])[my_h] = pr;
    float ps = pr;  // per-head sum over the 8 keys
    ps += __shfl_xor_sync(0xffffffffu, ps, 4);
    ps += __shfl_xor_sync(0xffffffffu, ps, 8);
    ps += __shfl_xor_sync(0xffffffffu, ps, 16);
    if (lane < kG) l_run = l_run * s_alpha[warp][lane] + ps;
    __syncwarp();
    float al[kG];
#pragma unroll
    for (int h = 0; h < kG; ++h) al[h] = s_alpha[warp][h];
#pragma unroll
    for (int h = 0; h < kG; ++h) {
      const uint64_t a2 = f2(al[h], al[h]);
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) acc2[h][jj] = fmul2(acc2[h][jj], a2);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4 pp = s_p[warp][2 * i + half];
      const float ph[kG] = {pp.x, pp.y, pp.z, pp.w};
      uint64_t vf[4];
      bf8x2(vr[i], vf);
#pragma unroll
      for (int h = 0; h < kG; ++h) {
        const uint64_t p2 = f2(ph[h], ph[h]);
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) acc2[h][jj] = ffma2(p2, vf[jj], acc2[h][jj]);
      }
    }
    __syncwarp();  // s_p / s_alpha reuse by the next half page
  };
  // the loads of kStage - 1 half pages are in flight while one is processed
  auto issue = [&](int u, int slot) {
    if (u < u1) {
      const int page = bt[u >> 1];
      const __nv_bfloat16* kt = p.pool.base + p.pool.tile_off(page, p.layer, 0, kvh) +
                                static_cast<int64_t>((u & 1) * 8) * kHd + sl * 8;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int key = 2 * i + half;
        cp_async16(&s_kv[warp][slot][0][i][lane], kt + key * kHd);
        cp_async16(&s_kv[warp][slot][1][i][lane], kt + kv_stride + key * kHd);
      }
    }
    cp_async_commit();  // possibly empty: keeps the group count uniform
  };
#pragma unroll
  for (int k = 0; k < kStage - 1; ++k) issue(u0 + warp + k * kWarps, k);
  for (int k = 0, u = u0 + warp; u < u1; ++k, u += kWarps) {
    issue(u + (kStage - 1) * kWarps, (k + kStage - 1) % kStage);
    cp_async_wait<kStage - 1>();
    const int slot = k % kStage;
    uint4 kr[4], vr[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      kr[i] = s_kv[warp][slot][0][i][lane];
      vr[i] = s_kv[warp][slot][1][i][lane];
    }
    process(u, kr, vr);
  }
  cp_async_wait<0>();
  // merge the two key halves, then the warps
  float acc[kG][8];
#pragma unroll
  for (int h = 0; h < kG; ++h)
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      acc[h][2 * jj] = f2lo(acc2[h][jj]);
      acc[h][2 * jj + 1] = f2hi(acc2[h][jj]);
    }
#pragma unroll
  for (int h = 0; h < kG; ++h)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[h][j] += __shfl_xor_sync(0xffffffffu, acc[h][j], 16);
  if (lane < kG) {
    s_m[warp][lane] = m_run;
    s_l[warp][lane] = l_run;
  }
  if (half == 0) {
#pragma unroll
    for (int h = 0; h < kG; ++h)
#pragma unroll
      for (int j = 0; j < 8; ++j) s_acc[warp][h][sl * 8 + j] = acc[h][j];
  }
  __syncthreads();
  const int d = threadIdx.x;  // 128 threads = 128 dims
#pragma unroll
  for (int h = 0; h < kG; ++h) {
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) M = fmaxf(M, s_m[w][h]);
    float L = 0.f, O = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const float wt = s_m[w][h] == -INFINITY ? 0.f : ex2f(s_m[w][h] - M);
      L += wt * s_l[w][h];
      O += wt * s_acc[w][h][d];
    }
    if (n_split == 1) {
      p.o[(static_cast<int64_t>(qrow) * p.H + kvh * kG + h) * kHd + d] = __float2bfloat16_rn(O / L);
    } else {
      const int64_t row = (static_cast<int64_t>(item) * n_split + split) * kG + h;
      part_o[row * kHd + d] = O;
      if (d == 0) part_ml[row] = make_float2(M, L);
    }
  }
}

__global__ void __launch_bounds__(kHd)
decode_combine_kernel(AttnParams p, int n_split, const float* __restrict__ part_o,
                      const float2* __restrict__ part_ml) {
  const int item = blockIdx.x;
  const int req = item / p.Hkv, kvh = item % p.Hkv;
  const int qrow = p.q_start[req] + p.q_len[req] - 1;
  const int d = threadIdx.x;
#pragma unroll
  for (int h = 0; h < kG; ++h) {
    float M = -INFINITY;
    for (int s = 0; s < n_split; ++s)
      M = fmaxf(M, part_ml[(static_cast<int64_t>(item) * n_split + s) * kG + h].x);
    float L = 0.f, O = 0.f;
    for (int s = 0; s < n_split; ++s) {
      const int64_t row = (static_cast<int64_t>(item) * n_split + s) * kG + h;
      const float2 ml = part_ml[row];
      const float wt = ml.x == -INFINITY ? 0.f : ex2f(ml.x - M);
      L += wt * ml.y;
      O += wt * part_o[row * kHd + d];
    }
    p.o[(static_cast<int64_t>(qrow) * p.H + kvh * kG + h) * kHd + d] = __float2bfloat16_rn(O / L);
  }
}

}  // namespace

bool decode_attention_supported(const AttnParams& p) {
  return p.H == kG * p.Hkv && p.pool.head_dim == kHd && p.pool.block_tokens == kB;
}

// Splits per item so that ~2 CTAs per SM are in flight (a 64-request decode step, 512 items,
// needs no split and no combine pass), bounded by the partial workspace rows (max_rows) and by
// one split per 4 half pages.
int decode_attention_splits(int n_items, int max_ctx, int max_rows) {
  const int units = (max_ctx + 7) / 8;
  int s = std::max(1, (2 * kNumSMs + n_items - 1) / std::max(1, n_items));
  s = std::min(s, std::max(1, units / 4));
  s = std::min(s, std::max(1, max_rows / std::max(1, n_items * kG)));
  return s;
}

void paged_attention_decode(const AttnParams& p, int n_req, int n_split, float* part_o,
                            float2* part_ml, cudaStream_t s) {
  if (n_req <= 0) return;
  if (!decode_attention_supported(p)) throw Error(GLMX_ERR_ARG, "decode attention: unsupported geometry");
  const int items = n_req * p.Hkv;
  decode_attn_kernel<false><<<dim3(items, n_split), kWarps * 32, 0, s>>>(p, DecodeRope{}, n_split,
                                                                       part_o, part_ml);
  GLMX_CHECK_LAUNCH();
  if (n_split > 1) {
    decode_combine_kernel<<<items, kHd, 0, s>>>(p, n_split, part_o, part_ml);
    GLMX_CHECK_LAUNCH();
  }
}

void paged_attention_decode_rope(const AttnParams& p, const DecodeRope& r, int n_req, int n_split,
                                 float* part_o, float2* part_ml, cudaStream_t s) {
  if (n_req <= 0) return;
  if (!decode_attention_supported(p)) throw Error(GLMX_ERR_ARG, "decode attention: unsupported geometry");
  const int items = n_req * p.Hkv;
  decode_attn_kernel<true><<<dim3(items, n_split), kWarps * 32, 0, s>>>(p, r, n_split, part_o, part_ml);
  GLMX_CHECK_LAUNCH();
  if (n_split > 1) {
    decode_combine_kernel<<<items, kHd, 0, s>>>(p, n_split, part_o, part_ml);
    GLMX_CHECK_LAUNCH();
  }
}

}  // namespace glmx
