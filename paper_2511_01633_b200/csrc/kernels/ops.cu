#include <cfloat>

#include "common.cuh"
#include "ops.cuh"

namespace glmx {

namespace {

__global__ void init_normal_kernel(__nv_bfloat16* p, uint64_t n, uint64_t seed, float std) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t a = mix64(seed ^ (i * 0xd1b54a32d192ed03ULL));
    uint64_t b = mix64(a ^ 0x8cb92ba72f3d8dd7ULL);
    float u1 = (static_cast<float>(a >> 40) + 1.0f) * (1.0f / 16777217.0f);  // (0, 1]
    float u2 = static_cast<float>(b >> 40) * (1.0f / 16777216.0f);
    float z = sqrtf(-2.0f * logf(u1)) * cospif(2.0f * u2);
    p[i] = __float2bfloat16(z * std);
  }
}

__global__ void init_const_kernel(__nv_bfloat16* p, uint64_t n, float v) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    p[i] = __float2bfloat16(v);
}

__global__ void embed_kernel(const int32_t* __restrict__ tok, const __nv_bfloat16* __restrict__ E,
                             int d, float* __restrict__ x) {
  const int t = blockIdx.x;
  const __nv_bfloat16* row = E + static_cast<int64_t>(tok[t]) * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x)
    x[static_cast<int64_t>(t) * d + i] = __bfloat162float(row[i]);
}

template <int NT>
__device__ __forceinline__ float block_sum(float v, float* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < NT / 32 ? red[l] : 0.f;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (l == 0) red[0] = v;
  }
  __syncthreads();
  return red[0];
}

template <int NT>
__global__ void __launch_bounds__(NT)
rmsnorm_kernel(const float* __restrict__ x, const int32_t* __restrict__ rows, int d,
               const __nv_bfloat16* __restrict__ w, float eps, __nv_bfloat16* __restrict__ out) {
  __shared__ float red[32];
  const int t = blockIdx.x;
  const int64_t src = rows ? rows[t] : t;
  const float4* xr = reinterpret_cast<const float4*>(x + src * d);
  float ss = 0.f;
  for (int i = threadIdx.x; i < d / 4; i += NT) {
    float4 v = xr[i];
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  ss = block_sum<NT>(ss, red);
  const float inv = rsqrtf(ss / static_cast<float>(d) + eps);
  __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(out + static_cast<int64_t>(t) * d);
  const __nv_bfloat162* w2 = reinterpret_cast<const __nv_bfloat162*>(w);
  for (int i = threadIdx.x; i < d / 4; i += NT) {
    float4 v = xr[i];
    float2 wa = __bfloat1622float2(w2[2 * i]), wb = __bfloat1622float2(w2[2 * i + 1]);
    o[2 * i] = __floats2bfloat162_rn(v.x * inv * wa.x, v.y * inv * wa.y);
    o[2 * i + 1] = __floats2bfloat162_rn(v.z * inv * wb.x, v.w * inv * wb.y);
  }
}

// d = 4096 (the Llama-3-8B width): the row stays in registers (4 float4 per thread, all issued
// before the reduction), a single read of x; 8-byte bf16 stores.
template <int NT, int D>
__global__ void __launch_bounds__(NT)
rmsnorm_reg_kernel(const float* __restrict__ x, const int32_t* __restrict__ rows,
                   const __nv_bfloat16* __restrict__ w, float eps, __nv_bfloat16* __restrict__ out) {
  constexpr int kV = D / 4 / NT;  // float4 per thread
  __shared__ float red[32];
  pdl_wait();
  const int t = blockIdx.x;
  const int64_t src = rows ? rows[t] : t;
  const float4* xr = reinterpret_cast<const float4*>(x + src * D);
  float4 v[kV];
  uint2 wr[kV];  // the weights are loaded together with x, not after the reduction
  const uint2* w4 = reinterpret_cast<const uint2*>(w);
#pragma unroll
  for (int k = 0; k < kV; ++k) {
    v[k] = __ldcs(xr + threadIdx.x + k * NT);
    wr[k] = __ldg(w4 + threadIdx.x + k * NT);
  }
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < kV; ++k) ss += v[k].x * v[k].x + v[k].y * v[k].y + v[k].z * v[k].z + v[k].w * v[k].w;
  ss = block_sum<NT>(ss, red);
  const float inv = rsqrtf(ss / static_cast<float>(D) + eps);
  uint2* o = reinterpret_cast<uint2*>(out + static_cast<int64_t>(t) * D);
#pragma unroll
  for (int k = 0; k < kV; ++k) {
    const int i = threadIdx.x + k * NT;
    const uint2 wv = wr[k];
    const float2 wa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv.x));
    const float2 wb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv.y));
    __nv_bfloat162 a = __floats2bfloat162_rn(v[k].x * inv * wa.x, v[k].y * inv * wa.y);
    __nv_bfloat162 b = __floats2bfloat162_rn(v[k].z * inv * wb.x, v[k].w * inv * wb.y);
    o[i] = make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
  }
}

// K2: RoPE + KV append, kTok tokens per CTA.  The CTA first builds the cos/sin tables of its
// tokens in shared memory (fp32 angle pos * inv_freq, accurate sincosf: positions reach 32k), then
// every (token, head slot, 8-element chunk) work unit is two 16-byte loads (the rotate-half
// partners c and c + hd/2) and two 16-byte stores.  Head slots: H query heads (-> q_out), Hkv K
// heads (roped -> pool page), Hkv V heads (copied -> pool page).  A warp covers 4 heads x 8 chunks
// of one token: every load and store instruction moves two fully used 128-byte lines.  All of a
// thread's loads are issued before its first store (kUnroll units in flight per thread).
template <int kTok, int kUnroll>
__global__ void __launch_bounds__(256)
rope_kv_append_kernel(const __nv_bfloat16* __restrict__ qkv, const int32_t* __restrict__ pos,
                      const int64_t* __restrict__ slot, int T, int H, int Hkv, int hd,
                      const float* __restrict__ inv_freq, PoolGeom pool, uint32_t layer,
                      __nv_bfloat16* __restrict__ q_out) {
  __shared__ float cs_tab[kTok][128], sn_tab[kTok][128];
  const int t_base = blockIdx.x * kTok;
  const int half = hd / 2;
  const int heads = H + 2 * Hkv;
  const int chunks = half / 8;
  const int per_tok = heads * chunks;
  const int units = kTok * per_tok;
  uint4 av[kUnroll], bv[kUnroll];
  auto load = [&](int u0) {
#pragma unroll
    for (int k = 0; k < kUnroll; ++k) {
      const int u = u0 + k * blockDim.x;
      const int tt = u / per_tok, w = u % per_tok;
      const int t = t_base + tt;
      if (u < units && t < T) {
        const __nv_bfloat16* src = qkv + (static_cast<int64_t>(t) * heads + w / chunks) * hd + (w % chunks) * 8;
        av[k] = __ldcs(reinterpret_cast<const uint4*>(src));
        bv[k] = __ldcs(reinterpret_cast<const uint4*>(src + half));
      }
    }
  };
  auto process = [&](int u0) {
#pragma unroll
    for (int k = 0; k < kUnroll; ++k) {
      const int u = u0 + k * blockDim.x;
      const int tt = u / per_tok, w = u % per_tok;
      const int t = t_base + tt;
      if (u >= units || t >= T) continue;
      const int h = w / chunks, c = w % chunks;
      __nv_bfloat16* dst;
      bool rotate = true;
      if (h < H) {
        dst = q_out + (static_cast<int64_t>(t) * H + h) * hd + c * 8;
      } else {
        const int kv = h < H + Hkv ? 0 : 1;
        const int kh = h - H - kv * Hkv;
        const int64_t sl = slot[t];
        dst = pool.base + pool.tile_off(sl / pool.block_tokens, layer, kv, kh) +
              static_cast<int64_t>(sl % pool.block_tokens) * hd + c * 8;
        rotate = kv == 0;
      }
      if (!rotate) {
        *reinterpret_cast<uint4*>(dst) = av[k];
        *reinterpret_cast<uint4*>(dst + half) = bv[k];
        continue;
      }
      const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&av[k]);
      const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&bv[k]);
      uint4 ra, rb;
      __nv_bfloat162* ra2 = reinterpret_cast<__nv_bfloat162*>(&ra);
      __nv_bfloat162* rb2 = reinterpret_cast<__nv_bfloat162*>(&rb);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 a = __bfloat1622float2(a2[q]), b = __bfloat1622float2(b2[q]);
        const int i = c * 8 + 2 * q;
        const float c0 = cs_tab[tt][i], s0 = sn_tab[tt][i], c1 = cs_tab[tt][i + 1], s1 = sn_tab[tt][i + 1];
        ra2[q] = __floats2bfloat162_rn(a.x * c0 - b.x * s0, a.y * c1 - b.y * s1);
        rb2[q] = __floats2bfloat162_rn(b.x * c0 + a.x * s0, b.y * c1 + a.y * s1);
      }
      *reinterpret_cast<uint4*>(dst) = ra;
      *reinterpret_cast<uint4*>(dst + half) = rb;
    }
  };
  // the first loads are in flight while the cos/sin tables are built
  load(threadIdx.x);
  for (int i = threadIdx.x; i < kTok * half; i += blockDim.x) {
    const int tt = i / half, k = i % half;
    const int t = min(t_base + tt, T - 1);
    sincosf(static_cast<float>(pos[t]) * inv_freq[k], &sn_tab[tt][k], &cs_tab[tt][k]);
  }
  __syncthreads();
  process(threadIdx.x);
  for (int u0 = threadIdx.x + blockDim.x * kUnroll; u0 < units; u0 += blockDim.x * kUnroll) {
    load(u0);
    process(u0);
  }
}


// K2, warp-per-(token, head group) form (head_dim 128: 8 lanes per head, 4 heads per pass, 16
// heads per warp = blockIdx.y's group): a lane's cos/sin of its 8 rotation pairs come from the
// forward's RoPE table (rope_table: one sincosf per (token, pair) per forward instead of per layer
// and head group; the large-argument sincosf path was a third of K2's issue slots) and are reused
// across the warp's heads; the 4 passes issue all 8 loads of a lane before any store.
// Small prefill batches (a few hundred tokens) still spread over the SMs with one round trip per
// warp; mid-size batches (~3-5k tokens) fill the machine in one wave instead of the 1.2 waves of
// 2-token CTAs.
template <int kPassU>
__global__ void __launch_bounds__(256)
rope_kv_append_warp_kernel(const __nv_bfloat16* __restrict__ qkv, const float2* __restrict__ rope_cs,
                           const int64_t* __restrict__ slot, int T, int H, int Hkv, PoolGeom pool,
                           uint32_t layer, __nv_bfloat16* __restrict__ q_out) {
  constexpr int kHd = 128, kHalf = 64, kChunks = 8, kHeadsPerPass = 32 / kChunks;
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= T) return;
  const int c = lane % kChunks, hsub = lane / kChunks;
  const int heads = H + 2 * Hkv;
  const int pass_lo = blockIdx.y * kPassU, pass_hi = min((heads + kHeadsPerPass - 1) / kHeadsPerPass,
                                                        pass_lo + kPassU);
  if (pass_lo >= pass_hi) return;
  const int64_t sl = slot[t];
  const __nv_bfloat16* row = qkv + static_cast<int64_t>(t) * heads * kHd + c * 8;
  // the grid's y dimension covers kPassU passes per warp: one group, loads issued before the
  // cos/sin of the rotation pairs are computed (V-only groups skip them)
  const int p0 = pass_lo;
  {
    uint4 av[kPassU], bv[kPassU];
#pragma unroll
    for (int i = 0; i < kPassU; ++i) {
      const int h = (p0 + i) * kHeadsPerPass + hsub;
      if (h < heads) {
        av[i] = __ldcs(reinterpret_cast<const uint4*>(row + h * kHd));
        bv[i] = __ldcs(reinterpret_cast<const uint4*>(row + h * kHd + kHalf));
      }
    }
    float cs[8], sn[8];
    if (p0 * kHeadsPerPass < H + Hkv) {  // the token's (cos, sin) row of the forward's table
      const float4* tab = reinterpret_cast<const float4*>(rope_cs + static_cast<int64_t>(t) * kHalf + c * 8);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float4 v = __ldg(tab + j);
        cs[2 * j] = v.x;
        sn[2 * j] = v.y;
        cs[2 * j + 1] = v.z;
        sn[2 * j + 1] = v.w;
      }
    }
#pragma unroll
    for (int i = 0; i < kPassU; ++i) {
      const int h = (p0 + i) * kHeadsPerPass + hsub;
      if (h >= heads) continue;
      __nv_bfloat16* dst;
      bool rotate = true;
      if (h < H) {
        dst = q_out + (static_cast<int64_t>(t) * H + h) * kHd + c * 8;
      } else {
        const int kv = h < H + Hkv ? 0 : 1;
        const int kh = h - H - kv * Hkv;
        dst = pool.base + pool.tile_off(sl / pool.block_tokens, layer, kv, kh) +
              static_cast<int64_t>(sl % pool.block_tokens) * kHd + c * 8;
        rotate = kv == 0;
      }
      if (!rotate) {
        *reinterpret_cast<uint4*>(dst) = av[i];
        *reinterpret_cast<uint4*>(dst + kHalf) = bv[i];
        continue;
      }
      const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&av[i]);
      const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&bv[i]);
      uint4 ra, rb;
      __nv_bfloat162* ra2 = reinterpret_cast<__nv_bfloat162*>(&ra);
      __nv_bfloat162* rb2 = reinterpret_cast<__nv_bfloat162*>(&rb);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 a = __bfloat1622float2(a2[q]), b = __bfloat1622float2(b2[q]);
        const float c0 = cs[2 * q], s0 = sn[2 * q], c1 = cs[2 * q + 1], s1 = sn[2 * q + 1];
        ra2[q] = __floats2bfloat162_rn(a.x * c0 - b.x * s0, a.y * c1 - b.y * s1);
        rb2[q] = __floats2bfloat162_rn(b.x * c0 + a.x * s0, b.y * c1 + a.y * s1);
      }
      *reinterpret_cast<uint4*>(dst) = ra;
      *reinterpret_cast<uint4*>(dst + kHalf) = rb;
    }
  }
}

// 8 outputs per thread: two 16-byte loads (gate, up), one 16-byte store; the 64-bit integer
// divide is hoisted by iterating rows in the grid's y dimension.
__global__ void __launch_bounds__(256)
swiglu_kernel(const __nv_bfloat16* __restrict__ gu, int T, int ff, __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  const int vec_per_row = ff / 8;
  for (int t = blockIdx.y; t < T; t += gridDim.y) {
    const uint4* g4 = reinterpret_cast<const uint4*>(gu + static_cast<int64_t>(t) * 2 * ff);
    const uint4* u4 = g4 + vec_per_row;
    uint4* o4 = reinterpret_cast<uint4*>(out + static_cast<int64_t>(t) * ff);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < vec_per_row; i += gridDim.x * blockDim.x) {
      const uint4 gv = g4[i], uv = u4[i];
      const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gv);
      const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&uv);
      uint4 ov;
      __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&ov);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 gf = __bfloat1622float2(g2[k]), uf = __bfloat1622float2(u2[k]);
        o2[k] = __floats2bfloat162_rn(gf.x / (1.f + __expf(-gf.x)) * uf.x,
                                      gf.y / (1.f + __expf(-gf.y)) * uf.y);
      }
      o4[i] = ov;
    }
  }
}

// Greedy argmax over the vocabulary, split across CTAs: grid (slices, rows); a CTA reduces its
// slice with 16-byte loads to one 64-bit key (orderable value << 32 | ~index: the max key is the
// first maximal index) and atomicMax-es it into keys[row]; argmax_finalize turns keys into ids.
// Values must exceed -FLT_MAX (NaN never wins); a row without one yields 0x7fffffff as before.
__device__ __forceinline__ unsigned long long argmax_key(float v, int i) {
  if (!(v > -FLT_MAX)) return 0ull;
  const uint32_t b = v == 0.f ? 0u : __float_as_uint(v);  // -0 == +0, as the float compare
  const uint32_t o = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  return (static_cast<unsigned long long>(o) << 32) | (0xFFFFFFFFu - static_cast<uint32_t>(i));
}

__global__ void __launch_bounds__(256)
argmax_slice_kernel(const float* __restrict__ logits, int V, int slice,
                    unsigned long long* __restrict__ keys) {
  const int row = blockIdx.y;
  const float* r = logits + static_cast<int64_t>(row) * V;
  const int lo = blockIdx.x * slice, hi = min(V, lo + slice);
  unsigned long long best = 0;
  if ((V & 3) == 0) {  // rows 16-byte aligned: float4 loads
    for (int i = lo + 4 * threadIdx.x; i < hi; i += 4 * blockDim.x) {
      const float4 x = *reinterpret_cast<const float4*>(r + i);
      const unsigned long long k0 = argmax_key(x.x, i), k1 = argmax_key(x.y, i + 1);
      const unsigned long long k2 = argmax_key(x.z, i + 2), k3 = argmax_key(x.w, i + 3);
      best = max(best, max(max(k0, k1), max(k2, k3)));
    }
  } else {
    for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) best = max(best, argmax_key(r[i], i));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0 && best) atomicMax(keys + row, best);
}

__global__ void argmax_finalize_kernel(const unsigned long long* __restrict__ keys, int n,
                                       int32_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long k = keys[i];
  out[i] = k ? static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(k)) : 0x7fffffff;
}

// First maximal index per row (greedy decode; ties -> lowest id like a first-max scan).
__global__ void __launch_bounds__(1024)
argmax_kernel(const float* __restrict__ logits, int V, int32_t* __restrict__ out) {
  __shared__ float sv[32];
  __shared__ int si[32];
  const float* row = logits + static_cast<int64_t>(blockIdx.x) * V;
  float best = -FLT_MAX;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    float v = row[i];
    if (v > best) {  // strided scan visits increasing i: keeps the first max of this thread
      best = v;
      bi = i;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    float ov = __shfl_xor_sync(0xffffffffu, best, o);
    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    sv[w] = best;
    si[w] = bi;
  }
  __syncthreads();
  if (w == 0) {
    best = l < static_cast<int>(blockDim.x >> 5) ? sv[l] : -FLT_MAX;
    bi = l < static_cast<int>(blockDim.x >> 5) ? si[l] : 0x7fffffff;
    for (int o = 16; o > 0; o >>= 1) {
      float ov = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) {
        best = ov;
        bi = oi;
      }
    }
    if (l == 0) out[blockIdx.x] = bi;
  }
}

// K4: one CTA per (page, slice); 16-byte vectorised, 4 loads in flight per thread.
__global__ void __launch_bounds__(256)
pool_copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, uint64_t page_vec,
                 const int32_t* __restrict__ sp, const int32_t* __restrict__ dp, int slices) {
  const int i = blockIdx.y;
  const uint64_t per = ceil_div(page_vec, slices);
  const uint64_t b = blockIdx.x * per, e = min(page_vec, b + per);
  const uint4* s = src + static_cast<uint64_t>(sp[i]) * page_vec;
  uint4* d = dst + static_cast<uint64_t>(dp[i]) * page_vec;
  uint64_t j = b + threadIdx.x;
  for (; j + 3 * 256 < e; j += 4 * 256) {
    uint4 v0 = s[j], v1 = s[j + 256], v2 = s[j + 512], v3 = s[j + 768];
    d[j] = v0;
    d[j + 256] = v1;
    d[j + 512] = v2;
    d[j + 768] = v3;
  }
  for (; j < e; j += 256) d[j] = s[j];
}

__global__ void kv_gather_kernel(PoolGeom pool, uint32_t layer, uint32_t kv,
                                 const int32_t* __restrict__ pages, __nv_bfloat16* __restrict__ out) {
  const int i = blockIdx.x;  // page index in list
  const int B = pool.block_tokens, hd = pool.head_dim, Hkv = pool.n_kv_heads;
  for (int e = threadIdx.x; e < B * Hkv * hd; e += blockDim.x) {
    const int tok = e / (Hkv * hd), h = (e / hd) % Hkv, c = e % hd;
    out[(static_cast<int64_t>(i) * B + tok) * Hkv * hd + h * hd + c] =
        pool.base[pool.tile_off(pages[i], layer, kv, h) + static_cast<int64_t>(tok) * hd + c];
  }
}

int grid_for(uint64_t n, int threads) {
  return static_cast<int>(std::min<uint64_t>(ceil_div(n, threads), kNumSMs * 32));
}

}  // namespace

void init_normal_bf16(__nv_bfloat16* p, uint64_t n, uint64_t seed, float std, cudaStream_t s) {
  init_normal_kernel<<<grid_for(n, 256), 256, 0, s>>>(p, n, seed, std);
  GLMX_CHECK_LAUNCH();
}

void init_const_bf16(__nv_bfloat16* p, uint64_t n, float v, cudaStream_t s) {
  init_const_kernel<<<grid_for(n, 256), 256, 0, s>>>(p, n, v);
  GLMX_CHECK_LAUNCH();
}

void embed_gather(const int32_t* tokens, int T, const __nv_bfloat16* embed, int d, float* x,
                  cudaStream_t s) {
  if (T <= 0) return;
  embed_kernel<<<T, 256, 0, s>>>(tokens, embed, d, x);
  GLMX_CHECK_LAUNCH();
}

void rmsnorm(const float* x, const int32_t* rows, int T, int d, const __nv_bfloat16* w,
             float eps, __nv_bfloat16* out, cudaStream_t s) {
  if (T <= 0) return;
  if (d == 4096)
    launch_pdl(rmsnorm_reg_kernel<256, 4096>, dim3(T), dim3(256), 0, s, x, rows, w, eps, out);
  else
    rmsnorm_kernel<256><<<T, 256, 0, s>>>(x, rows, d, w, eps, out);
  GLMX_CHECK_LAUNCH();
}

__global__ void rope_table_kernel(const int32_t* __restrict__ pos, int T, int half,
                                  const float* __restrict__ inv_freq, float2* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<int64_t>(T) * half) return;
  float sn, cs;
  sincosf(static_cast<float>(pos[i / half]) * inv_freq[i % half], &sn, &cs);
  out[i] = make_float2(cs, sn);
}

void rope_table(const int32_t* pos, int T, int half, const float* inv_freq, float2* out,
                cudaStream_t s) {
  if (T <= 0) return;
  const int64_t n = static_cast<int64_t>(T) * half;
  rope_table_kernel<<<static_cast<int>(ceil_div(n, 256)), 256, 0, s>>>(pos, T, half, inv_freq, out);
  GLMX_CHECK_LAUNCH();
}

void rope_kv_append(const __nv_bfloat16* qkv, const int32_t* pos, const int64_t* slot, int T,
                    int H, int Hkv, int hd, const float* inv_freq, const float2* rope_cs,
                    const PoolGeom& pool, uint32_t layer, __nv_bfloat16* q_out, cudaStream_t s) {
  if (T <= 0) return;
  if (hd > 256 || hd % 16) throw Error(GLMX_ERR_ARG, "head_dim must be a multiple of 16, <= 256");
  if (hd == 128) {
    // 3 passes (12 heads) per warp, 3 warps (tokens) per CTA: the 12 passes of a token split
    // into 4 warps (Q | Q | Q+K | K+V), so every batch size spreads over the SMs with 3 loads in
    // flight per lane.  Differential sweep with the input dirty in L2 (scripts/micro/k2_cfg.cu,
    // profiles/r2_k2_launch_shapes.txt): 450 tokens 4.1 us (was 5.1 with 1 pass x 2 warps),
    // 1536 6.6 (was 8.1 with 4 passes x 8 warps), 4096 13.3 (was 14.3), elsewhere equal.
    const int passes = static_cast<int>(ceil_div(H + 2 * Hkv, 4));
    if (!rope_cs) throw Error(GLMX_ERR_ARG, "head_dim 128 append needs the forward's RoPE table");
    constexpr int kPassU = 3, kWarps = 3;
    launch_pdl(rope_kv_append_warp_kernel<kPassU>,
               dim3(static_cast<int>(ceil_div(T, kWarps)), static_cast<int>(ceil_div(passes, kPassU))),
               dim3(kWarps * 32), 0, s, qkv, rope_cs, slot, T, H, Hkv, pool, layer, q_out);
    GLMX_CHECK_LAUNCH();
    return;
  }
  constexpr int kTok = 2, kUnroll = 3;
  rope_kv_append_kernel<kTok, kUnroll><<<static_cast<int>(ceil_div(T, kTok)), 256, 0, s>>>(
      qkv, pos, slot, T, H, Hkv, hd, inv_freq, pool, layer, q_out);
  GLMX_CHECK_LAUNCH();
}

void swiglu(const __nv_bfloat16* gu, int T, int ff, __nv_bfloat16* out, cudaStream_t s) {
  if (T <= 0) return;
  if (ff % 8) throw Error(GLMX_ERR_ARG, "d_ff must be a multiple of 8");
  const int xb = static_cast<int>(ceil_div(ff / 8, 256));
  dim3 grid(xb, std::min(T, 65535));
  launch_pdl(swiglu_kernel, grid, dim3(256), 0, s, gu, T, ff, out);
  GLMX_CHECK_LAUNCH();
}

__global__ void gather_i32_kernel(const int32_t* __restrict__ src, const int32_t* __restrict__ idx,
                                  int n, int32_t* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

__global__ void gather2_i32_kernel(const int32_t* __restrict__ a, int na, const int32_t* __restrict__ b,
                                   const int32_t* __restrict__ idx, int n, int32_t* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const int k = idx[i];
    dst[i] = k < na ? a[k] : b[k - na];
  }
}

void gather2_i32(const int32_t* a, int na, const int32_t* b, const int32_t* idx, int n, int32_t* dst,
                 cudaStream_t s) {
  if (n <= 0) return;
  gather2_i32_kernel<<<static_cast<int>(ceil_div(n, 256)), 256, 0, s>>>(a, na, b, idx, n, dst);
  GLMX_CHECK_LAUNCH();
}

void gather_i32(const int32_t* src, const int32_t* idx, int n, int32_t* dst, cudaStream_t s) {
  if (n <= 0) return;
  gather_i32_kernel<<<static_cast<int>(ceil_div(n, 256)), 256, 0, s>>>(src, idx, n, dst);
  GLMX_CHECK_LAUNCH();
}

void argmax_rows(const float* logits, int n, int V, int32_t* out, void* keys, cudaStream_t s) {
  if (n <= 0) return;
  if (!keys) {  // one CTA per row
    argmax_kernel<<<n, 1024, 0, s>>>(logits, V, out);
    GLMX_CHECK_LAUNCH();
    return;
  }
  // ~2 CTAs per SM over all rows, slices a multiple of 1024 elements
  const int slices = std::max(1, std::min(static_cast<int>(ceil_div(V, 1024)),
                                          static_cast<int>(ceil_div(2 * kNumSMs, n))));
  const int slice = static_cast<int>(ceil_div(ceil_div(V, slices), 1024) * 1024);
  unsigned long long* k = static_cast<unsigned long long*>(keys);
  GLMX_CUDA(cudaMemsetAsync(k, 0, static_cast<size_t>(n) * 8, s));
  argmax_slice_kernel<<<dim3(static_cast<int>(ceil_div(V, slice)), n), 256, 0, s>>>(logits, V, slice, k);
  GLMX_CHECK_LAUNCH();
  argmax_finalize_kernel<<<static_cast<int>(ceil_div(n, 256)), 256, 0, s>>>(k, n, out);
  GLMX_CHECK_LAUNCH();
}

void pool_copy_pages(const __nv_bfloat16* src_base, __nv_bfloat16* dst_base, uint64_t page_elems,
                     const int32_t* src_pages, const int32_t* dst_pages, int n, cudaStream_t s) {
  if (n <= 0) return;
  const uint64_t page_vec = page_elems * sizeof(__nv_bfloat16) / sizeof(uint4);
  const int slices = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(64, page_vec / 4096)));
  dim3 grid(slices, n);
  pool_copy_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<const uint4*>(src_base),
                                        reinterpret_cast<uint4*>(dst_base), page_vec, src_pages,
                                        dst_pages, slices);
  GLMX_CHECK_LAUNCH();
}

void kv_gather(const PoolGeom& pool, uint32_t layer, uint32_t kv, const int32_t* pages, int n,
               __nv_bfloat16* out, cudaStream_t s) {
  if (n <= 0) return;
  kv_gather_kernel<<<n, 256, 0, s>>>(pool, layer, kv, pages, out);
  GLMX_CHECK_LAUNCH();
}

}  // namespace glmx
