// K2 launch-shape sweep (dev tool, not part of libglmx): times rope_kv_append_warp_kernel for
// several (passes per warp, threads per CTA) shapes and batch sizes, with the QKV input written
// just before every launch (memset -> dirty lines in L2, as the QKV GEMM leaves them in the step)
// and one CUDA event pair per launch (as the engine's per-kernel breakdown times it).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2511_01633_b200/csrc -I../../include \
//        k2_cfg.cu -o /tmp/k2_cfg && /tmp/k2_cfg
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <numeric>
#include <random>
#include <vector>

#include "kernels/ops.cu"

using namespace glmx;

#define CK(x)                                                               \
  do {                                                                      \
    cudaError_t e = (x);                                                    \
    if (e != cudaSuccess) {                                                 \
      std::printf("%s: %s\n", #x, cudaGetErrorString(e));                   \
      return 1;                                                             \
    }                                                                       \
  } while (0)

#define CKA(x)                                                  \
  do {                                                          \
    if ((x) != cudaSuccess) {                                   \
      std::printf("cuda error at line %d\n", __LINE__);         \
      std::abort();                                             \
    }                                                           \
  } while (0)

template <int U>
void launch(int threads, int T, int H, int Hkv, const __nv_bfloat16* qkv, const float2* cs,
            const int64_t* slot, const PoolGeom& pool, __nv_bfloat16* q_out, cudaStream_t s) {
  const int passes = (H + 2 * Hkv + 3) / 4;
  const int wpc = threads / 32;
  rope_kv_append_warp_kernel<U><<<dim3((T + wpc - 1) / wpc, (passes + U - 1) / U), threads, 0, s>>>(
      qkv, cs, slot, T, H, Hkv, pool, 3, q_out);
}

int main() {
  const int H = 32, Hkv = 8, hd = 128, L = 32, B = 16, kMaxT = 8192, kPages = 1024;
  PoolGeom pool{nullptr, L, static_cast<uint32_t>(Hkv), B, hd};
  CK(cudaMalloc(&pool.base, static_cast<size_t>(kPages) * pool.page_elems() * 2));
  __nv_bfloat16 *qkv, *q_out;
  float2* cs;
  int64_t* slot;
  CK(cudaMalloc(&qkv, static_cast<size_t>(kMaxT) * (H + 2 * Hkv) * hd * 2));
  CK(cudaMalloc(&q_out, static_cast<size_t>(kMaxT) * H * hd * 2));
  CK(cudaMalloc(&cs, static_cast<size_t>(kMaxT) * 64 * 8));
  CK(cudaMemset(cs, 0, static_cast<size_t>(kMaxT) * 64 * 8));
  std::vector<int64_t> hs(static_cast<size_t>(kPages) * B);
  std::iota(hs.begin(), hs.end(), 0);
  std::shuffle(hs.begin(), hs.end(), std::mt19937(1));
  CK(cudaMalloc(&slot, hs.size() * 8));
  CK(cudaMemcpy(slot, hs.data(), hs.size() * 8, cudaMemcpyHostToDevice));
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  struct Cfg { int u, threads; };
  const Cfg cfgs[] = {{1, 64}, {1, 128}, {1, 256}, {2, 64}, {2, 128}, {2, 256}, {4, 128}, {4, 256}, {3, 96}, {3, 192}};
  const int Ts[] = {256, 450, 768, 1024, 1536, 2048, 3072, 4096, 6144, 8192};
  // clocks up first: ~1 s of back-to-back launches
  for (int r = 0; r < 20000; ++r) launch<4>(256, 4096, H, Hkv, qkv, cs, slot, pool, q_out, s);
  CK(cudaStreamSynchronize(s));
  for (int T : Ts) {
    const double bytes = static_cast<double>(T) * (H + 2 * Hkv) * hd * 2 * 2;
    for (const Cfg& c : cfgs) {
      // differential timing (event timestamps tick in ~2 us steps on this part): one event pair
      // around `reps` x (memset + K2) minus one around `reps` x memset alone
      const int reps = 200;
      const size_t qb = static_cast<size_t>(T) * (H + 2 * Hkv) * hd * 2;
      auto run = [&](bool k2) -> float {
        CKA(cudaEventRecord(a, s));
        for (int r = 0; r < reps; ++r) {
          CKA(cudaMemsetAsync(qkv, r & 0xff, qb, s));
          if (!k2) continue;
          if (c.u == 1) launch<1>(c.threads, T, H, Hkv, qkv, cs, slot, pool, q_out, s);
          else if (c.u == 2) launch<2>(c.threads, T, H, Hkv, qkv, cs, slot, pool, q_out, s);
          else if (c.u == 3) launch<3>(c.threads, T, H, Hkv, qkv, cs, slot, pool, q_out, s);
          else launch<4>(c.threads, T, H, Hkv, qkv, cs, slot, pool, q_out, s);
        }
        CKA(cudaGetLastError());
        CKA(cudaEventRecord(b, s));
        CKA(cudaEventSynchronize(b));
        float ms = 0.f;
        CKA(cudaEventElapsedTime(&ms, a, b));
        return ms;
      };
      run(true);
      const float with = run(true), without = run(false);
      const double us = (with - without) / reps * 1e3;
      std::printf("{\"T\": %d, \"passes_per_warp\": %d, \"threads\": %d, \"us\": %.2f, \"gbs\": %.0f}\n", T,
                  c.u, c.threads, us, bytes / (us * 1e-6) / 1e9);
    }
  }
  return 0;
}
