// cuBLASLt algorithm sweep for the decode GEMMs: Y[n][N] = X[n][K] W[N][K]^T (column-major
// C(N x n) = W^T' X), bf16 in, fp32 accumulate, bf16 or fp32 (beta = 1) out.  Prints every
// heuristic candidate's median time (algo -1 = cublasGemmEx); nvcc -O3 -arch=sm_100a lt_tune.cu -lcublasLt -lcublas -o lt_tune [prefill]
#include <cublas_v2.h>
#include <cublasLt.h>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <cuda_bf16.h>
#include <cstdio>
#include <vector>

#define CK(x) do { auto r = (x); if ((int)r) { printf("err %d line %d\n", (int)r, __LINE__); return 1; } } while (0)

static cublasHandle_t g_blas;

// random operands: all-zero inputs draw far less power and overstate throughput under the cap
__global__ void fill_rand(__nv_bfloat16* p, size_t n, unsigned seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned h = (unsigned)i * 2654435761u ^ seed;
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
    p[i] = __float2bfloat16(((h & 0xffff) / 32768.f - 1.f) * 0.05f);
  }
}

int run(cublasLtHandle_t lt, int n, int K, int N, bool acc, void* ws, size_t ws_bytes) {
  __nv_bfloat16 *W, *X; void* Y;
  CK(cudaMalloc(&W, (size_t)N * K * 2)); CK(cudaMalloc(&X, (size_t)n * K * 2));
  CK(cudaMalloc(&Y, (size_t)n * N * 4));
  fill_rand<<<1184, 256>>>(W, (size_t)N * K, 1u); fill_rand<<<1184, 256>>>(X, (size_t)n * K, 2u); cudaMemset(Y, 0, (size_t)n * N * 4);
  cublasLtMatmulDesc_t op; CK(cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F));
  cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
  CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta)));
  CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb)));
  cublasLtMatrixLayout_t a, b, c;
  CK(cublasLtMatrixLayoutCreate(&a, CUDA_R_16BF, K, N, K));
  CK(cublasLtMatrixLayoutCreate(&b, CUDA_R_16BF, K, n, K));
  CK(cublasLtMatrixLayoutCreate(&c, acc ? CUDA_R_32F : CUDA_R_16BF, N, n, N));
  cublasLtMatmulPreference_t pref; CK(cublasLtMatmulPreferenceCreate(&pref));
  CK(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &ws_bytes, sizeof(ws_bytes)));
  cublasLtMatmulHeuristicResult_t res[32]; int got = 0;
  CK(cublasLtMatmulAlgoGetHeuristic(lt, op, a, b, c, c, pref, 32, res, &got));
  float alpha = 1.f, beta = acc ? 1.f : 0.f;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  // candidate -1 is what the engine calls (runtime.cpp gemm: cublasGemmEx, default heuristic);
  // rounds interleave the candidates so power-cap drift hits all of them alike; median of rounds
  auto launch = [&](int i) {
    if (i < 0)
      cublasGemmEx(g_blas, CUBLAS_OP_T, CUBLAS_OP_N, N, n, K, &alpha, W, CUDA_R_16BF, K, X, CUDA_R_16BF, K,
                   &beta, Y, acc ? CUDA_R_32F : CUDA_R_16BF, N, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
    else
      cublasLtMatmul(lt, op, &alpha, W, a, X, b, &beta, Y, c, Y, c, &res[i].algo, ws, ws_bytes, 0);
  };
  const int kRounds = 7, kIters = 10;
  std::vector<std::vector<float>> t(got + 1);
  for (int r = 0; r < kRounds; ++r)
    for (int i = -1; i < got; ++i) {
      for (int w = 0; w < 2; ++w) launch(i);
      cudaEventRecord(e0);
      for (int w = 0; w < kIters; ++w) launch(i);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      t[i + 1].push_back(ms / kIters);
    }
  for (int i = -1; i < got; ++i) {
    auto v = t[i + 1]; std::sort(v.begin(), v.end()); float ms = v[v.size() / 2];
    int tile = 0, cta = 0, splitk = 0;
    if (i >= 0) {
      cublasLtMatmulAlgoConfigGetAttribute(&res[i].algo, CUBLASLT_ALGO_CONFIG_TILE_ID, &tile, sizeof(tile), nullptr);
      cublasLtMatmulAlgoConfigGetAttribute(&res[i].algo, CUBLASLT_ALGO_CONFIG_CLUSTER_SHAPE_ID, &cta, sizeof(cta), nullptr);
      cublasLtMatmulAlgoConfigGetAttribute(&res[i].algo, CUBLASLT_ALGO_CONFIG_SPLITK_NUM, &splitk, sizeof(splitk), nullptr);
    }
    printf("{\"n\": %d, \"K\": %d, \"N\": %d, \"acc\": %d, \"algo\": %d, \"tile\": %d, \"cluster\": %d, \"splitk\": %d, \"ms\": %.5f, \"gbs\": %.0f, \"tflops\": %.1f}\n",
           n, K, N, (int)acc, i, tile, cta, splitk, ms, (double)N * K * 2 / ms / 1e6, 2.0 * n * N * K / ms / 1e9);
  }
  cudaFree(W); cudaFree(X); cudaFree(Y);
  return 0;
}

int main(int argc, char** argv) {
  cublasLtHandle_t lt; cublasLtCreate(&lt);
  cublasCreate(&g_blas);
  size_t ws_bytes = 64ull << 20; void* ws; cudaMalloc(&ws, ws_bytes);
  int shapes[4][3] = {{4096, 6144, 0}, {4096, 4096, 1}, {4096, 28672, 0}, {14336, 4096, 1}};
  cublasSetWorkspace(g_blas, ws, ws_bytes);
  std::vector<int> ns = {64, 8};
  if (argc > 1 && !strcmp(argv[1], "prefill"))  // the C2 forwards' batch token counts
    ns = {384, 466, 525, 636, 764, 5841, 5885, 7763, 8194};
  for (int n : ns)
    for (auto& s : shapes) run(lt, n, s[0], s[1], s[2] != 0, ws, ws_bytes);
  return 0;
}
