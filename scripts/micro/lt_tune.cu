// cuBLASLt algorithm sweep for the decode GEMMs: Y[n][N] = X[n][K] W[N][K]^T (column-major
// C(N x n) = W^T' X), bf16 in, fp32 accumulate, bf16 or fp32 (beta = 1) out.  Prints every
// heuristic candidate's mean time; nvcc -O3 -arch=sm_100a lt_tune.cu -lcublasLt -o lt_tune
#include <cublasLt.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <vector>

#define CK(x) do { auto r = (x); if ((int)r) { printf("err %d line %d\n", (int)r, __LINE__); return 1; } } while (0)

int run(cublasLtHandle_t lt, int n, int K, int N, bool acc, void* ws, size_t ws_bytes) {
  __nv_bfloat16 *W, *X; void* Y;
  CK(cudaMalloc(&W, (size_t)N * K * 2)); CK(cudaMalloc(&X, (size_t)n * K * 2));
  CK(cudaMalloc(&Y, (size_t)n * N * 4));
  cudaMemset(W, 0, (size_t)N * K * 2); cudaMemset(X, 0, (size_t)n * K * 2); cudaMemset(Y, 0, (size_t)n * N * 4);
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
  for (int i = 0; i < got; ++i) {
    for (int w = 0; w < 3; ++w)
      cublasLtMatmul(lt, op, &alpha, W, a, X, b, &beta, Y, c, Y, c, &res[i].algo, ws, ws_bytes, 0);
    cudaEventRecord(e0);
    for (int w = 0; w < 20; ++w)
      cublasLtMatmul(lt, op, &alpha, W, a, X, b, &beta, Y, c, Y, c, &res[i].algo, ws, ws_bytes, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 20;
    printf("{\"n\": %d, \"K\": %d, \"N\": %d, \"acc\": %d, \"algo\": %d, \"ms\": %.5f, \"gbs\": %.0f}\n", n, K, N, (int)acc, i, ms,
           (double)N * K * 2 / ms / 1e6);
  }
  cudaFree(W); cudaFree(X); cudaFree(Y);
  return 0;
}

int main() {
  cublasLtHandle_t lt; cublasLtCreate(&lt);
  size_t ws_bytes = 64ull << 20; void* ws; cudaMalloc(&ws, ws_bytes);
  int shapes[4][3] = {{4096, 6144, 0}, {4096, 4096, 1}, {4096, 28672, 0}, {14336, 4096, 1}};
  for (int n : {64, 8})
    for (auto& s : shapes) run(lt, n, s[0], s[1], s[2] != 0, ws, ws_bytes);
  return 0;
}
