// Prefill GEMM algorithm table.  The engine's four per-layer projections (QKV, O, gate/up, down)
// run through cuBLAS; cublasGemmEx's default heuristic picks a tile per (M, N, K) that, at some
// of the C2 batch sizes, quantises badly against 148 SMs (5-15% slower than the best cuBLASLt
// candidate for that shape; scripts/micro/lt_tune.cu, profiles/r1_gemm_algo_sweep.jsonl).
// GemmTuner times the cuBLASLt heuristic candidates against cublasGemmEx once per (projection,
// M bucket) — explicitly, through glmx_model_tune_gemms, while the device is otherwise idle — and
// the forward then launches the winner.  Buckets without a winner, and M above the tuned range,
// keep cublasGemmEx.  Both paths are the cuBLAS library; only the algorithm choice differs.
#pragma once

#include <cublasLt.h>
#include <cublas_v2.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <vector>

namespace glmx {

enum GemmShape { kGemmQKV = 0, kGemmO = 1, kGemmGU = 2, kGemmDown = 3, kGemmShapes = 4 };

class GemmTuner {
 public:
  GemmTuner() = default;
  GemmTuner(const GemmTuner&) = delete;
  GemmTuner& operator=(const GemmTuner&) = delete;
  ~GemmTuner();

  // M buckets: 128 wide up to 2048, 256 wide up to 16384 (aligned to the 128/256-row tiles
  // cuBLAS uses, so a bucket's tile count is that of its upper edge), 2048 wide above (tens of
  // waves: the tail wave no longer matters).
  static int bucket(int T);
  static int bucket_hi(int b);

  // Y[T][out] (+)= X[T][in] W[out][in]^T with the tuned algorithm; false = no entry (the caller
  // launches cublasGemmEx).
  bool run(int shape, cudaStream_t s, const __nv_bfloat16* X, const __nv_bfloat16* W, void* Y,
           bool y_fp32, bool acc, int T, int in, int out, void* ws, size_t ws_bytes);

  // Times cublasGemmEx and up to kCandidates cuBLASLt candidates at M = bucket_hi(b) on X/W/Y
  // (interleaved rounds, median) and records the winner if it beats cublasGemmEx by > 2%.
  // Returns 1 if an entry was recorded.
  int tune(int shape, int b, cublasHandle_t blas, cudaStream_t s, const __nv_bfloat16* X,
           const __nv_bfloat16* W, void* Y, bool y_fp32, bool acc, int in, int out, void* ws,
           size_t ws_bytes);

  int entries() const;

 private:
  static constexpr int kCandidates = 6, kMaxCandidates = 16;
  struct Entry {
    bool has = false;
    cublasLtMatmulAlgo_t algo{};
  };
  void ensure_handle();
  cublasLtHandle_t lt_ = nullptr;
  cublasLtMatmulDesc_t desc_ = nullptr;
  std::vector<Entry> table_[kGemmShapes];
};

}  // namespace glmx
