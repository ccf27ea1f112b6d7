// Decode GEMMs on tcgen05 (gemv_tc.cu): Y[n][N] (+)= X[n][K] . W[N][K]^T for n <= 64.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace glmx {

// TMA map over a row-major bf16 [rows][cols] matrix: box [box_rows][64] (W: 128 rows, X: 64)
void make_gemv_map(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows, void* out_map);
bool gemv_tc_supported(int n, int K, int N);
int gemv_tc_splits(int K, int N);
size_t gemv_tc_part_floats(int K, int N);  // fp32 split-partial workspace for this shape
// mode 0: bf16 store, 1: fp32 store, 2: fp32 accumulate (y += X W^T).  counters: N / 128 ints,
// zero on first use and left zero (self-resetting).
void gemv_tc(const void* w_map, const void* x_map, int n, int K, int N, int mode, void* y,
             float* part, int* counters, cudaStream_t s);

}  // namespace glmx
