// K5 — exact nearest-neighbour scan of RetrieveNode (index.cpp:41-56) on the GPU.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace glmx {

// best[q] must be zeroed; after the call best[q] = (orderable(score) << 32) | ~row of the
// top-1 row for query q (cosine descending, ties to the lowest row = lowest id).
// packed: fp32x2 (FFMA2) arithmetic, same bits, ~2x fewer FP instructions — for the standalone
// bulk scans (workload generation); the per-rotation RetrieveNode runs beside the prefill GEMMs,
// where the denser FP work slowed them (power cap), and uses the scalar form
void nearest_top1(const float* emb, int n_rows, int dpad, const float* queries, int n_q,
                  unsigned long long* best, cudaStream_t s, bool packed = false);

}  // namespace glmx
