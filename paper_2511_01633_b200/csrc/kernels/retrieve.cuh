// K5 — exact nearest-neighbour scan of RetrieveNode (index.cpp:41-56) on the GPU.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace glmx {

// best[q] must be zeroed; after the call best[q] = (orderable(score) << 32) | ~row of the
// top-1 row for query q (cosine descending, ties to the lowest row = lowest id).
void nearest_top1(const float* emb, int n_rows, int dpad, const float* queries, int n_q,
                  unsigned long long* best, cudaStream_t s);

}  // namespace glmx
