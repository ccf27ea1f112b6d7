// Graph ingest on the GPU (kernels/ingest.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace glmx {

struct DeviceCsr {
  const uint32_t* und_off = nullptr;
  const int32_t* und_idx = nullptr;
  const uint32_t* dir_off = nullptr;
  const int32_t* dir_idx = nullptr;
  const int32_t* w_total = nullptr;
  const int32_t* w_by_type = nullptr;
  std::vector<void*> allocs;  // owned device buffers (freed by the graph)
};

// src/dst/etype: host edge arrays (node indices in id order).  Fills `out` with device arrays and
// w_total_host with the total degrees.
void build_graph_device(const int32_t* src, const int32_t* dst, const int32_t* etype, uint64_t E,
                        uint32_t N, DeviceCsr& out, std::vector<int32_t>& w_total_host,
                        cudaStream_t s);

}  // namespace glmx
