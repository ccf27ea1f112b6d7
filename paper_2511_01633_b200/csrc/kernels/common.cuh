// Device-side helpers shared by the sm_100a kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>

#include "../host/common.hpp"

#define GLMX_CUDA(call)                                                                      \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      throw ::glmx::Error(GLMX_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define GLMX_CHECK_LAUNCH() GLMX_CUDA(cudaGetLastError())

namespace glmx {

// Programmatic dependent launch: a kernel that reads its predecessor's output is launched with
// programmatic stream serialization so its grid is set up (and its CTAs fill SMs as the
// predecessor's last CTAs retire) before the predecessor has finished; pdl_wait() at the kernel's
// top blocks until the predecessor grid has completed and its writes are visible.  A kernel
// launched without the attribute passes pdl_wait() at once.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  GLMX_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}


constexpr int kNumSMs = 148;

__host__ __device__ inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

__device__ __forceinline__ bool dev_is_space(unsigned char c) {
  return c == ' ' || (c >= '\t' && c <= '\r');
}

__device__ __forceinline__ uint64_t dev_fnv1a(const char* p, uint32_t n,
                                              uint64_t h = 14695981039346656037ULL) {
  for (uint32_t i = 0; i < n; ++i) {
    h ^= static_cast<unsigned char>(p[i]);
    h *= 1099511628211ULL;
  }
  return h;
}

// Deterministic counter-based normal sample (weights init): splitmix64 -> Box-Muller.
__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

}  // namespace glmx
