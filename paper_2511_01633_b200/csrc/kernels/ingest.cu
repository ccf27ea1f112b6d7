// Graph ingest on the GPU (build_indexes, graph_store.cpp:108-124, and the
// neighbour sets of Retriever::node_info, retriever.cpp:79-105): from the edge list (node indices
// in id order + edge type) build, with cub radix sorts,
//   * the undirected and the out-only neighbour CSRs, de-duplicated and ascending,
//   * total_degree (every edge counts once at each endpoint),
//   * the by-edge-type weight: per node the largest count of incident edges of one type.
// Same arrays as HostGraph's host build, bit for bit; the K1 kernels read them in place.
#include <cub/cub.cuh>

#include "common.cuh"
#include "ingest.cuh"

namespace glmx {

namespace {

__global__ void pair_keys_kernel(const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                                 uint64_t E, uint64_t* __restrict__ und, uint64_t* __restrict__ dir,
                                 uint64_t* __restrict__ typ, const int32_t* __restrict__ etype) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < E;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t u = static_cast<uint32_t>(src[e]), v = static_cast<uint32_t>(dst[e]);
    und[2 * e] = (u << 32) | v;
    und[2 * e + 1] = (v << 32) | u;
    dir[e] = (u << 32) | v;
    typ[2 * e] = (u << 24) | static_cast<uint32_t>(etype[e]);
    typ[2 * e + 1] = (v << 24) | static_cast<uint32_t>(etype[e]);
  }
}

__global__ void csr_fill_kernel(const uint64_t* __restrict__ keys, const int* __restrict__ n_keys,
                                uint32_t* __restrict__ count, int32_t* __restrict__ idx) {
  const int n = *n_keys;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    atomicAdd(count + (keys[i] >> 32), 1u);
    idx[i] = static_cast<int32_t>(keys[i] & 0xFFFFFFFFu);
  }
}

__global__ void degree_kernel(const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                              uint64_t E, int32_t* __restrict__ w) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < E;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    atomicAdd(w + src[e], 1);
    atomicAdd(w + dst[e], 1);
  }
}

__global__ void type_max_kernel(const uint64_t* __restrict__ keys, const int* __restrict__ runs,
                                const int* __restrict__ n_runs, int32_t* __restrict__ w) {
  const int n = *n_runs;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    atomicMax(w + (keys[i] >> 24), runs[i]);
}

int grid_of(uint64_t n) { return static_cast<int>(std::min<uint64_t>(ceil_div(std::max<uint64_t>(n, 1), 256), kNumSMs * 16)); }

}  // namespace

void build_graph_device(const int32_t* h_src, const int32_t* h_dst, const int32_t* h_etype,
                        uint64_t E, uint32_t N, DeviceCsr& out, std::vector<int32_t>& w_total_host,
                        cudaStream_t s) {
  auto dalloc = [&](size_t bytes) {
    void* p = nullptr;
    GLMX_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
    out.allocs.push_back(p);
    return p;
  };
  std::vector<void*> tmp;
  auto talloc = [&](size_t bytes) {
    void* p = nullptr;
    GLMX_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
    tmp.push_back(p);
    return p;
  };
  try {
    int32_t* src = static_cast<int32_t*>(talloc(E * 4));
    int32_t* dst = static_cast<int32_t*>(talloc(E * 4));
    int32_t* et = static_cast<int32_t*>(talloc(E * 4));
    if (E) {
      GLMX_CUDA(cudaMemcpyAsync(src, h_src, E * 4, cudaMemcpyHostToDevice, s));
      GLMX_CUDA(cudaMemcpyAsync(dst, h_dst, E * 4, cudaMemcpyHostToDevice, s));
      GLMX_CUDA(cudaMemcpyAsync(et, h_etype, E * 4, cudaMemcpyHostToDevice, s));
    }
    uint64_t* und = static_cast<uint64_t*>(talloc(2 * E * 8));
    uint64_t* dir = static_cast<uint64_t*>(talloc(E * 8));
    uint64_t* typ = static_cast<uint64_t*>(talloc(2 * E * 8));
    uint64_t* sorted = static_cast<uint64_t*>(talloc(2 * E * 8));
    uint64_t* uniq = static_cast<uint64_t*>(talloc(2 * E * 8));
    int* d_n = static_cast<int*>(talloc(16));
    int* runs = static_cast<int*>(talloc(2 * E * 4));
    if (E) pair_keys_kernel<<<grid_of(E), 256, 0, s>>>(src, dst, E, und, dir, typ, et);
    GLMX_CHECK_LAUNCH();
    size_t need = 0, t = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, t, und, sorted, static_cast<int>(2 * E));
    need = std::max(need, t);
    cub::DeviceSelect::Unique(nullptr, t, sorted, uniq, d_n, static_cast<int>(2 * E));
    need = std::max(need, t);
    cub::DeviceRunLengthEncode::Encode(nullptr, t, sorted, uniq, runs, d_n, static_cast<int>(2 * E));
    need = std::max(need, t);
    cub::DeviceScan::ExclusiveSum(nullptr, t, static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                  static_cast<int>(N + 1));
    need = std::max(need, t);
    void* temp = talloc(need);
    // neighbour CSR (undirected or out-only) from one key array of n pairs
    auto csr = [&](uint64_t* keys, uint64_t n, const uint32_t*& off_out, const int32_t*& idx_out) {
      size_t tb = need;
      GLMX_CUDA(cub::DeviceRadixSort::SortKeys(temp, tb, keys, sorted, static_cast<int>(n), 0, 64, s));
      tb = need;
      GLMX_CUDA(cub::DeviceSelect::Unique(temp, tb, sorted, uniq, d_n, static_cast<int>(n), s));
      int n_uniq = 0;
      GLMX_CUDA(cudaMemcpyAsync(&n_uniq, d_n, 4, cudaMemcpyDeviceToHost, s));
      GLMX_CUDA(cudaStreamSynchronize(s));
      uint32_t* count = static_cast<uint32_t*>(talloc((N + 1) * 4));
      uint32_t* off = static_cast<uint32_t*>(dalloc((N + 1) * 4));
      int32_t* idx = static_cast<int32_t*>(dalloc(static_cast<size_t>(n_uniq) * 4));
      GLMX_CUDA(cudaMemsetAsync(count, 0, (N + 1) * 4, s));
      if (n_uniq) csr_fill_kernel<<<grid_of(n_uniq), 256, 0, s>>>(uniq, d_n, count, idx);
      GLMX_CHECK_LAUNCH();
      tb = need;
      GLMX_CUDA(cub::DeviceScan::ExclusiveSum(temp, tb, count, off, static_cast<int>(N + 1), s));
      off_out = off;
      idx_out = idx;
    };
    csr(und, 2 * E, out.und_off, out.und_idx);
    csr(dir, E, out.dir_off, out.dir_idx);
    // total degree
    int32_t* wt = static_cast<int32_t*>(dalloc(N * 4));
    GLMX_CUDA(cudaMemsetAsync(wt, 0, N * 4, s));
    if (E) degree_kernel<<<grid_of(E), 256, 0, s>>>(src, dst, E, wt);
    GLMX_CHECK_LAUNCH();
    out.w_total = wt;
    // by edge type: runs of equal (node, type) keys; per node the longest run
    int32_t* wb = static_cast<int32_t*>(dalloc(N * 4));
    GLMX_CUDA(cudaMemsetAsync(wb, 0, N * 4, s));
    if (E) {
      size_t tb = need;
      GLMX_CUDA(cub::DeviceRadixSort::SortKeys(temp, tb, typ, sorted, static_cast<int>(2 * E), 0, 64, s));
      tb = need;
      GLMX_CUDA(cub::DeviceRunLengthEncode::Encode(temp, tb, sorted, uniq, runs, d_n, static_cast<int>(2 * E), s));
      type_max_kernel<<<grid_of(2 * E), 256, 0, s>>>(uniq, runs, d_n, wb);
      GLMX_CHECK_LAUNCH();
    }
    out.w_by_type = wb;
    w_total_host.resize(N);
    GLMX_CUDA(cudaMemcpyAsync(w_total_host.data(), wt, N * 4, cudaMemcpyDeviceToHost, s));
    GLMX_CUDA(cudaStreamSynchronize(s));
  } catch (...) {
    for (void* p : tmp) cudaFree(p);
    throw;
  }
  for (void* p : tmp) cudaFree(p);
}

}  // namespace glmx
