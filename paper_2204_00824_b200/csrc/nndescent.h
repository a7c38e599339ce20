// Host interface of the GPU nn_descent (nndescent.cu, its own translation unit).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace tsdg_dev {

constexpr uint32_t kNdMaxK = 128;  // GPU limit on the list width k

struct NnDescentStats {
    uint64_t offers;    // pool offers that passed the chunk-start filter
    uint64_t chunks;    // local-join chunks merged
    uint64_t reruns;    // chunks re-run smaller (offer buffer full)
    uint64_t launches;  // kernels launched
};

// tsdg::nn_descent (knn_graph.cpp:141-251) on device rows d_vec (n x ld floats, ld a
// multiple of 4, zero padded), k = the clamped k_eff (2 <= n, 1 <= k <= min(n-1, 128)),
// max_sample = max(1, round(sample_rate * k)).  Writes n x k (ids, dists) ascending by
// (dist, id) into d_ids / d_dists.  Synchronous on `st`; throws std::runtime_error on a
// CUDA error.
void nn_descent_device(const float* d_vec, uint32_t n, uint32_t d, uint32_t ld, uint32_t k,
                       int metric, uint32_t iterations, uint32_t max_sample, uint64_t seed,
                       uint32_t* d_ids, float* d_dists, cudaStream_t st, NnDescentStats* stats);

}  // namespace tsdg_dev
