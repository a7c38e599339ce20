// Host-side costs on the small-batch call path: cudaPointerGetAttributes on mapped
// pinned memory (the zero-copy alias check), an empty cluster launch + stream sync.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/bin/host_overheads tools/micro/host_overheads.cu
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __cluster_dims__(1, 1, 1) empty_kernel(int* p) {
    if (p && threadIdx.x == 1000) p[0] = 1;
}

int main() {
    float* h = nullptr;
    cudaHostAlloc(&h, 1 << 20, cudaHostAllocMapped);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaFree(0);
    using clk = std::chrono::steady_clock;
    const int N = 20000;
    cudaPointerAttributes a{};
    for (int i = 0; i < 100; ++i) cudaPointerGetAttributes(&a, h + (i & 255));
    auto t0 = clk::now();
    for (int i = 0; i < N; ++i) cudaPointerGetAttributes(&a, h + (i & 255));
    const double attr_us = std::chrono::duration<double, std::micro>(clk::now() - t0).count() / N;
    for (int i = 0; i < 100; ++i) empty_kernel<<<10, 128, 0, st>>>(nullptr);
    cudaStreamSynchronize(st);
    t0 = clk::now();
    for (int i = 0; i < 2000; ++i) {
        empty_kernel<<<10, 128, 0, st>>>(nullptr);
        cudaStreamSynchronize(st);
    }
    const double launch_sync_us = std::chrono::duration<double, std::micro>(clk::now() - t0).count() / 2000;
    t0 = clk::now();
    for (int i = 0; i < 2000; ++i) empty_kernel<<<10, 128, 0, st>>>(nullptr);
    const double launch_us = std::chrono::duration<double, std::micro>(clk::now() - t0).count() / 2000;
    cudaStreamSynchronize(st);
    printf("{\"cudaPointerGetAttributes_us\": %.3f, \"empty_launch_plus_sync_us\": %.2f, \"launch_only_us\": %.2f}\n",
           attr_us, launch_sync_us, launch_us);
    return 0;
}
