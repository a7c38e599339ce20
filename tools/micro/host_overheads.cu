// Host-side costs on the small-batch call path: cudaPointerGetAttributes on mapped
// pinned memory (the zero-copy alias check), an empty cluster launch + stream sync.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/bin/host_overheads tools/micro/host_overheads.cu
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __cluster_dims__(1, 1, 1) empty_kernel(int* p) {
    if (p && threadIdx.x == 1000) p[0] = 1;
}
__global__ void plain_kernel(int* p) {
    extern __shared__ int sm[];
    if (p && threadIdx.x == 1000) p[0] = sm[0];
}

// GPU time (events) of a 10-CTA x 128-thread launch: plain, with dynamic shared
// memory, as one 10-CTA cluster (non-portable size), both.
static float event_us(bool cluster, size_t smem, cudaStream_t st) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(10);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    if (cluster) {
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 10;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
    }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9f, sum = 0.0f;
    for (int i = 0; i < 220; ++i) {
        cudaEventRecord(a, st);
        cudaLaunchKernelEx(&cfg, plain_kernel, (int*)nullptr);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, a, b);
        if (i >= 20) sum += ms;
        if (ms < best) best = ms;
    }
    return sum / 200 * 1e3f;
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
    cudaFuncSetAttribute(plain_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(plain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    printf("{\"event_us_plain\": %.2f, \"event_us_smem77k\": %.2f, \"event_us_cluster10\": %.2f, "
           "\"event_us_cluster10_smem77k\": %.2f, \"err\": \"%s\"}\n",
           event_us(false, 0, st), event_us(false, 77 * 1024, st), event_us(true, 0, st),
           event_us(true, 77 * 1024, st), cudaGetErrorString(cudaGetLastError()));
    printf("{\"cudaPointerGetAttributes_us\": %.3f, \"empty_launch_plus_sync_us\": %.2f, \"launch_only_us\": %.2f}\n",
           attr_us, launch_sync_us, launch_us);
    return 0;
}
