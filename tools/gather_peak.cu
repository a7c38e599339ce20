// Random row-gather bandwidth on this GPU: the practical ceiling of the search
// kernels' memory traffic (rows of `row_bytes` at uniformly random row ids of an
// n-row table, no reuse beyond what L2 catches by chance).  Development tool.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_peak tools/gather_peak.cu
//   ./gather_peak [n_rows=1000000] [row_bytes=512]
//
// Variants: (a) LDG.128 per lane, 8 rows in flight per warp, max occupancy;
//           (b) TMA 1-D bulk copies of whole rows into shared memory, 16 rows per
//               mbarrier round per warp (the best-first kernel's staging pattern).
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

__global__ void gather_ldg(const float4* __restrict__ tab, uint32_t n, uint32_t vec_per_row,
                           uint32_t iters, float* sink) {
    const uint32_t lane = threadIdx.x & 31, gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    float4 acc = make_float4(0, 0, 0, 0);
    for (uint32_t it = 0; it < iters; ++it) {
        float4 v[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const uint32_t row = hash32(gw * 7919u + it * 8u + r) % n;
            v[r] = lane < vec_per_row ? __ldg(tab + (size_t)row * vec_per_row + lane) : make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) { acc.x += v[r].x; acc.y += v[r].y; acc.z += v[r].z; acc.w += v[r].w; }
    }
    if (acc.x == 12345.f) sink[0] = acc.y + acc.z + acc.w;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void gather_tma(const char* __restrict__ tab, uint32_t n, uint32_t row_bytes,
                           uint32_t iters, float* sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t pitch = row_bytes + 16;
    unsigned char* st = sm + wib * (16 * pitch + 16);
    uint64_t* bar = reinterpret_cast<uint64_t*>(st + 16 * pitch);
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    uint32_t parity = 0;
    float acc = 0;
    for (uint32_t it = 0; it < iters; ++it) {
        asm volatile("fence.proxy.async.shared::cta;");
        __syncwarp();
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                         "r"(16 * row_bytes));
        __syncwarp();
        if (lane < 16) {
            const uint32_t row = hash32(gw * 7919u + it * 16u + lane) % n;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(st + lane * pitch)),
                "l"(tab + (size_t)row * row_bytes), "r"(row_bytes), "r"(smem_u32(bar))
                : "memory");
        }
        asm volatile(
            "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                smem_u32(bar)),
            "r"(parity)
            : "memory");
        parity ^= 1;
        if (lane < 16) acc += reinterpret_cast<const float*>(st + lane * pitch)[lane];
    }
    if (acc == 12345.f) sink[0] = acc;
}

int main(int argc, char** argv) {
    const uint32_t n = argc > 1 ? (uint32_t)atoi(argv[1]) : 1000000u;
    const uint32_t row_bytes = argc > 2 ? (uint32_t)atoi(argv[2]) : 512u;
    char* tab;
    float* sink;
    cudaMalloc(&tab, (size_t)n * row_bytes);
    cudaMemset(tab, 1, (size_t)n * row_bytes);
    cudaMalloc(&sink, 4);
    char* flush;
    const size_t fb = 512ull << 20;
    cudaMalloc(&flush, fb);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    // (a) LDG
    for (int wps : {16, 32, 48, 64}) {
        const uint32_t iters = 64;
        const int threads = 256, blocks = sms * wps / 8;
        gather_ldg<<<blocks, threads>>>((const float4*)tab, n, row_bytes / 16, 4, sink);
        cudaMemset(flush, 0, fb);
        cudaEventRecord(a);
        gather_ldg<<<blocks, threads>>>((const float4*)tab, n, row_bytes / 16, iters, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = (double)blocks * (threads / 32) * iters * 8 * row_bytes;
        printf("{\"variant\": \"ldg\", \"warps_per_sm\": %d, \"GBps\": %.1f}\n", wps, bytes / ms / 1e6);
    }
    // (b) TMA rounds of 16 rows per warp
    for (int wps : {8, 16, 24}) {
        const uint32_t iters = 64;
        const int threads = 32;
        const int blocks = sms * wps;
        const size_t smem = 16 * (row_bytes + 16) + 16;
        cudaFuncSetAttribute(gather_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        gather_tma<<<blocks, threads, smem>>>(tab, n, row_bytes, 4, sink);
        cudaMemset(flush, 0, fb);
        cudaEventRecord(a);
        gather_tma<<<blocks, threads, smem>>>(tab, n, row_bytes, iters, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = (double)blocks * iters * 16 * row_bytes;
        printf("{\"variant\": \"tma16\", \"warps_per_sm\": %d, \"GBps\": %.1f, \"err\": \"%s\"}\n", wps,
               bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
