// Micro-benchmark of warp_merge_halves (greedy.cuh): cycles per call on one warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/micro/merge_bench tools/micro/merge_bench.cu
#include <cstdio>
#include "../../paper_2204_00824_b200/csrc/greedy.cuh"
using namespace tsdg_dev;
__global__ void bench(const float* td_in, const uint32_t* ti_in, int iters, long long* out, uint32_t* sink) {
    const int lane = threadIdx.x & 31;
    float rd = __int_as_float(0x7f800000);
    uint32_t ri = kInvalid;
    unsigned acc = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int o = (it & 63) * 32;
        const float td = td_in[o + lane];
        const uint32_t ti = ti_in[o + lane];
        acc += warp_merge_halves(rd, ri, td, ti, lane) ? 1u : 0u;
    }
    long long t1 = clock64();
    if (lane == 0) { out[0] = (t1 - t0) / iters; sink[0] = acc + ri; }
}
int main() {
    const int N = 64 * 32;
    float* hd = new float[N]; uint32_t* hi = new uint32_t[N];
    uint64_t s = 12345;
    for (int i = 0; i < N; ++i) { s = s * 6364136223846793005ull + 1; hd[i] = (float)((s >> 33) % 100000) / 1000.f; hi[i] = (uint32_t)((s >> 20) % 5000); }
    float* dd; uint32_t* di; long long* dout; uint32_t* sink;
    cudaMalloc(&dd, N * 4); cudaMalloc(&di, N * 4); cudaMalloc(&dout, 8); cudaMalloc(&sink, 4);
    cudaMemcpy(dd, hd, N * 4, cudaMemcpyHostToDevice); cudaMemcpy(di, hi, N * 4, cudaMemcpyHostToDevice);
    bench<<<1, 32>>>(dd, di, 100, dout, sink);
    bench<<<1, 32>>>(dd, di, 10000, dout, sink);
    long long c; cudaMemcpy(&c, dout, 8, cudaMemcpyDeviceToHost);
    printf("{\"warp_merge_halves_cycles\": %lld}\n", c);
    // sort alone
    return 0;
}
