// Cycles per call of the pieces of warp_merge_halves (greedy.cuh), one warp.
#include <cstdio>
#include "../../paper_2204_00824_b200/csrc/greedy.cuh"
using namespace tsdg_dev;
template <int PART>
__global__ void bench(const float* td_in, const uint32_t* ti_in, int iters, long long* out, uint32_t* sink) {
    const int lane = threadIdx.x & 31;
    float rd = __int_as_float(0x7f800000);
    uint32_t ri = kInvalid;
    unsigned acc = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int o = (it & 63) * 32;
        float td = td_in[o + lane];
        uint32_t ti = ti_in[o + lane];
        if (PART == 0) { acc += warp_merge_halves(rd, ri, td, ti, lane); }
        if (PART == 1) { warp_sort32(td, ti, lane); acc += ti; }
        if (PART == 2) {  // dup loop
            bool dup = false;
#pragma unroll 8
            for (int t = 0; t < 32; ++t) dup |= __shfl_sync(kFull, ri ^ (uint32_t)it, t) == ti;
            acc += dup;
        }
        if (PART == 3) {  // fns compaction
            const unsigned vm = __ballot_sync(kFull, lane < 16 && (ti & 1u));
            const uint32_t want = 31u - (uint32_t)lane;
            const bool has = want < (uint32_t)__popc(vm);
            const int src = has ? (int)__fns(vm, 0, (int)want + 1) : 0;
            acc += __shfl_sync(kFull, ti, src);
        }
        if (PART == 4) {  // merge network
            float nd = td; uint32_t ni = ti;
#pragma unroll
            for (int j = 16; j > 0; j >>= 1) {
                const float od = __shfl_xor_sync(kFull, nd, j);
                const uint32_t oi = __shfl_xor_sync(kFull, ni, j);
                cx(nd, ni, od, oi, (lane & j) == 0);
            }
            acc += ni;
        }
    }
    long long t1 = clock64();
    if (lane == 0) { out[PART] = (t1 - t0) / iters; sink[PART] = acc + ri; }
}
int main() {
    const int N = 64 * 32;
    float* hd = new float[N]; uint32_t* hi = new uint32_t[N];
    uint64_t s = 12345;
    for (int i = 0; i < N; ++i) { s = s * 6364136223846793005ull + 1; hd[i] = (float)((s >> 33) % 100000) / 1000.f; hi[i] = (uint32_t)((s >> 20) % 5000); }
    float* dd; uint32_t* di; long long* dout; uint32_t* sink;
    cudaMalloc(&dd, N * 4); cudaMalloc(&di, N * 4); cudaMalloc(&dout, 128); cudaMalloc(&sink, 128);
    cudaMemcpy(dd, hd, N * 4, cudaMemcpyHostToDevice); cudaMemcpy(di, hi, N * 4, cudaMemcpyHostToDevice);
    bench<0><<<1, 32>>>(dd, di, 10000, dout, sink);
    bench<1><<<1, 32>>>(dd, di, 10000, dout, sink);
    bench<2><<<1, 32>>>(dd, di, 10000, dout, sink);
    bench<3><<<1, 32>>>(dd, di, 10000, dout, sink);
    bench<4><<<1, 32>>>(dd, di, 10000, dout, sink);
    long long c[5]; cudaMemcpy(c, dout, 40, cudaMemcpyDeviceToHost);
    printf("{\"merge\": %lld, \"sort32\": %lld, \"dup_loop\": %lld, \"fns_compact\": %lld, \"merge_net\": %lld}\n", c[0], c[1], c[2], c[3], c[4]);
    return 0;
}
