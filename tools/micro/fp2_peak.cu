// Issue-rate probe for the packed fp32 pipe on sm_100a: independent FADD2 / FMUL2
// streams (8 accumulators per thread), scalar FADD for comparison, and the exact-scan
// inner step (SUB2 + MUL2 + ADD2 per packed pair, with and without the opaque AND
// that keeps ptxas from contracting MUL2 + ADD2 into FFMA2).  Prints lane-ops per
// SM per cycle.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp2_peak tools/micro/fp2_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;
__device__ __forceinline__ u64 add2(u64 a, u64 b) { u64 r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 sub2(u64 a, u64 b) { u64 r; asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 mul2(u64 a, u64 b) { u64 r; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 and64(u64 a, u64 b) { u64 r; asm volatile("and.b64 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }

constexpr int ITERS = 4096;

template <int MODE>
__global__ void probe(u64* out, u64 seed, u64 keep) {
    u64 acc[8], x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { acc[i] = seed * (i + 1) + threadIdx.x; x[i] = seed ^ (i * 77); }
    float s[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i] = (float)(seed + i);
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) acc[i] = add2(acc[i], x[i]);
            else if (MODE == 1) acc[i] = mul2(acc[i], x[i]);
            else if (MODE == 2) s[i] = s[i] + (float)it;
            else if (MODE == 3) { u64 d = sub2(x[i], acc[i]); acc[i] = add2(acc[i], and64(mul2(d, d), keep)); }
            else { u64 d = sub2(x[i], acc[i]); acc[i] = add2(acc[i], mul2(d, d)); }
        }
    }
    u64 r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r ^= acc[i] ^ (u64)__float_as_uint(s[i]);
    if (r == 0x1234567) out[0] = r;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    u64* out;
    cudaMalloc(&out, 8);
    const char* names[5] = {"FADD2", "FMUL2", "FADD scalar", "SUB2+MUL2+AND+ADD2 (scan step)", "SUB2+MUL2+ADD2 (contractible)"};
    // lane-ops per iteration per thread: packed = 2 per instruction
    const double ops[5] = {16, 16, 8, 48, 48};
    for (int mode = 0; mode < 5; ++mode) {
        const int blocks = sms * 8, threads = 256;
        void (*k)(u64*, u64, u64) = mode == 0 ? probe<0> : mode == 1 ? probe<1> : mode == 2 ? probe<2> : mode == 3 ? probe<3> : probe<4>;
        k<<<blocks, threads>>>(out, 3, ~0ull);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) k<<<blocks, threads>>>(out, 3, ~0ull);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double lane_ops = 5.0 * blocks * threads * (double)ITERS * ops[mode];
        const double per_s = lane_ops / (ms * 1e-3);
        printf("{\"op\": \"%s\", \"Gops\": %.1f, \"lane_ops_per_sm_clk_at_max\": %.1f}\n", names[mode],
               per_s / 1e9, per_s / sms / (clk * 1e3));
    }
    return 0;
}
