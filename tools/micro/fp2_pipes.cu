// Which fp32 pipe does each packed / scalar op use on sm_100a?  Every block runs
// 16 independent chains per thread of one op mix; lane-ops per SM per cycle come
// from clock64() around the loop (no dependence on the SM clock the GPU settles at).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/bin/fp2_pipes tools/micro/fp2_pipes.cu
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;
__device__ __forceinline__ u64 add2(u64 a, u64 b) { u64 r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 mul2(u64 a, u64 b) { u64 r; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ float add1(float a, float b) { float r; asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float fma1(float a, float b, float c) { float r; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r; }

constexpr int ITERS = 2048;

// lane-ops per thread per iteration for each mode
__host__ __device__ constexpr int ops_of(int m) {
    return m == 0 ? 32 : m == 1 ? 32 : m == 2 ? 32 : m == 3 ? 16 : m == 4 ? 16 : m == 5 ? 24 : m == 6 ? 24 : m == 10 ? 48 : 96;  // modes >= 7: 3 ops x 2 lanes x 16
}

template <int MODE>
__global__ void probe(u64* out, u64 seed, unsigned long long* cyc) {
    u64 a[16];
    float f[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) { a[i] = seed * (i + 3) + threadIdx.x; f[i] = (float)(seed + i); }
    const u64 x = seed ^ 0x3f8000003f800000ull, nz = seed & 0x8000000080000000ull;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (MODE == 0) a[i] = add2(a[i], x);                 // FADD2: 2 lane-ops
            else if (MODE == 1) a[i] = mul2(a[i], x);            // FMUL2
            else if (MODE == 2) a[i] = fma2(a[i], x, nz);        // FFMA2 (counted as 2, not 4)
            else if (MODE == 3) f[i] = add1(f[i], 1.0f);         // FADD: 1
            else if (MODE == 4) f[i] = fma1(f[i], 1.0001f, 0.5f);  // FFMA
            else if (MODE == 5) { if (i & 1) f[i] = add1(f[i], 1.0f); else a[i] = add2(a[i], x); }  // mix
            else if (MODE == 6) { if (i & 1) f[i] = fma1(f[i], 1.0001f, 0.5f); else a[i] = fma2(a[i], x, nz); }
            else if (MODE == 10) {  // all scalar: sub, fma(nz), add on one float chain (48 ops)
                float d = add1(f[i], 1.5f);
                d = fma1(d, d, __uint_as_float((unsigned)nz));
                f[i] = add1(f[i], d);
            }
            else if (MODE == 7) { u64 d = add2(a[i], x); d = fma2(d, d, nz); a[i] = add2(a[i], d); }  // scan step: 3 x 2
            else {
                // the same step with part of the work as scalar ops
                u64 d = add2(a[i], x);
                float lo = __uint_as_float((unsigned)d), hi = __uint_as_float((unsigned)(d >> 32));
                float alo = __uint_as_float((unsigned)a[i]), ahi = __uint_as_float((unsigned)(a[i] >> 32));
                const float z = __uint_as_float((unsigned)nz);
                if (MODE == 8) {  // SUB2, scalar FFMA x2, scalar FADD x2
                    lo = fma1(lo, lo, z); hi = fma1(hi, hi, z);
                    alo = add1(alo, lo); ahi = add1(ahi, hi);
                    a[i] = (u64)__float_as_uint(alo) | ((u64)__float_as_uint(ahi) << 32);
                } else {  // MODE 9: SUB2, FFMA2, scalar FADD x2
                    d = fma2(d, d, nz);
                    lo = __uint_as_float((unsigned)d); hi = __uint_as_float((unsigned)(d >> 32));
                    alo = add1(alo, lo); ahi = add1(ahi, hi);
                    a[i] = (u64)__float_as_uint(alo) | ((u64)__float_as_uint(ahi) << 32);
                }
            }
        }
    }
    const unsigned long long t1 = clock64();
    u64 r = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) r ^= a[i] ^ (u64)__float_as_uint(f[i]);
    if (r == 0x1234567) out[0] = r;
    if (threadIdx.x == 0) atomicMax(cyc, t1 - t0);
}

template <int MODE>
void run(int sms, u64* out, unsigned long long* cyc, const char* name) {
    const int per_sm = 4, threads = 256;  // 32 warps per SM
    unsigned long long zero = 0, c = 0;
    probe<MODE><<<sms * per_sm, threads>>>(out, 3, cyc);
    cudaMemcpy(cyc, &zero, 8, cudaMemcpyHostToDevice);
    probe<MODE><<<sms * per_sm, threads>>>(out, 3, cyc);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double ops = (double)per_sm * threads * ITERS * ops_of(MODE);
    printf("{\"op\": \"%s\", \"lane_ops_per_sm_per_cycle\": %.1f}\n", name, ops / (double)c);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    u64* out;
    unsigned long long* cyc;
    cudaMalloc(&out, 8);
    cudaMalloc(&cyc, 8);
    run<0>(sms, out, cyc, "FADD2");
    run<1>(sms, out, cyc, "FMUL2");
    run<2>(sms, out, cyc, "FFMA2 (2 per lane)");
    run<3>(sms, out, cyc, "FADD");
    run<4>(sms, out, cyc, "FFMA (1 per lane)");
    run<5>(sms, out, cyc, "FADD2 + FADD 1:1");
    run<6>(sms, out, cyc, "FFMA2 + FFMA 1:1");
    run<7>(sms, out, cyc, "scan step SUB2 FFMA2 ADD2");
    run<8>(sms, out, cyc, "scan step SUB2, 2 FFMA, 2 FADD");
    run<9>(sms, out, cyc, "scan step SUB2, FFMA2, 2 FADD");
    run<10>(sms, out, cyc, "scan step scalar FADD, FFMA, FADD");
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
