// TMA row gathers on sm_100a: 32 random 512-byte rows of a 1M x 128 fp32 table into
// shared memory slots of 132 floats (the kernels' conflict-free pitch), issued as
//   (a) 32 one-row bulk copies (cp.async.bulk, one per lane; what the kernels do), or
//   (b) 8 tile::gather4 tensor copies (4 rows each, box {132, 1}: columns 128..131
//       are out of bounds and zero-filled, which yields the padded pitch).  The
//       destination of a tensor copy must be 128-byte aligned, so 4-row groups sit
//       at a 2176-byte stride (17 x 128) — (a)'s 528-byte slot layout is rejected
//       with "misaligned address".
// Checks the staged bytes and reports cycles from issue to mbarrier completion
// (median over CTAs; one CTA per SM, 8 rounds each, L2-cold rows).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/bin/gather4_probe tools/micro/gather4_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

constexpr int N = 1 << 20, D = 128, P = 132, G = 544, ROUNDS = 8;  // G: floats per 4-row group

__device__ __forceinline__ int slot_off(int mode, int s) { return mode == 0 ? s * P : (s >> 2) * G + (s & 3) * P; }

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void probe(const float* __restrict__ vec, const __grid_constant__ CUtensorMap tm,
                      const uint32_t* __restrict__ ids, unsigned long long* cyc, int* bad, uint32_t shift) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
    float* st = reinterpret_cast<float*>(sm + 128 + shift);
    const int lane = threadIdx.x;
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    uint32_t parity = 0;
    unsigned long long total = 0;
    for (int r = 0; r < ROUNDS; ++r) {
        const uint32_t e = ids[(blockIdx.x * ROUNDS + r) * 32 + lane];
        __syncwarp();
        const unsigned long long t0 = clock64();
        if (MODE == 0) {
            if (lane == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar)), "r"(32 * D * 4) : "memory");
            __syncwarp();
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(sa(st + lane * P)), "l"(vec + (size_t)e * D), "r"(D * 4), "r"(sa(bar)) : "memory");
        } else {
            if (lane == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar)), "r"(32 * P * 4) : "memory");
            __syncwarp();
            const uint32_t e0 = __shfl_sync(~0u, e, lane), e1 = __shfl_sync(~0u, e, lane + 1),
                           e2 = __shfl_sync(~0u, e, lane + 2), e3 = __shfl_sync(~0u, e, lane + 3);
            if ((lane & 3) == 0)
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                             " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
                             ::"r"(sa(st + slot_off(1, lane))), "l"(&tm), "r"(sa(bar)), "r"(0), "r"(e0), "r"(e1), "r"(e2), "r"(e3)
                             : "memory");
        }
        asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}"
                     ::"r"(sa(bar)), "r"(parity) : "memory");
        parity ^= 1u;
        total += clock64() - t0;
        // check row `lane`
        for (int j = 0; j < D; ++j)
            if (st[slot_off(MODE, lane) + j] != vec[(size_t)e * D + j]) atomicAdd(bad, 1);
        if (MODE == 1)
            for (int j = D; j < P; ++j)
                if (st[slot_off(MODE, lane) + j] != 0.0f) atomicAdd(bad, 1);
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
    }
    if (lane == 0) cyc[blockIdx.x] = total / ROUNDS;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* vec;
    cudaMalloc(&vec, (size_t)N * D * 4);
    std::vector<float> h((size_t)N * D);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (float)(i % 9973) * 0.5f + 1.0f;
    cudaMemcpy(vec, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    const int blocks = sms;
    std::vector<uint32_t> hid((size_t)blocks * ROUNDS * 32);
    uint64_t x = 88172645463325252ull;
    for (auto& v : hid) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; v = (uint32_t)(x % N); }
    uint32_t* ids;
    cudaMalloc(&ids, hid.size() * 4);
    cudaMemcpy(ids, hid.data(), hid.size() * 4, cudaMemcpyHostToDevice);
    unsigned long long* cyc;
    int* bad;
    cudaMalloc(&cyc, blocks * 8);
    cudaMalloc(&bad, 4);

    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    CUtensorMap tm;
    cuuint64_t gdim[2] = {D, N}, gstr[1] = {D * 4};
    cuuint32_t box[2] = {P, 1}, es[2] = {1, 1};
    CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, vec, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("{\"encode\": %d}\n", (int)cr);
    const size_t smem = 128 + 256 + 8 * G * 4;
    for (int mode = 0; mode < 2; ++mode) {
        for (uint32_t shift : {0u, 128u}) {
            auto k = mode == 0 ? probe<0> : probe<1>;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaMemset(bad, 0, 4);
            // flush L2 between runs by touching other rows is not needed: ids differ per run
            for (int rep = 0; rep < 2; ++rep) k<<<blocks, 32, smem>>>(vec, tm, ids, cyc, bad, shift);
            cudaError_t e = cudaDeviceSynchronize();
            std::vector<unsigned long long> hc(blocks);
            cudaMemcpy(hc.data(), cyc, blocks * 8, cudaMemcpyDeviceToHost);
            int hb = -1;
            cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
            std::sort(hc.begin(), hc.end());
            printf("{\"mode\": \"%s\", \"smem_shift\": %u, \"err\": \"%s\", \"bad\": %d, \"cycles_median\": %llu}\n",
                   mode == 0 ? "32 x cp.async.bulk" : "8 x gather4", shift, cudaGetErrorString(e), hb, hc[blocks / 2]);
            if (e != cudaSuccess) return 1;
        }
    }
    return 0;
}
