// Device helpers shared by the TSDG search kernels (sm_100a).
//
// - splitmix64 / fork: common.hpp:27-61 of the reference.  splitmix64 is a counter
//   generator, so draw i of a stream with state s is mix64(s + (i+1)*golden): the
//   32 start draws of a search (bestfirst_search.cpp:57-63, greedy_search.cpp:18-22)
//   are computed by 32 lanes at once.
// - closer(): the global (dist, id) tie rule, common.hpp:22-25.
// - exact distances: sequential fp32, one rounding per op, no FMA — the reference's
//   compiled l2_sqr/dot (vectors.hpp:36-49) is a sequential addss chain.
// - TMA 1-D bulk copies (cp.async.bulk ... mbarrier::complete_tx) for row staging.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tsdg_dev {

// Phase-cycle instrumentation (development build only: -DTSDG_PHASES builds
// libtsdg_gpu_phases.so; tools/phase_profile.py reads the counters).  Each warp
// accumulates clock64() deltas per phase into its own slot.
#ifdef TSDG_PHASES
__device__ unsigned long long g_phase[1 << 16][8];
__device__ __forceinline__ unsigned gwarp_id() { return (blockIdx.x * blockDim.x + threadIdx.x) >> 5; }
// Per-CTA event trace (globaltimer ns) for the small-batch kernels: thread 0 of CTA b
// writes slot i of g_trace[b] (tools/trace_small.py reads it).
__device__ unsigned long long g_trace[256][32];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define TR_MARK(i)                                                                      \
    {                                                                                   \
        if (threadIdx.x == 0 && blockIdx.x < 256 && (i) < 32)                           \
            tsdg_dev::g_trace[blockIdx.x][(i)] = tsdg_dev::gtimer();                    \
    }
// Per-hop, per-warp event trace of CTA 0 of the greedy cluster kernel (globaltimer):
// g_hop[warp][hop][event] (tools/hop_trace.py).
__device__ unsigned long long g_hop[4][32][8];
#define HOP_MARK(t, i)                                                                  \
    {                                                                                   \
        if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && (t) < 32 && (threadIdx.x >> 5) < 4) \
            tsdg_dev::g_hop[threadIdx.x >> 5][(t)][(i)] = tsdg_dev::gtimer();           \
    }
#define PH_DECL long long _ph = clock64();
#define PH_RESET _ph = clock64();
#define PH_MARK(i)                                                                      \
    {                                                                                   \
        const long long _n = clock64();                                                 \
        if ((threadIdx.x & 31) == 0) tsdg_dev::g_phase[tsdg_dev::gwarp_id() & 0xFFFF][i] += _n - _ph; \
        _ph = _n;                                                                       \
    }
#else
// empty statements (not nothing): `if (c) PH_MARK(i)` must not capture the next line
#define PH_DECL
#define PH_RESET
#define PH_MARK(i) {}
#define TR_MARK(i) {}
#define HOP_MARK(t, i) {}
#endif

constexpr uint32_t kInvalid = 0xFFFFFFFFu;
constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t mix64_hd(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t fork_state(uint64_t state, uint64_t index) {
    return mix64_hd(state ^ (0xD1B54A32D192ED03ULL * (index + 1)));
}
// below(n) of draw number i (0-based) of the stream whose state is s.
__device__ __forceinline__ uint32_t draw_below(uint64_t s, uint32_t i, uint32_t n) {
    return static_cast<uint32_t>(mix64(s + static_cast<uint64_t>(i + 1) * kGolden) % n);
}

__device__ __forceinline__ bool closer(float da, uint32_t ia, float db, uint32_t ib) {
    if (da != db) return da < db;
    return ia < ib;
}

// Warp arg-min by closer(); every lane gets the winner.  Two REDUX.MIN (the distance
// as an order-preserving key, -0 == +0 as in closer(); then the smallest id holding
// that distance) and one shuffle for the winner's distance bits, instead of a 5-step
// shuffle butterfly.
__device__ __forceinline__ void warp_argmin(float& d, uint32_t& id) {
    uint32_t b = __float_as_uint(d);
    if ((b << 1) == 0) b = 0;
    const uint32_t key = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    const uint32_t mk = __reduce_min_sync(kFull, key);
    const uint32_t mi = __reduce_min_sync(kFull, key == mk ? id : 0xFFFFFFFFu);
    const unsigned who = __ballot_sync(kFull, key == mk && id == mi);
    d = __shfl_sync(kFull, d, __ffs(who) - 1);
    id = mi;
}

// compare-exchange keeping min (keep_min) or max of (d,id) vs partner's
__device__ __forceinline__ void cx(float& d, uint32_t& id, float od, uint32_t oi, bool keep_min) {
    const bool other_first = closer(od, oi, d, id);
    if (keep_min == other_first) {
        d = od;
        id = oi;
    }
}

// Ascending bitonic sort of 32 keys, one per lane.
__device__ __forceinline__ void warp_sort32(float& d, uint32_t& id, int lane) {
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const float od = __shfl_xor_sync(kFull, d, j);
            const uint32_t oi = __shfl_xor_sync(kFull, id, j);
            const bool up = (lane & k) == 0;
            const bool lower = (lane & j) == 0;
            cx(d, id, od, oi, lower == up);
        }
    }
}

// ---- exact (reference-rounding) distance accumulation -----------------------
// L2: acc += (q - r)^2 ; IP/cos: acc += q * r.  Finalise with finish_exact().
template <int METRIC>
__device__ __forceinline__ float acc_exact(float acc, float q, float r) {
    if (METRIC == 0) {
        const float diff = __fsub_rn(q, r);
        return __fadd_rn(acc, __fmul_rn(diff, diff));
    } else {
        return __fadd_rn(acc, __fmul_rn(q, r));
    }
}
template <int METRIC>
__device__ __forceinline__ float finish_exact(float acc) {
    if (METRIC == 0) return acc;
    if (METRIC == 1) return __fsub_rn(1.0f, acc);
    return -acc;
}
template <int METRIC>
__device__ __forceinline__ float acc4_exact(float acc, float4 q, float4 r) {
    acc = acc_exact<METRIC>(acc, q.x, r.x);
    acc = acc_exact<METRIC>(acc, q.y, r.y);
    acc = acc_exact<METRIC>(acc, q.z, r.z);
    acc = acc_exact<METRIC>(acc, q.w, r.w);
    return acc;
}

// Sequential exact distance reading both vectors from generic memory (slow path).
template <int METRIC>
__device__ float distance_exact_generic(const float* q, const float* r, uint32_t d) {
    float acc = 0.0f;
    for (uint32_t i = 0; i < d; ++i) acc = acc_exact<METRIC>(acc, q[i], __ldg(r + i));
    return finish_exact<METRIC>(acc);
}

// ---- mbarrier + TMA bulk copy ----------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
                 : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_addr(bar);
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(a),
        "r"(parity)
        : "memory");
}
// 1-D bulk copy global -> shared, completion counted on `bar` (bytes % 16 == 0).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
        "[%3];" ::"r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
// Order this thread's prior generic-proxy smem accesses before later async-proxy
// (TMA) writes to the same buffer.
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// Bulk L2 prefetch of `bytes` (multiple of 16) starting at a 16-byte aligned address.
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// L2 prefetch hint for a global address.
__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

}  // namespace tsdg_dev
