// Exact top-k scan: ground truth (bench.cpp:35-57 ground_truth, reference.cpp:96-111
// ref::exact_topk) and the exhaustive k-NN graph (knn_graph.cpp:64-86
// brute_force_knn).  Both keep, per query, the k smallest (dist, id) pairs over
// every base row under the reference's total order (common.hpp:22-25), with the
// reference's distance value bit for bit: sequential fp32 accumulation in
// dimension order, one rounding per sub / mul / add, no FMA (vectors.hpp:36-49).
//
// Shape: a GEMM-like tile sweep, but exact sequential fp32 (not tensor cores): the
// answer has to equal the reference's, ties included, and a mul+add split cannot be
// expressed on tcgen05.  The packed f32x2 pipe (FADD2/FMUL2 — one rounding per
// element, so still exact) gives two pair-dims per lane per instruction.
//
//   CTA = 32 queries x one split of the base rows; 256 threads, 8 warps.
//   Base tile of 128 rows, dims in chunks of 32: the chunk is loaded to registers
//   (LDG.128, next chunk in flight while the current one is reduced) and stored
//   transposed (dim-major) in shared memory; queries the same way, each value
//   duplicated as an (x, x) pair so one LDS.128 yields two packed operands.
//   Thread (tq, tb) owns queries 2tq, 2tq+1 x rows {4tb..4tb+3, 64+4tb..64+4tb+3}:
//   8 packed accumulators (16 pair distances) whose per-dim update is 8 SUB2 +
//   8 MUL2 (L2) + 8 ADD2 (+ 16 ALU-pipe LOP3, see opaque()) for 3 LDS.128.
//   After a tile, pairs closer than the query's current k-th (a stale, looser bound
//   is fine) are appended to the query's candidate buffer (P entries in shared
//   memory); when a buffer could overflow on the next tile it is sorted (warp
//   bitonic) and cut to k, which also tightens the bound.  The split's final top-k
//   goes to global memory; splits are merged per query by merge_splits_kernel.
#pragma once

#include "stage.cuh"  // f32x2 helpers

namespace tsdg_dev {

constexpr uint32_t kScanQT = 32;        // queries per CTA
constexpr uint32_t kScanBT = 128;       // base rows per tile
constexpr uint32_t kScanDC = 32;        // dims per chunk
constexpr uint32_t kScanThreads = 256;
constexpr uint32_t kScanBPitch = kScanBT + 4;  // floats per dim row of the base tile

struct ScanArgs {
    const float* base;      // n rows, stride ld_b floats (ld_b % 4 == 0)
    const float* queries;   // nq rows, stride ld_q floats (ld_q % 4 == 0)
    uint32_t n, nq, d, ld_b, ld_q;
    uint32_t k;             // results per query
    uint32_t P;             // candidate buffer entries per query (power of 2, >= k + BT)
    uint32_t rows_per_split;
    uint64_t self_base;     // exclude_self: query q is base row self_base + q
    int exclude_self;
    unsigned long long keep;  // all ones (host); see opaque()
    uint32_t* out_ids;      // [split][nq][k]
    float* out_dists;
};

__device__ __forceinline__ unsigned long long f2_dup(float x) {
    return (unsigned long long)__float_as_uint(x) | ((unsigned long long)__float_as_uint(x) << 32);
}
__device__ __forceinline__ unsigned long long f2_add(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
// ptxas contracts a packed mul.rn.f32x2 feeding an add.rn.f32x2 into one FFMA2 (a
// single rounding: not the reference's value).  Masking the product with a value it
// cannot see (all ones, from the kernel arguments) keeps the two roundings; the two
// LOP3 run on the ALU pipe, off the FMA pipe this loop is bound by.
__device__ __forceinline__ unsigned long long opaque(unsigned long long x, unsigned long long keep) {
    unsigned long long r;
    asm("and.b64 %0, %1, %2;" : "=l"(r) : "l"(x), "l"(keep));
    return r;
}

// Ascending bitonic sort by closer() of P entries (power of 2) in shared memory, one
// warp.
__device__ __forceinline__ void warp_sort_smem(float* dd, uint32_t* ii, uint32_t P, int lane) {
    for (uint32_t size = 2; size <= P; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = lane; i < (P >> 1); i += 32) {
                const uint32_t a = 2 * i - (i & (stride - 1));
                const uint32_t b = a + stride;
                const bool asc = (a & size) == 0;
                const float da = dd[a], db = dd[b];
                const uint32_t ia = ii[a], ib = ii[b];
                if (asc ? closer(db, ib, da, ia) : closer(da, ia, db, ib)) {
                    dd[a] = db;
                    ii[a] = ib;
                    dd[b] = da;
                    ii[b] = ia;
                }
            }
            __syncwarp();
        }
    }
}

template <int METRIC>
__global__ void __launch_bounds__(kScanThreads, 2) exact_scan_kernel(const ScanArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned long long* qs = reinterpret_cast<unsigned long long*>(smem);          // [DC][QT]
    float* bs = reinterpret_cast<float*>(smem + kScanDC * kScanQT * 8);              // [DC][BPitch]
    float* cd = bs + kScanDC * kScanBPitch;                                          // [QT][P]
    uint32_t* ci = reinterpret_cast<uint32_t*>(cd + kScanQT * a.P);                 // [QT][P]
    uint32_t* cnt = ci + kScanQT * a.P;                                              // [QT]
    float* thr_d = reinterpret_cast<float*>(cnt + kScanQT);                          // [QT]
    uint32_t* thr_i = reinterpret_cast<uint32_t*>(thr_d + kScanQT);                 // [QT]

    const float kInf = __int_as_float(0x7f800000);
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t tq = tid >> 4, tb = tid & 15u;
    const uint32_t q0 = blockIdx.x * kScanQT;
    const uint32_t r_begin = blockIdx.y * a.rows_per_split;
    const uint32_t r_end = min(a.n, r_begin + a.rows_per_split);
    if (tid < kScanQT) {
        cnt[tid] = 0;
        thr_d[tid] = kInf;
        thr_i[tid] = kInvalid;
    }

    // chunk loader: base 128 rows x 32 dims = 1024 float4 (4 per thread), queries
    // 32 x 32 = 256 float4 (1 per thread)
    float4 rb[4], rq;
    auto load_chunk = [&](uint32_t row0, uint32_t c0) {
#pragma unroll
        for (uint32_t t = 0; t < 4; ++t) {
            const uint32_t f = tid + t * kScanThreads;
            const uint32_t row = row0 + (f >> 3), dim = c0 + (f & 7u) * 4;
            rb[t] = (row < r_end && dim < a.ld_b)
                        ? __ldg(reinterpret_cast<const float4*>(a.base + (size_t)row * a.ld_b + dim))
                        : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        const uint32_t q = q0 + (tid >> 3), dim = c0 + (tid & 7u) * 4;
        rq = (q < a.nq && dim < a.ld_q)
                 ? __ldg(reinterpret_cast<const float4*>(a.queries + (size_t)q * a.ld_q + dim))
                 : make_float4(0.f, 0.f, 0.f, 0.f);
    };
    auto store_chunk = [&]() {
#pragma unroll
        for (uint32_t t = 0; t < 4; ++t) {
            const uint32_t f = tid + t * kScanThreads;
            const uint32_t row = f >> 3, dim = (f & 7u) * 4;
            bs[(dim + 0) * kScanBPitch + row] = rb[t].x;
            bs[(dim + 1) * kScanBPitch + row] = rb[t].y;
            bs[(dim + 2) * kScanBPitch + row] = rb[t].z;
            bs[(dim + 3) * kScanBPitch + row] = rb[t].w;
        }
        const uint32_t q = tid >> 3, dim = (tid & 7u) * 4;
        qs[(dim + 0) * kScanQT + q] = f2_dup(rq.x);
        qs[(dim + 1) * kScanQT + q] = f2_dup(rq.y);
        qs[(dim + 2) * kScanQT + q] = f2_dup(rq.z);
        qs[(dim + 3) * kScanQT + q] = f2_dup(rq.w);
    };

    for (uint32_t row0 = r_begin; row0 < r_end; row0 += kScanBT) {
        // acc[2*qi + h*... ]: query qi (0..1) x row pair p (0..3):
        //   p=0: rows 4tb+0,1  p=1: 4tb+2,3  p=2: 64+4tb+0,1  p=3: 64+4tb+2,3
        unsigned long long acc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = 0ull;
        load_chunk(row0, 0);
        for (uint32_t c0 = 0; c0 < a.d; c0 += kScanDC) {
            __syncthreads();  // previous chunk fully consumed
            store_chunk();
            __syncthreads();
            if (c0 + kScanDC < a.d) load_chunk(row0, c0 + kScanDC);  // in flight meanwhile
            const uint32_t dims = min(kScanDC, a.d - c0);
            const unsigned long long* qp = qs + 2 * tq;
            const float* bp0 = bs + 4 * tb;
            const float* bp1 = bs + 64 + 4 * tb;
            auto step = [&](uint32_t t) {
                const ulonglong2 qv = *reinterpret_cast<const ulonglong2*>(qp + t * kScanQT);
                const ulonglong2 b0 = *reinterpret_cast<const ulonglong2*>(bp0 + t * kScanBPitch);
                const ulonglong2 b1 = *reinterpret_cast<const ulonglong2*>(bp1 + t * kScanBPitch);
                const unsigned long long bv[4] = {b0.x, b0.y, b1.x, b1.y};
                const unsigned long long qq[2] = {qv.x, qv.y};
#pragma unroll
                for (int qi = 0; qi < 2; ++qi) {
#pragma unroll
                    for (int p = 0; p < 4; ++p) {
                        unsigned long long tt;
                        if (METRIC == 0) {
                            const unsigned long long df = f2_sub(qq[qi], bv[p]);
                            tt = f2_mul(df, df);
                        } else {
                            tt = f2_mul(qq[qi], bv[p]);
                        }
                        acc[qi * 4 + p] = f2_add(acc[qi * 4 + p], opaque(tt, a.keep));
                    }
                }
            };
            if (dims == kScanDC) {
#pragma unroll 8
                for (uint32_t t = 0; t < kScanDC; ++t) step(t);
            } else {
                for (uint32_t t = 0; t < dims; ++t) step(t);
            }
        }

        // ---- filter: append pairs closer than the query's current bound ----------
#pragma unroll
        for (int qi = 0; qi < 2; ++qi) {
            const uint32_t ql = 2 * tq + qi;
            const uint32_t q = q0 + ql;
            if (q >= a.nq) continue;
            const float td = thr_d[ql];
            const uint32_t ti = thr_i[ql];
#pragma unroll
            for (int p = 0; p < 4; ++p) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t row = row0 + (p >> 1) * 64 + 4 * tb + (p & 1) * 2 + h;
                    if (row >= r_end) continue;
                    if (a.exclude_self && (uint64_t)row == a.self_base + q) continue;
                    const float acc_v = h ? f2_hi(acc[qi * 4 + p]) : f2_lo(acc[qi * 4 + p]);
                    const float dist = finish_exact<METRIC>(acc_v);
                    if (closer(dist, row, td, ti)) {
                        const uint32_t pos = atomicAdd(&cnt[ql], 1u);
                        cd[ql * a.P + pos] = dist;
                        ci[ql * a.P + pos] = row;
                    }
                }
            }
        }
        __syncthreads();
        // ---- compact buffers that could overflow on the next tile ------------------
        const bool last = row0 + kScanBT >= r_end;
        for (uint32_t ql = warp; ql < kScanQT; ql += kScanThreads / 32) {
            const uint32_t c = cnt[ql];
            if (!last && c <= a.P - kScanBT) continue;
            float* dd = cd + ql * a.P;
            uint32_t* ii = ci + ql * a.P;
            for (uint32_t i = c + lane; i < a.P; i += 32) {
                dd[i] = kInf;
                ii[i] = kInvalid;
            }
            __syncwarp();
            warp_sort_smem(dd, ii, a.P, (int)lane);
            const uint32_t kept = min(c, a.k);
            if (lane == 0) {
                cnt[ql] = kept;
                if (kept == a.k) {
                    thr_d[ql] = dd[a.k - 1];
                    thr_i[ql] = ii[a.k - 1];
                }
            }
            __syncwarp();
        }
        __syncthreads();
    }

    // ---- write this split's top-k (sorted; padded with sentinels) -----------------
    for (uint32_t ql = warp; ql < kScanQT; ql += kScanThreads / 32) {
        const uint32_t q = q0 + ql;
        if (q >= a.nq) continue;
        const uint32_t c = cnt[ql];  // sorted, <= k (every split ends with a compaction)
        const size_t o = ((size_t)blockIdx.y * a.nq + q) * a.k;
        for (uint32_t i = lane; i < a.k; i += 32) {
            const bool ok = r_end > r_begin && i < c;
            a.out_ids[o + i] = ok ? ci[ql * a.P + i] : kInvalid;
            a.out_dists[o + i] = ok ? cd[ql * a.P + i] : kInf;
        }
    }
}

// Per query, merge S sorted split lists (disjoint row ranges) into the first k by
// (dist, id).  One warp per query; lane s < S tracks list s.
static __global__ void merge_splits_kernel(const uint32_t* in_ids, const float* in_dists, uint32_t S,
                                    uint32_t nq, uint32_t k, uint32_t* out_ids, float* out_dists) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (q >= nq) return;
    const float kInf = __int_as_float(0x7f800000);
    uint32_t pos = 0;
    auto head = [&](float& d, uint32_t& i) {
        if (lane < S && pos < k) {
            const size_t o = ((size_t)lane * nq + q) * k + pos;
            d = in_dists[o];
            i = in_ids[o];
        } else {
            d = kInf;
            i = kInvalid;
        }
    };
    float hd;
    uint32_t hi;
    head(hd, hi);
    for (uint32_t r = 0; r < k; ++r) {
        float bd = hd;
        uint32_t bi = hi;
        warp_argmin(bd, bi);
        if (lane == 0) {
            out_ids[(size_t)q * k + r] = bi;
            out_dists[(size_t)q * k + r] = bd;
        }
        if (bi != kInvalid && hi == bi && hd == bd) {  // this lane's list supplied it
            ++pos;
            head(hd, hi);
        }
    }
}

}  // namespace tsdg_dev
