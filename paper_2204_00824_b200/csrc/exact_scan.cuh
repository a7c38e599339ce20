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
//   CTA = 32 queries x one split of the base rows; 128 threads, 4 warps.
//   Base tile of 128 rows, dims in chunks of 32, double-buffered: the rows go
//   straight to shared memory row-major (cp.async, 16 B per lane, coalesced), the
//   query chunk dim-major through registers.  Thread (tq, tb) owns queries
//   4tq..4tq+3 x rows tb + 16i (i < 8): 16 packed accumulators, each an even/odd
//   query pair against one row.  The row value is the scalar operand of the packed
//   SUB2 (ptxas encodes the (x, x) broadcast as an operand modifier, `R.F32`), so
//   per 4 dims a thread issues 8 + 4 LDS.128 for 192 packed FP instructions
//   (16 x (SUB2 + FFMA2-with-(-0) + ADD2) per dim, see scan_step) — three times the
//   FP work per shared-memory access of the round-1 layout, which was bound by its
//   barriers and LSU, and no ALU-pipe masking.
//   One barrier per chunk: the next chunk's loads are issued right after it, into
//   the buffer every thread has finished with.
//   After a tile, pairs closer than the query's current k-th (a stale, looser bound
//   is fine) are appended to the query's candidate buffer (P entries in shared
//   memory); when a buffer could overflow on the next tile its new entries are
//   sorted and merged into the sorted prefix, cut to k (scan_compact), which also
//   tightens the bound.  The split's final top-k
//   goes to global memory; splits are merged per query by merge_splits_kernel.
#pragma once

#include <cuda.h>  // CUtensorMap

#include "stage.cuh"  // f32x2 helpers, cp_async16

namespace tsdg_dev {

constexpr uint32_t kScanQT = 32;        // queries per CTA
constexpr uint32_t kScanBT = 128;       // base rows per tile (64 with 3 CTAs per SM: same C2 time, C4 2% slower)
constexpr int kScanRPT = kScanBT / 16;   // rows per thread (tb + 16 i)
constexpr int kScanMinBlocks = kScanBT == 64 ? 3 : 2;  // CTAs per SM (shared memory)
constexpr uint32_t kScanDC = 32;        // dims per chunk
constexpr uint32_t kScanThreads = 128;
constexpr uint32_t kScanRPitch = kScanDC + 4;  // floats per staged row (conflict-free LDS.128)
constexpr uint32_t kScanRowBuf = kScanBT * kScanRPitch;  // floats per row buffer
constexpr uint32_t kScanQBuf = kScanDC * kScanQT;        // floats per query buffer

constexpr uint32_t kScanSortN = 128;  // per-warp sort scratch (entries)

// Dynamic shared memory of exact_scan_kernel for candidate buffers of P entries (+
// 1 KB to align the row buffers for the 128-byte TMA swizzle, + two mbarriers).
constexpr size_t scan_smem_bytes(uint32_t P) {
    return 1024 + 2 * (size_t)(kScanRowBuf + kScanQBuf) * 4 + (size_t)kScanQT * P * 8 +
           (size_t)(kScanThreads / 32) * kScanSortN * 8 + kScanQT * 16 + 8 + 16;
}

struct ScanArgs {
    const float* base;      // n rows, stride ld_b floats (ld_b % 4 == 0, 16-byte aligned)
    const float* queries;   // nq rows, stride ld_q floats (ld_q % 4 == 0)
    uint32_t n, nq, d, ld_b, ld_q;
    uint32_t k;             // results per query
    uint32_t P;             // candidate buffer entries per query (k + BT)
    uint32_t rows_per_split;
    uint64_t self_base;     // exclude_self: query q is base row self_base + q
    int exclude_self;
    unsigned long long keep;  // all ones (host); nz = keep & sign bits, see scan_step()
    uint32_t* out_ids;      // [split][nq][k]
    float* out_dists;
};

__device__ __forceinline__ unsigned long long f2_dup(float x) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %1};" : "=l"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ unsigned long long f2_add(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
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

// Compaction of one query's candidate buffer (one warp): entries [0, sorted) are the
// sorted best-so-far (<= k), [sorted, cnt) new unsorted appends.  The new entries are
// taken in batches of up to kScanSortN: sorted in the warp's scratch (bitonic over the
// next power of 2), then merged with the sorted prefix by co-rank search, keeping the
// first min(k, .) — the same set and order as sorting the whole buffer, at a fraction
// of the cost once the prefix holds k entries and few rows pass the bound per tile.
// A batch's merge output [0, nk) never reaches the unread appends (nk <= prefix +
// batch).
__device__ __forceinline__ void scan_compact(float* dd, uint32_t* ii, uint32_t sorted, uint32_t cnt,
                                             uint32_t k, float* sd, uint32_t* si, uint32_t lane) {
    const float kInf = __int_as_float(0x7f800000);
    constexpr int kOut = (384 + 31) / 32;  // outputs per lane (k <= 384)
    for (uint32_t b0 = sorted; b0 < cnt; b0 += kScanSortN) {
        const uint32_t m = min(kScanSortN, cnt - b0);
        uint32_t M = 2;
        while (M < m) M <<= 1;
        for (uint32_t i = lane; i < M; i += 32) {
            sd[i] = i < m ? dd[b0 + i] : kInf;
            si[i] = i < m ? ii[b0 + i] : kInvalid;
        }
        __syncwarp();
        warp_sort_smem(sd, si, M, (int)lane);
        const uint32_t na = sorted, nk = min(k, na + m);
        float od[kOut];
        uint32_t oi[kOut];
#pragma unroll
        for (int t = 0; t < kOut; ++t) {
            const uint32_t o = lane + 32u * t;
            if (o >= nk) break;
            // co-rank: i entries of the prefix and o - i of the batch precede output o
            uint32_t lo = o > m ? o - m : 0u, hi = min(o, na);
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (closer(dd[mid], ii[mid], sd[o - mid - 1], si[o - mid - 1])) lo = mid + 1;
                else hi = mid;
            }
            const uint32_t j = o - lo;
            const bool from_a = j >= m || (lo < na && closer(dd[lo], ii[lo], sd[j], si[j]));
            od[t] = from_a ? dd[lo] : sd[j];
            oi[t] = from_a ? ii[lo] : si[j];
        }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < kOut; ++t) {
            const uint32_t o = lane + 32u * t;
            if (o >= nk) break;
            dd[o] = od[t];
            ii[o] = oi[t];
        }
        __syncwarp();
        sorted = nk;
    }
}

// One packed update: accumulators of the query pair qq against row value b.  The
// product is formed as fma(x, y, nz) with nz = (-0, -0) read from the kernel
// arguments: x * y + (-0) is x * y rounded once (for every x * y, signed zeros
// included), and ptxas cannot fold an addend it cannot see into the following add,
// so the reference's two roundings stay (a plain mul.rn.f32x2 feeding add.rn.f32x2
// is contracted into one FFMA2).  Three FP-pipe instructions per packed update, no
// ALU-pipe masking.
template <int METRIC>
__device__ __forceinline__ void scan_step(unsigned long long& acc, unsigned long long qq, float b,
                                          unsigned long long nz) {
    unsigned long long tt;
    if (METRIC == 0) {
        const unsigned long long df = f2_sub(qq, f2_dup(b));
        tt = f2_fma(df, df, nz);
    } else {
        tt = f2_fma(qq, f2_dup(b), nz);
    }
    acc = f2_add(acc, tt);
}

// First half of scan_step for the sweep form: L2 leaves the difference (squared in
// a second sweep), IP / cosine the finished product.
template <int METRIC>
__device__ __forceinline__ void scan_prod(unsigned long long& tt, unsigned long long qq, float b,
                                          unsigned long long nz) {
    if (METRIC == 0) tt = f2_sub(qq, f2_dup(b));
    else tt = f2_fma(qq, f2_dup(b), nz);
}

// TMA: the row chunks arrive by one 2-D tensor copy per chunk (box {32 dims, 128
// rows}, 128-byte swizzle: 16-byte unit u of row r lands at unit u ^ (r & 7), so the
// eight rows an LDS.128 phase reads sit in eight different bank groups), completion
// counted on one mbarrier per buffer — instead of 8 cp.async (and their address
// arithmetic) per thread per chunk.  Otherwise rows go by cp.async into 36-float
// rows.
template <int METRIC, bool TMA>
__global__ void __launch_bounds__(kScanThreads, kScanMinBlocks)
    exact_scan_kernel(const ScanArgs a, const __grid_constant__ CUtensorMap tm) {
    extern __shared__ __align__(16) unsigned char smem_dyn[];
    // 1024-byte aligned start (offset from the shared array itself, so that the
    // compiler keeps every access below in the shared state space)
    unsigned char* smem = smem_dyn + ((1024u - (smem_addr(smem_dyn) & 1023u)) & 1023u);
    float* rs = reinterpret_cast<float*>(smem);                                      // [2][BT][RPitch]
    float* qs = rs + 2 * kScanRowBuf;                                                // [2][DC][QT]
    float* cd = qs + 2 * kScanQBuf;                                                  // [QT][P]
    uint32_t* ci = reinterpret_cast<uint32_t*>(cd + kScanQT * a.P);                 // [QT][P]
    float* sd = reinterpret_cast<float*>(ci + kScanQT * a.P);                        // [warps][SortN]
    uint32_t* si = reinterpret_cast<uint32_t*>(sd + kScanThreads / 32 * kScanSortN);  // [warps][SortN]
    uint32_t* cnt = si + kScanThreads / 32 * kScanSortN;                             // [QT]
    uint32_t* srt = cnt + kScanQT;                                                   // [QT] sorted prefix
    float* thr_d = reinterpret_cast<float*>(srt + kScanQT);                          // [QT]
    uint32_t* thr_i = reinterpret_cast<uint32_t*>(thr_d + kScanQT);                 // [QT]
    uint64_t* bars = reinterpret_cast<uint64_t*>(thr_i + kScanQT + ((smem_addr(thr_i + kScanQT) & 7u) ? 1 : 0));  // [2]

    const float kInf = __int_as_float(0x7f800000);
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t tq = tid >> 4, tb = tid & 15u;
    const uint32_t q0 = blockIdx.x * kScanQT;
    const uint32_t r_begin = blockIdx.y * a.rows_per_split;
    const uint32_t r_end = min(a.n, r_begin + a.rows_per_split);
    if (tid < kScanQT) {
        cnt[tid] = 0;
        srt[tid] = 0;
        thr_d[tid] = kInf;
        thr_i[tid] = kInvalid;
    }
    if (TMA) {
        if (tid == 0) {
            mbar_init(&bars[0], 1);
            mbar_init(&bars[1], 1);
        }
        __syncthreads();
    }
    const unsigned long long nz = a.keep & 0x8000000080000000ull;  // (-0, -0), opaque
    const uint32_t nchunks = (a.d + kScanDC - 1) / kScanDC;
    const uint32_t ntiles = r_end > r_begin ? (r_end - r_begin + kScanBT - 1) / kScanBT : 0;
    const uint32_t steps = ntiles * nchunks;

    // step s = (tile s / nchunks, chunk s % nchunks) -> buffer s & 1
    // rows: 128 rows x 32 dims = 1024 x 16 B, 8 cp.async per thread (8 lanes per row)
    // queries: 32 x 32 dims = 256 float4, 2 per thread, through registers (lane ->
    // query, so the transposed stores are conflict-free)
    float4 rq[2];
    auto issue = [&](uint32_t s) {
        const uint32_t row0 = r_begin + (s / nchunks) * kScanBT, c0 = (s % nchunks) * kScanDC;
        float* rb = rs + (s & 1u) * kScanRowBuf;
        if (TMA) {
            if (tid == 0) {
                mbar_arrive_expect_tx(&bars[s & 1u], kScanBT * kScanDC * 4);
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_addr(rb)),
                    "l"(&tm), "r"(c0), "r"(row0), "r"(smem_addr(&bars[s & 1u]))
                    : "memory");
            }
        } else {
#pragma unroll
            for (uint32_t t = 0; t < (uint32_t)kScanRPT; ++t) {
                const uint32_t f = tid + t * kScanThreads;
                const uint32_t r = f >> 3, dim = c0 + (f & 7u) * 4;
                if (row0 + r < r_end && dim < a.ld_b)
                    cp_async16(rb + r * kScanRPitch + (f & 7u) * 4, a.base + (size_t)(row0 + r) * a.ld_b + dim);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
#pragma unroll
        for (uint32_t t = 0; t < 2; ++t) {
            const uint32_t f = tid + t * kScanThreads;
            const uint32_t q = q0 + (f & 31u), dim = c0 + (f >> 5) * 4;
            rq[t] = (q < a.nq && dim < a.ld_q)
                        ? __ldg(reinterpret_cast<const float4*>(a.queries + (size_t)q * a.ld_q + dim))
                        : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    auto store_q = [&](uint32_t s) {
        float* qb = qs + (s & 1u) * kScanQBuf;
#pragma unroll
        for (uint32_t t = 0; t < 2; ++t) {
            const uint32_t f = tid + t * kScanThreads;
            const uint32_t q = f & 31u, dim = (f >> 5) * 4;
            qb[(dim + 0) * kScanQT + q] = rq[t].x;
            qb[(dim + 1) * kScanQT + q] = rq[t].y;
            qb[(dim + 2) * kScanQT + q] = rq[t].z;
            qb[(dim + 3) * kScanQT + q] = rq[t].w;
        }
    };

    // acc[2 * i + qp]: row tb + 16 i x queries (4tq + 2qp, 4tq + 2qp + 1)
    unsigned long long acc[2 * kScanRPT];
    if (steps > 0) {
        issue(0);
        store_q(0);
    }
    for (uint32_t s = 0; s < steps; ++s) {
        const uint32_t c = s % nchunks;
        const uint32_t row0 = r_begin + (s / nchunks) * kScanBT;
        if (c == 0) {
#pragma unroll
            for (int i = 0; i < 2 * kScanRPT; ++i) acc[i] = 0ull;
        }
        if (TMA) mbar_wait(&bars[s & 1u], (s >> 1) & 1u);
        else asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();  // step s staged by all; step s - 1 consumed by all
        if (s + 1 < steps) issue(s + 1);
        // row tb + 16 i: TMA rows are kScanDC floats with the 16-byte units swizzled by
        // (row & 7) = (tb & 7); cp.async rows are kScanRPitch floats, unswizzled
        const uint32_t rp = TMA ? kScanDC : kScanRPitch, sw = TMA ? (tb & 7u) : 0u;
        const float* rb = rs + (s & 1u) * kScanRowBuf + tb * rp;
        const float* qb = qs + (s & 1u) * kScanQBuf + 4 * tq;
        const uint32_t dims = min(kScanDC, a.d - c * kScanDC);
        if (dims == kScanDC) {
#pragma unroll 2
            for (uint32_t j4 = 0; j4 < kScanDC; j4 += 4) {
                float4 bv[kScanRPT];
#pragma unroll
                for (int i = 0; i < kScanRPT; ++i)
                    bv[i] = *reinterpret_cast<const float4*>(rb + i * 16 * rp + (((j4 >> 2) ^ sw) << 2));
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const ulonglong2 qv = *reinterpret_cast<const ulonglong2*>(qb + (j4 + jj) * kScanQT);
                    // one dim in three sweeps over the 2 * RPT accumulators, so that
                    // dependent instructions sit 2 * RPT apart (the per-accumulator
                    // sub -> fma -> add chain otherwise stalls on fixed latencies)
                    unsigned long long tt[2 * kScanRPT];
#pragma unroll
                    for (int i = 0; i < kScanRPT; ++i) {
                        const float b = jj == 0 ? bv[i].x : jj == 1 ? bv[i].y : jj == 2 ? bv[i].z : bv[i].w;
                        scan_prod<METRIC>(tt[2 * i + 0], qv.x, b, nz);
                        scan_prod<METRIC>(tt[2 * i + 1], qv.y, b, nz);
                    }
                    if (METRIC == 0) {
#pragma unroll
                        for (int i = 0; i < 2 * kScanRPT; ++i) tt[i] = f2_fma(tt[i], tt[i], nz);
                    }
#pragma unroll
                    for (int i = 0; i < 2 * kScanRPT; ++i) acc[i] = f2_add(acc[i], tt[i]);
                }
            }
        } else {
            for (uint32_t j = 0; j < dims; ++j) {
                const ulonglong2 qv = *reinterpret_cast<const ulonglong2*>(qb + j * kScanQT);
#pragma unroll
                for (int i = 0; i < kScanRPT; ++i) {
                    const float b = rb[i * 16 * rp + ((((j >> 2) ^ sw) << 2) | (j & 3u))];
                    scan_step<METRIC>(acc[2 * i + 0], qv.x, b, nz);
                    scan_step<METRIC>(acc[2 * i + 1], qv.y, b, nz);
                }
            }
        }
        if (s + 1 < steps) store_q(s + 1);  // buffer (s + 1) & 1 was released at the barrier
        if (c + 1 < nchunks) continue;

        // ---- tile done: append pairs closer than the query's current bound ---------
#pragma unroll
        for (int qp = 0; qp < 2; ++qp) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t ql = 4 * tq + 2 * qp + h;
                const uint32_t q = q0 + ql;
                if (q >= a.nq) continue;
                const float td = thr_d[ql];
                const uint32_t ti = thr_i[ql];
#pragma unroll
                for (int i = 0; i < kScanRPT; ++i) {
                    const uint32_t row = row0 + tb + 16 * i;
                    if (row >= r_end) continue;
                    if (a.exclude_self && (uint64_t)row == a.self_base + q) continue;
                    const unsigned long long v = acc[2 * i + qp];
                    const float dist = finish_exact<METRIC>(h ? f2_hi(v) : f2_lo(v));
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
        const bool last = s + 1 == steps;
        for (uint32_t ql = warp; ql < kScanQT; ql += kScanThreads / 32) {
            const uint32_t cq = cnt[ql];
            if (last ? cq == srt[ql] : cq <= a.P - kScanBT) continue;
            scan_compact(cd + ql * a.P, ci + ql * a.P, srt[ql], cq, a.k, sd + warp * kScanSortN,
                         si + warp * kScanSortN, lane);
            const uint32_t kept = min(cq, a.k);
            if (lane == 0) {
                cnt[ql] = kept;
                srt[ql] = kept;
                if (kept == a.k) {
                    thr_d[ql] = cd[ql * a.P + a.k - 1];
                    thr_i[ql] = ci[ql * a.P + a.k - 1];
                }
            }
            __syncwarp();
        }
        // the next step's barrier orders these updates before the next filter
    }
    __syncthreads();

    // ---- write this split's top-k (sorted; padded with sentinels) -----------------
    for (uint32_t ql = warp; ql < kScanQT; ql += kScanThreads / 32) {
        const uint32_t q = q0 + ql;
        if (q >= a.nq) continue;
        const uint32_t cq = cnt[ql];  // sorted, <= k (every split ends with a compaction)
        const size_t o = ((size_t)blockIdx.y * a.nq + q) * a.k;
        for (uint32_t i = lane; i < a.k; i += 32) {
            const bool ok = r_end > r_begin && i < cq;
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
