// Large-batch best-first search, FAST mode (paper Alg. 2) — register-direct,
// warp-cooperative distances, branch-free structure operations.
//
// Same search as bf_kernel (bestfirst.cuh): the reference's lossy C / V / R kept
// exactly (segmented.cpp:8-111), the same expansion order, admission test and
// eviction revival (bestfirst_search.cpp:73-97).  What differs is how a hop is
// executed, which is what bounds throughput (a warp's hop is a chain of dependent
// memory round trips and short-latency instructions; ncu: profiles/r2*_bf_fast_c2.md):
//
//   * no shared-memory staging, no TMA / mbarrier: the whole warp reads ONE row
//     per LDG.128 (lane l holds floats [4l, 4l+4) of each 128-float segment) into
//     registers, B rows per batch; the query sits in registers (d <= 128) or in
//     shared memory (larger d).  The row address is one IMAD.WIDE per row;
//   * each lane forms packed f32x2 partial sums (FADD2 + FMUL2/FFMA2) and the B row
//     sums are finished by a transposed butterfly (log2(B) exchange steps of B/2,
//     B/4, ... shuffles, then plain xor steps): ~1-2 shuffles per row;
//   * all edges of a hop (up to 64 per super-chunk) are classified at once — V
//     does not change during a hop and an edge can only leave C (eviction) before
//     its turn, so "in C at the hop start" plus eviction revival is exactly the
//     sequential loop's test — and every needed row is gathered in one pass before
//     the admission replay;
//   * C and V keep sentinel-filled slots (id 0xFFFFFFFF, dist +inf) instead of
//     size fields: membership is 8 LDS.128 + compares with no branches, a full
//     segment is "slot 31 is not the sentinel", the FIFO write slot of a V segment
//     is (adds to that segment) mod 32 held in lane s's register;
//   * rows past the first batch of a hop are pulled into L2 by per-lane 128-byte
//     line prefetches (row_prefetch; a bulk prefetch per row is the slower option)
//     as soon as the hop's needed set
//     is known, so only the first batch waits on DRAM (C2: 0.85 -> 0.79 ms);
//   * per-warp shared memory drops from 12.7 KB to ~4.5 KB (d = 128, m = 8).
//
// Distances use FMA and a tree order, so only recall-level parity applies (north
// star: recall@1/@10 within 0.5 pt of the reference); deterministic mode keeps the
// staged kernel.
#pragma once

#include "bestfirst.cuh"

namespace tsdg_dev {

constexpr int kFastWarps = 2;  // independent queries per CTA

__device__ __forceinline__ ulonglong2 ldg_row16(const void* p) {
    ulonglong2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0, %1}, [%2];"
                 : "=l"(r.x), "=l"(r.y)
                 : "l"(p));
    return r;
}

// Reduce B per-lane values (one per row) across the warp.  On return lane l holds
// the full sum of row `row` (the same value in groups of 32/B lanes).
template <int B>
__device__ __forceinline__ float bfly_reduce(float (&v)[B], int lane, uint32_t& row) {
    constexpr int LOG2B = B == 1 ? 0 : B == 2 ? 1 : B == 4 ? 2 : B == 8 ? 3 : B == 16 ? 4 : 5;
    row = 0;
#pragma unroll
    for (int st = 0; st < LOG2B; ++st) {
        const int off = 16 >> st;
        const int h = B >> (st + 1);
        const bool up = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < h; ++i) {
            const float send = up ? v[i] : v[i + h];
            const float keep = up ? v[i + h] : v[i];
            v[i] = keep + __shfl_xor_sync(kFull, send, off);
        }
        if (up) row += (uint32_t)h;
    }
#pragma unroll
    for (int off = 16 >> LOG2B; off > 0; off >>= 1) v[0] += __shfl_xor_sync(kFull, v[0], off);
    return v[0];
}

// First 4-float step of a row (no accumulator yet).
template <int METRIC>
__device__ __forceinline__ unsigned long long part4_first(ulonglong2 q, ulonglong2 r) {
    if (METRIC == 0) {
        const unsigned long long d01 = f2_sub(q.x, r.x), d23 = f2_sub(q.y, r.y);
        return f2_fma(d23, d23, f2_mul(d01, d01));
    }
    return f2_fma(q.y, r.y, f2_mul(q.x, r.x));
}

// Row geometry.  SEG: 1 = rows of exactly 128 floats (query piece in registers, no
// predication), 2 = rows of < 128 floats (lanes >= ld4 idle), 0 = any length
// (128-float segments, query in shared memory).
struct FastGeom {
    const char* rb;        // vec + 16 * lane
    uint32_t rowbytes;     // 4 * ld
    uint32_t ld4;          // 16-byte pieces per row
    const ulonglong2* sq;  // query in shared memory (SEG 0)
};

// Distances of the rows lst[0..cnt) -> dl[0..cnt).  lst is padded with valid ids
// to a multiple of B (pad rows are loaded and discarded).
template <int METRIC, int B, int SEG>
__device__ __forceinline__ void eval_rows(const FastGeom& g, const uint32_t* lst, float* dl,
                                          uint32_t cnt, ulonglong2 q, int lane) {
    const ulonglong2 zero = make_ulonglong2(0ull, 0ull);
    for (uint32_t t0 = 0; t0 < cnt; t0 += B) {
        uint32_t id[B];
#pragma unroll
        for (int j = 0; j < B / 4; ++j) {
            const uint4 v = reinterpret_cast<const uint4*>(lst + t0)[j];
            id[4 * j] = v.x;
            id[4 * j + 1] = v.y;
            id[4 * j + 2] = v.z;
            id[4 * j + 3] = v.w;
        }
        unsigned long long acc[B];
        if (SEG != 0) {
            const bool act = SEG == 1 || (uint32_t)lane < g.ld4;
            ulonglong2 r[B];
#pragma unroll
            for (int i = 0; i < B; ++i)
                r[i] = act ? ldg_row16(g.rb + (size_t)id[i] * g.rowbytes) : zero;
#pragma unroll
            for (int i = 0; i < B; ++i) acc[i] = part4_first<METRIC>(q, r[i]);
        } else {
#pragma unroll
            for (int i = 0; i < B; ++i) acc[i] = 0ull;
            const uint32_t nseg = (g.ld4 + 31u) >> 5;
            for (uint32_t s = 0; s < nseg; ++s) {
                const uint32_t f = s * 32u + (uint32_t)lane;
                const bool act = f < g.ld4;
                const ulonglong2 qq = act ? g.sq[f] : zero;
                ulonglong2 r[B];
#pragma unroll
                for (int i = 0; i < B; ++i)
                    r[i] = act ? ldg_row16(g.rb + (size_t)id[i] * g.rowbytes + s * 512u) : zero;
#pragma unroll
                for (int i = 0; i < B; ++i) acc[i] = acc4_fast<METRIC>(acc[i], qq, r[i]);
            }
        }
        float v[B];
#pragma unroll
        for (int i = 0; i < B; ++i) v[i] = f2_lo(acc[i]) + f2_hi(acc[i]);
        uint32_t row;
        const float s = bfly_reduce<B>(v, lane, row);
        if (((uint32_t)lane & (32u / B - 1u)) == 0 && t0 + row < cnt) dl[t0 + row] = finish_exact<METRIC>(s);
    }
}

// Two-stage form (SEG != 0): batch t+1's loads are issued before batch t is
// reduced, so 2B rows are in flight per warp.
template <int METRIC, int B, int SEG>
__device__ __forceinline__ void issue_batch(const FastGeom& g, const uint32_t* lst, uint32_t t0,
                                            ulonglong2 (&r)[B], int lane) {
    const ulonglong2 zero = make_ulonglong2(0ull, 0ull);
    const bool act = SEG == 1 || (uint32_t)lane < g.ld4;
#pragma unroll
    for (int j = 0; j < B / 4; ++j) {
        const uint4 v = reinterpret_cast<const uint4*>(lst + t0)[j];
        r[4 * j] = act ? ldg_row16(g.rb + (size_t)v.x * g.rowbytes) : zero;
        r[4 * j + 1] = act ? ldg_row16(g.rb + (size_t)v.y * g.rowbytes) : zero;
        r[4 * j + 2] = act ? ldg_row16(g.rb + (size_t)v.z * g.rowbytes) : zero;
        r[4 * j + 3] = act ? ldg_row16(g.rb + (size_t)v.w * g.rowbytes) : zero;
    }
}
template <int METRIC, int B>
__device__ __forceinline__ void reduce_batch(const ulonglong2 (&r)[B], ulonglong2 q, float* dl,
                                             uint32_t t0, uint32_t cnt, int lane) {
    float v[B];
#pragma unroll
    for (int i = 0; i < B; ++i) {
        const unsigned long long acc = part4_first<METRIC>(q, r[i]);
        v[i] = f2_lo(acc) + f2_hi(acc);
    }
    uint32_t row;
    const float s = bfly_reduce<B>(v, lane, row);
    if (((uint32_t)lane & (32u / B - 1u)) == 0 && t0 + row < cnt) dl[t0 + row] = finish_exact<METRIC>(s);
}
template <int METRIC, int B, int SEG>
__device__ __forceinline__ void eval_rows_pipe(const FastGeom& g, const uint32_t* lst, float* dl,
                                               uint32_t cnt, ulonglong2 q, int lane) {
    if (cnt == 0) return;
    ulonglong2 ra[B], rb[B];
    issue_batch<METRIC, B, SEG>(g, lst, 0, ra, lane);
    for (uint32_t t0 = 0;;) {
        if (t0 + B < cnt) issue_batch<METRIC, B, SEG>(g, lst, t0 + B, rb, lane);
        reduce_batch<METRIC, B>(ra, q, dl, t0, cnt, lane);
        t0 += B;
        if (t0 >= cnt) break;
        if (t0 + B < cnt) issue_batch<METRIC, B, SEG>(g, lst, t0 + B, ra, lane);
        reduce_batch<METRIC, B>(rb, q, dl, t0, cnt, lane);
        t0 += B;
        if (t0 >= cnt) break;
    }
}
template <int METRIC, int B, int SEG, bool PIPE>
__device__ __forceinline__ void eval_list(const FastGeom& g, const uint32_t* lst, float* dl,
                                          uint32_t cnt, ulonglong2 q, int lane) {
    if (PIPE && SEG != 0) eval_rows_pipe<METRIC, B, SEG>(g, lst, dl, cnt, q, lane);
    else eval_rows<METRIC, B, SEG>(g, lst, dl, cnt, q, lane);
}

// One row, whole warp; every lane gets the distance.
template <int METRIC, int SEG>
__device__ __forceinline__ float eval_one(const FastGeom& g, uint32_t e, ulonglong2 q, int lane) {
    const ulonglong2 zero = make_ulonglong2(0ull, 0ull);
    unsigned long long acc = 0ull;
    if (SEG != 0) {
        const bool act = SEG == 1 || (uint32_t)lane < g.ld4;
        acc = part4_first<METRIC>(q, act ? ldg_row16(g.rb + (size_t)e * g.rowbytes) : zero);
    } else {
        const uint32_t nseg = (g.ld4 + 31u) >> 5;
        for (uint32_t s = 0; s < nseg; ++s) {
            const uint32_t f = s * 32u + (uint32_t)lane;
            const bool act = f < g.ld4;
            const ulonglong2 qq = act ? g.sq[f] : zero;
            acc = acc4_fast<METRIC>(acc, qq, act ? ldg_row16(g.rb + (size_t)e * g.rowbytes + s * 512u) : zero);
        }
    }
    float v = f2_lo(acc) + f2_hi(acc);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
    return finish_exact<METRIC>(v);
}

// ---- C and V in sentinel form (segmented.cpp:8-79) ------------------------------
struct FastCV {
    uint32_t* cid;
    float* cdist;
    uint32_t* vid;
    uint32_t m;
};

// 32 ids of one segment row (16-byte aligned) contain e?  No branches.
__device__ __forceinline__ bool scan32(const uint32_t* row, uint32_t e) {
    const uint4* p = reinterpret_cast<const uint4*>(row);
    bool hit = false;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        const uint4 v = p[t];
        hit |= (v.x == e) | (v.y == e) | (v.z == e) | (v.w == e);
    }
    return hit;
}

// SegmentedQueue::push (segmented.cpp:13-34).  Returns the id displaced from C
// (kInvalid if none, or if the newcomer itself was dropped).  Warp-uniform call.
__device__ __forceinline__ uint32_t fc_push(const FastCV& cv, uint32_t e, float dist,
                                            uint32_t& total, uint32_t& evictions, int lane) {
    const uint32_t base = seg_of(e, cv.m) * kSegPitch;
    const uint32_t my_i = cv.cid[base + lane];
    const float my_d = cv.cdist[base + lane];
    const uint32_t li = __shfl_sync(kFull, my_i, 31);
    const float ld = __shfl_sync(kFull, my_d, 31);
    uint32_t displaced = kInvalid;
    if (li != kInvalid) {  // full segment: drop the farthest of (segment, newcomer)
        ++evictions;
        if (!closer(dist, e, ld, li)) return kInvalid;
        displaced = li;
        --total;
    }
    const uint32_t pos = __popc(__ballot_sync(kFull, closer(my_d, my_i, dist, e)));
    const uint32_t ui = __shfl_up_sync(kFull, my_i, 1);
    const float ud = __shfl_up_sync(kFull, my_d, 1);
    __syncwarp();
    if ((uint32_t)lane >= pos) {
        const bool me = (uint32_t)lane == pos;
        cv.cid[base + lane] = me ? e : ui;
        cv.cdist[base + lane] = me ? dist : ud;
    }
    ++total;
    __syncwarp();
    return displaced;
}

// SegmentedQueue::pop_min (segmented.cpp:36-53), total > 0.  Warp-uniform call.
__device__ __forceinline__ void fc_pop_min(const FastCV& cv, float& pd, uint32_t& pu,
                                           uint32_t& total, int lane) {
    float hd = __int_as_float(0x7f800000);
    uint32_t hi = kInvalid;
    if ((uint32_t)lane < cv.m) {
        hd = cv.cdist[lane * kSegPitch];
        hi = cv.cid[lane * kSegPitch];
    }
    warp_argmin(hd, hi);
    pd = hd;
    pu = hi;
    const uint32_t base = seg_of(hi, cv.m) * kSegPitch;
    const uint32_t ni = lane < 31 ? cv.cid[base + lane + 1] : kInvalid;
    const float nd = lane < 31 ? cv.cdist[base + lane + 1] : __int_as_float(0x7f800000);
    __syncwarp();
    cv.cid[base + lane] = ni;
    cv.cdist[base + lane] = nd;
    --total;
    __syncwarp();
}

// SegmentedVisited::add (segmented.cpp:68-79): dedup, then the FIFO slot.  Lane s
// holds vcnt = number of ids ever written to segment s.  Warp-uniform call.
__device__ __forceinline__ void fv_add(const FastCV& cv, uint32_t u, uint32_t& vcnt, int lane) {
    const uint32_t s = seg_of(u, cv.m);
    const uint32_t base = s * kSegPitch;
    const bool hit = __any_sync(kFull, cv.vid[base + lane] == u);
    const uint32_t c = __shfl_sync(kFull, vcnt, (int)s);
    __syncwarp();
    if (!hit) {
        if (lane == 0) cv.vid[base + (c & 31u)] = u;
        if ((uint32_t)lane == s) ++vcnt;
    }
    __syncwarp();
}

// Rank-compact the needed lanes of two 32-edge chunks into lst (chunk 0 first),
// padded to a multiple of B with the last needed id (a row already in flight in
// the same batch, so padding costs no DRAM traffic).
__device__ __forceinline__ uint32_t compact2(uint32_t* lst, bool need0, uint32_t e0, bool need1,
                                             uint32_t e1, uint32_t& rk0, uint32_t& rk1, int lane,
                                             uint32_t B) {
    const unsigned lt = (1u << lane) - 1u;
    const unsigned nm0 = __ballot_sync(kFull, need0), nm1 = __ballot_sync(kFull, need1);
    const uint32_t c0 = __popc(nm0), cnt = c0 + __popc(nm1);
    rk0 = __popc(nm0 & lt);
    rk1 = c0 + __popc(nm1 & lt);
    if (need0) lst[rk0] = e0;
    if (need1) lst[rk1] = e1;
    const uint32_t padded = (cnt + B - 1) / B * B;
    if (padded != cnt) {  // warp-uniform; cnt > 0 here
        const int src = nm1 ? 31 - __clz(nm1) : 31 - __clz(nm0);
        const uint32_t pad = __shfl_sync(kFull, nm1 ? e1 : e0, src);
        if ((uint32_t)lane + cnt < padded) lst[cnt + lane] = pad;
    }
    __syncwarp();
    return cnt;
}

// L2 prefetch of row e by the lane that wants it: per-lane 128-byte line prefetches
// (CCTL, all lanes in one instruction per line) by default; with prefetch bit 2 one
// bulk prefetch per row (UBLKPF — a uniform-datapath op, serialised over lanes).
__device__ __forceinline__ void row_prefetch(const BfArgs& a, bool want, uint32_t e,
                                             uint32_t rowbytes) {
    const char* p = reinterpret_cast<const char*>(a.vec + (size_t)e * a.ld);
    if (a.prefetch & 4u) {
        if (want) bulk_prefetch_l2(p, rowbytes);
    } else if (want) {
        for (uint32_t o = 0; o < rowbytes; o += 128) prefetch_l2(p + o);
    }
}

// Group mode (GRP = 2 or 4 warps, one query): the leader warp runs the search; at
// every row evaluation of more than B rows the helper warps take the rows past the
// leader's share, share rows each.  ctl (shared memory): [0] command (1 evaluate,
// 0 exit), [1] rows, [2] the share (a multiple of B), [3] the current query.  One
// evaluation = one "go" and one "done" barrier on all GRP warps — the non-.aligned
// named barrier 1 (the warps reach it from different code), never __syncthreads().
template <int GRP>
__device__ __forceinline__ void group_barrier() {
    asm volatile("barrier.sync 1, %0;" ::"n"(GRP * 32) : "memory");
}
template <int METRIC, int B, int SEG, bool PIPE, int GRP>
__device__ __forceinline__ void coop_eval(const FastGeom& g, const uint32_t* lst, float* dl,
                                          uint32_t cnt, ulonglong2 q, int lane,
                                          volatile uint32_t* ctl) {
    if (GRP == 1 || cnt <= (uint32_t)B) {
        eval_list<METRIC, B, SEG, PIPE>(g, lst, dl, cnt, q, lane);
        return;
    }
    const uint32_t share = ((cnt + GRP - 1) / GRP + B - 1) / B * B;  // < cnt when cnt > B
    if (lane == 0) {
        ctl[0] = 1u;
        ctl[1] = cnt;
        ctl[2] = share;
    }
    group_barrier<GRP>();  // go
    eval_list<METRIC, B, SEG, PIPE>(g, lst, dl, min(share, cnt), q, lane);
    group_barrier<GRP>();  // done: the helpers' dl entries are visible
}

// Admission replay of one 32-edge chunk in edge order (bestfirst_search.cpp:85-96).
// Evictions revive a later queued edge of this chunk (re-evaluated at once) and,
// for chunk 0, queued edges of the next chunk (`revived1`, evaluated before it).
template <int METRIC, int SEG, bool FIRST>
__device__ __forceinline__ void admit_chunk(const BfArgs& a, const FastCV& cv, const FastGeom& g,
                                            ulonglong2 q, RReg& rr, uint32_t& rn, float& rfar,
                                            uint32_t e, float& dist, bool need, bool inC,
                                            uint32_t e1, unsigned& pending1, unsigned& revivable1,
                                            unsigned& revived1, uint32_t& ctotal,
                                            uint32_t& evictions, uint32_t& evals, int lane) {
    const float kInf = __int_as_float(0x7f800000);
    unsigned pending = __ballot_sync(kFull, need);
    unsigned revivable = __ballot_sync(kFull, inC);
    const bool pf_adj = (a.prefetch & 2u) != 0;
    while (pending) {
        const bool ok = ((pending >> lane) & 1u) && (dist < rfar || rn < a.k);
        const unsigned adm = __ballot_sync(kFull, ok);
        if (adm == 0) break;
        const int p = __ffs(adm) - 1;
        const uint32_t ep = __shfl_sync(kFull, e, p);
        const float dp = __shfl_sync(kFull, dist, p);
        if (pf_adj && lane < 2) {
            prefetch_l2(a.adj + (size_t)ep * a.R + lane * 32u);
            if (lane == 0) prefetch_l2(a.degcut + ep);
        }
        r_push_reg(rr, rn, ep, dp, lane);
        const uint32_t gone = fc_push(cv, ep, dp, ctotal, evictions, lane);
        if (rn > a.k) --rn;  // pop_furthest
        rfar = rn ? __shfl_sync(kFull, rr.d, rn - 1) : kInf;
        pending &= (p == 31) ? 0u : (~0u << (p + 1));
        if (FIRST && pending1) {
            // a repeated target later in the hop is now in C (graphs from the
            // reference builder have none; kept so arbitrary CSR input stays sane)
            pending1 &= ~__ballot_sync(kFull, ((pending1 >> lane) & 1u) && e1 == ep);
        }
        if (gone != kInvalid) {
            const unsigned hit =
                __ballot_sync(kFull, lane > p && ((revivable >> lane) & 1u) && e == gone);
            if (hit) {
                const int h = __ffs(hit) - 1;
                const float rd = eval_one<METRIC, SEG>(g, gone, q, lane);
                if (lane == h) dist = rd;
                revivable &= ~(1u << h);
                pending |= (1u << h);
                ++evals;
            }
            if (FIRST) {
                const unsigned hit1 =
                    __ballot_sync(kFull, ((revivable1 >> lane) & 1u) && e1 == gone);
                revivable1 &= ~hit1;
                revived1 |= hit1;
            }
        }
    }
}

// MINB = resident CTAs per SM the register cap is set for: 12 -> 80 registers
// (24 warps / SM), 16 -> 64 registers (32 warps / SM).
//
// GRP > 1: the CTA's GRP warps search ONE query together (leader + helpers,
// coop_eval): for batches smaller than the resident query slots (a rank's slice of a
// strong-scaled batch), where one warp per query leaves most of the GPU idle.
template <int METRIC, int B, int SEG, int MINB, bool PIPE, int GRP>
__global__ void __launch_bounds__((GRP == 4 ? 4 : kFastWarps) * 32, GRP == 4 ? MINB / 2 : MINB)
    bf_fast_kernel(const BfArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    unsigned char* ws = smem_raw + (GRP > 1 ? 0u : (threadIdx.x >> 5) * a.warp_smem);
    volatile uint32_t* ctl = reinterpret_cast<volatile uint32_t*>(smem_raw + a.warp_smem);
    FastCV cv;
    cv.cid = reinterpret_cast<uint32_t*>(ws + a.off_cid);
    cv.cdist = reinterpret_cast<float*>(ws + a.off_cdist);
    cv.vid = reinterpret_cast<uint32_t*>(ws + a.off_vid);
    cv.m = a.m;
    uint32_t* lst = reinterpret_cast<uint32_t*>(ws + a.off_lst);
    float* dl = reinterpret_cast<float*>(ws + a.off_dl);
    float* sqf = reinterpret_cast<float*>(ws + a.off_query);
    FastGeom g;
    g.rb = reinterpret_cast<const char*>(a.vec) + 16 * lane;
    g.rowbytes = a.ld * 4u;
    g.ld4 = a.ld >> 2;
    g.sq = reinterpret_cast<const ulonglong2*>(sqf);
    const float kInf = __int_as_float(0x7f800000);
    const uint32_t seg_words = a.m * kSegPitch;  // multiple of 4

    if (GRP > 1 && (threadIdx.x >> 5) != 0) {  // helper warp
        const uint32_t hw = threadIdx.x >> 5;
        uint32_t cur = kInvalid;
        ulonglong2 q = make_ulonglong2(0ull, 0ull);
        for (;;) {
            group_barrier<GRP>();  // go
            if (ctl[0] == 0u) break;
            const uint32_t qi = ctl[3], cnt = ctl[1], share = ctl[2];
            if (SEG != 0 && qi != cur) {
                cur = qi;
                const float* gq = a.queries + (size_t)qi * a.d;
                q = (uint32_t)lane < g.ld4 ? *reinterpret_cast<const ulonglong2*>(gq + 4 * lane)
                                           : make_ulonglong2(0ull, 0ull);
            }
            const uint32_t b0 = hw * share;
            if (b0 < cnt) eval_list<METRIC, B, SEG, PIPE>(g, lst + b0, dl + b0, min(cnt - b0, share), q, lane);
            group_barrier<GRP>();  // done
        }
        return;
    }

    for (;;) {
        uint32_t qi = 0;
        if (lane == 0) qi = atomicAdd(a.work_counter, 1u) - a.work_base;
        qi = __shfl_sync(kFull, qi, 0);
        if (qi >= a.nq) break;
        if (GRP > 1 && lane == 0) ctl[3] = qi;

        const float* gq = a.queries + (size_t)qi * a.d;
        ulonglong2 q = make_ulonglong2(0ull, 0ull);
        __syncwarp();
        if (SEG != 0) {
            // host guarantees d == ld (multiple of 4) and 16-byte aligned query rows
            if ((uint32_t)lane < g.ld4) q = *reinterpret_cast<const ulonglong2*>(gq + 4 * lane);
        } else {
            for (uint32_t i = lane; i < a.ld; i += 32) sqf[i] = i < a.d ? gq[i] : 0.0f;
        }
        {
            const uint4 inv = make_uint4(kInvalid, kInvalid, kInvalid, kInvalid);
            const uint32_t fi = __float_as_uint(kInf);
            const uint4 infs = make_uint4(fi, fi, fi, fi);
            for (uint32_t i = lane; i < seg_words / 4; i += 32) {
                reinterpret_cast<uint4*>(cv.cid)[i] = inv;
                reinterpret_cast<uint4*>(cv.cdist)[i] = infs;
                reinterpret_cast<uint4*>(cv.vid)[i] = inv;
            }
        }
        __syncwarp();

        uint32_t hops = 0, evals = 0, evictions = 0, examined = 0, ctotal = 0, rn = 0, vcnt = 0;
        RReg rr{kInf, kInvalid};

        // 32 uniform start draws with replacement; best by closer (:57-63)
        const uint64_t s0 = fork_state(a.seed, a.qbase + qi);
        const uint32_t v0 = draw_below(s0, (uint32_t)lane, a.n);
        lst[lane] = v0;
        if (a.prefetch & 1u) row_prefetch(a, lane >= B, v0, g.rowbytes);
        __syncwarp();
        coop_eval<METRIC, B, SEG, PIPE, GRP>(g, lst, dl, 32, q, lane, ctl);
        __syncwarp();
        float sd = dl[lane];
        uint32_t si = v0;
        warp_argmin(sd, si);
        evals += 32;
        r_push_reg(rr, rn, si, sd, lane);
        fc_push(cv, si, sd, ctotal, evictions, lane);
        float rfar = __shfl_sync(kFull, rr.d, rn - 1);

        while (ctotal > 0 && hops < a.hop_limit) {  // :73
            ++hops;
            float pd;
            uint32_t u;
            fc_pop_min(cv, pd, u, ctotal, lane);
            if (pd > __fadd_rn(rfar, a.delta)) break;  // :79
            const uint32_t* arow = a.adj + (size_t)u * a.R;
            const uint32_t deg = __ldg(a.degcut + u);
            uint32_t ea = (uint32_t)lane < a.R ? __ldg(arow + lane) : kInvalid;
            uint32_t eb = (uint32_t)lane + 32 < a.R ? __ldg(arow + 32 + lane) : kInvalid;
            fv_add(cv, u, vcnt, lane);
            examined += deg;
            for (uint32_t base = 0; base < deg; base += 64) {
                if (base) {
                    ea = base + lane < a.R ? __ldg(arow + base + lane) : kInvalid;
                    eb = base + 32 + lane < a.R ? __ldg(arow + base + 32 + lane) : kInvalid;
                }
                const bool two = base + 32 < deg;  // warp-uniform
                const bool valid0 = base + lane < deg;
                const bool valid1 = two && base + 32 + lane < deg;
                const uint32_t e0 = valid0 ? ea : kInvalid;
                const uint32_t e1 = valid1 ? eb : kInvalid;
                const uint32_t o0 = seg_of(e0, a.m) * kSegPitch;
                const bool sV0 = valid0 && scan32(cv.vid + o0, e0);
                const bool sC0 = valid0 && scan32(cv.cid + o0, e0);
                bool sV1 = false, sC1 = false;
                if (two) {
                    const uint32_t o1 = seg_of(e1, a.m) * kSegPitch;
                    sV1 = valid1 && scan32(cv.vid + o1, e1);
                    sC1 = valid1 && scan32(cv.cid + o1, e1);
                }
                const bool inC0 = sC0 && !sV0, inC1 = sC1 && !sV1;
                const bool need0 = valid0 && !sV0 && !sC0;
                const bool need1 = valid1 && !sV1 && !sC1;
                uint32_t rk0, rk1;
                const uint32_t cnt = compact2(lst, need0, e0, need1, e1, rk0, rk1, lane, B);
                if (a.prefetch & 1u) {  // rows beyond the first batch -> L2
                    row_prefetch(a, need0 && rk0 >= (uint32_t)B, e0, g.rowbytes);
                    row_prefetch(a, need1 && rk1 >= (uint32_t)B, e1, g.rowbytes);
                }
                coop_eval<METRIC, B, SEG, PIPE, GRP>(g, lst, dl, cnt, q, lane, ctl);
                __syncwarp();
                float dist0 = need0 ? dl[rk0] : kInf;
                float dist1 = need1 ? dl[rk1] : kInf;
                evals += cnt;
                unsigned pending1 = __ballot_sync(kFull, need1);
                unsigned revivable1 = __ballot_sync(kFull, inC1);
                unsigned revived1 = 0;
                admit_chunk<METRIC, SEG, true>(a, cv, g, q, rr, rn, rfar, e0, dist0, need0, inC0, e1,
                                               pending1, revivable1, revived1, ctotal, evictions,
                                               evals, lane);
                if (two) {
                    if (revived1) {
                        // queued edges of chunk 1 evicted during chunk 0: evaluate now
                        const bool rv = (revived1 >> lane) & 1u;
                        uint32_t r0, r1;
                        __syncwarp();
                        const uint32_t rc = compact2(lst, rv, e1, false, 0u, r0, r1, lane, B);
                        coop_eval<METRIC, B, SEG, PIPE, GRP>(g, lst, dl, rc, q, lane, ctl);
                        __syncwarp();
                        if (rv) dist1 = dl[r0];
                        evals += rc;
                    }
                    const bool n1 = (((pending1 | revived1) >> lane) & 1u) != 0;
                    unsigned dummy0 = 0, dummy1 = 0, dummy2 = 0;
                    admit_chunk<METRIC, SEG, false>(a, cv, g, q, rr, rn, rfar, e1, dist1, n1,
                                                    ((revivable1 >> lane) & 1u) != 0, 0u, dummy0,
                                                    dummy1, dummy2, ctotal, evictions, evals, lane);
                }
                __syncwarp();
            }
        }

        uint32_t* oi = a.out_ids + (size_t)qi * a.k;
        float* od = a.out_dists ? a.out_dists + (size_t)qi * a.k : nullptr;
        if ((uint32_t)lane < a.k) {
            oi[lane] = (uint32_t)lane < rn ? rr.i : kInvalid;
            if (od) od[lane] = (uint32_t)lane < rn ? rr.d : kInf;
        }
        if (lane == 0) {
            if (a.out_counts) a.out_counts[qi] = rn;
            if (a.out_stats) {
                tsdg_query_stats st;
                st.hops = hops;
                st.distance_evals = evals;
                st.queue_evictions = evictions;
                st.edges_examined = examined;
                a.out_stats[qi] = st;
            }
        }
        __syncwarp();
    }
    if (GRP > 1) {  // release the helpers
        if (lane == 0) ctl[0] = 0u;
        group_barrier<GRP>();
    }
}

using BfFastKernel = void (*)(BfArgs);
// bf_fast.cu: the instantiation for (metric, row class, variant)
//   variant 0: B = 8, 80 registers (24 warps / SM)      [default, other row classes]
//           1: B = 8, 64 registers (32 warps / SM)      [default, L2 / 128-float rows]
//           2: B = 16, 80 registers
//           3: B = 16, 96 registers (20 warps / SM)
//           4: B = 8 two-stage, 80 registers
//           5: B = 8 two-stage, 96 registers
//           6: B = 4, 64 registers
//           7: B = 4, 80 registers
//           8: B = 8, 72 registers (28 warps / SM)
// grp: warps per query (1; 2 / 4 = the group forms, in variant 0's register budget;
// a group launch has 32 * grp threads per CTA, one query per CTA).
BfFastKernel bf_fast_kernel_for(int metric, int seg, int variant, int grp = 1);

}  // namespace tsdg_dev
