// Large-batch best-first search (paper Alg. 2) — one warp per query, persistent
// grid sized for occupancy, queries handed out by an atomic counter.
//
// Restates tsdg::search_impl<SegmentedQueue, SegmentedVisited>
// (bestfirst_search.cpp:50-108) with the reference's lossy structures kept
// exactly, per warp, in shared memory (segmented.cpp:8-111):
//   C  m segments x 32 (dist,id) sorted ascending; id e lives in segment e % m; a
//      push into a full segment drops the farthest of (segment, newcomer)
//   V  m FIFO rings x 32 ids, dedup-on-add, oldest overwritten when full
//   R  TopK(k): sorted, dedup push, pop farthest.  k <= 31 keeps R in registers
//      (lane i <-> entry i); larger k uses a shared-memory array.
// C and V are segment-major with a 36-word pitch: lane i <-> slot i of one segment
// is conflict-free, and 32 lanes scanning their own segments with LDS.128 hit
// distinct bank groups (pitch/4 = 9 is odd).
//
// One expansion of u (a hop):
//   * deg_cut[u] and the first 64 adjacency entries are loaded together;
//   * edges are processed in chunks of 32 (lane j <-> edge base+j): V/C
//     membership for the chunk, the non-skipped rows gathered (stage.cuh) and
//     reduced — bit-identical to the CPU in deterministic mode;
//   * admission is replayed in edge order with ballots: once |R| = k the farthest
//     distance only shrinks, so the first lane passing the test under the current
//     state IS the next admission.  A C-push that evicts an id sitting later in
//     the chunk (skipped because it was queued) revives that edge, exactly as the
//     sequential loop would see it;
//   * optional L2 prefetch (off by default, measured neutral): the rows of the next
//     chunk, and the adjacency row + deg_cut entry of every admitted node.
#pragma once

#include "../../include/tsdg_gpu.h"
#include "stage.cuh"

namespace tsdg_dev {

constexpr int kBfWarps = 4;       // queries per CTA
constexpr uint32_t kSegPitch = 36; // words per segment row (C and V)

struct BfArgs {
    const float* vec;       // n x ld
    const uint32_t* adj;    // n x R
    const uint32_t* degcut; // n
    const float* queries;   // nq x d (caller layout)
    uint32_t ld, R, n, d;
    uint32_t nq;
    uint64_t qbase;
    uint32_t k, hop_limit;
    float delta;
    uint32_t m;
    uint64_t seed;
    uint32_t* out_ids;
    float* out_dists;
    uint32_t* out_counts;
    tsdg_query_stats* out_stats;
    uint32_t* work_counter;
    uint32_t work_base;     // counter value at launch (tsdg_gpu.cu next_counter)
    uint32_t dch;           // staged dims per row per round (multiple of 8, <= 128)
    uint32_t slots;         // staged rows per gather round (1..32)
    uint32_t prefetch;      // bit 0: next-chunk rows (L2), bit 1: admitted adjacency (L2)
    uint32_t batch_min;     // batched admission when >= this many candidates pass the
                            // current bound (0: never; sequential replay only)
    // per-warp shared-memory carve (bytes)
    uint32_t warp_smem, off_query, off_stage, off_cid, off_cdist, off_csize, off_vid,
        off_vsize, off_voldest, off_rid, off_rdist, off_bar, off_rowid;
    uint32_t off_lst, off_dl;  // bf_fast_kernel: needed-row ids / distances (64 + pad)
    const void* tmap;          // kStageG4: tensor map of vec (global memory)
    uint32_t gpitch;           // kStageG4: floats between 4-slot groups
};

struct BfWarp {
    WarpStage st;
    uint32_t* cid;
    float* cdist;
    uint32_t* csize;
    uint32_t* vid;
    uint32_t* vsize;
    uint32_t* voldest;
    uint32_t* rid;   // smem R (large k)
    float* rdist;
};

// e % m without a hardware divide when m is a power of two (the usual 8 / 16)
__device__ __forceinline__ uint32_t seg_of(uint32_t e, uint32_t m) {
    return (m & (m - 1)) == 0 ? (e & (m - 1)) : e % m;
}

// ---- membership scans: each lane its own segment, 8 x LDS.128 ------------------
__device__ __forceinline__ bool seg_scan(const uint32_t* base, uint32_t sz, uint32_t e) {
    const uint4* p = reinterpret_cast<const uint4*>(base);
    bool hit = false;
#pragma unroll
    for (uint32_t t = 0; t < 8; ++t) {
        if (4 * t < sz) {
            const uint4 v = p[t];
            hit |= (v.x == e) & (4 * t + 0 < sz);
            hit |= (v.y == e) & (4 * t + 1 < sz);
            hit |= (v.z == e) & (4 * t + 2 < sz);
            hit |= (v.w == e) & (4 * t + 3 < sz);
        }
    }
    return hit;
}
__device__ __forceinline__ bool v_contains(const BfWarp& w, uint32_t m, uint32_t e) {
    const uint32_t s = seg_of(e, m);
    return seg_scan(w.vid + s * kSegPitch, w.vsize[s], e);
}
__device__ __forceinline__ bool c_contains(const BfWarp& w, uint32_t m, uint32_t e) {
    const uint32_t s = seg_of(e, m);
    return seg_scan(w.cid + s * kSegPitch, w.csize[s], e);
}

// segmented.cpp:68-79 (warp-uniform call)
__device__ __forceinline__ void v_add(BfWarp& w, uint32_t m, uint32_t u, int lane) {
    const uint32_t s = seg_of(u, m);
    uint32_t* seg = w.vid + s * kSegPitch;
    const uint32_t sz = w.vsize[s];
    const bool hit = lane < (int)sz && seg[lane] == u;
    const unsigned any_hit = __ballot_sync(kFull, hit);
    __syncwarp();  // every lane's read of the segment before lane 0 writes it
    if (any_hit == 0 && lane == 0) {
        if (sz < 32) {
            seg[sz] = u;
            w.vsize[s] = sz + 1;
        } else {
            const uint32_t o = w.voldest[s];
            seg[o] = u;
            w.voldest[s] = (o + 1) & 31u;
        }
    }
    __syncwarp();
}

// segmented.cpp:13-34.  Returns the id displaced from C (kInvalid if none, or if
// the newcomer itself was dropped).  Warp-uniform call.
__device__ __forceinline__ uint32_t c_push(BfWarp& w, uint32_t m, uint32_t e, float dist,
                                           uint32_t& total, uint32_t& evictions, int lane) {
    const uint32_t s = seg_of(e, m);
    uint32_t* sid = w.cid + s * kSegPitch;
    float* sdist = w.cdist + s * kSegPitch;
    uint32_t sz = w.csize[s];
    const float my_d = lane < (int)sz ? sdist[lane] : 0.f;
    const uint32_t my_i = lane < (int)sz ? sid[lane] : 0u;
    uint32_t displaced = kInvalid;
    if (sz == 32) {
        const float md = __shfl_sync(kFull, my_d, 31);
        const uint32_t mi = __shfl_sync(kFull, my_i, 31);
        ++evictions;
        if (!closer(dist, e, md, mi)) return kInvalid;
        displaced = mi;
        sz = 31;
        --total;
    }
    const bool after = lane < (int)sz && closer(dist, e, my_d, my_i);
    const unsigned gm = __ballot_sync(kFull, after);
    const uint32_t pos = gm ? (uint32_t)(__ffs(gm) - 1) : sz;
    __syncwarp();
    if (lane < (int)sz && (uint32_t)lane >= pos) {
        sdist[lane + 1] = my_d;
        sid[lane + 1] = my_i;
    }
    if ((uint32_t)lane == pos) {
        sdist[pos] = dist;
        sid[pos] = e;
    }
    if (lane == 0) w.csize[s] = sz + 1;
    ++total;
    __syncwarp();
    return displaced;
}

// segmented.cpp:36-53 (requires total > 0).  Warp-uniform call.
__device__ __forceinline__ void c_pop_min(BfWarp& w, uint32_t m, float& pd, uint32_t& pu,
                                          uint32_t& total, int lane) {
    float hd = __int_as_float(0x7f800000);
    uint32_t hi = kInvalid;
    for (uint32_t s = lane; s < m; s += 32) {
        if (w.csize[s] != 0) {
            const float d = w.cdist[s * kSegPitch];
            const uint32_t i = w.cid[s * kSegPitch];
            if (closer(d, i, hd, hi)) {
                hd = d;
                hi = i;
            }
        }
    }
    warp_argmin(hd, hi);
    pd = hd;
    pu = hi;
    const uint32_t s = seg_of(hi, m);
    uint32_t* sid = w.cid + s * kSegPitch;
    float* sdist = w.cdist + s * kSegPitch;
    const uint32_t sz = w.csize[s];
    const bool mv = lane >= 1 && lane < (int)sz;
    const float sd = mv ? sdist[lane] : 0.f;
    const uint32_t si = mv ? sid[lane] : 0u;
    __syncwarp();
    if (mv) {
        sdist[lane - 1] = sd;
        sid[lane - 1] = si;
    }
    if (lane == 0) w.csize[s] = sz - 1;
    --total;
    __syncwarp();
}

// ---- TopK R --------------------------------------------------------------------
// Register form (k <= 31): lane i holds entry i for i < rn.
struct RReg {
    float d;
    uint32_t i;
};
// segmented.cpp:94-101: no-op on a duplicate id, else sorted insert.
__device__ __forceinline__ void r_push_reg(RReg& r, uint32_t& rn, uint32_t e, float dist,
                                           int lane) {
    const bool live = lane < (int)rn;
    if (__any_sync(kFull, live && r.i == e)) return;
    const uint32_t pos = __popc(__ballot_sync(kFull, live && !closer(dist, e, r.d, r.i)));
    const float ud = __shfl_up_sync(kFull, r.d, 1);
    const uint32_t ui = __shfl_up_sync(kFull, r.i, 1);
    if ((uint32_t)lane == pos) {
        r.d = dist;
        r.i = e;
    } else if ((uint32_t)lane > pos && (uint32_t)lane <= rn) {
        r.d = ud;
        r.i = ui;
    }
    ++rn;
}
// Shared-memory form (any k).
__device__ __forceinline__ void r_push_smem(BfWarp& w, uint32_t& rn, uint32_t e, float dist,
                                            int lane) {
    bool dup = false;
    uint32_t before = 0;
    for (uint32_t c = 0; c < rn; c += 32) {
        const uint32_t i = c + lane;
        bool front = false;
        if (i < rn) {
            const uint32_t ri = w.rid[i];
            dup |= (ri == e);
            front = !closer(dist, e, w.rdist[i], ri);
        }
        before += __popc(__ballot_sync(kFull, front));
    }
    if (__any_sync(kFull, dup)) return;
    const uint32_t pos = before;
    if (rn > pos) {
        const uint32_t top = (rn - 1) & ~31u;
        for (int c = (int)top; c >= (int)(pos & ~31u); c -= 32) {
            const uint32_t i = (uint32_t)c + lane;
            const bool mv = i >= pos && i < rn;
            const uint32_t ri = mv ? w.rid[i] : 0u;
            const float rd = mv ? w.rdist[i] : 0.f;
            __syncwarp();
            if (mv) {
                w.rid[i + 1] = ri;
                w.rdist[i + 1] = rd;
            }
            __syncwarp();
        }
    }
    if (lane == 0) {
        w.rid[pos] = e;
        w.rdist[pos] = dist;
    }
    ++rn;
    __syncwarp();
}

// Number of entries of a sorted 32-lane list (lane t holds entry t; padded with
// (+inf, kInvalid) sentinels) that are strictly closer than (xd, xi).  Per-lane
// binary search through shuffles with per-lane source lanes.
__device__ __forceinline__ uint32_t count_closer32(float vd, uint32_t vi, float xd, uint32_t xi) {
    uint32_t pos = 0;
#pragma unroll
    for (uint32_t step = 16; step > 0; step >>= 1) {
        const float pd = __shfl_sync(kFull, vd, (int)(pos + step - 1));
        const uint32_t pi = __shfl_sync(kFull, vi, (int)(pos + step - 1));
        if (closer(pd, pi, xd, xi)) pos += step;
    }
    const float ld = __shfl_sync(kFull, vd, 31);
    const uint32_t li = __shfl_sync(kFull, vi, 31);
    if (pos == 31 && closer(ld, li, xd, xi)) pos = 32;
    return pos;
}

// Batched admission of one chunk for k <= 31 (R in registers, lane i = entry i).
//
// The reference admits the chunk's candidates one by one in edge order with the
// test dist < R.furthest().dist || |R| < k (bestfirst_search.cpp:91).  A rejected
// candidate is never closer than the current k-th distance, so counting it in the
// multiset does not move the k-th smallest distance; hence candidate j is admitted
// iff fewer than k of {R} u {needed candidates before j} have distance <= dist_j.
// The final R is the k smallest by (dist, id) of R u admitted (each push + pop of
// the farthest keeps exactly that).  C's final content without a full segment is
// order independent and no eviction happens.  Two cases make order matter and fall
// back to the sequential replay (returns false, nothing modified): a needed id
// already held by R (TopK::push is then a no-op) and a C segment that would overflow.
__device__ __forceinline__ bool admit_batch_reg(BfWarp& w, uint32_t m, uint32_t k, RReg& rr,
                                                uint32_t& rn, float& rfar, bool need, float dist,
                                                uint32_t e, uint32_t& ctotal, uint32_t& evictions,
                                                int lane) {
    const float kInf = __int_as_float(0x7f800000);
    const unsigned nm = __ballot_sync(kFull, need);
    if (nm == 0) return true;
    const float rdv = (uint32_t)lane < rn ? rr.d : kInf;
    const uint32_t riv = (uint32_t)lane < rn ? rr.i : kInvalid;
    bool dup = false;
    for (uint32_t i = 0; i < rn; ++i) {
        const uint32_t ri = __shfl_sync(kFull, riv, (int)i);  // every lane: no short-circuit
        dup |= need && ri == e;
    }
    if (__any_sync(kFull, dup)) return false;
    // #R entries with distance <= dist (R sorted; padded with +inf)
    uint32_t cnt = 0;
#pragma unroll
    for (uint32_t step = 16; step > 0; step >>= 1) {
        const float v = __shfl_sync(kFull, rdv, (int)(cnt + step - 1));
        if (v <= dist) cnt += step;
    }
    // + earlier needed candidates with distance <= dist
    unsigned mm = nm & ((1u << lane) - 1u);
    unsigned rest = nm;
    while (rest) {
        const int i = __ffs(rest) - 1;
        rest &= rest - 1;
        const float di = __shfl_sync(kFull, dist, i);
        if ((mm >> i) & 1u) cnt += (di <= dist) ? 1u : 0u;
    }
    const bool admit = need && cnt < k;
    const unsigned am = __ballot_sync(kFull, admit);
    if (am == 0) return true;
    const uint32_t s = seg_of(e, m);
    const unsigned same = __match_any_sync(kFull, admit ? s : 0xFFFFFFFFu) & am;
    const bool over = admit && (w.csize[s] + __popc(same) > 32u);
    if (__any_sync(kFull, over)) return false;
    // R <- k smallest of R u A
    float ad = admit ? dist : kInf;
    uint32_t ai = admit ? e : kInvalid;
    warp_sort32(ad, ai, lane);
    const uint32_t na = __popc(am);
    const uint32_t rank_r = (uint32_t)lane + count_closer32(ad, ai, rdv, riv);
    const uint32_t rank_a = (uint32_t)lane + count_closer32(rdv, riv, ad, ai);
    float* sd = w.cdist + m * kSegPitch;  // scratch row after C (carved by the host)
    uint32_t* si = w.cid + m * kSegPitch;
    __syncwarp();
    if ((uint32_t)lane < rn && rank_r < k) {
        sd[rank_r] = rdv;
        si[rank_r] = riv;
    }
    if ((uint32_t)lane < na && rank_a < k) {
        sd[rank_a] = ad;
        si[rank_a] = ai;
    }
    __syncwarp();
    rn = min(k, rn + na);
    if ((uint32_t)lane < rn) {
        rr.d = sd[lane];
        rr.i = si[lane];
    }
    __syncwarp();
    rfar = __shfl_sync(kFull, rr.d, (int)rn - 1);
    // C pushes (no segment overflows: order independent, no evictions)
    rest = am;
    while (rest) {
        const int p = __ffs(rest) - 1;
        rest &= rest - 1;
        c_push(w, m, __shfl_sync(kFull, e, p), __shfl_sync(kFull, dist, p), ctotal, evictions,
               lane);
    }
    return true;
}

__device__ __forceinline__ void prefetch_rows(const BfArgs& a, bool want, uint32_t e) {
    if (want) {
        const char* p = reinterpret_cast<const char*>(a.vec + (size_t)e * a.ld);
        const uint32_t bytes = min(a.ld * 4u, 512u);
        for (uint32_t o = 0; o < bytes; o += 128) prefetch_l2(p + o);
    }
}

// minBlocks 4 caps registers at 128 without spills (ptxas otherwise targets 72
// registers and spills; measured 9% slower on C2)
#ifndef TSDG_BF_MIN_BLOCKS
#define TSDG_BF_MIN_BLOCKS 4
#endif
template <int METRIC, bool FAST, int STAGE, bool KREG>
__global__ void __launch_bounds__(kBfWarps * 32, TSDG_BF_MIN_BLOCKS) bf_kernel(const BfArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    unsigned char* ws = smem_raw + (threadIdx.x >> 5) * a.warp_smem;
    BfWarp w;
    w.st.sq = reinterpret_cast<float*>(ws + a.off_query);
    w.st.stage = reinterpret_cast<float*>(ws + a.off_stage);
    w.st.bar = reinterpret_cast<uint64_t*>(ws + a.off_bar);
    w.st.parity = 0;
    w.st.rowid = a.off_rowid ? reinterpret_cast<uint32_t*>(ws + a.off_rowid) : nullptr;
    w.cid = reinterpret_cast<uint32_t*>(ws + a.off_cid);
    w.cdist = reinterpret_cast<float*>(ws + a.off_cdist);
    w.csize = reinterpret_cast<uint32_t*>(ws + a.off_csize);
    w.vid = reinterpret_cast<uint32_t*>(ws + a.off_vid);
    w.vsize = reinterpret_cast<uint32_t*>(ws + a.off_vsize);
    w.voldest = reinterpret_cast<uint32_t*>(ws + a.off_voldest);
    w.rid = reinterpret_cast<uint32_t*>(ws + a.off_rid);
    w.rdist = reinterpret_cast<float*>(ws + a.off_rdist);
    if (STAGE != kStageLdgsts) {
        if (lane == 0) mbar_init(w.st.bar, 1);
        __syncwarp();
    }
    const Geom g{a.vec, a.ld, a.d, a.dch, a.slots, 0, a.tmap, a.gpitch};
    const float kInf = __int_as_float(0x7f800000);
    const bool pf_rows = (a.prefetch & 1u) != 0;
    const bool pf_adj = (a.prefetch & 2u) != 0;

    for (;;) {
        uint32_t q = 0;
        if (lane == 0) q = atomicAdd(a.work_counter, 1u) - a.work_base;
        q = __shfl_sync(kFull, q, 0);
        if (q >= a.nq) break;

        const float* gq = a.queries + (size_t)q * a.d;
        __syncwarp();
        for (uint32_t i = lane; i < a.ld; i += 32) w.st.sq[i] = i < a.d ? gq[i] : 0.0f;
        for (uint32_t i = lane; i < a.m; i += 32) {
            w.csize[i] = 0;
            w.vsize[i] = 0;
            w.voldest[i] = 0;
        }
        __syncwarp();

        uint32_t hops = 0, evals = 0, evictions = 0, examined = 0, ctotal = 0, rn = 0;
        RReg rr{kInf, kInvalid};
        PH_DECL

        // 32 uniform start draws with replacement; best by closer (:57-63)
        const uint64_t s0 = fork_state(a.seed, a.qbase + q);
        const uint32_t v0 = draw_below(s0, (uint32_t)lane, a.n);
        float sd = gather_eval<METRIC, FAST, STAGE>(w.st, g, true, v0, lane);
        uint32_t si = v0;
        warp_argmin(sd, si);
        evals += 32;
        if (KREG) r_push_reg(rr, rn, si, sd, lane);
        else r_push_smem(w, rn, si, sd, lane);
        c_push(w, a.m, si, sd, ctotal, evictions, lane);
        float rfar = KREG ? __shfl_sync(kFull, rr.d, rn - 1) : w.rdist[rn - 1];
        PH_MARK(0)

        while (ctotal > 0 && hops < a.hop_limit) {  // :73
            ++hops;
            float pd;
            uint32_t u;
            c_pop_min(w, a.m, pd, u, ctotal, lane);
            if (pd > __fadd_rn(rfar, a.delta)) break;  // :79
            // issue the dependent loads first (unless the speculation already did), then
            // V.add while they fly
            const uint32_t* arow = a.adj + (size_t)u * a.R;
            const uint32_t deg = __ldg(a.degcut + u);
            uint32_t e_next = (uint32_t)lane < a.R ? __ldg(arow + lane) : kInvalid;
            uint32_t e_next2 = (uint32_t)lane + 32 < a.R ? __ldg(arow + 32 + lane) : kInvalid;
            v_add(w, a.m, u, lane);
            examined += deg;
            PH_MARK(1)
            for (uint32_t base = 0; base < deg; base += 32) {
                const uint32_t j = base + lane;
                const bool valid = j < deg;
                const uint32_t e = valid ? e_next : kInvalid;
                e_next = e_next2;
                const uint32_t j2 = base + 64 + lane;
                e_next2 = (base + 64 < deg && j2 < a.R) ? __ldg(arow + j2) : kInvalid;
                // both scans unconditionally: independent LDS streams overlap
                const bool sV = valid && v_contains(w, a.m, e);
                const bool sC = valid && c_contains(w, a.m, e);
                const bool inV = sV;
                const bool inC = sC && !sV;
                const bool need = valid && !inV && !inC;
                if (pf_rows && base + 32 < deg) {
                    // next chunk: prefetch rows of edges not visited (V is fixed for
                    // this expansion; C-membership is re-checked at that chunk)
                    const bool nv = base + 32 + lane < deg && !v_contains(w, a.m, e_next);
                    prefetch_rows(a, nv, e_next);
                }
                PH_MARK(2)
                float dist = gather_eval<METRIC, FAST, STAGE>(w.st, g, need, e, lane);
                PH_RESET
                unsigned pending = __ballot_sync(kFull, need);
                unsigned revivable = __ballot_sync(kFull, inC);
                evals += __popc(pending);
                if (KREG && a.batch_min &&
                    (uint32_t)__popc(__ballot_sync(kFull, need && (dist < rfar || rn < a.k))) >= a.batch_min &&
                    admit_batch_reg(w, a.m, a.k, rr, rn, rfar, need, dist, e, ctotal, evictions, lane))
                    pending = 0;
                while (pending) {
                    const bool ok = ((pending >> lane) & 1u) && (dist < rfar || rn < a.k);
                    const unsigned adm = __ballot_sync(kFull, ok);
                    if (adm == 0) break;
                    const int p = __ffs(adm) - 1;
                    const uint32_t ep = __shfl_sync(kFull, e, p);
                    const float dp = __shfl_sync(kFull, dist, p);
                    if (pf_adj && lane == 0) {
                        prefetch_l2(a.adj + (size_t)ep * a.R);
                        prefetch_l2(a.degcut + ep);
                    }
                    if (KREG) r_push_reg(rr, rn, ep, dp, lane);
                    else r_push_smem(w, rn, ep, dp, lane);
                    const uint32_t gone = c_push(w, a.m, ep, dp, ctotal, evictions, lane);
                    if (rn > a.k) --rn;  // pop_furthest
                    if (KREG) rfar = rn ? __shfl_sync(kFull, rr.d, rn - 1) : kInf;
                    else rfar = rn ? w.rdist[rn - 1] : kInf;
                    pending &= (p == 31) ? 0u : (~0u << (p + 1));
                    if (gone != kInvalid) {
                        const unsigned hit = __ballot_sync(
                            kFull, lane > p && ((revivable >> lane) & 1u) && e == gone);
                        if (hit) {
                            const int h = __ffs(hit) - 1;
                            const float rd =
                                gather_eval<METRIC, FAST, STAGE>(w.st, g, lane == h, e, lane);
                            if (lane == h) dist = rd;
                            revivable &= ~(1u << h);
                            pending |= (1u << h);
                            ++evals;
                        }
                    }
                }
                PH_MARK(5)
            }
        }

        uint32_t* oi = a.out_ids + (size_t)q * a.k;
        float* od = a.out_dists ? a.out_dists + (size_t)q * a.k : nullptr;
        if (KREG) {
            if ((uint32_t)lane < a.k) {
                oi[lane] = (uint32_t)lane < rn ? rr.i : kInvalid;
                if (od) od[lane] = (uint32_t)lane < rn ? rr.d : kInf;
            }
        } else {
            for (uint32_t i = lane; i < a.k; i += 32) {
                oi[i] = i < rn ? w.rid[i] : kInvalid;
                if (od) od[i] = i < rn ? w.rdist[i] : kInf;
            }
        }
        if (lane == 0) {
            if (a.out_counts) a.out_counts[q] = rn;
            if (a.out_stats) {
                tsdg_query_stats st;
                st.hops = hops;
                st.distance_evals = evals;
                st.queue_evictions = evictions;
                st.edges_examined = examined;
                a.out_stats[q] = st;
            }
        }
        __syncwarp();
    }
}

}  // namespace tsdg_dev
