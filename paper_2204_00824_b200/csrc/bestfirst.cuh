// Large-batch best-first search (paper Alg. 2) — one warp per query, persistent.
//
// Deterministic restatement of tsdg::search_impl<SegmentedQueue, SegmentedVisited>
// (bestfirst_search.cpp:50-108) with the reference's segmented structures
// (segmented.cpp:8-111) kept exactly in shared memory:
//   C  m x 32 sorted (dist,id) segments, id e in segment e % m, full segment drops
//      its farthest element (possibly the newcomer)           segmented.cpp:13-61
//   V  m x 32 FIFO rings of ids, dedup-on-add                 segmented.cpp:63-87
//   R  TopK(k), sorted, dedup push, pop farthest               segmented.cpp:89-111
// Both C and V are stored slot-major with an odd segment pitch P, so a warp
// touching one segment (lane i <-> slot i) and 32 lanes each scanning their own
// segment are both bank-conflict free.
//
// Per expansion the lambda-prefix of u (deg_cut[u] edges of the padded
// adjacency row) is processed in chunks of 32 edges, lane j <-> edge base+j:
//   1. membership flags (V, C) are evaluated for the whole chunk;
//   2. the rows of the non-skipped edges are gathered into shared memory with TMA
//      1-D bulk copies (one cp.async.bulk per lane, completion on one mbarrier),
//      and every lane reduces its own row sequentially in the reference's fp32
//      order (no FMA) — distances are bit-identical to the CPU's;
//   3. admission is replayed in edge order with ballots: only admissions change
//      the state that later edges see (R's farthest can only shrink once |R| = k),
//      so the first lane passing the test under the current state IS the next
//      admission.  A C-push that evicts an id sitting later in the chunk (skipped
//      because it was queued) revives that edge, as the sequential loop would see.
#pragma once

#include "common.cuh"
#include "../../include/tsdg_gpu.h"

namespace tsdg_dev {

constexpr int kBfWarps = 4;  // queries per CTA

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
    uint32_t m, P;
    uint64_t seed;
    uint32_t* out_ids;
    float* out_dists;
    uint32_t* out_counts;
    tsdg_query_stats* out_stats;
    uint32_t* work_counter;
    uint32_t dch;           // staged dims per row per round (multiple of 8)
    // per-warp shared-memory carve (bytes)
    uint32_t warp_smem, off_query, off_stage, off_cid, off_cdist, off_csize, off_vid,
        off_vsize, off_voldest, off_rid, off_rdist, off_bar;
};

struct BfWarp {
    float* sq;
    float* stage;
    uint32_t* cid;
    float* cdist;
    uint32_t* csize;
    uint32_t* vid;
    uint32_t* vsize;
    uint32_t* voldest;
    uint32_t* rid;
    float* rdist;
    uint64_t* bar;
    uint32_t parity;
};

// ---- segmented visited table V ------------------------------------------------
__device__ __forceinline__ bool v_contains(const BfWarp& w, const BfArgs& a, uint32_t e) {
    const uint32_t s = e % a.m;
    const uint32_t sz = w.vsize[s];
    bool hit = false;
    for (uint32_t i = 0; i < sz; ++i) hit |= (w.vid[i * a.P + s] == e);
    return hit;
}
// segmented.cpp:68-79 (warp-uniform call)
__device__ __forceinline__ void v_add(BfWarp& w, const BfArgs& a, uint32_t u, int lane) {
    const uint32_t s = u % a.m;
    const uint32_t sz = w.vsize[s];
    const bool hit = lane < (int)sz && w.vid[lane * a.P + s] == u;
    if (__ballot_sync(kFull, hit) == 0 && lane == 0) {
        if (sz < 32) {
            w.vid[sz * a.P + s] = u;
            w.vsize[s] = sz + 1;
        } else {
            const uint32_t o = w.voldest[s];
            w.vid[o * a.P + s] = u;
            w.voldest[s] = (o + 1) & 31u;
        }
    }
    __syncwarp();
}

// ---- segmented expansion queue C ------------------------------------------------
__device__ __forceinline__ bool c_contains(const BfWarp& w, const BfArgs& a, uint32_t e) {
    const uint32_t s = e % a.m;
    const uint32_t sz = w.csize[s];
    bool hit = false;
    for (uint32_t i = 0; i < sz; ++i) hit |= (w.cid[i * a.P + s] == e);
    return hit;
}
// segmented.cpp:13-34.  Returns the id displaced from C (kInvalid if none or if
// the newcomer itself was dropped).  Warp-uniform call.
__device__ __forceinline__ uint32_t c_push(BfWarp& w, const BfArgs& a, uint32_t e, float dist,
                                           uint32_t& total, uint32_t& evictions, int lane) {
    const uint32_t s = e % a.m;
    uint32_t sz = w.csize[s];
    uint32_t displaced = kInvalid;
    if (sz == 32) {
        const float md = w.cdist[31 * a.P + s];
        const uint32_t mi = w.cid[31 * a.P + s];
        ++evictions;
        if (!closer(dist, e, md, mi)) return kInvalid;
        displaced = mi;
        sz = 31;
        --total;
    }
    float sd = 0.f;
    uint32_t si = 0;
    bool after = false;
    if (lane < (int)sz) {
        sd = w.cdist[lane * a.P + s];
        si = w.cid[lane * a.P + s];
        after = closer(dist, e, sd, si);
    }
    const unsigned gm = __ballot_sync(kFull, after);
    const uint32_t pos = gm ? (uint32_t)(__ffs(gm) - 1) : sz;
    __syncwarp();
    if (lane < (int)sz && (uint32_t)lane >= pos) {
        w.cdist[(lane + 1) * a.P + s] = sd;
        w.cid[(lane + 1) * a.P + s] = si;
    }
    if ((uint32_t)lane == pos) {
        w.cdist[pos * a.P + s] = dist;
        w.cid[pos * a.P + s] = e;
    }
    if (lane == 0) w.csize[s] = sz + 1;
    ++total;
    __syncwarp();
    return displaced;
}
// segmented.cpp:36-53 (requires total > 0).  Warp-uniform call.
__device__ __forceinline__ void c_pop_min(BfWarp& w, const BfArgs& a, float& pd, uint32_t& pu,
                                          uint32_t& total, int lane) {
    float hd = __int_as_float(0x7f800000);
    uint32_t hi = kInvalid;
    if (lane < (int)a.m && w.csize[lane] != 0) {
        hd = w.cdist[lane];  // slot 0 of segment `lane` is at index 0 * P + lane
        hi = w.cid[lane];
    }
    warp_argmin(hd, hi);
    pd = hd;
    pu = hi;
    const uint32_t s = hi % a.m;
    const uint32_t sz = w.csize[s];
    float sd = 0.f;
    uint32_t si = 0;
    if (lane >= 1 && lane < (int)sz) {
        sd = w.cdist[lane * a.P + s];
        si = w.cid[lane * a.P + s];
    }
    __syncwarp();
    if (lane >= 1 && lane < (int)sz) {
        w.cdist[(lane - 1) * a.P + s] = sd;
        w.cid[(lane - 1) * a.P + s] = si;
    }
    if (lane == 0) w.csize[s] = sz - 1;
    --total;
    __syncwarp();
}

// ---- TopK R ----------------------------------------------------------------------
// segmented.cpp:94-101: no-op on duplicate id, else sorted insert.  Warp-uniform.
__device__ __forceinline__ void r_push(BfWarp& w, uint32_t& rn, uint32_t e, float dist,
                                       int lane) {
    bool dup = false;
    uint32_t before = 0;  // entries that stay in front: !closer(new, entry)
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
    // shift [pos, rn) up by one, top chunk first
    if (rn > pos) {
        const uint32_t top = (rn - 1) & ~31u;
        for (int c = (int)top; c >= (int)(pos & ~31u); c -= 32) {
            const uint32_t i = (uint32_t)c + lane;
            const bool mv = i >= pos && i < rn;
            uint32_t ri = 0;
            float rd = 0.f;
            if (mv) {
                ri = w.rid[i];
                rd = w.rdist[i];
            }
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

// ---- gather + exact distances -----------------------------------------------------
// Each lane with `need` gets the exact distance between the staged query and row e.
template <int METRIC>
__device__ __forceinline__ float gather_distances(BfWarp& w, const BfArgs& a, bool need,
                                                  uint32_t e, int lane) {
    const unsigned nm = __ballot_sync(kFull, need);
    if (nm == 0) return __int_as_float(0x7f800000);
    const uint32_t cnt = __popc(nm);
    const float* grow = a.vec + (size_t)(need ? e : 0) * a.ld;
    float* mine = w.stage + lane * (a.dch + 4);
    float acc = 0.0f;
    for (uint32_t c0 = 0; c0 < a.ld; c0 += a.dch) {
        const uint32_t cw = min(a.dch, a.ld - c0);
        fence_proxy_async_smem();  // prior generic reads of the stage before TMA writes
        __syncwarp();
        if (lane == 0) mbar_arrive_expect_tx(w.bar, cnt * cw * 4u);
        __syncwarp();
        if (need) bulk_g2s(mine, grow + c0, cw * 4u, w.bar);
        mbar_wait(w.bar, w.parity);
        w.parity ^= 1u;
        if (need && c0 < a.d) {
            const uint32_t lim = min(cw, a.d - c0);
            const uint32_t quads = lim >> 2;
            const float4* r4 = reinterpret_cast<const float4*>(mine);
            const float4* q4 = reinterpret_cast<const float4*>(w.sq + c0);
#pragma unroll 8
            for (uint32_t i = 0; i < quads; ++i) acc = acc4_exact<METRIC>(acc, q4[i], r4[i]);
            for (uint32_t i = quads * 4; i < lim; ++i)
                acc = acc_exact<METRIC>(acc, w.sq[c0 + i], mine[i]);
        }
    }
    return need ? finish_exact<METRIC>(acc) : __int_as_float(0x7f800000);
}

template <int METRIC>
__global__ void __launch_bounds__(kBfWarps * 32) bf_det_kernel(const BfArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    unsigned char* ws = smem_raw + (threadIdx.x >> 5) * a.warp_smem;
    BfWarp w;
    w.sq = reinterpret_cast<float*>(ws + a.off_query);
    w.stage = reinterpret_cast<float*>(ws + a.off_stage);
    w.cid = reinterpret_cast<uint32_t*>(ws + a.off_cid);
    w.cdist = reinterpret_cast<float*>(ws + a.off_cdist);
    w.csize = reinterpret_cast<uint32_t*>(ws + a.off_csize);
    w.vid = reinterpret_cast<uint32_t*>(ws + a.off_vid);
    w.vsize = reinterpret_cast<uint32_t*>(ws + a.off_vsize);
    w.voldest = reinterpret_cast<uint32_t*>(ws + a.off_voldest);
    w.rid = reinterpret_cast<uint32_t*>(ws + a.off_rid);
    w.rdist = reinterpret_cast<float*>(ws + a.off_rdist);
    w.bar = reinterpret_cast<uint64_t*>(ws + a.off_bar);
    w.parity = 0;
    if (lane == 0) mbar_init(w.bar, 1);
    __syncwarp();
    const float kInf = __int_as_float(0x7f800000);

    for (;;) {
        uint32_t q = 0;
        if (lane == 0) q = atomicAdd(a.work_counter, 1u);
        q = __shfl_sync(kFull, q, 0);
        if (q >= a.nq) break;

        const float* gq = a.queries + (size_t)q * a.d;
        for (uint32_t i = lane; i < a.ld; i += 32) w.sq[i] = i < a.d ? gq[i] : 0.0f;
        for (uint32_t i = lane; i < a.m; i += 32) {
            w.csize[i] = 0;
            w.vsize[i] = 0;
            w.voldest[i] = 0;
        }
        __syncwarp();

        uint32_t hops = 0, evals = 0, evictions = 0, examined = 0, ctotal = 0, rn = 0;

        // 32 uniform start draws with replacement; best by closer (:57-63)
        const uint64_t s0 = fork_state(a.seed, a.qbase + q);
        const uint32_t v = draw_below(s0, (uint32_t)lane, a.n);
        float sd = gather_distances<METRIC>(w, a, true, v, lane);
        uint32_t si = v;
        warp_argmin(sd, si);
        evals += 32;
        r_push(w, rn, si, sd, lane);
        c_push(w, a, si, sd, ctotal, evictions, lane);
        float rfar = w.rdist[rn - 1];

        while (ctotal > 0 && hops < a.hop_limit) {  // :73
            ++hops;
            float pd;
            uint32_t u;
            c_pop_min(w, a, pd, u, ctotal, lane);
            if (pd > __fadd_rn(rfar, a.delta)) break;  // :79
            v_add(w, a, u, lane);
            const uint32_t deg = __ldg(a.degcut + u);
            examined += deg;
            const uint32_t* arow = a.adj + (size_t)u * a.R;
            for (uint32_t base = 0; base < deg; base += 32) {
                const uint32_t j = base + lane;
                const bool valid = j < deg;
                const uint32_t e = valid ? __ldg(arow + j) : kInvalid;
                const bool inV = valid && v_contains(w, a, e);
                const bool inC = valid && !inV && c_contains(w, a, e);
                const bool need = valid && !inV && !inC;
                float dist = gather_distances<METRIC>(w, a, need, e, lane);
                unsigned pending = __ballot_sync(kFull, need);
                unsigned revivable = __ballot_sync(kFull, inC);
                evals += __popc(pending);
                while (pending) {
                    const bool ok = ((pending >> lane) & 1u) && (dist < rfar || rn < a.k);
                    const unsigned adm = __ballot_sync(kFull, ok);
                    if (adm == 0) break;
                    const int p = __ffs(adm) - 1;
                    const uint32_t ep = __shfl_sync(kFull, e, p);
                    const float dp = __shfl_sync(kFull, dist, p);
                    r_push(w, rn, ep, dp, lane);
                    const uint32_t gone = c_push(w, a, ep, dp, ctotal, evictions, lane);
                    if (rn > a.k) --rn;  // pop_furthest
                    rfar = rn ? w.rdist[rn - 1] : kInf;
                    pending &= (p == 31) ? 0u : (~0u << (p + 1));
                    if (gone != kInvalid) {
                        const unsigned hit = __ballot_sync(
                            kFull, lane > p && ((revivable >> lane) & 1u) && e == gone);
                        if (hit) {
                            const int h = __ffs(hit) - 1;
                            if (lane == h)
                                dist = distance_exact_generic<METRIC>(
                                    w.sq, a.vec + (size_t)e * a.ld, a.d);
                            revivable &= ~(1u << h);
                            pending |= (1u << h);
                            ++evals;
                        }
                    }
                }
            }
        }

        uint32_t* oi = a.out_ids + (size_t)q * a.k;
        float* od = a.out_dists ? a.out_dists + (size_t)q * a.k : nullptr;
        for (uint32_t i = lane; i < a.k; i += 32) {
            oi[i] = i < rn ? w.rid[i] : kInvalid;
            if (od) od[i] = i < rn ? w.rdist[i] : kInf;
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
