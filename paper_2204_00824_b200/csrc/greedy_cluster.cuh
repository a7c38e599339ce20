// Small-batch multi-start greedy search (paper Alg. 1), latency-oriented form:
// one CTA per (query, walk), one thread-block CLUSTER per query.
//
// Inside a CTA, one hop's lambda-prefix (up to deg_cut[u] edges) is spread over
// the CTA's warps: warp w evaluates groups w, w+W, ... of 32 edges (lane = edge
// position mod 32, exactly the reference's lane mapping, greedy_search.cpp:49-58)
// and keeps its per-lane strict-< minimum together with the group index; the
// partials are combined in shared memory as min-by-(dist, group) — the
// reference's sequential lane_update over groups in order (rank_list.cpp:8-18)
// lets an earlier group keep a tie, which is exactly "smaller group wins".  Warp 0
// then runs merge_halves / next-node selection (warp_merge_halves) and the hop
// loop continues with the whole CTA.
//
// The t0 walks of a query run on the t0 CTAs of one cluster (t0 <= 16; 8 is the
// portable limit, up to 16 with the non-portable attribute).  When all walks are
// done, CTA rank 0 reads every walk's 32-slot R_ij from its siblings' shared
// memory over DSMEM, pools the finite entries, sorts by (dist, id), drops
// adjacent duplicate ids and writes the first k (greedy_search.cpp:85-103) — no
// second kernel, no global round trip.  For t0 > 16 the same kernel writes the
// walks to global memory and greedy_merge_kernel finishes.
#pragma once

#include <cooperative_groups.h>

#include "greedy.cuh"

namespace tsdg_dev {

namespace cg = cooperative_groups;

constexpr int kGcWarps = 4;
constexpr int kGcThreads = kGcWarps * 32;

struct GcArgs {
    const float* vec;
    const uint32_t* adj;
    const uint32_t* degcut;
    const float* queries;
    uint32_t ld, R, n, d;
    uint32_t nq, t0, hop_limit, k;
    uint64_t seed;
    const uint64_t* walk_states;  // optional explicit RNG state per walk
    uint32_t* out_ids;
    float* out_dists;
    uint32_t* out_counts;
    tsdg_query_stats* out_stats;
    uint32_t* walk_ids;  // non-cluster mode
    float* walk_dists;
    uint32_t* walk_hops;
    uint32_t* walk_evals;
    int cluster;         // 1: the t0 CTAs of a query form one cluster
    uint32_t merge_warp;    // 1: warp 0 only combines / merges, warps 1.. evaluate the
                            // hop's edges (its merge then overlaps their gathers)
    uint32_t slice;         // edges per evaluating warp per round (16 or 32)
    uint32_t early_next;    // 1: next node from the evaluating warps' minima
    uint32_t adj_prefetch;  // 1: L2-prefetch the adjacency head + deg_cut of every
                            // evaluated node (the next hop's u is one of them)
    uint32_t share0;        // 1: warp 0 has no slab of its own (uses warp 1's: it
                            // gathers only in select_start, before warp 1 starts)
    uint32_t spec_next;     // 1: the evaluating warps run hop t+1 while warp 0 merges
                            // hop t (dropped if that merge changed nothing)
    uint32_t npow2;      // pool size for the in-cluster merge
    uint32_t dch, slots;
    uint32_t stage;       // host: StageKind the kernel was chosen for
    const void* tmap;     // kStageG4: tensor map of vec (global memory)
    uint32_t gpitch;      // kStageG4: floats between 4-slot groups
    uint32_t off_query, off_stage, off_bar, off_ctl, off_list, off_pool, off_rowid, off_pos;
};

struct GcCtl {
    uint32_t u;
    uint32_t improved;
    uint32_t imp[2];  // spec_next: hop t's merge result in imp[t & 1]
    uint32_t hops;
    uint32_t evals;
    uint32_t u_next;  // next node, published before the merge (L2 warm-up)
    // per evaluating warp: its smallest distance of the hop (orderable key), the id
    // holding it and how many candidates share it (the early next-node pick); two
    // sets, by hop parity (with spec_next the next hop's values arrive while this
    // hop's are still being read)
    uint32_t best_k[8];
    uint32_t best_i[8];
    uint32_t best_n[8];
};

// float -> uint32 with the same order (closer() on distances; -0 == +0)
__device__ __forceinline__ uint32_t gc_fkey(float d) {
    uint32_t b = __float_as_uint(d);
    if ((b << 1) == 0) b = 0;
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ void cluster_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}

// Output targets of one query (device memory, or mapped host memory on the
// zero-copy host-pointer path).
struct GcOut {
    uint32_t* ids;  // k entries for this query
    float* dists;   // or nullptr
    uint32_t* count;
    tsdg_query_stats* stats;  // or nullptr
};

// Shared-memory views of one CTA (carved by the host, GcArgs::off_*).
struct GcSmem {
    float* sq;
    GcCtl* ctl;
    float* list_d;
    uint32_t* list_i;
    float* pool_d;     // rank 0: the t0 walk lists, pushed by the walks over DSMEM
    uint32_t* pool_i;
    uint32_t* scan;
    uint32_t* walk_cnt;  // rank 0: 2 x t0 (hops, evals) pushed by the walks
    float* pos_d;        // distance / id by adjacency position (R entries each), two
    uint32_t* pos_i;     // sets by hop parity: set b at pos_d + 2 R b, pos_i + 2 R b
};

__device__ __forceinline__ GcSmem gc_smem(const GcArgs& a, unsigned char* smem_raw) {
    GcSmem m;
    m.sq = reinterpret_cast<float*>(smem_raw + a.off_query);
    m.pos_d = reinterpret_cast<float*>(smem_raw + a.off_pos);
    m.pos_i = reinterpret_cast<uint32_t*>(smem_raw + a.off_pos) + a.R;
    m.ctl = reinterpret_cast<GcCtl*>(smem_raw + a.off_ctl);
    m.list_d = reinterpret_cast<float*>(smem_raw + a.off_list);
    m.list_i = reinterpret_cast<uint32_t*>(smem_raw + a.off_list + 32 * 4);
    m.pool_d = reinterpret_cast<float*>(smem_raw + a.off_pool);
    m.pool_i = reinterpret_cast<uint32_t*>(smem_raw + a.off_pool + a.npow2 * 4);
    m.scan = m.pool_i + a.npow2;
    m.walk_cnt = m.scan + kGcThreads + 1;
    return m;
}

// The next hop expands one of the nodes evaluated in this hop (the closest of
// R_temp), so their deg_cut entries and adjacency heads can be pulled into L2 as soon
// as their ids are known.  Off by default (TSDG_GC_ADJ_PREFETCH=1): on C2 it moved
// batch-1/8/64 latency by < 1% — the next hop's adjacency load already overlaps the
// warp-0 merge, so it is not on the critical path.
__device__ __forceinline__ void gc_prefetch_adj(const GcArgs& a, bool valid, uint32_t e) {
    if (!a.adj_prefetch || !valid) return;
    const uint32_t* row = a.adj + (size_t)e * a.R;
    prefetch_l2(row);
    if (a.R > 32) prefetch_l2(row + 32);
    prefetch_l2(a.degcut + e);
}

// One walk (CTA) of query q: select_start + hops + (cluster mode) the in-cluster merge
// of the t0 walks into `o`.  gq: the query (any memory space the SM can read: device
// memory, or mapped host memory); s: the walk's RNG stream index.
template <int METRIC, bool FAST, int STAGE>
__device__ __forceinline__ void gc_query(const GcArgs& a, const GcSmem& m, WarpStage& w,
                                         uint32_t s, uint32_t walk, const float* gq,
                                         const GcOut& o) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float* sq = m.sq;
    GcCtl* ctl = m.ctl;
    const Geom g{a.vec, a.ld, a.d, a.dch, a.slots, 0, a.tmap, a.gpitch};
    const float kInf = __int_as_float(0x7f800000);

    TR_MARK(0)
    // the walks push into rank 0's shared memory when they end: arrive now, wait
    // before the push (every CTA of the cluster has started by then)
    if (a.cluster) cluster_arrive_relaxed();
    for (uint32_t i = threadIdx.x; i < a.ld; i += blockDim.x) sq[i] = i < a.d ? gq[i] : 0.0f;
    __syncthreads();
    TR_MARK(1)

    // select_start (greedy_search.cpp:12-25) by warp 0
    if (warp == 0) {
        const uint64_t st = a.walk_states ? a.walk_states[walk] : fork_state(a.seed, s);
        const uint32_t v = draw_below(st, (uint32_t)lane, a.n);
        gc_prefetch_adj(a, true, v);
        float sd = gather_eval<METRIC, FAST, STAGE>(w, g, true, v, lane);
        uint32_t si = v;
        warp_argmin(sd, si);
        if (lane == 0) {
            ctl->u = si;
            ctl->improved = 1;
            ctl->imp[0] = 1;
            ctl->imp[1] = 1;
            ctl->hops = 0;
            ctl->evals = 32;
        }
    }
    __syncthreads();

    float rd = kInf;  // R_ij slot `lane` (warp 0)
    uint32_t ri = kInvalid;
    uint32_t t = 0;
    // Pipelined hops (whole rows in one round): each evaluating warp's first slice of
    // the next hop is issued as soon as the next node is known — while warp 0 runs
    // merge_halves — and completed at the top of the next hop.
    const bool pipe = a.ld <= a.dch && a.slots >= a.slice;  // TMA or LDGSTS split gathers
    // Evaluating warps: all, or warps 1.. when warp 0 is kept for combine + merge (its
    // merge then overlaps their gathers).  The hop's edges are spread over them in
    // slices of a.slice positions (warp ew takes positions r*nev*SL + ew*SL + [0, SL)
    // in round r).  Measured on C2 (batch 1, t0=10): slices of 32 / 28 / 24 / 20 / 16 /
    // 8 take 51 / 52 / 54 / 57 / 60 / 77 us — narrower slices push the ~58-edge
    // prefix into a second, un-pipelined round — so the default is 32 (TSDG_GC_SLICE).
    // Every evaluated position's distance lands in pos_d / pos_i and
    // warp 0 forms R_temp from them in the reference's order: lane j keeps the
    // strict-< minimum over positions j, j + 32, ... (lane_update, rank_list.cpp:8-18).
    const uint32_t ew0 = a.merge_warp ? 1u : 0u, nev = (uint32_t)kGcWarps - ew0;
    const bool evaluates = (uint32_t)warp >= ew0;
    const uint32_t ew = evaluates ? (uint32_t)warp - ew0 : 0u;
    const uint32_t SL = a.slice, P = nev * SL;
    const bool lane_on = evaluates && (uint32_t)lane < SL;
    const uint32_t j0 = lane_on ? ew * SL + lane : 0xFFFFFFFFu;  // round-0 position
    uint32_t deg = 0, e0 = kInvalid;
    // Speculative next hop (a.spec_next, with the merge warp, the early pick and the
    // pipelined gathers): there is no barrier at the end of a hop; warps 1-3 start
    // hop t+1 (its first slice is already in flight) while warp 0 still merges hop
    // t, and hop t+1's first barrier tells everyone whether that merge improved R_ij
    // — if not, the walk ended after hop t and hop t+1 is dropped (not counted, not
    // merged), so results and counters are the sequential loop's.  pos_* and the
    // early-pick words are double-buffered by hop parity.
    const bool spec = a.spec_next && a.merge_warp && a.early_next && pipe;
    uint32_t ucur = ctl->u;
    bool pend = false;  // this lane's row of the pre-issued slice
    if (pipe) {
        const uint32_t u = ctl->u;
        deg = __ldg(a.degcut + u);
        pend = j0 < deg;
        e0 = pend ? __ldg(a.adj + (size_t)u * a.R + j0) : kInvalid;
        gather_issue_s<STAGE>(w, g, pend, e0, lane);
        gc_prefetch_adj(a, pend, e0);
    }
    TR_MARK(2)
    PH_DECL
    PH_MARK(0)  // phase 0: query load + select_start
    while ((spec || ctl->improved) && t < a.hop_limit) {
        ++t;
        HOP_MARK(t, 0)
        const uint32_t u = spec ? ucur : ctl->u;
        const uint32_t hb = spec ? (t & 1u) : 0u;  // parity set of pos_* / best_*
        float* pos_d = m.pos_d + (size_t)hb * 2 * a.R;
        uint32_t* pos_i = m.pos_i + (size_t)hb * 2 * a.R;
        const uint32_t* arow = a.adj + (size_t)u * a.R;
        if (!pipe) {
            // deg and this warp's first adjacency slice load together (no deg -> row
            // dependency on the hop's critical path)
            e0 = j0 < a.R ? __ldg(arow + j0) : kInvalid;
            deg = __ldg(a.degcut + u);
        }
        const uint32_t ngroups = (deg + 31) / 32;
        // this warp's smallest distance of the hop (one REDUX per round), its holder
        // and its multiplicity
        uint32_t bk = 0xFFFFFFFFu, bi = kInvalid, bn = 0;
        auto track = [&](bool valid, float dist, uint32_t e) {
            const uint32_t key = valid ? gc_fkey(dist) : 0xFFFFFFFFu;
            const uint32_t mk = __reduce_min_sync(kFull, key);
            const unsigned hit = __ballot_sync(kFull, valid && key == mk);
            if (hit == 0u) return;  // warp-uniform
            const uint32_t mi = __shfl_sync(kFull, e, __ffs(hit) - 1);
            if (mk < bk) {
                bk = mk;
                bi = mi;
                bn = __popc(hit);
            } else if (mk == bk) {
                bn += __popc(hit);
                bi = min(bi, mi);
            }
        };
        if (pipe) {  // the first slice was issued during the previous hop's merge
            const float dist = gather_complete<METRIC, FAST, STAGE>(w, g, pend, lane);
            if (pend) {
                pos_d[j0] = dist;
                pos_i[j0] = e0;
            }
            if (a.early_next && evaluates) track(pend, dist, e0);
            pend = false;
            HOP_MARK(t, 1)
        }
        for (uint32_t r0 = pipe ? P : 0; evaluates && r0 < deg; r0 += P) {
            const uint32_t j = r0 + ew * SL + lane;
            const bool valid = lane_on && j < deg;
            const uint32_t e = valid ? (r0 == 0 ? e0 : __ldg(arow + j)) : kInvalid;
            gc_prefetch_adj(a, valid, e);
            const float dist = gather_eval<METRIC, FAST, STAGE>(w, g, valid, e, lane);
            if (valid) {
                pos_d[j] = dist;
                pos_i[j] = e;
            }
            if (a.early_next) track(valid, dist, e);
        }
        if (a.early_next && evaluates && lane == 0) {
            ctl->best_k[hb * 4 + ew] = bk;
            ctl->best_i[hb * 4 + ew] = bi;
            ctl->best_n[hb * 4 + ew] = bn;
        }
        PH_MARK(1)  // adjacency + gather + distances
        HOP_MARK(t, 2)
        __syncthreads();
        HOP_MARK(t, 3)
        if (spec && !ctl->imp[(t - 1) & 1u]) {  // hop t-1's merge found nothing new: hop t was
            --t;                       // speculative — the walk ended after hop t-1
            break;
        }
        PH_MARK(2)  // barrier: slowest warp's gather
        // The next node is the minimum of R_temp by closer (greedy_search.cpp:63-67).
        // When the hop's smallest distance is held by exactly one candidate, that
        // candidate wins its lane slot (nothing before it in the slot is as close) and
        // is the minimum of R_temp: every warp takes it from the evaluating warps'
        // minima right after the barrier and starts the next adjacency load while warp
        // 0 forms R_temp and merges.  A tie at the minimum falls back to warp 0's
        // selection from R_temp (one more barrier).
        uint32_t un = kInvalid;
        bool early = false;
        if (a.early_next) {
            uint32_t gk = 0xFFFFFFFFu, gid = kInvalid, gn = 0;
            for (uint32_t v = 0; v < nev; ++v) {
                const uint32_t k2 = ctl->best_k[hb * 4 + v];
                if (k2 < gk) {
                    gk = k2;
                    gid = ctl->best_i[hb * 4 + v];
                    gn = ctl->best_n[hb * 4 + v];
                } else if (k2 == gk) {
                    gn += ctl->best_n[hb * 4 + v];
                }
            }
            early = gn == 1u;  // CTA-uniform
            un = gid;
        }
        // warp 0 forms R_temp (and, without the early pick, the next node)
        float td = kInf;
        uint32_t ti = kInvalid, ni = kInvalid;
        if (warp == 0) {
            for (uint32_t gi = 0; gi < ngroups; ++gi) {
                const uint32_t j = gi * 32 + lane;
                if (j < deg) {
                    const float d = pos_d[j];
                    if (d < td) {  // strict: an earlier group keeps a tie
                        td = d;
                        ti = pos_i[j];
                    }
                }
            }
            if (early) {
                ni = un;  // the minimum of R_temp (see above)
            } else {
                float nd = td;
                ni = ti;
                warp_argmin(nd, ni);
                if (lane == 0) ctl->u_next = ni;
            }
        }
        if (!early) {
            __syncthreads();
            un = ctl->u_next;
        }
        HOP_MARK(t, 4)
        // next hop (wasted only if the walk stops here): deg + this warp's first group
        uint32_t ndeg = 0, ne = kInvalid;
        if (pipe && un != kInvalid) {
            ndeg = __ldg(a.degcut + un);
            ne = j0 < a.R ? __ldg(a.adj + (size_t)un * a.R + j0) : kInvalid;
        }
        if (warp == 0) {
            const bool updated = warp_merge_halves(rd, ri, td, ti, lane);
            if (lane == 0) {
                if (ni != kInvalid) ctl->u = ni;
                ctl->improved = updated ? 1u : 0u;
                ctl->imp[t & 1u] = updated ? 1u : 0u;
                ctl->evals += deg;
            }
            HOP_MARK(t, 5)
        } else if (!pipe && un != kInvalid) {
            // while warp 0 merges, the other warps pull the next hop's deg_cut entry,
            // adjacency row and neighbour rows into L2 (wasted only on the last hop)
            const uint32_t* nrow = a.adj + (size_t)un * a.R;
            const uint32_t nd = __ldg(a.degcut + un);
            const uint32_t rowb = a.ld * 4u;
            for (uint32_t j = (uint32_t)(warp - 1) * 32 + lane; j < nd; j += (kGcWarps - 1) * 32) {
                const char* r = reinterpret_cast<const char*>(a.vec + (size_t)__ldg(nrow + j) * a.ld);
                for (uint32_t o = 0; o < rowb; o += 128) prefetch_l2(r + o);
            }
        }
        if (pipe && un != kInvalid) {
            deg = ndeg;
            pend = j0 < ndeg;
            e0 = pend ? ne : kInvalid;
            if (e0 == 0xFFFFFFFEu) asm volatile("" ::: "memory");  // (phases build: e0 loaded)
            if (warp != 0) {
                HOP_MARK(t, 5)
            }
            PH_MARK(3)  // combine + (warp 0) merge_halves / (others) next adjacency
            gather_issue_s<STAGE>(w, g, pend, e0, lane);
            gc_prefetch_adj(a, pend, e0);
            PH_MARK(5)  // next hop's row copies issued
            HOP_MARK(t, 6)
        } else {
            PH_MARK(3)
        }
        if (spec) ucur = un;  // no end-of-hop barrier (see above)
        else __syncthreads();
        HOP_MARK(t, 7)
        TR_MARK(3 + t)
        PH_MARK(4)  // barrier
    }
    if (pipe) gather_complete<METRIC, FAST, STAGE>(w, g, pend, lane);  // drain a pre-issued group

    if (!a.cluster) {
        if (warp == 0) {
            a.walk_ids[(size_t)walk * 32 + lane] = ri;
            a.walk_dists[(size_t)walk * 32 + lane] = rd;
            if (lane == 0) {
                a.walk_hops[walk] = t;
                a.walk_evals[walk] = ctl->evals;
            }
        }
        return;
    }

    // ---- in-cluster merge (CTA rank 0 of the query's cluster) ----------------------
    // each walk pushes its sorted 32-slot list and counters into rank 0's shared
    // memory over DSMEM as soon as it ends, so the merge reads local memory only
    cg::cluster_group cluster = cg::this_cluster();
    cluster_wait();
    if (warp == 0) {
        float* rpd = cluster.map_shared_rank(m.pool_d, 0);
        uint32_t* rpi = cluster.map_shared_rank(m.pool_i, 0);
        rpd[s * 32 + lane] = ri != kInvalid ? rd : kInf;
        rpi[s * 32 + lane] = ri;
        if (lane == 0) {
            uint32_t* rwc = cluster.map_shared_rank(m.walk_cnt, 0);
            rwc[2 * s] = t;
            rwc[2 * s + 1] = ctl->evals;
        }
    }
    TR_MARK(27)
    cluster.sync();
    TR_MARK(28)
    PH_MARK(6)  // waiting for the slowest walk of the query
    if (cluster.block_rank() == 0) {
        float* pd = m.pool_d;
        uint32_t* pi = m.pool_i;
        uint32_t* scan = m.scan;
        uint32_t hsum = 0, esum = 0;
        if (warp == 0) {
            for (uint32_t r = lane; r < a.t0; r += 32) {
                hsum += m.walk_cnt[2 * r];
                esum += m.walk_cnt[2 * r + 1];
            }
            hsum = __reduce_add_sync(kFull, hsum);
            esum = __reduce_add_sync(kFull, esum);
        }
        uint32_t c = 0;
        if (a.k <= 64 && a.t0 <= 32) {
            // the t0 lists are sorted: a warp k-way merge of their heads (k steps)
            if (warp == 0) {
                c = warp_kway_unique(pd, pi, a.t0, 32, 32, a.k, lane,
                                     [&](uint32_t i, uint32_t id, float dd) {
                                         if (lane == 0) {
                                             o.ids[i] = id;
                                             if (o.dists) o.dists[i] = dd;
                                         }
                                     });
                for (uint32_t i = c + lane; i < a.k; i += 32) {
                    o.ids[i] = kInvalid;
                    if (o.dists) o.dists[i] = kInf;
                }
            }
        } else {
            for (uint32_t i = a.t0 * 32 + threadIdx.x; i < a.npow2; i += blockDim.x) {
                pd[i] = kInf;
                pi[i] = kInvalid;
            }
            __syncthreads();
            for (uint32_t kk = 2; kk <= a.npow2; kk <<= 1) {
                for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
                    for (uint32_t i = threadIdx.x; i < a.npow2; i += blockDim.x) {
                        const uint32_t p = i ^ j;
                        if (p > i) {
                            const bool up = (i & kk) == 0;
                            const bool p_first = closer(pd[p], pi[p], pd[i], pi[i]);
                            if (p_first == up) {
                                const float td = pd[i];
                                const uint32_t ti = pi[i];
                                pd[i] = pd[p];
                                pi[i] = pi[p];
                                pd[p] = td;
                                pi[p] = ti;
                            }
                        }
                    }
                    __syncthreads();
                }
            }
            const uint32_t per = (a.npow2 + blockDim.x - 1) / blockDim.x;
            const uint32_t b0 = threadIdx.x * per;
            uint32_t cnt = 0;
            for (uint32_t i = b0; i < b0 + per && i < a.npow2; ++i)
                cnt += (pi[i] != kInvalid && (i == 0 || pi[i] != pi[i - 1])) ? 1u : 0u;
            scan[threadIdx.x] = cnt;
            __syncthreads();
            if (threadIdx.x == 0) {
                uint32_t run = 0;
                for (uint32_t x = 0; x < blockDim.x; ++x) {
                    const uint32_t cc = scan[x];
                    scan[x] = run;
                    run += cc;
                }
                scan[blockDim.x] = run;
            }
            __syncthreads();
            uint32_t pos = scan[threadIdx.x];
            for (uint32_t i = b0; i < b0 + per && i < a.npow2; ++i) {
                if (pi[i] != kInvalid && (i == 0 || pi[i] != pi[i - 1])) {
                    if (pos < a.k) {
                        o.ids[pos] = pi[i];
                        if (o.dists) o.dists[pos] = pd[i];
                    }
                    ++pos;
                }
            }
            const uint32_t uniq = scan[blockDim.x];
            c = uniq < a.k ? uniq : a.k;
            for (uint32_t i = c + threadIdx.x; i < a.k; i += blockDim.x) {
                o.ids[i] = kInvalid;
                if (o.dists) o.dists[i] = kInf;
            }
        }
        if (threadIdx.x == 0) {
            if (o.count) *o.count = c;
            if (o.stats) {
                tsdg_query_stats st;
                st.hops = hsum;
                st.distance_evals = esum;
                st.queue_evictions = 0;
                st.edges_examined = esum - 32u * a.t0;
                *o.stats = st;
            }
        }
    }
    PH_MARK(7)  // rank 0: pool merge
    TR_MARK(29)
    cluster.sync();  // rank 0's pool is free again before the walks of a next query push
    TR_MARK(30)
}

template <int METRIC, bool FAST, int STAGE>
__global__ void __launch_bounds__(kGcThreads) greedy_cta_kernel(const GcArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t walk = blockIdx.x;
    const uint32_t q = walk / a.t0, s = walk % a.t0;
    const GcSmem m = gc_smem(a, smem_raw);
    WarpStage w;
    w.sq = m.sq;
    const uint32_t slab = a.share0 ? (warp > 0 ? warp - 1 : 0) : warp;
    w.stage = reinterpret_cast<float*>(smem_raw + a.off_stage) +
              (size_t)slab * (STAGE == kStageG4 ? a.slots / 4 * a.gpitch : a.slots * (a.dch + 4));
    w.bar = reinterpret_cast<uint64_t*>(smem_raw + a.off_bar) + warp;
    w.parity = 0;
    w.rowid = STAGE != kStageTma ? reinterpret_cast<uint32_t*>(smem_raw + a.off_rowid) + warp * 32 : nullptr;
    if (lane == 0) mbar_init(w.bar, 1);
    GcOut o;
    o.ids = a.out_ids ? a.out_ids + (size_t)q * a.k : nullptr;
    o.dists = a.out_dists ? a.out_dists + (size_t)q * a.k : nullptr;
    o.count = a.out_counts ? a.out_counts + q : nullptr;
    o.stats = a.out_stats ? a.out_stats + q : nullptr;
    gc_query<METRIC, FAST, STAGE>(a, m, w, s, walk, a.queries + (size_t)q * a.d, o);
}

}  // namespace tsdg_dev
