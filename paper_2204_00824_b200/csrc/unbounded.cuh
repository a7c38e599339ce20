// Best-first search with the reference's UNBOUNDED stand-ins (BestFirstParams::
// unbounded = true; bestfirst_search.cpp:14-47, selected at :121-124): an exact
// priority queue ordered by (dist, id) and exact visited / queued sets, instead
// of the lossy segmented C and V.  This is the "sequential CPU-style
// configuration" the reference uses to check the segmented design; it is not a
// throughput path.
//
// One warp per query with a private arena in global memory:
//   * open-addressing hash table of ids with a state per slot (1 = queued,
//     2 = expanded).  An id only ever moves queued -> expanded (a popped node is
//     either expanded or the search stops), so no deletions are needed; the
//     capacity covers every id the search can touch (<= distance evals + 1).
//   * binary min-heap of (dist, id) pairs — std::set<pair<float,NodeId>> order —
//     maintained by lane 0.
// Distances use the same staged exact/fast evaluation as bf_kernel; admission is
// the same sequential replay (no evictions can occur).
#pragma once

#include "bestfirst.cuh"

namespace tsdg_dev {

struct UbArgs {
    const float* vec;
    const uint32_t* adj;
    const uint32_t* degcut;
    const float* queries;
    uint32_t ld, R, n, d;
    uint32_t nq;
    uint64_t qbase;
    uint32_t k, hop_limit;
    float delta;
    uint64_t seed;
    uint32_t* out_ids;
    float* out_dists;
    uint32_t* out_counts;
    tsdg_query_stats* out_stats;
    uint32_t* work_counter;
    uint32_t work_base;     // counter value at launch (tsdg_gpu.cu next_counter)
    uint32_t dch, slots;
    // per-warp arena in global memory
    uint32_t* hkeys;   // [warps][hcap]
    uint8_t* hstate;   // [warps][hcap]
    float* heap_d;     // [warps][qcap]
    uint32_t* heap_i;  // [warps][qcap]
    uint32_t* rid;     // [warps][k + 2]
    float* rdist;      // [warps][k + 2]
    uint32_t hcap, qcap;
    int* overflow;     // set if an arena bound is hit (host reports an error)
    uint32_t warp_smem, off_query, off_stage, off_bar;
};

__device__ __forceinline__ uint32_t ub_hash(uint32_t id, uint32_t cap) {
    return (uint32_t)(mix64(id) & (cap - 1));
}

// state of id in the warp's table (0 = absent); per-lane lookup
__device__ __forceinline__ uint32_t ub_state(const uint32_t* keys, const uint8_t* state,
                                             uint32_t cap, uint32_t id) {
    uint32_t h = ub_hash(id, cap);
    for (uint32_t probe = 0; probe < cap; ++probe) {
        const uint32_t kk = keys[h];
        if (kk == id) return state[h];
        if (kk == kInvalid) return 0;
        h = (h + 1) & (cap - 1);
    }
    return 0;
}
// lane-0 insert or update
__device__ __forceinline__ bool ub_set(uint32_t* keys, uint8_t* state, uint32_t cap, uint32_t id,
                                       uint8_t st) {
    uint32_t h = ub_hash(id, cap);
    for (uint32_t probe = 0; probe < cap; ++probe) {
        const uint32_t kk = keys[h];
        if (kk == id || kk == kInvalid) {
            keys[h] = id;
            state[h] = st;
            return true;
        }
        h = (h + 1) & (cap - 1);
    }
    return false;
}

__device__ __forceinline__ bool heap_less(float da, uint32_t ia, float db, uint32_t ib) {
    return closer(da, ia, db, ib);
}
__device__ void heap_push(float* hd, uint32_t* hi, uint32_t& size, float d, uint32_t id) {
    uint32_t i = size++;
    while (i > 0) {
        const uint32_t p = (i - 1) >> 1;
        if (!heap_less(d, id, hd[p], hi[p])) break;
        hd[i] = hd[p];
        hi[i] = hi[p];
        i = p;
    }
    hd[i] = d;
    hi[i] = id;
}
__device__ void heap_pop(float* hd, uint32_t* hi, uint32_t& size, float& d, uint32_t& id) {
    d = hd[0];
    id = hi[0];
    --size;
    const float ld = hd[size];
    const uint32_t li = hi[size];
    uint32_t i = 0;
    for (;;) {
        const uint32_t c = 2 * i + 1;
        if (c >= size) break;
        uint32_t m = c;
        if (c + 1 < size && heap_less(hd[c + 1], hi[c + 1], hd[c], hi[c])) m = c + 1;
        if (!heap_less(hd[m], hi[m], ld, li)) break;
        hd[i] = hd[m];
        hi[i] = hi[m];
        i = m;
    }
    hd[i] = ld;
    hi[i] = li;
}

template <int METRIC, bool FAST>
__global__ void __launch_bounds__(32) bf_unbounded_kernel(const UbArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const uint32_t gw = blockIdx.x;  // one warp per CTA
    WarpStage w;
    w.sq = reinterpret_cast<float*>(smem_raw + a.off_query);
    w.stage = reinterpret_cast<float*>(smem_raw + a.off_stage);
    w.bar = reinterpret_cast<uint64_t*>(smem_raw + a.off_bar);
    w.parity = 0;
    w.rowid = nullptr;
    if (lane == 0) mbar_init(w.bar, 1);
    __syncwarp();
    const Geom g{a.vec, a.ld, a.d, a.dch, a.slots};
    const float kInf = __int_as_float(0x7f800000);
    uint32_t* keys = a.hkeys + (size_t)gw * a.hcap;
    uint8_t* hst = a.hstate + (size_t)gw * a.hcap;
    float* hd = a.heap_d + (size_t)gw * a.qcap;
    uint32_t* hi = a.heap_i + (size_t)gw * a.qcap;
    uint32_t* rid = a.rid + (size_t)gw * (a.k + 2);
    float* rdist = a.rdist + (size_t)gw * (a.k + 2);

    for (;;) {
        uint32_t q = 0;
        if (lane == 0) q = atomicAdd(a.work_counter, 1u) - a.work_base;
        q = __shfl_sync(kFull, q, 0);
        if (q >= a.nq) break;
        const float* gq = a.queries + (size_t)q * a.d;
        __syncwarp();
        for (uint32_t i = lane; i < a.ld; i += 32) w.sq[i] = i < a.d ? gq[i] : 0.0f;
        for (uint32_t i = lane; i < a.hcap; i += 32) keys[i] = kInvalid;
        __syncwarp();
        __threadfence_block();

        uint32_t hops = 0, evals = 0, examined = 0, qsize = 0, rn = 0, used = 0;
        bool over = false;
        const uint64_t s0 = fork_state(a.seed, a.qbase + q);
        const uint32_t v0 = draw_below(s0, (uint32_t)lane, a.n);
        float sd = gather_eval<METRIC, FAST, kStageTma>(w, g, true, v0, lane);
        uint32_t si = v0;
        warp_argmin(sd, si);
        evals += 32;
        if (lane == 0) {
            rid[0] = si;
            rdist[0] = sd;
            heap_push(hd, hi, qsize, sd, si);
            over |= !ub_set(keys, hst, a.hcap, si, 1);
            ++used;
        }
        rn = 1;
        qsize = __shfl_sync(kFull, qsize, 0);
        __syncwarp();
        __threadfence_block();
        float rfar = sd;

        while (qsize > 0 && hops < a.hop_limit) {
            ++hops;
            float pd = 0.f;
            uint32_t u = 0;
            if (lane == 0) {
                heap_pop(hd, hi, qsize, pd, u);
                ub_set(keys, hst, a.hcap, u, 2);  // queued -> expanded
            }
            pd = __shfl_sync(kFull, pd, 0);
            u = __shfl_sync(kFull, u, 0);
            qsize = __shfl_sync(kFull, qsize, 0);
            __syncwarp();
            __threadfence_block();
            if (pd > __fadd_rn(rfar, a.delta)) break;
            const uint32_t deg = __ldg(a.degcut + u);
            examined += deg;
            const uint32_t* arow = a.adj + (size_t)u * a.R;
            for (uint32_t base = 0; base < deg; base += 32) {
                const uint32_t j = base + lane;
                const bool valid = j < deg;
                const uint32_t e = valid ? __ldg(arow + j) : kInvalid;
                const bool seen = valid && ub_state(keys, hst, a.hcap, e) != 0;
                const bool need = valid && !seen;
                float dist = gather_eval<METRIC, FAST, kStageTma>(w, g, need, e, lane);
                unsigned pending = __ballot_sync(kFull, need);
                evals += __popc(pending);
                while (pending) {
                    const bool ok = ((pending >> lane) & 1u) && (dist < rfar || rn < a.k);
                    const unsigned adm = __ballot_sync(kFull, ok);
                    if (adm == 0) break;
                    const int p = __ffs(adm) - 1;
                    const uint32_t ep = __shfl_sync(kFull, e, p);
                    const float dp = __shfl_sync(kFull, dist, p);
                    if (lane == 0) {
                        // TopK push (segmented.cpp:94-101): dedup, sorted insert
                        bool dup = false;
                        for (uint32_t i = 0; i < rn; ++i) dup |= rid[i] == ep;
                        if (!dup) {
                            uint32_t pos = rn;
                            while (pos > 0 && closer(dp, ep, rdist[pos - 1], rid[pos - 1])) {
                                rid[pos] = rid[pos - 1];
                                rdist[pos] = rdist[pos - 1];
                                --pos;
                            }
                            rid[pos] = ep;
                            rdist[pos] = dp;
                            ++rn;
                        }
                        if (qsize + 1 >= a.qcap || used + 1 >= a.hcap / 2) over = true;
                        else {
                            heap_push(hd, hi, qsize, dp, ep);
                            over |= !ub_set(keys, hst, a.hcap, ep, 1);
                            ++used;
                        }
                        if (rn > a.k) --rn;
                    }
                    rn = __shfl_sync(kFull, rn, 0);
                    qsize = __shfl_sync(kFull, qsize, 0);
                    __syncwarp();
                    __threadfence_block();
                    rfar = rn ? rdist[rn - 1] : kInf;
                    pending &= (p == 31) ? 0u : (~0u << (p + 1));
                }
            }
        }
        uint32_t* oi = a.out_ids + (size_t)q * a.k;
        float* od = a.out_dists ? a.out_dists + (size_t)q * a.k : nullptr;
        for (uint32_t i = lane; i < a.k; i += 32) {
            oi[i] = i < rn ? rid[i] : kInvalid;
            if (od) od[i] = i < rn ? rdist[i] : kInf;
        }
        if (lane == 0) {
            if (over) atomicExch(a.overflow, 1);
            if (a.out_counts) a.out_counts[q] = rn;
            if (a.out_stats) {
                tsdg_query_stats st;
                st.hops = hops;
                st.distance_evals = evals;
                st.queue_evictions = 0;
                st.edges_examined = examined;
                a.out_stats[q] = st;
            }
        }
        __syncwarp();
    }
}

}  // namespace tsdg_dev
