// Small-batch multi-start greedy search (paper Alg. 1), deterministic.
//
// greedy_walk_kernel: one warp per (query, walk s).  Restates greedy_search_once
// (greedy_search.cpp:27-72) with select_start (:12-25):
//   - 32 start draws from stream Rng64(seed).fork(s) (the same streams for every
//     query of a call, greedy_search.cpp:83,88) — or an explicit state per walk;
//   - per hop, the lambda-prefix of u streams through the 32 lanes in groups of 32
//     (lane = position mod 32): lane j keeps its own R_temp slot with the strict-<
//     per-lane minimum of lane_update (rank_list.cpp:8-18) in registers;
//   - merge_halves (rank_list.cpp:20-49) as a warp operation: bitonic sort of
//     R_temp, id-dedup of its best 16 finite entries against R_ij by shuffles,
//     then a bitonic merge of R_ij with the reversed new entries (6 steps);
//   - u <- closest of R_temp (not R_ij); stop when the merge changed nothing.
// Rows are staged with the same TMA bulk-copy gather as the best-first kernel,
// so distances are the reference's sequential fp32 values bit for bit.
//
// greedy_merge_kernel: one CTA per query merges the t0 walks' 32-slot lists:
// finite entries, sort by (dist, id), unique by id, first k
// (greedy_search.cpp:85-103).
#pragma once

#include "bestfirst.cuh"

namespace tsdg_dev {

constexpr int kGrWarps = 4;

struct GrArgs {
    const float* vec;
    const uint32_t* adj;
    const uint32_t* degcut;
    const float* queries;
    uint32_t ld, R, n, d;
    uint32_t nq, t0, hop_limit;
    uint64_t seed;
    const uint64_t* walk_states;  // optional: explicit RNG state per walk
    uint32_t* walk_ids;           // (nq*t0) x 32
    float* walk_dists;
    uint32_t* walk_hops;          // nq*t0
    uint32_t* walk_evals;
    uint32_t* work_counter;
    uint32_t work_base;     // counter value at launch (tsdg_gpu.cu next_counter)
    uint32_t dch, slots;
    uint32_t warp_smem, off_query, off_stage, off_bar, off_rowid;
    const void* tmap;   // kStageG4: tensor map of vec (global memory)
    uint32_t gpitch;    // kStageG4: floats between 4-slot groups
};

// merge_halves (rank_list.cpp:20-49).  (rd, ri): R_ij slot `lane` (sorted);
// (td, ti): R_temp slot `lane`.  Returns the warp-uniform "updated".
//
// The reference pools R_ij with the best 16 finite newcomers, keeping the closer
// copy of a repeated id, sorts the pool and keeps 32.  A repeated id always carries
// the same distance (a pure function of the query and the node), so "keep the
// closer copy" never replaces anything: the pool is R_ij plus the newcomers whose
// id is new.  Both parts are already sorted (R_ij by contract, the newcomers as a
// subsequence of the sorted R_temp), so instead of sorting 64 keys the warp forms
// the bitonic sequence R_ij ++ reverse(newcomers), keeps the lower half of one
// half-cleaner step (the 32 smallest) and sorts it with 5 more steps.
// Index of the n-th (0-based) set bit of m, which has more than n bits set: the
// largest p with popc(m below p) <= n, by a 5-step binary search (no __fns loop).
__device__ __forceinline__ int nth_set_bit(unsigned m, unsigned n) {
    int pos = 0;
#pragma unroll
    for (int b = 16; b > 0; b >>= 1) {
        if ((unsigned)__popc(m & ((1u << (pos + b)) - 1u)) <= n) pos += b;
    }
    return pos;
}

__device__ __forceinline__ bool warp_merge_halves(float& rd, uint32_t& ri, float td,
                                                  uint32_t ti, int lane) {
    warp_sort32(td, ti, lane);  // incoming, ascending
    // repeated ids: against R_ij, and within the newcomers (adjacent once sorted)
    const uint32_t prev = __shfl_up_sync(kFull, ti, 1);
    bool dup = lane > 0 && prev == ti;
    // membership of the 16 candidates (lanes 0-15) in R_ij: two MATCH.ANY rounds, the
    // upper 16 lanes carrying R_ij's lower / upper half (instead of 32 broadcasts)
    const uint32_t r_lo = __shfl_sync(kFull, ri, lane & 15), r_hi = __shfl_sync(kFull, ri, (lane & 15) + 16);
    const unsigned m_lo = __match_any_sync(kFull, lane < 16 ? ti : r_lo);
    const unsigned m_hi = __match_any_sync(kFull, lane < 16 ? ti : r_hi);
    dup |= ((m_lo | m_hi) & 0xFFFF0000u) != 0u;
    const unsigned vm = __ballot_sync(kFull, lane < 16 && ti != kInvalid && !dup);
    // lane L takes newcomer number 31 - L (the reversed, compacted newcomer list)
    const uint32_t want = 31u - (uint32_t)lane;
    const bool has = want < (uint32_t)__popc(vm);
    const int src = has ? nth_set_bit(vm, want) : 0;
    const float sd = __shfl_sync(kFull, td, src);
    const uint32_t sid = __shfl_sync(kFull, ti, src);
    float nd = rd;
    uint32_t ni = ri;
    if (has && closer(sd, sid, nd, ni)) {  // half-cleaner: lower half keeps the min
        nd = sd;
        ni = sid;
    }
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) {
        const float od = __shfl_xor_sync(kFull, nd, j);
        const uint32_t oi = __shfl_xor_sync(kFull, ni, j);
        cx(nd, ni, od, oi, (lane & j) == 0);
    }
    const bool changed = (nd != rd) || (ni != ri);
    rd = nd;
    ri = ni;
    return __any_sync(kFull, changed);
}

template <int METRIC, bool FAST, int STAGE>
__global__ void __launch_bounds__(kGrWarps * 32) greedy_walk_kernel(const GrArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    unsigned char* ws = smem_raw + (threadIdx.x >> 5) * a.warp_smem;
    WarpStage w;
    w.sq = reinterpret_cast<float*>(ws + a.off_query);
    w.stage = reinterpret_cast<float*>(ws + a.off_stage);
    w.bar = reinterpret_cast<uint64_t*>(ws + a.off_bar);
    w.parity = 0;
    w.rowid = STAGE == kStageG4 ? reinterpret_cast<uint32_t*>(ws + a.off_rowid) : nullptr;
    const Geom g{a.vec, a.ld, a.d, a.dch, a.slots, 0, a.tmap, a.gpitch};
    if (STAGE != kStageLdgsts) {
        if (lane == 0) mbar_init(w.bar, 1);
        __syncwarp();
    }
    const float kInf = __int_as_float(0x7f800000);
    const uint32_t nwalks = a.nq * a.t0;
    uint32_t cur_q = kInvalid;

    for (;;) {
        uint32_t wk = 0;
        if (lane == 0) wk = atomicAdd(a.work_counter, 1u) - a.work_base;
        wk = __shfl_sync(kFull, wk, 0);
        if (wk >= nwalks) break;
        const uint32_t q = wk / a.t0;
        const uint32_t s = wk % a.t0;
        if (q != cur_q) {
            __syncwarp();
            const float* gq = a.queries + (size_t)q * a.d;
            for (uint32_t i = lane; i < a.ld; i += 32) w.sq[i] = i < a.d ? gq[i] : 0.0f;
            cur_q = q;
            __syncwarp();
        }
        const uint64_t st = a.walk_states ? a.walk_states[wk] : fork_state(a.seed, s);

        // select_start (greedy_search.cpp:12-25)
        const uint32_t v = draw_below(st, (uint32_t)lane, a.n);
        float sd = gather_eval<METRIC, FAST, STAGE>(w, g, true, v, lane);
        uint32_t si = v;
        warp_argmin(sd, si);
        uint32_t u = si;
        uint32_t evals = 32, t = 0;

        float rd = kInf;
        uint32_t ri = kInvalid;
        bool improved = true;
        uint32_t deg = __ldg(a.degcut + u);
        uint32_t e_next = (uint32_t)lane < a.R ? __ldg(a.adj + (size_t)u * a.R + lane) : kInvalid;
        while (improved && t < a.hop_limit) {
            ++t;
            float td = kInf;
            uint32_t ti = kInvalid;
            const uint32_t* arow = a.adj + (size_t)u * a.R;
            for (uint32_t base = 0; base < deg; base += 32) {
                const uint32_t j = base + lane;
                const bool valid = j < deg;
                const uint32_t e = valid ? e_next : kInvalid;
                const uint32_t j2 = base + 32 + lane;
                e_next = (base + 32 < deg && j2 < a.R) ? __ldg(arow + j2) : kInvalid;
                const float dist = gather_eval<METRIC, FAST, STAGE>(w, g, valid, e, lane);
                if (valid && dist < td) {  // lane_update: strict <, earlier group keeps ties
                    td = dist;
                    ti = e;
                }
            }
            evals += deg;
            // next node = minimum of R_temp (greedy_search.cpp:63-67), known before
            // merge_halves: its deg_cut entry and first adjacency entries load while
            // the merge runs
            float nd = td;
            uint32_t ni = ti;
            warp_argmin(nd, ni);
            if (ni != kInvalid) u = ni;
            deg = __ldg(a.degcut + u);
            e_next = (uint32_t)lane < a.R ? __ldg(a.adj + (size_t)u * a.R + lane) : kInvalid;
            const bool updated = warp_merge_halves(rd, ri, td, ti, lane);
            improved = updated;
        }
        a.walk_ids[(size_t)wk * 32 + lane] = ri;
        a.walk_dists[(size_t)wk * 32 + lane] = rd;
        if (lane == 0) {
            a.walk_hops[wk] = t;
            a.walk_evals[wk] = evals;
        }
    }
}

// One CTA per query: pool the t0 x 32 walk slots, sort, unique, first k.
constexpr int kMergeThreads = 256;

// k-way merge of up to 32 lists sorted by (dist, id) (list r = entries
// [r*stride, r*stride + len); an invalid id ends a list) into the first k DISTINCT ids
// in (dist, id) order — the reference's pool sort + unique + first k
// (greedy_search.cpp:85-103) without sorting the pool: lane r holds list r's head and
// each step takes the warp arg-min.  A repeated id carries the same distance, so every
// list holding it has it at its head at that step and all of them advance together.
// Warp-uniform call; out(i, id, dist) is invoked by every lane; returns the count.
template <class Out>
__device__ __forceinline__ uint32_t warp_kway_unique(const float* ld, const uint32_t* li,
                                                     uint32_t nlists, uint32_t len,
                                                     uint32_t stride, uint32_t k, int lane,
                                                     Out out) {
    const float kInf = __int_as_float(0x7f800000);
    uint32_t pos = 0;
    const bool mine = (uint32_t)lane < nlists;
    // head (pos) and the entry after it, loaded one step ahead so that advancing a
    // list is a register move (the distance of an invalid id is never used: the key
    // below ignores it)
    auto fetch = [&](uint32_t p, float& d, uint32_t& i) {
        const bool ok = mine && p < len;
        i = ok ? li[(size_t)lane * stride + p] : kInvalid;
        d = ok ? ld[(size_t)lane * stride + p] : kInf;
    };
    float hd, nd;
    uint32_t hi, ni;
    fetch(0, hd, hi);
    fetch(1, nd, ni);
    uint32_t cnt = 0;
    while (cnt < k) {
        // closer()-minimum of the heads by two REDUX.MIN: the distance (as an
        // order-preserving key; -0 == +0), then the smallest id holding it
        uint32_t kd = 0xFFFFFFFFu;
        if (hi != kInvalid) {
            uint32_t b = __float_as_uint(hd);
            if ((b << 1) == 0) b = 0;
            kd = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
        }
        const uint32_t mk = __reduce_min_sync(kFull, kd);
        if (mk == 0xFFFFFFFFu) break;  // every list exhausted
        const uint32_t bi = __reduce_min_sync(kFull, kd == mk ? hi : 0xFFFFFFFFu);
        const float bd = __shfl_sync(kFull, hd, __ffs(__ballot_sync(kFull, kd == mk && hi == bi)) - 1);
        out(cnt, bi, bd);
        ++cnt;
        if (hi == bi) {
            ++pos;
            hd = nd;
            hi = ni;
            fetch(pos + 1, nd, ni);
        }
    }
    return cnt;
}

__global__ void __launch_bounds__(kMergeThreads) greedy_merge_kernel(
    const uint32_t* walk_ids, const float* walk_dists, const uint32_t* walk_hops,
    const uint32_t* walk_evals, uint32_t t0, uint32_t k, uint32_t npow2, uint32_t* out_ids,
    float* out_dists, uint32_t* out_counts, tsdg_query_stats* out_stats) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* sd = reinterpret_cast<float*>(smem_raw);
    uint32_t* si = reinterpret_cast<uint32_t*>(sd + npow2);
    uint32_t* scan = si + npow2;  // kMergeThreads + 1
    const uint32_t q = blockIdx.x;
    const uint32_t total = t0 * 32;
    const float kInf = __int_as_float(0x7f800000);
    for (uint32_t i = threadIdx.x; i < npow2; i += blockDim.x) {
        float d = kInf;
        uint32_t id = kInvalid;
        if (i < total) {
            id = walk_ids[(size_t)q * total + i];
            d = id != kInvalid ? walk_dists[(size_t)q * total + i] : kInf;
        }
        sd[i] = d;
        si[i] = id;
    }
    __syncthreads();
    for (uint32_t kk = 2; kk <= npow2; kk <<= 1) {
        for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < npow2; i += blockDim.x) {
                const uint32_t p = i ^ j;
                if (p > i) {
                    const bool up = (i & kk) == 0;
                    const bool p_first = closer(sd[p], si[p], sd[i], si[i]);
                    if (p_first == up) {
                        const float td = sd[i];
                        const uint32_t ti = si[i];
                        sd[i] = sd[p];
                        si[i] = si[p];
                        sd[p] = td;
                        si[p] = ti;
                    }
                }
            }
            __syncthreads();
        }
    }
    // unique by id over adjacent entries (std::unique), then first k
    const uint32_t per = (npow2 + blockDim.x - 1) / blockDim.x;
    const uint32_t b0 = threadIdx.x * per;
    uint32_t cnt = 0;
    for (uint32_t i = b0; i < b0 + per && i < npow2; ++i)
        cnt += (si[i] != kInvalid && (i == 0 || si[i] != si[i - 1])) ? 1u : 0u;
    scan[threadIdx.x] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (uint32_t t = 0; t < blockDim.x; ++t) {
            const uint32_t c = scan[t];
            scan[t] = run;
            run += c;
        }
        scan[blockDim.x] = run;
    }
    __syncthreads();
    uint32_t pos = scan[threadIdx.x];
    for (uint32_t i = b0; i < b0 + per && i < npow2; ++i) {
        if (si[i] != kInvalid && (i == 0 || si[i] != si[i - 1])) {
            if (pos < k) {
                out_ids[(size_t)q * k + pos] = si[i];
                if (out_dists) out_dists[(size_t)q * k + pos] = sd[i];
            }
            ++pos;
        }
    }
    const uint32_t uniq = scan[blockDim.x];
    const uint32_t c = uniq < k ? uniq : k;
    for (uint32_t i = c + threadIdx.x; i < k; i += blockDim.x) {
        out_ids[(size_t)q * k + i] = kInvalid;
        if (out_dists) out_dists[(size_t)q * k + i] = kInf;
    }
    if (threadIdx.x == 0) {
        if (out_counts) out_counts[q] = c;
        if (out_stats) {
            uint32_t h = 0, e = 0;
            for (uint32_t s = 0; s < t0; ++s) {
                h += walk_hops[(size_t)q * t0 + s];
                e += walk_evals[(size_t)q * t0 + s];
            }
            tsdg_query_stats st;
            st.hops = h;
            st.distance_evals = e;
            st.queue_evictions = 0;
            st.edges_examined = e - 32u * t0;
            out_stats[q] = st;
        }
    }
}

// deg_cut: partition_point(lambda < cut) over each node's edges (diversify.cpp:34-42).
__global__ void deg_cut_kernel(const uint16_t* lam, uint32_t R, const uint32_t* deg_full,
                               uint32_t n, uint32_t cut, uint32_t* out) {
    const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    const uint16_t* row = lam + (size_t)u * R;
    uint32_t lo = 0, hi = deg_full[u];
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if ((uint32_t)row[mid] < cut) lo = mid + 1;
        else hi = mid;
    }
    out[u] = lo;
}

// Sharded-base merge: per query, union of S shard lists (local ids + base),
// ascending by (dist, global id), first k.  One CTA per query, smem bitonic.
__global__ void __launch_bounds__(kMergeThreads) merge_shards_kernel(
    const uint32_t* ids, const float* dists, const uint32_t* counts, const uint64_t* shard_base,
    uint32_t S, uint32_t nq, uint32_t k, uint32_t npow2, uint32_t* out_ids, float* out_dists,
    uint32_t* out_counts) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* sd = reinterpret_cast<float*>(smem_raw);
    uint32_t* si = reinterpret_cast<uint32_t*>(sd + npow2);
    const uint32_t q = blockIdx.x;
    const float kInf = __int_as_float(0x7f800000);
    uint32_t valid_total = 0;
    for (uint32_t s = 0; s < S; ++s) valid_total += min(counts[(size_t)s * nq + q], k);
    for (uint32_t i = threadIdx.x; i < npow2; i += blockDim.x) {
        float d = kInf;
        uint32_t id = kInvalid;
        if (i < S * k) {
            const uint32_t s = i / k, j = i % k;
            if (j < counts[(size_t)s * nq + q]) {
                const size_t off = ((size_t)s * nq + q) * k + j;
                id = (uint32_t)(shard_base[s] + ids[off]);
                d = dists[off];
            }
        }
        sd[i] = d;
        si[i] = id;
    }
    __syncthreads();
    for (uint32_t kk = 2; kk <= npow2; kk <<= 1) {
        for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < npow2; i += blockDim.x) {
                const uint32_t p = i ^ j;
                if (p > i) {
                    const bool up = (i & kk) == 0;
                    const bool p_first = closer(sd[p], si[p], sd[i], si[i]);
                    if (p_first == up) {
                        const float td = sd[i];
                        const uint32_t ti = si[i];
                        sd[i] = sd[p];
                        si[i] = si[p];
                        sd[p] = td;
                        si[p] = ti;
                    }
                }
            }
            __syncthreads();
        }
    }
    const uint32_t c = valid_total < k ? valid_total : k;
    for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
        out_ids[(size_t)q * k + i] = i < c ? si[i] : kInvalid;
        out_dists[(size_t)q * k + i] = i < c ? sd[i] : kInf;
    }
    if (threadIdx.x == 0 && out_counts) out_counts[q] = c;
}

}  // namespace tsdg_dev
