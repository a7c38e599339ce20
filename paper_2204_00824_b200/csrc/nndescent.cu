// GPU nn_descent: tsdg::nn_descent (knn_graph.cpp:141-251)
// on one B200, returning the reference's KnnGraph bit for bit (ids and fp32
// distances) for the same (set, k, metric, iterations, sample_rate, seed).
//
// Why an exact GPU form exists.  The reference's pools are k-min sets under
// closer() with distinct ids, and a pair's distance does not depend on which side
// offers it (the kernels are symmetric bit for bit).  A pool's final content is
// therefore the k smallest of (start pool u every offer), whatever the order of the
// offers, and an entry's "new" flag is order-independent too: an entry of the start
// pool that is still there at the end was never evicted (once k closer entries are in,
// the k-th only shrinks), so it keeps its flag; every other survivor was inserted
// during the iteration and is new (knn_graph.cpp:198-200 relies on the same fact).
// The GPU runs the local joins of a whole chunk of nodes at once, appends every offer
// that beats its target's worst entry at the chunk start to a buffer, sorts that
// buffer by (target, dist, id) and merges each target's run into its pool.
//
// Per iteration (knn_graph.cpp:176-244):
//   nd_sample_kernel   warp per node: flagged / unflagged pool entries in pool
//                      order, seeded partial Fisher-Yates samples (sample_ids,
//                      :120-130) with the reference's fork(1|2).fork(it).fork(u)
//                      streams, the sampled new flags cleared.
//   reverse lists      (v, u) pairs in u-major order, stable radix sort by v: each
//                      reverse list in ascending u, as the serial scatter (:190-193).
//   nd_join_kernel     CTA per node u: join_new / join_old (forward lists plus the
//                      fork(3|4) samples of the reverse lists, sorted, unique), every
//                      new-new (x < y) and new-old pair's exact distance by the
//                      diversification tile (div_tile: sequential fp32, one rounding
//                      per op), offers to both endpoints filtered by the targets'
//                      worst keys, appended through a shared-memory stage.
//   sort + merge       CUB radix sort of the offers by key then (stable) by target;
//                      nd_merge_kernel (warp per target) merges the sorted, de-
//                      duplicated run into the pool: k smallest distinct (dist, id).
// Initial lists (:157-167): warp per node, the fork(0).fork(u) draws accepted in draw
// order (self and repeats skipped), distances exact, sorted by closer().
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "diversify.cuh"
#include "nndescent.h"

namespace tsdg_dev {

constexpr uint32_t kNdWarps = 8;          // warps per CTA (init / sample / merge)
constexpr uint32_t kNdStage = 1024;       // join kernel's shared-memory offer stage
constexpr uint32_t kNdNegZero = 0x80000000u;  // offer flag: the distance is -0.0f

struct NdArgs {
    const float* vec;  // n x ld (padded rows)
    uint32_t n, d, ld, k, ms;
    int metric;
    uint64_t seed;
    uint32_t it;
    // pools: n x k ascending by (dist, id), flag 1 = new
    uint32_t* pool_id;
    float* pool_d;
    uint8_t* pool_new;
    unsigned long long* worst;  // n: key of each pool's last entry
    // forward samples
    uint32_t* fwd_new;  // n x ms
    uint32_t* fwd_old;
    uint32_t* cnt_new;  // n
    uint32_t* cnt_old;
    // reverse lists (CSR over rev_*_off, u ascending)
    const uint32_t* rev_new;
    const uint32_t* rev_old;
    const uint32_t* rev_new_off;  // n + 1
    const uint32_t* rev_old_off;
    // offers: target (bit 31: -0.0f) + key
    uint32_t* off_t;
    unsigned long long* off_key;
    unsigned long long* off_count;
    unsigned long long off_cap;
    uint32_t u0, u1;
    // merge input (sorted by target, key)
    const uint32_t* srt_t;
    const unsigned long long* srt_key;
    const uint32_t* seg_lo;  // n
    const uint32_t* seg_hi;
    unsigned long long keep;  // all ones (opaque())
};

// (dist, id) as one ascending 64-bit key: closer() order.  -0.0f and +0.0f compare
// equal under closer(), so both map to the key of +0.0f (the sign travels apart).
__device__ __forceinline__ unsigned long long nd_key(float d, uint32_t id) {
    uint32_t b = __float_as_uint(d);
    if ((b << 1) == 0) b = 0;
    b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    return ((unsigned long long)b << 32) | id;
}
__device__ __forceinline__ float nd_key_dist(unsigned long long key, bool neg_zero) {
    uint32_t b = (uint32_t)(key >> 32);
    b = (b & 0x80000000u) ? (b & 0x7FFFFFFFu) : ~b;
    if (neg_zero && b == 0) b = 0x80000000u;
    return __uint_as_float(b);
}

// Ascending bitonic sort of P (power of 2) 64-bit keys with a 32-bit payload, one warp.
__device__ __forceinline__ void nd_warp_sort(unsigned long long* key, uint32_t* val, uint32_t P,
                                             uint32_t lane) {
    for (uint32_t size = 2; size <= P; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = lane; i < (P >> 1); i += 32) {
                const uint32_t a = 2 * i - (i & (stride - 1));
                const uint32_t b = a + stride;
                const bool asc = (a & size) == 0;
                const unsigned long long ka = key[a], kb = key[b];
                if (asc ? (kb < ka) : (ka < kb)) {
                    key[a] = kb;
                    key[b] = ka;
                    const uint32_t t = val[a];
                    val[a] = val[b];
                    val[b] = t;
                }
            }
            __syncwarp();
        }
    }
}

template <int METRIC>
__device__ float nd_distance(const NdArgs& a, uint32_t u, uint32_t v) {
    const float* p = a.vec + (size_t)u * a.ld;
    const float* q = a.vec + (size_t)v * a.ld;
    float acc = 0.0f;
    uint32_t i = 0;
    for (; i + 4 <= a.d; i += 4)
        acc = acc4_exact<METRIC>(acc, __ldg(reinterpret_cast<const float4*>(p + i)),
                                 __ldg(reinterpret_cast<const float4*>(q + i)));
    for (; i < a.d; ++i) acc = acc_exact<METRIC>(acc, __ldg(p + i), __ldg(q + i));
    return finish_exact<METRIC>(acc);
}

// ---- initial random lists (knn_graph.cpp:157-167) -----------------------------------
template <int METRIC>
__global__ void __launch_bounds__(kNdWarps * 32) nd_init_kernel(const NdArgs a) {
    __shared__ unsigned long long skey[kNdWarps][kNdMaxK];
    __shared__ uint32_t sval[kNdWarps][kNdMaxK];
    __shared__ uint32_t sid[kNdWarps][kNdMaxK];
    const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    const uint32_t u = blockIdx.x * kNdWarps + w;
    if (u >= a.n) return;
    const uint64_t st = fork_state(fork_state(a.seed, 0), u);
    uint32_t placed = 0, draw = 0;
    while (placed < a.k) {
        const uint32_t v = draw_below(st, draw + lane, a.n);
        bool ok = v != u;
        for (uint32_t j = 0; j < placed; ++j) ok &= sid[w][j] != v;
        const unsigned same = __match_any_sync(kFull, v);
        if (same & ((1u << lane) - 1u)) ok = false;  // an earlier draw of this round
        const unsigned acc = __ballot_sync(kFull, ok);
        const uint32_t rank = __popc(acc & ((1u << lane) - 1u));
        const uint32_t room = a.k - placed;
        if (ok && rank < room) sid[w][placed + rank] = v;
        placed += min((uint32_t)__popc(acc), room);
        draw += 32;
        __syncwarp();
    }
    uint32_t P = 32;
    while (P < a.k) P <<= 1;
    for (uint32_t j = lane; j < P; j += 32) {
        if (j < a.k) {
            const uint32_t v = sid[w][j];
            const float dd = nd_distance<METRIC>(a, u, v);
            skey[w][j] = nd_key(dd, v);
            sval[w][j] = __float_as_uint(dd);
        } else {
            skey[w][j] = ~0ull;
            sval[w][j] = 0;
        }
    }
    __syncwarp();
    nd_warp_sort(skey[w], sval[w], P, lane);
    for (uint32_t j = lane; j < a.k; j += 32) {
        const size_t o = (size_t)u * a.k + j;
        a.pool_id[o] = (uint32_t)skey[w][j];
        a.pool_d[o] = __uint_as_float(sval[w][j]);
        a.pool_new[o] = 1;
    }
    if (lane == 0) a.worst[u] = skey[w][a.k - 1];
}

// ---- sampling pass (knn_graph.cpp:176-189) ------------------------------------------
// sample_ids (:120-130) on a shared-memory list: partial Fisher-Yates, draw i of the
// stream with state s picks j = i + below(len - i).
__device__ __forceinline__ uint32_t nd_sample_list(uint32_t* list, uint32_t len, uint32_t want,
                                                   uint64_t s, uint32_t lane) {
    if (len <= want) return len;
    if (lane == 0) {
        for (uint32_t i = 0; i < want; ++i) {
            const uint32_t j = i + draw_below(s, i, len - i);
            const uint32_t t = list[i];
            list[i] = list[j];
            list[j] = t;
        }
    }
    __syncwarp();
    return want;
}

__global__ void __launch_bounds__(kNdWarps * 32) nd_sample_kernel(const NdArgs a) {
    __shared__ uint32_t fl[kNdWarps][kNdMaxK];
    __shared__ uint32_t uf[kNdWarps][kNdMaxK];
    const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    const uint32_t u = blockIdx.x * kNdWarps + w;
    if (u >= a.n) return;
    const size_t o = (size_t)u * a.k;
    uint32_t nf = 0, nu = 0;
    for (uint32_t b = 0; b < a.k; b += 32) {
        const uint32_t j = b + lane;
        const bool in = j < a.k;
        const uint32_t id = in ? a.pool_id[o + j] : 0u;
        const bool f = in && a.pool_new[o + j];
        const unsigned mf = __ballot_sync(kFull, f), mu = __ballot_sync(kFull, in && !f);
        const unsigned below = (1u << lane) - 1u;
        if (f) fl[w][nf + __popc(mf & below)] = id;
        if (in && !f) uf[w][nu + __popc(mu & below)] = id;
        nf += __popc(mf);
        nu += __popc(mu);
    }
    __syncwarp();
    const uint64_t s_new = fork_state(fork_state(fork_state(a.seed, 1), a.it), u);
    const uint64_t s_old = fork_state(fork_state(fork_state(a.seed, 2), a.it), u);
    const uint32_t cn = nd_sample_list(fl[w], nf, a.ms, s_new, lane);
    const uint32_t co = nd_sample_list(uf[w], nu, a.ms, s_old, lane);
    for (uint32_t j = lane; j < cn; j += 32) a.fwd_new[(size_t)u * a.ms + j] = fl[w][j];
    for (uint32_t j = lane; j < co; j += 32) a.fwd_old[(size_t)u * a.ms + j] = uf[w][j];
    if (lane == 0) {
        a.cnt_new[u] = cn;
        a.cnt_old[u] = co;
    }
    // the sampled new entries become old (:182-188)
    for (uint32_t j = lane; j < a.k; j += 32) {
        if (!a.pool_new[o + j]) continue;
        const uint32_t id = a.pool_id[o + j];
        bool hit = false;
        for (uint32_t t = 0; t < cn; ++t) hit |= fl[w][t] == id;
        if (hit) a.pool_new[o + j] = 0;
    }
}

// (v, u) pairs of the forward samples in u-major order; padding sorts last.
__global__ void nd_rev_pairs_kernel(const uint32_t* fwd, const uint32_t* cnt, uint32_t n,
                                    uint32_t ms, uint32_t* keys, uint32_t* vals) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)n * ms) return;
    const uint32_t u = (uint32_t)(i / ms), j = (uint32_t)(i % ms);
    keys[i] = j < cnt[u] ? fwd[i] : 0xFFFFFFFFu;
    vals[i] = u;
}
// off[v] = first position of key >= v in the sorted keys (v = 0..n).
__global__ void nd_rev_offsets_kernel(const uint32_t* keys, size_t total, uint32_t n,
                                      uint32_t* off) {
    const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v > n) return;
    size_t lo = 0, hi = total;
    while (lo < hi) {
        const size_t mid = (lo + hi) >> 1;
        if (keys[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    off[v] = (uint32_t)lo;
}

// ---- local join (knn_graph.cpp:203-243) ---------------------------------------------
struct NdJoinSmem {
    DivStage st;
    uint32_t jn[2 * kNdMaxK];      // join_new (sorted, unique)
    uint32_t jall[4 * kNdMaxK];    // join_new then join_old
    uint32_t tmp[2 * kNdMaxK];     // list being built
    unsigned long long wi[kDivT], wj[kDivT];  // worst keys of the tile's rows / columns
    uint32_t stage_t[kNdStage];
    unsigned long long stage_k[kNdStage];
    uint32_t fy_a[kNdMaxK], fy_pos[kNdMaxK], fy_val[kNdMaxK];
    uint32_t nstage, nlist, nn, no;
    unsigned long long gbase;
};

// sample_ids of a reverse list in global memory (not modified: a chunk may be re-run),
// written to out[0..want): the partial Fisher-Yates over a sparse overlay.  Thread 0.
__device__ uint32_t nd_sample_global(const uint32_t* list, uint32_t len, uint32_t want, uint64_t s,
                                     uint32_t* out, NdJoinSmem& m) {
    if (len <= want) {
        for (uint32_t i = 0; i < len; ++i) out[i] = list[i];
        return len;
    }
    for (uint32_t i = 0; i < want; ++i) m.fy_a[i] = list[i];
    uint32_t ne = 0;  // overlay of positions >= want
    auto get = [&](uint32_t p) -> uint32_t {
        if (p < want) return m.fy_a[p];
        for (uint32_t e = 0; e < ne; ++e)
            if (m.fy_pos[e] == p) return m.fy_val[e];
        return list[p];
    };
    auto set = [&](uint32_t p, uint32_t v) {
        if (p < want) {
            m.fy_a[p] = v;
            return;
        }
        for (uint32_t e = 0; e < ne; ++e)
            if (m.fy_pos[e] == p) {
                m.fy_val[e] = v;
                return;
            }
        m.fy_pos[ne] = p;
        m.fy_val[ne] = v;
        ++ne;
    };
    for (uint32_t i = 0; i < want; ++i) {
        const uint32_t j = i + draw_below(s, i, len - i);
        const uint32_t vi = get(i), vj = get(j);
        set(i, vj);
        set(j, vi);
    }
    for (uint32_t i = 0; i < want; ++i) out[i] = m.fy_a[i];
    return want;
}

// Builds sort(unique(fwd ++ sample(rev))) into dst; returns its length.  All threads.
__device__ uint32_t nd_join_list(const NdArgs& a, NdJoinSmem& m, uint32_t u, const uint32_t* fwd,
                                 uint32_t cf, const uint32_t* rev, const uint32_t* rev_off,
                                 uint64_t s, uint32_t* dst) {
    const uint32_t tid = threadIdx.x;
    if (tid == 0) {
        for (uint32_t i = 0; i < cf; ++i) m.tmp[i] = fwd[(size_t)u * a.ms + i];
        const uint32_t lo = rev_off[u], hi = rev_off[u + 1];
        m.nlist = cf + nd_sample_global(rev + lo, hi - lo, a.ms, s, m.tmp + cf, m);
    }
    __syncthreads();
    const uint32_t len = m.nlist;
    uint32_t P = 2;
    while (P < len) P <<= 1;
    for (uint32_t i = len + tid; i < P; i += blockDim.x) m.tmp[i] = 0xFFFFFFFFu;
    __syncthreads();
    for (uint32_t size = 2; size <= P; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = tid; i < (P >> 1); i += blockDim.x) {
                const uint32_t x = 2 * i - (i & (stride - 1)), y = x + stride;
                const bool asc = (x & size) == 0;
                const uint32_t vx = m.tmp[x], vy = m.tmp[y];
                if (asc ? (vy < vx) : (vx < vy)) {
                    m.tmp[x] = vy;
                    m.tmp[y] = vx;
                }
            }
            __syncthreads();
        }
    }
    if (tid < 32) {  // unique, compacted by ballots
        uint32_t outn = 0;
        for (uint32_t b = 0; b < len; b += 32) {
            const uint32_t i = b + tid;
            const bool keep = i < len && (i == 0 || m.tmp[i] != m.tmp[i - 1]);
            const unsigned mk = __ballot_sync(kFull, keep);
            if (keep) dst[outn + __popc(mk & ((1u << tid) - 1u))] = m.tmp[i];
            outn += __popc(mk);
        }
        if (tid == 0) m.nlist = outn;
    }
    __syncthreads();
    return m.nlist;
}

template <int METRIC>
__global__ void __launch_bounds__(kDivThreads, 2) nd_join_kernel(const NdArgs a) {
    __shared__ NdJoinSmem m;
    const uint32_t tid = threadIdx.x;
    const uint32_t u = a.u0 + blockIdx.x;
    if (u >= a.u1) return;
    DivArgs da{};
    da.vec = a.vec;
    da.n = a.n;
    da.d = a.d;
    da.ld = a.ld;
    da.metric = a.metric;
    da.keep = a.keep;
    const uint64_t s3 = fork_state(fork_state(fork_state(a.seed, 3), a.it), u);
    const uint64_t s4 = fork_state(fork_state(fork_state(a.seed, 4), a.it), u);
    const uint32_t nn = nd_join_list(a, m, u, a.fwd_new, a.cnt_new[u], a.rev_new, a.rev_new_off, s3, m.jn);
    for (uint32_t i = tid; i < nn; i += blockDim.x) m.jall[i] = m.jn[i];
    __syncthreads();
    const uint32_t no = nd_join_list(a, m, u, a.fwd_old, a.cnt_old[u], a.rev_old, a.rev_old_off, s4,
                                     m.jall + nn);
    if (tid == 0) m.nstage = 0;
    __syncthreads();
    const uint32_t nall = nn + no;
    auto push = [&](uint32_t t, unsigned long long key) {
        const uint32_t p = atomicAdd(&m.nstage, 1u);
        if (p < kNdStage) {
            m.stage_t[p] = t;
            m.stage_k[p] = key;
        } else {  // stage full: straight to the global buffer
            const unsigned long long g = atomicAdd(a.off_count, 1ull);
            if (g < a.off_cap) {
                a.off_t[g] = t;
                a.off_key[g] = key;
            }
        }
    };
    for (uint32_t i0 = 0; i0 < nn; i0 += kDivT) {
        const uint32_t ni = min(kDivT, nn - i0);
        for (uint32_t j0 = 0; j0 < nall; j0 += kDivT) {
            const uint32_t nj = min(kDivT, nall - j0);
            if (j0 + nj <= nn && j0 + nj <= i0 + 1) continue;  // new-new pairs need x < y
            for (uint32_t t = tid; t < kDivT; t += blockDim.x) {
                m.wi[t] = t < ni ? a.worst[m.jn[i0 + t]] : 0ull;
                m.wj[t] = t < nj ? a.worst[m.jall[j0 + t]] : 0ull;
            }
            __syncthreads();
            div_tile<METRIC>(da, m.st, m.jn + i0, ni, m.jall + j0, nj,
                             [&](uint32_t i, uint32_t j, float dist) {
                                 const uint32_t gi = i0 + i, gj = j0 + j;
                                 if (gj < nn && gj <= gi) return;
                                 const uint32_t x = m.jn[gi], y = m.jall[gj];
                                 if (x == y) return;
                                 const uint32_t neg = __float_as_uint(dist) == 0x80000000u ? kNdNegZero : 0u;
                                 const unsigned long long kxy = nd_key(dist, y), kyx = nd_key(dist, x);
                                 if (kxy < m.wi[i]) push(x | neg, kxy);
                                 if (kyx < m.wj[j]) push(y | neg, kyx);
                             });
        }
    }
    __syncthreads();
    const uint32_t ns = min(m.nstage, kNdStage);
    if (tid == 0) m.gbase = ns ? atomicAdd(a.off_count, (unsigned long long)ns) : 0ull;
    __syncthreads();
    for (uint32_t i = tid; i < ns; i += blockDim.x) {
        const unsigned long long g = m.gbase + i;
        if (g < a.off_cap) {
            a.off_t[g] = m.stage_t[i];
            a.off_key[g] = m.stage_k[i];
        }
    }
}

// Run bounds of each target in the sorted offers.
__global__ void nd_segments_kernel(const uint32_t* srt_t, uint32_t m, uint32_t* lo, uint32_t* hi) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint32_t t = srt_t[i] & ~kNdNegZero;
    if (i == 0 || (srt_t[i - 1] & ~kNdNegZero) != t) lo[t] = i;
    if (i == m - 1 || (srt_t[i + 1] & ~kNdNegZero) != t) hi[t] = i + 1;
}

// ---- merge of each target's offers into its pool ------------------------------------
__global__ void __launch_bounds__(kNdWarps * 32) nd_merge_kernel(const NdArgs a) {
    __shared__ unsigned long long pk[kNdWarps][kNdMaxK], nk[kNdWarps][kNdMaxK];
    __shared__ uint32_t pd[kNdWarps][kNdMaxK], ndd[kNdWarps][kNdMaxK];
    __shared__ uint8_t pf[kNdWarps][kNdMaxK], nf[kNdWarps][kNdMaxK];
    __shared__ unsigned long long ck[kNdWarps][32];
    const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    const uint32_t t = blockIdx.x * kNdWarps + w;
    if (t >= a.n) return;
    const uint32_t lo = a.seg_lo[t], hi = a.seg_hi[t];
    if (lo >= hi) return;
    const uint32_t k = a.k;
    const size_t o = (size_t)t * k;
    for (uint32_t j = lane; j < k; j += 32) {
        const float dj = a.pool_d[o + j];
        pk[w][j] = nd_key(dj, a.pool_id[o + j]);
        pd[w][j] = __float_as_uint(dj);
        pf[w][j] = a.pool_new[o + j];
    }
    __syncwarp();
    unsigned long long worst = pk[w][k - 1], prev = ~0ull;
    bool changed = false;
    for (uint32_t b = lo; b < hi; b += 32) {
        const uint32_t i = b + lane;
        const bool in = i < hi;
        const unsigned long long c = in ? a.srt_key[i] : ~0ull;
        const uint32_t ct = in ? a.srt_t[i] : 0u;
        if (__shfl_sync(kFull, c, 0) >= worst) break;  // sorted: nothing later enters
        const unsigned long long before = __shfl_up_sync(kFull, c, 1);
        const bool dup = lane ? (c == before) : (c == prev);
        prev = __shfl_sync(kFull, c, 31);
        // position among the pool (no equal key when absent from the pool)
        uint32_t l = 0, h = k;
        while (l < h) {
            const uint32_t mid = (l + h) >> 1;
            if (pk[w][mid] < c) l = mid + 1;
            else h = mid;
        }
        const bool ok = in && c < worst && !dup && !(l < k && pk[w][l] == c);
        const unsigned mk = __ballot_sync(kFull, ok);
        if (!mk) continue;
        changed = true;
        const uint32_t crank = __popc(mk & ((1u << lane) - 1u));
        if (ok) ck[w][crank] = c;
        __syncwarp();
        const uint32_t nc = __popc(mk);
        // pool entry j moves to j + #(accepted candidates closer than it)
        for (uint32_t j = lane; j < k; j += 32) {
            uint32_t cl = 0, chh = nc;
            while (cl < chh) {
                const uint32_t mid = (cl + chh) >> 1;
                if (ck[w][mid] < pk[w][j]) cl = mid + 1;
                else chh = mid;
            }
            const uint32_t r = j + cl;
            if (r < k) {
                nk[w][r] = pk[w][j];
                ndd[w][r] = pd[w][j];
                nf[w][r] = pf[w][j];
            }
        }
        if (ok) {
            const uint32_t r = crank + l;
            if (r < k) {
                nk[w][r] = c;
                ndd[w][r] = __float_as_uint(nd_key_dist(c, (ct & kNdNegZero) != 0));
                nf[w][r] = 1;
            }
        }
        __syncwarp();
        for (uint32_t j = lane; j < k; j += 32) {
            pk[w][j] = nk[w][j];
            pd[w][j] = ndd[w][j];
            pf[w][j] = nf[w][j];
        }
        __syncwarp();
        worst = pk[w][k - 1];
    }
    if (!changed) return;
    for (uint32_t j = lane; j < k; j += 32) {
        a.pool_id[o + j] = (uint32_t)pk[w][j];
        a.pool_d[o + j] = __uint_as_float(pd[w][j]);
        a.pool_new[o + j] = pf[w][j];
    }
    if (lane == 0) a.worst[t] = worst;
}

// ---- host driver ----------------------------------------------------------------------
namespace {

void nd_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class T>
struct NdBuf {
    T* p = nullptr;
    cudaStream_t st;
    NdBuf(size_t n, cudaStream_t s) : st(s) {
        nd_check(cudaMallocAsync(reinterpret_cast<void**>(&p), std::max<size_t>(n, 1) * sizeof(T), s),
                 "cudaMallocAsync(nn_descent)");
    }
    ~NdBuf() { cudaFreeAsync(p, st); }
    NdBuf(const NdBuf&) = delete;
};

template <int METRIC>
void nd_launch_init(const NdArgs& a, cudaStream_t st) {
    nd_init_kernel<METRIC><<<(a.n + kNdWarps - 1) / kNdWarps, kNdWarps * 32, 0, st>>>(a);
}
template <int METRIC>
void nd_launch_join(const NdArgs& a, cudaStream_t st) {
    nd_join_kernel<METRIC><<<a.u1 - a.u0, kDivThreads, 0, st>>>(a);
}

// Reverse lists of one forward sample: CSR (off, vals) with u ascending per v.
void nd_reverse(const uint32_t* fwd, const uint32_t* cnt, uint32_t n, uint32_t ms, uint32_t* k_in,
                uint32_t* v_in, uint32_t* k_out, uint32_t* v_out, uint32_t* off, void*& tmp,
                size_t& tmp_bytes, cudaStream_t st, uint64_t& launches) {
    const size_t total = (size_t)n * ms;
    nd_rev_pairs_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(fwd, cnt, n, ms, k_in, v_in);
    size_t need = 0;
    nd_check(cub::DeviceRadixSort::SortPairs(nullptr, need, k_in, k_out, v_in, v_out, total, 0, 32, st),
             "cub sort (reverse lists)");
    if (need > tmp_bytes) {
        cudaFreeAsync(tmp, st);
        nd_check(cudaMallocAsync(&tmp, need, st), "cudaMallocAsync(cub)");
        tmp_bytes = need;
    }
    nd_check(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k_in, k_out, v_in, v_out, total, 0, 32, st),
             "cub sort (reverse lists)");
    nd_rev_offsets_kernel<<<(n + 1 + 255) / 256, 256, 0, st>>>(k_out, total, n, off);
    launches += 4;
}

}  // namespace

void nn_descent_device(const float* d_vec, uint32_t n, uint32_t d, uint32_t ld, uint32_t k,
                       int metric, uint32_t iterations, uint32_t max_sample, uint64_t seed,
                       uint32_t* d_ids, float* d_dists, cudaStream_t st, NnDescentStats* stats) {
    NdArgs a{};
    a.vec = d_vec;
    a.n = n;
    a.d = d;
    a.ld = ld;
    a.k = k;
    a.ms = max_sample;
    a.metric = metric;
    a.seed = seed;
    a.keep = ~0ull;
    const size_t nk = (size_t)n * k, nms = (size_t)n * max_sample;
    NdBuf<uint8_t> pool_new(nk, st);
    NdBuf<unsigned long long> worst(n, st);
    a.pool_id = d_ids;
    a.pool_d = d_dists;
    a.pool_new = pool_new.p;
    a.worst = worst.p;
    uint64_t launches = 0;
    if (metric == 0) nd_launch_init<0>(a, st);
    else if (metric == 1) nd_launch_init<1>(a, st);
    else nd_launch_init<2>(a, st);
    ++launches;
    nd_check(cudaGetLastError(), "nd_init_kernel launch");
    NdBuf<uint32_t> fwd_new(nms, st), fwd_old(nms, st), cnt_new(n, st), cnt_old(n, st);
    NdBuf<uint32_t> rk_in(nms, st), rv_in(nms, st), rk_out(nms, st), rnew(nms, st), rold(nms, st);
    NdBuf<uint32_t> off_new((size_t)n + 1, st), off_old((size_t)n + 1, st);
    NdBuf<uint32_t> seg_lo(n, st), seg_hi(n, st);
    a.fwd_new = fwd_new.p;
    a.fwd_old = fwd_old.p;
    a.cnt_new = cnt_new.p;
    a.cnt_old = cnt_old.p;
    a.rev_new = rnew.p;
    a.rev_old = rold.p;
    a.rev_new_off = off_new.p;
    a.rev_old_off = off_old.p;
    a.seg_lo = seg_lo.p;
    a.seg_hi = seg_hi.p;
    // offer buffer: ~24 B per entry with the sorted copies; sized from free memory
    size_t free_b = 0, total_b = 0;
    nd_check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
    unsigned long long cap = std::min<unsigned long long>(
        std::max<unsigned long long>(1ull << 20, (unsigned long long)(free_b / 4 / 24)), 0x7FFFFFFFull);
    cap = std::min<unsigned long long>(cap, std::max<unsigned long long>(1ull << 20, (unsigned long long)n * 256));
    NdBuf<uint32_t> off_t(cap, st), srt_t(cap, st);
    NdBuf<unsigned long long> off_key(cap, st), srt_key(cap, st), off_count(1, st);
    a.off_t = off_t.p;
    a.off_key = off_key.p;
    a.off_count = off_count.p;
    a.off_cap = cap;
    a.srt_t = srt_t.p;
    a.srt_key = srt_key.p;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    uint32_t chunk = n;
    uint64_t offers = 0, chunks = 0, reruns = 0;
    unsigned long long* h_count = nullptr;
    nd_check(cudaMallocHost(&h_count, sizeof(unsigned long long)), "cudaMallocHost");
    try {
        for (uint32_t it = 0; it < iterations; ++it) {
            a.it = it;
            nd_sample_kernel<<<(n + kNdWarps - 1) / kNdWarps, kNdWarps * 32, 0, st>>>(a);
            ++launches;
            nd_check(cudaGetLastError(), "nd_sample_kernel launch");
            nd_reverse(fwd_new.p, cnt_new.p, n, max_sample, rk_in.p, rv_in.p, rk_out.p, rnew.p,
                       off_new.p, tmp, tmp_bytes, st, launches);
            nd_reverse(fwd_old.p, cnt_old.p, n, max_sample, rk_in.p, rv_in.p, rk_out.p, rold.p,
                       off_old.p, tmp, tmp_bytes, st, launches);
            uint32_t u0 = 0;
            while (u0 < n) {
                const uint32_t u1 = (uint32_t)std::min<uint64_t>(n, (uint64_t)u0 + chunk);
                a.u0 = u0;
                a.u1 = u1;
                nd_check(cudaMemsetAsync(off_count.p, 0, 8, st), "memset");
                if (metric == 0) nd_launch_join<0>(a, st);
                else if (metric == 1) nd_launch_join<1>(a, st);
                else nd_launch_join<2>(a, st);
                ++launches;
                nd_check(cudaGetLastError(), "nd_join_kernel launch");
                nd_check(cudaMemcpyAsync(h_count, off_count.p, 8, cudaMemcpyDeviceToHost, st), "D2H");
                nd_check(cudaStreamSynchronize(st), "nd_join_kernel");
                const unsigned long long m = *h_count;
                if (m > cap) {  // buffer too small for this chunk: nothing merged yet, redo smaller
                    const uint64_t want = std::max<uint64_t>(1, (uint64_t)(u1 - u0) * cap / m / 2);
                    chunk = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(want, chunk / 2));
                    ++reruns;
                    continue;
                }
                offers += m;
                ++chunks;
                if (m) {
                    size_t need = 0;
                    nd_check(cub::DeviceRadixSort::SortPairs(nullptr, need, off_key.p, srt_key.p, off_t.p,
                                                             srt_t.p, m, 0, 64, st),
                             "cub sort (offers)");
                    size_t need2 = 0;
                    nd_check(cub::DeviceRadixSort::SortPairs(nullptr, need2, srt_t.p, off_t.p, srt_key.p,
                                                             off_key.p, m, 0, 31, st),
                             "cub sort (offers)");
                    need = std::max(need, need2);
                    if (need > tmp_bytes) {
                        cudaFreeAsync(tmp, st);
                        nd_check(cudaMallocAsync(&tmp, need, st), "cudaMallocAsync(cub)");
                        tmp_bytes = need;
                    }
                    // by key, then stable by target (bit 31 = sign of a zero distance, ignored)
                    nd_check(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, off_key.p, srt_key.p, off_t.p,
                                                             srt_t.p, m, 0, 64, st),
                             "cub sort (offers)");
                    nd_check(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, srt_t.p, off_t.p, srt_key.p,
                                                             off_key.p, m, 0, 31, st),
                             "cub sort (offers)");
                    // sorted result now in (off_t, off_key)
                    NdArgs b = a;
                    b.srt_t = off_t.p;
                    b.srt_key = off_key.p;
                    nd_check(cudaMemsetAsync(seg_lo.p, 0, (size_t)n * 4, st), "memset");
                    nd_check(cudaMemsetAsync(seg_hi.p, 0, (size_t)n * 4, st), "memset");
                    nd_segments_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(off_t.p, (uint32_t)m,
                                                                                  seg_lo.p, seg_hi.p);
                    nd_merge_kernel<<<(n + kNdWarps - 1) / kNdWarps, kNdWarps * 32, 0, st>>>(b);
                    launches += 4;
                    nd_check(cudaGetLastError(), "nd_merge_kernel launch");
                }
                u0 = u1;
            }
        }
        nd_check(cudaStreamSynchronize(st), "nn_descent");
    } catch (...) {
        cudaStreamSynchronize(st);
        cudaFreeAsync(tmp, st);
        cudaFreeHost(h_count);
        throw;
    }
    cudaFreeAsync(tmp, st);
    cudaFreeHost(h_count);
    if (stats) {
        stats->offers = offers;
        stats->chunks = chunks;
        stats->reruns = reruns;
        stats->launches = launches;
    }
}

}  // namespace tsdg_dev
