// GPU two-stage diversification: tsdg::build
// (diversify.cpp:152-209) from a k-NN graph, producing the reference's TsdgGraph
// exactly — same edges, same lambda, same fp32 distances, same (lambda, dist, target)
// order — given the same KnnGraph.
//
//   stage 1 (stage1_relaxed_gd, diversify.cpp:44-69)   one CTA per node: all pairwise
//       distances of the k candidates (exact sequential fp32, tiled like the exact
//       scan), folded at once into an "i relax-occludes j" bit matrix; the greedy pass
//       over candidates in order is then a walk over 128-bit masks.
//   reverse edges (add_reverse_edges, :71-124)        count, prefix, fill, then per
//       node dedup by target keeping the smallest distance.
//   stage 2 (stage2_soft_gd, :126-150)                 one CTA per node: distances to
//       the owner (the reference's dist_matches re-check), order by (dist, target),
//       pairwise occlusion counts lambda, filter lambda <= lambda0, order by
//       (lambda, dist, target), cap at max_degree.
// Distances are the reference kernel's value bit for bit: each pair accumulates
// in dimension order with one rounding per sub / mul / add (vectors.hpp:36-49);
// the kernels are symmetric in their arguments, as every call site here is.
#pragma once

#include "exact_scan.cuh"  // opaque(), f32x2 helpers

namespace tsdg_dev {

constexpr uint32_t kDivThreads = 256;
constexpr uint32_t kDivT = 128;     // tile rows (both sides)
constexpr uint32_t kDivDC = 16;     // dims per staged chunk
constexpr uint32_t kDivJP = kDivT + 4;
constexpr uint32_t kDivMaxK = 128;  // stage-1 candidates per node (GPU limit)

struct DivArgs {
    const float* vec;  // n x ld
    uint32_t n, d, ld;
    int metric;
    unsigned long long keep;  // all ones; its sign bits give the opaque (-0, -0) addend
    // stage 1
    const uint32_t* knn_ids;  // n x k
    const float* knn_dists;
    uint32_t k;
    float alpha;
    uint32_t* s1_ids;    // n x k (kept prefix)
    float* s1_dists;
    uint32_t* s1_cnt;    // n
    int* err;            // 1: candidates unsorted, 2: target out of range
    // augmented lists (CSR over aug_off)
    const unsigned long long* aug_off;  // n + 1
    uint32_t* aug_ids;
    float* aug_dists;
    uint32_t* aug_cnt;   // after dedup
    uint32_t* tmp_ids;   // scratch, same layout
    float* tmp_dists;
    uint32_t* tmp_cnt;   // stage-2 occlusion counts
    // stage 2 output (same layout, compacted)
    uint32_t lambda0, max_degree;
    uint32_t* out_ids;
    uint16_t* out_lambda;
    float* out_dists;
    uint32_t* out_cnt;
};

// Shared staging of one 128 x 128 tile, dims in chunks of 16: i side duplicated as
// (x, x) pairs (one LDS.128 = two packed operands), j side plain, both dim-major.
struct DivStage {
    unsigned long long is[kDivDC][kDivT];
    float js[kDivDC][kDivJP];
};

// Exact distances of the pairs (ids_i[0..ni) x ids_j[0..nj)), ni, nj <= 128.  Thread
// (ti, tj) of the 16 x 16 grid owns i rows 8ti..8ti+7 and j columns {4tj..4tj+3,
// 64+4tj..64+4tj+3}; consume(i, j, dist) is called by the owner for every pair in
// range.  ids_* may point to global or shared memory; every thread must call.
template <int METRIC, class F>
__device__ __forceinline__ void div_tile(const DivArgs& a, DivStage& st, const uint32_t* ids_i,
                                         uint32_t ni, const uint32_t* ids_j, uint32_t nj,
                                         F&& consume) {
    const uint32_t tid = threadIdx.x, ti = tid >> 4, tj = tid & 15u;
    unsigned long long acc[8][4];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = 0ull;
    float4 ri[2], rj[2];
    auto load = [&](uint32_t c0) {
#pragma unroll
        for (uint32_t t = 0; t < 2; ++t) {
            const uint32_t f = tid + t * kDivThreads;  // 512 float4 per side
            const uint32_t row = f >> 2, dim = c0 + (f & 3u) * 4;
            const bool okd = dim < a.ld;
            ri[t] = (row < ni && okd)
                        ? __ldg(reinterpret_cast<const float4*>(a.vec + (size_t)ids_i[row] * a.ld + dim))
                        : make_float4(0.f, 0.f, 0.f, 0.f);
            rj[t] = (row < nj && okd)
                        ? __ldg(reinterpret_cast<const float4*>(a.vec + (size_t)ids_j[row] * a.ld + dim))
                        : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    load(0);
    for (uint32_t c0 = 0; c0 < a.d; c0 += kDivDC) {
        __syncthreads();
#pragma unroll
        for (uint32_t t = 0; t < 2; ++t) {
            const uint32_t f = tid + t * kDivThreads;
            const uint32_t row = f >> 2, dim = (f & 3u) * 4;
            st.is[dim + 0][row] = f2_dup(ri[t].x);
            st.is[dim + 1][row] = f2_dup(ri[t].y);
            st.is[dim + 2][row] = f2_dup(ri[t].z);
            st.is[dim + 3][row] = f2_dup(ri[t].w);
            st.js[dim + 0][row] = rj[t].x;
            st.js[dim + 1][row] = rj[t].y;
            st.js[dim + 2][row] = rj[t].z;
            st.js[dim + 3][row] = rj[t].w;
        }
        __syncthreads();
        if (c0 + kDivDC < a.d) load(c0 + kDivDC);
        const uint32_t dims = min(kDivDC, a.d - c0);
        // (-0, -0) from the arguments: fma(x, y, nz) is x * y rounded once and stays a
        // separate rounding from the add (exact_scan.cuh scan_step)
        const unsigned long long nz = a.keep & 0x8000000080000000ull;
        for (uint32_t t = 0; t < dims; ++t) {
            const ulonglong2* ip = reinterpret_cast<const ulonglong2*>(&st.is[t][8 * ti]);
            const ulonglong2 i01 = ip[0], i23 = ip[1], i45 = ip[2], i67 = ip[3];
            const ulonglong2 j0 = *reinterpret_cast<const ulonglong2*>(&st.js[t][4 * tj]);
            const ulonglong2 j1 = *reinterpret_cast<const ulonglong2*>(&st.js[t][64 + 4 * tj]);
            const unsigned long long iv[8] = {i01.x, i01.y, i23.x, i23.y, i45.x, i45.y, i67.x, i67.y};
            const unsigned long long jv[4] = {j0.x, j0.y, j1.x, j1.y};
#pragma unroll
            for (int r = 0; r < 8; ++r) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    unsigned long long tt;
                    if (METRIC == 0) {
                        const unsigned long long df = f2_sub(iv[r], jv[c]);
                        tt = f2_fma(df, df, nz);
                    } else {
                        tt = f2_fma(iv[r], jv[c], nz);
                    }
                    acc[r][c] = f2_add(acc[r][c], tt);
                }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const uint32_t i = 8 * ti + r;
        if (i >= ni) continue;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t j = (c >> 1) * 64 + 4 * tj + (c & 1) * 2 + h;
                if (j >= nj) continue;
                const float v = h ? f2_hi(acc[r][c]) : f2_lo(acc[r][c]);
                consume(i, j, finish_exact<METRIC>(v));
            }
        }
    }
    __syncthreads();  // staging reusable by the next tile
}

// (d0i < d0j) && (dij < d0j), diversify.hpp occludes(); relaxed: alpha * both sides.
__device__ __forceinline__ bool occludes_relaxed_dev(float d0i, float d0j, float dij, float alpha) {
    return __fmul_rn(alpha, d0i) < d0j && __fmul_rn(alpha, dij) < d0j;
}

// ---- stage 1: one CTA per node ------------------------------------------------
template <int METRIC>
__global__ void __launch_bounds__(kDivThreads, 2) div_stage1_kernel(const DivArgs a) {
    __shared__ DivStage st;
    __shared__ uint32_t cid[kDivMaxK];
    __shared__ float cdist[kDivMaxK];
    __shared__ uint32_t occ[kDivMaxK][kDivMaxK / 32];  // occ[j] bit i: i relax-occludes j
    __shared__ int bad;
    const uint32_t u = blockIdx.x, tid = threadIdx.x;
    const uint32_t k = a.k;
    if (tid == 0) bad = 0;
    for (uint32_t j = tid; j < k; j += kDivThreads) {
        cid[j] = a.knn_ids[(size_t)u * k + j];
        cdist[j] = a.knn_dists[(size_t)u * k + j];
    }
    for (uint32_t w = tid; w < kDivMaxK * kDivMaxK / 32; w += kDivThreads) (&occ[0][0])[w] = 0;
    __syncthreads();
    for (uint32_t j = tid; j < k; j += kDivThreads) {
        if (cid[j] >= a.n) atomicOr(&bad, 2);
        if (j > 0 && cdist[j] < cdist[j - 1]) atomicOr(&bad, 1);  // diversify.cpp:48-53
    }
    __syncthreads();
    if (bad) {
        if (tid == 0) {
            atomicOr(a.err, bad);
            a.s1_cnt[u] = 0;
        }
        return;
    }
    div_tile<METRIC>(a, st, cid, k, cid, k, [&](uint32_t i, uint32_t j, float dij) {
        if (i < j && occludes_relaxed_dev(cdist[i], cdist[j], dij, a.alpha))
            atomicOr(&occ[j][i >> 5], 1u << (i & 31u));
    });
    __syncthreads();
    if (tid == 0) {  // the greedy filter: j survives iff no kept i < j occludes it
        uint32_t kept[kDivMaxK / 32] = {0, 0, 0, 0};
        uint32_t nk = 0;
        for (uint32_t j = 0; j < k; ++j) {
            const bool o = (occ[j][0] & kept[0]) | (occ[j][1] & kept[1]) | (occ[j][2] & kept[2]) |
                           (occ[j][3] & kept[3]);
            if (!o) {
                kept[j >> 5] |= 1u << (j & 31u);
                a.s1_ids[(size_t)u * k + nk] = cid[j];
                a.s1_dists[(size_t)u * k + nk] = cdist[j];
                ++nk;
            }
        }
        a.s1_cnt[u] = nk;
    }
}

// ---- reverse edges ---------------------------------------------------------------
static __global__ void div_rev_count_kernel(const DivArgs a, uint32_t* rev_cnt) {
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t u = (uint32_t)(t / a.k), j = (uint32_t)(t % a.k);
    if (u >= a.n || j >= a.s1_cnt[u]) return;
    atomicAdd(&rev_cnt[a.s1_ids[(size_t)u * a.k + j]], 1u);
}

// forward entries first (stage-1 order), reverse entries appended (order fixed later
// by the dedup + (dist, target) ranking, so the atomic append order does not matter)
static __global__ void div_fill_kernel(const DivArgs a, uint32_t* cursor) {
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t u = (uint32_t)(t / a.k), j = (uint32_t)(t % a.k);
    if (u >= a.n || j >= a.s1_cnt[u]) return;
    const uint32_t v = a.s1_ids[(size_t)u * a.k + j];
    const float dist = a.s1_dists[(size_t)u * a.k + j];
    const unsigned long long fo = a.aug_off[u] + j;
    a.tmp_ids[fo] = v;
    a.tmp_dists[fo] = dist;
    const unsigned long long ro = a.aug_off[v] + a.s1_cnt[v] + atomicAdd(&cursor[v], 1u);
    a.tmp_ids[ro] = u;
    a.tmp_dists[ro] = dist;
}

// sort by (target, dist) + unique by target (diversify.cpp:101-110): entry j survives
// iff no other entry has its target with a smaller (dist, index).  Warp per node.
static __global__ void div_dedup_kernel(const DivArgs a) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t u = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (u >= a.n) return;
    const unsigned long long o = a.aug_off[u];
    const uint32_t m = (uint32_t)(a.aug_off[u + 1] - o);
    uint32_t out = 0;
    for (uint32_t j0 = 0; j0 < m; j0 += 32) {
        const uint32_t j = j0 + lane;
        const bool vj = j < m;
        const uint32_t tj = vj ? a.tmp_ids[o + j] : kInvalid;
        const float dj = vj ? a.tmp_dists[o + j] : 0.f;
        bool dup = false;
        for (uint32_t i = 0; i < m && vj; ++i) {
            if (i == j) continue;
            if (a.tmp_ids[o + i] != tj) continue;
            const float di = a.tmp_dists[o + i];
            if (di < dj || (di == dj && i < j)) {
                dup = true;
                break;
            }
        }
        const bool keepj = vj && !dup;
        const unsigned km = __ballot_sync(kFull, keepj);
        if (keepj) {
            const uint32_t pos = out + __popc(km & ((1u << lane) - 1u));
            a.aug_ids[o + pos] = tj;
            a.aug_dists[o + pos] = dj;
        }
        out += __popc(km);
    }
    if (lane == 0) a.aug_cnt[u] = out;
}

// diversify.cpp:26-31 dist_matches
__device__ __forceinline__ bool dist_matches_dev(float x, float y) {
    const float m = fmaxf(1.0f, fmaxf(fabsf(x), fabsf(y)));
    return fabsf(__fsub_rn(x, y)) <= __fmul_rn(1e-5f, m);
}
__device__ __forceinline__ bool cand_before(float di, uint32_t ti, float dj, uint32_t tj) {
    return di != dj ? di < dj : ti < tj;  // candidate_order, diversify.cpp:16-19
}

// ---- stage 2: one CTA per node ---------------------------------------------------
template <int METRIC>
__global__ void __launch_bounds__(kDivThreads, 2) div_stage2_kernel(const DivArgs a) {
    __shared__ DivStage st;
    __shared__ uint32_t owner;
    const uint32_t u = blockIdx.x, tid = threadIdx.x;
    const unsigned long long o = a.aug_off[u];
    const uint32_t m = a.aug_cnt[u];
    uint32_t* ids = a.aug_ids + o;     // deduped, then fixed distances
    float* dists = a.aug_dists + o;
    uint32_t* sid = a.tmp_ids + o;     // sorted by (dist, target)
    float* sdist = a.tmp_dists + o;
    uint32_t* cnt = a.tmp_cnt + o;
    if (tid == 0) owner = u;
    __syncthreads();
    // (1) dist_matches re-check against the owner's row (diversify.cpp:111-117)
    for (uint32_t j0 = 0; j0 < m; j0 += kDivT) {
        const uint32_t nj = min(kDivT, m - j0);
        div_tile<METRIC>(a, st, &owner, 1, ids + j0, nj, [&](uint32_t, uint32_t j, float e) {
            const float cur = dists[j0 + j];
            if (!dist_matches_dev(cur, e)) dists[j0 + j] = e;
        });
    }
    __syncthreads();
    // (2) order by (dist, target): rank = number of entries before it
    for (uint32_t j = tid; j < m; j += kDivThreads) {
        const float dj = dists[j];
        const uint32_t tj = ids[j];
        uint32_t r = 0;
        for (uint32_t i = 0; i < m; ++i) r += cand_before(dists[i], ids[i], dj, tj) ? 1u : 0u;
        sid[r] = tj;
        sdist[r] = dj;
        cnt[r] = 0;
    }
    __syncthreads();
    // (3) lambda_j = #{i != j : occludes(d0i, d0j, dij)}; d0i < d0j implies i < j here
    for (uint32_t i0 = 0; i0 < m; i0 += kDivT) {
        for (uint32_t j0 = i0; j0 < m; j0 += kDivT) {
            const uint32_t ni = min(kDivT, m - i0), nj = min(kDivT, m - j0);
            div_tile<METRIC>(a, st, sid + i0, ni, sid + j0, nj, [&](uint32_t i, uint32_t j, float dij) {
                const float d0i = sdist[i0 + i], d0j = sdist[j0 + j];
                if (d0i < d0j && dij < d0j) atomicAdd(&cnt[j0 + j], 1u);
            });
        }
    }
    __syncthreads();
    // (4) keep lambda <= lambda0, order by (lambda, dist, target), cap at max_degree
    uint32_t* oid = a.out_ids + o;
    uint16_t* olam = a.out_lambda + o;
    float* odist = a.out_dists + o;
    for (uint32_t j = tid; j < m; j += kDivThreads) {
        const uint32_t lj = min(cnt[j], 65535u);
        if (lj > a.lambda0) continue;
        const float dj = sdist[j];
        uint32_t r = 0;
        for (uint32_t i = 0; i < m; ++i) {
            const uint32_t li = min(cnt[i], 65535u);
            if (li > a.lambda0) continue;
            // edge_order (diversify.cpp:21-25); sdist/sid are already (dist, target)-sorted
            r += (li < lj || (li == lj && i < j)) ? 1u : 0u;
        }
        if (a.max_degree == 0 || r < a.max_degree) {
            oid[r] = sid[j];
            olam[r] = (uint16_t)lj;
            odist[r] = dj;
        }
    }
    if (tid == 0) {
        uint32_t kept = 0;
        for (uint32_t j = 0; j < m; ++j) kept += min(cnt[j], 65535u) <= a.lambda0 ? 1u : 0u;
        a.out_cnt[u] = a.max_degree ? min(kept, a.max_degree) : kept;
    }
}

}  // namespace tsdg_dev
