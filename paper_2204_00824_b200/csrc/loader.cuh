// Direct file -> device index loading: the raw bytes of a
// reference .tsdg file (diversify.cpp:274-306) and an fvecs/bvecs file
// (io.cpp:58-121) are streamed to HBM unchanged and decoded there, one warp per
// node / record, straight into the search layout (padded adjacency + lambdas,
// padded fp32 rows).  The host only walks the TSDG degree fields once to get each
// node's byte offset (the records are variable-length).
//
// Validation on the device mirrors the reference loaders' checks: a record
// dimension that differs from the first record's, a non-finite component, an edge
// target >= n.  The kernels only flag the smallest offending record / node; the
// host then re-parses on the CPU to produce the reference's exact message
// (error path only).
#pragma once
#include <cstdint>

namespace tsdg_dev {

__device__ __forceinline__ uint32_t ld_le32(const unsigned char* p) {
    return uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 | uint32_t(p[3]) << 24;
}

// records [0, nrec) of `raw` (each 4 + cb*d bytes) -> out rows [row0, row0+nrec),
// ld floats each, zero padded.  bad: atomicMin of the first failing global record.
__global__ void unpack_vectors_kernel(const unsigned char* __restrict__ raw, uint32_t nrec,
                                      uint32_t row0, uint32_t d, uint32_t cb, uint32_t ld,
                                      float* __restrict__ out, unsigned long long* bad) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    const uint64_t rec = 4ull + (uint64_t)cb * d;
    for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nrec; r += nw) {
        const unsigned char* p = raw + rec * r;
        bool ok = lane != 0 || ld_le32(p) == d;
        float* o = out + (uint64_t)(row0 + r) * ld;
        for (uint32_t j = lane; j < ld; j += 32) {
            float v = 0.0f;
            if (j < d) {
                if (cb == 4) v = __uint_as_float(ld_le32(p + 4 + 4ull * j));
                else v = (float)p[4 + j];
                ok &= isfinite(v);
            }
            o[j] = v;
        }
        if (__any_sync(0xFFFFFFFFu, !ok) && lane == 0) atomicMin(bad, (unsigned long long)(row0 + r));
    }
}

// TSDG node records (deg u32, deg x (target u32, lambda u16, dist f32)) of nodes
// [u0, u1), node u at byte node_off[u] - base of `raw` -> adjacency / lambda rows
// of stride R (pads 0xFFFFFFFF / 0xFFFF) and deg_full.  bad: atomicMin of the
// first node with an out-of-range target (>= n).
__global__ void unpack_graph_kernel(const unsigned char* __restrict__ raw,
                                    const uint64_t* __restrict__ node_off, uint64_t base,
                                    uint32_t u0, uint32_t u1, uint32_t n, uint32_t R,
                                    uint32_t* __restrict__ adj, uint16_t* __restrict__ lam,
                                    uint32_t* __restrict__ deg_full, unsigned long long* bad) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t u = u0 + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5); u < u1; u += nw) {
        const unsigned char* p = raw + (node_off[u] - base);
        const uint32_t deg = ld_le32(p);
        bool ok = true;
        for (uint32_t j = lane; j < R; j += 32) {
            uint32_t t = 0xFFFFFFFFu;
            uint16_t l = 0xFFFF;
            if (j < deg) {
                const unsigned char* e = p + 4 + 10ull * j;
                t = ld_le32(e);
                l = (uint16_t)(e[4] | e[5] << 8);
                ok &= t < n;
            }
            adj[(uint64_t)u * R + j] = t;
            lam[(uint64_t)u * R + j] = l;
        }
        if (lane == 0) deg_full[u] = deg;
        if (__any_sync(0xFFFFFFFFu, !ok) && lane == 0) atomicMin(bad, (unsigned long long)u);
    }
}

}  // namespace tsdg_dev
