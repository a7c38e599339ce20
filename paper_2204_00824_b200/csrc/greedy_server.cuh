// Persistent small-batch server (paper Alg. 1, the latency regime): the cluster
// kernel of greedy_cluster.cuh kept resident and fed through mapped host memory, so
// a request costs no kernel launch, no copy engine and no stream synchronisation.
//
//   host:   writes the queries into the mapped request buffer, then req->seq (release)
//   CTA 0:  polls req->seq over the bus (acquire, system scope) and republishes it in
//           device memory; every other CTA polls that device word (L2)
//   walks:  cluster c runs queries c, c + C, c + 2C, ... of the request: each of its
//           t0 CTAs reads the query straight from host memory, walks (gc_query), and
//           rank 0 merges the t0 lists and writes ids / distances / count straight
//           into the mapped response buffer
//   done:   rank 0 of every cluster fences (system scope) and counts itself done; the
//           last one stores resp->seq, which the host is spinning on.
//
// The server owns its clusters until stopped (req->stop), so it is sized to what can
// be co-resident (tsdg_gpu_server_create checks cudaOccupancyMaxActiveClusters).
#pragma once

#include "greedy_cluster.cuh"

namespace tsdg_dev {

struct GsReq {  // mapped host memory, written by the host
    uint32_t seq;
    uint32_t nq;
    uint32_t stop;
    uint32_t pad;
};
struct GsResp {  // mapped host memory, written by the device
    uint32_t seq;
    uint32_t pad[3];
};

struct GsArgs {
    GcArgs a;
    const GsReq* req;
    const float* req_queries;  // max_batch x d (mapped)
    GsResp* resp;
    uint32_t* resp_ids;        // max_batch x k (mapped)
    float* resp_dists;
    uint32_t* resp_counts;
    uint32_t nclusters;
    uint32_t* dev_seq;   // device memory: the request CTA 0 saw (0xFFFFFFFF = stop)
    uint32_t* dev_done;  // device memory: clusters finished with the current request
};

constexpr uint32_t kServerStop = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int METRIC, bool FAST>
__global__ void __launch_bounds__(kGcThreads) greedy_server_kernel(const GsArgs sa) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const GcArgs& a = sa.a;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t cl = blockIdx.x / a.t0, s = blockIdx.x % a.t0;
    const GcSmem m = gc_smem(a, smem_raw);
    WarpStage w;
    w.sq = m.sq;
    w.stage = reinterpret_cast<float*>(smem_raw + a.off_stage) + (size_t)warp * a.slots * (a.dch + 4);
    w.bar = reinterpret_cast<uint64_t*>(smem_raw + a.off_bar) + warp;
    w.parity = 0;
    w.rowid = nullptr;
    if (lane == 0) mbar_init(w.bar, 1);
    uint32_t* seen = &m.ctl->hops;  // reused as the broadcast slot before each request
    uint32_t last = 0;
    for (;;) {
        if (threadIdx.x == 0) {
            uint32_t cur;
            if (blockIdx.x == 0) {
                for (;;) {
                    cur = ld_acquire_sys(&sa.req->seq);
                    if (cur != last) break;
                    if (ld_acquire_sys(&sa.req->stop)) {
                        cur = kServerStop;
                        break;
                    }
                    __nanosleep(32);
                }
                st_release_gpu(sa.dev_seq, cur);
            } else {
                for (;;) {
                    cur = ld_acquire_gpu(sa.dev_seq);
                    if (cur != last) break;
                    __nanosleep(64);
                }
            }
            *seen = cur;
        }
        __syncthreads();
        const uint32_t cur = *seen;
        __syncthreads();
        if (cur == kServerStop) return;
        last = cur;
        const uint32_t nq = ld_acquire_sys(&sa.req->nq);
        for (uint32_t q = cl; q < nq; q += sa.nclusters) {
            GcOut o;
            o.ids = sa.resp_ids + (size_t)q * a.k;
            o.dists = sa.resp_dists ? sa.resp_dists + (size_t)q * a.k : nullptr;
            o.count = sa.resp_counts + q;
            o.stats = nullptr;
            gc_query<METRIC, FAST, kStageTma>(a, m, w, s, blockIdx.x, sa.req_queries + (size_t)q * a.d, o);
        }
        if (s == 0 && threadIdx.x == 0) {
            __threadfence_system();  // this cluster's results reach host memory first
            const uint32_t prev = atomicAdd(sa.dev_done, 1u);
            if (prev == sa.nclusters - 1) {
                *sa.dev_done = 0;
                __threadfence_system();
                st_release_sys(&sa.resp->seq, cur);
            }
        }
    }
}

}  // namespace tsdg_dev
