// Host side of libtsdg_gpu.so: the C-ABI declared in include/tsdg_gpu.h.
//
// Owns the device index (vector store + padded adjacency + lambdas + cached
// deg_cut tables), validates parameters exactly like the reference front ends
// (bestfirst_search.cpp:112-150, greedy_search.cpp:74-127), sizes the
// persistent kernels for occupancy on the B200's 148 SMs and launches them.
#include <cuda.h>  // CUtensorMap (encoded through the runtime's driver entry point)
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <utility>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <thread>
#include <string>
#include <vector>

#include "../../include/tsdg_gpu.h"
#include <cub/device/device_scan.cuh>

#include "bf_fast.cuh"
#include "diversify.cuh"
#include "exact_scan.cuh"
#include "greedy_cluster.cuh"
#include "loader.cuh"
#include "nndescent.h"
#include "unbounded.cuh"

using namespace tsdg_dev;

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

struct Error {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw Error{code, msg}; }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(TSDG_ERUNTIME, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return TSDG_OK;
    } catch (const Error& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return TSDG_ERUNTIME;
    }
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cuda_check(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

uint32_t round_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

template <class T>
T* dev_alloc(size_t count, cudaStream_t st) {
    T* p = nullptr;
    if (count == 0) count = 1;
    cuda_check(cudaMallocAsync(&p, sizeof(T) * count, st), "cudaMallocAsync");
    return p;
}

}  // namespace

void tsdg_set_error(const std::string& msg) { g_err = msg; }

// Host-side TSDG produced by tsdg_gpu_build (the reference's TsdgGraph fields).
struct tsdg_gpu_graph {
    uint32_t n = 0, k = 0;
    int metric = 0;
    float alpha = 1.2f;
    uint16_t lambda0 = 9;
    std::vector<uint64_t> offsets;
    std::vector<uint32_t> targets;
    std::vector<uint16_t> lambdas;
    std::vector<float> dists;
};

// Replicated index over several devices (one tsdg_gpu_index each).
struct tsdg_gpu_multi {
    std::vector<tsdg_gpu_index*> parts;
};

// Sharded base: one tsdg_gpu_index per shard (local ids), global id = offset + local.
struct tsdg_gpu_sharded {
    std::vector<tsdg_gpu_index*> shards;
    std::vector<uint64_t> offsets;
    uint32_t d = 0;
    // persistent workspace (grow-only, sized for nq_cap queries x k_cap results):
    // per shard its queries and top-k on its own device, an event marking them
    // ready; on the first shard's device the gathered [shard][query][k] block and
    // the merged output.  Serialised by mu.
    std::mutex mu;
    size_t nq_cap = 0, k_cap = 0;
    std::vector<float*> sq;
    std::vector<uint32_t*> sid, scnt;
    std::vector<float*> sdist;
    std::vector<cudaEvent_t> done;
    uint32_t *gid = nullptr, *gcnt = nullptr, *oid = nullptr, *ocnt = nullptr;
    float *gdist = nullptr, *odist = nullptr;
};

struct tsdg_gpu_index {
    int device = 0;
    int sm_count = 148;
    uint32_t n = 0, d = 0, ld = 0, R = 0, max_degree = 0;
    int metric = 0;
    float* vec = nullptr;
    uint32_t* adj = nullptr;
    uint16_t* lam = nullptr;
    uint32_t* deg_full = nullptr;
    uint32_t* counters = nullptr;  // work counters, one per launch slot (never reset:
    uint32_t counter_slot = 0;     // each launch starts from the slot's known value)
    uint32_t counter_val[64] = {};
    cudaEvent_t slot_done[64] = {};        // recorded after each launch on a slot
    cudaStream_t slot_stream[64] = {};     // the stream of that launch
    bool slot_used[64] = {};
    std::map<uint32_t, uint32_t*> degcut;
    std::mutex mu;
    cudaStream_t stream = nullptr;   // for the host-pointer entry points
    cudaStream_t stream2 = nullptr;  // second pipeline stream (copy/compute overlap)
    // grow-only device scratch for the host-pointer entry points
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    // 2-D tensor map of the vectors for TMA tile::gather4 (greedy kernels), made on
    // first use; device copy (64-byte aligned) or nullptr when not encodable
    void* tmap = nullptr;
    uint32_t tmap_box = 0;
    bool tmap_tried = false;
};

namespace {

constexpr uint32_t kCounterSlots = 64;

// Work-queue tickets without a memset per launch: a persistent kernel hands out work
// with atomicAdd on its slot and every warp exits after exactly one fetch past the
// end, so a launch advances the slot by (work items + warps).  The kernel subtracts
// the slot's value at launch time (`base`).  Callers hold idx->mu.
//  - A slot is reused only after its previous launch: a launch on another stream
//    first waits on the event recorded after that launch (same stream: in order), so
//    any number of in-flight launches over any streams never share a live counter.
//  - The host value advances only when the launch was accepted; a rejected launch
//    (bad configuration, no kernel image, ...) never ran and left the word as it was.
struct Ticket {
    uint32_t* ptr;
    uint32_t base;
    uint32_t slot;
};
Ticket next_counter(tsdg_gpu_index* idx, cudaStream_t st) {
    (void)cudaGetLastError();  // commit_counter reads the launch's own status
    const uint32_t slot = idx->counter_slot++ % kCounterSlots;
    if (idx->slot_used[slot] && idx->slot_stream[slot] != st)
        cuda_check(cudaStreamWaitEvent(st, idx->slot_done[slot], 0), "cudaStreamWaitEvent(slot)");
    return Ticket{idx->counters + slot, idx->counter_val[slot], slot};
}
void commit_counter(tsdg_gpu_index* idx, const Ticket& t, uint64_t items, uint64_t warps,
                    cudaStream_t st) {
    if (cudaPeekAtLastError() != cudaSuccess) return;  // not launched: word unchanged
    idx->counter_val[t.slot] += (uint32_t)(items + warps);
    cuda_check(cudaEventRecord(idx->slot_done[t.slot], st), "cudaEventRecord(slot)");
    idx->slot_stream[t.slot] = st;
    idx->slot_used[t.slot] = true;
}

// Cached per-(kernel, device) launch attributes: the host side of a small-batch call
// is part of its latency.
std::mutex g_attr_mu;
std::map<std::pair<const void*, int>, int> g_smem_attr;
std::map<std::tuple<const void*, int, int, size_t>, int> g_occ;
int cur_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}
void set_smem(const void* kern, size_t smem, const char* what) {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    int& v = g_smem_attr[{kern, cur_device()}];
    if ((int)smem > v) {
        cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), what);
        v = (int)smem;
    }
}
int occupancy(const void* kern, int threads, size_t smem) {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    const auto key = std::make_tuple(kern, cur_device(), threads, smem);
    auto it = g_occ.find(key);
    if (it != g_occ.end()) return it->second;
    int per_sm = 0;
    cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem),
               "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
    g_occ[key] = per_sm;
    return per_sm;
}

const uint32_t* get_degcut(tsdg_gpu_index* idx, uint32_t cut, cudaStream_t st) {
    auto it = idx->degcut.find(cut);
    if (it != idx->degcut.end()) return it->second;
    uint32_t* out = nullptr;
    cuda_check(cudaMalloc(&out, sizeof(uint32_t) * std::max<uint32_t>(idx->n, 1)), "cudaMalloc(degcut)");
    if (idx->n) {
        deg_cut_kernel<<<(idx->n + 255) / 256, 256, 0, st>>>(idx->lam, idx->R, idx->deg_full,
                                                             idx->n, cut, out);
        g_launches++;
        cuda_check(cudaGetLastError(), "deg_cut_kernel");
        // the table is shared by later launches on any stream
        cuda_check(cudaStreamSynchronize(st), "deg_cut_kernel");
    }
    idx->degcut[cut] = out;
    return out;
}

// Staged dims per row per gather round: the whole (padded) row when it fits in
// 128 floats, else 128-float chunks.
uint32_t staging_dims(uint32_t ld) { return std::min<uint32_t>(round_up(ld, 8), 128); }

struct Carve {
    uint32_t total = 0;
    uint32_t take(uint32_t bytes, uint32_t align = 16) {
        total = round_up(total, align);
        const uint32_t off = total;
        total += bytes;
        return off;
    }
};

void fill_bf_layout(BfArgs& a) {
    Carve c;
    a.off_bar = c.take(8, 8);
    a.off_query = c.take(a.ld * 4);
    a.gpitch = round_up(4 * (a.dch + 4), 32);
    a.off_stage = c.take(a.tmap ? a.slots / 4 * a.gpitch * 4 : a.slots * (a.dch + 4) * 4, 128);
    a.off_cid = c.take((a.m + 1) * kSegPitch * 4);    // + one scratch row (batched admission)
    a.off_cdist = c.take((a.m + 1) * kSegPitch * 4);
    a.off_csize = c.take(a.m * 4);
    a.off_vid = c.take(a.m * kSegPitch * 4);
    a.off_vsize = c.take(a.m * 4);
    a.off_voldest = c.take(a.m * 4);
    const bool kreg = a.k <= 31;
    a.off_rid = c.take(kreg ? 0 : round_up(a.k + 2, 32) * 4);
    a.off_rdist = c.take(kreg ? 0 : round_up(a.k + 2, 32) * 4);
    a.off_rowid = c.take(32 * 4);
    a.warp_smem = round_up(c.total, 128);
}

// Tuning knobs (environment, read per launch): TSDG_STAGE=tma (default)|ldgsts,
// TSDG_PREFETCH=<bits> (1: next-chunk rows, 2: admitted adjacency; default 0:
// measured neutral-to-slower on C2, see profiles/),
// TSDG_BATCH_MIN=<n> (batched admission when >= n candidates pass the bound; default
// 0 = off: its fixed cost exceeded the sequential replay's on C2, 1.27 vs 1.16 ms),
// TSDG_BF_WARPS=<warps per CTA> (default 1: finest shared-memory granularity),
// TSDG_SLOTS=<staged rows per gather round> (default 16).
int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v && *v ? std::atoi(v) : dflt;
}
bool env_is(const char* name, const char* val) {
    const char* v = std::getenv(name);
    return v && std::strcmp(v, val) == 0;
}

using BfKernel = void (*)(BfArgs);

template <int METRIC, bool FAST>
BfKernel pick_bf(int stage, bool kreg) {
    if (stage == kStageG4 && !FAST)  // gather4 staging: deterministic mode, whole rows
        return kreg ? bf_kernel<METRIC, false, kStageG4, true> : bf_kernel<METRIC, false, kStageG4, false>;
    if (stage != kStageLdgsts)
        return kreg ? bf_kernel<METRIC, FAST, kStageTma, true> : bf_kernel<METRIC, FAST, kStageTma, false>;
    return kreg ? bf_kernel<METRIC, FAST, kStageLdgsts, true> : bf_kernel<METRIC, FAST, kStageLdgsts, false>;
}
BfKernel pick_bf(int metric, bool fast, int stage, bool kreg) {
    if (metric == 0) return fast ? pick_bf<0, true>(stage, kreg) : pick_bf<0, false>(stage, kreg);
    if (metric == 1) return fast ? pick_bf<1, true>(stage, kreg) : pick_bf<1, false>(stage, kreg);
    return fast ? pick_bf<2, true>(stage, kreg) : pick_bf<2, false>(stage, kreg);
}

// bf_fast_kernel per-warp carve: query (generic path), C and V in sentinel form
// (no size fields), needed-row ids and distances.
void fill_bf_fast_layout(BfArgs& a) {
    Carve c;
    a.off_query = c.take(a.ld * 4);
    a.off_cid = c.take(a.m * kSegPitch * 4);
    a.off_cdist = c.take(a.m * kSegPitch * 4);
    a.off_vid = c.take(a.m * kSegPitch * 4);
    a.off_lst = c.take(64 * 4);
    a.off_dl = c.take(64 * 4);
    a.warp_smem = round_up(c.total, 16);
}

template <class K>
int grid_for(K kernel, int threads, size_t smem, int sm_count, uint32_t work_warps,
             int warps_per_cta) {
    const int per_sm = occupancy(reinterpret_cast<const void*>(kernel), threads, smem);
    if (per_sm < 1) fail(TSDG_ERUNTIME, "kernel does not fit on an SM (shared memory)");
    const uint32_t need = (work_warps + warps_per_cta - 1) / warps_per_cta;
    return (int)std::max<uint32_t>(1, std::min<uint32_t>(need, (uint32_t)(per_sm * sm_count)));
}

void validate_bf(const tsdg_gpu_index* idx, const tsdg_bf_params* p) {
    if (!p) fail(TSDG_EINVAL, "bestfirst_search: null params");
    if (idx->n == 0) fail(TSDG_EINVAL, "bestfirst_search: empty graph");
    if (p->k < 1 || p->hop_limit < 1 || p->m_segments < 1 || p->lambda_cut < 1 ||
        p->delta < 0.0f || std::isnan(p->delta))
        fail(TSDG_EINVAL, "bestfirst_search: invalid parameters");
    if (!p->unbounded && p->m_segments > 32)
        fail(TSDG_EINVAL, "bestfirst_search: GPU path supports m_segments <= 32");
    if (p->k > 1024) fail(TSDG_EINVAL, "bestfirst_search: GPU path supports k <= 1024");
}

// unbounded=true: exact queue / visited set (unbounded.cuh), per-warp arena in HBM
void launch_unbounded(tsdg_gpu_index* idx, const float* d_queries, uint32_t nq, uint64_t qbase,
                      const tsdg_bf_params* p, int mode, uint32_t* d_ids, float* d_dists,
                      uint32_t* d_counts, tsdg_query_stats* d_stats, cudaStream_t st) {
    UbArgs a{};
    a.vec = idx->vec;
    a.adj = idx->adj;
    a.degcut = get_degcut(idx, p->lambda_cut, st);
    a.queries = d_queries;
    a.ld = idx->ld;
    a.R = idx->R;
    a.n = idx->n;
    a.d = idx->d;
    a.nq = nq;
    a.qbase = qbase;
    a.k = p->k;
    a.hop_limit = p->hop_limit;
    a.delta = p->delta;
    a.seed = p->seed;
    a.out_ids = d_ids;
    a.out_dists = d_dists;
    a.out_counts = d_counts;
    a.out_stats = d_stats;
    const Ticket tk = next_counter(idx, st);
    a.work_counter = tk.ptr;
    a.work_base = tk.base;
    a.dch = staging_dims(idx->ld);
    a.slots = 32;
    // every id the search can touch: <= min(n, 1 + hop_limit * max degree)
    const uint64_t touch = std::min<uint64_t>(idx->n, 1ull + (uint64_t)p->hop_limit * idx->max_degree) + 32;
    uint64_t hcap = 64;
    while (hcap < 2 * touch + 2) hcap <<= 1;
    a.hcap = (uint32_t)hcap;
    a.qcap = (uint32_t)(touch + 2);
    const size_t per_warp = hcap * 5 + (size_t)a.qcap * 8 + (size_t)(p->k + 2) * 8;
    const size_t budget = size_t(2) << 30;
    uint32_t warps = (uint32_t)std::max<size_t>(1, std::min<size_t>(budget / per_warp, 4u * idx->sm_count));
    warps = std::min(warps, nq);
    char* arena = dev_alloc<char>(per_warp * warps + 256, st);
    size_t off = 0;
    auto take = [&](size_t bytes) { char* r = arena + off; off += (bytes + 15) & ~size_t(15); return r; };
    a.hkeys = reinterpret_cast<uint32_t*>(take(hcap * 4 * warps));
    a.hstate = reinterpret_cast<uint8_t*>(take(hcap * warps));
    a.heap_d = reinterpret_cast<float*>(take((size_t)a.qcap * 4 * warps));
    a.heap_i = reinterpret_cast<uint32_t*>(take((size_t)a.qcap * 4 * warps));
    a.rid = reinterpret_cast<uint32_t*>(take((size_t)(p->k + 2) * 4 * warps));
    a.rdist = reinterpret_cast<float*>(take((size_t)(p->k + 2) * 4 * warps));
    int* over = dev_alloc<int>(1, st);
    cuda_check(cudaMemsetAsync(over, 0, sizeof(int), st), "memset");
    a.overflow = over;
    Carve c;
    a.off_bar = c.take(8, 8);
    a.off_query = c.take(a.ld * 4);
    a.off_stage = c.take(a.slots * (a.dch + 4) * 4, 128);
    a.warp_smem = round_up(c.total, 128);
    void (*kern)(UbArgs);
    const bool fast = mode == TSDG_MODE_FAST;
    if (idx->metric == 0) kern = fast ? bf_unbounded_kernel<0, true> : bf_unbounded_kernel<0, false>;
    else if (idx->metric == 1) kern = fast ? bf_unbounded_kernel<1, true> : bf_unbounded_kernel<1, false>;
    else kern = fast ? bf_unbounded_kernel<2, true> : bf_unbounded_kernel<2, false>;
    set_smem(reinterpret_cast<const void*>(kern), a.warp_smem, "cudaFuncSetAttribute(unbounded)");
    kern<<<warps, 32, a.warp_smem, st>>>(a);
    commit_counter(idx, tk, nq, warps, st);
    g_launches++;
    cuda_check(cudaGetLastError(), "bf_unbounded_kernel launch");
    int h_over = 0;
    cuda_check(cudaMemcpyAsync(&h_over, over, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
    cudaFreeAsync(arena, st);
    cudaFreeAsync(over, st);
    cuda_check(cudaStreamSynchronize(st), "bf_unbounded_kernel");
    if (h_over) fail(TSDG_ERUNTIME, "bestfirst_search(unbounded): arena capacity exceeded");
}

const void* vectors_tmap(tsdg_gpu_index* idx, uint32_t box, cudaStream_t st);

void launch_bestfirst(tsdg_gpu_index* idx, const float* d_queries, uint32_t nq, uint64_t qbase,
                      const tsdg_bf_params* p, int mode, uint32_t* d_ids, float* d_dists,
                      uint32_t* d_counts, tsdg_query_stats* d_stats, cudaStream_t st) {
    if (nq == 0) return;
    if (p->unbounded) {
        launch_unbounded(idx, d_queries, nq, qbase, p, mode, d_ids, d_dists, d_counts, d_stats, st);
        return;
    }
    BfArgs a{};
    a.vec = idx->vec;
    a.adj = idx->adj;
    a.degcut = get_degcut(idx, p->lambda_cut, st);
    a.queries = d_queries;
    a.ld = idx->ld;
    a.R = idx->R;
    a.n = idx->n;
    a.d = idx->d;
    a.nq = nq;
    a.qbase = qbase;
    a.k = p->k;
    a.hop_limit = p->hop_limit;
    a.delta = p->delta;
    a.m = p->m_segments;
    a.seed = p->seed;
    a.out_ids = d_ids;
    a.out_dists = d_dists;
    a.out_counts = d_counts;
    a.out_stats = d_stats;
    const Ticket tk = next_counter(idx, st);
    a.work_counter = tk.ptr;
    a.work_base = tk.base;
    a.dch = staging_dims(idx->ld);
    a.slots = (uint32_t)std::max(1, std::min(32, env_int("TSDG_SLOTS", 16)));
    a.prefetch = (uint32_t)env_int("TSDG_PREFETCH", 0);
    a.batch_min = (uint32_t)std::max(0, env_int("TSDG_BATCH_MIN", 0));
    // fast mode, k <= 31, rows of at most 128 floats: register-direct warp-cooperative
    // kernel (bf_fast.cuh).  Wider rows keep the staged kernel: at d = 960 (C4) the
    // register-direct form measured 24.0 ms vs 15.9 ms for the staged deterministic
    // kernel (its query no longer fits in registers and a row takes 8 batch rounds).
    // TSDG_FAST_KERNEL=staged / =register forces either.
    const bool reg_fast = env_is("TSDG_FAST_KERNEL", "register") ||
                          (idx->ld <= 128 && !env_is("TSDG_FAST_KERNEL", "staged"));
    if (mode == TSDG_MODE_FAST && a.k <= 31 && reg_fast) {
        // bit 0: bulk L2 prefetch of the rows past a hop's first batch (default, C2:
        // 0.85 -> 0.79 ms); bit 1: L2 prefetch of admitted nodes' adjacency (slower)
        a.prefetch = (uint32_t)env_int("TSDG_FAST_PREFETCH", 1);
        fill_bf_fast_layout(a);
        // row class: 1 = 128 floats, 2 = fewer (query in registers), 0 = generic
        const bool reg_q = idx->ld <= 128 && idx->ld == idx->d &&
                           (reinterpret_cast<uintptr_t>(d_queries) & 15u) == 0;
        const int seg = reg_q ? (idx->ld == 128 ? 1 : 2) : 0;
        // Group forms (2 or 4 warps per query) when the batch leaves most resident
        // query slots empty (a strong-scaled rank's slice): pairs below one query per
        // CTA slot of the one-warp-per-query launch.  TSDG_FAST_GROUP=1|2|4 (or
        // TSDG_FAST_PAIR=0|1) forces.
        // variant 1 (64 registers, 32 warps / SM) for L2 over 128-float rows: C2 0.7025
        // vs 0.7086 ms for variant 0 (80 registers; before the REDUX arg-min variant 1
        // spilled and was slower, 0.863 ms) — profiles/fast_variants_r2b.jsonl
        const int variant = env_int("TSDG_FAST_VARIANT", idx->metric == 0 && seg == 1 ? 1 : 0);
        const BfKernel single = bf_fast_kernel_for(idx->metric, seg, variant);
        const size_t smem1 = (size_t)a.warp_smem * kFastWarps;
        set_smem(reinterpret_cast<const void*>(single), smem1, "cudaFuncSetAttribute(bf_fast)");
        const int slots = grid_for(single, kFastWarps * 32, smem1, idx->sm_count, 0xFFFFFFFFu, 1);
        int grp = nq <= (uint32_t)slots ? 2 : 1;
        const int pair_env = env_int("TSDG_FAST_PAIR", -1);
        if (pair_env >= 0) grp = pair_env == 1 ? 2 : 1;
        const int grp_env = env_int("TSDG_FAST_GROUP", 0);
        if (grp_env == 1 || grp_env == 2 || grp_env == 4) grp = grp_env;
        // (the group forms keep the 80-register budget: a pair in 64 registers took
        // 0.249 vs 0.208 ms for a 1250-query slice)
        const BfKernel kern = grp > 1 ? bf_fast_kernel_for(idx->metric, seg, 0, grp) : single;
        const size_t smem = grp > 1 ? (size_t)a.warp_smem + 16 : smem1;
        const int threads = (grp == 4 ? 4 : kFastWarps) * 32;
        if (grp > 1) set_smem(reinterpret_cast<const void*>(kern), smem, "cudaFuncSetAttribute(bf_fast group)");
        // work fetches: one per query plus one final per fetching warp (the leader only
        // in the group forms)
        const int grid = grp > 1 ? grid_for(kern, threads, smem, idx->sm_count, nq, 1)
                                 : grid_for(kern, threads, smem, idx->sm_count, nq, kFastWarps);
        kern<<<grid, threads, smem, st>>>(a);
        commit_counter(idx, tk, nq, (uint64_t)grid * (grp > 1 ? 1 : kFastWarps), st);
        g_launches++;
        cuda_check(cudaGetLastError(), "bf_fast_kernel launch");
        return;
    }
    // row staging (TSDG_STAGE=g4|tma|ldgsts): deterministic mode with whole rows
    // (ld <= dch) and slots in groups of 4 uses gather4 tensor copies (C2 bench point:
    // 1.100 vs 1.147 ms, identical results; tools/det_stage.py); else one bulk copy
    // per row
    int stage = env_is("TSDG_STAGE", "ldgsts") ? kStageLdgsts : kStageTma;
    a.tmap = nullptr;
    if (stage == kStageTma && !env_is("TSDG_STAGE", "tma") && mode != TSDG_MODE_FAST && idx->ld <= a.dch &&
        a.slots % 4 == 0) {
        a.tmap = vectors_tmap(idx, a.dch + 4, st);
        if (a.tmap) stage = kStageG4;
    }
    fill_bf_layout(a);
    const int wpc = std::max(1, std::min(kBfWarps, env_int("TSDG_BF_WARPS", 1)));
    const size_t smem = (size_t)a.warp_smem * wpc;
    const BfKernel kern = pick_bf(idx->metric, mode == TSDG_MODE_FAST, stage, a.k <= 31);
    set_smem(reinterpret_cast<const void*>(kern), smem, "cudaFuncSetAttribute(bf)");
    const int grid = grid_for(kern, wpc * 32, smem, idx->sm_count, nq, wpc);
    kern<<<grid, wpc * 32, smem, st>>>(a);
    commit_counter(idx, tk, nq, (uint64_t)grid * wpc, st);
    g_launches++;
    cuda_check(cudaGetLastError(), "bf_kernel launch");
}

void validate_greedy(const tsdg_gpu_index* idx, uint32_t k, const tsdg_greedy_params* p) {
    if (!p) fail(TSDG_EINVAL, "small_batch_search: null params");
    if (k < 1) fail(TSDG_EINVAL, "small_batch_search: k must be >= 1");
    if (p->t0 < 1) fail(TSDG_EINVAL, "small_batch_search: t0 must be >= 1");
    if ((uint64_t)k > 32ull * p->t0) fail(TSDG_EINVAL, "small_batch_search: k exceeds 32 * t0");
    if (p->lambda_cut < 1) fail(TSDG_EINVAL, "greedy_search_once: lambda_cut must be >= 1");
    if (p->hop_limit < 1) fail(TSDG_EINVAL, "greedy_search_once: hop limit must be >= 1");
    if (idx->n == 0) fail(TSDG_EINVAL, "select_start: empty graph");
    if (p->t0 > 256) fail(TSDG_EINVAL, "small_batch_search: GPU path supports t0 <= 256");
}

struct WalkBuffers {
    uint32_t* ids = nullptr;
    float* dists = nullptr;
    uint32_t* hops = nullptr;
    uint32_t* evals = nullptr;
};

WalkBuffers alloc_walks(uint32_t walks, cudaStream_t st) {
    WalkBuffers b;
    cuda_check(cudaMallocAsync(&b.ids, sizeof(uint32_t) * 32 * walks, st), "cudaMallocAsync");
    cuda_check(cudaMallocAsync(&b.dists, sizeof(float) * 32 * walks, st), "cudaMallocAsync");
    cuda_check(cudaMallocAsync(&b.hops, sizeof(uint32_t) * walks, st), "cudaMallocAsync");
    cuda_check(cudaMallocAsync(&b.evals, sizeof(uint32_t) * walks, st), "cudaMallocAsync");
    return b;
}
void free_walks(WalkBuffers& b, cudaStream_t st) {
    cudaFreeAsync(b.ids, st);
    cudaFreeAsync(b.dists, st);
    cudaFreeAsync(b.hops, st);
    cudaFreeAsync(b.evals, st);
}

void launch_walks(tsdg_gpu_index* idx, const float* d_queries, uint32_t nq, uint32_t t0,
                  uint32_t hop_limit, uint32_t cut, uint64_t seed, const uint64_t* d_states,
                  WalkBuffers& wb, cudaStream_t st, bool fast = false) {
    GrArgs a{};
    a.vec = idx->vec;
    a.adj = idx->adj;
    a.degcut = get_degcut(idx, cut, st);
    a.queries = d_queries;
    a.ld = idx->ld;
    a.R = idx->R;
    a.n = idx->n;
    a.d = idx->d;
    a.nq = nq;
    a.t0 = t0;
    a.hop_limit = hop_limit;
    a.seed = seed;
    a.walk_states = d_states;
    a.walk_ids = wb.ids;
    a.walk_dists = wb.dists;
    a.walk_hops = wb.hops;
    a.walk_evals = wb.evals;
    const Ticket tk = next_counter(idx, st);
    a.work_counter = tk.ptr;
    a.work_base = tk.base;
    a.dch = staging_dims(idx->ld);
    a.slots = 32;
    // row staging: gather4 tensor copies for L2 rows of <= dch floats (C2, t0=10,
    // batch 256 / 1024 / 4096: 162 / 388 / 1304 vs 180 / 430 / 1437 us with one bulk
    // copy per row, bit-exact); TSDG_GR_STAGE=tma forces per-row copies
    if (!env_is("TSDG_GR_STAGE", "tma") && !env_is("TSDG_STAGE", "ldgsts") && idx->ld <= a.dch &&
        idx->metric == 0)
        a.tmap = vectors_tmap(idx, a.dch + 4, st);
    const bool g4 = a.tmap != nullptr;
    a.gpitch = round_up(4 * (a.dch + 4), 32);
    Carve c;
    a.off_bar = c.take(8, 8);
    a.off_query = c.take(a.ld * 4);
    a.off_stage = c.take(g4 ? a.slots / 4 * a.gpitch * 4 : a.slots * (a.dch + 4) * 4, 128);
    a.off_rowid = c.take(g4 ? 32 * 4 : 0);
    a.warp_smem = round_up(c.total, 128);
    const int wpc = std::max(1, std::min(kGrWarps, env_int("TSDG_GR_WARPS", 1)));
    const size_t smem = (size_t)a.warp_smem * wpc;
    using GrKernel = void (*)(GrArgs);
    const bool tma = !env_is("TSDG_STAGE", "ldgsts");
    GrKernel kern;
    if (g4)
        kern = fast ? greedy_walk_kernel<0, true, kStageG4> : greedy_walk_kernel<0, false, kStageG4>;
    else if (idx->metric == 0)
        kern = fast ? (tma ? greedy_walk_kernel<0, true, kStageTma> : greedy_walk_kernel<0, true, kStageLdgsts>)
                    : (tma ? greedy_walk_kernel<0, false, kStageTma> : greedy_walk_kernel<0, false, kStageLdgsts>);
    else if (idx->metric == 1)
        kern = fast ? greedy_walk_kernel<1, true, kStageLdgsts> : greedy_walk_kernel<1, false, kStageLdgsts>;
    else
        kern = fast ? greedy_walk_kernel<2, true, kStageLdgsts> : greedy_walk_kernel<2, false, kStageLdgsts>;
    set_smem(reinterpret_cast<const void*>(kern), smem, "cudaFuncSetAttribute(greedy)");
    const int grid = grid_for(kern, wpc * 32, smem, idx->sm_count, nq * t0, wpc);
    kern<<<grid, wpc * 32, smem, st>>>(a);
    commit_counter(idx, tk, (uint64_t)nq * t0, (uint64_t)grid * wpc, st);
    g_launches++;
    cuda_check(cudaGetLastError(), "greedy_walk_kernel launch");
}

// Tensor map of the vectors for tile::gather4 row gathers: 2-D {ld, n} fp32, row
// stride ld * 4 bytes, box {box, 1} (box = the staging pitch dch + 4: the columns past
// ld are out of bounds and arrive as zeros).  Encoded once per index through the
// driver entry point (no libcuda link); nullptr when the driver rejects it (the
// kernels then stage with one bulk copy per row).  Caller holds idx->mu.
// 2-D fp32 tensor map {cols, rows} with row stride ld floats and box {bc, br};
// false when the driver entry point or the encoding is unavailable.
bool encode_tmap_2d(CUtensorMap* tm, const float* base, uint64_t cols, uint64_t rows, uint64_t ld,
                    uint32_t bc, uint32_t br, CUtensorMapSwizzle swz) {
    using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                CUtensorMapFloatOOBfill);
    static Encode enc = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        (void)cudaGetLastError();
        return reinterpret_cast<Encode>(fn);
    }();
    if (!enc || rows == 0 || bc > 256 || br > 256 || (bc * 4) % 16 || (ld * 4) % 16 ||
        (reinterpret_cast<uintptr_t>(base) & 15u))
        return false;
    const cuuint64_t gdim[2] = {cols, rows};
    const cuuint64_t gstride[1] = {ld * 4};
    const cuuint32_t bdim[2] = {bc, br};
    const cuuint32_t estride[2] = {1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), gdim, gstride, bdim, estride,
               CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

const void* vectors_tmap(tsdg_gpu_index* idx, uint32_t box, cudaStream_t st) {
    if (idx->tmap_tried) return idx->tmap_box == box ? idx->tmap : nullptr;
    idx->tmap_tried = true;
    alignas(64) CUtensorMap tm;
    if (!encode_tmap_2d(&tm, idx->vec, idx->ld, idx->n, idx->ld, box, 1, CU_TENSOR_MAP_SWIZZLE_NONE))
        return nullptr;
    void* dev = nullptr;
    cuda_check(cudaMalloc(&dev, sizeof(CUtensorMap)), "cudaMalloc(tensor map)");
    cuda_check(cudaMemcpyAsync(dev, &tm, sizeof(CUtensorMap), cudaMemcpyHostToDevice, st), "H2D tensor map");
    cuda_check(cudaStreamSynchronize(st), "tensor map upload");
    idx->tmap = dev;
    idx->tmap_box = box;
    return dev;
}

// At index creation (no caller stream, no stream capture in progress): the tensor
// map the gather4 staging of the greedy and deterministic kernels uses, so that a
// launch never has to allocate or synchronise for it.
void make_vectors_tmap(tsdg_gpu_index* idx) {
    const uint32_t dch = staging_dims(idx->ld);
    if (idx->ld <= dch) vectors_tmap(idx, dch + 4, idx->stream);
}

// CTA-per-walk / cluster-per-query greedy (greedy_cluster.cuh).  Returns false when
// the cluster launch is not possible (then the caller merges walks itself).
// GcArgs + shared-memory carve of the CTA-per-walk kernels.
size_t fill_gc_args(GcArgs& a, tsdg_gpu_index* idx, uint32_t k, const tsdg_greedy_params* p,
                    bool cluster, cudaStream_t st, uint32_t stage_req = kStageG4,
                    uint32_t compact_slots = 0) {
    a.vec = idx->vec;
    a.adj = idx->adj;
    a.degcut = get_degcut(idx, p->lambda_cut, st);
    a.adj_prefetch = (uint32_t)env_int("TSDG_GC_ADJ_PREFETCH", 0);  // measured: no gain (C2 batch 1/8/64)
    a.merge_warp = (uint32_t)env_int("TSDG_GC_MERGE_WARP", 1);
    a.slice = a.merge_warp ? (uint32_t)std::max(1, std::min(32, env_int("TSDG_GC_SLICE", 32))) : 32u;
    a.early_next = (uint32_t)env_int("TSDG_GC_EARLY", 1);
    a.spec_next = (uint32_t)env_int("TSDG_GC_SPEC", 1);
    a.ld = idx->ld;
    a.R = idx->R;
    a.n = idx->n;
    a.d = idx->d;
    a.t0 = p->t0;
    a.hop_limit = p->hop_limit;
    a.k = k;
    a.seed = p->seed;
    a.cluster = cluster ? 1 : 0;
    a.npow2 = 32;
    while (a.npow2 < p->t0 * 32) a.npow2 <<= 1;
    a.dch = staging_dims(idx->ld);
    a.slots = 32;
    // compact slab (launch_greedy_cta, for grids above one wave): fewer row slots per
    // warp and warp 0 (the merge warp, which gathers only in select_start) borrowing
    // warp 1's slab, so that more CTAs fit on an SM
    a.share0 = 0;
    if (compact_slots && a.merge_warp) {
        a.slots = compact_slots;
        a.slice = std::min(a.slice, compact_slots);
        a.share0 = 1;
    }
    // row staging (TSDG_GC_STAGE=g4|tma|ldgsts): tile::gather4 tensor copies by
    // default when the rows fit one staging round (ld <= dch) and the tensor map
    // encodes; else one bulk copy per row
    a.stage = kStageTma;
    a.tmap = nullptr;
    if (env_is("TSDG_GC_STAGE", "ldgsts")) {
        a.stage = kStageLdgsts;
    } else if (stage_req == kStageG4 && !env_is("TSDG_GC_STAGE", "tma") && idx->ld <= a.dch) {
        a.tmap = vectors_tmap(idx, a.dch + 4, st);
        if (a.tmap) a.stage = kStageG4;
    }
    a.gpitch = round_up(4 * (a.dch + 4), 32);
    const uint32_t warp_stage = a.stage == kStageG4 ? a.slots / 4 * a.gpitch : a.slots * (a.dch + 4);
    Carve c;
    a.off_bar = c.take(8 * kGcWarps, 8);
    a.off_ctl = c.take(sizeof(GcCtl));
    a.off_list = c.take(32 * 8);
    a.off_query = c.take(a.ld * 4);
    a.off_pos = c.take((size_t)idx->R * 16);  // two parity sets of (distance, id)
    a.off_stage = c.take((kGcWarps - a.share0) * warp_stage * 4, 128);
    a.off_pool = c.take(a.cluster ? a.npow2 * 8 + (kGcThreads + 1) * 4 + 2 * a.t0 * 4 : 0);
    a.off_rowid = c.take(kGcWarps * 32 * 4);
    return round_up(c.total, 128);
}

template <int M>
void (*pick_gc(bool fast, uint32_t stage))(GcArgs) {
    if (stage == kStageG4) return fast ? greedy_cta_kernel<M, true, kStageG4> : greedy_cta_kernel<M, false, kStageG4>;
    if (stage == kStageLdgsts)
        return fast ? greedy_cta_kernel<M, true, kStageLdgsts> : greedy_cta_kernel<M, false, kStageLdgsts>;
    return fast ? greedy_cta_kernel<M, true, kStageTma> : greedy_cta_kernel<M, false, kStageTma>;
}

bool launch_greedy_cta(tsdg_gpu_index* idx, const float* d_queries, uint32_t nq, uint32_t k,
                       const tsdg_greedy_params* p, bool fast, const uint64_t* d_states,
                       uint32_t* d_ids, float* d_dists, uint32_t* d_counts,
                       tsdg_query_stats* d_stats, WalkBuffers* wb, cudaStream_t st) {
    GcArgs a{};
    size_t smem = fill_gc_args(a, idx, k, p, wb == nullptr, st);
    int smem_sm = 0, resv = 0;
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, idx->device);
    cudaDeviceGetAttribute(&resv, cudaDevAttrReservedSharedMemoryPerBlock, idx->device);
    const uint64_t walks = (uint64_t)nq * p->t0;
    // more walks than one wave of CTAs: the compact slab (20 row slots per warp, the
    // merge warp borrowing a gather warp's slab) when it fits more CTAs per SM.
    // TSDG_GC_COMPACT=0|1 forces.
    {
        const int cenv = env_int("TSDG_GC_COMPACT", -1);
        const uint64_t per = (uint64_t)smem_sm / (smem + resv);
        bool want = cenv == 1 || (cenv < 0 && walks > per * (uint64_t)idx->sm_count);
        if (want && a.merge_warp) {
            GcArgs b{};
            const size_t smem_c = fill_gc_args(b, idx, k, p, wb == nullptr, st, kStageG4, 20);
            if (cenv == 1 || (uint64_t)smem_sm / (smem_c + resv) > per) {
                a = b;
                smem = smem_c;
            }
        }
    }
    if (a.stage == kStageG4 && !env_is("TSDG_GC_STAGE", "g4") && !a.share0) {
        // the gather4 slab is ~3% larger (128-byte aligned 4-slot groups): when that
        // costs a resident CTA per SM and the grid needs it, stage per row instead
        // (C2, t0=10, batch 64: 117 vs 94 us)
        GcArgs b{};
        const size_t smem_t = fill_gc_args(b, idx, k, p, wb == nullptr, st, kStageTma);
        const uint64_t per_g4 = (uint64_t)smem_sm / (smem + resv), per_t = (uint64_t)smem_sm / (smem_t + resv);
        if (per_g4 < per_t && (uint64_t)nq * p->t0 > per_g4 * (uint64_t)idx->sm_count) {
            a = b;
            smem = smem_t;
        }
    }
    a.queries = d_queries;
    a.nq = nq;
    a.walk_states = d_states;
    a.out_ids = d_ids;
    a.out_dists = d_dists;
    a.out_counts = d_counts;
    a.out_stats = d_stats;
    if (wb) {
        a.walk_ids = wb->ids;
        a.walk_dists = wb->dists;
        a.walk_hops = wb->hops;
        a.walk_evals = wb->evals;
    }
    using GcKernel = void (*)(GcArgs);
    GcKernel kern;
    // row staging (fill_gc_args): gather4 tensor copies, TMA bulk copies (one per row)
    // or LDGSTS (one coalesced 512 B row per warp instruction).  All pipelined across
    // hops; C2 batch 1, t0=10: TMA 51 us, LDGSTS 59 us (its 32 cp.async per lane
    // issue slower)
    if (idx->metric == 0) kern = pick_gc<0>(fast, a.stage);
    else if (idx->metric == 1) kern = pick_gc<1>(fast, a.stage);
    else kern = pick_gc<2>(fast, a.stage);
    set_smem(reinterpret_cast<const void*>(kern), smem, "cudaFuncSetAttribute(greedy_cta)");
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(nq * p->t0);
    cfg.blockDim = dim3(kGcThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    if (a.cluster) {
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = p->t0;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        // cluster feasibility per (kernel, device, t0, smem), checked once
        static std::map<std::tuple<const void*, int, uint32_t, size_t>, bool> ok_cache;
        std::lock_guard<std::mutex> lk(g_attr_mu);
        const auto key = std::make_tuple(reinterpret_cast<const void*>(kern), cur_device(), p->t0, smem);
        auto it = ok_cache.find(key);
        if (it == ok_cache.end()) {
            if (p->t0 > 8)
                cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                           "cudaFuncSetAttribute(non-portable cluster)");
            int nclusters = 0;
            const bool ok = cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) == cudaSuccess &&
                            nclusters >= 1;
            if (!ok) cudaGetLastError();
            it = ok_cache.emplace(key, ok).first;
        }
        if (!it->second) return false;
    }
    cuda_check(cudaLaunchKernelEx(&cfg, kern, a), "greedy_cta_kernel launch");
    g_launches++;
    return true;
}

// Kernel choice for Alg. 1: the latency-oriented CTA/cluster kernel for small
// batches (the paper's small-batch regime), the warp-per-walk
// kernel when there are enough walks to fill the GPU.  TSDG_GREEDY=cta|warp forces.
bool use_cta_greedy(const tsdg_gpu_index* idx, uint32_t nq, uint32_t t0) {
    if (env_is("TSDG_GREEDY", "cta")) return true;
    if (env_is("TSDG_GREEDY", "warp")) return false;
    // measured crossover on C2 (profiles/greedy_crossover_r2.jsonl): the cluster kernel
    // is faster up to ~4.5 walks per SM (t0=10: 64 queries 94 vs 125 us; 128 queries
    // 158 vs 132 us; t0=16: 32 queries 94 vs 122 us, 64 queries 155 vs 130 us)
    const int mx = env_int("TSDG_GREEDY_CTA_MAX_WALKS", 0);
    const uint64_t limit = mx > 0 ? (uint64_t)mx : (uint64_t)idx->sm_count * 9 / 2;
    return (uint64_t)nq * t0 <= limit;
}

void launch_greedy(tsdg_gpu_index* idx, const float* d_queries, uint32_t nq, uint32_t k,
                   const tsdg_greedy_params* p, int mode, uint32_t* d_ids, float* d_dists,
                   uint32_t* d_counts, tsdg_query_stats* d_stats, cudaStream_t st) {
    if (nq == 0) return;
    const bool fast = mode == TSDG_MODE_FAST;
    const bool cta = use_cta_greedy(idx, nq, p->t0);
    if (cta && p->t0 <= 16 &&
        launch_greedy_cta(idx, d_queries, nq, k, p, fast, nullptr, d_ids, d_dists, d_counts,
                          d_stats, nullptr, st))
        return;
    WalkBuffers wb = alloc_walks(nq * p->t0, st);
    if (cta) {
        launch_greedy_cta(idx, d_queries, nq, k, p, fast, nullptr, nullptr, nullptr, nullptr,
                          nullptr, &wb, st);
    } else {
        launch_walks(idx, d_queries, nq, p->t0, p->hop_limit, p->lambda_cut, p->seed, nullptr, wb,
                     st, fast);
    }
    uint32_t npow2 = 32;
    while (npow2 < p->t0 * 32) npow2 <<= 1;
    const size_t smem = (size_t)npow2 * 8 + (kMergeThreads + 1) * 4;
    cuda_check(cudaFuncSetAttribute(greedy_merge_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
               "cudaFuncSetAttribute(merge)");
    greedy_merge_kernel<<<nq, kMergeThreads, smem, st>>>(wb.ids, wb.dists, wb.hops, wb.evals,
                                                         p->t0, k, npow2, d_ids, d_dists,
                                                         d_counts, d_stats);
    g_launches++;
    cuda_check(cudaGetLastError(), "greedy_merge_kernel launch");
    free_walks(wb, st);
}

void check_cosine_queries(const tsdg_gpu_index* idx, const float* queries, uint32_t nq) {
    // require_metric_ready (vectors.cpp:83-95), applied to host query buffers.
    if (idx->metric != TSDG_METRIC_COSINE || !queries) return;
    for (uint32_t q = 0; q < nq; ++q) {
        float sq = 0.0f;
        const float* r = queries + (size_t)q * idx->d;
        for (uint32_t i = 0; i < idx->d; ++i) sq += r[i] * r[i];
        if (std::fabs(sq - 1.0f) > 1e-4f)
            fail(TSDG_EINVAL, "Cosine requires unit-normalized vectors (row " + std::to_string(q) +
                                  " has squared norm " + std::to_string(sq) +
                                  "); pass the set through normalized_copy first");
    }
}


}  // namespace

namespace {

// ---- exact top-k scan (ground truth / brute-force k-NN graph) ----------------
constexpr uint32_t kScanMaxK = 384;
// Candidate buffer per query: k kept + one tile of appended rows.
uint32_t scan_buffer(uint32_t k) { return round_up(k + kScanBT, 4); }

void launch_exact_topk(const float* d_base, uint32_t n, uint32_t ld_b, const float* d_queries,
                       uint32_t nq, uint32_t ld_q, uint32_t d, uint32_t k, int metric,
                       int exclude_self, uint64_t self_base, uint32_t* d_ids, float* d_dists,
                       cudaStream_t st) {
    if (nq == 0) return;
    if (k < 1 || k > kScanMaxK) fail(TSDG_EINVAL, "exact_topk: need 1 <= k <= 384");
    if (d < 1 || ld_b % 4 || ld_q % 4 || ld_b < d || ld_q < d)
        fail(TSDG_EINVAL, "exact_topk: row strides must be multiples of 4 floats and >= d");
    if (metric < 0 || metric > 2) fail(TSDG_EINVAL, "invalid metric");
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    int sms = 148;
    cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "attr");
    ScanArgs a{};
    a.base = d_base;
    a.queries = d_queries;
    a.n = n;
    a.nq = nq;
    a.d = d;
    a.ld_b = ld_b;
    a.ld_q = ld_q;
    a.k = k;
    a.P = scan_buffer(k);
    a.exclude_self = exclude_self;
    a.self_base = self_base;
    a.keep = ~0ull;
    const size_t smem = scan_smem_bytes(a.P);
    // row chunks by one TMA tensor copy each (128-byte swizzle) when the base can be
    // described by a tensor map (16-byte aligned, fewer than 2^31 rows: TMA
    // coordinates are signed 32-bit); else 8 cp.async per thread.  TSDG_SCAN_TMA=0
    // forces cp.async.
    alignas(64) CUtensorMap tm{};
    const bool tma = !env_is("TSDG_SCAN_TMA", "0") && n < (1u << 31) &&
                     encode_tmap_2d(&tm, d_base, ld_b, n, ld_b, kScanDC, kScanBT, CU_TENSOR_MAP_SWIZZLE_128B);
    using ScanKernel = void (*)(ScanArgs, CUtensorMap);
    ScanKernel kern;
    if (tma) kern = metric == 0 ? exact_scan_kernel<0, true> : metric == 1 ? exact_scan_kernel<1, true>
                                                                           : exact_scan_kernel<2, true>;
    else kern = metric == 0 ? exact_scan_kernel<0, false> : metric == 1 ? exact_scan_kernel<1, false>
                                                                        : exact_scan_kernel<2, false>;
    set_smem(reinterpret_cast<const void*>(kern), smem, "cudaFuncSetAttribute(exact_scan)");
    const int per_sm = occupancy(reinterpret_cast<const void*>(kern), kScanThreads, smem);
    const uint32_t slots = (uint32_t)std::max(1, per_sm) * (uint32_t)sms;
    const uint32_t qtiles = (nq + kScanQT - 1) / kScanQT;
    // split the base rows so that the grid is >= ~4 waves; each split >= 8 tiles
    uint32_t S = std::max<uint32_t>(1, (4 * slots + qtiles - 1) / qtiles);
    S = std::min<uint32_t>(S, std::max<uint32_t>(1, n / (8 * kScanBT)));
    if (env_int("TSDG_SCAN_SPLITS", 0) > 0) S = (uint32_t)env_int("TSDG_SCAN_SPLITS", 0);
    // merge_splits_kernel follows one split list per lane
    S = std::min<uint32_t>(S, 32);
    uint32_t rows = round_up((std::max<uint32_t>(n, 1) + S - 1) / S, kScanBT);
    S = std::max<uint32_t>(1, (n + rows - 1) / rows);
    a.rows_per_split = rows;
    uint32_t* tids = d_ids;
    float* tdist = d_dists;
    if (S > 1) {
        tids = dev_alloc<uint32_t>((size_t)S * nq * k, st);
        tdist = dev_alloc<float>((size_t)S * nq * k, st);
    }
    a.out_ids = tids;
    a.out_dists = tdist;
    kern<<<dim3(qtiles, S), kScanThreads, smem, st>>>(a, tm);
    g_launches++;
    cuda_check(cudaGetLastError(), "exact_scan_kernel launch");
    if (S > 1) {
        merge_splits_kernel<<<(nq + 7) / 8, 256, 0, st>>>(tids, tdist, S, nq, k, d_ids, d_dists);
        g_launches++;
        cuda_check(cudaGetLastError(), "merge_splits_kernel launch");
        cudaFreeAsync(tids, st);
        cudaFreeAsync(tdist, st);
    }
}

// Host rows (n x d, dense) -> device rows padded to ld = round_up(d, 4), zero fill.
float* upload_rows(const float* h, uint32_t n, uint32_t d, uint32_t ld, cudaStream_t st) {
    float* p = dev_alloc<float>((size_t)std::max<uint32_t>(n, 1) * ld, st);
    if (!n) return p;
    if (ld == d) {
        cuda_check(cudaMemcpyAsync(p, h, (size_t)n * d * 4, cudaMemcpyHostToDevice, st), "H2D rows");
    } else {
        cuda_check(cudaMemsetAsync(p, 0, (size_t)n * ld * 4, st), "memset rows");
        cuda_check(cudaMemcpy2DAsync(p, ld * 4, h, d * 4, d * 4, n, cudaMemcpyHostToDevice, st),
                   "H2D rows");
    }
    return p;
}

void scan_to_host(const float* d_base, uint32_t n, uint32_t ld, const float* d_queries, uint32_t nq,
                  uint32_t d, uint32_t k, int metric, int exclude_self, uint32_t* ids,
                  float* dists, cudaStream_t st) {
    uint32_t* di = dev_alloc<uint32_t>((size_t)nq * k, st);
    float* dd = dev_alloc<float>((size_t)nq * k, st);
    launch_exact_topk(d_base, n, ld, d_queries, nq, ld, d, k, metric, exclude_self, 0, di, dd, st);
    cuda_check(cudaMemcpyAsync(ids, di, (size_t)nq * k * 4, cudaMemcpyDeviceToHost, st), "D2H ids");
    if (dists)
        cuda_check(cudaMemcpyAsync(dists, dd, (size_t)nq * k * 4, cudaMemcpyDeviceToHost, st),
                   "D2H dists");
    cudaFreeAsync(di, st);
    cudaFreeAsync(dd, st);
    cuda_check(cudaStreamSynchronize(st), "exact_topk");
}

// ---- GPU two-stage diversification (diversify.cuh) ------------------------------
template <class T>
struct DevBuf {
    T* p = nullptr;
    cudaStream_t st;
    DevBuf(size_t n, cudaStream_t s) : st(s) { p = dev_alloc<T>(n, s); }
    ~DevBuf() { cudaFreeAsync(p, st); }
    DevBuf(const DevBuf&) = delete;
};

__global__ void div_total_kernel(const uint32_t* a, const uint32_t* b, uint32_t n,
                                 unsigned long long* out) {
    const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u < n) out[u + 1] = (unsigned long long)a[u] + (b ? b[u] : 0u);
    if (u == 0) out[0] = 0;
}
__global__ void div_gather_kernel(const unsigned long long* src_off, const unsigned long long* dst_off,
                                  const uint32_t* cnt, uint32_t n, const uint32_t* ids,
                                  const uint16_t* lam, const float* dists, uint32_t* o_ids,
                                  uint16_t* o_lam, float* o_dists) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t u = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (u >= n) return;
    for (uint32_t j = lane; j < cnt[u]; j += 32) {
        o_ids[dst_off[u] + j] = ids[src_off[u] + j];
        o_lam[dst_off[u] + j] = lam[src_off[u] + j];
        o_dists[dst_off[u] + j] = dists[src_off[u] + j];
    }
}

// offsets[0..n] = prefix sums of a[u] (+ b[u]); returns the total.
unsigned long long div_prefix(const uint32_t* a, const uint32_t* b, uint32_t n,
                              unsigned long long* off, cudaStream_t st) {
    div_total_kernel<<<(std::max<uint32_t>(n, 1) + 255) / 256, 256, 0, st>>>(a, b, n, off);
    g_launches++;
    size_t tmp = 0;
    cuda_check(cub::DeviceScan::InclusiveSum(nullptr, tmp, off + 1, off + 1, (int)n, st), "cub scan");
    DevBuf<char> t(tmp, st);
    cuda_check(cub::DeviceScan::InclusiveSum(t.p, tmp, off + 1, off + 1, (int)n, st), "cub scan");
    unsigned long long total = 0;
    cuda_check(cudaMemcpyAsync(&total, off + n, 8, cudaMemcpyDeviceToHost, st), "D2H total");
    cuda_check(cudaStreamSynchronize(st), "prefix");
    return total;
}

void gpu_build(const float* base, uint32_t n, uint32_t d, const uint32_t* knn_ids,
               const float* knn_dists, uint32_t k, float alpha, uint16_t lambda0,
               uint32_t max_degree, int metric, tsdg_gpu_graph& g, uint64_t* stats,
               cudaStream_t st) {
    const uint32_t ld = round_up(d, 4);
    DevBuf<float> vec_keep(0, st);
    cudaFreeAsync(vec_keep.p, st);  // adopt the uploaded rows instead
    vec_keep.p = upload_rows(base, n, d, ld, st);
    DivArgs a{};
    a.vec = vec_keep.p;
    a.n = n;
    a.d = d;
    a.ld = ld;
    a.metric = metric;
    a.keep = ~0ull;
    a.k = k;
    a.alpha = alpha;
    a.lambda0 = lambda0;
    a.max_degree = max_degree;
    const size_t nk = (size_t)n * k;
    DevBuf<uint32_t> kid(nk, st), s1i(nk, st), s1c(n, st), rc(n, st), cur(n, st), acnt(n, st),
        ocnt(n, st);
    DevBuf<float> kd(nk, st), s1d(nk, st);
    DevBuf<int> err(1, st);
    DevBuf<unsigned long long> aoff(n + 1, st), foff(n + 1, st);
    cuda_check(cudaMemcpyAsync(kid.p, knn_ids, nk * 4, cudaMemcpyHostToDevice, st), "H2D knn");
    cuda_check(cudaMemcpyAsync(kd.p, knn_dists, nk * 4, cudaMemcpyHostToDevice, st), "H2D knn");
    cuda_check(cudaMemsetAsync(err.p, 0, 4, st), "memset");
    cuda_check(cudaMemsetAsync(rc.p, 0, (size_t)n * 4, st), "memset");
    cuda_check(cudaMemsetAsync(cur.p, 0, (size_t)n * 4, st), "memset");
    a.knn_ids = kid.p;
    a.knn_dists = kd.p;
    a.s1_ids = s1i.p;
    a.s1_dists = s1d.p;
    a.s1_cnt = s1c.p;
    a.err = err.p;
    auto s1 = metric == 0 ? div_stage1_kernel<0> : metric == 1 ? div_stage1_kernel<1> : div_stage1_kernel<2>;
    s1<<<n, kDivThreads, 0, st>>>(a);
    g_launches++;
    cuda_check(cudaGetLastError(), "div_stage1_kernel launch");
    int herr = 0;
    cuda_check(cudaMemcpyAsync(&herr, err.p, 4, cudaMemcpyDeviceToHost, st), "D2H err");
    cuda_check(cudaStreamSynchronize(st), "div_stage1_kernel");
    if (herr & 1) fail(TSDG_EINVAL, "stage1_relaxed_gd: candidates must be sorted ascending by distance");
    if (herr & 2) fail(TSDG_EINVAL, "add_reverse_edges: target out of range");
    const unsigned blocks_nk = (unsigned)((nk + 255) / 256);
    div_rev_count_kernel<<<blocks_nk, 256, 0, st>>>(a, rc.p);
    g_launches++;
    const unsigned long long s1_edges = div_prefix(s1c.p, nullptr, n, foff.p, st);  // stage-1 count
    const unsigned long long total = div_prefix(s1c.p, rc.p, n, aoff.p, st);
    DevBuf<uint32_t> aid(total, st), tid_(total, st), tcnt(total, st), oid(total, st);
    DevBuf<float> adist(total, st), tdist(total, st), odist(total, st);
    DevBuf<uint16_t> olam(total, st);
    a.aug_off = aoff.p;
    a.aug_ids = aid.p;
    a.aug_dists = adist.p;
    a.aug_cnt = acnt.p;
    a.tmp_ids = tid_.p;
    a.tmp_dists = tdist.p;
    a.tmp_cnt = tcnt.p;
    a.out_ids = oid.p;
    a.out_lambda = olam.p;
    a.out_dists = odist.p;
    a.out_cnt = ocnt.p;
    div_fill_kernel<<<blocks_nk, 256, 0, st>>>(a, cur.p);
    g_launches++;
    div_dedup_kernel<<<(n + 7) / 8, 256, 0, st>>>(a);
    g_launches++;
    auto s2 = metric == 0 ? div_stage2_kernel<0> : metric == 1 ? div_stage2_kernel<1> : div_stage2_kernel<2>;
    s2<<<n, kDivThreads, 0, st>>>(a);
    g_launches++;
    cuda_check(cudaGetLastError(), "div_stage2_kernel launch");
    const unsigned long long aug_edges = div_prefix(acnt.p, nullptr, n, foff.p, st);
    const unsigned long long fin = div_prefix(ocnt.p, nullptr, n, foff.p, st);
    DevBuf<uint32_t> fid(fin, st);
    DevBuf<uint16_t> flam(fin, st);
    DevBuf<float> fdist(fin, st);
    div_gather_kernel<<<(n + 7) / 8, 256, 0, st>>>(aoff.p, foff.p, ocnt.p, n, oid.p, olam.p, odist.p,
                                                   fid.p, flam.p, fdist.p);
    g_launches++;
    g.offsets.resize((size_t)n + 1);
    g.targets.resize(fin);
    g.lambdas.resize(fin);
    g.dists.resize(fin);
    static_assert(sizeof(unsigned long long) == sizeof(uint64_t), "u64");
    cuda_check(cudaMemcpyAsync(g.offsets.data(), foff.p, ((size_t)n + 1) * 8, cudaMemcpyDeviceToHost, st), "D2H");
    if (fin) {
        cuda_check(cudaMemcpyAsync(g.targets.data(), fid.p, fin * 4, cudaMemcpyDeviceToHost, st), "D2H");
        cuda_check(cudaMemcpyAsync(g.lambdas.data(), flam.p, fin * 2, cudaMemcpyDeviceToHost, st), "D2H");
        cuda_check(cudaMemcpyAsync(g.dists.data(), fdist.p, fin * 4, cudaMemcpyDeviceToHost, st), "D2H");
    }
    cuda_check(cudaStreamSynchronize(st), "gpu_build");
    if (stats) {
        stats[0] = (uint64_t)n * k;
        stats[1] = s1_edges;
        stats[2] = aug_edges;
        stats[3] = fin;
    }
}

void write_tsdg_file(const tsdg_gpu_graph& g, const char* path) {
    FILE* f = std::fopen(path, "wb");
    if (!f) fail(TSDG_ERUNTIME, std::string(path) + ": cannot open for writing");
    std::vector<unsigned char> buf;
    auto put = [&](const void* p, size_t nb) {
        const unsigned char* c = static_cast<const unsigned char*>(p);
        buf.insert(buf.end(), c, c + nb);
    };
    const uint32_t version = 1;
    const uint64_t n64 = g.n;
    const uint8_t metric = (uint8_t)g.metric;
    put("TSDG", 4);  // little-endian host (x86-64 / aarch64), as the reference's LeWriter
    put(&version, 4);
    put(&n64, 8);
    put(&metric, 1);
    put(&g.k, 4);
    put(&g.alpha, 4);
    put(&g.lambda0, 2);
    for (uint32_t u = 0; u < g.n; ++u) {
        const uint32_t deg = (uint32_t)(g.offsets[u + 1] - g.offsets[u]);
        put(&deg, 4);
        for (uint64_t e = g.offsets[u]; e < g.offsets[u + 1]; ++e) {
            put(&g.targets[e], 4);
            put(&g.lambdas[e], 2);
            put(&g.dists[e], 4);
        }
        if (buf.size() > (64u << 20)) {
            if (std::fwrite(buf.data(), 1, buf.size(), f) != buf.size()) {
                std::fclose(f);
                fail(TSDG_ERUNTIME, std::string(path) + ": write failed");
            }
            buf.clear();
        }
    }
    const bool ok = std::fwrite(buf.data(), 1, buf.size(), f) == buf.size();
    if (std::fclose(f) != 0 || !ok) fail(TSDG_ERUNTIME, std::string(path) + ": write failed");
}

}  // namespace

namespace {
// Runs fn(i) on one host thread per device; returns the first failure (status,
// message) in device order.
template <class F>
void run_per_device(size_t ndev, F&& fn) {
    std::vector<int> rc(ndev, TSDG_OK);
    std::vector<std::string> msg(ndev);
    std::vector<std::thread> th;
    for (size_t i = 0; i < ndev; ++i)
        th.emplace_back([&, i] {
            rc[i] = fn(i);
            if (rc[i] != TSDG_OK) msg[i] = tsdg_gpu_last_error();
        });
    for (auto& t : th) t.join();
    for (size_t i = 0; i < ndev; ++i)
        if (rc[i] != TSDG_OK) fail(rc[i], msg[i]);
}
// Sharded index workspace: release (also of a partially built index), and grow-only
// reservation for nq queries x k results.
void sharded_release_buffers(tsdg_gpu_sharded* sh) {
    for (size_t i = 0; i < sh->shards.size() && i < sh->sid.size(); ++i) {
        if (!sh->shards[i]) continue;
        DeviceGuard dg(sh->shards[i]->device);
        cudaStreamSynchronize(sh->shards[i]->stream);
        cudaFree(sh->sq[i]);
        cudaFree(sh->sid[i]);
        cudaFree(sh->sdist[i]);
        cudaFree(sh->scnt[i]);
        sh->sq[i] = nullptr;
        sh->sid[i] = sh->scnt[i] = nullptr;
        sh->sdist[i] = nullptr;
    }
    if (!sh->shards.empty() && sh->shards[0]) {
        DeviceGuard dg(sh->shards[0]->device);
        cudaStreamSynchronize(sh->shards[0]->stream);
        for (void* p : {(void*)sh->gid, (void*)sh->gdist, (void*)sh->gcnt, (void*)sh->oid,
                        (void*)sh->odist, (void*)sh->ocnt})
            cudaFree(p);
    }
    sh->gid = sh->gcnt = sh->oid = sh->ocnt = nullptr;
    sh->gdist = sh->odist = nullptr;
    sh->nq_cap = sh->k_cap = 0;
}
void sharded_free(tsdg_gpu_sharded* sh) {
    sharded_release_buffers(sh);
    for (size_t i = 0; i < sh->done.size(); ++i) {
        if (!sh->done[i]) continue;
        DeviceGuard dg(sh->shards[i] ? sh->shards[i]->device : 0);
        cudaEventDestroy(sh->done[i]);
        sh->done[i] = nullptr;
    }
    for (auto*& p : sh->shards) {
        if (p) tsdg_gpu_index_destroy(p);
        p = nullptr;
    }
}
void sharded_reserve(tsdg_gpu_sharded* sh, size_t nq, size_t k) {
    if (nq <= sh->nq_cap && k <= sh->k_cap) return;
    const size_t nqc = std::max(nq, sh->nq_cap), kc = std::max(k, sh->k_cap);
    sharded_release_buffers(sh);
    const size_t S = sh->shards.size(), blk = nqc * kc;
    auto alloc = [](auto*& p, size_t count, const char* what) {
        cuda_check(cudaMalloc(reinterpret_cast<void**>(&p), std::max<size_t>(count, 1) * sizeof(*p)), what);
    };
    for (size_t i = 0; i < S; ++i) {
        DeviceGuard dg(sh->shards[i]->device);
        alloc(sh->sq[i], nqc * sh->d, "cudaMalloc(shard queries)");
        alloc(sh->sid[i], blk, "cudaMalloc(shard ids)");
        alloc(sh->sdist[i], blk, "cudaMalloc(shard dists)");
        alloc(sh->scnt[i], nqc, "cudaMalloc(shard counts)");
    }
    DeviceGuard dg(sh->shards[0]->device);
    alloc(sh->gid, S * blk, "cudaMalloc(gather)");
    alloc(sh->gdist, S * blk, "cudaMalloc(gather)");
    alloc(sh->gcnt, S * nqc, "cudaMalloc(gather)");
    alloc(sh->oid, blk, "cudaMalloc(merge)");
    alloc(sh->odist, blk, "cudaMalloc(merge)");
    alloc(sh->ocnt, nqc, "cudaMalloc(merge)");
    sh->nq_cap = nqc;
    sh->k_cap = kc;
}

// Device alias of a host buffer [p, p + bytes) when it lies in one mapped pinned
// allocation (cudaHostAlloc / cudaMallocHost / registered-mapped memory, e.g. torch
// pin_memory()); nullptr otherwise (pageable memory: the copy pipeline is used).
template <class T>
T* mapped_alias(T* p, size_t bytes) {
    if (!p || bytes == 0) return nullptr;
    cudaPointerAttributes a{}, b{};
    const char* last = reinterpret_cast<const char*>(p) + bytes - 1;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess || cudaPointerGetAttributes(&b, last) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (a.type != cudaMemoryTypeHost || b.type != cudaMemoryTypeHost || !a.devicePointer || !b.devicePointer)
        return nullptr;
    if (static_cast<const char*>(b.devicePointer) - static_cast<const char*>(a.devicePointer) !=
        static_cast<ptrdiff_t>(bytes - 1))
        return nullptr;
    return static_cast<T*>(a.devicePointer);
}

// contiguous slice [begin, end) of nq for part i of ndev
void slice_of(uint32_t nq, size_t ndev, size_t i, uint32_t& b, uint32_t& e) {
    b = (uint32_t)((uint64_t)nq * i / ndev);
    e = (uint32_t)((uint64_t)nq * (i + 1) / ndev);
}
}  // namespace

// tsdg_io.cpp (host parsing; error messages in the reference's wording)
uint32_t tsdg_vector_component_bytes(const std::string& path);
int tsdg_vector_file_shape(const std::string& path, uint32_t* n, uint32_t* d, std::string& err);
int tsdg_parse_vector_file(const std::string& path, float* out, uint32_t* n, uint32_t* d,
                           std::string& err);
int tsdg_parse_header_bytes(const std::string& path, const unsigned char* p, size_t size,
                            tsdg_graph_header* h, uint64_t* body_off, std::string& err);
std::string tsdg_truncated_message(const std::string& path, uint64_t file_size);

namespace {

// Frees whatever an index holds (also a partially built one).
void free_index(tsdg_gpu_index* idx) {
    DeviceGuard dg(idx->device);
    if (idx->stream) cudaStreamSynchronize(idx->stream);
    if (idx->stream2) cudaStreamSynchronize(idx->stream2);
    for (auto& kv : idx->degcut) cudaFree(kv.second);
    if (idx->scratch) cudaFree(idx->scratch);
    if (idx->tmap) cudaFree(idx->tmap);
    cudaFree(idx->vec);
    cudaFree(idx->adj);
    cudaFree(idx->lam);
    cudaFree(idx->deg_full);
    cudaFree(idx->counters);
    for (auto& e : idx->slot_done)
        if (e) cudaEventDestroy(e);
    if (idx->stream) cudaStreamDestroy(idx->stream);
    if (idx->stream2) cudaStreamDestroy(idx->stream2);
    delete idx;
}
struct IndexOwner {
    tsdg_gpu_index* p = new tsdg_gpu_index();
    ~IndexOwner() {
        if (p) free_index(p);
    }
    tsdg_gpu_index* release() { return std::exchange(p, nullptr); }
};

// Device, streams, the stream-ordered pool policy and the work counters.
void init_index_runtime(tsdg_gpu_index* idx, int device) {
    idx->device = device;
    cudaDeviceProp prop{};
    cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    idx->sm_count = prop.multiProcessorCount;
    cuda_check(cudaStreamCreateWithFlags(&idx->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaStreamCreateWithFlags(&idx->stream2, cudaStreamNonBlocking), "cudaStreamCreate");
    // keep stream-ordered allocations cached across calls (no re-mapping per search)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cuda_check(cudaMalloc(&idx->counters, kCounterSlots * 4), "cudaMalloc(counters)");
    cuda_check(cudaMemset(idx->counters, 0, kCounterSlots * 4), "cudaMemset(counters)");
    for (auto& e : idx->slot_done)
        cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate(slot)");
}

// File byte ranges -> device, through two pinned staging buffers: the read of
// chunk i+1 (split over several threads) overlaps the H2D copy and the decode of
// chunk i.  push() copies into the stager's own device buffer and enqueues
// decode(dev) after it (stream order protects the buffer); push_to() copies
// straight to a caller device address.  visit(host, bytes) runs on the host copy
// while its H2D copy is in flight.
// Two pinned host buffers + their copy-done events, shared by the loads of one call.
struct PinnedPair {
    size_t bytes;
    cudaStream_t st;
    unsigned char* host[2] = {};
    cudaEvent_t done[2] = {};
    uint64_t next = 0;  // alternates across the stagers that share the pair
    PinnedPair(size_t b, cudaStream_t s) : bytes(b), st(s) {
        for (int i = 0; i < 2; ++i) {
            cuda_check(cudaMallocHost(&host[i], bytes), "cudaMallocHost(stager)");
            cuda_check(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming), "cudaEventCreate");
        }
    }
    ~PinnedPair() {
        cudaStreamSynchronize(st);
        for (int i = 0; i < 2; ++i) {
            if (host[i]) cudaFreeHost(host[i]);
            if (done[i]) cudaEventDestroy(done[i]);
        }
    }
};

class FileStager {
public:
    FileStager(const std::string& path, PinnedPair& pin, bool dev_buffers)
        : path_(path), chunk_(pin.bytes), st_(pin.st), pin_(pin) {
        fd_ = open(path.c_str(), O_RDONLY);
        if (fd_ < 0) fail(TSDG_ERUNTIME, path + ": cannot open for reading");
        struct stat sb {};
        if (fstat(fd_, &sb) != 0) fail(TSDG_ERUNTIME, path + ": cannot stat");
        size_ = (uint64_t)sb.st_size;
        for (int b = 0; b < 2; ++b) {
            host_[b] = pin.host[b];
            done_[b] = pin.done[b];
            if (dev_buffers) cuda_check(cudaMalloc(&dev_[b], chunk_), "cudaMalloc(stager)");
        }
    }
    ~FileStager() {
        cudaStreamSynchronize(st_);
        for (int b = 0; b < 2; ++b)
            if (dev_[b]) cudaFree(dev_[b]);
        if (fd_ >= 0) close(fd_);
    }
    uint64_t size() const { return size_; }
    void read_at(uint64_t off, size_t bytes, unsigned char* dst) {
        // a few threads per chunk: one pread stream does not saturate the page cache
        constexpr size_t kPart = 8ull << 20;
        const size_t parts = std::min<size_t>(8, (bytes + kPart - 1) / kPart);
        std::vector<std::thread> th;
        std::atomic<bool> ok{true};
        auto part = [&](size_t i) {
            const size_t b0 = bytes * i / parts, b1 = bytes * (i + 1) / parts;
            size_t got = b0;
            while (got < b1) {
                const ssize_t r = pread(fd_, dst + got, b1 - got, (off_t)(off + got));
                if (r <= 0) {
                    ok = false;
                    return;
                }
                got += (size_t)r;
            }
        };
        for (size_t i = 1; i < parts; ++i) th.emplace_back(part, i);
        if (parts) part(0);
        for (auto& t : th) t.join();
        if (!ok) fail(TSDG_ERUNTIME, path_ + ": read failed near byte offset " + std::to_string(off));
    }
    template <class Decode, class Visit>
    void push(uint64_t off, size_t bytes, Decode&& decode, Visit&& visit) {
        const int b = stage(off, bytes);
        cuda_check(cudaMemcpyAsync(dev_[b], host_[b], bytes, cudaMemcpyHostToDevice, st_), "H2D file chunk");
        cuda_check(cudaEventRecord(done_[b], st_), "cudaEventRecord");
        decode(static_cast<const unsigned char*>(dev_[b]));
        visit(static_cast<const unsigned char*>(host_[b]), bytes);
    }
    template <class Visit>
    void push_to(uint64_t off, size_t bytes, unsigned char* dst, Visit&& visit) {
        const int b = stage(off, bytes);
        cuda_check(cudaMemcpyAsync(dst, host_[b], bytes, cudaMemcpyHostToDevice, st_), "H2D file chunk");
        cuda_check(cudaEventRecord(done_[b], st_), "cudaEventRecord");
        visit(static_cast<const unsigned char*>(host_[b]), bytes);
    }

private:
    int stage(uint64_t off, size_t bytes) {
        const int b = (int)(pin_.next++ & 1);
        cuda_check(cudaEventSynchronize(done_[b]), "stager wait");  // H2D from host_[b] finished
        read_at(off, bytes, host_[b]);
        return b;
    }
    std::string path_;
    size_t chunk_;
    cudaStream_t st_;
    PinnedPair& pin_;
    int fd_ = -1;
    uint64_t size_ = 0;
    unsigned char* host_[2] = {};
    unsigned char* dev_[2] = {};
    cudaEvent_t done_[2] = {};
};

constexpr size_t kStageChunk = 32ull << 20;

int decode_grid(const tsdg_gpu_index* idx) { return idx->sm_count * 8; }

// vectors file -> idx->vec (n x ld, zero padded); d_bad <- first bad record
void load_vectors_to_device(tsdg_gpu_index* idx, const std::string& path, PinnedPair& pin,
                            unsigned long long* d_bad) {
    const uint32_t cb = tsdg_vector_component_bytes(path);
    const uint64_t rec = 4ull + (uint64_t)cb * idx->d;
    const uint32_t per = (uint32_t)std::max<uint64_t>(1, pin.bytes / rec);
    if (per * rec > pin.bytes) fail(TSDG_ERUNTIME, path + ": record exceeds the staging chunk");
    FileStager fs(path, pin, true);
    for (uint32_t r0 = 0; r0 < idx->n; r0 += per) {
        const uint32_t nr = std::min(per, idx->n - r0);
        fs.push((uint64_t)r0 * rec, (size_t)nr * rec,
                [&](const unsigned char* dev) {
                    unpack_vectors_kernel<<<decode_grid(idx), 256, 0, idx->stream>>>(
                        dev, nr, r0, idx->d, cb, idx->ld, idx->vec, d_bad);
                    g_launches++;
                    cuda_check(cudaGetLastError(), "unpack_vectors_kernel launch");
                },
                [](const unsigned char*, size_t) {});
    }
}

// TSDG file -> idx->adj / lam / deg_full in ONE read of the file: the body streams
// into a transient device copy while the host walks the degree fields of each
// staged chunk (node byte offsets, max degree, truncation check); then the node
// offsets go up and one decode kernel builds the padded rows.
void load_graph_to_device(tsdg_gpu_index* idx, const std::string& path, uint64_t body_off,
                          PinnedPair& pin, unsigned long long* d_bad) {
    FileStager fs(path, pin, false);
    const uint64_t body = fs.size() > body_off ? fs.size() - body_off : 0;
    DevBuf<unsigned char> raw(std::max<uint64_t>(body, 1), idx->stream);
    std::vector<uint64_t> node_off((size_t)idx->n + 1);
    uint64_t pos = 0;  // body offset of the next node record
    uint32_t u = 0, maxdeg = 0;
    unsigned char tail[4] = {};  // the 4 body bytes before the current chunk
    uint64_t cs = 0;             // current chunk start (body offset)
    auto walk = [&](const unsigned char* h, size_t bytes) {
        const uint64_t ce = cs + bytes;
        auto byte_at = [&](uint64_t x) { return x >= cs ? h[x - cs] : tail[4 - (cs - x)]; };
        while (u < idx->n && pos + 4 <= ce) {
            const uint32_t deg = uint32_t(byte_at(pos)) | uint32_t(byte_at(pos + 1)) << 8 |
                                 uint32_t(byte_at(pos + 2)) << 16 | uint32_t(byte_at(pos + 3)) << 24;
            node_off[u++] = pos;
            maxdeg = std::max(maxdeg, deg);
            pos += 4 + 10ull * deg;
        }
        unsigned char nt[4] = {};
        for (int i = 0; i < 4; ++i) {
            const int64_t x = (int64_t)ce - 4 + i;  // body offset of new tail byte i
            if (x >= (int64_t)cs) nt[i] = h[x - (int64_t)cs];
            else if (x >= 0) nt[i] = tail[4 - ((int64_t)cs - x)];
        }
        std::memcpy(tail, nt, 4);
        cs = ce;
    };
    for (uint64_t off = 0; off < body; off += pin.bytes) {
        const size_t bytes = (size_t)std::min<uint64_t>(pin.bytes, body - off);
        fs.push_to(body_off + off, bytes, raw.p + off, walk);
    }
    if (u < idx->n || pos > body) fail(TSDG_ERUNTIME, tsdg_truncated_message(path, fs.size()));
    node_off[idx->n] = pos;
    idx->max_degree = maxdeg;
    idx->R = std::max<uint32_t>(4, round_up(maxdeg, 4));
    const size_t rows = std::max<uint32_t>(idx->n, 1);
    cuda_check(cudaMalloc(&idx->adj, rows * idx->R * 4), "cudaMalloc(adj)");
    cuda_check(cudaMalloc(&idx->lam, rows * idx->R * 2), "cudaMalloc(lam)");
    cuda_check(cudaMalloc(&idx->deg_full, rows * 4), "cudaMalloc(deg)");
    DevBuf<uint64_t> d_off(node_off.size(), idx->stream);
    cuda_check(cudaMemcpyAsync(d_off.p, node_off.data(), node_off.size() * 8, cudaMemcpyHostToDevice,
                               idx->stream),
               "H2D node offsets");
    if (idx->n) {
        unpack_graph_kernel<<<decode_grid(idx), 256, 0, idx->stream>>>(
            raw.p, d_off.p, 0, 0, idx->n, idx->n, idx->R, idx->adj, idx->lam, idx->deg_full, d_bad);
        g_launches++;
        cuda_check(cudaGetLastError(), "unpack_graph_kernel launch");
    }
    // node_off must outlive the async copy
    cuda_check(cudaStreamSynchronize(idx->stream), "graph decode");
}

}  // namespace

extern "C" {

const char* tsdg_gpu_last_error(void) { return g_err.c_str(); }
int tsdg_gpu_abi_version(void) { return TSDG_GPU_ABI_VERSION; }
uint64_t tsdg_gpu_launch_count(void) { return g_launches.load(); }

int tsdg_gpu_host_buffer_mapped(const void* p, uint64_t bytes) {
    return mapped_alias(p, (size_t)bytes) != nullptr ? 1 : 0;
}

int tsdg_gpu_index_create(const float* base, uint32_t n, uint32_t d, const uint64_t* offsets,
                          const uint32_t* targets, const uint16_t* lambdas, int metric,
                          int device, tsdg_gpu_index** out) {
    return guarded([&] {
        if (!out) fail(TSDG_EINVAL, "index_create: null out");
        *out = nullptr;
        if (d < 1) fail(TSDG_EINVAL, "index_create: d must be >= 1");
        if (metric < 0 || metric > 2) fail(TSDG_EINVAL, "invalid metric");
        if (n > 0 && (!base || !offsets || !targets || !lambdas))
            fail(TSDG_EINVAL, "index_create: null input array");
        uint32_t maxdeg = 0;
        for (uint32_t u = 0; u < n; ++u) {
            if (offsets[u + 1] < offsets[u]) fail(TSDG_EINVAL, "index_create: offsets not monotone");
            maxdeg = std::max<uint32_t>(maxdeg, (uint32_t)(offsets[u + 1] - offsets[u]));
        }
        const uint64_t E = n ? offsets[n] : 0;
        for (uint64_t j = 0; j < E; ++j)
            if (targets[j] >= n) fail(TSDG_EINVAL, "index_create: edge target out of range");
        DeviceGuard dg(device);
        IndexOwner own;
        tsdg_gpu_index* idx = own.p;
        idx->n = n;
        idx->d = d;
        idx->ld = round_up(d, 4);
        idx->metric = metric;
        idx->max_degree = maxdeg;
        idx->R = std::max<uint32_t>(4, round_up(maxdeg, 4));
        init_index_runtime(idx, device);
        // vectors, rows padded to ld floats (16-byte aligned for TMA bulk copies)
        const size_t nv = (size_t)std::max<uint32_t>(n, 1) * idx->ld;
        cuda_check(cudaMalloc(&idx->vec, nv * sizeof(float)), "cudaMalloc(vectors)");
        if (n) {
            if (idx->ld == d) {
                cuda_check(cudaMemcpy(idx->vec, base, (size_t)n * d * 4, cudaMemcpyHostToDevice),
                           "cudaMemcpy(vectors)");
            } else {
                cuda_check(cudaMemset(idx->vec, 0, nv * sizeof(float)), "cudaMemset");
                cuda_check(cudaMemcpy2D(idx->vec, idx->ld * 4, base, d * 4, d * 4, n,
                                        cudaMemcpyHostToDevice),
                           "cudaMemcpy2D(vectors)");
            }
        }
        // padded adjacency + lambdas + full degrees
        const size_t na = (size_t)std::max<uint32_t>(n, 1) * idx->R;
        std::vector<uint32_t> hadj(na, kInvalid);
        std::vector<uint16_t> hlam(na, 0xFFFF);
        std::vector<uint32_t> hdeg(std::max<uint32_t>(n, 1), 0);
        for (uint32_t u = 0; u < n; ++u) {
            const uint64_t b = offsets[u], e = offsets[u + 1];
            hdeg[u] = (uint32_t)(e - b);
            std::memcpy(&hadj[(size_t)u * idx->R], targets + b, (e - b) * 4);
            std::memcpy(&hlam[(size_t)u * idx->R], lambdas + b, (e - b) * 2);
        }
        cuda_check(cudaMalloc(&idx->adj, na * 4), "cudaMalloc(adj)");
        cuda_check(cudaMalloc(&idx->lam, na * 2), "cudaMalloc(lam)");
        cuda_check(cudaMalloc(&idx->deg_full, hdeg.size() * 4), "cudaMalloc(deg)");
        cuda_check(cudaMemcpy(idx->adj, hadj.data(), na * 4, cudaMemcpyHostToDevice), "cudaMemcpy(adj)");
        cuda_check(cudaMemcpy(idx->lam, hlam.data(), na * 2, cudaMemcpyHostToDevice), "cudaMemcpy(lam)");
        cuda_check(cudaMemcpy(idx->deg_full, hdeg.data(), hdeg.size() * 4, cudaMemcpyHostToDevice),
                   "cudaMemcpy(deg)");
        make_vectors_tmap(idx);
        *out = own.release();
    });
}

int tsdg_gpu_index_create_from_file(const char* tsdg_path, const float* base, uint32_t n,
                                    uint32_t d, int device, tsdg_gpu_index** out) {
    tsdg_graph_header h{};
    int rc = tsdg_read_tsdg_header(tsdg_path, &h);
    if (rc) return rc;
    if (h.n != n) {
        g_err = "index_create_from_file: graph has " + std::to_string(h.n) + " nodes, base has " +
                std::to_string(n);
        return TSDG_EINVAL;
    }
    std::vector<uint64_t> off(h.n + 1);
    std::vector<uint32_t> tgt(h.num_edges);
    std::vector<uint16_t> lam(h.num_edges);
    rc = tsdg_read_tsdg(tsdg_path, off.data(), tgt.data(), lam.data(), nullptr);
    if (rc) return rc;
    return tsdg_gpu_index_create(base, n, d, off.data(), tgt.data(), lam.data(), h.metric, device,
                                 out);
}

int tsdg_gpu_index_create_from_files(const char* tsdg_path, const char* vectors_path, int device,
                                     tsdg_gpu_index** out) {
    return guarded([&] {
        if (!out) fail(TSDG_EINVAL, "index_create_from_files: null out");
        *out = nullptr;
        if (!tsdg_path || !vectors_path) fail(TSDG_EINVAL, "index_create_from_files: null path");
        const std::string gpath(tsdg_path), vpath(vectors_path);
        // TSDG_LOAD_TRACE=1: phase times on stderr (development)
        const bool trace = env_int("TSDG_LOAD_TRACE", 0) != 0;
        auto t_last = std::chrono::steady_clock::now();
        auto mark = [&](const char* what) {
            if (!trace) return;
            const auto t = std::chrono::steady_clock::now();
            std::fprintf(stderr, "[load] %-16s %8.1f ms\n", what,
                         std::chrono::duration<double, std::milli>(t - t_last).count());
            t_last = t;
        };
        std::string err;
        uint32_t vn = 0, vd = 0;
        if (int rc = tsdg_vector_file_shape(vpath, &vn, &vd, err)) fail(rc, err);
        // TSDG header (27 bytes; a shorter file fails in the parse with the
        // reference-worded truncation message)
        tsdg_graph_header h{};
        uint64_t body_off = 0;
        {
            unsigned char hb[64] = {};
            const int fd = open(gpath.c_str(), O_RDONLY);
            if (fd < 0) fail(TSDG_ERUNTIME, gpath + ": cannot open for reading");
            const ssize_t got = pread(fd, hb, sizeof(hb), 0);
            close(fd);
            if (got == 0) fail(TSDG_ERUNTIME, tsdg_truncated_message(gpath, 0));
            if (got < 0) fail(TSDG_ERUNTIME, gpath + ": read failed");
            if (int rc = tsdg_parse_header_bytes(gpath, hb, (size_t)got, &h, &body_off, err)) fail(rc, err);
        }
        mark("shape+header");
        if (h.n != vn)
            fail(TSDG_EINVAL, "index_create_from_files: graph has " + std::to_string(h.n) +
                                  " nodes, base has " + std::to_string(vn));
        if (h.metric > 2) fail(TSDG_EINVAL, "invalid metric");
        DeviceGuard dg(device);
        IndexOwner own;
        tsdg_gpu_index* idx = own.p;
        idx->n = vn;
        idx->d = vd;
        idx->ld = round_up(vd, 4);
        idx->metric = h.metric;
        init_index_runtime(idx, device);
        mark("runtime");
        const size_t rows = std::max<uint32_t>(vn, 1);
        cuda_check(cudaMalloc(&idx->vec, rows * idx->ld * sizeof(float)), "cudaMalloc(vectors)");
        DevBuf<unsigned long long> bad(2, idx->stream);
        cuda_check(cudaMemsetAsync(bad.p, 0xFF, 2 * sizeof(unsigned long long), idx->stream), "memset");
        PinnedPair pin(kStageChunk, idx->stream);
        mark("alloc");
        load_vectors_to_device(idx, vpath, pin, bad.p);
        if (trace) cudaStreamSynchronize(idx->stream);
        mark("vectors");
        load_graph_to_device(idx, gpath, body_off, pin, bad.p + 1);
        mark("graph");
        unsigned long long hbad[2];
        cuda_check(cudaMemcpyAsync(hbad, bad.p, sizeof(hbad), cudaMemcpyDeviceToHost, idx->stream), "D2H");
        cuda_check(cudaStreamSynchronize(idx->stream), "index_create_from_files");
        if (hbad[0] != ~0ull) {
            // the host parse reports the first bad record in the reference's wording
            uint32_t pn = 0, pd = 0;
            if (int rc = tsdg_parse_vector_file(vpath, nullptr, &pn, &pd, err)) fail(rc, err);
            fail(TSDG_ERUNTIME, vpath + ": invalid record " + std::to_string(hbad[0]));
        }
        if (hbad[1] != ~0ull)
            fail(TSDG_EINVAL, "index_create_from_files: edge target out of range at node " +
                                  std::to_string(hbad[1]));
        make_vectors_tmap(idx);
        *out = own.release();
    });
}

int tsdg_gpu_index_destroy(tsdg_gpu_index* idx) {
    return guarded([&] {
        if (idx) free_index(idx);
    });
}

int tsdg_gpu_index_info(const tsdg_gpu_index* idx, uint32_t* n, uint32_t* d, int* metric,
                        uint32_t* max_degree, int* device, uint32_t* row_stride,
                        uint32_t* adj_stride) {
    if (!idx) {
        g_err = "index_info: null index";
        return TSDG_EINVAL;
    }
    if (n) *n = idx->n;
    if (d) *d = idx->d;
    if (metric) *metric = idx->metric;
    if (max_degree) *max_degree = idx->max_degree;
    if (device) *device = idx->device;
    if (row_stride) *row_stride = idx->ld;
    if (adj_stride) *adj_stride = idx->R;
    return TSDG_OK;
}

int tsdg_gpu_deg_cut(tsdg_gpu_index* idx, uint32_t lambda_cut, uint32_t* out) {
    return guarded([&] {
        if (!idx) fail(TSDG_EINVAL, "deg_cut: null index");
        std::lock_guard<std::mutex> lk(idx->mu);
        DeviceGuard dg(idx->device);
        const uint32_t* dc = get_degcut(idx, lambda_cut, idx->stream);
        if (out && idx->n) {
            cuda_check(cudaMemcpyAsync(out, dc, sizeof(uint32_t) * idx->n, cudaMemcpyDeviceToHost,
                                       idx->stream),
                       "cudaMemcpyAsync(deg_cut)");
        }
        cuda_check(cudaStreamSynchronize(idx->stream), "cudaStreamSynchronize");
    });
}

int tsdg_gpu_search_bestfirst_device(tsdg_gpu_index* idx, const float* d_queries, uint32_t nq,
                                     uint64_t query_index_base, const tsdg_bf_params* params,
                                     int mode, uint32_t* d_ids, float* d_dists,
                                     uint32_t* d_counts, tsdg_query_stats* d_stats,
                                     void* stream) {
    return guarded([&] {
        if (!idx) fail(TSDG_EINVAL, "bestfirst_search: null index");
        validate_bf(idx, params);
        if (nq && (!d_queries || !d_ids)) fail(TSDG_EINVAL, "bestfirst_search: null buffer");
        std::lock_guard<std::mutex> lk(idx->mu);
        DeviceGuard dg(idx->device);
        launch_bestfirst(idx, d_queries, nq, query_index_base, params, mode, d_ids, d_dists,
                         d_counts, d_stats, static_cast<cudaStream_t>(stream));
    });
}

int tsdg_gpu_search_bestfirst(tsdg_gpu_index* idx, const float* queries, uint32_t nq,
                              uint64_t query_index_base, const tsdg_bf_params* params,
                              int mode, uint32_t* ids, float* dists, uint32_t* counts,
                              tsdg_query_stats* stats) {
    return guarded([&] {
        if (!idx) fail(TSDG_EINVAL, "bestfirst_search: null index");
        if (nq == 0) return;  // the reference's per-query loop never runs
        validate_bf(idx, params);
        if (!queries || !ids) fail(TSDG_EINVAL, "bestfirst_search: null buffer");
        check_cosine_queries(idx, queries, nq);
        std::lock_guard<std::mutex> lk(idx->mu);
        DeviceGuard dg(idx->device);
        const uint32_t k = params->k;
        // Zero-copy when every buffer is mapped pinned host memory (TSDG_ZERO_COPY=0
        // disables): the kernel reads each query from host memory once (into shared
        // memory) and writes its results straight back over the bus, so the upload
        // and download overlap the whole search instead of bracketing it.
        if (env_int("TSDG_ZERO_COPY", 1)) {
            const float* zq = mapped_alias(queries, (size_t)nq * idx->d * 4);
            uint32_t* zi = mapped_alias(ids, (size_t)nq * k * 4);
            float* zd = mapped_alias(dists, (size_t)nq * k * 4);
            uint32_t* zc = mapped_alias(counts, (size_t)nq * 4);
            tsdg_query_stats* zs = mapped_alias(stats, (size_t)nq * sizeof(tsdg_query_stats));
            if (env_int("TSDG_DEBUG_PATH", 0))
                std::fprintf(stderr, "[tsdg] bestfirst host call: q=%p i=%p d=%p c=%p s=%p -> %s\n",
                             (const void*)zq, (void*)zi, (void*)zd, (void*)zc, (void*)zs,
                             (zq && zi && (zd || !dists) && (zc || !counts) && (zs || !stats))
                                 ? "zero-copy" : "copy pipeline");
            if (zq && zi && (zd || !dists) && (zc || !counts) && (zs || !stats)) {
                launch_bestfirst(idx, zq, nq, query_index_base, params, mode, zi, zd, zc, zs,
                                 idx->stream);
                cuda_check(cudaStreamSynchronize(idx->stream), "bestfirst_search");
                return;
            }
        }
        // grow-only scratch: queries | ids | dists | counts | stats
        const size_t bq = (size_t)nq * idx->d * 4, bi = (size_t)nq * k * 4, bc = (size_t)nq * 4,
                     bs = (size_t)nq * sizeof(tsdg_query_stats);
        auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
        const size_t need = al(bq) + 2 * al(bi) + al(bc) + al(bs);
        if (need > idx->scratch_bytes) {
            cuda_check(cudaStreamSynchronize(idx->stream), "sync");
            cuda_check(cudaStreamSynchronize(idx->stream2), "sync");
            if (idx->scratch) cudaFree(idx->scratch);
            idx->scratch = nullptr;
            idx->scratch_bytes = 0;
            cuda_check(cudaMalloc(&idx->scratch, need), "cudaMalloc(scratch)");
            idx->scratch_bytes = need;
        }
        char* base = static_cast<char*>(idx->scratch);
        float* dq = reinterpret_cast<float*>(base);
        uint32_t* di = reinterpret_cast<uint32_t*>(base + al(bq));
        float* dd = reinterpret_cast<float*>(base + al(bq) + al(bi));
        uint32_t* dc = reinterpret_cast<uint32_t*>(base + al(bq) + 2 * al(bi));
        tsdg_query_stats* ds =
            reinterpret_cast<tsdg_query_stats*>(base + al(bq) + 2 * al(bi) + al(bc));
        // Copy/compute pipeline (2 chunks measured best on C2: 1.27 vs 1.31 ms for 1, 1.32
        // for 4, TSDG_E2E_CHUNKS overrides): the batch is cut into chunks alternating between two
        // streams, so chunk c+1's upload overlaps chunk c's search and chunk c-1's
        // download.  Each chunk keeps its global query index (RNG stream fork(base+q)).
        get_degcut(idx, params->lambda_cut, idx->stream);
        const int env_chunks = env_int("TSDG_E2E_CHUNKS", 0);
        const uint32_t nchunks = env_chunks > 0 ? (uint32_t)env_chunks : (nq >= 4096 ? 2 : 1);
        // chunk boundaries: the first chunk may be smaller (TSDG_E2E_FIRST = percent of
        // the batch) so the first search starts after a shorter upload
        const int first_pct = env_int("TSDG_E2E_FIRST", 25);  // measured: 25% best (1.25 vs 1.28 ms)
        std::vector<uint32_t> bounds(1, 0);
        if (nchunks == 2 && first_pct > 0 && first_pct < 100) {
            bounds.push_back((uint32_t)((uint64_t)nq * first_pct / 100));
        } else {
            const uint32_t csz = (nq + nchunks - 1) / nchunks;
            for (uint32_t c = 1; c < nchunks; ++c) bounds.push_back(std::min(nq, c * csz));
        }
        bounds.push_back(nq);
        for (uint32_t c = 0; c + 1 < bounds.size(); ++c) {
            const uint32_t q0 = bounds[c];
            if (q0 >= nq) break;
            const uint32_t cn = bounds[c + 1] - q0;
            if (cn == 0) continue;
            cudaStream_t st = (c & 1) ? idx->stream2 : idx->stream;
            cuda_check(cudaMemcpyAsync(dq + (size_t)q0 * idx->d, queries + (size_t)q0 * idx->d,
                                       (size_t)cn * idx->d * 4, cudaMemcpyHostToDevice, st),
                       "cudaMemcpyAsync(queries)");
            launch_bestfirst(idx, dq + (size_t)q0 * idx->d, cn, query_index_base + q0, params, mode,
                             di + (size_t)q0 * k, dd + (size_t)q0 * k, dc + q0,
                             stats ? ds + q0 : nullptr, st);
            cuda_check(cudaMemcpyAsync(ids + (size_t)q0 * k, di + (size_t)q0 * k, (size_t)cn * k * 4,
                                       cudaMemcpyDeviceToHost, st),
                       "D2H ids");
            if (dists)
                cuda_check(cudaMemcpyAsync(dists + (size_t)q0 * k, dd + (size_t)q0 * k,
                                           (size_t)cn * k * 4, cudaMemcpyDeviceToHost, st),
                           "D2H dists");
            if (counts)
                cuda_check(cudaMemcpyAsync(counts + q0, dc + q0, (size_t)cn * 4,
                                           cudaMemcpyDeviceToHost, st),
                           "D2H counts");
            if (stats)
                cuda_check(cudaMemcpyAsync(stats + q0, ds + q0, (size_t)cn * sizeof(tsdg_query_stats),
                                           cudaMemcpyDeviceToHost, st),
                           "D2H stats");
        }
        cuda_check(cudaStreamSynchronize(idx->stream), "bestfirst_search");
        cuda_check(cudaStreamSynchronize(idx->stream2), "bestfirst_search");
    });
}

int tsdg_gpu_search_greedy_device(tsdg_gpu_index* idx, const float* d_queries, uint32_t nq,
                                  uint32_t k, const tsdg_greedy_params* params, int mode,
                                  uint32_t* d_ids, float* d_dists, uint32_t* d_counts,
                                  tsdg_query_stats* d_stats, void* stream) {
    return guarded([&] {
        if (!idx) fail(TSDG_EINVAL, "small_batch_search: null index");
        validate_greedy(idx, k, params);
        if (nq && (!d_queries || !d_ids)) fail(TSDG_EINVAL, "small_batch_search: null buffer");
        std::lock_guard<std::mutex> lk(idx->mu);
        DeviceGuard dg(idx->device);
        launch_greedy(idx, d_queries, nq, k, params, mode, d_ids, d_dists, d_counts, d_stats,
                      static_cast<cudaStream_t>(stream));
    });
}

int tsdg_gpu_search_greedy(tsdg_gpu_index* idx, const float* queries, uint32_t nq, uint32_t k,
                           const tsdg_greedy_params* params, int mode, uint32_t* ids,
                           float* dists, uint32_t* counts, tsdg_query_stats* stats) {
    return guarded([&] {
        if (!idx) fail(TSDG_EINVAL, "small_batch_search: null index");
        if (nq == 0) return;  // the reference's per-query loop never runs
        validate_greedy(idx, k, params);
        if (!queries || !ids) fail(TSDG_EINVAL, "small_batch_search: null buffer");
        check_cosine_queries(idx, queries, nq);
        std::lock_guard<std::mutex> lk(idx->mu);
        DeviceGuard dg(idx->device);
        cudaStream_t st = idx->stream;
        // zero-copy with mapped pinned buffers (see tsdg_gpu_search_bestfirst): at
        // small batch this removes two copy round trips from the call's latency
        if (env_int("TSDG_ZERO_COPY", 1)) {
            const float* zq = mapped_alias(queries, (size_t)nq * idx->d * 4);
            uint32_t* zi = mapped_alias(ids, (size_t)nq * k * 4);
            float* zd = mapped_alias(dists, (size_t)nq * k * 4);
            uint32_t* zc = mapped_alias(counts, (size_t)nq * 4);
            tsdg_query_stats* zs = mapped_alias(stats, (size_t)nq * sizeof(tsdg_query_stats));
            if (zq && zi && (zd || !dists) && (zc || !counts) && (zs || !stats)) {
                launch_greedy(idx, zq, nq, k, params, mode, zi, zd, zc, zs, st);
                cuda_check(cudaStreamSynchronize(st), "small_batch_search");
                return;
            }
        }
        float* dq = dev_alloc<float>((size_t)nq * idx->d, st);
        uint32_t* di = dev_alloc<uint32_t>((size_t)nq * k, st);
        float* dd = dev_alloc<float>((size_t)nq * k, st);
        uint32_t* dc = dev_alloc<uint32_t>(nq, st);
        tsdg_query_stats* ds = stats ? dev_alloc<tsdg_query_stats>(nq, st) : nullptr;
        cuda_check(cudaMemcpyAsync(dq, queries, (size_t)nq * idx->d * 4, cudaMemcpyHostToDevice, st),
                   "cudaMemcpyAsync(queries)");
        launch_greedy(idx, dq, nq, k, params, mode, di, dd, dc, ds, st);
        cuda_check(cudaMemcpyAsync(ids, di, (size_t)nq * k * 4, cudaMemcpyDeviceToHost, st), "D2H ids");
        if (dists)
            cuda_check(cudaMemcpyAsync(dists, dd, (size_t)nq * k * 4, cudaMemcpyDeviceToHost, st),
                       "D2H dists");
        if (counts)
            cuda_check(cudaMemcpyAsync(counts, dc, (size_t)nq * 4, cudaMemcpyDeviceToHost, st),
                       "D2H counts");
        if (stats)
            cuda_check(cudaMemcpyAsync(stats, ds, (size_t)nq * sizeof(tsdg_query_stats),
                                       cudaMemcpyDeviceToHost, st),
                       "D2H stats");
        cudaFreeAsync(dq, st);
        cudaFreeAsync(di, st);
        cudaFreeAsync(dd, st);
        cudaFreeAsync(dc, st);
        if (ds) cudaFreeAsync(ds, st);
        cuda_check(cudaStreamSynchronize(st), "small_batch_search");
    });
}


int tsdg_gpu_greedy_once(tsdg_gpu_index* idx, const float* queries, uint32_t nq,
                         const uint64_t* rng_states, uint32_t hop_limit, uint32_t lambda_cut,
                         uint32_t* ids32, float* dists32, tsdg_query_stats* stats) {
    return guarded([&] {
        if (!idx) fail(TSDG_EINVAL, "greedy_search_once: null index");
        if (lambda_cut < 1) fail(TSDG_EINVAL, "greedy_search_once: lambda_cut must be >= 1");
        if (hop_limit < 1) fail(TSDG_EINVAL, "greedy_search_once: hop limit must be >= 1");
        if (idx->n == 0) fail(TSDG_EINVAL, "select_start: empty graph");
        if (nq == 0) return;
        if (!queries || !rng_states || !ids32) fail(TSDG_EINVAL, "greedy_search_once: null buffer");
        std::lock_guard<std::mutex> lk(idx->mu);
        DeviceGuard dg(idx->device);
        cudaStream_t st = idx->stream;
        float* dq = dev_alloc<float>((size_t)nq * idx->d, st);
        uint64_t* dst = dev_alloc<uint64_t>(nq, st);
        cuda_check(cudaMemcpyAsync(dq, queries, (size_t)nq * idx->d * 4, cudaMemcpyHostToDevice, st), "H2D");
        cuda_check(cudaMemcpyAsync(dst, rng_states, (size_t)nq * 8, cudaMemcpyHostToDevice, st), "H2D");
        WalkBuffers wb = alloc_walks(nq, st);
        launch_walks(idx, dq, nq, 1, hop_limit, lambda_cut, 0, dst, wb, st);
        cuda_check(cudaMemcpyAsync(ids32, wb.ids, (size_t)nq * 32 * 4, cudaMemcpyDeviceToHost, st), "D2H");
        if (dists32)
            cuda_check(cudaMemcpyAsync(dists32, wb.dists, (size_t)nq * 32 * 4, cudaMemcpyDeviceToHost, st),
                       "D2H");
        std::vector<uint32_t> h(nq), e(nq);
        cuda_check(cudaMemcpyAsync(h.data(), wb.hops, (size_t)nq * 4, cudaMemcpyDeviceToHost, st), "D2H");
        cuda_check(cudaMemcpyAsync(e.data(), wb.evals, (size_t)nq * 4, cudaMemcpyDeviceToHost, st), "D2H");
        free_walks(wb, st);
        cudaFreeAsync(dq, st);
        cudaFreeAsync(dst, st);
        cuda_check(cudaStreamSynchronize(st), "greedy_search_once");
        if (stats) {
            for (uint32_t q = 0; q < nq; ++q) {
                stats[q].hops = h[q];
                stats[q].distance_evals = e[q];
                stats[q].queue_evictions = 0;
                stats[q].edges_examined = e[q] - 32;
            }
        }
    });
}

int tsdg_gpu_merge_shards_device(const uint32_t* d_ids, const float* d_dists,
                                 const uint32_t* d_counts, const uint64_t* shard_base,
                                 uint32_t shards, uint32_t nq, uint32_t k, uint32_t* d_out_ids,
                                 float* d_out_dists, uint32_t* d_out_counts, void* stream) {
    return guarded([&] {
        if (shards < 1 || k < 1) fail(TSDG_EINVAL, "merge_shards: need shards >= 1 and k >= 1");
        if (nq == 0) return;
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        uint32_t npow2 = 32;
        while (npow2 < shards * k) npow2 <<= 1;
        const size_t smem = (size_t)npow2 * 8;
        if (smem > 200 * 1024) fail(TSDG_EINVAL, "merge_shards: shards * k too large");
        uint64_t* dbase = dev_alloc<uint64_t>(shards, st);
        cuda_check(cudaMemcpyAsync(dbase, shard_base, shards * 8, cudaMemcpyHostToDevice, st), "H2D");
        cuda_check(cudaFuncSetAttribute(merge_shards_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                   "cudaFuncSetAttribute(merge_shards)");
        merge_shards_kernel<<<nq, kMergeThreads, smem, st>>>(d_ids, d_dists, d_counts, dbase,
                                                             shards, nq, k, npow2, d_out_ids,
                                                             d_out_dists, d_out_counts);
        g_launches++;
        cuda_check(cudaGetLastError(), "merge_shards_kernel launch");
        cudaFreeAsync(dbase, st);
    });
}


// ---- exact top-k: ground truth / brute-force k-NN graph -------------------------
int tsdg_gpu_exact_topk_device(const float* d_base, uint32_t n, uint32_t ld_base,
                               const float* d_queries, uint32_t nq, uint32_t ld_queries,
                               uint32_t d, uint32_t k, int metric, int exclude_self,
                               uint64_t self_base, uint32_t* d_ids, float* d_dists, void* stream) {
    return guarded([&] {
        if ((nq && (!d_queries || !d_ids || !d_dists)) || (n && !d_base))
            fail(TSDG_EINVAL, "exact_topk: null pointer");
        launch_exact_topk(d_base, n, ld_base, d_queries, nq, ld_queries, d, k, metric, exclude_self,
                          self_base, d_ids, d_dists, (cudaStream_t)stream);
    });
}

int tsdg_gpu_ground_truth(const float* base, uint32_t n, const float* queries, uint32_t nq,
                          uint32_t d, uint32_t k_gt, int metric, int device, uint32_t* ids,
                          float* dists) {
    return guarded([&] {
        // bench.cpp:38-41
        if (k_gt < 1 || k_gt > n) fail(TSDG_EINVAL, "ground_truth: need 1 <= K_gt <= n");
        if (d < 1) fail(TSDG_EINVAL, "ground_truth: dim mismatch");
        if (!base || (nq && (!queries || !ids))) fail(TSDG_EINVAL, "ground_truth: null pointer");
        DeviceGuard dg(device);
        cudaStream_t st;
        cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
        const uint32_t ld = round_up(d, 4);
        float* db = upload_rows(base, n, d, ld, st);
        float* dq = upload_rows(queries, nq, d, ld, st);
        try {
            if (nq) scan_to_host(db, n, ld, dq, nq, d, k_gt, metric, 0, ids, dists, st);
        } catch (...) {
            cudaFreeAsync(db, st);
            cudaFreeAsync(dq, st);
            cudaStreamDestroy(st);
            throw;
        }
        cudaFreeAsync(db, st);
        cudaFreeAsync(dq, st);
        cuda_check(cudaStreamSynchronize(st), "ground_truth");
        cudaStreamDestroy(st);
    });
}

int tsdg_gpu_index_ground_truth(tsdg_gpu_index* idx, const float* queries, uint32_t nq,
                                uint32_t k_gt, uint32_t* ids, float* dists) {
    return guarded([&] {
        if (!idx) fail(TSDG_EINVAL, "ground_truth: null index");
        if (k_gt < 1 || k_gt > idx->n) fail(TSDG_EINVAL, "ground_truth: need 1 <= K_gt <= n");
        if (nq && (!queries || !ids)) fail(TSDG_EINVAL, "ground_truth: null pointer");
        std::lock_guard<std::mutex> lk(idx->mu);
        DeviceGuard dg(idx->device);
        cudaStream_t st = idx->stream;
        float* dq = upload_rows(queries, nq, idx->d, idx->ld, st);
        if (nq) scan_to_host(idx->vec, idx->n, idx->ld, dq, nq, idx->d, k_gt, idx->metric, 0, ids,
                             dists, st);
        cudaFreeAsync(dq, st);
        cuda_check(cudaStreamSynchronize(st), "ground_truth");
    });
}

int tsdg_gpu_brute_force_knn(const float* base, uint32_t n, uint32_t d, uint32_t k, int metric,
                             int device, uint32_t* ids, float* dists, uint32_t* k_eff) {
    return guarded([&] {
        // knn_graph.cpp:17-26 (clamp_k)
        if (n < 2) fail(TSDG_EINVAL, "brute_force_knn: need at least 2 vectors");
        if (k < 1) fail(TSDG_EINVAL, "brute_force_knn: k must be >= 1");
        if (k > n - 1) {
            std::fprintf(stderr, "brute_force_knn: k=%u clamped to n-1=%u\n", k, n - 1);
            k = n - 1;
        }
        if (k_eff) *k_eff = k;
        if (d < 1) fail(TSDG_EINVAL, "brute_force_knn: d must be >= 1");
        if (!base || !ids) fail(TSDG_EINVAL, "brute_force_knn: null pointer");
        DeviceGuard dg(device);
        cudaStream_t st;
        cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
        const uint32_t ld = round_up(d, 4);
        float* db = upload_rows(base, n, d, ld, st);
        try {
            scan_to_host(db, n, ld, db, n, d, k, metric, 1, ids, dists, st);
        } catch (...) {
            cudaFreeAsync(db, st);
            cudaStreamDestroy(st);
            throw;
        }
        cudaFreeAsync(db, st);
        cuda_check(cudaStreamSynchronize(st), "brute_force_knn");
        cudaStreamDestroy(st);
    });
}

int tsdg_gpu_nn_descent(const float* base, uint32_t n, uint32_t d, uint32_t k, int metric,
                        uint32_t iterations, double sample_rate, uint64_t seed, int device,
                        uint32_t* ids, float* dists, uint32_t* k_eff, uint64_t* stats4) {
    return guarded([&] {
        if (metric < 0 || metric > 2) fail(TSDG_EINVAL, "invalid metric");
        // knn_graph.cpp:144-146, then clamp_k (:17-26)
        if (!(sample_rate > 0.0 && sample_rate <= 1.0))
            fail(TSDG_EINVAL, "nn_descent: sample_rate must be in (0, 1]");
        if (n < 2) fail(TSDG_EINVAL, "nn_descent: need at least 2 vectors");
        if (k < 1) fail(TSDG_EINVAL, "nn_descent: k must be >= 1");
        if (k > n - 1) {
            std::fprintf(stderr, "nn_descent: k=%u clamped to n-1=%u\n", k, n - 1);
            k = n - 1;
        }
        if (k_eff) *k_eff = k;
        if (k > kNdMaxK) fail(TSDG_EINVAL, "nn_descent: GPU path supports k <= 128");
        if (n > 0x7FFFFFFFu) fail(TSDG_EINVAL, "nn_descent: GPU path supports n < 2^31");
        if (d < 1) fail(TSDG_EINVAL, "nn_descent: d must be >= 1");
        if (!base || !ids || !dists) fail(TSDG_EINVAL, "nn_descent: null pointer");
        // knn_graph.cpp:170-171: std::round(sample_rate * k_eff), at least 1
        const uint32_t ms = (uint32_t)std::max(1.0, std::round(sample_rate * (double)k));
        DeviceGuard dg(device);
        cudaStream_t st;
        cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
        const uint32_t ld = round_up(d, 4);
        float* db = nullptr;
        uint32_t* di = nullptr;
        float* dd = nullptr;
        auto release = [&] {
            cudaFreeAsync(db, st);
            cudaFreeAsync(di, st);
            cudaFreeAsync(dd, st);
            cudaStreamSynchronize(st);
            cudaStreamDestroy(st);
        };
        try {
            db = upload_rows(base, n, d, ld, st);
            di = dev_alloc<uint32_t>((size_t)n * k, st);
            dd = dev_alloc<float>((size_t)n * k, st);
            NnDescentStats ns{};
            nn_descent_device(db, n, d, ld, k, metric, iterations, ms, seed, di, dd, st, &ns);
            g_launches += ns.launches;
            cuda_check(cudaMemcpyAsync(ids, di, (size_t)n * k * 4, cudaMemcpyDeviceToHost, st), "D2H ids");
            cuda_check(cudaMemcpyAsync(dists, dd, (size_t)n * k * 4, cudaMemcpyDeviceToHost, st), "D2H dists");
            cuda_check(cudaStreamSynchronize(st), "nn_descent");
            if (stats4) {
                stats4[0] = ns.offers;
                stats4[1] = ns.chunks;
                stats4[2] = ns.reruns;
                stats4[3] = ns.launches;
            }
        } catch (...) {
            release();
            throw;
        }
        release();
    });
}

// ---- GPU two-stage diversification --------------------------------------------------
int tsdg_gpu_build(const float* base, uint32_t n, uint32_t d, const uint32_t* knn_ids,
                   const float* knn_dists, uint32_t k, float alpha, uint16_t lambda0,
                   uint32_t max_degree, int metric, int device, tsdg_gpu_graph** out,
                   uint64_t* stats4) {
    return guarded([&] {
        if (!out) fail(TSDG_EINVAL, "build: null out");
        *out = nullptr;
        if (!(alpha >= 1.0f)) fail(TSDG_EINVAL, "build: alpha must be >= 1");
        if (metric < 0 || metric > 2) fail(TSDG_EINVAL, "invalid metric");
        if (d < 1) fail(TSDG_EINVAL, "build: d must be >= 1");
        if (k < 1 || k > kDivMaxK) fail(TSDG_EINVAL, "build: GPU path supports 1 <= knn k <= 128");
        if (n > 0 && (!base || !knn_ids || !knn_dists)) fail(TSDG_EINVAL, "build: null input");
        auto g = std::make_unique<tsdg_gpu_graph>();
        g->n = n;
        g->k = k;
        g->metric = metric;
        g->alpha = alpha;
        g->lambda0 = lambda0;
        if (n == 0) {
            g->offsets.assign(1, 0);
            if (stats4) stats4[0] = stats4[1] = stats4[2] = stats4[3] = 0;
        } else {
            DeviceGuard dg(device);
            cudaStream_t st;
            cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
            try {
                gpu_build(base, n, d, knn_ids, knn_dists, k, alpha, lambda0, max_degree, metric, *g,
                          stats4, st);
            } catch (...) {
                cudaStreamSynchronize(st);
                cudaStreamDestroy(st);
                throw;
            }
            cudaStreamDestroy(st);
        }
        *out = g.release();
    });
}

int tsdg_gpu_graph_info(const tsdg_gpu_graph* g, uint64_t* n, uint64_t* num_edges,
                        uint32_t* max_degree) {
    return guarded([&] {
        if (!g) fail(TSDG_EINVAL, "graph_info: null graph");
        if (n) *n = g->n;
        if (num_edges) *num_edges = g->targets.size();
        if (max_degree) {
            uint32_t m = 0;
            for (uint32_t u = 0; u < g->n; ++u)
                m = std::max<uint32_t>(m, (uint32_t)(g->offsets[u + 1] - g->offsets[u]));
            *max_degree = m;
        }
    });
}

int tsdg_gpu_graph_copy(const tsdg_gpu_graph* g, uint64_t* offsets, uint32_t* targets,
                        uint16_t* lambdas, float* dists) {
    return guarded([&] {
        if (!g) fail(TSDG_EINVAL, "graph_copy: null graph");
        if (offsets) std::memcpy(offsets, g->offsets.data(), g->offsets.size() * 8);
        if (targets) std::memcpy(targets, g->targets.data(), g->targets.size() * 4);
        if (lambdas) std::memcpy(lambdas, g->lambdas.data(), g->lambdas.size() * 2);
        if (dists) std::memcpy(dists, g->dists.data(), g->dists.size() * 4);
    });
}

int tsdg_gpu_graph_save(const tsdg_gpu_graph* g, const char* path) {
    return guarded([&] {
        if (!g || !path) fail(TSDG_EINVAL, "graph_save: null argument");
        write_tsdg_file(*g, path);
    });
}

int tsdg_gpu_graph_destroy(tsdg_gpu_graph* g) {
    delete g;
    return TSDG_OK;
}


// ---- replicated multi-device index (one process, several GPUs) ---------------------

int tsdg_gpu_multi_create(const float* base, uint32_t n, uint32_t d, const uint64_t* offsets,
                          const uint32_t* targets, const uint16_t* lambdas, int metric,
                          const int* devices, int ndev, tsdg_gpu_multi** out) {
    return guarded([&] {
        if (!out) fail(TSDG_EINVAL, "multi_create: null out");
        *out = nullptr;
        if (ndev < 1 || !devices) fail(TSDG_EINVAL, "multi_create: need at least one device");
        auto m = std::make_unique<tsdg_gpu_multi>();
        m->parts.assign((size_t)ndev, nullptr);
        try {
            run_per_device((size_t)ndev, [&](size_t i) {
                return tsdg_gpu_index_create(base, n, d, offsets, targets, lambdas, metric,
                                             devices[i], &m->parts[i]);
            });
        } catch (...) {
            for (auto* p : m->parts)
                if (p) tsdg_gpu_index_destroy(p);
            throw;
        }
        *out = m.release();
    });
}

int tsdg_gpu_multi_destroy(tsdg_gpu_multi* m) {
    if (!m) return TSDG_OK;
    int rc = TSDG_OK;
    for (auto* p : m->parts) {
        const int r = tsdg_gpu_index_destroy(p);
        if (rc == TSDG_OK) rc = r;
    }
    delete m;
    return rc;
}

int tsdg_gpu_multi_search_bestfirst(tsdg_gpu_multi* m, const float* queries, uint32_t nq,
                                    uint64_t query_index_base, const tsdg_bf_params* params,
                                    int mode, uint32_t* ids, float* dists, uint32_t* counts,
                                    tsdg_query_stats* stats) {
    return guarded([&] {
        if (!m) fail(TSDG_EINVAL, "bestfirst_search: null index");
        if (nq == 0) return;
        if (!params) fail(TSDG_EINVAL, "bestfirst_search: null params");
        if (!queries || !ids) fail(TSDG_EINVAL, "bestfirst_search: null buffer");
        const uint32_t d = m->parts[0]->d, k = params->k;
        run_per_device(m->parts.size(), [&](size_t i) {
            uint32_t b, e;
            slice_of(nq, m->parts.size(), i, b, e);
            if (b == e) return (int)TSDG_OK;
            // query q keeps its stream fork(query_index_base + q): identical results
            // for any device count
            return tsdg_gpu_search_bestfirst(m->parts[i], queries + (size_t)b * d, e - b,
                                             query_index_base + b, params, mode,
                                             ids + (size_t)b * k, dists ? dists + (size_t)b * k : nullptr,
                                             counts ? counts + b : nullptr, stats ? stats + b : nullptr);
        });
    });
}

int tsdg_gpu_multi_search_greedy(tsdg_gpu_multi* m, const float* queries, uint32_t nq, uint32_t k,
                                 const tsdg_greedy_params* params, int mode, uint32_t* ids,
                                 float* dists, uint32_t* counts, tsdg_query_stats* stats) {
    return guarded([&] {
        if (!m) fail(TSDG_EINVAL, "small_batch_search: null index");
        if (nq == 0) return;
        if (!queries || !ids) fail(TSDG_EINVAL, "small_batch_search: null buffer");
        const uint32_t d = m->parts[0]->d;
        run_per_device(m->parts.size(), [&](size_t i) {
            uint32_t b, e;
            slice_of(nq, m->parts.size(), i, b, e);
            if (b == e) return (int)TSDG_OK;
            return tsdg_gpu_search_greedy(m->parts[i], queries + (size_t)b * d, e - b, k, params, mode,
                                          ids + (size_t)b * k, dists ? dists + (size_t)b * k : nullptr,
                                          counts ? counts + b : nullptr, stats ? stats + b : nullptr);
        });
    });
}


// ---- sharded base in one process (SURVEY.md §8(e), C5 layout) ----------------------
int tsdg_gpu_sharded_create_from_files(const char* const* tsdg_paths, const float* const* bases,
                                       const uint32_t* shard_n, const uint64_t* shard_offset,
                                       uint32_t nshards, uint32_t d, const int* devices,
                                       tsdg_gpu_sharded** out) {
    return guarded([&] {
        if (!out) fail(TSDG_EINVAL, "sharded_create: null out");
        *out = nullptr;
        if (nshards < 1 || !tsdg_paths || !bases || !shard_n || !shard_offset || !devices)
            fail(TSDG_EINVAL, "sharded_create: need at least one shard and its arrays");
        auto sh = std::make_unique<tsdg_gpu_sharded>();
        sh->d = d;
        sh->offsets.assign(shard_offset, shard_offset + nshards);
        sh->shards.assign(nshards, nullptr);
        try {
            run_per_device(nshards, [&](size_t i) {
                return tsdg_gpu_index_create_from_file(tsdg_paths[i], bases[i], shard_n[i], d,
                                                       devices[i], &sh->shards[i]);
            });
            // the per-shard top-k travel to the first shard's device: direct peer
            // access over NVLink where the pair supports it (else the copy is staged)
            const int m = devices[0];
            for (uint32_t i = 1; i < nshards; ++i) {
                const int dv = devices[i];
                if (dv == m) continue;
                int can = 0;
                cuda_check(cudaDeviceCanAccessPeer(&can, m, dv), "cudaDeviceCanAccessPeer");
                if (!can) continue;
                DeviceGuard dg(m);
                const cudaError_t e = cudaDeviceEnablePeerAccess(dv, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else cuda_check(e, "cudaDeviceEnablePeerAccess");
            }
            sh->sq.assign(nshards, nullptr);
            sh->sid.assign(nshards, nullptr);
            sh->scnt.assign(nshards, nullptr);
            sh->sdist.assign(nshards, nullptr);
            sh->done.assign(nshards, nullptr);
            for (uint32_t i = 0; i < nshards; ++i) {
                DeviceGuard dg(devices[i]);
                cuda_check(cudaEventCreateWithFlags(&sh->done[i], cudaEventDisableTiming), "event");
            }
        } catch (...) {
            sharded_free(sh.get());
            throw;
        }
        *out = sh.release();
    });
}

int tsdg_gpu_sharded_destroy(tsdg_gpu_sharded* sh) {
    if (!sh) return TSDG_OK;
    return guarded([&] {
        sharded_free(sh);
        delete sh;
    });
}

int tsdg_gpu_sharded_search_bestfirst(tsdg_gpu_sharded* sh, const float* queries, uint32_t nq,
                                      uint64_t query_index_base, const tsdg_bf_params* params,
                                      int mode, uint32_t* ids, float* dists, uint32_t* counts) {
    return guarded([&] {
        if (!sh) fail(TSDG_EINVAL, "bestfirst_search: null index");
        if (nq == 0) return;
        if (!params) fail(TSDG_EINVAL, "bestfirst_search: null params");
        if (!queries || !ids) fail(TSDG_EINVAL, "bestfirst_search: null buffer");
        const uint32_t S = (uint32_t)sh->shards.size(), k = params->k, d = sh->d;
        for (uint32_t i = 0; i < S; ++i) validate_bf(sh->shards[i], params);
        // every shard searches every query on its own device; the per-shard top-k
        // (local ids) are copied peer-to-peer (NVLink) into one [shard][query][k]
        // block on the first shard's device and merged by (dist, global id) there.
        // The workspace persists across calls; a failed shard leaves nothing behind.
        std::lock_guard<std::mutex> slk(sh->mu);
        sharded_reserve(sh, nq, k);
        const size_t blk = (size_t)nq * k;
        try {
            run_per_device(S, [&](size_t i) {
                return guarded([&] {
                    tsdg_gpu_index* idx = sh->shards[i];
                    std::lock_guard<std::mutex> lk(idx->mu);
                    DeviceGuard dg(idx->device);
                    cudaStream_t st = idx->stream;
                    float* dq = sh->sq[i];
                    cuda_check(cudaMemcpyAsync(dq, queries, (size_t)nq * d * 4, cudaMemcpyHostToDevice, st),
                               "H2D queries");  // rows of d floats (the kernels' query stride)
                    launch_bestfirst(idx, dq, nq, query_index_base, params, mode, sh->sid[i], sh->sdist[i],
                                     sh->scnt[i], nullptr, st);
                    cuda_check(cudaEventRecord(sh->done[i], st), "event record");
                });
            });
            tsdg_gpu_index* m = sh->shards[0];
            std::lock_guard<std::mutex> lk(m->mu);
            DeviceGuard dg(m->device);
            cudaStream_t st = m->stream;
            for (uint32_t i = 0; i < S; ++i) {
                const int dev = sh->shards[i]->device;
                cuda_check(cudaStreamWaitEvent(st, sh->done[i], 0), "wait shard");
                cuda_check(cudaMemcpyPeerAsync(sh->gid + i * blk, m->device, sh->sid[i], dev, blk * 4, st),
                           "peer ids");
                cuda_check(cudaMemcpyPeerAsync(sh->gdist + i * blk, m->device, sh->sdist[i], dev, blk * 4, st),
                           "peer dists");
                cuda_check(cudaMemcpyPeerAsync(sh->gcnt + (size_t)i * nq, m->device, sh->scnt[i], dev,
                                               (size_t)nq * 4, st),
                           "peer counts");
            }
            const int rc = tsdg_gpu_merge_shards_device(sh->gid, sh->gdist, sh->gcnt, sh->offsets.data(), S,
                                                        nq, k, sh->oid, sh->odist, sh->ocnt, st);
            if (rc != TSDG_OK) fail(rc, tsdg_gpu_last_error());
            cuda_check(cudaMemcpyAsync(ids, sh->oid, blk * 4, cudaMemcpyDeviceToHost, st), "D2H ids");
            if (dists)
                cuda_check(cudaMemcpyAsync(dists, sh->odist, blk * 4, cudaMemcpyDeviceToHost, st), "D2H dists");
            if (counts)
                cuda_check(cudaMemcpyAsync(counts, sh->ocnt, (size_t)nq * 4, cudaMemcpyDeviceToHost, st),
                           "D2H counts");
            cuda_check(cudaStreamSynchronize(st), "sharded search");
        } catch (...) {
            for (auto* idx : sh->shards) {  // no shard work left in flight on the workspace
                DeviceGuard dg(idx->device);
                cudaStreamSynchronize(idx->stream);
            }
            throw;
        }
    });
}

}  // extern "C"

#ifdef TSDG_PHASES
// Development build only: per-phase cycle totals summed over warps (see common.cuh).
// Per-CTA globaltimer trace of the small-batch kernels (out: 256 x 32 u64), reset after.
extern "C" int tsdg_gpu_trace_read(unsigned long long* out) {
    if (cudaMemcpyFromSymbol(out, tsdg_dev::g_trace, 256 * 32 * 8) != cudaSuccess) return 2;
    static unsigned long long zero[256][32];
    cudaMemcpyToSymbol(tsdg_dev::g_trace, zero, sizeof(zero));
    return 0;
}
extern "C" int tsdg_gpu_hop_trace_read(unsigned long long* out) {  // 4 x 32 x 8 u64, reset after
    if (cudaMemcpyFromSymbol(out, tsdg_dev::g_hop, 4 * 32 * 8 * 8) != cudaSuccess) return 2;
    static unsigned long long zero[4][32][8];
    cudaMemcpyToSymbol(tsdg_dev::g_hop, zero, sizeof(zero));
    return 0;
}
extern "C" int tsdg_gpu_phase_read(unsigned long long* out8, int reset) {
    static unsigned long long host[1 << 16][8];
    if (cudaMemcpyFromSymbol(host, tsdg_dev::g_phase, sizeof(host)) != cudaSuccess) return 2;
    for (int i = 0; i < 8; ++i) out8[i] = 0;
    for (int w = 0; w < (1 << 16); ++w)
        for (int i = 0; i < 8; ++i) out8[i] += host[w][i];
    if (reset) {
        std::memset(host, 0, sizeof(host));
        cudaMemcpyToSymbol(tsdg_dev::g_phase, host, sizeof(host));
    }
    return 0;
}
#endif
