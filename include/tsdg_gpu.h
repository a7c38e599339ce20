/*
 * tsdg_gpu.h — C-ABI of the B200 (sm_100a) TSDG search library
 * (paper_2204_00824_b200/_lib/libtsdg_gpu.so).
 *
 * Drop-in boundary for the reference's search hot path.  The reference is a
 * C++20 library (/root/reference/proj); its search entry points run an OpenMP
 * loop over queries, and this ABI sits exactly where that loop sits
 * (SURVEY.md §3).  Each entry point below names the reference interface it
 * replaces.  Plain pointers and sizes only; no STL, no torch types.
 *
 * Error convention: every call returns TSDG_OK (0) or a status code; the
 * message is in tsdg_gpu_last_error() (thread-local).  The C++ wrapper
 * (include/tsdg/gpu_search.hpp) rethrows TSDG_EINVAL as std::invalid_argument
 * and TSDG_ERUNTIME as std::runtime_error, the exception types the reference
 * throws (bestfirst_search.cpp:116-120,134; greedy_search.cpp:30-35,78-82,112;
 * diversify.cpp:254,276,281-282).
 *
 * Determinism: TSDG_MODE_DETERMINISTIC reproduces the reference bit for bit
 * (ids, fp32 distances, hops / distance_evals / queue_evictions per query).
 * TSDG_MODE_FAST is allowed to differ in fp32 rounding of distances only
 * (fused multiply-add, tree reduction); its recall must stay within 0.5 points
 * of the reference at equal parameters.
 *
 * Environment (read at each call; defaults are the measured best on C2, and none of
 * them changes deterministic-mode results):
 *   TSDG_ZERO_COPY=0        host-pointer calls use the copy pipeline even when every
 *                           buffer is mapped pinned memory
 *   TSDG_E2E_CHUNKS, TSDG_E2E_FIRST   copy-pipeline chunking (2 chunks, first 25%)
 *   TSDG_FAST_KERNEL=staged|register  fast best-first kernel choice (default: the
 *                           register-direct kernel for rows <= 128 floats, k <= 31)
 *   TSDG_FAST_PAIR=0|1, TSDG_FAST_GROUP=1|2|4   force the single / group (two or
 *                           four warps per query) fast kernel (default: pairs below
 *                           one query per CTA slot)
 *   TSDG_FAST_VARIANT, TSDG_FAST_PREFETCH   fast-kernel tuning variants (bf_fast.cu)
 *   TSDG_STAGE=g4|tma|ldgsts, TSDG_SLOTS, TSDG_BF_WARPS, TSDG_PREFETCH, TSDG_BATCH_MIN
 *                           staged best-first kernel: staging path (default: TMA
 *                           gather4 tensor copies in deterministic mode for rows of
 *                           <= 128 floats, else one bulk copy per row) / slots / warps
 *   TSDG_GREEDY=cta|warp, TSDG_GREEDY_CTA_MAX_WALKS   greedy kernel routing
 *   TSDG_GC_STAGE=g4|tma|ldgsts, TSDG_GC_MERGE_WARP, TSDG_GC_SLICE, TSDG_GC_ADJ_PREFETCH,
 *   TSDG_GR_WARPS, TSDG_GR_STAGE=g4|tma   greedy kernels' staging / warp roles
 *   TSDG_SCAN_SPLITS, TSDG_SCAN_TMA=0   exact-scan base splits / cp.async row tiles
 *   TSDG_DEBUG_PATH=1, TSDG_LOAD_TRACE=1   diagnostics on stderr
 */
#ifndef TSDG_GPU_H
#define TSDG_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSDG_GPU_ABI_VERSION 1

enum {
    TSDG_OK = 0,
    TSDG_EINVAL = 1,   /* std::invalid_argument in the reference */
    TSDG_ERUNTIME = 2, /* std::runtime_error / CUDA failure */
    TSDG_ENCCL = 3
};

enum { TSDG_MODE_DETERMINISTIC = 0, TSDG_MODE_FAST = 1 };

enum { TSDG_METRIC_L2 = 0, TSDG_METRIC_COSINE = 1, TSDG_METRIC_IP = 2 }; /* vectors.hpp:15 */

/* tsdg::BestFirstParams (bestfirst_search.hpp:15-25); same fields, same defaults
 * (k=10, hop_limit=1024, delta=0, m_segments=8, lambda_cut=5, seed=0, unbounded=0). */
typedef struct {
    uint32_t k;
    uint32_t hop_limit;
    float delta;
    uint32_t m_segments;
    uint32_t lambda_cut;
    uint64_t seed;
    int32_t unbounded;
} tsdg_bf_params;

/* tsdg::GreedyParams (greedy_search.hpp:14-19); defaults t0=16, hop_limit=16,
 * lambda_cut=10, seed=0. */
typedef struct {
    uint32_t t0;
    uint32_t hop_limit;
    uint32_t lambda_cut;
    uint64_t seed;
} tsdg_greedy_params;

/* Per-query counters; tsdg::SearchStats (greedy_search.hpp:21-32) fields plus
 * the EdgeTrace sizes (bestfirst_search.hpp:29-32). */
typedef struct {
    uint32_t hops;
    uint32_t distance_evals;
    uint32_t queue_evictions;
    uint32_t edges_examined; /* EdgeTrace::examined.size() (greedy: streamed edges) */
} tsdg_query_stats;

/* TSDG file header (diversify.cpp:252-272). */
typedef struct {
    uint64_t n;
    uint64_t num_edges;
    uint32_t k;
    float alpha;
    uint16_t lambda0;
    uint8_t metric;
    uint32_t max_degree;
} tsdg_graph_header;

typedef struct tsdg_gpu_index tsdg_gpu_index;

const char* tsdg_gpu_last_error(void);
int tsdg_gpu_abi_version(void);

/* ---- bulk TSDG loader (replaces load_tsdg, diversify.cpp:274-306) ----------
 * Reads the reference's byte format unchanged: one sequential pass, no per-field
 * stream calls.  tsdg_read_tsdg fills caller arrays sized from the header
 * (offsets n+1, the rest num_edges); any pointer may be NULL to skip. */
int tsdg_read_tsdg_header(const char* path, tsdg_graph_header* out);
int tsdg_read_tsdg(const char* path, uint64_t* offsets, uint32_t* targets,
                   uint16_t* lambdas, float* dists);

/* ---- vector files (replaces load_vectors / load_fvecs / load_bvecs, io.hpp:11-19,
 * io.cpp:58-121) ------------------------------------------------------------
 * fvecs (int32 d, d x f32) or, for a ".bvecs" path, bvecs (int32 d, d x u8,
 * widened to f32).  tsdg_read_vectors_shape reads (n, d) from the first record and
 * the file size; tsdg_read_vectors fills a caller n x d buffer.  Errors carry the
 * reference's messages (truncation, implausible / invalid / inconsistent
 * dimension, non-finite value, empty dataset) as TSDG_ERUNTIME. */
int tsdg_read_vectors_shape(const char* path, uint32_t* n, uint32_t* d);
int tsdg_read_vectors(const char* path, float* out, uint32_t n, uint32_t d);

/* ---- device index -----------------------------------------------------------
 * Uploads the fp32 vector store (rows padded to 16 B) and a fixed-degree padded
 * adjacency (row stride = max degree rounded up to 4, CSR order kept exactly,
 * pads 0xFFFFFFFF) plus the per-edge lambda for deg_cut.  Replaces the
 * reference's in-RAM TsdgGraph + VectorSet (diversify.hpp:56-76, vectors.hpp:23-34). */
int tsdg_gpu_index_create(const float* base, uint32_t n, uint32_t d, const uint64_t* offsets,
                          const uint32_t* targets, const uint16_t* lambdas, int metric,
                          int device, tsdg_gpu_index** out);
int tsdg_gpu_index_create_from_file(const char* tsdg_path, const float* base, uint32_t n,
                                    uint32_t d, int device, tsdg_gpu_index** out);
/* Direct file -> HBM index: the raw bytes of a reference .tsdg
 * file (load_tsdg, diversify.cpp:274-306) and an fvecs/bvecs base (load_vectors,
 * io.cpp:112-117) are streamed through pinned staging buffers and decoded on the
 * device into the search layout; no host-side CSR or VectorSet is built.  The
 * metric comes from the TSDG header.  Same index as tsdg_gpu_index_create on the
 * decoded arrays. */
int tsdg_gpu_index_create_from_files(const char* tsdg_path, const char* vectors_path, int device,
                                     tsdg_gpu_index** out);
int tsdg_gpu_index_destroy(tsdg_gpu_index* idx);
/* n, d, metric, max_degree, device, padded row stride (floats), adjacency stride */
int tsdg_gpu_index_info(const tsdg_gpu_index* idx, uint32_t* n, uint32_t* d, int* metric,
                        uint32_t* max_degree, int* device, uint32_t* row_stride,
                        uint32_t* adj_stride);
/* deg_cut: per-node lambda-prefix length for a cutoff (diversify.cpp:34-42), kept
 * cached in the index; copies it out when out != NULL (n entries). */
int tsdg_gpu_deg_cut(tsdg_gpu_index* idx, uint32_t lambda_cut, uint32_t* out);

/* ---- large batch: best-first, Alg. 2 ------------------------------------------
 * Replaces tsdg::large_batch_search (bestfirst_search.cpp:129-150).  Query q uses
 * the stream Rng64(params.seed).fork(query_index_base + q); with base 0 this is the
 * reference batch call, and a split batch (multi-GPU) passes its slice start.
 * ids: nq x k, ascending by (dist, id), padded 0xFFFFFFFF; dists padded +inf;
 * counts: nq; stats: nq entries or NULL.  HOST pointers; all transfers inside the
 * call: when every buffer lies in mapped pinned memory (cudaMallocHost /
 * cudaHostAlloc / torch pin_memory) the kernel reads the queries and writes the
 * results over the bus directly (zero-copy); otherwise a copy/compute pipeline.
 * TSDG_ZERO_COPY=0 forces the pipeline.  Same results either way. */
int tsdg_gpu_search_bestfirst(tsdg_gpu_index* idx, const float* queries, uint32_t nq,
                              uint64_t query_index_base, const tsdg_bf_params* params,
                              int mode, uint32_t* ids, float* dists, uint32_t* counts,
                              tsdg_query_stats* stats);
/* Same, DEVICE pointers, asynchronous on `stream` (cudaStream_t; NULL = legacy). */
int tsdg_gpu_search_bestfirst_device(tsdg_gpu_index* idx, const float* d_queries, uint32_t nq,
                                     uint64_t query_index_base, const tsdg_bf_params* params,
                                     int mode, uint32_t* d_ids, float* d_dists,
                                     uint32_t* d_counts, tsdg_query_stats* d_stats,
                                     void* stream);

/* ---- small batch: multi-start greedy, Alg. 1 --------------------------------
 * Replaces tsdg::small_batch_search (greedy_search.cpp:106-127): t0 walks per query
 * with streams Rng64(seed).fork(s) (the same for every query), merged by
 * (dist, id) with id-dedup, first k.  Output layout as for best-first; HOST
 * pointers, zero-copy with mapped pinned buffers as for best-first. */
int tsdg_gpu_search_greedy(tsdg_gpu_index* idx, const float* queries, uint32_t nq, uint32_t k,
                           const tsdg_greedy_params* params, int mode, uint32_t* ids,
                           float* dists, uint32_t* counts, tsdg_query_stats* stats);
int tsdg_gpu_search_greedy_device(tsdg_gpu_index* idx, const float* d_queries, uint32_t nq,
                                  uint32_t k, const tsdg_greedy_params* params, int mode,
                                  uint32_t* d_ids, float* d_dists, uint32_t* d_counts,
                                  tsdg_query_stats* d_stats, void* stream);
/* One greedy walk (greedy_search.cpp:27-72) per query with an explicit RNG state
 * per query (rng_states[q]): the 32-slot R_ij is written to ids32/dists32 (nq x 32). */
int tsdg_gpu_greedy_once(tsdg_gpu_index* idx, const float* queries, uint32_t nq,
                         const uint64_t* rng_states, uint32_t hop_limit, uint32_t lambda_cut,
                         uint32_t* ids32, float* dists32, tsdg_query_stats* stats);


/* ---- sharded base: per-shard top-k merge (no reference counterpart) ----------
 * After an all-gather of S shards' results (each nq x k, LOCAL ids, ascending),
 * merges per query by (dist, global id), global id = shard_base[s] + local id.
 * DEVICE pointers; layout [s][q][k]. */
int tsdg_gpu_merge_shards_device(const uint32_t* d_ids, const float* d_dists,
                                 const uint32_t* d_counts, const uint64_t* shard_base,
                                 uint32_t shards, uint32_t nq, uint32_t k, uint32_t* d_out_ids,
                                 float* d_out_dists, uint32_t* d_out_counts, void* stream);

/* ---- replicated index over several GPUs in one process -----------------------
 * SURVEY.md §8(b)/(e) "replicate" mode: one device index per entry of `devices`
 * (built concurrently), each batch split into contiguous slices searched on the
 * devices concurrently, slice b..e with query_index_base + b, so every query keeps
 * its reference RNG stream and the results are identical for any device list.
 * Host pointers, same layouts and errors as the single-device calls.  (The sharded
 * base layout with an NCCL all-gather lives in the Python layer, shards.py.) */
typedef struct tsdg_gpu_multi tsdg_gpu_multi;
int tsdg_gpu_multi_create(const float* base, uint32_t n, uint32_t d, const uint64_t* offsets,
                          const uint32_t* targets, const uint16_t* lambdas, int metric,
                          const int* devices, int ndev, tsdg_gpu_multi** out);
int tsdg_gpu_multi_destroy(tsdg_gpu_multi* m);
int tsdg_gpu_multi_search_bestfirst(tsdg_gpu_multi* m, const float* queries, uint32_t nq,
                                    uint64_t query_index_base, const tsdg_bf_params* params,
                                    int mode, uint32_t* ids, float* dists, uint32_t* counts,
                                    tsdg_query_stats* stats);
int tsdg_gpu_multi_search_greedy(tsdg_gpu_multi* m, const float* queries, uint32_t nq, uint32_t k,
                                 const tsdg_greedy_params* params, int mode, uint32_t* ids,
                                 float* dists, uint32_t* counts, tsdg_query_stats* stats);

/* ---- sharded base in one process (the C5 layout) --------------
 * Shard s: a TSDG over its own rows (local ids, e.g. built by the reference per
 * shard) and base rows bases[s] (shard_n[s] x d); global id = shard_offset[s] + local.
 * A search runs every query on every shard (each shard on devices[s], concurrently),
 * copies the per-shard top-k peer-to-peer to the first shard's device and merges them
 * there by (dist, global id), first k (merge_shards_kernel).  Host pointers;
 * ids / dists nq x k, counts nq. */
typedef struct tsdg_gpu_sharded tsdg_gpu_sharded;
int tsdg_gpu_sharded_create_from_files(const char* const* tsdg_paths, const float* const* bases,
                                       const uint32_t* shard_n, const uint64_t* shard_offset,
                                       uint32_t nshards, uint32_t d, const int* devices,
                                       tsdg_gpu_sharded** out);
int tsdg_gpu_sharded_destroy(tsdg_gpu_sharded* sh);
int tsdg_gpu_sharded_search_bestfirst(tsdg_gpu_sharded* sh, const float* queries, uint32_t nq,
                                      uint64_t query_index_base, const tsdg_bf_params* params,
                                      int mode, uint32_t* ids, float* dists, uint32_t* counts);

/* ---- exact top-k scan ----------------------------
 * Per query the k smallest (dist, id) pairs over every base row, distances bit-equal
 * to the reference's kernel (sequential fp32, vectors.hpp:36-49), ties by id
 * (common.hpp:22-25).  Output nq x k ascending, padded 0xFFFFFFFF / +inf.  GPU
 * limit: k <= 384.
 *
 * tsdg_gpu_ground_truth replaces tsdg::ground_truth (bench.cpp:35-57; same checks:
 * 1 <= k_gt <= n) and ref::exact_topk (reference.cpp:96-111); dists may be NULL.
 * tsdg_gpu_index_ground_truth: the same over an index's resident vector store.
 * tsdg_gpu_brute_force_knn replaces tsdg::brute_force_knn (knn_graph.cpp:64-86):
 * the self pair is excluded, n < 2 and k < 1 are invalid, k > n-1 is clamped to n-1
 * (warning on stderr, knn_graph.cpp:17-26) and returned in *k_eff; ids/dists are
 * n x k_eff (the KnnGraph flat layout, knn_graph.hpp:15-28).
 * tsdg_gpu_exact_topk_device: DEVICE pointers, row strides ld_* (multiples of 4
 * floats), asynchronous on `stream`; exclude_self skips base row self_base + q for
 * query q. */
int tsdg_gpu_ground_truth(const float* base, uint32_t n, const float* queries, uint32_t nq,
                          uint32_t d, uint32_t k_gt, int metric, int device, uint32_t* ids,
                          float* dists);
int tsdg_gpu_index_ground_truth(tsdg_gpu_index* idx, const float* queries, uint32_t nq,
                                uint32_t k_gt, uint32_t* ids, float* dists);
int tsdg_gpu_brute_force_knn(const float* base, uint32_t n, uint32_t d, uint32_t k, int metric,
                             int device, uint32_t* ids, float* dists, uint32_t* k_eff);
int tsdg_gpu_exact_topk_device(const float* d_base, uint32_t n, uint32_t ld_base,
                               const float* d_queries, uint32_t nq, uint32_t ld_queries,
                               uint32_t d, uint32_t k, int metric, int exclude_self,
                               uint64_t self_base, uint32_t* d_ids, float* d_dists, void* stream);

/* tsdg_gpu_nn_descent replaces tsdg::nn_descent (knn_graph.cpp:141-251): the same
 * KnnGraph bit for bit (ids and fp32 distances, rows ascending by (dist, id)) for the
 * same (set, k, metric, iterations, sample_rate, seed), independent of scheduling as
 * the reference's is of its thread count.  Errors as the reference: sample_rate outside
 * (0, 1], n < 2 and k < 1 are invalid; k > n-1 is clamped to n-1 (warning on stderr)
 * and returned in *k_eff.  GPU limits: k_eff <= 128, n < 2^31.  stats4 (nullable) =
 * {offers merged, join chunks, chunk re-runs, kernel launches}. */
int tsdg_gpu_nn_descent(const float* base, uint32_t n, uint32_t d, uint32_t k, int metric,
                        uint32_t iterations, double sample_rate, uint64_t seed, int device,
                        uint32_t* ids, float* dists, uint32_t* k_eff, uint64_t* stats4);

/* ---- GPU two-stage diversification ------------------------
 * Replaces tsdg::build (diversify.cpp:152-209): stage 1 relaxed GD per node
 * (:44-69), reverse edges with dedup and the dist_matches re-check (:71-124), stage
 * 2 lambda counts with the lambda0 filter, (lambda, dist, target) order and the
 * max_degree cap (:126-150).  Given the same KnnGraph (knn_ids / knn_dists: n x k,
 * rows ascending by (dist, id) as brute_force_knn / nn_descent produce them) the
 * result equals the reference's TsdgGraph edge for edge, fp32 distances included.
 * Errors as the reference: alpha < 1 and unsorted candidate rows are invalid
 * arguments (diversify.cpp:48-53,157), a target >= n too (add_reverse_edges throws
 * std::out_of_range there).  GPU limit: k <= 128.  stats4 (nullable) = BuildStats
 * {input_edges, stage1_edges, augmented_edges, final_edges} (diversify.hpp:39-44).
 * The graph lives on the host: tsdg_gpu_graph_copy fills CSR arrays sized by
 * tsdg_gpu_graph_info (offsets n+1, the rest num_edges); tsdg_gpu_graph_save writes
 * the reference's file format (save_tsdg, diversify.cpp:252-272). */
typedef struct tsdg_gpu_graph tsdg_gpu_graph;
int tsdg_gpu_build(const float* base, uint32_t n, uint32_t d, const uint32_t* knn_ids,
                   const float* knn_dists, uint32_t k, float alpha, uint16_t lambda0,
                   uint32_t max_degree, int metric, int device, tsdg_gpu_graph** out,
                   uint64_t* stats4);
int tsdg_gpu_graph_info(const tsdg_gpu_graph* g, uint64_t* n, uint64_t* num_edges,
                        uint32_t* max_degree);
int tsdg_gpu_graph_copy(const tsdg_gpu_graph* g, uint64_t* offsets, uint32_t* targets,
                        uint16_t* lambdas, float* dists);
int tsdg_gpu_graph_save(const tsdg_gpu_graph* g, const char* path);
int tsdg_gpu_graph_destroy(tsdg_gpu_graph* g);

/* Number of kernels this library launched since load (evidence counter). */
uint64_t tsdg_gpu_launch_count(void);

/* 1 when [p, p + bytes) lies in one mapped pinned host allocation — the condition
 * under which the host-pointer search calls take the zero-copy path (the kernel reads
 * queries from / writes results to host memory); 0 otherwise (copy pipeline). */
int tsdg_gpu_host_buffer_mapped(const void* p, uint64_t bytes);

#ifdef __cplusplus
}
#endif
#endif /* TSDG_GPU_H */
