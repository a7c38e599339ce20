/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load this; the product path never does.
 *
 * Plain-C restatement of the reference's search hot path
 * (/root/reference/proj, cited per function in tsdg_oracle.c).  Pinned against
 * the reference itself: tests/test_oracle.py compares every entry point with
 * oracle/_ref/libtsdg_ref.so (the unmodified reference) and with the committed
 * golden vectors in tests/golden/ (made by tests/golden/make_golden.py).
 *
 * Status codes: 0 ok, 1 invalid argument (std::invalid_argument in the
 * reference), 2 runtime/allocation.
 */
#ifndef TSDG_ORACLE_H
#define TSDG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    uint32_t n;               /* nodes == base rows */
    uint32_t d;               /* dimension */
    int metric;               /* 0 L2 (squared), 1 cosine (1-dot), 2 inner product (-dot) */
    const float* base;        /* n x d row-major */
    const uint64_t* offsets;  /* n + 1, CSR (diversify.hpp:61) */
    const uint32_t* targets;  /* edge targets, per node sorted by (lambda, dist, target) */
    const uint16_t* lambdas;  /* occlusion factor per edge */
} tsdg_o_graph;

typedef struct {
    uint32_t k, hop_limit;
    float delta;
    uint32_t m_segments, lambda_cut;
    uint64_t seed;
    int unbounded;            /* not restated: must be 0 (see tsdg_oracle.c) */
} tsdg_o_bf_params;

typedef struct {
    uint32_t t0, hop_limit, lambda_cut;
    uint64_t seed;
} tsdg_o_greedy_params;

uint64_t tsdg_o_mix64(uint64_t z);
uint64_t tsdg_o_fork(uint64_t state, uint64_t index);
float tsdg_o_distance(const float* a, const float* b, uint32_t d, int metric);

/* one bestfirst_search with explicit RNG state; stats3 = hops, evals, evictions;
 * trace2 = expanded, examined counts. ids/dists have room for k. */
int tsdg_o_bestfirst(const tsdg_o_graph* g, const float* query, uint64_t rng_state,
                     const tsdg_o_bf_params* p, uint32_t* ids, float* dists, uint32_t* count,
                     uint64_t* stats3, uint64_t* trace2);

/* large_batch_search with per-query stream Rng64(seed).fork(query_index_base + q). */
int tsdg_o_large_batch(const tsdg_o_graph* g, const float* queries, uint32_t nq,
                       uint64_t query_index_base, const tsdg_o_bf_params* p, uint32_t* ids,
                       float* dists, uint32_t* counts, uint64_t* stats);

int tsdg_o_greedy_once(const tsdg_o_graph* g, const float* query, uint64_t rng_state,
                       uint32_t hop_limit, uint32_t lambda_cut, uint32_t* ids32,
                       float* dists32, uint64_t* stats3);

int tsdg_o_small_batch(const tsdg_o_graph* g, const float* queries, uint32_t nq, uint32_t k,
                       const tsdg_o_greedy_params* p, uint32_t* ids, float* dists,
                       uint32_t* counts, uint64_t* stats);

int tsdg_o_lane_update(uint32_t* slot_ids, float* slot_dists, const uint32_t* lanes,
                       const uint32_t* ids, const float* dists, uint32_t nb);
int tsdg_o_merge_halves(uint32_t* rij_ids, float* rij_dists, const uint32_t* tmp_ids,
                        const float* tmp_dists, int* updated);
int tsdg_o_segmented_replay(uint32_t m, const uint8_t* ops, const uint32_t* ids,
                            const float* dists, uint32_t n_ops, uint32_t* out,
                            float* out_dist, uint64_t* sizes, uint64_t* evictions);
int tsdg_o_topk_replay(uint32_t k, const uint8_t* ops, const uint32_t* ids,
                       const float* dists, uint32_t n_ops, uint32_t* out,
                       uint32_t* final_ids, float* final_dists, uint32_t* final_n);
int tsdg_o_exact_topk(const float* base, uint32_t n, const float* queries, uint32_t nq,
                      uint32_t d, uint32_t k, int metric, uint32_t* ids, float* dists);
int tsdg_o_brute_force_knn(const float* base, uint32_t n, uint32_t d, uint32_t k, int metric,
                           uint32_t* ids, float* dists);

#ifdef __cplusplus
}
#endif
#endif
