// TEST INFRASTRUCTURE ONLY — never linked into the product path.
//
// extern "C" shim over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src/*.cpp by oracle/Makefile into oracle/_ref/).  It lets
// pytest (ctypes), bench.py's cpu_baseline leg and the dataset tool call the
// reference's own functions with plain pointers:
//   - search:      tsdg::large_batch_search / small_batch_search / bestfirst_search
//                  (bestfirst_search.cpp:112-150, greedy_search.cpp:74-127)
//   - primitives:  lane_update / merge_halves (rank_list.cpp:8-49),
//                  SegmentedQueue / SegmentedVisited / TopK (segmented.cpp:8-111)
//   - data:        make_synthetic_split (bench.cpp:114-129), ground_truth (bench.cpp:35-57)
//   - graph build: brute_force_knn / nn_descent (knn_graph.cpp:64-251) + build (diversify.cpp:152-209)
//   - file I/O:    save_tsdg / load_tsdg (diversify.cpp:252-306)
// Nothing here re-implements reference logic; it only marshals arguments.

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "tsdg/bench.hpp"
#include "tsdg/bestfirst_search.hpp"
#include "tsdg/diversify.hpp"
#include "tsdg/greedy_search.hpp"
#include "tsdg/io.hpp"
#include "tsdg/knn_graph.hpp"
#include "tsdg/rank_list.hpp"
#include "tsdg/reference.hpp"
#include "tsdg/segmented.hpp"

using namespace tsdg;

namespace {

thread_local std::string g_err;

// 0 ok, 1 invalid_argument, 2 runtime_error / other, 3 domain_error, 4 logic_error
template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

VectorSet make_set(const float* data, std::uint32_t n, std::uint32_t d) {
    VectorSet s;
    s.n = n;
    s.d = d;
    s.data.assign(data, data + static_cast<std::size_t>(n) * d);
    return s;
}

struct Fixture {
    TsdgGraph graph;
    VectorSet base;
};

BestFirstParams bf_params(std::uint32_t k, std::uint32_t hop_limit, float delta,
                          std::uint32_t m, std::uint32_t cut, std::uint64_t seed,
                          int unbounded) {
    BestFirstParams p;
    p.k = k;
    p.hop_limit = hop_limit;
    p.delta = delta;
    p.m_segments = m;
    p.lambda_cut = cut;
    p.seed = seed;
    p.unbounded = unbounded != 0;
    return p;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_num_threads() {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void ref_set_num_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}

// ---- RNG (common.hpp:27-61) -------------------------------------------------
std::uint64_t ref_mix64(std::uint64_t z) { return mix64(z); }

// Draws `count` values of Rng64(seed).fork(fork_index).below(n) in order.
void ref_rng_below_stream(std::uint64_t seed, std::uint64_t fork_index, int do_fork,
                          std::uint32_t n, std::uint32_t count, std::uint32_t* out) {
    Rng64 r = do_fork ? Rng64(seed).fork(fork_index) : Rng64(seed);
    for (std::uint32_t i = 0; i < count; ++i) out[i] = r.below(n);
}

// ---- data -------------------------------------------------------------------
int ref_make_synthetic_split(std::uint32_t n, std::uint32_t nq, std::uint32_t d,
                             std::uint32_t clusters, float spread, std::uint64_t seed,
                             float* base_out, float* queries_out) {
    return guarded([&] {
        auto [b, q] = make_synthetic_split(n, nq, d, clusters, spread, seed);
        std::memcpy(base_out, b.data.data(), b.data.size() * sizeof(float));
        std::memcpy(queries_out, q.data.data(), q.data.size() * sizeof(float));
    });
}

int ref_make_synthetic(std::uint32_t n, std::uint32_t d, std::uint32_t clusters,
                       float spread, std::uint64_t seed, float* out) {
    return guarded([&] {
        const auto s = make_synthetic(n, d, clusters, spread, seed);
        std::memcpy(out, s.data.data(), s.data.size() * sizeof(float));
    });
}

int ref_ground_truth(const float* base, std::uint32_t n, const float* queries,
                     std::uint32_t nq, std::uint32_t d, std::uint32_t k_gt, int metric,
                     std::uint32_t* ids_out) {
    return guarded([&] {
        const auto gt = ground_truth(make_set(base, n, d), make_set(queries, nq, d), k_gt,
                                     static_cast<Metric>(metric));
        for (std::uint32_t q = 0; q < nq; ++q) {
            std::copy(gt.ids[q].begin(), gt.ids[q].end(),
                      ids_out + static_cast<std::size_t>(q) * k_gt);
        }
    });
}

float ref_distance(const float* a, const float* b, std::uint32_t d, int metric) {
    return kernel_for(static_cast<Metric>(metric))(a, b, d);
}

// ---- graph build + file I/O -------------------------------------------------
// method 0 = brute_force_knn, 1 = nn_descent. Writes the TSDG file to `path`.
int ref_build_tsdg(const float* base, std::uint32_t n, std::uint32_t d, int metric,
                   int method, std::uint32_t knn_k, std::uint32_t iterations,
                   double sample_rate, std::uint64_t knn_seed, float alpha,
                   std::uint32_t lambda0, std::uint32_t max_degree, const char* path,
                   std::uint64_t* stats4) {
    return guarded([&] {
        const VectorSet set = make_set(base, n, d);
        const auto m = static_cast<Metric>(metric);
        const KnnGraph knn = method == 0
                                 ? brute_force_knn(set, knn_k, m)
                                 : nn_descent(set, knn_k, m, iterations, sample_rate, knn_seed);
        DiversifyParams p;
        p.alpha = alpha;
        p.lambda0 = static_cast<std::uint16_t>(lambda0);
        p.max_degree = max_degree;
        BuildStats bs;
        const TsdgGraph g = build(set, knn, p, m, &bs);
        save_tsdg(g, path);
        if (stats4) {
            stats4[0] = bs.input_edges;
            stats4[1] = bs.stage1_edges;
            stats4[2] = bs.augmented_edges;
            stats4[3] = bs.final_edges;
        }
    });
}

// tsdg::normalized_copy (vectors.cpp:68-80).
int ref_normalized_copy(const float* data, std::uint32_t n, std::uint32_t d, float* out) {
    return guarded([&] {
        const auto v = normalized_copy(make_set(data, n, d));
        std::copy(v.data.begin(), v.data.end(), out);
    });
}

// tsdg::load_vectors (io.cpp:112-117): shape first (out == NULL), then the data.
int ref_load_vectors(const char* path, std::uint32_t* n, std::uint32_t* d, float* out) {
    return guarded([&] {
        const VectorSet v = load_vectors(path);
        *n = v.n;
        *d = v.d;
        if (out) std::copy(v.data.begin(), v.data.end(), out);
    });
}

// tsdg::run_bench_file (bench.cpp:189-362), unmodified; writes the CSV.
int ref_run_bench_file(const char* config_path, const char* csv_out) {
    return guarded([&] { run_bench_file(config_path, csv_out); });
}

// tsdg::nn_descent (knn_graph.cpp:141-251) rows: n x k_eff (id, dist).
int ref_nn_descent(const float* base, std::uint32_t n, std::uint32_t d, int metric,
                   std::uint32_t k, std::uint32_t iterations, double sample_rate,
                   std::uint64_t seed, std::uint32_t* ids_out, float* dists_out,
                   std::uint32_t* k_eff) {
    return guarded([&] {
        const auto g = nn_descent(make_set(base, n, d), k, static_cast<Metric>(metric),
                                  iterations, sample_rate, seed);
        *k_eff = g.k;
        for (std::size_t i = 0; i < g.flat.size(); ++i) {
            ids_out[i] = g.flat[i].id;
            dists_out[i] = g.flat[i].dist;
        }
    });
}

// tsdg::build (diversify.cpp:152-209) from an explicit KnnGraph; saved with save_tsdg.
int ref_build_from_knn(const float* base, std::uint32_t n, std::uint32_t d, int metric,
                       const std::uint32_t* knn_ids, const float* knn_dists, std::uint32_t k,
                       float alpha, std::uint32_t lambda0, std::uint32_t max_degree,
                       const char* path, std::uint64_t* stats4) {
    return guarded([&] {
        KnnGraph knn;
        knn.n = n;
        knn.k = k;
        knn.flat.resize(static_cast<std::size_t>(n) * k);
        for (std::size_t i = 0; i < knn.flat.size(); ++i) knn.flat[i] = {knn_ids[i], knn_dists[i]};
        DiversifyParams p;
        p.alpha = alpha;
        p.lambda0 = static_cast<std::uint16_t>(lambda0);
        p.max_degree = max_degree;
        BuildStats bs;
        const TsdgGraph g = build(make_set(base, n, d), knn, p, static_cast<Metric>(metric), &bs);
        save_tsdg(g, path);
        if (stats4) {
            stats4[0] = bs.input_edges;
            stats4[1] = bs.stage1_edges;
            stats4[2] = bs.augmented_edges;
            stats4[3] = bs.final_edges;
        }
    });
}

// Saves an explicit CSR adjacency through tsdg_from_adjacency + save_tsdg
// (diversify.cpp:211-272); validates ordering exactly like the reference.
int ref_save_csr(std::uint32_t n, int metric, std::uint32_t k, float alpha,
                 std::uint32_t lambda0, const std::uint64_t* offsets,
                 const std::uint32_t* targets, const std::uint16_t* lambdas,
                 const float* dists, const char* path) {
    return guarded([&] {
        std::vector<std::vector<TsdgEdge>> adj(n);
        for (std::uint32_t u = 0; u < n; ++u) {
            for (std::uint64_t j = offsets[u]; j < offsets[u + 1]; ++j) {
                adj[u].push_back({targets[j], lambdas[j], dists[j]});
            }
        }
        const auto g = tsdg_from_adjacency(n, static_cast<Metric>(metric), k, alpha,
                                           static_cast<std::uint16_t>(lambda0), adj);
        save_tsdg(g, path);
    });
}

// ---- fixtures: graph + base held by the reference types ---------------------
void* ref_fixture_load(const char* tsdg_path, const float* base, std::uint32_t n,
                       std::uint32_t d) {
    auto* fx = new Fixture;
    const int rc = guarded([&] {
        fx->graph = load_tsdg(tsdg_path);
        fx->base = make_set(base, n, d);
    });
    if (rc != 0) {
        delete fx;
        return nullptr;
    }
    return fx;
}

// Both inputs through the reference's own loaders: load_tsdg (diversify.cpp:274-306)
// and load_vectors (io.cpp:112-117) — bench.py's reference arm.
void* ref_fixture_load_files(const char* tsdg_path, const char* vectors_path) {
    auto* fx = new Fixture;
    const int rc = guarded([&] {
        fx->graph = load_tsdg(tsdg_path);
        fx->base = load_vectors(vectors_path);
    });
    if (rc != 0) {
        delete fx;
        return nullptr;
    }
    return fx;
}

std::uint32_t ref_fixture_d(void* h) { return static_cast<Fixture*>(h)->base.d; }

void ref_fixture_free(void* h) { delete static_cast<Fixture*>(h); }

std::uint32_t ref_fixture_n(void* h) { return static_cast<Fixture*>(h)->graph.n; }
std::uint64_t ref_fixture_edges(void* h) {
    return static_cast<Fixture*>(h)->graph.edges.size();
}

// Copies the loaded CSR out (offsets n+1, then edges).
void ref_fixture_csr(void* h, std::uint64_t* offsets, std::uint32_t* targets,
                     std::uint16_t* lambdas, float* dists) {
    const auto& g = static_cast<Fixture*>(h)->graph;
    std::copy(g.offsets.begin(), g.offsets.end(), offsets);
    for (std::size_t i = 0; i < g.edges.size(); ++i) {
        targets[i] = g.edges[i].target;
        lambdas[i] = g.edges[i].lambda;
        dists[i] = g.edges[i].dist;
    }
}

// The reference batch front end, called exactly as bench.cpp:329-333 does
// (ids only; stats summed). ids_out is nq x k padded with 0xFFFFFFFF.
int ref_large_batch_search(void* h, const float* queries, std::uint32_t nq,
                           std::uint32_t k, std::uint32_t hop_limit, float delta,
                           std::uint32_t m, std::uint32_t cut, std::uint64_t seed,
                           int unbounded, std::uint32_t* ids_out, std::uint32_t* counts,
                           std::uint64_t* stats3) {
    return guarded([&] {
        const auto* fx = static_cast<Fixture*>(h);
        const VectorSet qs = make_set(queries, nq, fx->base.d);
        SearchStats st;
        const auto res = large_batch_search(fx->graph, fx->base, qs,
                                            bf_params(k, hop_limit, delta, m, cut, seed,
                                                      unbounded),
                                            &st);
        for (std::uint32_t q = 0; q < nq; ++q) {
            counts[q] = static_cast<std::uint32_t>(res[q].size());
            for (std::uint32_t i = 0; i < k; ++i) {
                ids_out[static_cast<std::size_t>(q) * k + i] =
                    i < res[q].size() ? res[q][i] : kInvalidId;
            }
        }
        if (stats3) {
            stats3[0] = st.hops;
            stats3[1] = st.distance_evals;
            stats3[2] = st.queue_evictions;
        }
    });
}

int ref_small_batch_search(void* h, const float* queries, std::uint32_t nq, std::uint32_t k,
                           std::uint32_t t0, std::uint32_t hop_limit, std::uint32_t cut,
                           std::uint64_t seed, std::uint32_t* ids_out, std::uint32_t* counts,
                           std::uint64_t* stats3) {
    return guarded([&] {
        const auto* fx = static_cast<Fixture*>(h);
        const VectorSet qs = make_set(queries, nq, fx->base.d);
        GreedyParams p;
        p.t0 = t0;
        p.hop_limit = hop_limit;
        p.lambda_cut = cut;
        p.seed = seed;
        SearchStats st;
        const auto res = small_batch_search(fx->graph, fx->base, qs, k, p, &st);
        for (std::uint32_t q = 0; q < nq; ++q) {
            counts[q] = static_cast<std::uint32_t>(res[q].size());
            for (std::uint32_t i = 0; i < k; ++i) {
                ids_out[static_cast<std::size_t>(q) * k + i] =
                    i < res[q].size() ? res[q][i] : kInvalidId;
            }
        }
        if (stats3) {
            stats3[0] = st.hops;
            stats3[1] = st.distance_evals;
            stats3[2] = st.queue_evictions;
        }
    });
}

// Per-query stats: one bestfirst_search per query with Rng64(seed).fork(base+q),
// the stream large_batch_search hands query q (bestfirst_search.cpp:136-143).
// stats_out is nq x 3 (hops, evals, evictions); trace sizes nq x 2
// (expanded, examined) when non-null.
int ref_bestfirst_per_query(void* h, const float* queries, std::uint32_t nq,
                            std::uint64_t query_index_base, std::uint32_t k,
                            std::uint32_t hop_limit, float delta, std::uint32_t m,
                            std::uint32_t cut, std::uint64_t seed, int unbounded,
                            std::uint32_t* ids_out, std::uint32_t* counts,
                            std::uint64_t* stats_out, std::uint64_t* trace_sizes) {
    return guarded([&] {
        const auto* fx = static_cast<Fixture*>(h);
        const auto p = bf_params(k, hop_limit, delta, m, cut, seed, unbounded);
        const Rng64 base(seed);
        std::string err;
#pragma omp parallel for schedule(dynamic, 8)
        for (std::int64_t qi = 0; qi < static_cast<std::int64_t>(nq); ++qi) {
            try {
                const auto q = static_cast<std::uint32_t>(qi);
                SearchStats st;
                EdgeTrace tr;
                const auto res = bestfirst_search(
                    fx->graph, fx->base,
                    std::span<const float>(queries + static_cast<std::size_t>(q) * fx->base.d,
                                           fx->base.d),
                    p, base.fork(query_index_base + q), &st, trace_sizes ? &tr : nullptr);
                counts[q] = static_cast<std::uint32_t>(res.size());
                for (std::uint32_t i = 0; i < k; ++i) {
                    ids_out[static_cast<std::size_t>(q) * k + i] =
                        i < res.size() ? res[i] : kInvalidId;
                }
                stats_out[3 * q + 0] = st.hops;
                stats_out[3 * q + 1] = st.distance_evals;
                stats_out[3 * q + 2] = st.queue_evictions;
                if (trace_sizes) {
                    trace_sizes[2 * q + 0] = tr.expanded.size();
                    trace_sizes[2 * q + 1] = tr.examined.size();
                }
            } catch (const std::exception& e) {
#pragma omp critical
                err = e.what();
            }
        }
        if (!err.empty()) throw std::invalid_argument(err);
    });
}

// Full EdgeTrace of one query: expanded ids (cap entries) and examined targets.
int ref_bestfirst_trace(void* h, const float* query, std::uint64_t rng_seed, int fork,
                        std::uint64_t fork_index, std::uint32_t k, std::uint32_t hop_limit,
                        float delta, std::uint32_t m, std::uint32_t cut, int unbounded,
                        std::uint32_t* ids_out, std::uint32_t* count,
                        std::uint32_t* expanded, std::uint32_t* n_expanded,
                        std::uint32_t* examined, std::uint32_t* n_examined,
                        std::uint32_t cap) {
    return guarded([&] {
        const auto* fx = static_cast<Fixture*>(h);
        const auto p = bf_params(k, hop_limit, delta, m, cut, 0, unbounded);
        const Rng64 r = fork ? Rng64(rng_seed).fork(fork_index) : Rng64(rng_seed);
        EdgeTrace tr;
        const auto res = bestfirst_search(fx->graph, fx->base,
                                          std::span<const float>(query, fx->base.d), p, r,
                                          nullptr, &tr);
        *count = static_cast<std::uint32_t>(res.size());
        std::copy(res.begin(), res.end(), ids_out);
        *n_expanded = static_cast<std::uint32_t>(tr.expanded.size());
        *n_examined = static_cast<std::uint32_t>(tr.examined.size());
        for (std::size_t i = 0; i < tr.expanded.size() && i < cap; ++i) expanded[i] = tr.expanded[i];
        for (std::size_t i = 0; i < tr.examined.size() && i < cap; ++i) {
            examined[2 * i] = tr.examined[i].first;
            examined[2 * i + 1] = tr.examined[i].second;
        }
    });
}

// Per-query greedy: small_batch_search_one per query (greedy_search.cpp:74-104).
int ref_greedy_per_query(void* h, const float* queries, std::uint32_t nq, std::uint32_t k,
                         std::uint32_t t0, std::uint32_t hop_limit, std::uint32_t cut,
                         std::uint64_t seed, std::uint32_t* ids_out, std::uint32_t* counts,
                         std::uint64_t* stats_out) {
    return guarded([&] {
        const auto* fx = static_cast<Fixture*>(h);
        GreedyParams p;
        p.t0 = t0;
        p.hop_limit = hop_limit;
        p.lambda_cut = cut;
        p.seed = seed;
        std::string err;
#pragma omp parallel for schedule(dynamic, 1)
        for (std::int64_t qi = 0; qi < static_cast<std::int64_t>(nq); ++qi) {
            try {
                const auto q = static_cast<std::uint32_t>(qi);
                SearchStats st;
                const auto res = small_batch_search_one(
                    fx->graph, fx->base,
                    std::span<const float>(queries + static_cast<std::size_t>(q) * fx->base.d,
                                           fx->base.d),
                    k, p, &st);
                counts[q] = static_cast<std::uint32_t>(res.size());
                for (std::uint32_t i = 0; i < k; ++i) {
                    ids_out[static_cast<std::size_t>(q) * k + i] =
                        i < res.size() ? res[i] : kInvalidId;
                }
                stats_out[3 * q + 0] = st.hops;
                stats_out[3 * q + 1] = st.distance_evals;
                stats_out[3 * q + 2] = st.queue_evictions;
            } catch (const std::exception& e) {
#pragma omp critical
                err = e.what();
            }
        }
        if (!err.empty()) throw std::invalid_argument(err);
    });
}

// One greedy_search_once (greedy_search.cpp:27-72); out is the 32-slot R_ij.
int ref_greedy_search_once(void* h, const float* query, std::uint64_t rng_seed, int fork,
                           std::uint64_t fork_index, std::uint32_t hop_limit,
                           std::uint32_t cut, std::uint32_t* ids32, float* dists32,
                           std::uint64_t* stats3) {
    return guarded([&] {
        const auto* fx = static_cast<Fixture*>(h);
        GreedyParams p;
        p.hop_limit = hop_limit;
        p.lambda_cut = cut;
        const Rng64 r = fork ? Rng64(rng_seed).fork(fork_index) : Rng64(rng_seed);
        SearchStats st;
        const RankList rl = greedy_search_once(
            fx->graph, fx->base, std::span<const float>(query, fx->base.d), p, r, &st);
        for (std::uint32_t i = 0; i < kLaneWidth; ++i) {
            ids32[i] = rl.slot[i].id;
            dists32[i] = rl.slot[i].dist;
        }
        if (stats3) {
            stats3[0] = st.hops;
            stats3[1] = st.distance_evals;
            stats3[2] = st.queue_evictions;
        }
    });
}

// ---- primitives -------------------------------------------------------------
// lane_update over `nb` entries (rank_list.cpp:8-18); slots are in/out.
int ref_lane_update(std::uint32_t* slot_ids, float* slot_dists, const std::uint32_t* lanes,
                    const std::uint32_t* ids, const float* dists, std::uint32_t nb) {
    return guarded([&] {
        RankList r;
        for (std::uint32_t i = 0; i < kLaneWidth; ++i) r.slot[i] = {slot_ids[i], slot_dists[i]};
        std::vector<LaneEntry> batch(nb);
        for (std::uint32_t i = 0; i < nb; ++i) batch[i] = {lanes[i], ids[i], dists[i]};
        lane_update(r, batch);
        for (std::uint32_t i = 0; i < kLaneWidth; ++i) {
            slot_ids[i] = r.slot[i].id;
            slot_dists[i] = r.slot[i].dist;
        }
    });
}

// merge_halves (rank_list.cpp:20-49); r_ij in/out, returns updated via *updated.
int ref_merge_halves(std::uint32_t* rij_ids, float* rij_dists, const std::uint32_t* tmp_ids,
                     const float* tmp_dists, int* updated) {
    return guarded([&] {
        RankList a, t;
        for (std::uint32_t i = 0; i < kLaneWidth; ++i) {
            a.slot[i] = {rij_ids[i], rij_dists[i]};
            t.slot[i] = {tmp_ids[i], tmp_dists[i]};
        }
        *updated = merge_halves(a, t) ? 1 : 0;
        for (std::uint32_t i = 0; i < kLaneWidth; ++i) {
            rij_ids[i] = a.slot[i].id;
            rij_dists[i] = a.slot[i].dist;
        }
    });
}

// Replays an op sequence on SegmentedQueue + SegmentedVisited (segmented.cpp).
// op: 0 push(id,dist) if !contains, 1 pop_min, 2 visited.add(id), 3 visited.contains(id).
// out[i] per op: push -> 1 if pushed (precondition held) else 0; pop -> popped id
// (0xFFFFFFFF if empty); add -> 0; contains -> 0/1.  out_dist[i] = popped dist.
// Also records queue.size() after each op and the final eviction count.
int ref_segmented_replay(std::uint32_t m, const std::uint8_t* ops, const std::uint32_t* ids,
                         const float* dists, std::uint32_t n_ops, std::uint32_t* out,
                         float* out_dist, std::uint64_t* sizes, std::uint64_t* evictions) {
    return guarded([&] {
        SegmentedQueue q(m);
        SegmentedVisited v(m);
        for (std::uint32_t i = 0; i < n_ops; ++i) {
            out[i] = 0;
            out_dist[i] = 0.0f;
            switch (ops[i]) {
                case 0:
                    if (!q.contains(ids[i])) {
                        q.push(ids[i], dists[i]);
                        out[i] = 1;
                    }
                    break;
                case 1: {
                    const auto p = q.pop_min();
                    out[i] = p ? p->id : kInvalidId;
                    out_dist[i] = p ? p->dist : kInfDist;
                    break;
                }
                case 2:
                    v.add(ids[i]);
                    break;
                default:
                    out[i] = v.contains(ids[i]) ? 1 : 0;
                    break;
            }
            sizes[i] = q.size();
        }
        *evictions = q.evictions();
    });
}

// Replays push / pop_furthest on TopK(k) (segmented.cpp:89-111).
// op 0 push(id,dist) -> out 1/0; op 1 pop_furthest.  Final sorted contents out.
int ref_topk_replay(std::uint32_t k, const std::uint8_t* ops, const std::uint32_t* ids,
                    const float* dists, std::uint32_t n_ops, std::uint32_t* out,
                    std::uint32_t* final_ids, float* final_dists, std::uint32_t* final_n) {
    return guarded([&] {
        TopK t(k);
        for (std::uint32_t i = 0; i < n_ops; ++i) {
            if (ops[i] == 0) {
                out[i] = t.push(ids[i], dists[i]) ? 1 : 0;
            } else {
                t.pop_furthest();
                out[i] = 0;
            }
        }
        const auto& s = t.sorted_ascending();
        *final_n = static_cast<std::uint32_t>(s.size());
        for (std::size_t i = 0; i < s.size(); ++i) {
            final_ids[i] = s[i].id;
            final_dists[i] = s[i].dist;
        }
    });
}

// Exact top-k by (dist, id) (reference.cpp:96-111).
int ref_exact_topk(const float* base, std::uint32_t n, const float* queries,
                   std::uint32_t nq, std::uint32_t d, std::uint32_t k, int metric,
                   std::uint32_t* ids_out, float* dists_out) {
    return guarded([&] {
        const auto r = ref::exact_topk(make_set(base, n, d), make_set(queries, nq, d), k,
                                       static_cast<Metric>(metric));
        for (std::uint32_t q = 0; q < nq; ++q) {
            for (std::uint32_t i = 0; i < k; ++i) {
                const bool ok = i < r[q].size();
                ids_out[static_cast<std::size_t>(q) * k + i] = ok ? r[q][i].id : kInvalidId;
                dists_out[static_cast<std::size_t>(q) * k + i] = ok ? r[q][i].dist : kInfDist;
            }
        }
    });
}

// tsdg::brute_force_knn (knn_graph.cpp:64-86), unmodified; k_eff = clamped k.
int ref_brute_force_knn(const float* base, std::uint32_t n, std::uint32_t d, std::uint32_t k,
                        int metric, std::uint32_t* ids_out, float* dists_out,
                        std::uint32_t* k_eff) {
    return guarded([&] {
        const auto g = brute_force_knn(make_set(base, n, d), k, static_cast<Metric>(metric));
        *k_eff = g.k;
        for (std::size_t i = 0; i < g.flat.size(); ++i) {
            ids_out[i] = g.flat[i].id;
            dists_out[i] = g.flat[i].dist;
        }
    });
}

}  // extern "C"
