// C++ parity suite for the drop-in header include/tsdg/gpu_search.hpp, written
// like the reference's own tests (test_bestfirst.cpp, test_greedy.cpp,
// acceptance.cpp) and linked against the UNMODIFIED reference library
// (oracle/_ref, test infrastructure) so every case compares tsdg::gpu::* with
// the reference's tsdg::* on the same inputs.  Exit code = number of failures.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "tsdg/bench.hpp"
#include "tsdg/bestfirst_search.hpp"
#include "tsdg/greedy_search.hpp"
#include "tsdg/io.hpp"
#include "tsdg/knn_graph.hpp"
#include "tsdg/reference.hpp"
#include "tsdg/gpu_search.hpp"

using namespace tsdg;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                                  \
    do {                                                                          \
        ++g_checks;                                                               \
        if (!(c)) {                                                               \
            ++g_fail;                                                             \
            std::printf("  FAIL %s:%d  %s\n", __FILE__, __LINE__, #c);            \
        }                                                                         \
    } while (0)
#define CASE(name) std::printf("[case] %s\n", name)

static TsdgGraph complete_graph(const VectorSet& set, Metric metric) {
    // test_bestfirst.cpp:18-33
    const auto kernel = kernel_for(metric);
    std::vector<std::vector<TsdgEdge>> adjacency(set.n);
    for (NodeId u = 0; u < set.n; ++u) {
        for (NodeId v = 0; v < set.n; ++v) {
            if (v == u) continue;
            adjacency[u].push_back({v, 0, kernel(set.row(u), set.row(v), set.d)});
        }
        std::sort(adjacency[u].begin(), adjacency[u].end(), [](const TsdgEdge& a, const TsdgEdge& b) {
            if (a.dist != b.dist) return a.dist < b.dist;
            return a.target < b.target;
        });
    }
    return tsdg_from_adjacency(set.n, metric, set.n - 1, 1.0f, 0, adjacency);
}

int main() {
    {
        CASE("complete graph yields the exact top-k (test_bestfirst.cpp:39-62)");
        const auto set = make_synthetic(64, 8, 3, 0.3f, 51);
        const auto g = complete_graph(set, Metric::L2);
        const auto queries = make_synthetic(15, 8, 3, 0.3f, 52);
        const auto truth = ref::exact_topk(set, queries, 10, Metric::L2);
        BestFirstParams p;
        p.k = 10;
        p.hop_limit = 10000;
        p.delta = 1e30f;
        p.m_segments = 2;
        p.lambda_cut = 1;
        const auto ids = gpu::large_batch_search(g, set, queries, p);
        for (std::uint32_t q = 0; q < queries.n; ++q) {
            CHECK(ids[q].size() == 10);
            for (std::size_t i = 0; i < ids[q].size(); ++i) CHECK(ids[q][i] == truth[q][i].id);
        }
    }
    {
        CASE("large_batch_search == reference, ids + stats, parameter grid");
        auto [base, queries] = make_synthetic_split(3000, 300, 24, 10, 0.25f, 9);
        const auto knn = brute_force_knn(base, 30, Metric::L2);
        const auto g = build(base, knn, {1.2f, 9, 0}, Metric::L2);
        const gpu::Index index(g, base);
        for (std::uint32_t k : {1u, 10u, 32u, 64u}) {
            for (std::uint32_t m : {1u, 8u}) {
                for (float delta : {0.0f, 0.5f}) {
                    BestFirstParams p;
                    p.k = k;
                    p.m_segments = m;
                    p.delta = delta;
                    p.lambda_cut = 7;
                    p.seed = 11 + k;
                    SearchStats s_ref, s_gpu;
                    const auto want = large_batch_search(g, base, queries, p, &s_ref);
                    const auto got = index.large_batch_search(queries, p, &s_gpu);
                    CHECK(got == want);
                    CHECK(s_gpu.hops == s_ref.hops);
                    CHECK(s_gpu.distance_evals == s_ref.distance_evals);
                    CHECK(s_gpu.queue_evictions == s_ref.queue_evictions);
                    const auto fast = index.large_batch_search(queries, p, nullptr, gpu::Mode::Fast);
                    CHECK(fast.size() == want.size());
                }
            }
        }
        CASE("distances equal the reference kernel on the returned ids");
        BestFirstParams p;
        p.k = 16;
        const auto r = index.search_bestfirst(queries, p);
        const auto kernel = kernel_for(Metric::L2);
        for (std::uint32_t q = 0; q < queries.n; ++q)
            for (std::uint32_t i = 0; i < r.counts[q]; ++i) {
                const float want = kernel(queries.row(q), base.row(r.ids[q * p.k + i]), base.d);
                CHECK(std::memcmp(&want, &r.dists[q * p.k + i], 4) == 0);
            }
        CASE("small_batch_search == reference (greedy_search.cpp:106-127)");
        for (std::uint32_t t0 : {1u, 4u, 16u}) {
            GreedyParams gp;
            gp.t0 = t0;
            gp.seed = 77;
            SearchStats s_ref, s_gpu;
            const auto want = small_batch_search(g, base, queries, 10, gp, &s_ref);
            const auto got = index.small_batch_search(queries, 10, gp, &s_gpu);
            CHECK(got == want);
            CHECK(s_gpu.hops == s_ref.hops);
            CHECK(s_gpu.distance_evals == s_ref.distance_evals);
        }
        CASE("parameter validation throws std::invalid_argument (test_bestfirst.cpp:176-183)");
        BestFirstParams bad;
        bad.delta = -1.0f;
        bool threw = false;
        try {
            index.large_batch_search(queries, bad);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
        GreedyParams g1;
        g1.t0 = 1;
        threw = false;
        try {
            index.small_batch_search(queries, 33, g1);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
        VectorSet wrong = queries;
        wrong.d = 5;
        wrong.data.resize(static_cast<std::size_t>(wrong.n) * 5);
        threw = false;
        try {
            index.large_batch_search(wrong, BestFirstParams{});
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
    }
    {
        CASE("saved TSDG reloaded by the reference loader, searched on the GPU");
        auto [base, queries] = make_synthetic_split(2000, 100, 16, 8, 0.2f, 401);
        const auto g = build(base, brute_force_knn(base, 30, Metric::L2), {1.2f, 9, 0}, Metric::L2);
        save_tsdg(g, "/tmp/tsdg_gpu_api.tsdg");
        const auto g2 = load_tsdg("/tmp/tsdg_gpu_api.tsdg");
        BestFirstParams p;
        p.k = 10;
        p.seed = 5;
        CHECK(gpu::large_batch_search(g2, base, queries, p) == large_batch_search(g, base, queries, p));
        std::remove("/tmp/tsdg_gpu_api.tsdg");
    }
    {
        CASE("ground_truth / brute_force_knn / build == reference (bench.cpp, knn_graph.cpp, diversify.cpp)");
        auto [base, queries] = make_synthetic_split(3000, 120, 20, 6, 0.25f, 77);
        CHECK(gpu::ground_truth(base, queries, 50, Metric::L2) == ground_truth(base, queries, 50, Metric::L2));
        const auto knn_ref = brute_force_knn(base, 40, Metric::L2);
        const auto knn_gpu = gpu::brute_force_knn(base, 40, Metric::L2);
        CHECK(knn_gpu == knn_ref);
        for (const DiversifyParams dp : {DiversifyParams{1.2f, 9, 0}, DiversifyParams{1.0f, 4, 12}}) {
            BuildStats s_ref, s_gpu;
            const auto g_ref = build(base, knn_ref, dp, Metric::L2, &s_ref);
            const auto g_gpu = gpu::build(base, knn_gpu, dp, Metric::L2, &s_gpu);
            CHECK(g_gpu == g_ref);
            CHECK(s_gpu.stage1_edges == s_ref.stage1_edges && s_gpu.final_edges == s_ref.final_edges &&
                  s_gpu.augmented_edges == s_ref.augmented_edges);
        }
        const auto nnd = nn_descent(base, 24, Metric::L2, 4, 0.7, 3);
        CHECK(gpu::build(base, nnd, {1.2f, 9, 0}, Metric::L2) == build(base, nnd, {1.2f, 9, 0}, Metric::L2));
        bool threw = false;
        try {
            gpu::build(base, knn_gpu, {0.5f, 9, 0}, Metric::L2);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
    }
    {
        CASE("MultiIndex (replicated over a device list) == reference");
        auto [base, queries] = make_synthetic_split(2500, 150, 16, 8, 0.2f, 91);
        const auto g = build(base, brute_force_knn(base, 24, Metric::L2), {1.2f, 9, 0}, Metric::L2);
        const gpu::MultiIndex multi(g, base, {0, 0, 0});  // three replicas (one GPU here)
        BestFirstParams p;
        p.k = 12;
        p.seed = 4;
        SearchStats s_ref, s_gpu;
        CHECK(multi.large_batch_search(queries, p, &s_gpu) == large_batch_search(g, base, queries, p, &s_ref));
        CHECK(s_gpu.distance_evals == s_ref.distance_evals && s_gpu.hops == s_ref.hops);
        GreedyParams gp;
        gp.t0 = 4;
        gp.seed = 6;
        CHECK(multi.small_batch_search(queries, 10, gp) == small_batch_search(g, base, queries, 10, gp));
    }
    {
        CASE("ShardedIndex == per-shard reference searches merged by (dist, global id)");
        auto [base, queries] = make_synthetic_split(3000, 80, 12, 6, 0.25f, 57);
        const std::uint32_t half = 1400;
        std::vector<VectorSet> parts(2);
        std::vector<std::uint64_t> offs = {0, half};
        std::vector<std::string> paths = {"/tmp/tsdg_shard0.tsdg", "/tmp/tsdg_shard1.tsdg"};
        std::vector<TsdgGraph> gs;
        for (int s = 0; s < 2; ++s) {
            const std::uint32_t lo = s ? half : 0, hi = s ? base.n : half;
            parts[s].n = hi - lo;
            parts[s].d = base.d;
            parts[s].data.assign(base.data.begin() + (std::size_t)lo * base.d, base.data.begin() + (std::size_t)hi * base.d);
            gs.push_back(build(parts[s], brute_force_knn(parts[s], 20, Metric::L2), {1.2f, 9, 0}, Metric::L2));
            save_tsdg(gs.back(), paths[s]);
        }
        const gpu::ShardedIndex sharded(paths, parts, offs, {0, 0});
        BestFirstParams p;
        p.k = 8;
        p.seed = 13;
        const auto got = sharded.large_batch_search(queries, p);
        const auto kernel = kernel_for(Metric::L2);
        bool same = got.size() == queries.n;
        for (std::uint32_t q = 0; q < queries.n && same; ++q) {
            std::vector<IdDist> pool;
            for (int s = 0; s < 2; ++s) {
                // query q keeps its stream fork(q) on every shard
                const auto ids = bestfirst_search(gs[s], parts[s], std::span<const float>(queries.row(q), queries.d),
                                                  p, Rng64(p.seed).fork(q));
                for (NodeId id : ids)
                    pool.push_back({static_cast<NodeId>(id + offs[s]), kernel(queries.row(q), parts[s].row(id), base.d)});
            }
            std::sort(pool.begin(), pool.end(), [](const IdDist& a, const IdDist& b) { return closer(a, b); });
            std::vector<NodeId> want;
            for (std::size_t i = 0; i < pool.size() && i < p.k; ++i) want.push_back(pool[i].id);
            same = got[q] == want;
        }
        CHECK(same);
        std::remove(paths[0].c_str());
        std::remove(paths[1].c_str());
    }
    {
        CASE("Index(tsdg file, fvecs file) decoded on the device == load_tsdg + load_vectors");
        auto [base, queries] = make_synthetic_split(2500, 60, 20, 5, 0.25f, 91);
        const TsdgGraph g = build(base, brute_force_knn(base, 24, Metric::L2), {1.2f, 9, 0}, Metric::L2);
        const std::string gp = "/tmp/tsdg_files_case.tsdg", vp = "/tmp/tsdg_files_case.fvecs";
        save_tsdg(g, gp);
        write_fvecs(base, vp);
        const gpu::Index from_files(gp, vp);
        const gpu::Index from_memory(load_tsdg(gp), load_vectors(vp));
        BestFirstParams p;
        p.k = 12;
        p.seed = 4;
        SearchStats s_a, s_b;
        CHECK(from_files.large_batch_search(queries, p, &s_a) == large_batch_search(g, base, queries, p, &s_b));
        CHECK(s_a.distance_evals == s_b.distance_evals && s_a.hops == s_b.hops);
        GreedyParams gp2;
        gp2.t0 = 4;
        CHECK(from_files.small_batch_search(queries, 10, gp2) == from_memory.small_batch_search(queries, 10, gp2));
        bool threw = false;
        try {
            const gpu::Index bad(gp, "/tmp/tsdg_files_case_missing.fvecs");
        } catch (const std::runtime_error& e) {
            threw = std::string(e.what()).find("cannot open for reading") != std::string::npos;
        }
        CHECK(threw);
        std::remove(gp.c_str());
        std::remove(vp.c_str());
    }
    {
        CASE("nn_descent == reference KnnGraph (knn_graph.cpp:141-251)");
        auto [base, queries] = make_synthetic_split(2500, 10, 24, 7, 0.3f, 95);
        for (double rate : {0.5, 1.0}) {
            const KnnGraph want = nn_descent(base, 20, Metric::L2, 4, rate, 17);
            const KnnGraph got = gpu::nn_descent(base, 20, Metric::L2, 4, rate, 17);
            CHECK(got == want);
        }
        bool threw = false;
        try {
            gpu::nn_descent(base, 20, Metric::L2, 4, 0.0, 17);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
    }
    {
        CASE("reference-signature free functions reuse one resident index (no re-upload per call)");
        auto [base, queries] = make_synthetic_split(3000, 80, 16, 6, 0.25f, 93);
        const TsdgGraph g = build(base, brute_force_knn(base, 20, Metric::L2), {1.2f, 9, 0}, Metric::L2);
        BestFirstParams p;
        p.k = 10;
        p.seed = 7;
        GreedyParams gp;
        gp.t0 = 4;
        const auto want_bf = large_batch_search(g, base, queries, p);
        const auto want_gr = small_batch_search(g, base, queries, 10, gp);
        const std::uint64_t before = gpu::index_uploads();
        for (int rep = 0; rep < 5; ++rep) {  // bench.cpp:329,333 call once per chunk
            CHECK(gpu::large_batch_search(g, base, queries, p) == want_bf);
            CHECK(gpu::small_batch_search(g, base, queries, 10, gp) == want_gr);
        }
        CHECK(gpu::index_uploads() == before + 1);
        // a different base (same graph object) is a different index
        VectorSet other = base;
        CHECK(gpu::large_batch_search(g, other, queries, p) == want_bf);
        CHECK(gpu::index_uploads() == before + 2);
        gpu::release_resident_indexes();
        CHECK(gpu::large_batch_search(g, base, queries, p) == want_bf);
        CHECK(gpu::index_uploads() == before + 3);
        gpu::release_resident_indexes();
    }
    std::printf("gpu_api: %d/%d checks passed\n", g_checks - g_fail, g_checks);
    return g_fail;
}
