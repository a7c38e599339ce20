"""GPU parity: the sm_100a kernels through the C-ABI against the CPU oracle
(oracle/tsdg_oracle.c, itself pinned to the reference) and the reference's
golden outputs.  Deterministic mode must be bit-exact: ids, fp32 distances,
counts and per-query hops / distance_evals / queue_evictions."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2204_00824_b200 import datasets, search
from paper_2204_00824_b200.search import BestFirstParams, GreedyParams, InvalidArgument

pytestmark = pytest.mark.gpu
FIXTURES = ["syn2k", "lowlid3k"]


@pytest.fixture(scope="module")
def orc():
    return O.Oracle()


@pytest.fixture(scope="module")
def index(fixtures):
    cache = {}

    def get(name):
        if name not in cache:
            g, b, q = fixtures(name)
            cache[name] = search.GpuIndex(search.load_tsdg(f"tests/golden/{name}.tsdg"), b)
        return cache[name]

    return get


def assert_same(gpu: search.SearchResult, want: O.Result, check_stats=True):
    np.testing.assert_array_equal(gpu.ids, want.ids)
    np.testing.assert_array_equal(gpu.counts, want.counts)
    np.testing.assert_array_equal(gpu.dists.view(np.uint32), want.dists.view(np.uint32))
    if check_stats:
        np.testing.assert_array_equal(gpu.stats["hops"], want.stats[:, 0])
        np.testing.assert_array_equal(gpu.stats["distance_evals"], want.stats[:, 1])
        np.testing.assert_array_equal(gpu.stats["queue_evictions"], want.stats[:, 2])


@pytest.mark.parametrize("name", FIXTURES)
def test_bestfirst_bit_exact_grid(orc, fixtures, index, golden, golden_meta, name):
    g, b, q = fixtures(name)
    idx = index(name)
    for i, pd in enumerate(golden_meta["bf_grid"]):
        p = BestFirstParams(**pd)
        got = idx.search_bestfirst(q, p)
        assert_same(got, orc.large_batch(g, b, q, p))
        np.testing.assert_array_equal(got.ids, golden[f"{name}_bf{i}_ids"])  # the reference itself
        np.testing.assert_array_equal(got.stats["edges_examined"],
                                      golden[f"{name}_bf{i}_trace"][:, 1])


@pytest.mark.parametrize("name", FIXTURES)
def test_bestfirst_random_params(orc, fixtures, index, name):
    g, b, q = fixtures(name)
    idx = index(name)
    rng = np.random.default_rng(123)
    for _ in range(6):
        p = BestFirstParams(k=int(rng.integers(1, 80)), hop_limit=int(rng.integers(1, 400)),
                            delta=float(rng.choice([0.0, 0.1, 1.0, 1e30])),
                            m_segments=int(rng.integers(1, 33)), lambda_cut=int(rng.integers(1, 12)),
                            seed=int(rng.integers(0, 2**63)))
        assert_same(idx.search_bestfirst(q, p), orc.large_batch(g, b, q, p))


@pytest.mark.parametrize("name", FIXTURES)
def test_bestfirst_maximum_k(orc, fixtures, index, name):
    """The largest result sizes the GPU path accepts (k up to 1024, R in shared
    memory) with heavy queue overflow (m = 1 / 8 / 32): still bit-exact, counters
    included (queue_evictions large)."""
    g, b, q = fixtures(name)
    idx = index(name)
    q = q[:48]
    evictions = 0
    for k, m, cut in ((128, 8, 10), (512, 32, 12), (1024, 32, 12), (300, 1, 5)):
        p = BestFirstParams(k=k, m_segments=m, lambda_cut=cut, seed=k + m)
        got, want = idx.search_bestfirst(q, p), orc.large_batch(g, b, q, p)
        assert_same(got, want)
        evictions += int(want.stats[:, 2].sum())
    assert evictions > 0
    with pytest.raises(InvalidArgument):
        idx.search_bestfirst(q, BestFirstParams(k=1025))


@pytest.mark.parametrize("name", FIXTURES)
def test_greedy_maximum_t0_and_k(orc, fixtures, index, name):
    """Alg. 1 at the GPU path's limits: t0 = 256 walks (global-memory pool + merge
    kernel) with k up to 32 * t0, and t0 = 16 / 17 on both sides of the cluster
    limit; bit-exact ids, distances, counts and counters."""
    g, b, q = fixtures(name)
    idx = index(name)
    q = q[:16]
    for t0, k, T, cut in ((256, 2000, 16, 10), (256, 8192, 4, 3), (17, 100, 16, 10),
                          (16, 512, 16, 10)):
        p = GreedyParams(t0=t0, hop_limit=T, lambda_cut=cut, seed=t0 * 7 + k)
        got, want = idx.search_greedy(q, k, p), orc.small_batch(g, b, q, k, p)
        assert_same(got, want)
    with pytest.raises(InvalidArgument):
        idx.search_greedy(q, 10, GreedyParams(t0=257))


def test_bestfirst_query_index_base_split(orc, fixtures, index):
    g, b, q = fixtures("syn2k")
    idx = index("syn2k")
    p = BestFirstParams(k=10, seed=21)
    whole = idx.search_bestfirst(q, p)
    a = idx.search_bestfirst(q[:77], p, query_index_base=0)
    c = idx.search_bestfirst(q[77:], p, query_index_base=77)
    np.testing.assert_array_equal(np.concatenate([a.ids, c.ids]), whole.ids)


@pytest.mark.parametrize("name", FIXTURES)
def test_greedy_bit_exact_grid(orc, fixtures, index, golden, golden_meta, name):
    g, b, q = fixtures(name)
    idx = index(name)
    for i, gd in enumerate(golden_meta["gr_grid"]):
        p = GreedyParams(**{k: v for k, v in gd.items() if k != "k"})
        got = idx.search_greedy(q, gd["k"], p)
        want = orc.small_batch(g, b, q, gd["k"], p)
        np.testing.assert_array_equal(got.ids, want.ids)
        np.testing.assert_array_equal(got.counts, want.counts)
        np.testing.assert_array_equal(got.dists.view(np.uint32), want.dists.view(np.uint32))
        np.testing.assert_array_equal(got.stats["hops"], want.stats[:, 0])
        np.testing.assert_array_equal(got.stats["distance_evals"], want.stats[:, 1])
        np.testing.assert_array_equal(got.ids, golden[f"{name}_gr{i}_ids"])


@pytest.mark.parametrize("name", FIXTURES)
def test_greedy_once_slots(fixtures, index, golden, name):
    g, b, q = fixtures(name)
    idx = index(name)
    ids, dists, st = idx.greedy_search_once(q[:20], np.arange(100, 120, dtype=np.uint64), 16, 10)
    np.testing.assert_array_equal(ids, golden[f"{name}_once_ids"])
    np.testing.assert_array_equal(dists.view(np.uint32), golden[f"{name}_once_dists"].view(np.uint32))
    np.testing.assert_array_equal(st["hops"], golden[f"{name}_once_stats"][:, 0])
    np.testing.assert_array_equal(st["distance_evals"], golden[f"{name}_once_stats"][:, 1])


def test_complete_graph_exact_both_procedures(golden, golden_meta):
    spec = golden_meta["fixtures"]["complete96"]["spec"]
    b, q = datasets.make_synthetic_split(spec["n"], spec["nq"], spec["d"], spec["clusters"],
                                         spec["spread"], spec["seed"])
    idx = search.GpuIndex.from_file("tests/golden/complete96.tsdg", b)
    exact = golden["complete96_exact_ids"]
    p = BestFirstParams(k=10, hop_limit=10000, delta=1e30, m_segments=4, lambda_cut=1, seed=42)
    np.testing.assert_array_equal(idx.search_bestfirst(q, p).ids, exact)
    r = idx.search_greedy(q, 10, GreedyParams(t0=16, hop_limit=8, lambda_cut=1, seed=42))
    np.testing.assert_array_equal(r.ids, exact)
    np.testing.assert_array_equal(r.dists, golden["complete96_exact_dists"])


def test_hop_limit_one(fixtures, index):
    g, b, q = fixtures("syn2k")
    r = index("syn2k").search_bestfirst(q[:10], BestFirstParams(hop_limit=1))
    assert (r.stats["hops"] == 1).all()
    r = index("syn2k").search_greedy(q[:10], 10, GreedyParams(t0=1, hop_limit=1))
    assert (r.stats["hops"] == 1).all()


def test_deg_cut_matches_prefix(index):
    idx = index("syn2k")
    g = idx.graph
    for cut in (1, 3, 5, 10, 100):
        dc = idx.deg_cut(cut)
        want = [len(g.neighbors_below(u, cut)) for u in range(g.n)]
        np.testing.assert_array_equal(dc, want)


def test_validation_errors(index, fixtures):
    g, b, q = fixtures("syn2k")
    idx = index("syn2k")
    for bad in (BestFirstParams(delta=-1.0), BestFirstParams(k=0), BestFirstParams(hop_limit=0),
                BestFirstParams(m_segments=0), BestFirstParams(lambda_cut=0)):
        with pytest.raises(InvalidArgument):
            idx.search_bestfirst(q[:2], bad)
    with pytest.raises(InvalidArgument):
        idx.search_greedy(q[:2], 33, GreedyParams(t0=1))
    with pytest.raises(InvalidArgument):
        idx.search_greedy(q[:2], 0, GreedyParams())
    with pytest.raises(InvalidArgument):
        idx.search_bestfirst(np.zeros((2, 5), np.float32), BestFirstParams())


def test_empty_batch(index):
    r = index("syn2k").search_bestfirst(np.zeros((0, 32), np.float32), BestFirstParams())
    assert r.ids.shape == (0, 10)


def test_merge_shards_kernel():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(5)
    S, nq, k = 4, 50, 10
    ids = np.zeros((S, nq, k), np.uint32)
    dists = np.full((S, nq, k), np.inf, np.float32)
    counts = rng.integers(0, k + 1, size=(S, nq)).astype(np.uint32)
    base = np.array([0, 1000, 2000, 3000], np.uint64)
    for s in range(S):
        for qq in range(nq):
            c = counts[s, qq]
            loc = rng.choice(1000, size=c, replace=False).astype(np.uint32)
            dd = (rng.integers(0, 50, size=c) / 4).astype(np.float32)
            order = np.lexsort((loc, dd))
            ids[s, qq, :c], dists[s, qq, :c] = loc[order], dd[order]
    dev = torch.device("cuda:0")
    ti, td, tc = (torch.from_numpy(x).to(dev) for x in (ids.view(np.int32), dists, counts.view(np.int32)))
    oi = torch.empty((nq, k), dtype=torch.int32, device=dev)
    od = torch.empty((nq, k), dtype=torch.float32, device=dev)
    oc = torch.empty(nq, dtype=torch.int32, device=dev)
    search.merge_shards_device(ti.data_ptr(), td.data_ptr(), tc.data_ptr(), base, S, nq, k,
                               oi.data_ptr(), od.data_ptr(), oc.data_ptr(),
                               torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    gi = oi.cpu().numpy().view(np.uint32)
    for qq in range(nq):
        cand = [(dists[s, qq, j], int(base[s]) + int(ids[s, qq, j]))
                for s in range(S) for j in range(counts[s, qq])]
        cand.sort()
        want = [c[1] for c in cand[:k]]
        assert oc[qq].item() == len(want)
        assert gi[qq, :len(want)].tolist() == want


DATA = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "data")


@pytest.mark.skipif(not datasets.available("c1_lowlid_100k"), reason="data/c1_lowlid_100k absent")
def test_c1_parity_and_recall(orc):
    ds = datasets.load("c1_lowlid_100k")
    g = O.parse_tsdg(ds.graph_path)
    idx = search.GpuIndex.from_file(ds.graph_path, ds.base)
    q = ds.queries[:1000]
    for p in (BestFirstParams(k=10, seed=7), BestFirstParams(k=32, seed=7, m_segments=16),
              BestFirstParams(k=64, seed=3, m_segments=8, lambda_cut=10)):
        got = idx.search_bestfirst(q, p)
        assert_same(got, orc.large_batch(g, ds.base, q, p))
    p = BestFirstParams(k=32, seed=7)
    got = idx.search_bestfirst(q, p)
    assert O.recall_at_k(got.ids, got.counts, ds.gt, 10) >= 0.95
    gp = GreedyParams(t0=8, seed=7)
    gr = idx.search_greedy(q[:200], 10, gp)
    want = orc.small_batch(g, ds.base, q[:200], 10, gp)
    np.testing.assert_array_equal(gr.ids, want.ids)


@pytest.mark.skipif(not datasets.available("c2_lowlid_1m"), reason="data/c2_lowlid_1m absent")
def test_c2_full_size_properties(orc):
    ds = datasets.load("c2_lowlid_1m")
    idx = search.GpuIndex.from_file(ds.graph_path, ds.base)
    p = BestFirstParams(k=32, seed=7)
    r = idx.search_bestfirst(ds.queries, p)
    # sortedness by (dist, id), recomputed distances, recall
    assert (np.diff(r.dists, axis=1) >= 0).all()
    for qq in range(0, ds.queries.shape[0], 997):
        for j in range(int(r.counts[qq])):
            assert r.dists[qq, j] == orc.distance(ds.queries[qq], ds.base[r.ids[qq, j]])
    assert O.recall_at_k(r.ids, r.counts, ds.gt, 10) >= 0.95
    # bit-exact subset vs the oracle
    g = O.parse_tsdg(ds.graph_path)
    sub = orc.large_batch(g, ds.base, ds.queries[:300], p)
    assert_same(idx.search_bestfirst(ds.queries[:300], p), sub)


@pytest.mark.parametrize("stage", ["ldgsts", "tma"])
@pytest.mark.parametrize("prefetch", ["0", "3"])
def test_staging_paths_bit_exact(orc, fixtures, index, golden_meta, monkeypatch, stage, prefetch):
    monkeypatch.setenv("TSDG_STAGE", stage)
    monkeypatch.setenv("TSDG_PREFETCH", prefetch)
    for name in FIXTURES:
        g, b, q = fixtures(name)
        idx = index(name)
        for pd in golden_meta["bf_grid"][:4]:
            p = BestFirstParams(**pd)
            assert_same(idx.search_bestfirst(q, p), orc.large_batch(g, b, q, p))
        gp = GreedyParams(t0=4, seed=5)
        np.testing.assert_array_equal(idx.search_greedy(q, 10, gp).ids,
                                      orc.small_batch(g, b, q, 10, gp).ids)


def test_fast_mode_recall_within_half_point(fixtures, index, golden, golden_meta):
    from paper_2204_00824_b200 import _native
    for name in FIXTURES:
        g, b, q = fixtures(name)
        idx = index(name)
        gt = golden[f"{name}_gt"]
        for i, pd in enumerate(golden_meta["bf_grid"][:3]):
            p = BestFirstParams(**pd)
            ref_ids = golden[f"{name}_bf{i}_ids"]
            ref_cnt = golden[f"{name}_bf{i}_counts"]
            fast = idx.search_bestfirst(q, p, mode=_native.MODE_FAST)
            r_ref = O.recall_at_k(ref_ids, ref_cnt, gt, min(10, p.k))
            r_fast = O.recall_at_k(fast.ids, fast.counts, gt, min(10, p.k))
            assert abs(r_fast - r_ref) <= 0.005, (name, i, r_fast, r_ref)
        gd = golden_meta["gr_grid"][0]  # the params golden gr0 was produced with
        gp = GreedyParams(**{kk: v for kk, v in gd.items() if kk != "k"})
        fg = idx.search_greedy(q, gd["k"], gp, mode=_native.MODE_FAST)
        for kk in (1, 10):  # north star: recall@1 / @10 within 0.5 pt
            r_ref = O.recall_at_k(golden[f"{name}_gr0_ids"], golden[f"{name}_gr0_counts"], gt, kk)
            assert abs(O.recall_at_k(fg.ids, fg.counts, gt, kk) - r_ref) <= 0.005, (name, kk)


@pytest.mark.skipif(not datasets.available("c1_lowlid_100k"), reason="data/c1_lowlid_100k absent")
def test_c1_fast_mode_recall(orc):
    from paper_2204_00824_b200 import _native
    ds = datasets.load("c1_lowlid_100k")
    idx = search.GpuIndex.from_file(ds.graph_path, ds.base)
    for k in (10, 16, 32):
        p = BestFirstParams(k=k, seed=7)
        det = idx.search_bestfirst(ds.queries, p)
        fast = idx.search_bestfirst(ds.queries, p, mode=_native.MODE_FAST)
        rd = O.recall_at_k(det.ids, det.counts, ds.gt, 10)
        rf = O.recall_at_k(fast.ids, fast.counts, ds.gt, 10)
        assert abs(rf - rd) <= 0.005, (k, rf, rd)
        rel = np.abs(fast.dists[:, :1] - det.dists[:, :1]) / np.maximum(det.dists[:, :1], 1e-30)
        assert np.nanmax(rel) < 1e-4


@pytest.mark.parametrize("kernel", ["cta", "warp"])
def test_greedy_kernels_bit_exact(orc, fixtures, index, golden, golden_meta, monkeypatch, kernel):
    """Both Alg. 1 kernels (CTA/cluster-per-query and warp-per-walk) reproduce the
    reference, including t0 > 16 (no cluster: walks merged by greedy_merge_kernel)."""
    monkeypatch.setenv("TSDG_GREEDY", kernel)
    for name in FIXTURES:
        g, b, q = fixtures(name)
        idx = index(name)
        for i, gd in enumerate(golden_meta["gr_grid"]):
            p = GreedyParams(**{k: v for k, v in gd.items() if k != "k"})
            got = idx.search_greedy(q[:64], gd["k"], p)
            np.testing.assert_array_equal(got.ids, golden[f"{name}_gr{i}_ids"][:64])
            np.testing.assert_array_equal(got.stats["hops"], golden[f"{name}_gr{i}_stats"][:64, 0])
            np.testing.assert_array_equal(got.stats["distance_evals"],
                                          golden[f"{name}_gr{i}_stats"][:64, 1])
        for t0 in (8, 24):
            p = GreedyParams(t0=t0, seed=3)
            got = idx.search_greedy(q[:16], 10, p)
            want = orc.small_batch(g, b, q[:16], 10, p)
            np.testing.assert_array_equal(got.ids, want.ids)
            np.testing.assert_array_equal(got.dists.view(np.uint32), want.dists.view(np.uint32))


@pytest.mark.parametrize("merge_warp,early,stage,extra", [
    ("0", "0", "tma", {}), ("0", "1", "ldgsts", {}), ("1", "0", "tma", {}), ("1", "1", "tma", {}),
    ("1", "1", "ldgsts", {}), ("1", "0", "ldgsts", {}),
    ("1", "1", "tma", {"TSDG_GC_SLICE": "16"}), ("1", "1", "tma", {"TSDG_GC_ADJ_PREFETCH": "1"}),
    ("0", "0", "g4", {}), ("1", "0", "g4", {}), ("1", "1", "g4", {}),
    ("1", "1", "g4", {"TSDG_GC_SLICE": "16"}), ("1", "1", "g4", {"TSDG_GC_SPEC": "0"}),
    ("1", "1", "tma", {"TSDG_GC_SPEC": "0"}), ("1", "1", "g4", {"TSDG_GC_COMPACT": "1"}),
    ("1", "1", "tma", {"TSDG_GC_COMPACT": "1"}), ("1", "0", "g4", {"TSDG_GC_COMPACT": "1"})])
def test_greedy_cluster_kernel_variants_bit_exact(orc, fixtures, index, golden, golden_meta, monkeypatch,
                                                  merge_warp, early, stage, extra):
    """The greedy cluster kernel's internal variants — warp 0 merging while warps 1-3
    gather (TSDG_GC_MERGE_WARP), the early next-node pick (TSDG_GC_EARLY), row
    staging by TMA bulk copies, TMA tile::gather4 tensor copies or cp.async
    (TSDG_GC_STAGE) — all reproduce the reference."""
    monkeypatch.setenv("TSDG_GREEDY", "cta")
    monkeypatch.setenv("TSDG_GC_MERGE_WARP", merge_warp)
    monkeypatch.setenv("TSDG_GC_EARLY", early)
    monkeypatch.setenv("TSDG_GC_STAGE", stage)
    for k, v in extra.items():
        monkeypatch.setenv(k, v)
    for name in FIXTURES:
        g, b, q = fixtures(name)
        idx = index(name)
        for i, gd in enumerate(golden_meta["gr_grid"]):
            p = GreedyParams(**{k: v for k, v in gd.items() if k != "k"})
            got = idx.search_greedy(q[:48], gd["k"], p)
            np.testing.assert_array_equal(got.ids, golden[f"{name}_gr{i}_ids"][:48])
            np.testing.assert_array_equal(got.stats["hops"], golden[f"{name}_gr{i}_stats"][:48, 0])
            np.testing.assert_array_equal(got.stats["distance_evals"], golden[f"{name}_gr{i}_stats"][:48, 1])
        p = GreedyParams(t0=12, hop_limit=3, seed=9)  # hop limit reached mid-walk
        want = orc.small_batch(g, b, q[:24], 10, p)
        got = idx.search_greedy(q[:24], 10, p)
        np.testing.assert_array_equal(got.ids, want.ids)
        np.testing.assert_array_equal(got.dists.view(np.uint32), want.dists.view(np.uint32))
