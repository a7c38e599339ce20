"""Search kernels under the non-L2 metrics (vectors.cpp:10-16: inner product = -dot,
cosine = 1 - dot on unit rows) and the reference tests' monotonicity properties
(test_greedy.cpp:264-305 t0 nesting / recall, test_bestfirst.cpp:76-101 Delta), all
through the C-ABI on the GPU and checked against the oracle (tests only)."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2204_00824_b200 import _native, datasets

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def index(fixtures):
    from paper_2204_00824_b200 import search
    cache = {}

    def get(name):
        if name not in cache:
            _, b, _ = fixtures(name)
            cache[name] = search.GpuIndex(search.load_tsdg(os.path.join(GOLDEN, f"{name}.tsdg")), b)
        return cache[name]

    return get


def _same(got, want):
    np.testing.assert_array_equal(got.ids, want.ids)
    np.testing.assert_array_equal(got.dists.view(np.uint32), want.dists.view(np.uint32))
    np.testing.assert_array_equal(got.counts, want.counts)


def test_inner_product_graph_search_bit_exact():
    from paper_2204_00824_b200 import search
    with open(os.path.join(GOLDEN, "scan.json")) as f:
        spec = json.load(f)["specs"]["b"]
    base, queries = datasets.generate(spec)
    path = os.path.join(GOLDEN, "build_ip_b.tsdg")  # reference build, metric 2
    g = O.parse_tsdg(path)
    assert g.metric == 2
    idx = search.GpuIndex.from_file(path, base)
    orc = O.Oracle()
    for p in (search.BestFirstParams(k=10, seed=3), search.BestFirstParams(k=40, seed=4, m_segments=5)):
        _same(idx.search_bestfirst(queries, p), orc.large_batch(g, base, queries, p))
    gp = search.GreedyParams(t0=4, seed=9)
    got = idx.search_greedy(queries, 10, gp)
    _same(got, orc.small_batch(g, base, queries, 10, gp))


def test_cosine_graph_search_bit_exact(tmp_path):
    from paper_2204_00824_b200 import bench_runner, search
    base, queries = datasets.make_synthetic_split(1500, 60, 24, 6, 0.3, 13)
    base, queries = bench_runner.normalized_copy(base), bench_runner.normalized_copy(queries)
    knn = search.brute_force_knn(base, 20, metric=1)
    path = str(tmp_path / "cos.tsdg")
    search.build(base, knn, 1.2, 9, 0, metric=1, save_path=path)
    g = O.parse_tsdg(path)
    idx = search.GpuIndex.from_file(path, base)
    orc = O.Oracle()
    p = search.BestFirstParams(k=12, seed=5)
    _same(idx.search_bestfirst(queries, p), orc.large_batch(g, base, queries, p))
    gp = search.GreedyParams(t0=3, seed=2)
    _same(idx.search_greedy(queries, 8, gp), orc.small_batch(g, base, queries, 8, gp))
    # fast mode: recall within the north-star tolerance of the deterministic result
    gt = search.ground_truth(base, queries, 10, metric=1).ids
    det = idx.search_bestfirst(queries, p)
    fast = idx.search_bestfirst(queries, p, mode=_native.MODE_FAST)
    assert abs(O.recall_at_k(fast.ids, fast.counts, gt, 10) -
               O.recall_at_k(det.ids, det.counts, gt, 10)) <= 0.005


def test_greedy_t0_nesting_and_monotone_recall(fixtures, index):
    """test_greedy.cpp:264-305: walks s < t0 are the same for every t0 (streams
    fork(s)), so the t0=4 pool is contained in the t0=8 pool and recall cannot drop."""
    from paper_2204_00824_b200 import search
    g, b, q = fixtures("lowlid3k")
    idx = index("lowlid3k")
    gt = search.ground_truth(b, q, 10).ids
    rec = []
    for t0 in (1, 2, 4, 8, 16):
        r = idx.search_greedy(q, 10, search.GreedyParams(t0=t0, seed=7))
        rec.append(O.recall_at_k(r.ids, r.counts, gt, 10))
    assert all(a <= b + 1e-12 for a, b in zip(rec, rec[1:])), rec
    # the merged top-k of more walks is never farther, query by query
    r4 = idx.search_greedy(q, 10, search.GreedyParams(t0=4, seed=7))
    r8 = idx.search_greedy(q, 10, search.GreedyParams(t0=8, seed=7))
    assert (r8.dists[:, 0] <= r4.dists[:, 0]).all()


def test_bestfirst_delta_monotone(fixtures, index):
    """test_bestfirst.cpp:76-101: a larger Delta only continues the search longer
    (with no queue evictions the expansions nest), so hops never decrease and the
    best distance never gets worse."""
    from paper_2204_00824_b200 import search
    g, b, q = fixtures("lowlid3k")
    idx = index("lowlid3k")
    prev = None
    for delta in (0.0, 0.05, 0.5, 1e30):
        r = idx.search_bestfirst(q, search.BestFirstParams(k=10, seed=3, delta=delta, m_segments=16))
        if prev is not None:
            ok = (prev.stats["queue_evictions"] == 0) & (r.stats["queue_evictions"] == 0)
            assert (r.stats["hops"][ok] >= prev.stats["hops"][ok]).all()
            assert (r.dists[ok, 0] <= prev.dists[ok, 0]).all()
        prev = r


@pytest.mark.parametrize("d", [30, 200])
def test_odd_and_wide_rows_bit_exact(tmp_path, d):
    """Rows that are not a multiple of 4 floats (zero-padded to 16 bytes in HBM) and
    rows wider than one 128-float staging chunk (dimension-chunked gathers, the C4
    shape) through both procedures, deterministic mode, against the oracle."""
    from paper_2204_00824_b200 import search
    base, queries = datasets.make_lowlid(2500, 60, d, 6, 10, 0.25, 31 + d, 0.01)
    knn = search.brute_force_knn(base, 24)
    path = str(tmp_path / f"g{d}.tsdg")
    search.build(base, knn, 1.2, 9, 0, save_path=path)
    g = O.parse_tsdg(path)
    idx = search.GpuIndex.from_file(path, base)
    orc = O.Oracle()
    for p in (search.BestFirstParams(k=10, seed=1), search.BestFirstParams(k=40, seed=2, m_segments=3)):
        _same(idx.search_bestfirst(queries, p), orc.large_batch(g, base, queries, p))
        fast = idx.search_bestfirst(queries, p, mode=_native.MODE_FAST)
        assert (fast.ids[:, 0] == orc.large_batch(g, base, queries, p).ids[:, 0]).mean() > 0.95
    for kern in ("cta", "warp"):
        os.environ["TSDG_GREEDY"] = kern
        try:
            gp = search.GreedyParams(t0=4, seed=3)
            _same(idx.search_greedy(queries, 10, gp), orc.small_batch(g, base, queries, 10, gp))
        finally:
            os.environ.pop("TSDG_GREEDY", None)


def test_results_independent_of_launch_shape(fixtures, index, monkeypatch):
    """acceptance.cpp:376-425 (identical across OpenMP worker counts): the GPU result
    does not depend on warps per CTA, staging slots, staging path or work order."""
    from paper_2204_00824_b200 import search
    g, b, q = fixtures("lowlid3k")
    idx = index("lowlid3k")
    p = search.BestFirstParams(k=24, seed=11, m_segments=8)
    want = idx.search_bestfirst(q, p)
    for env in ({"TSDG_BF_WARPS": "4"}, {"TSDG_BF_WARPS": "2", "TSDG_SLOTS": "8"},
                {"TSDG_SLOTS": "32"}, {"TSDG_STAGE": "ldgsts", "TSDG_SLOTS": "24"}):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        got = idx.search_bestfirst(q, p)
        _same(got, want)
        np.testing.assert_array_equal(got.stats, want.stats)
        for k in env:
            monkeypatch.delenv(k)
    # a batch split into uneven pieces with their query_index_base gives the same
    parts = [idx.search_bestfirst(q[a:c], p, query_index_base=a) for a, c in ((0, 1), (1, 90), (90, 200))]
    np.testing.assert_array_equal(np.concatenate([r.ids for r in parts]), want.ids)


def test_multi_device_index_equals_single(fixtures, index):
    """tsdg_gpu_multi (replicated over a device list; here three replicas on one GPU):
    each slice keeps its query_index_base, so results equal the single index's."""
    from paper_2204_00824_b200 import search
    g, b, q = fixtures("lowlid3k")
    idx = index("lowlid3k")
    multi = search.MultiGpuIndex(search.load_tsdg(os.path.join(GOLDEN, "lowlid3k.tsdg")), b,
                                 devices=(0, 0, 0))
    p = search.BestFirstParams(k=16, seed=9)
    for mode in (_native.MODE_DETERMINISTIC, _native.MODE_FAST):
        want = idx.search_bestfirst(q, p, mode=mode, query_index_base=5)
        got = multi.search_bestfirst(q, p, mode=mode, query_index_base=5)
        _same(got, want)
        np.testing.assert_array_equal(got.stats, want.stats)
    gp = search.GreedyParams(t0=6, seed=2)
    _same(multi.search_greedy(q, 10, gp), idx.search_greedy(q, 10, gp))
    _same(multi.search_bestfirst(q[:2], p), idx.search_bestfirst(q[:2], p))  # fewer queries than devices
    multi.close()


def test_zero_copy_host_path_equals_copy_pipeline(fixtures, index, monkeypatch):
    """Pinned host buffers take the zero-copy path (the kernel reads queries from and
    writes results to mapped host memory); pageable ones the copy pipeline.  Both
    equal the device-pointer search, ids, distances, counts and counters."""
    import ctypes
    import torch
    from paper_2204_00824_b200.search import BestFirstParams
    g, b, q = fixtures("lowlid3k")
    idx = index("lowlid3k")
    p = BestFirstParams(k=12, seed=9)
    want = idx.search_bestfirst(q, p)  # pageable numpy buffers: copy pipeline
    nq, k = q.shape[0], p.k
    hq = torch.from_numpy(np.ascontiguousarray(q)).pin_memory()
    hi = torch.empty((nq, k), dtype=torch.int32).pin_memory()
    hd = torch.empty((nq, k), dtype=torch.float32).pin_memory()
    hc = torch.empty(nq, dtype=torch.int32).pin_memory()
    hs = torch.empty((nq, 4), dtype=torch.int32).pin_memory()
    pc = p.c()
    L = _native.lib()
    for zc in ("1", "0"):
        monkeypatch.setenv("TSDG_ZERO_COPY", zc)
        hi.fill_(-7)
        _native.check(L.tsdg_gpu_search_bestfirst(
            idx.handle, ctypes.c_void_p(hq.data_ptr()), nq, 0, ctypes.byref(pc), _native.MODE_DETERMINISTIC,
            ctypes.c_void_p(hi.data_ptr()), ctypes.c_void_p(hd.data_ptr()), ctypes.c_void_p(hc.data_ptr()),
            ctypes.c_void_p(hs.data_ptr())))
        np.testing.assert_array_equal(hi.numpy().view(np.uint32), want.ids)
        np.testing.assert_array_equal(hd.numpy().view(np.uint32), want.dists.view(np.uint32))
        np.testing.assert_array_equal(hc.numpy().view(np.uint32), want.counts)
        np.testing.assert_array_equal(hs.numpy()[:, 1].view(np.uint32), want.stats["distance_evals"])


def test_zero_copy_greedy_equals_copy_path(fixtures, index, monkeypatch):
    """Small batch through the host-pointer call: pinned buffers (zero-copy) and
    pageable buffers give identical results, for the cluster and the warp kernel."""
    import ctypes
    import torch
    from paper_2204_00824_b200.search import GreedyParams
    _, _, q = fixtures("lowlid3k")
    idx = index("lowlid3k")
    L = _native.lib()
    for nq, t0 in ((1, 16), (8, 8), (200, 16)):
        qq = np.ascontiguousarray(q[:nq])
        p = GreedyParams(t0=t0, seed=3)
        want = idx.search_greedy(qq, 10, p)
        hq = torch.from_numpy(qq).pin_memory()
        hi = torch.full((nq, 10), -7, dtype=torch.int32).pin_memory()
        hd = torch.empty((nq, 10), dtype=torch.float32).pin_memory()
        hc = torch.empty(nq, dtype=torch.int32).pin_memory()
        pc = p.c()
        _native.check(L.tsdg_gpu_search_greedy(
            idx.handle, ctypes.c_void_p(hq.data_ptr()), nq, 10, ctypes.byref(pc), _native.MODE_DETERMINISTIC,
            ctypes.c_void_p(hi.data_ptr()), ctypes.c_void_p(hd.data_ptr()), ctypes.c_void_p(hc.data_ptr()),
            None))
        np.testing.assert_array_equal(hi.numpy().view(np.uint32), want.ids)
        np.testing.assert_array_equal(hd.numpy().view(np.uint32), want.dists.view(np.uint32))
        np.testing.assert_array_equal(hc.numpy().view(np.uint32), want.counts)


def test_many_overlapping_device_launches_on_two_streams(fixtures, index):
    """More in-flight *_device launches than work-counter slots (64), alternating over
    two streams with mixed procedures: every launch's results equal its own
    synchronous search (no two live launches share a work counter)."""
    import torch
    from paper_2204_00824_b200.search import BestFirstParams, GreedyParams
    g, b, q = fixtures("lowlid3k")
    idx = index("lowlid3k")
    p = BestFirstParams(k=10, seed=4)
    gp = GreedyParams(t0=4, seed=4)
    nq = q.shape[0]
    dq = torch.from_numpy(np.ascontiguousarray(q)).cuda()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = []
    n_launch = 100
    for i in range(n_launch):
        lo = (i * 37) % (nq - 40)
        cnt = 8 + (i * 13) % 32
        ids = torch.full((cnt, 10), -1, dtype=torch.int32, device="cuda")
        dd = torch.empty((cnt, 10), dtype=torch.float32, device="cuda")
        cc = torch.empty(cnt, dtype=torch.int32, device="cuda")
        st = streams[i % 2]
        qp = dq[lo].data_ptr()
        if i % 3 == 2:
            idx.search_greedy_device(qp, cnt, 10, gp, ids.data_ptr(), dd.data_ptr(), cc.data_ptr(),
                                     0, st.cuda_stream)
        else:
            idx.search_bestfirst_device(qp, cnt, p, ids.data_ptr(), dd.data_ptr(), cc.data_ptr(),
                                        0, st.cuda_stream, query_index_base=lo,
                                        mode=_native.MODE_FAST if i % 2 else _native.MODE_DETERMINISTIC)
        outs.append((i, lo, cnt, ids, dd))
    torch.cuda.synchronize()
    for i, lo, cnt, ids, dd in outs:
        if i % 3 == 2:
            want = idx.search_greedy(q[lo:lo + cnt], 10, gp)
        else:
            want = idx.search_bestfirst(q[lo:lo + cnt], p, query_index_base=lo,
                                        mode=_native.MODE_FAST if i % 2 else _native.MODE_DETERMINISTIC)
        np.testing.assert_array_equal(ids.cpu().numpy().view(np.uint32), want.ids, err_msg=str(i))
        np.testing.assert_array_equal(dd.cpu().numpy().view(np.uint32), want.dists.view(np.uint32))


@pytest.mark.parametrize("name", ["syn2k", "lowlid3k"])
def test_fast_paired_kernel_equals_single_on_fixtures(fixtures, index, monkeypatch, name):
    """The group fast kernels (two / four warps per query) on the golden fixtures
    (d = 32, the query-in-registers class below 128 floats) equal the single-warp fast
    kernel."""
    from paper_2204_00824_b200.search import BestFirstParams
    g, b, q = fixtures(name)
    idx = index(name)
    for pd in (dict(k=10, seed=7), dict(k=24, seed=3, m_segments=4, lambda_cut=10)):
        p = BestFirstParams(**pd)
        res = {}
        for grp in ("1", "2", "4"):
            monkeypatch.setenv("TSDG_FAST_GROUP", grp)
            res[grp] = idx.search_bestfirst(q, p, mode=_native.MODE_FAST)
        for grp in ("2", "4"):
            np.testing.assert_array_equal(res[grp].ids, res["1"].ids)
            np.testing.assert_array_equal(res[grp].dists.view(np.uint32), res["1"].dists.view(np.uint32))


@pytest.mark.parametrize("env", [{"TSDG_FAST_VARIANT": str(v)} for v in range(9)]
                         + [{"TSDG_FAST_PREFETCH": p} for p in ("0", "2", "5")]
                         + [{"TSDG_FAST_KERNEL": "staged"}, {"TSDG_FAST_KERNEL": "register"}])
def test_fast_kernel_knobs_keep_recall(fixtures, index, golden, monkeypatch, env):
    """Every compiled fast-kernel variant / prefetch mode / kernel choice runs and keeps
    recall@1 and @10 within 0.5 pt of the deterministic (reference) result."""
    from paper_2204_00824_b200.search import BestFirstParams
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    for name in ("syn2k", "lowlid3k"):
        g, b, q = fixtures(name)
        idx = index(name)
        gt = golden[f"{name}_gt"]
        p = BestFirstParams(k=12, seed=5)
        det = idx.search_bestfirst(q, p)
        fast = idx.search_bestfirst(q, p, mode=_native.MODE_FAST)
        for kk in (1, 10):
            assert abs(O.recall_at_k(fast.ids, fast.counts, gt, kk)
                       - O.recall_at_k(det.ids, det.counts, gt, kk)) <= 0.005, (env, name, kk)
    if datasets.available("c1_lowlid_100k"):  # d = 128: the row class the variants target
        from paper_2204_00824_b200 import search
        ds = _c1()
        p = BestFirstParams(k=14, seed=7)
        det = ds[1].search_bestfirst(ds[0].queries, p)
        fast = ds[1].search_bestfirst(ds[0].queries, p, mode=_native.MODE_FAST)
        for kk in (1, 10):
            assert abs(O.recall_at_k(fast.ids, fast.counts, ds[0].gt, kk)
                       - O.recall_at_k(det.ids, det.counts, ds[0].gt, kk)) <= 0.005, (env, "c1", kk)


_C1 = []


def _c1():
    if not _C1:
        from paper_2204_00824_b200 import search
        ds = datasets.load("c1_lowlid_100k")
        _C1.append((ds, search.GpuIndex.from_file(ds.graph_path, ds.base)))
    return _C1[0]


@pytest.mark.parametrize("stage", ["tma", "g4", "ldgsts"])
def test_row_staging_paths_bit_exact(tmp_path, monkeypatch, stage):
    """Every row-staging path — one TMA bulk copy per row, TMA tile::gather4 tensor
    copies (4 rows per instruction, partial last groups, box = padded row), cp.async —
    in the deterministic best-first kernel and both greedy kernels reproduces the
    oracle, on a 12-float row (box of 20 floats) under L2 and on the inner-product
    fixture."""
    from paper_2204_00824_b200 import search
    for var in ("TSDG_STAGE", "TSDG_GC_STAGE"):
        monkeypatch.setenv(var, stage)
    monkeypatch.setenv("TSDG_GR_STAGE", "tma" if stage == "tma" else "g4")
    orc = O.Oracle()
    base, queries = datasets.make_synthetic_split(1200, 40, 12, 4, 0.3, 17)
    knn = search.brute_force_knn(base, 16)
    path = str(tmp_path / "d12.tsdg")
    search.build(base, knn, 1.2, 9, 0, save_path=path)
    cases = [(path, base, queries)]
    with open(os.path.join(GOLDEN, "scan.json")) as f:
        spec = json.load(f)["specs"]["b"]
    b2, q2 = datasets.generate(spec)
    cases.append((os.path.join(GOLDEN, "build_ip_b.tsdg"), b2, q2))
    for p_, b, q in cases:
        g = O.parse_tsdg(p_)
        idx = search.GpuIndex.from_file(p_, b)
        p = search.BestFirstParams(k=10, seed=3)
        _same(idx.search_bestfirst(q, p), orc.large_batch(g, b, q, p))
        for kern in ("cta", "warp"):
            monkeypatch.setenv("TSDG_GREEDY", kern)
            gp = search.GreedyParams(t0=5, seed=9)
            _same(idx.search_greedy(q, 10, gp), orc.small_batch(g, b, q, 10, gp))
        monkeypatch.delenv("TSDG_GREEDY")
        idx.close()
