"""GPU nn_descent (tsdg_gpu_nn_descent) against the reference's tsdg::nn_descent
(knn_graph.cpp:141-251): the KnnGraph must be identical, ids and fp32 distance bits,
for the same (set, k, metric, iterations, sample_rate, seed).  Pinned on the golden
KnnGraph the reference wrote (tests/golden/build_lowlid3k_knn.npz) and on the live
reference library (oracle/_ref) over a grid of shapes, metrics and sample rates."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2204_00824_b200 import datasets, search
from paper_2204_00824_b200.search import InvalidArgument

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _same(g: search.KnnGraph, ids, dists):
    np.testing.assert_array_equal(g.ids, ids)
    np.testing.assert_array_equal(g.dists.view(np.uint32), np.ascontiguousarray(dists).view(np.uint32))


def test_golden_lowlid3k_knn(golden_meta):
    """make_golden_build.py: ref.nn_descent(lowlid3k base, k=32, 4 iterations, 0.6, seed 7)."""
    spec = dict(golden_meta["fixtures"]["lowlid3k"]["spec"])
    spec.setdefault("latent", 0)
    spec.setdefault("noise", 0.0)
    base, _ = datasets.generate(spec)
    z = np.load(os.path.join(ROOT, "tests", "golden", "build_lowlid3k_knn.npz"))
    st = {}
    g = search.nn_descent(base, 32, 4, 0.6, 7, stats=st)
    assert g.k == 32
    _same(g, z["ids"], z["dists"])
    assert st["offers"] > 0 and st["chunks"] >= 4


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("n,d,k,iters,rate,seed,metric", [
    (2000, 32, 16, 3, 0.5, 7, 0),
    (3000, 20, 24, 4, 1.0, 11, 0),     # d not a multiple of 4, full sampling
    (1500, 16, 8, 6, 0.3, 3, 0),
    (2500, 24, 40, 2, 0.8, 5, 2),      # inner product (negative distances)
    (2000, 12, 20, 3, 0.5, 9, 1),      # cosine on normalized rows
    (64, 8, 100, 3, 0.5, 1, 0),        # k clamped to n - 1
    (300, 8, 128, 2, 1.0, 2, 0),       # the GPU's widest list
    (20000, 64, 32, 5, 0.5, 7, 0),
])
def test_matches_reference(n, d, k, iters, rate, seed, metric):
    ref = O.Ref()
    base, _ = datasets.make_synthetic_split(n, 1, d, 12, 0.3, seed + 100)
    if metric == 1:
        base = ref.normalized_copy(base)
    ids, dists = ref.nn_descent(base, k, iters, rate, seed, metric=metric)
    g = search.nn_descent(base, k, iters, rate, seed, metric=metric)
    assert g.k == ids.shape[1]
    _same(g, ids, dists)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_iteration_prefix_and_quality():
    """knn_graph.hpp:37-40: a+1 iterations extend a run of a; quality non-decreasing;
    zero iterations = the random initial lists."""
    ref = O.Ref()
    base, _ = datasets.make_lowlid(4000, 1, 32, latent=8, seed=3)
    gt_ids, _ = ref.brute_force_knn(base, 16)
    prev = -1.0
    for it in (0, 1, 2, 4):
        g = search.nn_descent(base, 16, it, 0.5, 13)
        ids, dists = ref.nn_descent(base, 16, it, 0.5, 13)
        _same(g, ids, dists)
        q = np.mean([len(set(g.ids[u]) & set(gt_ids[u])) / 16 for u in range(4000)])
        assert q >= prev
        prev = q
    assert prev > 0.9


def test_validation_errors():
    base = np.random.default_rng(0).standard_normal((50, 8)).astype(np.float32)
    with pytest.raises(InvalidArgument, match="sample_rate"):
        search.nn_descent(base, 10, 2, 0.0, 1)
    with pytest.raises(InvalidArgument, match="sample_rate"):
        search.nn_descent(base, 10, 2, 1.5, 1)
    with pytest.raises(InvalidArgument, match="k must be"):
        search.nn_descent(base, 0, 2, 0.5, 1)
    with pytest.raises(InvalidArgument, match="at least 2"):
        search.nn_descent(base[:1], 4, 2, 0.5, 1)


def test_c2_graph_rebuilt_on_gpu_byte_identical(tmp_path):
    """Full size: the GPU nn_descent + GPU build with the parameters the reference used
    for data/c2_lowlid_1m (nn_descent k=64, 5 iterations, 0.5, seed 7; build(1.2, 9))
    rewrite the reference's graph file byte for byte."""
    import json
    if not datasets.available("c2_lowlid_1m"):
        pytest.skip("data/c2_lowlid_1m absent")
    ds = datasets.load("c2_lowlid_1m")
    gm = ds.meta["graph"]
    assert gm["builder"] == "nndescent"
    knn = search.nn_descent(ds.base, gm["knn_k"], gm["iters"], gm["sample_rate"], gm["knn_seed"])
    out = str(tmp_path / "gpu.tsdg")
    search.build(ds.base, knn, gm["alpha"], gm["lambda0"], 0, save_path=out)
    with open(out, "rb") as a, open(ds.graph_path, "rb") as b:
        assert a.read() == b.read()
