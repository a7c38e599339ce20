"""Exact top-k scan: GPU ground truth and brute-force k-NN graph (SURVEY.md §8(f)
rows 1 and 4).  The oracle's C restatement is pinned against golden vectors made by
the unmodified reference (tests/golden/make_golden_scan.py); the GPU kernels
(csrc/exact_scan.cuh, through the C-ABI) must then reproduce both bit for bit:
ids, and fp32 distance bits."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2204_00824_b200 import datasets

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def scan_golden():
    with open(os.path.join(GOLDEN, "scan.json")) as f:
        meta = json.load(f)
    g = np.load(os.path.join(GOLDEN, "scan.npz"))
    data = {}
    for name, spec in meta["specs"].items():
        b, q = datasets.generate(spec)
        assert datasets.checksums(b, q) == meta["checksums"][name]
        data[name] = (b, q)
    return meta, g, data


def _bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


# ---------------------------------------------------------------- CPU: oracle pinned
@pytest.mark.parametrize("name", ["a", "b", "tiny"])
def test_oracle_exact_topk_matches_reference(scan_golden, name):
    meta, g, data = scan_golden
    b, q = data[name]
    orc = O.Oracle()
    ids, dists = orc.exact_topk(b, q, 37)
    np.testing.assert_array_equal(ids, g[f"{name}_topk_ids"])
    np.testing.assert_array_equal(_bits(dists), _bits(g[f"{name}_topk_dists"]))
    gt = g[f"{name}_gt"]
    ids, _ = orc.exact_topk(b, q, gt.shape[1])
    np.testing.assert_array_equal(ids, gt)


@pytest.mark.parametrize("name", ["a", "b", "tiny"])
def test_oracle_brute_force_knn_matches_reference(scan_golden, name):
    meta, g, data = scan_golden
    b, _ = data[name]
    orc = O.Oracle()
    for k in (16, 100):
        key = f"{name}_knn{k}"
        if f"{key}_ids" not in g.files:
            continue
        ids, dists = orc.brute_force_knn(b, k)
        assert ids.shape[1] == meta["cases"][key]["k_eff"]
        np.testing.assert_array_equal(ids, g[f"{key}_ids"])
        np.testing.assert_array_equal(_bits(dists), _bits(g[f"{key}_dists"]))
    ids, dists = orc.brute_force_knn(b, 16, metric=2)
    np.testing.assert_array_equal(ids, g[f"{name}_knn16ip_ids"])


# ---------------------------------------------------------------- GPU: bit-exact
@pytest.mark.gpu
@pytest.mark.parametrize("name", ["a", "b", "tiny"])
def test_gpu_ground_truth_bit_exact(scan_golden, name):
    from paper_2204_00824_b200 import search
    meta, g, data = scan_golden
    b, q = data[name]
    gt = g[f"{name}_gt"]
    r = search.ground_truth(b, q, gt.shape[1])
    np.testing.assert_array_equal(r.ids, gt)
    ids, dists = search.exact_topk(b, q, 37)
    np.testing.assert_array_equal(ids, g[f"{name}_topk_ids"])
    np.testing.assert_array_equal(_bits(dists), _bits(g[f"{name}_topk_dists"]))
    r = search.ground_truth(b, q, g[f"{name}_gtip"].shape[1], metric=2)
    np.testing.assert_array_equal(r.ids, g[f"{name}_gtip"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["a", "b", "tiny"])
def test_gpu_brute_force_knn_bit_exact(scan_golden, name):
    from paper_2204_00824_b200 import search
    meta, g, data = scan_golden
    b, _ = data[name]
    for k in (16, 100):
        key = f"{name}_knn{k}"
        if f"{key}_ids" not in g.files:
            continue
        kg = search.brute_force_knn(b, k)
        assert kg.k == meta["cases"][key]["k_eff"]
        np.testing.assert_array_equal(kg.ids, g[f"{key}_ids"])
        np.testing.assert_array_equal(_bits(kg.dists), _bits(g[f"{key}_dists"]))
    kg = search.brute_force_knn(b, 16, metric=2)
    np.testing.assert_array_equal(kg.ids, g[f"{name}_knn16ip_ids"])
    np.testing.assert_array_equal(_bits(kg.dists), _bits(g[f"{name}_knn16ip_dists"]))


@pytest.mark.gpu
def test_gpu_scan_few_queries_max_splits():
    """A handful of queries over a base long enough for the launcher's largest split
    count (the merge follows at most 32 split lists, one per lane): same ids and
    distance bits as the oracle, for small and large k."""
    from paper_2204_00824_b200 import search
    spec = {"kind": "lowlid", "n": 60000, "nq": 3, "d": 12, "latent": 6, "clusters": 10,
            "spread": 0.25, "seed": 21, "noise": 0.01}
    b, q = datasets.generate(spec)
    orc = O.Oracle()
    for k in (10, 300):
        wi, wd = orc.exact_topk(b, q, k)
        r = search.ground_truth(b, q, k)
        np.testing.assert_array_equal(r.ids, wi)
        np.testing.assert_array_equal(_bits(r.dists), _bits(wd))


@pytest.mark.gpu
def test_gpu_scan_splits_and_index_form(scan_golden):
    """Many queries (several base splits + the device merge) and the index-resident
    form agree with the oracle; larger k exercises the 512-entry candidate buffer."""
    from paper_2204_00824_b200 import search
    spec = {"kind": "lowlid", "n": 20000, "nq": 3000, "d": 40, "latent": 8, "clusters": 20,
            "spread": 0.25, "seed": 9, "noise": 0.01}
    b, q = datasets.generate(spec)
    orc = O.Oracle()
    want_i, want_d = orc.exact_topk(b, q[:200], 10)
    r = search.ground_truth(b, q, 10)
    np.testing.assert_array_equal(r.ids[:200], want_i)
    np.testing.assert_array_equal(_bits(r.dists[:200]), _bits(want_d))
    assert (np.diff(r.dists, axis=1) >= 0).all()
    wi, wd = orc.exact_topk(b, q[:50], 300)
    r3 = search.ground_truth(b, q[:50], 300)
    np.testing.assert_array_equal(r3.ids, wi)
    np.testing.assert_array_equal(_bits(r3.dists), _bits(wd))
    # index-resident vectors (graph irrelevant here: a trivial one-edge-per-node ring)
    n = b.shape[0]
    g = search.TsdgGraph(n, 0, 1, 1.2, 9, np.arange(n + 1, dtype=np.uint64),
                         ((np.arange(n) + 1) % n).astype(np.uint32), np.zeros(n, np.uint16),
                         np.zeros(n, np.float32))
    idx = search.GpuIndex(g, b)
    ri = idx.ground_truth(q[:200], 10)
    np.testing.assert_array_equal(ri.ids, want_i)
    idx.close()


@pytest.mark.gpu
def test_gpu_scan_validation():
    from paper_2204_00824_b200 import search
    b = np.random.default_rng(0).standard_normal((10, 4)).astype(np.float32)
    with pytest.raises(search.InvalidArgument, match="1 <= K_gt <= n"):
        search.ground_truth(b, b[:2], 11)
    with pytest.raises(search.InvalidArgument, match="at least 2 vectors"):
        search.brute_force_knn(b[:1], 3)
    kg = search.brute_force_knn(b, 50)  # clamped to n-1 like clamp_k
    assert kg.k == 9 and kg.ids.shape == (10, 9)
    assert not (kg.ids == np.arange(10)[:, None]).any()  # no self loops
