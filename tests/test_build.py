"""GPU two-stage diversification (tsdg::build, diversify.cpp:152-209; SURVEY.md §8(f)
row 2).  Parity is pinned on files written by the unmodified reference from the same
KnnGraph (tests/golden/make_golden_build.py): the GPU result saved in the reference's
format must be byte-identical (edges, lambda, fp32 distances, order, header)."""
import json
import os

import numpy as np
import pytest

from paper_2204_00824_b200 import datasets

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _spec(name):
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        s = dict(json.load(f)["fixtures"][name]["spec"])
    s.setdefault("latent", 0)
    s.setdefault("noise", 0.0)
    return s


def _bytes(p):
    with open(p, "rb") as f:
        return f.read()


def test_golden_build_fixtures_present():
    with open(os.path.join(GOLDEN, "build.json")) as f:
        meta = json.load(f)
    assert set(meta) >= {"lowlid3k", "syn2k", "syn2k_a1_l3_m10", "ip_b"}
    z = np.load(os.path.join(GOLDEN, "build_lowlid3k_knn.npz"))
    assert z["ids"].shape == (3000, 32)
    assert (np.diff(z["dists"], axis=1) >= 0).all()  # KnnGraph rows ascending


@pytest.mark.gpu
def test_gpu_build_matches_reference_files(tmp_path):
    from paper_2204_00824_b200 import search
    with open(os.path.join(GOLDEN, "build.json")) as f:
        meta = json.load(f)
    # nn_descent KnnGraph (reference) -> lowlid3k.tsdg
    base, _ = datasets.generate(_spec("lowlid3k"))
    z = np.load(os.path.join(GOLDEN, "build_lowlid3k_knn.npz"))
    st = search.BuildStats()
    out = tmp_path / "a.tsdg"
    g = search.build(base, search.KnnGraph(3000, 32, z["ids"], z["dists"]), 1.2, 9, 0,
                     save_path=str(out), stats=st)
    assert _bytes(out) == _bytes(os.path.join(GOLDEN, "lowlid3k.tsdg"))
    assert [st.input_edges, st.stage1_edges, st.augmented_edges, st.final_edges] == meta["lowlid3k"]
    assert g.n == 3000 and int(g.offsets[-1]) == meta["lowlid3k"][3]
    # GPU brute-force k-NN graph (bit-exact with the reference's) -> syn2k.tsdg, and a
    # second parameter point (alpha 1, lambda0 3, max_degree 10)
    base, _ = datasets.generate(_spec("syn2k"))
    knn = search.brute_force_knn(base, 24)
    out = tmp_path / "b.tsdg"
    search.build(base, knn, 1.2, 9, 0, save_path=str(out), stats=st)
    assert _bytes(out) == _bytes(os.path.join(GOLDEN, "syn2k.tsdg"))
    assert [st.input_edges, st.stage1_edges, st.augmented_edges, st.final_edges] == meta["syn2k"]
    out = tmp_path / "c.tsdg"
    search.build(base, knn, 1.0, 3, 10, save_path=str(out))
    assert _bytes(out) == _bytes(os.path.join(GOLDEN, "build_syn2k_a1_l3_m10.tsdg"))
    # inner product
    with open(os.path.join(GOLDEN, "scan.json")) as f:
        spec_b = json.load(f)["specs"]["b"]
    base, _ = datasets.generate(spec_b)
    knn = search.brute_force_knn(base, 16, metric=2)
    out = tmp_path / "d.tsdg"
    search.build(base, knn, 1.2, 9, 0, metric=2, save_path=str(out))
    assert _bytes(out) == _bytes(os.path.join(GOLDEN, "build_ip_b.tsdg"))


@pytest.mark.gpu
def test_gpu_build_validation():
    from paper_2204_00824_b200 import search
    base, _ = datasets.generate(_spec("syn2k"))
    knn = search.brute_force_knn(base, 8)
    with pytest.raises(search.InvalidArgument, match="alpha must be >= 1"):
        search.build(base, knn, 0.9)
    bad = search.KnnGraph(knn.n, knn.k, knn.ids.copy(), knn.dists.copy())
    bad.dists[5, :] = bad.dists[5, ::-1]
    with pytest.raises(search.InvalidArgument, match="sorted ascending by distance"):
        search.build(base, bad)
    bad = search.KnnGraph(knn.n, knn.k, knn.ids.copy(), knn.dists.copy())
    bad.ids[7, 3] = base.shape[0] + 5
    with pytest.raises(search.InvalidArgument, match="target out of range"):
        search.build(base, bad)


@pytest.mark.gpu
@pytest.mark.skipif(not datasets.available("c1_lowlid_100k"), reason="data/c1_lowlid_100k absent")
def test_gpu_pipeline_rebuilds_c1_graph(tmp_path):
    """Config C1 end to end on the GPU: brute-force k-NN graph (k=100) + build(1.2, 9)
    gives the reference-built data/c1_lowlid_100k/graph.tsdg byte for byte."""
    from paper_2204_00824_b200 import search
    ds = datasets.load("c1_lowlid_100k")
    knn = search.brute_force_knn(ds.base, 100)
    out = tmp_path / "c1.tsdg"
    search.build(ds.base, knn, 1.2, 9, 0, save_path=str(out))
    assert _bytes(out) == _bytes(ds.graph_path)
