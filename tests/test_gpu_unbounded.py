"""GPU: BestFirstParams.unbounded = true — the reference's exact std::set queue and
visited set (bestfirst_search.cpp:14-47) — against the oracle's restatement,
which tests/test_oracle.py pins to the live reference."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2204_00824_b200 import datasets, search
from paper_2204_00824_b200.search import BestFirstParams

pytestmark = pytest.mark.gpu


def test_unbounded_bit_exact(fixtures):
    orc = O.Oracle()
    for name in ("syn2k", "lowlid3k"):
        g, b, q = fixtures(name)
        idx = search.GpuIndex(search.load_tsdg(f"tests/golden/{name}.tsdg"), b)
        for p in (BestFirstParams(k=10, seed=4, unbounded=True, delta=0.5, lambda_cut=10),
                  BestFirstParams(k=32, seed=9, unbounded=True),
                  BestFirstParams(k=10, seed=2, unbounded=True, hop_limit=24, delta=4.0)):
            got = idx.search_bestfirst(q, p)
            want = orc.large_batch(g, b, q, p)
            np.testing.assert_array_equal(got.ids, want.ids)
            np.testing.assert_array_equal(got.dists.view(np.uint32), want.dists.view(np.uint32))
            np.testing.assert_array_equal(got.stats["hops"], want.stats[:, 0])
            np.testing.assert_array_equal(got.stats["distance_evals"], want.stats[:, 1])


def test_segmented_equals_unbounded_without_overflow(fixtures):
    # test_bestfirst.cpp:103-123: hop limit 24 keeps every segment below capacity
    g, b, q = fixtures("syn2k")
    idx = search.GpuIndex(search.load_tsdg("tests/golden/syn2k.tsdg"), b)
    p = BestFirstParams(k=10, hop_limit=24, delta=4.0, seed=10)
    seg = idx.search_bestfirst(q, p)
    assert (seg.stats["queue_evictions"] == 0).all()
    ub = idx.search_bestfirst(q, BestFirstParams(k=10, hop_limit=24, delta=4.0, seed=10,
                                                 unbounded=True))
    np.testing.assert_array_equal(seg.ids, ub.ids)


def test_unbounded_complete_graph_exact(golden, golden_meta):
    spec = golden_meta["fixtures"]["complete96"]["spec"]
    b, q = datasets.make_synthetic_split(spec["n"], spec["nq"], spec["d"], spec["clusters"],
                                         spec["spread"], spec["seed"])
    idx = search.GpuIndex.from_file("tests/golden/complete96.tsdg", b)
    p = BestFirstParams(k=10, hop_limit=100000, delta=1e30, lambda_cut=1, seed=42, unbounded=True)
    np.testing.assert_array_equal(idx.search_bestfirst(q, p).ids, golden["complete96_exact_ids"])
