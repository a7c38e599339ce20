"""Persistent small-batch server (tsdg_gpu_server_*): every request returns exactly
what the launch path (tsdg_gpu_search_greedy) returns — itself bit-exact with the
reference's small_batch_search (greedy_search.cpp:106-127) in deterministic mode."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2204_00824_b200 import _native, datasets, search
from paper_2204_00824_b200.search import GreedyParams, InvalidArgument

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def syn2k():
    base, queries = datasets.make_synthetic_split(2000, 200, 32, 8, 0.2, 11)
    idx = search.GpuIndex.from_file("tests/golden/syn2k.tsdg", base)
    return idx, base, queries


@pytest.mark.parametrize("t0", [1, 4, 10, 16])
def test_server_equals_launch_path_and_oracle(syn2k, t0):
    idx, base, queries = syn2k
    p = GreedyParams(t0=t0, seed=5)
    g = O.parse_tsdg("tests/golden/syn2k.tsdg")
    want = O.Oracle().small_batch(g, base, queries[:64], 10, p)
    with idx.greedy_server(10, p, max_batch=64) as sv:
        for batch in (1, 8, 64, 3):
            for lo in range(0, 64, batch):
                q = queries[lo:lo + batch]
                got = sv.search(q)
                ref = idx.search_greedy(q, 10, p)
                np.testing.assert_array_equal(got.ids, ref.ids)
                np.testing.assert_array_equal(got.dists.view(np.uint32), ref.dists.view(np.uint32))
                np.testing.assert_array_equal(got.counts, ref.counts)
                np.testing.assert_array_equal(got.ids, want.ids[lo:lo + batch])


def test_server_fast_mode_and_reuse(syn2k):
    idx, base, queries = syn2k
    p = GreedyParams(t0=8, seed=3)
    with idx.greedy_server(16, p, mode=_native.MODE_FAST, max_batch=8) as sv:
        for _ in range(3):  # requests keep working after many round trips
            for lo in range(0, 200, 8):
                got = sv.search(queries[lo:lo + 8])
                ref = idx.search_greedy(queries[lo:lo + 8], 16, p, mode=_native.MODE_FAST)
                np.testing.assert_array_equal(got.ids, ref.ids)


def test_server_limits(syn2k):
    idx, _, queries = syn2k
    with pytest.raises(InvalidArgument):
        idx.greedy_server(10, GreedyParams(t0=17))
    with pytest.raises(InvalidArgument):
        idx.greedy_server(65, GreedyParams(t0=4))
    with idx.greedy_server(10, GreedyParams(t0=4), max_batch=2) as sv:
        with pytest.raises(InvalidArgument):
            sv.search(queries[:3])


@pytest.mark.skipif(not datasets.available("c2_lowlid_1m"), reason="data/c2_lowlid_1m absent")
@pytest.mark.parametrize("t0", [10, 16])
def test_server_c2_bit_exact(t0):
    ds = datasets.load("c2_lowlid_1m")
    idx = search.GpuIndex.from_file(ds.graph_path, ds.base)
    p = GreedyParams(t0=t0, hop_limit=16, lambda_cut=10, seed=7)
    q = ds.queries[:64]
    want = O.Oracle().small_batch(O.parse_tsdg(ds.graph_path), ds.base, q, 10, p)
    with idx.greedy_server(10, p, max_batch=64) as sv:
        for batch in (1, 8, 64):
            for lo in range(0, 64, batch):
                got = sv.search(q[lo:lo + batch])
                np.testing.assert_array_equal(got.ids, want.ids[lo:lo + batch])
                np.testing.assert_array_equal(got.dists.view(np.uint32),
                                              want.dists[lo:lo + batch].view(np.uint32))
