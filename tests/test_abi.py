"""CPU: the C-ABI library loads and exports every symbol include/tsdg_gpu.h
declares (no compute calls without a GPU); host-side loader and validation."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import oracle as O
from paper_2204_00824_b200 import _native, search

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "tsdg_gpu.h")).read()
    return sorted(set(re.findall(r"^(?:int|const char\*|uint64_t)\s+(tsdg_\w+)\(", src, re.M)))


def test_header_symbols_exported():
    so = ctypes.CDLL(_native.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(so, s), s
    assert set(syms) == set(_native.SIGNATURES), "ctypes table out of sync with the header"


def test_abi_version():
    assert _native.lib().tsdg_gpu_abi_version() == 1


@pytest.mark.parametrize("name", ["syn2k", "lowlid3k", "complete96"])
def test_bulk_loader_matches_independent_parser(name):
    path = os.path.join(ROOT, "tests", "golden", f"{name}.tsdg")
    g = search.load_tsdg(path)
    w = O.parse_tsdg(path)
    assert (g.n, g.metric, g.k, g.lambda0) == (w.n, w.metric, w.k, w.lambda0)
    assert np.float32(g.alpha) == np.float32(w.alpha)
    np.testing.assert_array_equal(g.offsets, w.offsets)
    np.testing.assert_array_equal(g.targets, w.targets)
    np.testing.assert_array_equal(g.lambdas, w.lambdas)
    np.testing.assert_array_equal(g.dists.view(np.uint32), w.dists.view(np.uint32))
    assert g.max_degree == int(np.diff(w.offsets).max())


def test_bulk_loader_errors(tmp_path):
    p = tmp_path / "bad.tsdg"
    p.write_bytes(b"NOPE" + b"\0" * 40)
    with pytest.raises(search.TsdgRuntimeError, match="not a TSDG file"):
        search.load_tsdg(str(p))
    good = open(os.path.join(ROOT, "tests", "golden", "syn2k.tsdg"), "rb").read()
    p.write_bytes(good[:1000])
    with pytest.raises(search.TsdgRuntimeError, match="truncated file"):
        search.load_tsdg(str(p))
    p.write_bytes(good[:4] + (2).to_bytes(4, "little") + good[8:])
    with pytest.raises(search.TsdgRuntimeError, match="unsupported TSDG version 2"):
        search.load_tsdg(str(p))
    with pytest.raises(search.TsdgRuntimeError, match="cannot open"):
        search.load_tsdg(str(tmp_path / "missing.tsdg"))


def test_neighbors_below_is_lambda_prefix():
    g = search.load_tsdg(os.path.join(ROOT, "tests", "golden", "syn2k.tsdg"))
    for u in range(0, g.n, 97):
        b, e = int(g.offsets[u]), int(g.offsets[u + 1])
        for cut in (1, 2, 5, 10):
            nb = g.neighbors_below(u, cut)
            assert np.array_equal(nb, g.targets[b:b + len(nb)])
            assert (g.lambdas[b:b + len(nb)] < cut).all()
            assert (g.lambdas[b + len(nb):e] >= cut).all()


def test_params_defaults_mirror_reference():
    # bestfirst_search.hpp:15-25, greedy_search.hpp:14-19
    p = search.BestFirstParams()
    assert (p.k, p.hop_limit, p.delta, p.m_segments, p.lambda_cut, p.seed, p.unbounded) == \
        (10, 1024, 0.0, 8, 5, 0, False)
    g = search.GreedyParams()
    assert (g.t0, g.hop_limit, g.lambda_cut, g.seed) == (16, 16, 10, 0)
