import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: larger CPU-side cases")


@pytest.fixture(scope="session")
def golden():
    return np.load(os.path.join(GOLDEN, "golden.npz"))


@pytest.fixture(scope="session")
def golden_meta():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)


def fixture_data(meta, name):
    """(graph Csr, base, queries) for a golden fixture; vectors regenerated."""
    from oracle import oracle as O
    from paper_2204_00824_b200 import datasets

    spec = dict(meta["fixtures"][name]["spec"])
    spec.setdefault("latent", 0)
    spec.setdefault("noise", 0.0)
    base, queries = datasets.generate(spec)
    assert datasets.checksums(base, queries) == meta["fixtures"][name]["checksums"]
    graph = O.parse_tsdg(os.path.join(GOLDEN, f"{name}.tsdg"))
    return graph, base, queries


@pytest.fixture(scope="session")
def fixtures(golden_meta):
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = fixture_data(golden_meta, name)
        return cache[name]

    return get
