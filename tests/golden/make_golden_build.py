"""Golden fixtures for the GPU two-stage diversification (tsdg::build,
diversify.cpp:152-209), produced by the UNMODIFIED reference (oracle/_ref):

    python tests/golden/make_golden_build.py

  build_lowlid3k_knn.npz   the reference's nn_descent KnnGraph of the lowlid3k fixture
                           (k=32, 4 iterations, sample 0.6, seed 7); the reference's
                           build(1.2, 9) of it is tests/golden/lowlid3k.tsdg (checked)
  build_syn2k_a1_l3_m10.tsdg  build(alpha=1.0, lambda0=3, max_degree=10) of the syn2k
                           fixture's brute_force_knn(k=24)
  build_ip_b.tsdg          build(1.2, 9) under inner product (metric 2) of scan fixture
                           "b"'s brute_force_knn(k=16, metric 2)
  build.json               stats (BuildStats) of every case
"""
from __future__ import annotations

import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2204_00824_b200 import datasets  # noqa: E402


def main() -> None:
    ref = O.Ref()
    gm = json.load(open(os.path.join(HERE, "golden.json")))
    sm = json.load(open(os.path.join(HERE, "scan.json")))
    meta = {}

    def spec_of(name):
        s = dict(gm["fixtures"][name]["spec"])
        s.setdefault("latent", 0)
        s.setdefault("noise", 0.0)
        return s

    # (1) nn_descent KnnGraph of lowlid3k -> the committed lowlid3k.tsdg
    base, _ = datasets.generate(spec_of("lowlid3k"))
    ids, dists = ref.nn_descent(base, 32, 4, 0.6, 7)
    np.savez_compressed(os.path.join(HERE, "build_lowlid3k_knn.npz"), ids=ids, dists=dists)
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "g.tsdg")
        meta["lowlid3k"] = ref.build_from_knn(base, ids, dists, p, 1.2, 9, 0)
        assert open(p, "rb").read() == open(os.path.join(HERE, "lowlid3k.tsdg"), "rb").read()

    # (2) syn2k brute k=24 with alpha=1.0, lambda0=3, max_degree=10
    base, _ = datasets.generate(spec_of("syn2k"))
    ids, dists = ref.brute_force_knn(base, 24)
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "g.tsdg")
        meta["syn2k"] = ref.build_from_knn(base, ids, dists, p, 1.2, 9, 0)
        assert open(p, "rb").read() == open(os.path.join(HERE, "syn2k.tsdg"), "rb").read()
    meta["syn2k_a1_l3_m10"] = ref.build_from_knn(
        base, ids, dists, os.path.join(HERE, "build_syn2k_a1_l3_m10.tsdg"), 1.0, 3, 10)

    # (3) inner product
    base, _ = datasets.generate(sm["specs"]["b"])
    ids, dists = ref.brute_force_knn(base, 16, metric=2)
    meta["ip_b"] = ref.build_from_knn(base, ids, dists, os.path.join(HERE, "build_ip_b.tsdg"),
                                      1.2, 9, 0, metric=2)
    with open(os.path.join(HERE, "build.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(meta)


if __name__ == "__main__":
    main()
