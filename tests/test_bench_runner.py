"""GPU port of the JSON bench runner (run_bench_file, bench.cpp:189-362; SURVEY.md
§8(f) row 4).  Reference CSVs come from the unmodified reference
(tests/golden/make_golden_bench.py); in deterministic mode every column except qps
must be identical, string for string."""
import csv
import glob
import os

import numpy as np
import pytest

from paper_2204_00824_b200 import bench_runner as B

HERE = os.path.dirname(os.path.abspath(__file__))
CONFIGS = sorted(glob.glob(os.path.join(HERE, "golden", "bench", "*.json")))


def _rows(path):
    with open(path) as f:
        return list(csv.reader(f))


def test_helpers_match_reference_semantics(tmp_path):
    assert B.metric_from_name("cosine") == 1 and B.metric_from_name("innerproduct") == 2
    with pytest.raises(B.InvalidArgument, match="unknown metric"):
        B.metric_from_name("hamming")
    assert B.mix64(0) == 0 and B.mix64(7 + 40) == B.mix64(47)
    assert B._fmt(0.5) == "0.5" and B._fmt(1e30) == "1e+30" and B._fmt(1234567.0) == "1.23457e+06"
    # fvecs / bvecs / ivecs round trips and the reference's error cases
    x = np.random.default_rng(1).standard_normal((5, 3)).astype(np.float32)
    rec = b"".join(np.int32(3).tobytes() + r.tobytes() for r in x)
    (tmp_path / "a.fvecs").write_bytes(rec)
    np.testing.assert_array_equal(B.load_vectors(str(tmp_path / "a.fvecs")), x)
    bv = b"".join(np.int32(4).tobytes() + bytes([i, 2, 3, 255]) for i in range(3))
    (tmp_path / "a.bvecs").write_bytes(bv)
    assert B.load_vectors(str(tmp_path / "a.bvecs"))[2, 3] == 255.0
    (tmp_path / "bad.fvecs").write_bytes(rec[:-4])  # truncated last record
    with pytest.raises(B.TsdgRuntimeError):
        B.load_vectors(str(tmp_path / "bad.fvecs"))
    iv = np.int32(2).tobytes() + np.array([4, 9], "<i4").tobytes() + np.int32(0).tobytes()
    (tmp_path / "g.ivecs").write_bytes(iv)
    lists = B.load_ivecs(str(tmp_path / "g.ivecs"))
    assert [list(l) for l in lists] == [[4, 9], []]
    (tmp_path / "n.ivecs").write_bytes(np.int32(-1).tobytes())
    with pytest.raises(B.TsdgRuntimeError, match="negative record length"):
        B.load_ivecs(str(tmp_path / "n.ivecs"))
    # recall (bench.cpp:59-78)
    assert B.recall_at_k([np.array([1, 3, 9])], [np.array([3, 9, 1])], 3, 2) == 0.5


def test_normalized_copy_matches_reference():
    from oracle import oracle as O
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    from paper_2204_00824_b200 import datasets
    b, _ = datasets.make_synthetic_split(500, 1, 20, 5, 0.3, 9)
    got = B.normalized_copy(b)
    want = O.Ref().normalized_copy(b)
    np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", CONFIGS, ids=[os.path.basename(c) for c in CONFIGS])
def test_gpu_runner_matches_reference_csv(cfg, tmp_path):
    out = tmp_path / "gpu.csv"
    B.run_bench_file(cfg, str(out))
    want = _rows(cfg[:-5] + ".ref.csv")
    got = _rows(out)
    assert got[0] == want[0]
    assert len(got) == len(want)
    qps = want[0].index("qps")
    for g, w in zip(got[1:], want[1:]):
        assert [x for i, x in enumerate(g) if i != qps] == [x for i, x in enumerate(w) if i != qps]
        assert float(g[qps]) > 0
