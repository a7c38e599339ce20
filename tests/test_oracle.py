"""CPU: the oracle restatement (oracle/tsdg_oracle.c) against the reference's
outputs — the committed golden vectors (tests/golden/make_golden.py ran the
unmodified reference) and, where oracle/_ref exists, the live reference."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2204_00824_b200 import datasets
from paper_2204_00824_b200.search import BestFirstParams, GreedyParams

FIXTURES = ["syn2k", "lowlid3k"]


@pytest.fixture(scope="module")
def orc():
    return O.Oracle()


def test_datagen_matches_reference_generator(golden_meta):
    # bench.cpp:80-129 restated in tools/datagen.c; checksums of the reference's output
    for key, want in golden_meta.items():
        if not key.startswith("gen_"):
            continue
        _, n, nq, d, c, seed = key.split("_")
        spread = 0.25 if int(n) == 1000 else 0.3
        b, q = datasets.make_synthetic_split(int(n), int(nq), int(d), int(c), spread, int(seed))
        assert {"base": datasets.fnv1a(b), "queries": datasets.fnv1a(q)} == want


@pytest.mark.parametrize("name", FIXTURES)
def test_bestfirst_matches_golden(orc, fixtures, golden, golden_meta, name):
    g, b, q = fixtures(name)
    for i, pd in enumerate(golden_meta["bf_grid"]):
        r = orc.large_batch(g, b, q, BestFirstParams(**pd))
        np.testing.assert_array_equal(r.ids, golden[f"{name}_bf{i}_ids"])
        np.testing.assert_array_equal(r.counts, golden[f"{name}_bf{i}_counts"])
        np.testing.assert_array_equal(r.stats, golden[f"{name}_bf{i}_stats"])


@pytest.mark.parametrize("name", FIXTURES)
def test_bestfirst_trace_sizes_match_golden(orc, fixtures, golden, golden_meta, name):
    g, b, q = fixtures(name)
    pd = golden_meta["bf_grid"][1]
    p = BestFirstParams(**pd)
    want = golden[f"{name}_bf1_trace"]
    for qi in range(0, q.shape[0], 17):
        _, _, _, tr = orc.bestfirst_trace(g, b, q[qi], p, orc.fork(p.seed, qi))
        np.testing.assert_array_equal(tr, want[qi])


@pytest.mark.parametrize("name", FIXTURES)
def test_greedy_matches_golden(orc, fixtures, golden, golden_meta, name):
    g, b, q = fixtures(name)
    for i, gd in enumerate(golden_meta["gr_grid"]):
        p = GreedyParams(**{k: v for k, v in gd.items() if k != "k"})
        r = orc.small_batch(g, b, q, gd["k"], p)
        np.testing.assert_array_equal(r.ids, golden[f"{name}_gr{i}_ids"])
        np.testing.assert_array_equal(r.counts, golden[f"{name}_gr{i}_counts"])
        np.testing.assert_array_equal(r.stats, golden[f"{name}_gr{i}_stats"])


@pytest.mark.parametrize("name", FIXTURES)
def test_greedy_once_matches_golden(orc, fixtures, golden, name):
    g, b, q = fixtures(name)
    for qi in range(20):
        ids, dists, st = orc.greedy_once(g, b, q[qi], 100 + qi, 16, 10)
        np.testing.assert_array_equal(ids, golden[f"{name}_once_ids"][qi])
        np.testing.assert_array_equal(dists.view(np.uint32),
                                      golden[f"{name}_once_dists"][qi].view(np.uint32))
        np.testing.assert_array_equal(st, golden[f"{name}_once_stats"][qi])


def test_merge_halves_matches_golden(orc, golden):
    for t in range(golden["mh_upd"].shape[0]):
        ri, rd, upd = orc.merge_halves(golden["mh_old_i"][t], golden["mh_old_d"][t],
                                       golden["mh_tmp_i"][t], golden["mh_tmp_d"][t])
        np.testing.assert_array_equal(ri, golden["mh_out_i"][t])
        np.testing.assert_array_equal(rd, golden["mh_out_d"][t])
        assert upd == bool(golden["mh_upd"][t])


def test_merge_halves_pinned(orc):
    # test_greedy.cpp:100-126
    rij_i = np.full(32, O.KINVALID, np.uint32)
    rij_d = np.full(32, np.inf, np.float32)
    ti = np.arange(100, 132, dtype=np.uint32)
    td = (32.0 - np.arange(32)).astype(np.float32)
    ri, rd, upd = orc.merge_halves(rij_i, rij_d, ti, td)
    assert upd
    np.testing.assert_array_equal(rd[:16], np.arange(1, 17, dtype=np.float32))
    np.testing.assert_array_equal(ri[:16], 131 - np.arange(16))
    assert (ri[16:] == O.KINVALID).all()
    ri2, rd2, upd2 = orc.merge_halves(ri, rd, np.full(32, O.KINVALID, np.uint32),
                                      np.full(32, np.inf, np.float32))
    assert not upd2 and np.array_equal(ri2, ri)
    dup_i = np.full(32, O.KINVALID, np.uint32)
    dup_d = np.full(32, np.inf, np.float32)
    dup_i[:16], dup_d[:16] = ri[:16], rd[:16]
    _, _, upd3 = orc.merge_halves(ri, rd, dup_i, dup_d)
    assert not upd3


def test_lane_update_pinned(orc, golden):
    si, sd = orc.lane_update(np.full(32, O.KINVALID, np.uint32), np.full(32, np.inf, np.float32),
                             [0, 1], [5, 9], np.array([0.5, 0.9], np.float32))
    si, sd = orc.lane_update(si, sd, [0], [7], np.array([0.6], np.float32))
    np.testing.assert_array_equal(si, golden["lane_pinned_i"])
    np.testing.assert_array_equal(sd, golden["lane_pinned_d"])
    assert si[0] == 5 and si[1] == 9 and (si[2:] == O.KINVALID).all()
    with pytest.raises(ValueError):
        orc.lane_update(si, sd, [32], [1], np.array([0.1], np.float32))


@pytest.mark.parametrize("m", [1, 3, 8])
def test_segmented_replay_matches_golden(orc, golden, m):
    o, od, sz, ev = orc.segmented_replay(m, golden[f"seg{m}_ops"], golden[f"seg{m}_ids"],
                                         golden[f"seg{m}_dists"])
    np.testing.assert_array_equal(o, golden[f"seg{m}_out"])
    np.testing.assert_array_equal(od, golden[f"seg{m}_outd"])
    np.testing.assert_array_equal(sz, golden[f"seg{m}_sizes"])
    assert ev == golden[f"seg{m}_ev"][0]


def test_topk_replay_matches_golden(orc, golden):
    o, fi, fd = orc.topk_replay(12, golden["topk_ops"], golden["topk_ids"], golden["topk_dists"])
    np.testing.assert_array_equal(o, golden["topk_out"])
    np.testing.assert_array_equal(fi, golden["topk_final_i"])
    np.testing.assert_array_equal(fd, golden["topk_final_d"])


def test_complete_graph_exact(orc, golden, golden_meta):
    # test_bestfirst.cpp:39-62 / acceptance.cpp:211-257 on the golden complete graph
    spec = golden_meta["fixtures"]["complete96"]["spec"]
    b, q = datasets.make_synthetic_split(spec["n"], spec["nq"], spec["d"], spec["clusters"],
                                         spec["spread"], spec["seed"])
    g = O.parse_tsdg("tests/golden/complete96.tsdg")
    exact = golden["complete96_exact_ids"]
    for unbounded in (False, True):
        p = BestFirstParams(k=10, hop_limit=10000, delta=1e30, m_segments=4, lambda_cut=1,
                            seed=42, unbounded=unbounded)
        r = orc.large_batch(g, b, q, p)
        np.testing.assert_array_equal(r.ids, exact)
    r = orc.small_batch(g, b, q, 10, GreedyParams(t0=16, hop_limit=8, lambda_cut=1, seed=42))
    np.testing.assert_array_equal(r.ids, exact)
    ids, dists = orc.exact_topk(b, q, 10)
    np.testing.assert_array_equal(ids, exact)


def test_parameter_validation(orc, fixtures):
    g, b, q = fixtures("syn2k")
    with pytest.raises(ValueError):
        orc.large_batch(g, b, q[:2], BestFirstParams(delta=-1.0))
    with pytest.raises(ValueError):
        orc.small_batch(g, b, q[:2], 33, GreedyParams(t0=1))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
class TestLiveReference:
    """The restatement against the running reference on fresh seeds."""

    @pytest.fixture(scope="class")
    def ref(self):
        return O.Ref()

    def test_bestfirst_unbounded_and_fresh_seeds(self, ref, orc, fixtures):
        g, b, q = fixtures("syn2k")
        fx = ref.fixture("tests/golden/syn2k.tsdg", b)
        for p in [BestFirstParams(k=12, seed=99, delta=0.3, m_segments=5, lambda_cut=7),
                  BestFirstParams(k=10, seed=4, unbounded=True, delta=0.5, lambda_cut=10),
                  BestFirstParams(k=48, seed=8, m_segments=2, hop_limit=64)]:
            ids, counts, st, _ = fx.bestfirst_per_query(q, p, qbase=5)
            r = orc.large_batch(g, b, q, p, qbase=5)
            np.testing.assert_array_equal(r.ids, ids)
            np.testing.assert_array_equal(r.stats, st)

    def test_batch_front_end_equals_per_query(self, ref, fixtures):
        g, b, q = fixtures("lowlid3k")
        fx = ref.fixture("tests/golden/lowlid3k.tsdg", b)
        p = BestFirstParams(k=10, seed=13)
        ids, counts, tot = fx.large_batch(q, p)
        ids2, counts2, st, _ = fx.bestfirst_per_query(q, p)
        np.testing.assert_array_equal(ids, ids2)
        np.testing.assert_array_equal(tot, st.sum(0))

    def test_segmented_random_ops(self, ref, orc):
        rng = np.random.default_rng(7)
        for m in (2, 5, 16):
            ops = rng.integers(0, 4, 5000).astype(np.uint8)
            ids = rng.integers(0, 150, 5000).astype(np.uint32)
            ds = (rng.integers(0, 300, 5000) / 8.0).astype(np.float32)
            a = orc.segmented_replay(m, ops, ids, ds)
            w = ref.segmented_replay(m, ops, ids, ds)
            for x, y in zip(a[:3], w[:3]):
                np.testing.assert_array_equal(x, y)
            assert a[3] == w[3]
