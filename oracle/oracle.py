"""TEST INFRASTRUCTURE ONLY — ctypes front end of the CPU oracle.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference leg
may import this module.  Two back ends:

  Oracle (libtsdg_oracle.so)  plain-C restatement of the reference search path
                              (oracle/tsdg_oracle.c, every function cites the
                              reference file:line it follows)
  Ref    (_ref/libtsdg_ref.so) the UNMODIFIED reference library compiled from
                              /root/reference by oracle/Makefile, behind the
                              extern "C" shim ref_shim.cpp

The restatement is pinned against Ref and against tests/golden/ (see
tests/test_oracle.py).  Graph files are parsed here with numpy, independently of
the product's bulk loader, so a loader bug cannot hide behind the oracle.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libtsdg_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtsdg_ref.so")
KINVALID = 0xFFFFFFFF


class OracleGraph(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint32), ("d", ctypes.c_uint32), ("metric", ctypes.c_int),
                ("base", ctypes.c_void_p), ("offsets", ctypes.c_void_p),
                ("targets", ctypes.c_void_p), ("lambdas", ctypes.c_void_p)]


class OracleBf(ctypes.Structure):
    _fields_ = [("k", ctypes.c_uint32), ("hop_limit", ctypes.c_uint32), ("delta", ctypes.c_float),
                ("m_segments", ctypes.c_uint32), ("lambda_cut", ctypes.c_uint32),
                ("seed", ctypes.c_uint64), ("unbounded", ctypes.c_int)]


class OracleGreedy(ctypes.Structure):
    _fields_ = [("t0", ctypes.c_uint32), ("hop_limit", ctypes.c_uint32),
                ("lambda_cut", ctypes.c_uint32), ("seed", ctypes.c_uint64)]


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class Csr:
    """CSR graph (the reference's TsdgGraph fields, diversify.hpp:56-76)."""
    n: int
    metric: int
    k: int
    alpha: float
    lambda0: int
    offsets: np.ndarray
    targets: np.ndarray
    lambdas: np.ndarray
    dists: np.ndarray


@dataclass
class Result:
    ids: np.ndarray      # nq x k, KINVALID-padded
    dists: np.ndarray    # nq x k, +inf padded
    counts: np.ndarray   # nq
    stats: np.ndarray    # nq x 3 (hops, evals, evictions)


def parse_tsdg(path: str) -> Csr:
    """Independent numpy parser of the TSDG format (diversify.cpp:252-306)."""
    raw = np.fromfile(path, np.uint8)
    if raw[:4].tobytes() != b"TSDG":
        raise RuntimeError(f"{path}: not a TSDG file")
    hdr = raw[:27].tobytes()
    version = int.from_bytes(hdr[4:8], "little")
    if version != 1:
        raise RuntimeError(f"{path}: unsupported TSDG version {version}")
    n = int.from_bytes(hdr[8:16], "little")
    metric = hdr[16]
    k = int.from_bytes(hdr[17:21], "little")
    alpha = float(np.frombuffer(hdr[21:25], "<f4")[0])
    lambda0 = int.from_bytes(hdr[25:27], "little")
    off = 27
    degs = np.empty(n, np.uint64)
    starts = np.empty(n, np.uint64)
    for u in range(n):
        d = int.from_bytes(raw[off:off + 4].tobytes(), "little")
        degs[u] = d
        starts[u] = off + 4
        off += 4 + 10 * d
    offsets = np.zeros(n + 1, np.uint64)
    offsets[1:] = np.cumsum(degs)
    E = int(offsets[-1])
    rec = np.empty((E, 10), np.uint8)
    for u in range(n):
        s, d = int(starts[u]), int(degs[u])
        rec[int(offsets[u]):int(offsets[u]) + d] = raw[s:s + 10 * d].reshape(d, 10)
    targets = rec[:, 0:4].copy().view("<u4").reshape(E).astype(np.uint32)
    lambdas = rec[:, 4:6].copy().view("<u2").reshape(E).astype(np.uint16)
    dists = rec[:, 6:10].copy().view("<f4").reshape(E).astype(np.float32)
    return Csr(n, int(metric), k, alpha, lambda0, offsets, targets, lambdas, dists)


def write_tsdg(g: Csr, path: str) -> None:
    """Byte-exact writer of the TSDG format (diversify.cpp:252-272)."""
    with open(path, "wb") as f:
        f.write(b"TSDG")
        f.write((1).to_bytes(4, "little"))
        f.write(int(g.n).to_bytes(8, "little"))
        f.write(bytes([int(g.metric)]))
        f.write(int(g.k).to_bytes(4, "little"))
        f.write(np.float32(g.alpha).tobytes())
        f.write(int(g.lambda0).to_bytes(2, "little"))
        for u in range(g.n):
            b, e = int(g.offsets[u]), int(g.offsets[u + 1])
            f.write((e - b).to_bytes(4, "little"))
            rec = np.zeros((e - b, 10), np.uint8)
            rec[:, 0:4] = g.targets[b:e].astype("<u4").view(np.uint8).reshape(-1, 4)
            rec[:, 4:6] = g.lambdas[b:e].astype("<u2").view(np.uint8).reshape(-1, 2)
            rec[:, 6:10] = g.dists[b:e].astype("<f4").view(np.uint8).reshape(-1, 4)
            f.write(rec.tobytes())


# ---------------------------------------------------------------- C restatement
class Oracle:
    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"{ORACLE_SO} missing (make -C oracle oracle)")
        self.so = ctypes.CDLL(ORACLE_SO)
        self.so.tsdg_o_distance.restype = ctypes.c_float
        self.so.tsdg_o_distance.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32,
                                            ctypes.c_int]
        self.so.tsdg_o_fork.restype = ctypes.c_uint64
        self.so.tsdg_o_fork.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        self.so.tsdg_o_mix64.restype = ctypes.c_uint64
        self.so.tsdg_o_mix64.argtypes = [ctypes.c_uint64]

    @staticmethod
    def _graph(g: Csr, base: np.ndarray):
        keep = (np.ascontiguousarray(base, np.float32),
                np.ascontiguousarray(g.offsets, np.uint64),
                np.ascontiguousarray(g.targets, np.uint32),
                np.ascontiguousarray(g.lambdas, np.uint16))
        og = OracleGraph(g.n, keep[0].shape[1], g.metric, keep[0].ctypes.data,
                         keep[1].ctypes.data, keep[2].ctypes.data, keep[3].ctypes.data)
        return og, keep

    def fork(self, state: int, index: int) -> int:
        return int(self.so.tsdg_o_fork(state & 0xFFFFFFFFFFFFFFFF, index))

    def distance(self, a, b, metric=0) -> np.float32:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        return np.float32(self.so.tsdg_o_distance(_p(a), _p(b), a.shape[-1], metric))

    def large_batch(self, g: Csr, base, queries, p, qbase: int = 0) -> Result:
        og, keep = self._graph(g, base)
        q = np.ascontiguousarray(queries, np.float32)
        nq, k = q.shape[0], int(p.k)
        ids = np.empty((nq, k), np.uint32)
        dists = np.empty((nq, k), np.float32)
        counts = np.empty(nq, np.uint32)
        stats = np.zeros((nq, 3), np.uint64)
        bp = OracleBf(p.k, p.hop_limit, p.delta, p.m_segments, p.lambda_cut,
                      p.seed & 0xFFFFFFFFFFFFFFFF, 1 if p.unbounded else 0)
        rc = self.so.tsdg_o_large_batch(ctypes.byref(og), _p(q), ctypes.c_uint32(nq),
                                        ctypes.c_uint64(qbase), ctypes.byref(bp), _p(ids),
                                        _p(dists), _p(counts), _p(stats))
        if rc:
            raise ValueError("oracle: invalid parameters")
        return Result(ids, dists, counts, stats)

    def bestfirst_trace(self, g: Csr, base, query, p, rng_state: int):
        """(ids, dists, stats3, (expanded, examined)) for one query."""
        og, keep = self._graph(g, base)
        q = np.ascontiguousarray(query, np.float32)
        ids = np.empty(p.k, np.uint32)
        dists = np.empty(p.k, np.float32)
        cnt = ctypes.c_uint32()
        stats = np.zeros(3, np.uint64)
        trace = np.zeros(2, np.uint64)
        bp = OracleBf(p.k, p.hop_limit, p.delta, p.m_segments, p.lambda_cut, 0,
                      1 if p.unbounded else 0)
        rc = self.so.tsdg_o_bestfirst(ctypes.byref(og), _p(q),
                                      ctypes.c_uint64(rng_state & 0xFFFFFFFFFFFFFFFF),
                                      ctypes.byref(bp), _p(ids), _p(dists), ctypes.byref(cnt),
                                      _p(stats), _p(trace))
        if rc:
            raise ValueError("oracle: invalid parameters")
        return ids[:cnt.value], dists[:cnt.value], stats, trace

    def small_batch(self, g: Csr, base, queries, k: int, p) -> Result:
        og, keep = self._graph(g, base)
        q = np.ascontiguousarray(queries, np.float32)
        nq = q.shape[0]
        ids = np.empty((nq, k), np.uint32)
        dists = np.empty((nq, k), np.float32)
        counts = np.empty(nq, np.uint32)
        stats = np.zeros((nq, 3), np.uint64)
        gp = OracleGreedy(p.t0, p.hop_limit, p.lambda_cut, p.seed & 0xFFFFFFFFFFFFFFFF)
        rc = self.so.tsdg_o_small_batch(ctypes.byref(og), _p(q), ctypes.c_uint32(nq),
                                        ctypes.c_uint32(k), ctypes.byref(gp), _p(ids), _p(dists),
                                        _p(counts), _p(stats))
        if rc:
            raise ValueError("oracle: invalid parameters")
        return Result(ids, dists, counts, stats)

    def greedy_once(self, g: Csr, base, query, rng_state: int, hop_limit=16, cut=10):
        og, keep = self._graph(g, base)
        q = np.ascontiguousarray(query, np.float32)
        ids = np.empty(32, np.uint32)
        dists = np.empty(32, np.float32)
        stats = np.zeros(3, np.uint64)
        rc = self.so.tsdg_o_greedy_once(ctypes.byref(og), _p(q),
                                        ctypes.c_uint64(rng_state & 0xFFFFFFFFFFFFFFFF),
                                        ctypes.c_uint32(hop_limit), ctypes.c_uint32(cut), _p(ids),
                                        _p(dists), _p(stats))
        if rc:
            raise ValueError("oracle: invalid parameters")
        return ids, dists, stats

    def lane_update(self, slot_ids, slot_dists, lanes, ids, dists):
        si = np.array(slot_ids, np.uint32)
        sd = np.array(slot_dists, np.float32)
        la = np.ascontiguousarray(lanes, np.uint32)
        rc = self.so.tsdg_o_lane_update(_p(si), _p(sd), _p(la), _p(np.ascontiguousarray(ids, np.uint32)),
                                        _p(np.ascontiguousarray(dists, np.float32)),
                                        ctypes.c_uint32(len(la)))
        if rc:
            raise ValueError("lane_update: invalid argument")
        return si, sd

    def merge_halves(self, rij_ids, rij_dists, tmp_ids, tmp_dists):
        ri = np.array(rij_ids, np.uint32)
        rd = np.array(rij_dists, np.float32)
        upd = ctypes.c_int()
        self.so.tsdg_o_merge_halves(_p(ri), _p(rd), _p(np.ascontiguousarray(tmp_ids, np.uint32)),
                                    _p(np.ascontiguousarray(tmp_dists, np.float32)),
                                    ctypes.byref(upd))
        return ri, rd, bool(upd.value)

    def segmented_replay(self, m, ops, ids, dists):
        n = len(ops)
        out = np.empty(n, np.uint32)
        od = np.empty(n, np.float32)
        sizes = np.empty(n, np.uint64)
        ev = ctypes.c_uint64()
        rc = self.so.tsdg_o_segmented_replay(ctypes.c_uint32(m), _p(np.ascontiguousarray(ops, np.uint8)),
                                             _p(np.ascontiguousarray(ids, np.uint32)),
                                             _p(np.ascontiguousarray(dists, np.float32)),
                                             ctypes.c_uint32(n), _p(out), _p(od), _p(sizes),
                                             ctypes.byref(ev))
        if rc:
            raise ValueError("segmented: invalid argument")
        return out, od, sizes, ev.value

    def topk_replay(self, k, ops, ids, dists):
        n = len(ops)
        out = np.empty(n, np.uint32)
        fi = np.empty(n + 1, np.uint32)
        fd = np.empty(n + 1, np.float32)
        fn = ctypes.c_uint32()
        rc = self.so.tsdg_o_topk_replay(ctypes.c_uint32(k), _p(np.ascontiguousarray(ops, np.uint8)),
                                        _p(np.ascontiguousarray(ids, np.uint32)),
                                        _p(np.ascontiguousarray(dists, np.float32)),
                                        ctypes.c_uint32(n), _p(out), _p(fi), _p(fd),
                                        ctypes.byref(fn))
        if rc:
            raise ValueError("topk: invalid argument")
        return out, fi[:fn.value], fd[:fn.value]

    def exact_topk(self, base, queries, k, metric=0):
        b = np.ascontiguousarray(base, np.float32)
        q = np.ascontiguousarray(queries, np.float32)
        ids = np.empty((q.shape[0], k), np.uint32)
        dists = np.empty((q.shape[0], k), np.float32)
        self.so.tsdg_o_exact_topk(_p(b), ctypes.c_uint32(b.shape[0]), _p(q),
                                  ctypes.c_uint32(q.shape[0]), ctypes.c_uint32(b.shape[1]),
                                  ctypes.c_uint32(k), ctypes.c_int(metric), _p(ids), _p(dists))
        return ids, dists

    def brute_force_knn(self, base, k, metric=0):
        """knn_graph.cpp:64-86 restated; k clamped to n-1 like clamp_k (:17-26)."""
        b = np.ascontiguousarray(base, np.float32)
        n = b.shape[0]
        k = min(k, n - 1)
        ids = np.empty((n, k), np.uint32)
        dists = np.empty((n, k), np.float32)
        rc = self.so.tsdg_o_brute_force_knn(_p(b), ctypes.c_uint32(n), ctypes.c_uint32(b.shape[1]),
                                            ctypes.c_uint32(k), ctypes.c_int(metric), _p(ids),
                                            _p(dists))
        if rc:
            raise ValueError("brute_force_knn: invalid argument")
        return ids, dists


# ---------------------------------------------------------------- the reference itself
def ref_available() -> bool:
    return os.path.exists(REF_SO)


class Ref:
    """The unmodified reference library (oracle/_ref/libtsdg_ref.so)."""

    def __init__(self):
        if not ref_available():
            raise RuntimeError(f"{REF_SO} missing (make -C oracle ref; needs /root/reference)")
        so = ctypes.CDLL(REF_SO)
        so.ref_last_error.restype = ctypes.c_char_p
        so.ref_fixture_load.restype = ctypes.c_void_p
        so.ref_fixture_load.argtypes = [ctypes.c_char_p, ctypes.c_void_p, ctypes.c_uint32,
                                        ctypes.c_uint32]
        so.ref_fixture_free.argtypes = [ctypes.c_void_p]
        so.ref_fixture_n.argtypes = [ctypes.c_void_p]
        so.ref_fixture_n.restype = ctypes.c_uint32
        so.ref_fixture_edges.argtypes = [ctypes.c_void_p]
        so.ref_fixture_edges.restype = ctypes.c_uint64
        so.ref_fixture_csr.argtypes = [ctypes.c_void_p] + [ctypes.c_void_p] * 4
        so.ref_mix64.restype = ctypes.c_uint64
        so.ref_mix64.argtypes = [ctypes.c_uint64]
        so.ref_distance.restype = ctypes.c_float
        so.ref_distance.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_int]
        so.ref_num_threads.restype = ctypes.c_int
        for name in ("ref_large_batch_search", "ref_small_batch_search", "ref_bestfirst_per_query",
                     "ref_greedy_per_query", "ref_greedy_search_once", "ref_bestfirst_trace"):
            getattr(so, name).argtypes = None
        self.so = so

    def err(self) -> str:
        return self.so.ref_last_error().decode()

    def check(self, rc):
        if rc == 1:
            raise ValueError(self.err())
        if rc:
            raise RuntimeError(self.err())

    def build_graph(self, base, path, *, method="brute", knn_k=30, iters=5, sample_rate=1.0,
                    knn_seed=7, alpha=1.2, lambda0=9, max_degree=0, metric=0):
        b = np.ascontiguousarray(base, np.float32)
        stats = (ctypes.c_uint64 * 4)()
        rc = self.so.ref_build_tsdg(_p(b), ctypes.c_uint32(b.shape[0]), ctypes.c_uint32(b.shape[1]),
                                    ctypes.c_int(metric), ctypes.c_int(0 if method == "brute" else 1),
                                    ctypes.c_uint32(knn_k), ctypes.c_uint32(iters),
                                    ctypes.c_double(sample_rate), ctypes.c_uint64(knn_seed),
                                    ctypes.c_float(alpha), ctypes.c_uint32(lambda0),
                                    ctypes.c_uint32(max_degree), path.encode(), stats)
        self.check(rc)
        return list(stats)

    def save_csr(self, g: Csr, path: str):
        rc = self.so.ref_save_csr(ctypes.c_uint32(g.n), ctypes.c_int(g.metric), ctypes.c_uint32(g.k),
                                  ctypes.c_float(g.alpha), ctypes.c_uint32(g.lambda0),
                                  _p(np.ascontiguousarray(g.offsets, np.uint64)),
                                  _p(np.ascontiguousarray(g.targets, np.uint32)),
                                  _p(np.ascontiguousarray(g.lambdas, np.uint16)),
                                  _p(np.ascontiguousarray(g.dists, np.float32)), path.encode())
        self.check(rc)

    def fixture(self, tsdg_path, base):
        b = np.ascontiguousarray(base, np.float32)
        h = self.so.ref_fixture_load(tsdg_path.encode(), _p(b), b.shape[0], b.shape[1])
        if not h:
            raise RuntimeError(self.err())
        return RefFixture(self, h, b.shape[1])

    def fixture_from_files(self, tsdg_path, vectors_path):
        """Graph and base loaded by the reference's own load_tsdg / load_vectors."""
        so = self.so
        so.ref_fixture_load_files.restype = ctypes.c_void_p
        so.ref_fixture_load_files.argtypes = [ctypes.c_char_p, ctypes.c_char_p]
        so.ref_fixture_d.restype = ctypes.c_uint32
        so.ref_fixture_d.argtypes = [ctypes.c_void_p]
        h = so.ref_fixture_load_files(tsdg_path.encode(), vectors_path.encode())
        if not h:
            raise RuntimeError(self.err())
        return RefFixture(self, h, so.ref_fixture_d(ctypes.c_void_p(h)))

    def make_synthetic_split(self, n, nq, d, clusters, spread, seed):
        b = np.empty((n, d), np.float32)
        q = np.empty((nq, d), np.float32)
        self.check(self.so.ref_make_synthetic_split(ctypes.c_uint32(n), ctypes.c_uint32(nq),
                                                    ctypes.c_uint32(d), ctypes.c_uint32(clusters),
                                                    ctypes.c_float(spread), ctypes.c_uint64(seed),
                                                    _p(b), _p(q)))
        return b, q

    def ground_truth(self, base, queries, k, metric=0):
        b = np.ascontiguousarray(base, np.float32)
        q = np.ascontiguousarray(queries, np.float32)
        out = np.empty((q.shape[0], k), np.uint32)
        self.check(self.so.ref_ground_truth(_p(b), ctypes.c_uint32(b.shape[0]), _p(q),
                                            ctypes.c_uint32(q.shape[0]), ctypes.c_uint32(b.shape[1]),
                                            ctypes.c_uint32(k), ctypes.c_int(metric), _p(out)))
        return out

    def lane_update(self, slot_ids, slot_dists, lanes, ids, dists):
        si = np.array(slot_ids, np.uint32)
        sd = np.array(slot_dists, np.float32)
        la = np.ascontiguousarray(lanes, np.uint32)
        self.check(self.so.ref_lane_update(_p(si), _p(sd), _p(la), _p(np.ascontiguousarray(ids, np.uint32)),
                                           _p(np.ascontiguousarray(dists, np.float32)),
                                           ctypes.c_uint32(len(la))))
        return si, sd

    def merge_halves(self, rij_ids, rij_dists, tmp_ids, tmp_dists):
        ri = np.array(rij_ids, np.uint32)
        rd = np.array(rij_dists, np.float32)
        upd = ctypes.c_int()
        self.check(self.so.ref_merge_halves(_p(ri), _p(rd), _p(np.ascontiguousarray(tmp_ids, np.uint32)),
                                            _p(np.ascontiguousarray(tmp_dists, np.float32)),
                                            ctypes.byref(upd)))
        return ri, rd, bool(upd.value)

    def segmented_replay(self, m, ops, ids, dists):
        n = len(ops)
        out = np.empty(n, np.uint32)
        od = np.empty(n, np.float32)
        sizes = np.empty(n, np.uint64)
        ev = ctypes.c_uint64()
        self.check(self.so.ref_segmented_replay(ctypes.c_uint32(m), _p(np.ascontiguousarray(ops, np.uint8)),
                                                _p(np.ascontiguousarray(ids, np.uint32)),
                                                _p(np.ascontiguousarray(dists, np.float32)),
                                                ctypes.c_uint32(n), _p(out), _p(od), _p(sizes),
                                                ctypes.byref(ev)))
        return out, od, sizes, ev.value

    def topk_replay(self, k, ops, ids, dists):
        n = len(ops)
        out = np.empty(n, np.uint32)
        fi = np.empty(n + 1, np.uint32)
        fd = np.empty(n + 1, np.float32)
        fn = ctypes.c_uint32()
        self.check(self.so.ref_topk_replay(ctypes.c_uint32(k), _p(np.ascontiguousarray(ops, np.uint8)),
                                           _p(np.ascontiguousarray(ids, np.uint32)),
                                           _p(np.ascontiguousarray(dists, np.float32)),
                                           ctypes.c_uint32(n), _p(out), _p(fi), _p(fd),
                                           ctypes.byref(fn)))
        return out, fi[:fn.value], fd[:fn.value]

    def exact_topk(self, base, queries, k, metric=0):
        b = np.ascontiguousarray(base, np.float32)
        q = np.ascontiguousarray(queries, np.float32)
        ids = np.empty((q.shape[0], k), np.uint32)
        dists = np.empty((q.shape[0], k), np.float32)
        self.check(self.so.ref_exact_topk(_p(b), ctypes.c_uint32(b.shape[0]), _p(q),
                                          ctypes.c_uint32(q.shape[0]), ctypes.c_uint32(b.shape[1]),
                                          ctypes.c_uint32(k), ctypes.c_int(metric), _p(ids), _p(dists)))
        return ids, dists

    def normalized_copy(self, x):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        self.check(self.so.ref_normalized_copy(_p(x), ctypes.c_uint32(x.shape[0]),
                                               ctypes.c_uint32(x.shape[1]), _p(out)))
        return out

    def load_vectors(self, path):
        """tsdg::load_vectors -> (n, d) float32; raises with the reference's message."""
        n, d = ctypes.c_uint32(), ctypes.c_uint32()
        self.check(self.so.ref_load_vectors(str(path).encode(), ctypes.byref(n), ctypes.byref(d),
                                            None))
        out = np.empty((n.value, d.value), np.float32)
        self.check(self.so.ref_load_vectors(str(path).encode(), ctypes.byref(n), ctypes.byref(d),
                                            _p(out)))
        return out

    def run_bench_file(self, config_path, csv_out):
        self.check(self.so.ref_run_bench_file(str(config_path).encode(), str(csv_out).encode()))

    def nn_descent(self, base, k, iterations, sample_rate, seed, metric=0):
        b = np.ascontiguousarray(base, np.float32)
        n = b.shape[0]
        kk = max(1, min(k, n - 1))
        ids = np.empty((n, kk), np.uint32)
        dists = np.empty((n, kk), np.float32)
        keff = ctypes.c_uint32()
        self.check(self.so.ref_nn_descent(_p(b), ctypes.c_uint32(n), ctypes.c_uint32(b.shape[1]),
                                          ctypes.c_int(metric), ctypes.c_uint32(k),
                                          ctypes.c_uint32(iterations), ctypes.c_double(sample_rate),
                                          ctypes.c_uint64(seed), _p(ids), _p(dists),
                                          ctypes.byref(keff)))
        return ids[:, :keff.value], dists[:, :keff.value]

    def build_from_knn(self, base, knn_ids, knn_dists, path, alpha=1.2, lambda0=9, max_degree=0,
                       metric=0):
        b = np.ascontiguousarray(base, np.float32)
        ki = np.ascontiguousarray(knn_ids, np.uint32)
        kd = np.ascontiguousarray(knn_dists, np.float32)
        stats = (ctypes.c_uint64 * 4)()
        self.check(self.so.ref_build_from_knn(_p(b), ctypes.c_uint32(b.shape[0]),
                                              ctypes.c_uint32(b.shape[1]), ctypes.c_int(metric),
                                              _p(ki), _p(kd), ctypes.c_uint32(ki.shape[1]),
                                              ctypes.c_float(alpha), ctypes.c_uint32(lambda0),
                                              ctypes.c_uint32(max_degree), str(path).encode(), stats))
        return list(stats)

    def brute_force_knn(self, base, k, metric=0):
        b = np.ascontiguousarray(base, np.float32)
        n = b.shape[0]
        kk = max(1, min(k, n - 1))
        ids = np.empty((n, kk), np.uint32)
        dists = np.empty((n, kk), np.float32)
        keff = ctypes.c_uint32()
        self.check(self.so.ref_brute_force_knn(_p(b), ctypes.c_uint32(n), ctypes.c_uint32(b.shape[1]),
                                               ctypes.c_uint32(k), ctypes.c_int(metric), _p(ids),
                                               _p(dists), ctypes.byref(keff)))
        return ids[:, :keff.value], dists[:, :keff.value]


class RefFixture:
    def __init__(self, ref: Ref, h, d):
        self.ref, self.h, self.d = ref, h, d

    def __del__(self):
        try:
            self.ref.so.ref_fixture_free(ctypes.c_void_p(self.h))
        except Exception:
            pass

    def csr(self) -> Csr:
        so = self.ref.so
        n = so.ref_fixture_n(ctypes.c_void_p(self.h))
        E = so.ref_fixture_edges(ctypes.c_void_p(self.h))
        off = np.empty(n + 1, np.uint64)
        t = np.empty(E, np.uint32)
        lam = np.empty(E, np.uint16)
        ds = np.empty(E, np.float32)
        so.ref_fixture_csr(ctypes.c_void_p(self.h), _p(off), _p(t), _p(lam), _p(ds))
        return Csr(n, 0, 0, 0.0, 0, off, t, lam, ds)

    def large_batch(self, queries, p):
        """The reference batch front end itself (ids, counts, summed stats)."""
        q = np.ascontiguousarray(queries, np.float32)
        nq, k = q.shape[0], int(p.k)
        ids = np.empty((nq, k), np.uint32)
        counts = np.empty(nq, np.uint32)
        stats = np.zeros(3, np.uint64)
        rc = self.ref.so.ref_large_batch_search(
            ctypes.c_void_p(self.h), _p(q), ctypes.c_uint32(nq), ctypes.c_uint32(k),
            ctypes.c_uint32(p.hop_limit), ctypes.c_float(p.delta), ctypes.c_uint32(p.m_segments),
            ctypes.c_uint32(p.lambda_cut), ctypes.c_uint64(p.seed & 0xFFFFFFFFFFFFFFFF),
            ctypes.c_int(1 if p.unbounded else 0), _p(ids), _p(counts), _p(stats))
        self.ref.check(rc)
        return ids, counts, stats

    def bestfirst_per_query(self, queries, p, qbase=0):
        q = np.ascontiguousarray(queries, np.float32)
        nq, k = q.shape[0], int(p.k)
        ids = np.empty((nq, k), np.uint32)
        counts = np.empty(nq, np.uint32)
        stats = np.zeros((nq, 3), np.uint64)
        trace = np.zeros((nq, 2), np.uint64)
        rc = self.ref.so.ref_bestfirst_per_query(
            ctypes.c_void_p(self.h), _p(q), ctypes.c_uint32(nq), ctypes.c_uint64(qbase),
            ctypes.c_uint32(k), ctypes.c_uint32(p.hop_limit), ctypes.c_float(p.delta),
            ctypes.c_uint32(p.m_segments), ctypes.c_uint32(p.lambda_cut),
            ctypes.c_uint64(p.seed & 0xFFFFFFFFFFFFFFFF), ctypes.c_int(1 if p.unbounded else 0),
            _p(ids), _p(counts), _p(stats), _p(trace))
        self.ref.check(rc)
        return ids, counts, stats, trace

    def small_batch(self, queries, k, p):
        q = np.ascontiguousarray(queries, np.float32)
        nq = q.shape[0]
        ids = np.empty((nq, k), np.uint32)
        counts = np.empty(nq, np.uint32)
        stats = np.zeros(3, np.uint64)
        rc = self.ref.so.ref_small_batch_search(
            ctypes.c_void_p(self.h), _p(q), ctypes.c_uint32(nq), ctypes.c_uint32(k),
            ctypes.c_uint32(p.t0), ctypes.c_uint32(p.hop_limit), ctypes.c_uint32(p.lambda_cut),
            ctypes.c_uint64(p.seed & 0xFFFFFFFFFFFFFFFF), _p(ids), _p(counts), _p(stats))
        self.ref.check(rc)
        return ids, counts, stats

    def greedy_per_query(self, queries, k, p):
        q = np.ascontiguousarray(queries, np.float32)
        nq = q.shape[0]
        ids = np.empty((nq, k), np.uint32)
        counts = np.empty(nq, np.uint32)
        stats = np.zeros((nq, 3), np.uint64)
        rc = self.ref.so.ref_greedy_per_query(
            ctypes.c_void_p(self.h), _p(q), ctypes.c_uint32(nq), ctypes.c_uint32(k),
            ctypes.c_uint32(p.t0), ctypes.c_uint32(p.hop_limit), ctypes.c_uint32(p.lambda_cut),
            ctypes.c_uint64(p.seed & 0xFFFFFFFFFFFFFFFF), _p(ids), _p(counts), _p(stats))
        self.ref.check(rc)
        return ids, counts, stats

    def greedy_once(self, query, rng_seed, fork_index=None, hop_limit=16, cut=10):
        q = np.ascontiguousarray(query, np.float32)
        ids = np.empty(32, np.uint32)
        dists = np.empty(32, np.float32)
        stats = np.zeros(3, np.uint64)
        rc = self.ref.so.ref_greedy_search_once(
            ctypes.c_void_p(self.h), _p(q), ctypes.c_uint64(rng_seed & 0xFFFFFFFFFFFFFFFF),
            ctypes.c_int(0 if fork_index is None else 1), ctypes.c_uint64(fork_index or 0),
            ctypes.c_uint32(hop_limit), ctypes.c_uint32(cut), _p(ids), _p(dists), _p(stats))
        self.ref.check(rc)
        return ids, dists, stats

    def bestfirst_trace(self, query, p, rng_seed, fork_index=None, cap=1 << 20):
        q = np.ascontiguousarray(query, np.float32)
        ids = np.empty(p.k, np.uint32)
        cnt = ctypes.c_uint32()
        exp = np.empty(cap, np.uint32)
        nexp = ctypes.c_uint32()
        exam = np.empty(2 * cap, np.uint32)
        nexam = ctypes.c_uint32()
        rc = self.ref.so.ref_bestfirst_trace(
            ctypes.c_void_p(self.h), _p(q), ctypes.c_uint64(rng_seed & 0xFFFFFFFFFFFFFFFF),
            ctypes.c_int(0 if fork_index is None else 1), ctypes.c_uint64(fork_index or 0),
            ctypes.c_uint32(p.k), ctypes.c_uint32(p.hop_limit), ctypes.c_float(p.delta),
            ctypes.c_uint32(p.m_segments), ctypes.c_uint32(p.lambda_cut),
            ctypes.c_int(1 if p.unbounded else 0), _p(ids), ctypes.byref(cnt), _p(exp),
            ctypes.byref(nexp), _p(exam), ctypes.byref(nexam), ctypes.c_uint32(cap))
        self.ref.check(rc)
        return ids[:cnt.value], exp[:nexp.value], exam[:2 * nexam.value].reshape(-1, 2)


# ---------------------------------------------------------------- helpers
def complete_graph(base: np.ndarray, metric: int = 0) -> Csr:
    """The reference tests' complete-graph fixture (test_bestfirst.cpp:18-33):
    every other node, lambda 0, sorted by (dist, target)."""
    o = Oracle()
    n = base.shape[0]
    offsets = np.zeros(n + 1, np.uint64)
    tg, lm, ds = [], [], []
    for u in range(n):
        d = np.array([o.distance(base[u], base[v], metric) if v != u else np.inf
                      for v in range(n)], np.float32)
        order = np.lexsort((np.arange(n), d))
        order = order[order != u]
        tg.append(order.astype(np.uint32))
        lm.append(np.zeros(n - 1, np.uint16))
        ds.append(d[order])
        offsets[u + 1] = offsets[u] + (n - 1)
    return Csr(n, metric, n - 1, 1.0, 0, offsets, np.concatenate(tg), np.concatenate(lm),
               np.concatenate(ds))


def recall_at_k(ids: np.ndarray, counts: np.ndarray, gt: np.ndarray, k: int) -> float:
    """bench.cpp:59-78: |results[0..k) ^ truth[0..k)| / (nq * k)."""
    hits = 0
    for q in range(ids.shape[0]):
        want = set(gt[q, :k].tolist())
        got = ids[q, :min(int(counts[q]), k)].tolist()
        hits += sum(1 for x in got if x in want)
    return hits / (ids.shape[0] * k)
