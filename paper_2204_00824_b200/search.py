"""Host-side mirror of the reference's C++ search API, over the B200 C-ABI.

Reference interface (paper_2204_00824, /root/reference/proj/include/tsdg):
  BestFirstParams        bestfirst_search.hpp:15-25   -> BestFirstParams
  GreedyParams           greedy_search.hpp:14-19      -> GreedyParams
  SearchStats            greedy_search.hpp:21-32      -> SearchStats
  load_tsdg              diversify.hpp:127            -> load_tsdg (bulk C loader)
  large_batch_search     bestfirst_search.hpp:47-51   -> large_batch_search / GpuIndex
  bestfirst_search       bestfirst_search.hpp:39-43   -> bestfirst_search
  small_batch_search     greedy_search.hpp:55-60      -> small_batch_search / GpuIndex
  small_batch_search_one greedy_search.hpp:49-52      -> small_batch_search_one
  greedy_search_once     greedy_search.hpp:43-45      -> greedy_search_once
  ground_truth           bench.hpp (bench.cpp:35-57)  -> ground_truth / GpuIndex.ground_truth
  exact_topk             reference.hpp (reference.cpp:96-111) -> exact_topk
  brute_force_knn        knn_graph.hpp:32             -> brute_force_knn
  build / save_tsdg      diversify.hpp:114,125        -> build (GPU two-stage diversification)
Same field names, defaults, argument meaning and exception types
(std::invalid_argument -> InvalidArgument(ValueError)); results come back as the
reference's list-of-id-lists, and the extended calls also return fp32 distances
and per-query counters.  Every call runs on the GPU; nothing here computes.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _native
from ._native import InvalidArgument, TsdgRuntimeError, check, lib

KINVALID = 0xFFFFFFFF
METRICS = {"l2": 0, "cos": 1, "cosine": 1, "ip": 2, "innerproduct": 2}


@dataclass
class BestFirstParams:
    k: int = 10
    hop_limit: int = 1024
    delta: float = 0.0
    m_segments: int = 8
    lambda_cut: int = 5
    seed: int = 0
    unbounded: bool = False

    def c(self) -> _native.BfParamsC:
        return _native.BfParamsC(self.k, self.hop_limit, self.delta, self.m_segments,
                                 self.lambda_cut, self.seed & 0xFFFFFFFFFFFFFFFF,
                                 1 if self.unbounded else 0)


@dataclass
class GreedyParams:
    t0: int = 16
    hop_limit: int = 16
    lambda_cut: int = 10
    seed: int = 0

    def c(self) -> _native.GreedyParamsC:
        return _native.GreedyParamsC(self.t0, self.hop_limit, self.lambda_cut,
                                     self.seed & 0xFFFFFFFFFFFFFFFF)


@dataclass
class SearchStats:
    hops: int = 0
    distance_evals: int = 0
    queue_evictions: int = 0

    def add(self, per_query: np.ndarray) -> None:
        self.hops += int(per_query["hops"].sum(dtype=np.uint64))
        self.distance_evals += int(per_query["distance_evals"].sum(dtype=np.uint64))
        self.queue_evictions += int(per_query["queue_evictions"].sum(dtype=np.uint64))


QUERY_STATS_DTYPE = np.dtype([("hops", np.uint32), ("distance_evals", np.uint32),
                              ("queue_evictions", np.uint32), ("edges_examined", np.uint32)])


@dataclass
class SearchResult:
    """ids/dists are nq x k (ascending by (dist, id), padded KINVALID / +inf)."""
    ids: np.ndarray
    dists: np.ndarray
    counts: np.ndarray
    stats: np.ndarray  # QUERY_STATS_DTYPE per query

    def lists(self) -> List[np.ndarray]:
        return [self.ids[q, : self.counts[q]].copy() for q in range(self.ids.shape[0])]


@dataclass
class TsdgGraph:
    """CSR TSDG as loaded from the reference's file format (diversify.hpp:56-76)."""
    n: int
    metric: int
    k: int
    alpha: float
    lambda0: int
    offsets: np.ndarray   # u64 n+1
    targets: np.ndarray   # u32 E
    lambdas: np.ndarray   # u16 E
    dists: np.ndarray     # f32 E
    max_degree: int = 0

    def neighbors_below(self, u: int, lambda_cut: int) -> np.ndarray:
        b, e = int(self.offsets[u]), int(self.offsets[u + 1])
        cut = int(np.searchsorted(self.lambdas[b:e], lambda_cut, side="left"))
        return self.targets[b:b + cut]


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def load_tsdg(path: str) -> TsdgGraph:
    h = _native.GraphHeaderC()
    check(lib().tsdg_read_tsdg_header(path.encode(), ctypes.byref(h)))
    off = np.empty(h.n + 1, np.uint64)
    tgt = np.empty(h.num_edges, np.uint32)
    lam = np.empty(h.num_edges, np.uint16)
    dst = np.empty(h.num_edges, np.float32)
    check(lib().tsdg_read_tsdg(path.encode(), _p(off), _p(tgt), _p(lam), _p(dst)))
    return TsdgGraph(int(h.n), int(h.metric), int(h.k), float(h.alpha), int(h.lambda0), off, tgt,
                     lam, dst, int(h.max_degree))


def read_vectors(path: str) -> np.ndarray:
    """fvecs / bvecs file -> (n, d) float32 (tsdg::load_vectors, io.cpp:112-117;
    bvecs components widened to float).  Errors carry the reference's messages."""
    n, d = ctypes.c_uint32(), ctypes.c_uint32()
    check(lib().tsdg_read_vectors_shape(path.encode(), ctypes.byref(n), ctypes.byref(d)))
    out = np.empty((n.value, d.value), np.float32)
    check(lib().tsdg_read_vectors(path.encode(), _p(out), n.value, d.value))
    return out


def _f32rows(a, d: Optional[int] = None) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    if a.ndim == 1:
        a = a.reshape(1, -1)
    if d is not None and a.shape[1] != d:
        raise InvalidArgument(f"dim mismatch ({a.shape[1]} vs {d})")
    return a


class GpuIndex:
    """Device-resident TSDG + vector store on one GPU (C-ABI tsdg_gpu_index)."""

    def __init__(self, graph: TsdgGraph, base, device: int = 0):
        base = _f32rows(base)
        if base.shape[0] != graph.n:
            raise InvalidArgument(f"graph has {graph.n} nodes, base has {base.shape[0]} rows")
        self.n, self.d = int(base.shape[0]), int(base.shape[1])
        self.metric = graph.metric
        self.device = device
        self.graph = graph
        h = ctypes.c_void_p()
        check(lib().tsdg_gpu_index_create(
            _p(base), self.n, self.d, _p(np.ascontiguousarray(graph.offsets, np.uint64)),
            _p(np.ascontiguousarray(graph.targets, np.uint32)),
            _p(np.ascontiguousarray(graph.lambdas, np.uint16)), int(graph.metric), device,
            ctypes.byref(h)))
        self._h = h
        self._read_info()

    @classmethod
    def from_file(cls, tsdg_path: str, base, device: int = 0) -> "GpuIndex":
        return cls(load_tsdg(tsdg_path), base, device)

    @classmethod
    def from_files(cls, tsdg_path: str, vectors_path: str, device: int = 0) -> "GpuIndex":
        """Index straight from a reference .tsdg file and an fvecs/bvecs base: the
        raw file bytes are decoded on the device (tsdg_gpu_index_create_from_files);
        no host graph or vector array is built."""
        self = cls.__new__(cls)
        h = ctypes.c_void_p()
        check(lib().tsdg_gpu_index_create_from_files(tsdg_path.encode(), vectors_path.encode(),
                                                     device, ctypes.byref(h)))
        self._h = h
        self.device = device
        self.graph = None
        self._read_info()
        return self

    def _read_info(self) -> None:
        info = [ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_int(), ctypes.c_uint32(),
                ctypes.c_int(), ctypes.c_uint32(), ctypes.c_uint32()]
        check(lib().tsdg_gpu_index_info(self._h, *[ctypes.byref(x) for x in info]))
        self.n, self.d, self.metric = info[0].value, info[1].value, info[2].value
        self.max_degree, self.row_stride, self.adj_stride = info[3].value, info[5].value, info[6].value

    def close(self) -> None:
        if getattr(self, "_h", None):
            check(lib().tsdg_gpu_index_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def ground_truth(self, queries, k_gt: int) -> GroundTruth:
        """Exact top-k_gt over the resident vector store (tsdg::ground_truth)."""
        q = _f32rows(queries, self.d)
        nq = q.shape[0]
        ids = np.empty((nq, max(k_gt, 1)), np.uint32)
        dists = np.empty((nq, max(k_gt, 1)), np.float32)
        check(lib().tsdg_gpu_index_ground_truth(self._h, _p(q), nq, int(k_gt), _p(ids), _p(dists)))
        return GroundTruth(int(k_gt), ids, dists)

    def deg_cut(self, lambda_cut: int) -> np.ndarray:
        out = np.empty(self.n, np.uint32)
        check(lib().tsdg_gpu_deg_cut(self._h, lambda_cut, _p(out)))
        return out

    # ---- large batch (Alg. 2) ------------------------------------------------
    def search_bestfirst(self, queries, params: BestFirstParams = BestFirstParams(), *,
                         query_index_base: int = 0, mode: int = _native.MODE_DETERMINISTIC
                         ) -> SearchResult:
        q = _f32rows(queries, self.d)
        nq, k = q.shape[0], int(params.k)
        ids = np.empty((nq, max(k, 1)), np.uint32)
        dists = np.empty((nq, max(k, 1)), np.float32)
        counts = np.empty(nq, np.uint32)
        stats = np.zeros(nq, QUERY_STATS_DTYPE)
        pc = params.c()
        check(lib().tsdg_gpu_search_bestfirst(self._h, _p(q), nq, query_index_base,
                                              ctypes.byref(pc), mode, _p(ids), _p(dists),
                                              _p(counts), _p(stats)))
        return SearchResult(ids, dists, counts, stats)

    def large_batch_search(self, queries, params: BestFirstParams = BestFirstParams(),
                           stats: Optional[SearchStats] = None, **kw) -> List[np.ndarray]:
        r = self.search_bestfirst(queries, params, **kw)
        if stats is not None:
            stats.add(r.stats)
        return r.lists()

    # ---- small batch (Alg. 1) ------------------------------------------------
    def search_greedy(self, queries, k: int, params: GreedyParams = GreedyParams(), *,
                      mode: int = _native.MODE_DETERMINISTIC) -> SearchResult:
        q = _f32rows(queries, self.d)
        nq = q.shape[0]
        kk = max(int(k), 1)
        ids = np.empty((nq, kk), np.uint32)
        dists = np.empty((nq, kk), np.float32)
        counts = np.empty(nq, np.uint32)
        stats = np.zeros(nq, QUERY_STATS_DTYPE)
        pc = params.c()
        check(lib().tsdg_gpu_search_greedy(self._h, _p(q), nq, int(k), ctypes.byref(pc), mode,
                                           _p(ids), _p(dists), _p(counts), _p(stats)))
        return SearchResult(ids, dists, counts, stats)

    def small_batch_search(self, queries, k: int, params: GreedyParams = GreedyParams(),
                           stats: Optional[SearchStats] = None, **kw) -> List[np.ndarray]:
        r = self.search_greedy(queries, k, params, **kw)
        if stats is not None:
            stats.add(r.stats)
        return r.lists()

    def greedy_search_once(self, queries, rng_states, hop_limit: int = 16,
                           lambda_cut: int = 10):
        """One walk per query with explicit RNG states (greedy_search.cpp:27-72).
        Returns (ids nq x 32, dists nq x 32, stats)."""
        q = _f32rows(queries, self.d)
        nq = q.shape[0]
        st = np.ascontiguousarray(np.broadcast_to(np.asarray(rng_states, np.uint64), (nq,)))
        ids = np.empty((nq, 32), np.uint32)
        dists = np.empty((nq, 32), np.float32)
        stats = np.zeros(nq, QUERY_STATS_DTYPE)
        check(lib().tsdg_gpu_greedy_once(self._h, _p(q), nq, _p(st), hop_limit, lambda_cut,
                                         _p(ids), _p(dists), _p(stats)))
        return ids, dists, stats

    # ---- device-pointer entry points (torch tensors / raw pointers) ----------
    def search_bestfirst_device(self, q_ptr: int, nq: int, params: BestFirstParams,
                                ids_ptr: int, dists_ptr: int, counts_ptr: int,
                                stats_ptr: int = 0, stream: int = 0, *,
                                query_index_base: int = 0,
                                mode: int = _native.MODE_DETERMINISTIC) -> None:
        pc = params.c()
        check(lib().tsdg_gpu_search_bestfirst_device(
            self._h, ctypes.c_void_p(q_ptr), nq, query_index_base, ctypes.byref(pc), mode,
            ctypes.c_void_p(ids_ptr), ctypes.c_void_p(dists_ptr or None),
            ctypes.c_void_p(counts_ptr or None), ctypes.c_void_p(stats_ptr or None),
            ctypes.c_void_p(stream or None)))

    def search_greedy_device(self, q_ptr: int, nq: int, k: int, params: GreedyParams,
                             ids_ptr: int, dists_ptr: int, counts_ptr: int,
                             stats_ptr: int = 0, stream: int = 0, *,
                             mode: int = _native.MODE_DETERMINISTIC) -> None:
        pc = params.c()
        check(lib().tsdg_gpu_search_greedy_device(
            self._h, ctypes.c_void_p(q_ptr), nq, k, ctypes.byref(pc), mode,
            ctypes.c_void_p(ids_ptr), ctypes.c_void_p(dists_ptr or None),
            ctypes.c_void_p(counts_ptr or None), ctypes.c_void_p(stats_ptr or None),
            ctypes.c_void_p(stream or None)))


class MultiGpuIndex:
    """Replicated index over several GPUs in one process (C-ABI tsdg_gpu_multi): a
    batch is split into contiguous slices searched concurrently, slice b.. with
    query_index_base + b — the results equal GpuIndex's for any device list."""

    def __init__(self, graph: TsdgGraph, base, devices=(0,)):
        base = _f32rows(base)
        if base.shape[0] != graph.n:
            raise InvalidArgument(f"graph has {graph.n} nodes, base has {base.shape[0]} rows")
        self.n, self.d = int(base.shape[0]), int(base.shape[1])
        devs = np.ascontiguousarray(list(devices), np.int32)
        h = ctypes.c_void_p()
        check(lib().tsdg_gpu_multi_create(
            _p(base), self.n, self.d, _p(np.ascontiguousarray(graph.offsets, np.uint64)),
            _p(np.ascontiguousarray(graph.targets, np.uint32)),
            _p(np.ascontiguousarray(graph.lambdas, np.uint16)), int(graph.metric), _p(devs),
            len(devs), ctypes.byref(h)))
        self._h = h

    def close(self) -> None:
        if getattr(self, "_h", None):
            check(lib().tsdg_gpu_multi_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def search_bestfirst(self, queries, params: BestFirstParams = BestFirstParams(), *,
                         query_index_base: int = 0, mode: int = _native.MODE_DETERMINISTIC
                         ) -> SearchResult:
        q = _f32rows(queries, self.d)
        nq, k = q.shape[0], int(params.k)
        ids = np.empty((nq, max(k, 1)), np.uint32)
        dists = np.empty((nq, max(k, 1)), np.float32)
        counts = np.empty(nq, np.uint32)
        stats = np.zeros(nq, QUERY_STATS_DTYPE)
        pc = params.c()
        check(lib().tsdg_gpu_multi_search_bestfirst(self._h, _p(q), nq, query_index_base,
                                                    ctypes.byref(pc), mode, _p(ids), _p(dists),
                                                    _p(counts), _p(stats)))
        return SearchResult(ids, dists, counts, stats)

    def search_greedy(self, queries, k: int, params: GreedyParams = GreedyParams(), *,
                      mode: int = _native.MODE_DETERMINISTIC) -> SearchResult:
        q = _f32rows(queries, self.d)
        nq = q.shape[0]
        ids = np.empty((nq, max(k, 1)), np.uint32)
        dists = np.empty((nq, max(k, 1)), np.float32)
        counts = np.empty(nq, np.uint32)
        stats = np.zeros(nq, QUERY_STATS_DTYPE)
        pc = params.c()
        check(lib().tsdg_gpu_multi_search_greedy(self._h, _p(q), nq, int(k), ctypes.byref(pc), mode,
                                                 _p(ids), _p(dists), _p(counts), _p(stats)))
        return SearchResult(ids, dists, counts, stats)


class ShardedGpuIndex:
    """Sharded base in one process (C-ABI tsdg_gpu_sharded): shard s = a TSDG file over
    its own rows, global id = offsets[s] + local id; every query searched on every
    shard (shard s on devices[s]), per-shard top-k merged by (dist, global id)."""

    def __init__(self, tsdg_paths, bases, offsets, devices=None):
        self._bases = [_f32rows(b) for b in bases]
        S = len(self._bases)
        self.d = int(self._bases[0].shape[1])
        devs = np.ascontiguousarray(list(devices) if devices is not None else [0] * S, np.int32)
        paths = (ctypes.c_char_p * S)(*[str(p).encode() for p in tsdg_paths])
        ptrs = (ctypes.c_void_p * S)(*[b.ctypes.data for b in self._bases])
        ns = np.ascontiguousarray([b.shape[0] for b in self._bases], np.uint32)
        offs = np.ascontiguousarray(list(offsets), np.uint64)
        h = ctypes.c_void_p()
        check(lib().tsdg_gpu_sharded_create_from_files(paths, ptrs, _p(ns), _p(offs), S, self.d,
                                                       _p(devs), ctypes.byref(h)))
        self._h = h

    def close(self) -> None:
        if getattr(self, "_h", None):
            check(lib().tsdg_gpu_sharded_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def search_bestfirst(self, queries, params: BestFirstParams = BestFirstParams(), *,
                         query_index_base: int = 0, mode: int = _native.MODE_DETERMINISTIC):
        q = _f32rows(queries, self.d)
        nq, k = q.shape[0], int(params.k)
        ids = np.empty((nq, max(k, 1)), np.uint32)
        dists = np.empty((nq, max(k, 1)), np.float32)
        counts = np.empty(nq, np.uint32)
        pc = params.c()
        check(lib().tsdg_gpu_sharded_search_bestfirst(self._h, _p(q), nq, query_index_base,
                                                      ctypes.byref(pc), mode, _p(ids), _p(dists),
                                                      _p(counts)))
        return ids, dists, counts


@dataclass
class GroundTruth:
    """tsdg::GroundTruth (bench.hpp): k ids per query, plus the fp32 distances."""
    k: int
    ids: np.ndarray    # nq x k u32
    dists: np.ndarray  # nq x k f32


@dataclass
class KnnGraph:
    """tsdg::KnnGraph (knn_graph.hpp:15-28): n x k neighbours ascending by (dist, id)."""
    n: int
    k: int
    ids: np.ndarray    # n x k u32
    dists: np.ndarray  # n x k f32


def ground_truth(base, queries, k_gt: int, metric: int = 0, device: int = 0) -> GroundTruth:
    """tsdg::ground_truth (bench.cpp:35-57) on the GPU: exact top-k_gt by (dist, id)."""
    b = _f32rows(base)
    q = _f32rows(queries)
    if q.shape[1] != b.shape[1]:
        raise InvalidArgument("ground_truth: dim mismatch")
    nq = q.shape[0]
    ids = np.empty((nq, max(k_gt, 1)), np.uint32)
    dists = np.empty((nq, max(k_gt, 1)), np.float32)
    check(lib().tsdg_gpu_ground_truth(_p(b), b.shape[0], _p(q), nq, b.shape[1], int(k_gt),
                                      int(metric), device, _p(ids), _p(dists)))
    return GroundTruth(int(k_gt), ids, dists)


def exact_topk(base, queries, k: int, metric: int = 0, device: int = 0):
    """ref::exact_topk (reference.cpp:96-111): (ids, dists), nq x k."""
    g = ground_truth(base, queries, k, metric, device)
    return g.ids, g.dists


def brute_force_knn(base, k: int, metric: int = 0, device: int = 0) -> KnnGraph:
    """tsdg::brute_force_knn (knn_graph.cpp:64-86) on the GPU: exact k-NN graph, self
    excluded, k clamped to n-1 (warning on stderr), same (dist, id) order."""
    b = _f32rows(base)
    n = b.shape[0]
    kk = max(1, min(int(k), max(n - 1, 1)))
    ids = np.empty((n, kk), np.uint32)
    dists = np.empty((n, kk), np.float32)
    keff = ctypes.c_uint32(0)
    check(lib().tsdg_gpu_brute_force_knn(_p(b), n, b.shape[1], int(k), int(metric), device,
                                         _p(ids), _p(dists), ctypes.byref(keff)))
    return KnnGraph(n, int(keff.value), ids, dists)


def nn_descent(base, k: int, iterations: int, sample_rate: float, seed: int, metric: int = 0,
               device: int = 0, stats: Optional[dict] = None) -> KnnGraph:
    """tsdg::nn_descent (knn_graph.cpp:141-251) on the GPU: the reference's KnnGraph
    bit for bit for the same (k, metric, iterations, sample_rate, seed); k clamped to
    n-1 (warning on stderr); sample_rate outside (0, 1] is an InvalidArgument."""
    b = _f32rows(base)
    n = b.shape[0]
    kk = max(1, min(int(k), max(n - 1, 1)))
    ids = np.empty((n, kk), np.uint32)
    dists = np.empty((n, kk), np.float32)
    keff = ctypes.c_uint32(0)
    st = np.zeros(4, np.uint64)
    check(lib().tsdg_gpu_nn_descent(_p(b), n, b.shape[1], int(k), int(metric), int(iterations),
                                    float(sample_rate), int(seed) & 0xFFFFFFFFFFFFFFFF, device,
                                    _p(ids), _p(dists), ctypes.byref(keff), _p(st)))
    if stats is not None:
        stats.update(offers=int(st[0]), chunks=int(st[1]), reruns=int(st[2]), launches=int(st[3]))
    return KnnGraph(n, int(keff.value), ids, dists)


@dataclass
class BuildStats:
    """tsdg::BuildStats (diversify.hpp:39-44)."""
    input_edges: int = 0
    stage1_edges: int = 0
    augmented_edges: int = 0
    final_edges: int = 0


def build(base, knn: KnnGraph, alpha: float = 1.2, lambda0: int = 9, max_degree: int = 0,
          metric: int = 0, device: int = 0, save_path: Optional[str] = None,
          stats: Optional[BuildStats] = None) -> TsdgGraph:
    """tsdg::build (diversify.cpp:152-209) on the GPU: the same TsdgGraph as the
    reference's from the same KnnGraph.  save_path writes it in the reference's file
    format (save_tsdg, diversify.cpp:252-272)."""
    b = _f32rows(base)
    ids = np.ascontiguousarray(knn.ids, np.uint32)
    dists = np.ascontiguousarray(knn.dists, np.float32)
    if ids.shape[0] != b.shape[0]:
        raise InvalidArgument("build: graph/set size mismatch")
    st = (ctypes.c_uint64 * 4)()
    g = ctypes.c_void_p()
    check(lib().tsdg_gpu_build(_p(b), b.shape[0], b.shape[1], _p(ids), _p(dists), ids.shape[1],
                               float(alpha), int(lambda0), int(max_degree), int(metric), device,
                               ctypes.byref(g), st))
    try:
        n, ne, md = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint32()
        check(lib().tsdg_gpu_graph_info(g, ctypes.byref(n), ctypes.byref(ne), ctypes.byref(md)))
        off = np.empty(n.value + 1, np.uint64)
        tgt = np.empty(ne.value, np.uint32)
        lam = np.empty(ne.value, np.uint16)
        dst = np.empty(ne.value, np.float32)
        check(lib().tsdg_gpu_graph_copy(g, _p(off), _p(tgt), _p(lam), _p(dst)))
        if save_path is not None:
            check(lib().tsdg_gpu_graph_save(g, str(save_path).encode()))
    finally:
        lib().tsdg_gpu_graph_destroy(g)
    if stats is not None:
        stats.input_edges, stats.stage1_edges, stats.augmented_edges, stats.final_edges = list(st)
    return TsdgGraph(int(n.value), int(metric), int(ids.shape[1]), float(np.float32(alpha)),
                     int(lambda0), off, tgt, lam, dst, int(md.value))


def merge_shards_device(ids_ptr: int, dists_ptr: int, counts_ptr: int, shard_base, shards: int,
                        nq: int, k: int, out_ids_ptr: int, out_dists_ptr: int,
                        out_counts_ptr: int, stream: int = 0) -> None:
    base = np.ascontiguousarray(shard_base, np.uint64)
    check(lib().tsdg_gpu_merge_shards_device(
        ctypes.c_void_p(ids_ptr), ctypes.c_void_p(dists_ptr), ctypes.c_void_p(counts_ptr),
        _p(base), shards, nq, k, ctypes.c_void_p(out_ids_ptr), ctypes.c_void_p(out_dists_ptr),
        ctypes.c_void_p(out_counts_ptr or None), ctypes.c_void_p(stream or None)))


# ---- reference-signature free functions (drop-in) --------------------------------
def _index_for(graph_or_index, base) -> GpuIndex:
    if isinstance(graph_or_index, GpuIndex):
        return graph_or_index
    return GpuIndex(graph_or_index, base)


def large_batch_search(graph, base, queries, params: BestFirstParams = BestFirstParams(),
                       stats: Optional[SearchStats] = None) -> List[np.ndarray]:
    """tsdg::large_batch_search (bestfirst_search.cpp:129-150)."""
    idx = _index_for(graph, base)
    if _f32rows(queries).shape[1] != idx.d:
        raise InvalidArgument("large_batch_search: dim mismatch")
    return idx.large_batch_search(queries, params, stats)


def bestfirst_search(graph, base, query, params: BestFirstParams, rng_index: int,
                     stats: Optional[SearchStats] = None) -> np.ndarray:
    """tsdg::bestfirst_search with the stream Rng64(params.seed).fork(rng_index)
    (the stream large_batch_search gives query rng_index)."""
    idx = _index_for(graph, base)
    r = idx.search_bestfirst(query, params, query_index_base=rng_index)
    if stats is not None:
        stats.add(r.stats)
    return r.lists()[0]


def small_batch_search(graph, base, queries, k: int, params: GreedyParams = GreedyParams(),
                       stats: Optional[SearchStats] = None) -> List[np.ndarray]:
    """tsdg::small_batch_search (greedy_search.cpp:106-127)."""
    idx = _index_for(graph, base)
    if _f32rows(queries).shape[1] != idx.d:
        raise InvalidArgument("small_batch_search: dim mismatch")
    return idx.small_batch_search(queries, k, params, stats)


def small_batch_search_one(graph, base, query, k: int, params: GreedyParams,
                           stats: Optional[SearchStats] = None) -> np.ndarray:
    """tsdg::small_batch_search_one (greedy_search.cpp:74-104)."""
    return small_batch_search(graph, base, _f32rows(query), k, params, stats)[0]


__all__ = ["BestFirstParams", "GreedyParams", "SearchStats", "SearchResult", "TsdgGraph",
           "GpuIndex", "load_tsdg", "large_batch_search", "bestfirst_search",
           "small_batch_search", "small_batch_search_one", "merge_shards_device",
           "GroundTruth", "KnnGraph", "ground_truth", "exact_topk", "brute_force_knn",
           "BuildStats", "build", "nn_descent", "MultiGpuIndex", "ShardedGpuIndex",
           "InvalidArgument", "TsdgRuntimeError", "KINVALID", "QUERY_STATS_DTYPE"]

