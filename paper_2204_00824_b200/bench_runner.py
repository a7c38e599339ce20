"""GPU port of the reference's JSON bench runner:
tsdg::run_bench_file (bench.cpp:189-362) with the same config keys and defaults,
the same sweep expansion and auto routing, the same per-chunk seeding
(bp.seed = mix64(seed + begin), bench.cpp:331-333), the same recall (bench.cpp:59-78)
and the same CSV (write_bench_csv, bench.cpp:177-187).  Every piece of work runs on
the B200: ground truth by the exact scan, the graph (when not loaded) by the GPU
brute-force k-NN or nn_descent + two-stage diversification, the searches by the best-first /
greedy kernels (deterministic mode by default: the same traversal, so recall,
mean_hops and mean_distance_evals equal the reference's row for row).

    python -m paper_2204_00824_b200.bench_runner config.json [out.csv] [--fast]

Graph method "nndescent" (bench.cpp:245-247, keys iterations / sample_rate / knn_seed
with the reference's defaults 10 / 1.0 / 7) runs the GPU nn_descent, which returns the
reference's KnnGraph bit for bit.
"""
from __future__ import annotations

import json
import math
import os
import struct
import sys
import time
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from . import _native, datasets
from .search import (BestFirstParams, GpuIndex, GreedyParams, InvalidArgument, KnnGraph,
                     SearchStats, TsdgRuntimeError, brute_force_knn, build, ground_truth,
                     load_tsdg, nn_descent)

METRIC_NAMES = {0: "l2", 1: "cos", 2: "ip"}


def metric_from_name(name: str) -> int:
    """vectors.cpp:29-34"""
    if name == "l2":
        return 0
    if name in ("cos", "cosine"):
        return 1
    if name in ("ip", "innerproduct"):
        return 2
    raise InvalidArgument(f"unknown metric '{name}' (expected l2, cos, or ip)")


def mix64(z: int) -> int:
    """common.hpp splitmix64 finaliser (uint64 arithmetic)."""
    m = 0xFFFFFFFFFFFFFFFF
    z &= m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def _fmt(v) -> str:
    """std::ostream default formatting of a double (precision 6, %g style)."""
    if isinstance(v, float):
        if math.isinf(v):
            return "inf" if v > 0 else "-inf"
        if math.isnan(v):
            return "nan"
        return f"{v:g}"
    return str(v)


# ---- file formats (io.cpp:75-164) ------------------------------------------------
def _load_records(path: str, dtype, name: str) -> np.ndarray:
    if not os.path.exists(path):
        raise TsdgRuntimeError(f"{path}: cannot open for reading")
    raw = np.fromfile(path, np.uint8)
    itemsize = np.dtype(dtype).itemsize
    if raw.size < 4:
        raise TsdgRuntimeError(f"{path}: empty dataset")
    d = int(np.frombuffer(raw[:4].tobytes(), "<i4")[0])
    if d <= 0:
        raise TsdgRuntimeError(f"{path}: invalid dimension {d} at record 0 (byte offset 0)")
    rec = 4 + itemsize * d
    if raw.size % rec:
        raise TsdgRuntimeError(f"{path}: truncated record")
    n = raw.size // rec
    r = raw.reshape(n, rec)
    dims = r[:, :4].copy().view("<i4").reshape(n)
    bad = np.nonzero(dims != d)[0]
    if bad.size:
        i = int(bad[0])
        raise TsdgRuntimeError(f"{path}: inconsistent dimension at record {i} (byte offset "
                               f"{i * rec}): got {int(dims[i])}, expected {d}")
    vals = r[:, 4:].copy().view(dtype).reshape(n, d).astype(np.float32)
    if not np.isfinite(vals).all():
        i, j = map(int, np.argwhere(~np.isfinite(vals))[0])
        raise TsdgRuntimeError(f"{path}: non-finite value at record {i} component {j}")
    return vals


def load_vectors(path: str) -> np.ndarray:
    """io.cpp:116-121: .bvecs widened to fp32, anything else read as fvecs."""
    if path.endswith(".bvecs"):
        return _load_records(path, np.uint8, "bvecs")
    return _load_records(path, "<f4", "fvecs")


def load_ivecs(path: str) -> List[np.ndarray]:
    """io.cpp:132-152"""
    if not os.path.exists(path):
        raise TsdgRuntimeError(f"{path}: cannot open for reading")
    raw = open(path, "rb").read()
    out, off = [], 0
    while off < len(raw):
        if off + 4 > len(raw):
            raise TsdgRuntimeError(f"{path}: truncated record length at byte offset {off}")
        (k,) = struct.unpack_from("<i", raw, off)
        if k < 0:
            raise TsdgRuntimeError(f"{path}: negative record length at byte offset {off}")
        if off + 4 + 4 * k > len(raw):
            raise TsdgRuntimeError(f"{path}: truncated record ids at byte offset {off}")
        out.append(np.frombuffer(raw, "<i4", k, off + 4).astype(np.uint32))
        off += 4 + 4 * k
    if not out:
        raise TsdgRuntimeError(f"{path}: empty dataset")
    return out


def normalized_copy(x: np.ndarray) -> np.ndarray:
    """vectors.cpp:68-80: norm = sqrt(dot(r, r)) with the reference's sequential fp32
    dot (one rounding per multiply and per add, dimension order), then r[j] / norm."""
    x = np.ascontiguousarray(x, np.float32)
    acc = np.zeros(x.shape[0], np.float32)
    for j in range(x.shape[1]):
        acc = acc + x[:, j] * x[:, j]
    norm = np.sqrt(acc)
    if (norm == 0).any():
        i = int(np.nonzero(norm == 0)[0][0])
        raise ValueError(f"normalized_copy: zero-norm vector at row {i}")
    return x / norm[:, None]


def recall_at_k(results: List[np.ndarray], gt_ids: List[np.ndarray], gt_k: int, k: int) -> float:
    """bench.cpp:59-78"""
    if k < 1:
        raise InvalidArgument("recall_at_k: k must be >= 1")
    if k > gt_k:
        raise InvalidArgument("recall_at_k: k exceeds ground-truth depth")
    if len(results) != len(gt_ids):
        raise InvalidArgument("recall_at_k: query count mismatch")
    hits = 0
    for r, g in zip(results, gt_ids):
        want = set(int(x) for x in g[:k])
        hits += sum(1 for x in r[:k] if int(x) in want)
    return hits / (len(results) * k)


@dataclass
class BenchRow:
    """tsdg::BenchRow (bench.hpp:47-57)"""
    dataset: str
    algorithm: str
    batch_size: int
    params: str
    k: int
    recall: float
    qps: float
    mean_hops: float
    mean_distance_evals: float


def write_bench_csv(rows: List[BenchRow], path: str) -> None:
    """bench.cpp:177-187"""
    with open(path, "w") as f:
        f.write("dataset,algorithm,batch_size,params,k,recall,qps,mean_hops,mean_distance_evals\n")
        for r in rows:
            f.write(",".join([r.dataset, r.algorithm, str(r.batch_size), r.params, str(r.k),
                              _fmt(r.recall), _fmt(r.qps), _fmt(r.mean_hops),
                              _fmt(r.mean_distance_evals)]) + "\n")


def _sweep(j: dict, key: str, fallback: float) -> List[float]:
    """bench.cpp:158-167 as_sweep"""
    if key not in j:
        return [float(fallback)]
    v = j[key]
    if isinstance(v, list):
        if not v:
            raise TsdgRuntimeError(f"empty sweep for {key}")
        return [float(x) for x in v]
    return [float(v)]


def run_bench_file(config_path: str, csv_out: str = "", device: int = 0,
                   mode: int = _native.MODE_DETERMINISTIC) -> List[BenchRow]:
    """tsdg::run_bench_file (bench.cpp:189-362) on the GPU."""
    if not os.path.exists(config_path):
        raise TsdgRuntimeError(f"{config_path}: cannot open config")
    with open(config_path) as f:
        cfg = json.load(f)
    dcfg = cfg["dataset"]
    metric = metric_from_name(dcfg.get("metric", "l2"))
    dataset_name = dcfg.get("name", "dataset")
    if "synthetic" in dcfg:
        s = dcfg["synthetic"]
        base, queries = datasets.make_synthetic_split(
            int(s["n"]), int(s.get("queries", 100)), int(s["d"]), int(s["clusters"]),
            float(s["spread"]), int(s.get("seed", 1)))
    else:
        base = load_vectors(dcfg["data"])
        queries = load_vectors(dcfg["queries"])
    if metric == 1:
        base, queries = normalized_copy(base), normalized_copy(queries)
    nq = queries.shape[0]

    gt_k = int(dcfg.get("gt_k", 100))
    if "gt" in dcfg:
        rows = load_ivecs(dcfg["gt"])
        if any(len(r) < gt_k for r in rows):
            raise TsdgRuntimeError("bench: ground-truth record shorter than gt_k")
        if len(rows) != nq:
            raise TsdgRuntimeError("bench: ground-truth record count does not match queries")
        gt_ids = rows
    else:
        gt_k = min(gt_k, base.shape[0])
        gt_ids = list(ground_truth(base, queries, gt_k, metric, device).ids)

    gcfg = cfg["graph"]
    if "tsdg" in gcfg:
        graph = load_tsdg(gcfg["tsdg"])
        if graph.metric != metric:
            raise TsdgRuntimeError("bench: graph metric does not match dataset metric")
    else:
        knn_k = int(gcfg.get("knn_k", 100))
        if gcfg.get("method", "brute") == "nndescent":
            knn = nn_descent(base, knn_k, int(gcfg.get("iterations", 10)),
                             float(gcfg.get("sample_rate", 1.0)), int(gcfg.get("knn_seed", 7)),
                             metric, device)
        else:
            knn = brute_force_knn(base, knn_k, metric, device)
        graph = build(base, knn, float(gcfg.get("alpha", 1.2)), int(gcfg.get("lambda0", 9)),
                      int(gcfg.get("max_degree", 0)), metric, device)
    threshold = int(cfg.get("routing", {}).get("small_batch_threshold", 256))

    points = []
    for r in cfg["runs"]:
        algorithm = r.get("algorithm", "auto")
        batch_size = int(r.get("batch_size", nq))
        if algorithm == "auto":
            algorithm = "greedy" if batch_size <= threshold else "bestfirst"
        k = int(r.get("k", 10))
        seed = int(r.get("seed", 7))
        greedy = algorithm == "greedy"
        t0s = _sweep(r, "t0", 16) if greedy else [0.0]
        hopss = _sweep(r, "T", 16 if greedy else 1024)
        cuts = _sweep(r, "lambda_cut", 10 if greedy else 5)
        deltas = [0.0] if greedy else _sweep(r, "delta", 0.0)
        for t0 in t0s:
            for hops in hopss:
                for cut in cuts:
                    for delta in deltas:
                        bs = max(1, min(batch_size, nq))
                        if greedy:
                            p = GreedyParams(int(t0), int(hops), int(cut), seed)
                            echo = f"t0={p.t0};T={p.hop_limit};lambda_cut={p.lambda_cut};seed={seed}"
                        else:
                            p = BestFirstParams(k, int(hops), float(np.float32(delta)),
                                                int(r.get("m_segments", 8)), int(cut), seed,
                                                bool(r.get("unbounded", False)))
                            echo = (f"T={p.hop_limit};delta={_fmt(float(delta))};"
                                    f"m_segments={p.m_segments};lambda_cut={p.lambda_cut};"
                                    f"seed={seed};unbounded={1 if p.unbounded else 0}")
                        echo += f";metric={METRIC_NAMES[metric]}"
                        points.append((algorithm, bs, k, p, echo))

    idx = GpuIndex(graph, base, device)
    out_rows = []
    try:
        for algorithm, bs, k, p, echo in points:
            def run_all():
                results: List[np.ndarray] = [None] * nq
                stats = SearchStats()
                for begin in range(0, nq, bs):
                    chunk = queries[begin:min(nq, begin + bs)]
                    if algorithm == "greedy":
                        part = idx.small_batch_search(chunk, k, p, stats, mode=mode)
                    else:
                        bp = BestFirstParams(**{**p.__dict__, "seed": mix64(p.seed + begin)})
                        part = idx.large_batch_search(chunk, bp, stats, mode=mode)
                    results[begin:begin + len(part)] = part
                return results, stats

            run_all()  # warm-up (bench.cpp:342)
            t0 = time.perf_counter()
            results, stats = run_all()
            seconds = time.perf_counter() - t0
            out_rows.append(BenchRow(
                dataset_name, algorithm, bs, echo, k,
                recall_at_k(results, gt_ids, gt_k, min(k, gt_k)),
                nq / seconds if seconds > 0 else 0.0,
                stats.hops / nq, stats.distance_evals / nq))
    finally:
        idx.close()
    if csv_out:
        write_bench_csv(out_rows, csv_out)
    return out_rows


def main(argv=None) -> None:
    argv = list(sys.argv[1:] if argv is None else argv)
    fast = "--fast" in argv
    argv = [a for a in argv if a != "--fast"]
    if not argv:
        raise SystemExit("usage: python -m paper_2204_00824_b200.bench_runner config.json [out.csv] [--fast]")
    rows = run_bench_file(argv[0], argv[1] if len(argv) > 1 else "",
                          mode=_native.MODE_FAST if fast else _native.MODE_DETERMINISTIC)
    for r in rows:
        print(f"{r.dataset} {r.algorithm} batch={r.batch_size} {r.params} k={r.k} "
              f"recall={_fmt(r.recall)} qps={_fmt(r.qps)} hops={_fmt(r.mean_hops)} "
              f"evals={_fmt(r.mean_distance_evals)}")


if __name__ == "__main__":
    main()
