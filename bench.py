"""Benchmark: QPS at recall@10 >= 0.95, SIFT1M-shaped TSDG search, batch 10K (config C2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step = one large-batch best-first search (paper Alg. 2) of the whole 10K-query
batch over the 1M x 128 fp32 low-LID clustered set (SURVEY.md §8(d) recipe 2),
TSDG built by the reference's CPU builder (nn_descent k=64 + build(1.2, 9),
tools/make_dataset.py) and loaded unchanged.  Search parameters are fixed at the
recall >= 0.95 operating point (k_search=14, delta=0, lambda_cut=5, m=8,
T=1024, seed=7: recall@10 0.957, identical for the reference's own search; the
sweep in profiles/recall_qps_c2_*.jsonl picks the cheapest point with a clear margin —
k_search=13 reaches 0.9504).

ours:      `value` = device-resident throughput (queries already in HBM; CUDA events
           on the launching stream around each step; L2 flushed between steps);
           `e2e`   = same search through the reference-facing C-ABI call with HOST
           buffers (pinned), H2D of the queries and D2H of ids/dists/counts inside
           the timed region (pinned buffers take the zero-copy path: the kernel
           reads each query from host memory and writes its results back over the
           bus while the search runs; TSDG_ZERO_COPY=0 selects the copy pipeline).
reference: the reference's own CPU large_batch_search (oracle/_ref, unmodified,
           OpenMP on all host cores) on the same config.
Multi-GPU (torchrun, one process per GPU): the index is replicated; each rank
searches its own 10K-query batch (query_index_base = rank * 10K, so every query
keeps its reference RNG stream) — weak scaling, no data-path collective.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DATASET = "c2_lowlid_1m"
PARAMS = dict(k=14, hop_limit=1024, delta=0.0, m_segments=8, lambda_cut=5, seed=7)
METRIC = "QPS at recall@10>=0.95 (SIFT1M-shape 1Mx128 fp32 L2, batch 10K)"
WORKLOAD = "C2: SIFT1M-shaped 1Mx128 fp32 L2 low-LID clustered, TSDG (reference nn_descent k=64 + build(1.2,9)), large batch 10K queries, best-first"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def recall_at_k(ids: np.ndarray, counts: np.ndarray, gt: np.ndarray, k: int) -> float:
    """bench.cpp:59-78: |results[0..k) & truth[0..k)| / (nq * k), vectorised."""
    nq = ids.shape[0]
    cols = np.arange(ids.shape[1])[None, :]
    got = np.where((cols < np.minimum(counts, k)[:, None]) & (cols < k), ids.astype(np.int64), -1)
    want = np.sort(gt[:, :k].astype(np.int64), axis=1)
    hits = 0
    for q in range(nq):  # sets are tiny (k <= 100); searchsorted per row
        g = got[q][got[q] >= 0]
        pos = np.searchsorted(want[q], g)
        pos = np.minimum(pos, k - 1)
        hits += int((want[q][pos] == g).sum())
    return hits / (nq * k)


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


def profiled_traffic(mode: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the search kernel, from
    the committed ncu capture of this configuration (profiles/traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        e = t.get(mode)
        return None if e is None else int(e["dram_bytes_read"] + e["dram_bytes_write"])
    except Exception:
        return None


SHARDED = "c5s_lowlid_2m_96"
C4 = "c4_lowlid_1m_960"


def _events_time(fn, steps, stream=None):
    import torch
    evs = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


def small_batch_section(idx, ds, dev, ref_fx=None):
    """C3: Alg. 1 (greedy, CTA/cluster-per-query procedure) on the C2 index at batch
    1 / 8 / 64, at the cheapest t0 whose recall@10 reaches 0.95 (the reference's
    small_batch_search gives the same ids: deterministic mode is bit-exact).
      device:  launch path, queries resident in HBM, CUDA events around each call
      e2e:     the host-pointer C-ABI call (tsdg_gpu_search_greedy) with pinned HOST
               query / result buffers (zero-copy: the kernel reads the queries from and
               writes the results to host memory), wall clock around each synchronous call
      reference: the reference's small_batch_search (oracle/_ref, all host threads)
               on the same queries, wall clock per call"""
    import torch

    from paper_2204_00824_b200.search import GreedyParams

    k = 10
    # cheapest t0 reaching recall@10 >= 0.95 on the first 2000 queries (untimed)
    t0_pick, sweep = None, {}
    for t0 in (8, 10, 12, 16):
        p = GreedyParams(t0=t0, hop_limit=16, lambda_cut=10, seed=7)
        r = idx.search_greedy(ds.queries[:2000], k, p)
        sweep[t0] = recall_at_k(r.ids, r.counts, ds.gt[:2000], 10)
        if sweep[t0] >= 0.95:
            t0_pick = t0
            break
    t0_pick = t0_pick or 16
    p = GreedyParams(t0=t0_pick, hop_limit=16, lambda_cut=10, seed=7)
    out = []
    for batch in (1, 8, 64):
        reps = 256 if batch == 1 else max(32, 1024 // batch)
        nq = reps * batch
        row = {"batch": batch, "t0": p.t0}
        dq = torch.from_numpy(ds.queries[:nq]).to(dev)
        ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
        dd = torch.empty((nq, k), dtype=torch.float32, device=dev)
        cc = torch.empty(nq, dtype=torch.int32, device=dev)
        st = torch.cuda.current_stream(dev).cuda_stream

        def call(j):
            idx.search_greedy_device(dq[j * batch].data_ptr(), batch, k, p, ids[j * batch].data_ptr(),
                                     dd[j * batch].data_ptr(), cc[j * batch].data_ptr(), 0, st)

        for j in range(3):
            call(j)
        torch.cuda.synchronize()
        times = []
        for j in range(reps):  # one call at a time: latency, not throughput
            times += _events_time(lambda: call(j), 1)
        row["recall_at_10"] = recall_at_k(ids.cpu().numpy().view(np.uint32), cc.cpu().numpy(),
                                          ds.gt[:nq], 10)
        row["recall_at_1"] = recall_at_k(ids.cpu().numpy().view(np.uint32), cc.cpu().numpy(),
                                         ds.gt[:nq], 1)
        lat = float(np.median(times))
        row["device"] = {"latency_us_p50": lat * 1e3, "latency_us_p99": float(np.percentile(times, 99)) * 1e3,
                         "qps": batch / lat * 1e3}
        dev_ids = ids.cpu().numpy().view(np.uint32).copy()
        # end to end with host buffers through the reference-facing C-ABI call
        hq = torch.from_numpy(ds.queries[:nq].copy()).pin_memory()
        hi = torch.empty((nq, k), dtype=torch.int32).pin_memory()
        hd = torch.empty((nq, k), dtype=torch.float32).pin_memory()
        hc = torch.empty(nq, dtype=torch.int32).pin_memory()
        L = _native_lib()
        pc = p.c()

        def lcall(j):
            o = j * batch
            _native_check(L.tsdg_gpu_search_greedy(
                idx.handle, ctypes.c_void_p(hq[o].data_ptr()), batch, k, ctypes.byref(pc), 0,
                ctypes.c_void_p(hi[o].data_ptr()), ctypes.c_void_p(hd[o].data_ptr()),
                ctypes.c_void_p(hc[o].data_ptr()), None))

        for j in range(3):
            lcall(j)
        lat_l = []
        for j in range(reps):
            t = time.perf_counter()
            lcall(j)
            lat_l.append(time.perf_counter() - t)
        assert np.array_equal(hi.numpy().view(np.uint32), dev_ids), "e2e result differs"
        m = float(np.median(lat_l))
        row["e2e"] = {"path": "tsdg_gpu_search_greedy, pinned host buffers (zero-copy)",
                      "latency_us_p50": m * 1e6, "latency_us_p99": float(np.percentile(lat_l, 99)) * 1e6,
                      "qps": batch / m, "h2d_bytes_per_call": batch * ds.queries.shape[1] * 4,
                      "d2h_bytes_per_call": batch * (k * 8 + 4)}
        if ref_fx is not None:
            rr = min(reps, 64 if batch < 64 else 8)
            ref_fx.small_batch(ds.queries[:batch], k, p)
            lat_r = []
            for j in range(rr):
                t = time.perf_counter()
                r_ids, _, _ = ref_fx.small_batch(ds.queries[j * batch:(j + 1) * batch], k, p)
                lat_r.append(time.perf_counter() - t)
                assert np.array_equal(r_ids, dev_ids[j * batch:(j + 1) * batch]), "reference differs"
            mr = float(np.median(lat_r))
            row["reference"] = {"latency_us_p50": mr * 1e6, "qps": batch / mr,
                                "cores": ref_fx.ref.so.ref_num_threads(), "calls": rr,
                                "ids_equal": True}
        out.append(row)
    return {"procedure": "greedy (paper Alg. 1), deterministic, C2 index, hop_limit 16, lambda_cut 10",
            "t0_rule": "cheapest t0 in (8, 10, 12, 16) with recall@10 >= 0.95 on 2000 queries",
            "t0_recall_sweep": {str(t): v for t, v in sweep.items()}, "points": out}


def _native_lib():
    from paper_2204_00824_b200 import _native
    return _native.lib()


def _native_check(rc):
    from paper_2204_00824_b200 import _native
    _native.check(rc)


def sharded_section(args, ws, rank, local, dev, dist):
    """Sharded base (C5 shape, scaled to 2M x 96 in 8 shards): each rank searches all
    queries on its 8/N shards, NCCL all-gather of per-shard top-k, device merge."""
    from paper_2204_00824_b200 import _native, datasets, shards
    from paper_2204_00824_b200.search import BestFirstParams, load_tsdg

    import torch

    d = os.path.join(datasets.DATA_DIR, SHARDED)
    if not os.path.exists(os.path.join(d, "meta.json")):
        return {"unavailable": f"data/{SHARDED} missing (tools/make_sharded.py)"}
    with open(os.path.join(d, "meta.json")) as f:
        meta = json.load(f)
    if 8 % ws:
        return {"unavailable": f"8 shards do not split over {ws} GPUs"}
    base, queries = datasets.generate(meta["spec"])
    table = [(s["offset"], s["n"]) for s in meta["shards"]]
    mine = shards.shards_of_rank(len(table), ws, rank)
    graphs, bases = {}, {}
    from tools import graph_pack
    for s in mine:
        path = os.path.join(d, f"shard_{s}.tsdg")
        off, n = table[s]
        if not os.path.exists(path):
            bpath, _ = datasets.ensure_fvecs(SHARDED, base, queries)
            graph_pack.unpack(os.path.join(d, f"shard_{s}.pk"), bpath, path, off)
        graphs[s] = load_tsdg(path)
        bases[s] = base[off:off + n]
    searcher = shards.ShardedSearcher(graphs, bases, table, device=local,
                                      group=dist.group.WORLD if ws > 1 else None)
    p = BestFirstParams(k=16, seed=7)
    qd = torch.from_numpy(queries).to(dev)
    mode = _native.MODE_FAST if args.mode == "fast" else _native.MODE_DETERMINISTIC
    for _ in range(3):
        ids, dists, counts = searcher.search(qd, p, mode=mode)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    steps = max(5, args.steps // 2)
    times = _events_time(lambda: searcher.search(qd, p, mode=mode), steps)
    total = sum(times) / 1e3
    if ws > 1:
        t = torch.tensor([total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = float(t.item())
    ids, dists, counts = searcher.search(qd, p, mode=mode)
    gt = np.fromfile(os.path.join(d, "gt.u32"), np.uint32).reshape(meta["gt_queries"], meta["gt_k"])
    nq_gt = gt.shape[0]
    rec = recall_at_k(ids[:nq_gt].cpu().numpy().view(np.uint32), counts[:nq_gt].cpu().numpy(), gt, 10)
    nq = queries.shape[0]
    return {"workload": f"{meta['spec']['n']}x{meta['spec']['d']} fp32 in {len(table)} shards "
                        "(Deep100M-shape scaled 50x), TSDG per shard from the reference builder",
            "params": {"k": p.k, "lambda_cut": p.lambda_cut, "m_segments": p.m_segments,
                       "delta": p.delta, "seed": p.seed}, "mode": args.mode,
            "n_gpus": ws, "shards_per_gpu": len(mine), "queries": nq,
            "value": nq * steps / total, "unit": "queries/s (every query searched on all shards)",
            "ms_per_step": total / steps * 1e3, "recall_at_10": rec,
            "collective": "all_gather_into_tensor (NCCL) of per-shard (ids, dists, counts)" if ws > 1 else "none (1 GPU)"}


def c4_section(args, dev):
    """GIST1M shape (1M x 960 fp32), batch 10K, replicated index, one GPU."""
    import torch

    from paper_2204_00824_b200 import _native, datasets
    from paper_2204_00824_b200.search import BestFirstParams, GpuIndex, load_tsdg

    if not datasets.available(C4):
        return {"unavailable": f"data/{C4} missing (tools/make_dataset.py --d 960)"}
    ds = datasets.load(C4)
    idx = GpuIndex(load_tsdg(ds.graph_path), ds.base, device=dev.index or 0)
    nq = ds.queries.shape[0]
    dq = torch.from_numpy(ds.queries).to(dev)
    best = None
    for k in (10, 16, 24, 32):
        p = BestFirstParams(k=k, seed=7)
        ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
        dd = torch.empty((nq, k), dtype=torch.float32, device=dev)
        cc = torch.empty(nq, dtype=torch.int32, device=dev)
        stt = torch.empty((nq, 4), dtype=torch.int32, device=dev)
        mode = _native.MODE_FAST if args.mode == "fast" else _native.MODE_DETERMINISTIC
        st = torch.cuda.current_stream(dev).cuda_stream

        def call():
            idx.search_bestfirst_device(dq.data_ptr(), nq, p, ids.data_ptr(), dd.data_ptr(),
                                        cc.data_ptr(), stt.data_ptr(), st, mode=mode)

        for _ in range(2):
            call()
        torch.cuda.synchronize()
        rec = recall_at_k(ids.cpu().numpy().view(np.uint32), cc.cpu().numpy(), ds.gt, 10)
        times = _events_time(call, 5)
        s = stt.cpu().numpy().astype(np.int64)
        alg = 4 * 960 * s[:, 1].sum() + 4 * s[:, 3].sum() + nq * (4 * 960 + 8 * k)
        ms = float(np.median(times))
        best = {"k_search": k, "recall_at_10": rec, "value": nq / ms * 1e3, "unit": "queries/s",
                "ms_per_batch": ms, "roofline_achieved_GBps": alg / ms / 1e6,
                "roofline_frac": alg / ms / 1e6 / peaks()[0], "alg_bytes_per_launch": int(alg)}
        if rec >= 0.95:
            break
    idx.close()
    traffic = profiled_traffic("c4_fast") if args.mode == "fast" else None
    return {"workload": "GIST1M-shaped 1M x 960 fp32 L2 low-LID (latent 26), batch 10K, "
                        "TSDG from the reference builder (nn_descent k=64)", **best,
            "traffic": traffic, "traffic_capture": "profiles/r2_bf_staged_c4.md (k_search=24)"}


def gpu_local_cpus(device: int):
    """Host CPUs attached to `device` (NVML CPU affinity), or None.  The host-pointer
    (zero-copy) path streams queries and results between pinned host memory and the
    GPU while the kernel runs, so the pinned buffers belong on the GPU's own NUMA node:
    the process runs on those CPUs while it allocates and times them (the CPU baseline
    gets every core back)."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(device)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, 16)
        cpus = {w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        avail = os.sched_getaffinity(0)
        cpus &= avail
        return cpus if cpus and cpus != avail else None
    except Exception:
        return None


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


PREPARE = os.path.join(ROOT, "paper_2204_00824_b200", "_lib", "tsdg_prepare")


def reference_inputs(name: str):
    """Input files of `name` in the reference's formats, made (untimed) by the
    tools/prepare_inputs.c executable when missing: base.fvecs / queries.fvecs
    (checksum-verified seeded vectors) and graph.tsdg (rebuilt byte-identically from
    graph.pk).  Returns (graph.tsdg, base.fvecs, queries.fvecs, gt).  Loads nothing
    of this repository into the calling process."""
    d = os.path.join(ROOT, "data", name)
    with open(os.path.join(d, "meta.json")) as f:
        meta = json.load(f)
    sp = meta["spec"]
    bpath, qpath, gpath = (os.path.join(d, x) for x in ("base.fvecs", "queries.fvecs", "graph.tsdg"))
    if not (os.path.exists(bpath) and os.path.exists(qpath)):
        subprocess.run([PREPARE, "vectors", sp["kind"], str(sp["n"]), str(sp["nq"]), str(sp["d"]),
                        str(sp.get("latent", 0)), str(sp["clusters"]), repr(float(sp["spread"])),
                        str(sp["seed"]), repr(float(sp.get("noise", 0.0))), bpath, qpath,
                        meta["checksums"]["base"], meta["checksums"]["queries"]], check=True)
    if not os.path.exists(gpath):
        subprocess.run([PREPARE, "unpack", os.path.join(d, "graph.pk"), bpath, gpath], check=True)
    gt = np.fromfile(os.path.join(d, "gt.u32"), np.uint32).reshape(sp["nq"], meta["gt_k"])
    return gpath, bpath, qpath, gt


def bench_config(ws: int, scaling: str) -> dict:
    """The `config` object, identical on both arms."""
    per_gpu = 10000 if scaling == "weak" else 10000 // ws
    return {"workload": WORKLOAD, "params": PARAMS, "scaling": scaling,
            "queries_per_gpu": per_gpu, "global_batch": 10000 * ws if scaling == "weak" else 10000,
            "parallelism": f"replicated index, {'each rank its own 10K batch' if scaling == 'weak' else 'the 10K batch split'} x{ws}"}


def reference_arm(args, ws, rank):
    """The reference's own CPU implementation, unmodified (oracle/_ref, compiled from
    /root/reference): graph and vectors read by its load_tsdg / load_vectors, search
    by its large_batch_search on all host threads; nothing of this repository's
    search (or any library of it) is loaded into this process."""
    if rank != 0:
        return
    from oracle import oracle as O

    gpath, bpath, qpath, gt = reference_inputs(DATASET)
    ref = O.Ref()
    threads = ref.so.ref_num_threads()
    fx = ref.fixture_from_files(gpath, bpath)
    queries = ref.load_vectors(qpath)

    class P:  # BestFirstParams fields as the shim reads them
        pass
    p = P()
    for kk, vv in PARAMS.items():
        setattr(p, kk, vv)
    p.unbounded = False
    nq_step = min(args.ref_queries, queries.shape[0])
    q = queries[:nq_step]
    for _ in range(args.warmup):
        fx.large_batch(q, p)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ids, counts, st = fx.large_batch(q, p)
    dt = time.perf_counter() - t0
    qps = nq_step * args.steps / dt
    rec = recall_at_k(ids, counts, gt[:nq_step], 10)
    rec1 = recall_at_k(ids, counts, gt[:nq_step], 1)
    one = ref_one_thread(ref, fx, queries, p)
    line = {
        "impl": "reference", "metric": METRIC, "value": qps, "unit": "queries/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (low-LID clustered, seeded)",
        "config": bench_config(ws, args.scaling),
        "recall_at_10": rec, "recall_at_1": rec1,
        "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": threads, "kind": "reference",
                         "sample": f"{nq_step} of the 10K C2 queries per step, reference "
                                   f"large_batch_search (OpenMP, {threads} threads); inputs read "
                                   "by the reference's load_tsdg / load_vectors"},
        "cpu_baseline_1thread": one,
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def ref_one_thread(ref, fx, queries, p, seconds_budget=8.0):
    """bench.cpp:321-345 also times the search on one thread: a bounded sample."""
    full = ref.so.ref_num_threads()
    ref.so.ref_set_num_threads(1)
    try:
        fx.large_batch(queries[:50], p)
        t0 = time.perf_counter()
        done = 0
        while time.perf_counter() - t0 < seconds_budget and done < queries.shape[0]:
            chunk = queries[done:done + 250]
            fx.large_batch(chunk, p)
            done += chunk.shape[0]
        dt = time.perf_counter() - t0
    finally:
        ref.so.ref_set_num_threads(full)
    return {"value": done / dt, "unit": "queries/s", "cores": 1, "kind": "reference",
            "sample": f"first {done} C2 queries on 1 thread (~{seconds_budget:.0f}s)"}


def cpu_baseline(ds, seconds_budget=15.0):
    """Reference CPU search on a bounded sample (rank 0, N=1)."""
    from oracle import oracle as O
    from paper_2204_00824_b200.search import BestFirstParams

    ref = O.Ref()
    threads = ref.so.ref_num_threads()
    fx = ref.fixture(ds.graph_path, ds.base)
    p = BestFirstParams(**PARAMS)
    q = ds.queries[:500]
    fx.large_batch(q, p)
    t0 = time.perf_counter()
    done = 0
    while time.perf_counter() - t0 < seconds_budget and done < ds.queries.shape[0]:
        chunk = ds.queries[done:done + 2000]
        fx.large_batch(chunk, p)
        done += chunk.shape[0]
    dt = time.perf_counter() - t0
    return {"value": done / dt, "unit": "queries/s", "cores": threads, "kind": "reference",
            "sample": f"first {done} C2 queries, reference large_batch_search "
                      f"(oracle/_ref, unmodified, OpenMP {threads} threads), ~{seconds_budget:.0f}s",
            "one_thread": ref_one_thread(ref, fx, ds.queries, p)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--ref-queries", type=int, default=10000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mode", choices=["det", "fast"], default="fast")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="weak: every rank searches its own 10K batch; strong: the 10K batch "
                         "is split across the ranks (query_index_base = slice start)")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the small-batch / sharded / C4 secondary measurements")
    args = ap.parse_args()
    ws, rank, local = dist_env()

    if args.impl == "reference":
        reference_arm(args, ws, rank)
        return

    from paper_2204_00824_b200 import datasets

    if not datasets.available(DATASET):
        # data/ is prepared offline (tools/prepare_data.sh); when it is absent (a fresh
        # checkout) it is rebuilt here, untimed: the graph by the reference's CPU
        # builder (oracle/_ref, as for every benchmark graph), ground truth on the GPU
        cmd = [sys.executable, os.path.join(ROOT, "tools", "make_dataset.py"), "--name", DATASET,
               "--kind", "lowlid", "--n", "1000000", "--nq", "10000", "--d", "128", "--latent", "16",
               "--builder", "nndescent", "--knn-k", "64", "--iters", "5", "--gt", "gpu"]
        if ws > 1:  # one builder; the other ranks wait for its meta.json
            if rank == 0:
                subprocess.run(cmd, check=True, stdout=sys.stderr)
            t_wait = time.time()
            while not datasets.available(DATASET) and time.time() - t_wait < 3600:
                time.sleep(5)
        elif os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libtsdg_ref.so")):
            subprocess.run(cmd, check=True, stdout=sys.stderr)
        if not datasets.available(DATASET):
            raise SystemExit(f"data/{DATASET} missing and oracle/_ref is not built: "
                             "bash tools/prepare_data.sh c2")
    ds = datasets.load(DATASET)

    import torch
    import torch.distributed as dist

    from paper_2204_00824_b200 import _native
    from paper_2204_00824_b200.search import BestFirstParams, GpuIndex, load_tsdg

    all_cpus = os.sched_getaffinity(0)
    local_cpus = gpu_local_cpus(int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local)).split(",")[local])
                                if os.environ.get("CUDA_VISIBLE_DEVICES", "").replace(",", "").isdigit()
                                else local)
    if local_cpus:
        os.sched_setaffinity(0, local_cpus)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    graph = load_tsdg(ds.graph_path)
    idx = GpuIndex(graph, ds.base, device=local)
    p = BestFirstParams(**PARAMS)
    k = p.k
    if args.scaling == "strong":  # this rank's contiguous slice of the one 10K batch
        from paper_2204_00824_b200 import shards
        lo, hi = shards.query_slice(ds.queries.shape[0], ws, rank)  # gloo-tested split
        queries, gt, qbase = ds.queries[lo:hi], ds.gt[lo:hi], lo
        total_q = ds.queries.shape[0]
    else:  # every rank its own 10K batch, RNG streams continued (query_index_base)
        queries, gt, qbase = ds.queries, ds.gt, rank * ds.queries.shape[0]
        total_q = ds.queries.shape[0] * ws
    nq = queries.shape[0]

    stream = torch.cuda.Stream(device=dev)
    sptr = stream.cuda_stream
    dq = torch.from_numpy(queries).to(dev)
    d_ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
    d_dists = torch.empty((nq, k), dtype=torch.float32, device=dev)
    d_counts = torch.empty(nq, dtype=torch.int32, device=dev)
    d_stats = torch.empty((nq, 4), dtype=torch.int32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    d = ds.base.shape[1]

    def max_over_ranks(x: float) -> float:
        if ws == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def device_timed(mode: int, clk_sampler=None):
        def step():
            idx.search_bestfirst_device(dq.data_ptr(), nq, p, d_ids.data_ptr(), d_dists.data_ptr(),
                                        d_counts.data_ptr(), d_stats.data_ptr(), sptr,
                                        query_index_base=qbase, mode=mode)

        # the clock sampler (nvidia-smi) starts before the warm-up so that its start-up
        # is outside the timed region; the warm-up is W >= 3 steps, extended to at least
        # 0.25 s of GPU work (clocks, TLBs over the 1.2 GB index)
        ctx = clk_sampler if clk_sampler is not None else _Null()
        ctx.__enter__()
        t_w = time.perf_counter()
        with torch.cuda.stream(stream):
            for _ in range(max(args.warmup, 3)):
                step()
        torch.cuda.synchronize()
        while time.perf_counter() - t_w < 0.25:
            with torch.cuda.stream(stream):
                for _ in range(5):
                    step()
            torch.cuda.synchronize()
        ids = d_ids.cpu().numpy().view(np.uint32).copy()
        counts = d_counts.cpu().numpy().view(np.uint32)
        stats = d_stats.cpu().numpy().astype(np.uint64)
        rec = recall_at_k(ids, counts, gt, 10)
        rec1 = recall_at_k(ids, counts, gt, 1)
        evals, examined = int(stats[:, 1].sum()), int(stats[:, 3].sum())
        alg_bytes = int(4 * d * evals + 4 * examined + nq * (4 * d + 8 * k))
        launches0 = _native.lib().tsdg_gpu_launch_count()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(float(i))  # L2 flush outside the events
                evs[i][0].record(stream)
                step()
                evs[i][1].record(stream)
        torch.cuda.synchronize()
        ctx.__exit__(None, None, None)
        launches = _native.lib().tsdg_gpu_launch_count() - launches0
        total_s = max_over_ranks(sum(a.elapsed_time(b) for a, b in evs) / 1e3)
        return {"total_s": total_s, "value": total_q * args.steps / total_s, "recall_at_10": rec,
                "recall_at_1": rec1,
                "alg_bytes": alg_bytes, "evals": evals, "examined": examined, "ids": ids,
                "launches": int(launches)}

    head_mode = _native.MODE_FAST if args.mode == "fast" else _native.MODE_DETERMINISTIC
    other_mode = _native.MODE_DETERMINISTIC if args.mode == "fast" else _native.MODE_FAST
    clk = ClockSampler(local)
    head = device_timed(head_mode, clk)
    other = device_timed(other_mode)
    det = head if head_mode == _native.MODE_DETERMINISTIC else other
    kernel_s = head["total_s"] / args.steps  # one search kernel per step (+ a 4-byte memset)

    # ---- end-to-end through the host-pointer C-ABI call -----------------------------
    hq = torch.from_numpy(queries).pin_memory()
    h_ids = torch.empty((nq, k), dtype=torch.int32).pin_memory()
    h_d = torch.empty((nq, k), dtype=torch.float32).pin_memory()
    h_c = torch.empty(nq, dtype=torch.int32).pin_memory()
    pc = p.c()
    L = _native.lib()

    def e2e_step():
        _native.check(L.tsdg_gpu_search_bestfirst(
            idx.handle, ctypes.c_void_p(hq.data_ptr()), nq, qbase, ctypes.byref(pc), head_mode,
            ctypes.c_void_p(h_ids.data_ptr()), ctypes.c_void_p(h_d.data_ptr()),
            ctypes.c_void_p(h_c.data_ptr()), None))

    for _ in range(2):
        e2e_step()
    if ws > 1:
        dist.barrier()
    e2e_times = []
    for i in range(args.steps):
        flush.fill_(float(i))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_step()  # synchronous: returns after the D2H copies landed
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = max_over_ranks(sum(e2e_times))
    zero_copy = all(L.tsdg_gpu_host_buffer_mapped(ctypes.c_void_p(t.data_ptr()), t.numel() * t.element_size())
                    for t in (hq, h_ids, h_d, h_c)) and os.environ.get("TSDG_ZERO_COPY", "1") != "0"
    e2e_val = total_q * args.steps / e2e_s
    assert np.array_equal(h_ids.numpy().view(np.uint32), head["ids"]), "e2e result differs"

    if local_cpus:  # the reference (CPU baseline, small-batch reference) gets every core
        os.sched_setaffinity(0, all_cpus)

    # ---- secondary workloads (not the headline): small batch, sharded base, C4 -----
    extras = {}
    if not args.no_extras:
        del flush
        torch.cuda.empty_cache()
        if rank == 0:
            ref_fx = None
            if ws == 1 and not args.no_cpu_baseline:
                try:
                    from oracle import oracle as O
                    ref_fx = O.Ref().fixture(ds.graph_path, ds.base)
                except Exception:  # reference not built on this host
                    ref_fx = None
            extras["small_batch"] = small_batch_section(idx, ds, dev, ref_fx)
            del ref_fx
        extras["sharded"] = sharded_section(args, ws, rank, local, dev, dist)
        if rank == 0:
            idx.close()
            del dq, d_ids, d_dists, d_counts, d_stats
            torch.cuda.empty_cache()
            extras["c4_gist_shape"] = c4_section(args, dev)

    if rank == 0:
        peak, peak_kind = peaks()
        achieved = head["alg_bytes"] / kernel_s / 1e9
        cpu = None
        if ws == 1 and not args.no_cpu_baseline:
            try:
                cpu = cpu_baseline(ds)
            except Exception as e:  # reference not built on this host
                cpu = {"value": None, "unavailable": str(e)}
        traffic = profiled_traffic(args.mode)
        line = {
            "metric": METRIC, "value": head["value"], "unit": "queries/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": head["total_s"] / args.steps * 1e3,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (low-LID clustered generator, seeded); graph built by the reference CPU builder",
            "config": bench_config(ws, args.scaling),
            "mode": args.mode,
            "recall_at_10": head["recall_at_10"], "recall_at_1": head["recall_at_1"],
            "recall_reference_order": {"recall_at_10": det["recall_at_10"],
                                       "recall_at_1": det["recall_at_1"],
                                       "note": "deterministic mode = the reference's results bit for bit"},
            "l2": "flushed between timed steps (256 MB write); inputs also exceed L2 "
                  "(512 MB vectors + padded adjacency)",
            "modes": {
                "det": {"value": det["value"], "recall_at_10": det["recall_at_10"],
                        "recall_at_1": det["recall_at_1"],
                        "note": "bit-exact with the reference (ids, distances, counters)"},
                "fast": {"value": (head if head is not det else other)["value"],
                         "recall_at_10": (head if head is not det else other)["recall_at_10"],
                         "recall_at_1": (head if head is not det else other)["recall_at_1"],
                         "note": "register-direct warp-cooperative gathers, FMA distances; "
                                 "recall@1/@10 must stay within 0.5 pt of det"},
            },
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "alg_bytes_per_step": head["alg_bytes"],
                         "alg_bytes_formula": "4*d*E_q + 4*A_q + 4*d + 8*k summed over queries",
                         "evals_per_query": head["evals"] / nq,
                         "edges_per_query": head["examined"] / nq},
            "e2e": {"value": e2e_val, "unit": "queries/s",
                    "h2d_bytes_per_step": int(queries.nbytes),
                    "d2h_bytes_per_step": int(nq * k * 8 + nq * 4),
                    "host_cpus": f"{len(local_cpus)} GPU-local CPUs (NVML affinity)" if local_cpus else "all",
                    "transfer": "zero-copy (kernel reads/writes pinned host memory)"
                    if zero_copy else "copy pipeline (2 chunks, 2 streams)"},
            "gpu_launches": head["launches"],
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            **extras,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
