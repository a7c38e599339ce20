"""Kernel-variant sweep on one GPU (development tool; bench.py is the contract).
Loads the C2 dataset once, then times each (mode, TSDG_STAGE, TSDG_PREFETCH)
variant with CUDA events, L2 flushed between steps.  Prints one JSON line each."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import recall_at_k  # noqa: E402  (bench.cpp:59-78, vectorised)
from paper_2204_00824_b200 import _native, datasets  # noqa: E402
from paper_2204_00824_b200.search import BestFirstParams, GpuIndex, load_tsdg  # noqa: E402

name = os.environ.get("SWEEP_DATASET", "c2_lowlid_1m")
# each variant: mode[:ENV=VALUE[:ENV=VALUE...]]  e.g.  fast:TSDG_SLOTS=16:TSDG_BATCH_MIN=8
variants = [v.split(":") for v in sys.argv[1:]] or [["fast"]]
ks = [int(x) for x in os.environ.get("SWEEP_K", "16").split(",")]
t = time.time()
ds = datasets.load(name)
idx = GpuIndex(load_tsdg(ds.graph_path), ds.base)
print(f"# setup {time.time()-t:.1f}s", flush=True)
dev = torch.device("cuda:0")
nq = ds.queries.shape[0]
# SWEEP_ORDER=pivot<N>: process queries grouped by their nearest of N random base rows
# (an upper-bound experiment for L2-locality-aware query scheduling)
if os.environ.get("SWEEP_ORDER", "").startswith("pivot"):
    npiv = int(os.environ["SWEEP_ORDER"][5:] or 64)
    piv = ds.base[np.random.default_rng(0).choice(ds.base.shape[0], npiv, replace=False)]
    d2 = ((ds.queries[:, None, :] - piv[None, :, :]) ** 2).sum(-1)
    perm = np.argsort(d2.argmin(1), kind="stable")
    ds.queries[:] = ds.queries[perm]
    ds.gt[:] = ds.gt[perm]
dq = torch.from_numpy(ds.queries).to(dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
stream = torch.cuda.Stream()
for k in ks:
    p = BestFirstParams(k=k, seed=7)
    ids = torch.empty((nq, k), dtype=torch.int32, device=dev)
    dd = torch.empty((nq, k), dtype=torch.float32, device=dev)
    cc = torch.empty(nq, dtype=torch.int32, device=dev)
    stt = torch.empty((nq, 4), dtype=torch.int32, device=dev)
    for var in variants:
        mode, envs = var[0], dict(kv.split("=", 1) for kv in var[1:])
        saved = {kk: os.environ.get(kk) for kk in envs}
        os.environ.update(envs)
        m = _native.MODE_FAST if mode == "fast" else _native.MODE_DETERMINISTIC

        def step():
            idx.search_bestfirst_device(dq.data_ptr(), nq, p, ids.data_ptr(), dd.data_ptr(),
                                        cc.data_ptr(), stt.data_ptr(), stream.cuda_stream, mode=m)

        with torch.cuda.stream(stream):
            for _ in range(3):
                step()
        torch.cuda.synchronize()
        times = []
        for i in range(10):
            with torch.cuda.stream(stream):
                flush.fill_(float(i))
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                step()
                b.record(stream)
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        st = stt.cpu().numpy().astype(np.int64)
        rec = recall_at_k(ids.cpu().numpy().view(np.uint32), cc.cpu().numpy(), ds.gt, 10)
        ms = float(np.median(times))
        alg = 4 * ds.base.shape[1] * st[:, 1].sum() + 4 * st[:, 3].sum() + nq * (4 * ds.base.shape[1] + 8 * k)
        for kk, vv in saved.items():
            if vv is None:
                os.environ.pop(kk, None)
            else:
                os.environ[kk] = vv
        print(json.dumps({"k": k, "mode": mode, "env": envs, "ms": ms,
                          "qps": nq / ms * 1e3, "recall10": rec, "alg_GBps": alg / ms / 1e6,
                          "evals_q": float(st[:, 1].mean()), "hops_q": float(st[:, 0].mean())}),
              flush=True)
