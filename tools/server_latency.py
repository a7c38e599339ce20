"""Small-batch latency on C2 through the host-pointer calls: the persistent server
(tsdg_gpu_server_search) vs the launch path (tsdg_gpu_search_greedy), wall clock
around each synchronous call with pinned buffers, recall@10 beside it.
python tools/server_latency.py [t0,...] [mode det|fast]"""
import json, os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from bench import recall_at_k
from paper_2204_00824_b200 import _native, datasets
from paper_2204_00824_b200.search import GpuIndex, GreedyParams, load_tsdg
t0s = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "10,16").split(",")]
mode = _native.MODE_FAST if (len(sys.argv) > 2 and sys.argv[2] == "fast") else _native.MODE_DETERMINISTIC
ds = datasets.load("c2_lowlid_1m")
idx = GpuIndex(load_tsdg(ds.graph_path), ds.base)
k = 10
for t0 in t0s:
    p = GreedyParams(t0=t0, hop_limit=16, lambda_cut=10, seed=7)
    for batch in (1, 8, 64):
        reps = 400 if batch == 1 else max(50, 2048 // batch)
        hq = torch.from_numpy(ds.queries[:reps * batch].copy()).pin_memory()
        hi = torch.empty((reps * batch, k), dtype=torch.int32).pin_memory()
        hd = torch.empty((reps * batch, k), dtype=torch.float32).pin_memory()
        hc = torch.empty(reps * batch, dtype=torch.int32).pin_memory()
        row = {"t0": t0, "batch": batch, "mode": "fast" if mode else "det"}
        with idx.greedy_server(k, p, mode=mode, max_batch=batch) as sv:
            def call(j):
                o = j * batch
                sv.search_into(hq[o].data_ptr(), batch, hi[o].data_ptr(), hd[o].data_ptr(), hc[o].data_ptr())
            for j in range(5):
                call(j)
            lat = []
            for j in range(reps):
                t = time.perf_counter(); call(j); lat.append(time.perf_counter() - t)
            row["server_us_p50"] = float(np.median(lat)) * 1e6
            row["server_us_p99"] = float(np.percentile(lat, 99)) * 1e6
            row["server_clusters"] = sv.clusters
        row["recall_at_10"] = recall_at_k(hi.numpy().view(np.uint32), hc.numpy(), ds.gt[:reps * batch], 10)
        L = _native.lib(); pc = p.c()
        import ctypes
        def lcall(j):
            o = j * batch
            _native.check(L.tsdg_gpu_search_greedy(idx.handle, ctypes.c_void_p(hq[o].data_ptr()), batch, k,
                                                   ctypes.byref(pc), mode, ctypes.c_void_p(hi[o].data_ptr()),
                                                   ctypes.c_void_p(hd[o].data_ptr()), ctypes.c_void_p(hc[o].data_ptr()), None))
        for j in range(5):
            lcall(j)
        lat = []
        for j in range(min(reps, 200)):
            t = time.perf_counter(); lcall(j); lat.append(time.perf_counter() - t)
        row["launch_us_p50"] = float(np.median(lat)) * 1e6
        print(json.dumps(row), flush=True)
