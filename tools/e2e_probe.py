"""Where the e2e time of the C2 bench step goes (k_search=14, fast mode):
  device      : *_device call, queries / results in HBM, CUDA events
  device_mapped: *_device call on the mapped aliases of pinned host buffers (the zero-copy
                kernel alone), CUDA events
  e2e_zero_copy / e2e_copy : the host-pointer call (TSDG_ZERO_COPY=1 / 0), wall clock
  host_call_tiny: the host-pointer call with nq = 1 (fixed host-side cost)
python tools/e2e_probe.py"""
import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2204_00824_b200 import _native, datasets  # noqa: E402
from paper_2204_00824_b200.search import BestFirstParams, GpuIndex, load_tsdg  # noqa: E402

ds = datasets.load("c2_lowlid_1m")
idx = GpuIndex(load_tsdg(ds.graph_path), ds.base)
nq, k = ds.queries.shape[0], 14
bp = BestFirstParams(k=k, seed=7)
p = bp.c()
L = _native.lib()
mode = _native.MODE_FAST
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
hq = torch.from_numpy(ds.queries).pin_memory()
hi = torch.empty((nq, k), dtype=torch.int32).pin_memory()
hd = torch.empty((nq, k), dtype=torch.float32).pin_memory()
hc = torch.empty(nq, dtype=torch.int32).pin_memory()
dq = hq.cuda()
di, dd, dc = hi.cuda(), hd.cuda(), hc.cuda()
st = torch.cuda.current_stream().cuda_stream


def events(fn, reps=15):
    ts = []
    for i in range(reps):
        flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return float(np.median(ts))


def wall(fn, reps=15):
    ts = []
    for i in range(reps):
        flush.fill_(float(i))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


def dev_call(q, i, d, c, n=nq):
    idx.search_bestfirst_device(q, n, bp, i, d, c, 0, st, mode=mode)


def host_call(n=nq):
    _native.check(L.tsdg_gpu_search_bestfirst(
        idx.handle, ctypes.c_void_p(hq.data_ptr()), n, 0, ctypes.byref(p), mode,
        ctypes.c_void_p(hi.data_ptr()), ctypes.c_void_p(hd.data_ptr()), ctypes.c_void_p(hc.data_ptr()),
        None))


out = {}
for _ in range(3):
    dev_call(dq.data_ptr(), di.data_ptr(), dd.data_ptr(), dc.data_ptr())
out["device_s"] = events(lambda: dev_call(dq.data_ptr(), di.data_ptr(), dd.data_ptr(), dc.data_ptr()))
# pinned torch tensors are mapped (unified addressing): the host pointer is the device alias
out["device_mapped_s"] = events(lambda: dev_call(hq.data_ptr(), hi.data_ptr(), hd.data_ptr(), hc.data_ptr()))
out["device_mapped_queries_only_s"] = events(
    lambda: dev_call(hq.data_ptr(), di.data_ptr(), dd.data_ptr(), dc.data_ptr()))
out["device_mapped_results_only_s"] = events(
    lambda: dev_call(dq.data_ptr(), hi.data_ptr(), hd.data_ptr(), hc.data_ptr()))
for zc in ("1", "0"):
    os.environ["TSDG_ZERO_COPY"] = zc
    for _ in range(2):
        host_call()
    out[f"e2e_zero_copy_{zc}_s"] = wall(host_call)
os.environ["TSDG_ZERO_COPY"] = "1"
out["host_call_tiny_s"] = wall(lambda: host_call(1), reps=50)
out["qps"] = {kk: nq / v for kk, v in out.items() if kk.endswith("_s") and "tiny" not in kk}
print(json.dumps(out), flush=True)
