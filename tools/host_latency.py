"""Small-batch latency of the host-pointer C-ABI call (wall clock around the
synchronous call): pinned buffers (zero-copy path) vs pageable (copy path).
Development tool."""
import ctypes, os, sys, time, json
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2204_00824_b200 import _native, datasets
from paper_2204_00824_b200.search import GpuIndex, GreedyParams, load_tsdg
ds = datasets.load("c2_lowlid_1m")
idx = GpuIndex(load_tsdg(ds.graph_path), ds.base)
L = _native.lib()
p = GreedyParams(t0=16, seed=7); pc = p.c()
for batch in (1, 8, 64):
    for pinned in (True, False):
        qs = [np.ascontiguousarray(ds.queries[(i % 150)*batch:(i % 150 + 1)*batch]) for i in range(200)]
        if pinned:
            hq = [torch.from_numpy(x).pin_memory() for x in qs]; ptrs = [t.data_ptr() for t in hq]
            hi = torch.empty((batch, 10), dtype=torch.int32).pin_memory(); hd = torch.empty((batch, 10)).pin_memory(); hc = torch.empty(batch, dtype=torch.int32).pin_memory()
            oi, od, oc = hi.data_ptr(), hd.data_ptr(), hc.data_ptr()
        else:
            ptrs = [x.ctypes.data for x in qs]
            ni = np.empty((batch, 10), np.uint32); nd = np.empty((batch, 10), np.float32); nc = np.empty(batch, np.uint32)
            oi, od, oc = ni.ctypes.data, nd.ctypes.data, nc.ctypes.data
        ts = []
        for i in range(200):
            t = time.perf_counter()
            _native.check(L.tsdg_gpu_search_greedy(idx.handle, ctypes.c_void_p(ptrs[i]), batch, 10, ctypes.byref(pc), 0,
                          ctypes.c_void_p(oi), ctypes.c_void_p(od), ctypes.c_void_p(oc), None))
            ts.append((time.perf_counter() - t) * 1e6)
        print(json.dumps({"batch": batch, "pinned_zero_copy": pinned, "host_call_us_p50": float(np.median(ts[20:])), "p99": float(np.percentile(ts[20:], 99))}))
