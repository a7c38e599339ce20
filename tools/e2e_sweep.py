"""e2e (host buffers through the C-ABI) timing vs the copy/compute chunk count."""
import ctypes, json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import torch
from paper_2204_00824_b200 import _native, datasets
from paper_2204_00824_b200.search import BestFirstParams, GpuIndex, load_tsdg
ds = datasets.load("c2_lowlid_1m")
idx = GpuIndex(load_tsdg(ds.graph_path), ds.base)
nq, k = ds.queries.shape[0], 16
p = BestFirstParams(k=16, seed=7).c()
hq = torch.from_numpy(ds.queries).pin_memory()
hi = torch.empty((nq, k), dtype=torch.int32).pin_memory(); hd = torch.empty((nq, k), dtype=torch.float32).pin_memory()
hc = torch.empty(nq, dtype=torch.int32).pin_memory()
L = _native.lib()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for ch in sys.argv[1:]:
    os.environ["TSDG_E2E_CHUNKS"] = ch
    def step():
        _native.check(L.tsdg_gpu_search_bestfirst(idx.handle, ctypes.c_void_p(hq.data_ptr()), nq, 0, ctypes.byref(p), 1,
            ctypes.c_void_p(hi.data_ptr()), ctypes.c_void_p(hd.data_ptr()), ctypes.c_void_p(hc.data_ptr()), None))
    for _ in range(3): step()
    ts = []
    for i in range(15):
        flush.fill_(float(i)); torch.cuda.synchronize()
        t0 = time.perf_counter(); step(); ts.append(time.perf_counter() - t0)
    print(json.dumps({"chunks": ch, "ms_median": 1e3 * float(np.median(ts)), "qps": nq / float(np.median(ts))}), flush=True)
