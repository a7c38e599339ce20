"""Per-hop, per-warp timeline of one walk (CTA 0) of the greedy cluster kernel, batch 1
on C2 — development tool, phases build:
  TSDG_LIB=paper_2204_00824_b200/_lib/libtsdg_gpu_phases.so python tools/hop_trace.py [t0]
Events (ns from the hop's start on warp 1): 0 top, 1 pre-issued slice landed + distances,
2 before barrier 1, 3 after barrier 1, 4 after the combine barrier, 5 warp 0: merge done /
warps 1-3: next adjacency loaded, 6 next rows issued, 7 after barrier 2.  Median over
calls of each (warp, event) offset."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2204_00824_b200 import _native, datasets  # noqa: E402
from paper_2204_00824_b200.search import GpuIndex, GreedyParams, load_tsdg  # noqa: E402

t0 = int(sys.argv[1]) if len(sys.argv) > 1 else 10
ds = datasets.load("c2_lowlid_1m")
idx = GpuIndex(load_tsdg(ds.graph_path), ds.base)
lib = _native.lib()
lib.tsdg_gpu_hop_trace_read.argtypes = [ctypes.c_void_p]
buf = np.zeros((4, 32, 8), np.uint64)
p = GreedyParams(t0=t0, hop_limit=16, lambda_cut=10, seed=7)
dq = torch.from_numpy(ds.queries[:64]).cuda()
ids = torch.empty((64, 10), dtype=torch.int32, device="cuda")
dd = torch.empty((64, 10), dtype=torch.float32, device="cuda")
cc = torch.empty(64, dtype=torch.int32, device="cuda")
offs = []
for i in range(64):
    idx.search_greedy_device(dq[i].data_ptr(), 1, 10, p, ids[i].data_ptr(), dd[i].data_ptr(),
                             cc[i].data_ptr(), 0, 0)
    torch.cuda.synchronize()
    lib.tsdg_gpu_hop_trace_read(buf.ctypes.data)
    if i < 3:
        continue
    T = buf.astype(np.int64)
    for h in range(2, 32):  # hop 1 is special (no pre-issue timing before it)
        if T[1, h, 0] == 0 or T[1, h, 7] == 0:
            continue
        base = T[1, h, 0]
        offs.append({(w, e): T[w, h, e] - base for w in range(4) for e in range(8) if T[w, h, e]})
keys = sorted({k for o in offs for k in o})
med = {f"w{w}e{e}": float(np.median([o[(w, e)] for o in offs if (w, e) in o])) for (w, e) in keys}
print(json.dumps({"t0": t0, "hops_sampled": len(offs), "median_ns": med}))
