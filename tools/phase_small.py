"""Per-phase cycles of greedy_cta_kernel (small batch, batch 1) on C2, development
build with -DTSDG_PHASES:  TSDG_LIB=paper_2204_00824_b200/_lib/libtsdg_gpu_phases.so
python tools/phase_small.py [t0]"""
import ctypes, json, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_2204_00824_b200 import _native, datasets
from paper_2204_00824_b200.search import GpuIndex, GreedyParams, load_tsdg
t0 = int(sys.argv[1]) if len(sys.argv) > 1 else 8
ds = datasets.load("c2_lowlid_1m")
idx = GpuIndex(load_tsdg(ds.graph_path), ds.base)
lib = _native.lib()
lib.tsdg_gpu_phase_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
out = np.zeros(8, np.uint64)
nq = 200
dq = torch.from_numpy(ds.queries[:nq]).cuda()
ids = torch.empty((nq, 10), dtype=torch.int32, device="cuda")
dd = torch.empty((nq, 10), dtype=torch.float32, device="cuda")
cc = torch.empty(nq, dtype=torch.int32, device="cuda")
st = torch.empty((nq, 4), dtype=torch.int32, device="cuda")
p = GreedyParams(t0=t0, seed=7)
for i in range(5):
    idx.search_greedy_device(dq[i].data_ptr(), 1, 10, p, ids[i].data_ptr(), dd[i].data_ptr(), cc[i].data_ptr(), st[i].data_ptr(), 0)
torch.cuda.synchronize()
lib.tsdg_gpu_phase_read(out.ctypes.data, 1)
for i in range(nq):
    idx.search_greedy_device(dq[i].data_ptr(), 1, 10, p, ids[i].data_ptr(), dd[i].data_ptr(), cc[i].data_ptr(), st[i].data_ptr(), 0)
torch.cuda.synchronize()
lib.tsdg_gpu_phase_read(out.ctypes.data, 1)
hops = int(st.cpu().numpy()[:, 0].sum())  # summed over walks
warps = nq * t0 * 4
names = ["start", "gather+dist", "barrier1", "combine+merge(w0)/next adjacency", "barrier2",
         "row copy issue", "cluster wait", "pool merge"]
print(json.dumps({"t0": t0, "walk_hops": hops / (nq * t0),
                  "cycles_per_walk_warp": {names[i]: round(float(out[i]) / warps) for i in range(8)},
                  "per_hop": {names[i]: round(float(out[i]) / (hops * 4)) for i in (1, 2, 3, 5, 4)}}))
