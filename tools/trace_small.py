"""Per-CTA globaltimer trace of greedy_cta_kernel (small batch) on C2 — development
tool, phases build:  TSDG_LIB=paper_2204_00824_b200/_lib/libtsdg_gpu_phases.so
python tools/trace_small.py [t0] [batch] [hop_limit]
Prints the median over calls of: CTA start skew, query load, select_start, hops,
the wait for the slowest walk of the cluster, the pool merge, and the CUDA-event time
of the same call."""
import ctypes, json, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_2204_00824_b200 import _native, datasets
from paper_2204_00824_b200.search import GpuIndex, GreedyParams, load_tsdg

t0 = int(sys.argv[1]) if len(sys.argv) > 1 else 16
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1
hl = int(sys.argv[3]) if len(sys.argv) > 3 else 16
ds = datasets.load("c2_lowlid_1m")
idx = GpuIndex(load_tsdg(ds.graph_path), ds.base)
lib = _native.lib()
lib.tsdg_gpu_trace_read.argtypes = [ctypes.c_void_p]
tr = np.zeros((256, 32), np.uint64)
calls = 40
dq = torch.from_numpy(ds.queries[:calls * batch]).cuda()
ids = torch.empty((calls * batch, 10), dtype=torch.int32, device="cuda")
dd = torch.empty((calls * batch, 10), dtype=torch.float32, device="cuda")
cc = torch.empty(calls * batch, dtype=torch.int32, device="cuda")
st = torch.empty((calls * batch, 4), dtype=torch.int32, device="cuda")
p = GreedyParams(t0=t0, hop_limit=hl, lambda_cut=10, seed=7)
rows = []
for i in range(calls + 3):
    j = i % calls
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    idx.search_greedy_device(dq[j * batch].data_ptr(), batch, 10, p, ids[j * batch].data_ptr(),
                             dd[j * batch].data_ptr(), cc[j * batch].data_ptr(), st[j * batch].data_ptr(), 0)
    b.record()
    torch.cuda.synchronize()
    lib.tsdg_gpu_trace_read(tr.ctypes.data)
    if i < 3:
        continue
    n = min(batch * t0, 256)  # the trace buffer holds 256 CTAs
    T = tr[:n].astype(np.int64)
    start = T[:, 0]
    t_begin = start.min()
    hops = [(T[c, 3:27] > 0).sum() for c in range(n)]
    hop_t = [(T[c, 3 + h - 1] - T[c, 2]) / max(h, 1) for c, h in enumerate(hops)]
    loop_end = np.array([T[c, 27] for c in range(n)])
    rows.append({
        "event_us": a.elapsed_time(b) * 1e3,
        "span_us": (T[:, 30].max() - t_begin) / 1e3,
        "start_skew_us": (start.max() - t_begin) / 1e3,
        "query_load_us": float(np.median(T[:, 1] - T[:, 0])) / 1e3,
        "select_start_us": float(np.median(T[:, 2] - T[:, 1])) / 1e3,
        "hops_mean": float(np.mean(hops)), "hops_max": int(max(hops)),
        "us_per_hop": float(np.median(hop_t)) / 1e3,
        "slowest_walk_end_us": (loop_end.max() - t_begin) / 1e3,
        "cluster_wait_us": float(np.median(T[:, 28] - T[:, 27])) / 1e3,
        "merge_us": float(np.median(T[::t0, 29] - T[::t0, 28])) / 1e3,
    })
out = {k: float(np.median([r[k] for r in rows])) for k in rows[0]}
print(json.dumps({"t0": t0, "batch": batch, "hop_limit": hl, **{k: round(v, 2) for k, v in out.items()}}))
