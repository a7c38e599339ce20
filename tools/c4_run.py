"""C4 (GIST1M-shaped 1M x 960 fp32, batch 10K) best-first search at one k_search, for
timing and for an ncu capture of the search kernel:

    python tools/c4_run.py [k_search] [fast|det] [steps]
    ncu --set full -k regex:bf_ -c 1 ... python tools/c4_run.py 24 fast 1

Prints one JSON line: ms per batch (events, L2 flushed), recall@10, algorithmic bytes
per launch (4*d*E_q + 4*A_q + 4*d + 8*k summed) and the roofline fraction."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import peaks, recall_at_k  # noqa: E402
from paper_2204_00824_b200 import _native, datasets  # noqa: E402
from paper_2204_00824_b200.search import BestFirstParams, GpuIndex, load_tsdg  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 24
mode = _native.MODE_DETERMINISTIC if (len(sys.argv) > 2 and sys.argv[2] == "det") else _native.MODE_FAST
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
ds = datasets.load("c4_lowlid_1m_960")
idx = GpuIndex(load_tsdg(ds.graph_path), ds.base)
nq, d = ds.queries.shape
p = BestFirstParams(k=k, seed=7)
dq = torch.from_numpy(ds.queries).cuda()
ids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
dd = torch.empty((nq, k), dtype=torch.float32, device="cuda")
cc = torch.empty(nq, dtype=torch.int32, device="cuda")
stt = torch.empty((nq, 4), dtype=torch.int32, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def step():
    idx.search_bestfirst_device(dq.data_ptr(), nq, p, ids.data_ptr(), dd.data_ptr(), cc.data_ptr(),
                                stt.data_ptr(), st, mode=mode)


if steps > 1:
    for _ in range(3):
        step()
ts = []
for i in range(steps):
    flush.fill_(float(i))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    step()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
s = stt.cpu().numpy().astype(np.int64)
alg = int(4 * d * s[:, 1].sum() + 4 * s[:, 3].sum() + nq * (4 * d + 8 * k))
ms = float(np.median(ts))
peak = peaks()[0]
print(json.dumps({"workload": "C4 GIST1M-shape 1M x 960, batch 10K", "k_search": k,
                  "mode": "det" if mode == _native.MODE_DETERMINISTIC else "fast",
                  "ms_per_batch": ms, "qps": nq / ms * 1e3,
                  "recall_at_10": recall_at_k(ids.cpu().numpy().view(np.uint32), cc.cpu().numpy(), ds.gt, 10),
                  "recall_at_1": recall_at_k(ids.cpu().numpy().view(np.uint32), cc.cpu().numpy(), ds.gt, 1),
                  "evals_per_query": float(s[:, 1].mean()), "edges_per_query": float(s[:, 3].mean()),
                  "alg_bytes_per_launch": alg, "achieved_GBps": alg / ms / 1e6,
                  "roofline_frac": alg / ms / 1e6 / peak}), flush=True)
