"""Greedy (Alg. 1) kernel routing on C2: CTA-per-walk cluster kernel vs warp-per-walk
kernel + merge, per-call latency (events) at growing batches, t0 from argv.
The launcher routes to the CTA kernel while nq * t0 <= TSDG_GREEDY_CTA_MAX_WALKS
(tsdg_gpu.cu use_cta_greedy); this measures where the crossover lies.

    python tools/greedy_crossover.py [t0]"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2204_00824_b200 import datasets  # noqa: E402
from paper_2204_00824_b200.search import GpuIndex, GreedyParams, load_tsdg  # noqa: E402

t0 = int(sys.argv[1]) if len(sys.argv) > 1 else 10
ds = datasets.load("c2_lowlid_1m")
idx = GpuIndex(load_tsdg(ds.graph_path), ds.base)
p = GreedyParams(t0=t0, hop_limit=16, lambda_cut=10, seed=7)
k = 10
dq = torch.from_numpy(ds.queries).cuda()
ids = torch.empty((10000, k), dtype=torch.int32, device="cuda")
dd = torch.empty((10000, k), dtype=torch.float32, device="cuda")
cc = torch.empty(10000, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for batch in (16, 32, 64, 128, 256, 512, 1024, 2048, 4096):
    for kern in ("cta", "warp"):
        os.environ["TSDG_GREEDY"] = kern
        reps = max(3, min(32, 4096 // batch))

        def call(j):
            o = (j * batch) % (10000 - batch)
            idx.search_greedy_device(dq[o].data_ptr(), batch, k, p, ids[o].data_ptr(), dd[o].data_ptr(),
                                     cc[o].data_ptr(), 0, st)
        for j in range(2):
            call(j)
        torch.cuda.synchronize()
        ts = []
        for j in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            call(j)
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        ms = float(np.median(ts))
        print(json.dumps({"t0": t0, "batch": batch, "kernel": kern, "walks": batch * t0,
                          "latency_us": ms * 1e3, "qps": batch / ms * 1e3}), flush=True)
