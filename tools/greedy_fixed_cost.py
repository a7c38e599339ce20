"""Small-batch fixed cost vs per-hop cost (development tool): batch-1 latency of the
greedy CTA kernel on C2 at hop limits T = 1, 2, 4, 8, 16 and t0 = 1, 2, 16, CUDA
events around the device call (so host submission is included) and the kernel time
alone (events around a second launch queued behind the first)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2204_00824_b200 import datasets  # noqa: E402
from paper_2204_00824_b200.search import GpuIndex, GreedyParams, load_tsdg  # noqa: E402

ds = datasets.load("c2_lowlid_1m")
idx = GpuIndex(load_tsdg(ds.graph_path), ds.base)
os.environ.setdefault("TSDG_GREEDY", "cta")
dq = torch.from_numpy(ds.queries[:256]).cuda()
ids = torch.empty((256, 10), dtype=torch.int32, device="cuda")
dd = torch.empty((256, 10), dtype=torch.float32, device="cuda")
cc = torch.empty(256, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for t0 in (1, 2, 16):
    for T in (1, 2, 4, 8, 16):
        p = GreedyParams(t0=t0, hop_limit=T, seed=7)

        def call(j):
            idx.search_greedy_device(dq[j].data_ptr(), 1, 10, p, ids[j].data_ptr(), dd[j].data_ptr(),
                                     cc[j].data_ptr(), 0, st)
        for j in range(5):
            call(j)
        torch.cuda.synchronize()
        single, queued = [], []
        for j in range(100):
            a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            a.record()
            call(j)
            b.record()
            call(j + 100)  # queued behind: its time excludes host submission
            c.record()
            c.synchronize()
            single.append(a.elapsed_time(b) * 1e3)
            queued.append(b.elapsed_time(c) * 1e3)
        print(json.dumps({"t0": t0, "hop_limit": T, "event_us_p50": float(np.median(single)),
                          "queued_us_p50": float(np.median(queued))}), flush=True)
