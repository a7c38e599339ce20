"""Tuning sweep of the fast best-first kernel's compiled variants on C2 (bench params):
rows per batch B and the register/occupancy target (bf_fast.cu pick()), plus the L2
prefetch switch.  Events around each step, L2 flushed between steps.

    python tools/fast_variants.py [variant,...] [prefetch,...]"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import PARAMS, recall_at_k  # noqa: E402
from paper_2204_00824_b200 import _native, datasets  # noqa: E402
from paper_2204_00824_b200.search import BestFirstParams, GpuIndex, load_tsdg  # noqa: E402

variants = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "0,1,2,3,4,5,6,7").split(",")]
prefetches = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1").split(",")]
ds = datasets.load("c2_lowlid_1m")
idx = GpuIndex(load_tsdg(ds.graph_path), ds.base)
p = BestFirstParams(**PARAMS)
nq, k = ds.queries.shape[0], p.k
dq = torch.from_numpy(ds.queries).cuda()
ids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
dd = torch.empty((nq, k), dtype=torch.float32, device="cuda")
cc = torch.empty(nq, dtype=torch.int32, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def step():
    idx.search_bestfirst_device(dq.data_ptr(), nq, p, ids.data_ptr(), dd.data_ptr(), cc.data_ptr(),
                                0, st, mode=_native.MODE_FAST)


for pf in prefetches:
    os.environ["TSDG_FAST_PREFETCH"] = str(pf)
    for v in variants:
        os.environ["TSDG_FAST_VARIANT"] = str(v)
        for _ in range(5):
            step()
        ts = []
        for i in range(20):
            flush.fill_(float(i))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            step()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        rec = recall_at_k(ids.cpu().numpy().view(np.uint32), cc.cpu().numpy(), ds.gt, 10)
        ms = float(np.median(ts))
        print(json.dumps({"variant": v, "prefetch": pf, "ms": ms, "qps": nq / ms * 1e3,
                          "recall_at_10": rec}), flush=True)
