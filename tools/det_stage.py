"""Deterministic best-first kernel on C2 (bench params, 10K batch): row staging by one
TMA bulk copy per row vs tile::gather4 tensor copies (TSDG_STAGE=tma|g4), events
around each step with L2 flushed in between; the two must return identical ids,
distance bits and counts.

    python tools/det_stage.py [slots,...]"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import PARAMS  # noqa: E402
from paper_2204_00824_b200 import _native, datasets  # noqa: E402
from paper_2204_00824_b200.search import BestFirstParams, GpuIndex, load_tsdg  # noqa: E402

ds = datasets.load("c2_lowlid_1m")
idx = GpuIndex(load_tsdg(ds.graph_path), ds.base)
p = BestFirstParams(**PARAMS)
nq, k = ds.queries.shape[0], p.k
dq = torch.from_numpy(ds.queries).cuda()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
ref = None
for slots in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "16").split(",")]:
    os.environ["TSDG_SLOTS"] = str(slots)
    for stage in ("tma", "g4"):
        os.environ["TSDG_STAGE"] = stage
        ids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
        dd = torch.empty((nq, k), dtype=torch.float32, device="cuda")
        cc = torch.empty(nq, dtype=torch.int32, device="cuda")

        def step():
            idx.search_bestfirst_device(dq.data_ptr(), nq, p, ids.data_ptr(), dd.data_ptr(), cc.data_ptr(), 0, st,
                                        mode=_native.MODE_DETERMINISTIC)
        for _ in range(3):
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
        out = (ids.cpu().numpy(), dd.cpu().numpy().view(np.uint32), cc.cpu().numpy())
        if ref is None:
            ref = out
        same = all(np.array_equal(x, y) for x, y in zip(out, ref))
        ms = float(np.median(ts))
        print(json.dumps({"slots": slots, "stage": stage, "ms": ms, "qps": nq / ms * 1e3,
                          "identical_to_first": same}), flush=True)
