"""Does processing order matter for L2 reuse?  Times the C2 fast search on the 10K
batch in its own order and re-ordered by nearest pivot (P base rows, host-side,
untimed), so that queries in flight together touch nearby graph regions.  Timing
only (the RNG stream follows the position, so ids differ in detail).

    python tools/order_probe.py [P,...]"""
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

ds = datasets.load("c2_lowlid_1m")
idx = GpuIndex(load_tsdg(ds.graph_path), ds.base)
p = BestFirstParams(**PARAMS)
nq, k = ds.queries.shape[0], p.k
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
rng = np.random.default_rng(0)
for P in [0] + [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "16,64,256,1024").split(",")]:
    if P == 0:
        order = np.arange(nq)
    else:
        piv = ds.base[rng.choice(ds.base.shape[0], P, replace=False)]
        d2 = ((ds.queries[:, None, :] - piv[None, :, :]) ** 2).sum(-1) if P <= 256 else None
        if d2 is None:
            d2 = np.stack([((ds.queries - piv[i]) ** 2).sum(-1) for i in range(P)], axis=1)
        order = np.argsort(d2.argmin(1), kind="stable")
    q = np.ascontiguousarray(ds.queries[order])
    dq = torch.from_numpy(q).cuda()
    ids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
    dd = torch.empty((nq, k), dtype=torch.float32, device="cuda")
    cc = torch.empty(nq, dtype=torch.int32, device="cuda")

    def step():
        idx.search_bestfirst_device(dq.data_ptr(), nq, p, ids.data_ptr(), dd.data_ptr(), cc.data_ptr(), 0, st,
                                    mode=_native.MODE_FAST)
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
    rec = recall_at_k(ids.cpu().numpy().view(np.uint32), cc.cpu().numpy(), ds.gt[order], 10)
    print(json.dumps({"pivots": P, "ms": float(np.median(ts)), "recall_at_10": rec}), flush=True)
