"""Strong-scaling proxy on one GPU: throughput of the C2 bench search (fast mode,
bench params) when a rank holds only a slice of the 10K batch — 10000 / N queries for
N = 1, 2, 4, 8 GPUs — with query_index_base = the slice start (bench.py --scaling
strong).  Events around each step, L2 flushed between steps.

    python tools/slice_scaling.py"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import PARAMS  # noqa: E402
from paper_2204_00824_b200 import _native, datasets, shards  # noqa: E402
from paper_2204_00824_b200.search import BestFirstParams, GpuIndex, load_tsdg  # noqa: E402

ds = datasets.load("c2_lowlid_1m")
idx = GpuIndex(load_tsdg(ds.graph_path), ds.base)
p = BestFirstParams(**PARAMS)
k = p.k
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for ws in (1, 2, 4, 8):
    lo, hi = shards.query_slice(ds.queries.shape[0], ws, 0)
    nq = hi - lo
    dq = torch.from_numpy(ds.queries[lo:hi]).cuda()
    ids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
    dd = torch.empty((nq, k), dtype=torch.float32, device="cuda")
    cc = torch.empty(nq, dtype=torch.int32, device="cuda")
    for mode, grp in ((_native.MODE_FAST, "1"), (_native.MODE_FAST, "2"), (_native.MODE_FAST, "4"),
                      (_native.MODE_DETERMINISTIC, "1")):
        os.environ["TSDG_FAST_GROUP"] = grp

        def step():
            idx.search_bestfirst_device(dq.data_ptr(), nq, p, ids.data_ptr(), dd.data_ptr(), cc.data_ptr(),
                                        0, st, query_index_base=lo, mode=mode)
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
        ms = float(np.median(ts))
        print(json.dumps({"gpus": ws, "queries_per_gpu": nq, "mode": "fast" if mode else "det",
                          "warps_per_query": int(grp) if mode == _native.MODE_FAST else 1,
                          "ms": ms, "qps_per_gpu": nq / ms * 1e3,
                          "projected_total_qps": ws * nq / ms * 1e3}), flush=True)
