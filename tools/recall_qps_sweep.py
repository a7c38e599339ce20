"""Recall@10 vs QPS on C2 (BASELINE config 2: "recall@10 vs QPS sweep"): GPU best-first
fast / deterministic at several k_search and lambda cuts, device-resident batch of 10K,
L2 flushed between steps, CUDA events; the reference CPU (oracle/_ref, all host
threads) timed on the first 2000 queries at the same points.  Development tool:
python tools/recall_qps_sweep.py [k,cut ...] > profiles/recall_qps_c2_r1.jsonl"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402  (reference-arm timing, as bench.py --impl reference)
from bench import recall_at_k  # noqa: E402
from paper_2204_00824_b200 import _native, datasets  # noqa: E402
from paper_2204_00824_b200.search import BestFirstParams, GpuIndex, load_tsdg  # noqa: E402

ds = datasets.load("c2_lowlid_1m")
idx = GpuIndex(load_tsdg(ds.graph_path), ds.base)
ref = O.Ref()
fx = ref.fixture(ds.graph_path, ds.base)
nq = ds.queries.shape[0]
dq = torch.from_numpy(ds.queries).cuda()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
# Delta is in squared-distance units (bestfirst_search.hpp:18); SURVEY §8(d) sweeps it
# as a multiple of the median squared distance to the 10th true neighbour
g10 = ds.gt[:, 9].astype(np.int64)
d10 = ((ds.queries.astype(np.float32) - ds.base[g10]) ** 2).sum(axis=1)
med10 = float(np.median(d10))


def parse(a):
    f = a.split(",")  # k,cut[,m[,delta_multiple]]
    return (int(f[0]), int(f[1]), int(f[2]) if len(f) > 2 else 8, float(f[3]) if len(f) > 3 else 0.0)


points = [parse(a) for a in sys.argv[1:]] or (
    [(k, 5, 8, 0.0) for k in (10, 12, 16, 24, 32, 48, 64)] + [(16, 3, 8, 0.0), (16, 10, 8, 0.0),
                                                             (32, 10, 8, 0.0)])
for k, cut, m, dmul in points:
    p = BestFirstParams(k=k, lambda_cut=cut, seed=7, m_segments=m, delta=dmul * med10)
    ids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
    dd = torch.empty((nq, k), dtype=torch.float32, device="cuda")
    cc = torch.empty(nq, dtype=torch.int32, device="cuda")
    st = torch.empty((nq, 4), dtype=torch.int32, device="cuda")
    line = {"k_search": k, "lambda_cut": cut, "m_segments": m, "delta": p.delta,
            "delta_over_median_d10": dmul}
    for name, mode in (("fast", _native.MODE_FAST), ("det", _native.MODE_DETERMINISTIC)):
        def step():
            idx.search_bestfirst_device(dq.data_ptr(), nq, p, ids.data_ptr(), dd.data_ptr(),
                                        cc.data_ptr(), st.data_ptr(), 0, mode=mode)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        ts = []
        for i in range(10):
            flush.fill_(float(i))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            step()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = float(np.median(ts))
        rec = recall_at_k(ids.cpu().numpy().view(np.uint32), cc.cpu().numpy(), ds.gt, 10)
        line[name] = {"qps": nq / ms * 1e3, "ms": ms, "recall_at_10": rec}
    q = ds.queries[:2000]
    fx.large_batch(q[:200], p)
    t0 = time.perf_counter()
    rids, rc, _ = fx.large_batch(q, p)
    sec = time.perf_counter() - t0
    line["reference_cpu"] = {"qps": 2000 / sec, "threads": ref.so.ref_num_threads(),
                             "recall_at_10_first2000": recall_at_k(rids, rc, ds.gt[:2000], 10)}
    print(json.dumps(line), flush=True)
