"""Small-batch (Alg. 1, greedy) latency on C2: batch 1 / 8 / 64, device-resident
queries, CUDA events around each call.  Development tool; bench.py carries the
same measurement in its JSON line under "small_batch"."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import recall_at_k  # noqa: E402  (bench.cpp:59-78, vectorised)
from paper_2204_00824_b200 import _native, datasets  # noqa: E402
from paper_2204_00824_b200.search import GpuIndex, GreedyParams, load_tsdg  # noqa: E402


def small_batch_latency(idx, queries, gt, batch, params, k=10, mode=0, reps=None, dev=None):
    dev = dev or torch.device("cuda:0")
    nq_total = min(queries.shape[0], 1024 if batch >= 8 else 256)
    reps = reps or max(1, nq_total // batch)
    dq = torch.from_numpy(queries[:reps * batch]).to(dev)
    ids = torch.empty((reps * batch, k), dtype=torch.int32, device=dev)
    dd = torch.empty((reps * batch, k), dtype=torch.float32, device=dev)
    cc = torch.empty(reps * batch, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    for i in range(min(3, reps)):  # warm-up
        idx.search_greedy_device(dq[i * batch].data_ptr(), batch, k, params, ids[i * batch].data_ptr(),
                                 dd[i * batch].data_ptr(), cc[i * batch].data_ptr(), 0, stream,
                                 mode=mode)
    torch.cuda.synchronize()
    times = []
    for i in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        idx.search_greedy_device(dq[i * batch].data_ptr(), batch, k, params, ids[i * batch].data_ptr(),
                                 dd[i * batch].data_ptr(), cc[i * batch].data_ptr(), 0, stream,
                                 mode=mode)
        b.record()
        b.synchronize()
        times.append(a.elapsed_time(b))
    rec = recall_at_k(ids.cpu().numpy().view(np.uint32), cc.cpu().numpy(), gt[:reps * batch], 10)
    lat = float(np.median(times))
    return {"batch": batch, "t0": params.t0, "latency_ms_p50": lat,
            "latency_ms_p99": float(np.percentile(times, 99)), "qps": batch / lat * 1e3,
            "recall_at_10": rec, "queries": reps * batch}


if __name__ == "__main__":
    ds = datasets.load(os.environ.get("SWEEP_DATASET", "c2_lowlid_1m"))
    idx = GpuIndex(load_tsdg(ds.graph_path), ds.base)
    for kern in os.environ.get("KERNELS", "cta,warp").split(","):
        os.environ["TSDG_GREEDY"] = kern
        for t0 in [int(x) for x in os.environ.get("T0S", "8,16").split(",")]:
            for batch in (1, 8, 64):
                mode = int(os.environ.get("MODE", "0"))
                r = small_batch_latency(idx, ds.queries, ds.gt, batch, GreedyParams(t0=t0, seed=7),
                                        mode=mode)
                r["kernel"] = kern
                r["mode"] = "fast" if mode else "det"
                print(json.dumps(r), flush=True)
    if os.environ.get("REF") == "1":
        # reference arm (as bench.py --impl reference): the unmodified reference's
        # small_batch_search on the host cores, wall clock per call, same batches
        import time
        from oracle import oracle as O
        ref = O.Ref()
        fx = ref.fixture(ds.graph_path, ds.base)
        for t0 in [int(x) for x in os.environ.get("T0S", "8,16").split(",")]:
            p = GreedyParams(t0=t0, seed=7)
            for batch in (1, 8, 64):
                reps = max(4, min(64, 512 // batch))
                fx.small_batch(ds.queries[:batch], 10, p)
                ts = []
                for i in range(reps):
                    q = ds.queries[i * batch:(i + 1) * batch]
                    t = time.perf_counter()
                    fx.small_batch(q, 10, p)
                    ts.append((time.perf_counter() - t) * 1e3)
                lat = float(np.median(ts))
                print(json.dumps({"batch": batch, "t0": t0, "latency_ms_p50": lat,
                                  "qps": batch / lat * 1e3, "impl": "reference_cpu",
                                  "threads": ref.so.ref_num_threads(), "queries": reps * batch}),
                      flush=True)
