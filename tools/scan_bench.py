"""Exact top-k scan on full-size inputs (development / evidence tool; one GPU).

  * ground truth at C2 (10K x 1M x 128, k=100) and C4 (10K x 1M x 960) through the
    index-resident form, checked id-for-id against the reference's ground_truth
    output stored in data/<name>/gt.u32 (tools/make_dataset.py);
  * brute-force k-NN graph (k=100) of the C1 base (100K x 128).

Prints one JSON line per case: seconds (CUDA events around the device call), pair
distances per second and the fp32-pipe roofline: 3 ops per pair-dim (sub, mul, add —
no FMA, the reference's rounding) against the packed-pipe rate measured by
tools/micro/fp2_pipes.cu (FADD2 / FMUL2: 127.7 lane-ops per SM per cycle, i.e. one
packed instruction per two cycles per SMSP; the kernel's own step — SUB2, FFMA2 with
a -0 addend, ADD2 — at best 112 in that probe)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2204_00824_b200 import _native, datasets  # noqa: E402

FP2_PEAK = 148 * 128 * 1.965e9  # fp32 lane-ops/s of the packed pipe (37.2 T), measured rate
STEP_CAP = 148 * 112 * 1.965e9  # the scan step's own best in the probe (32.6 T)


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return min(ts)


def gt_case(name, k=100):
    if not datasets.available(name):
        return {"case": f"ground_truth {name}", "unavailable": "dataset missing"}
    import ctypes

    from paper_2204_00824_b200.search import ground_truth
    ds = datasets.load(name)
    n, d = ds.base.shape
    nq = ds.queries.shape[0]
    # host-API form (upload + scan + download), checked against the reference's GT
    t0 = time.perf_counter()
    r = ground_truth(ds.base, ds.queries, k)
    host_s = time.perf_counter() - t0
    same = bool(np.array_equal(r.ids[:, :ds.gt.shape[1]], ds.gt[:, :k]))
    out = {"case": f"ground_truth {name}", "nq": nq, "n": n, "d": d, "k": k,
           "ids_equal_reference_gt": same, "host_call_s": host_s}
    if d % 4 == 0:  # device-resident form (rows already 16-byte strided)
        db = torch.from_numpy(ds.base).cuda()
        dq = torch.from_numpy(ds.queries).cuda()
        ids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
        dd = torch.empty((nq, k), dtype=torch.float32, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        L = _native.lib()

        def call():
            _native.check(L.tsdg_gpu_exact_topk_device(
                ctypes.c_void_p(db.data_ptr()), n, d, ctypes.c_void_p(dq.data_ptr()), nq, d, d, k,
                0, 0, 0, ctypes.c_void_p(ids.data_ptr()), ctypes.c_void_p(dd.data_ptr()),
                ctypes.c_void_p(st)))

        sec = timed(call)
        flops = 3.0 * nq * n * d
        out.update({"device_s": sec, "pairs_per_s": nq * n / sec,
                    "fp32_Tops": flops / sec / 1e12, "fp2_pipe_frac": flops / sec / FP2_PEAK,
                    "frac_of_probe_step": flops / sec / STEP_CAP})
    return out


def knn_case(name="c1_lowlid_100k", k=100):
    if not datasets.available(name):
        return {"case": f"brute_force_knn {name}", "unavailable": "dataset missing"}
    ds = datasets.load(name)
    from paper_2204_00824_b200.search import brute_force_knn
    n, d = ds.base.shape
    t0 = time.perf_counter()
    kg = brute_force_knn(ds.base, k)
    sec = time.perf_counter() - t0
    # spot-check 50 nodes with a float64 exact scan: the returned k distances must
    # be the k smallest (bit-exactness against the reference is in tests/test_scan.py)
    rows = np.arange(0, n, n // 50)[:50]
    ok = True
    base64 = ds.base.astype(np.float64)
    for r in rows:
        d2 = ((base64 - base64[r]) ** 2).sum(axis=1)
        d2[r] = np.inf
        want = np.sort(d2)[:k]
        got = np.sort(d2[kg.ids[r].astype(np.int64)])
        ok &= bool(np.allclose(got, want, rtol=1e-5, atol=1e-6))
    flops = 3.0 * n * n * d
    return {"case": f"brute_force_knn {name}", "n": n, "d": d, "k": kg.k,
            "host_call_s": sec, "fp32_Tops_incl_copies": flops / sec / 1e12,
            "float64_spot_check_50_nodes": ok}


if __name__ == "__main__":
    for name in sys.argv[1:] or ["c2_lowlid_1m", "c4_lowlid_1m_960", "knn"]:
        print(json.dumps(knn_case() if name == "knn" else gt_case(name)), flush=True)
