"""Per-phase cycle breakdown of bf_kernel on C2 (development build with
-DTSDG_PHASES).  Run: TSDG_LIB=paper_2204_00824_b200/_lib/libtsdg_gpu_phases.so \
python tools/phase_profile.py"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2204_00824_b200 import _native, datasets  # noqa: E402
from paper_2204_00824_b200.search import BestFirstParams, GpuIndex, load_tsdg  # noqa: E402

NAMES = ["start", "pop+adj", "contains", "gather_wait", "distance", "admission", "-", "-"]
ds = datasets.load("c2_lowlid_1m")
idx = GpuIndex(load_tsdg(ds.graph_path), ds.base)
lib = _native.lib()
lib.tsdg_gpu_phase_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
out = np.zeros(8, np.uint64)
nq = ds.queries.shape[0]
dq = torch.from_numpy(ds.queries).cuda()
for mode in (1, 0):
    for slots in os.environ.get("SLOTS", "16").split(","):
        os.environ["TSDG_SLOTS"] = slots
        p = BestFirstParams(k=16, seed=7)
        ids = torch.empty((nq, 16), dtype=torch.int32, device="cuda")
        dd = torch.empty((nq, 16), dtype=torch.float32, device="cuda")
        cc = torch.empty(nq, dtype=torch.int32, device="cuda")
        stt = torch.empty((nq, 4), dtype=torch.int32, device="cuda")
        idx.search_bestfirst_device(dq.data_ptr(), nq, p, ids.data_ptr(), dd.data_ptr(), cc.data_ptr(),
                                    stt.data_ptr(), 0, mode=mode)
        torch.cuda.synchronize()
        lib.tsdg_gpu_phase_read(out.ctypes.data, 1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        idx.search_bestfirst_device(dq.data_ptr(), nq, p, ids.data_ptr(), dd.data_ptr(), cc.data_ptr(),
                                    stt.data_ptr(), 0, mode=mode)
        b.record()
        torch.cuda.synchronize()
        lib.tsdg_gpu_phase_read(out.ctypes.data, 1)
        hops = int(stt.cpu().numpy()[:, 0].sum())
        tot = float(out.sum())
        print(json.dumps({"mode": "fast" if mode else "det", "slots": slots, "ms": a.elapsed_time(b),
                          "cycles_per_hop": tot / hops,
                          "share": {NAMES[i]: round(float(out[i]) / tot, 3) for i in range(6)},
                          "per_hop": {NAMES[i]: round(float(out[i]) / hops) for i in range(6)}}))
