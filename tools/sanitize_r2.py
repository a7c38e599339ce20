"""Small workloads over the round-2 kernels for compute-sanitizer (memcheck /
racecheck / synccheck): GPU nn_descent, the exact scan, the fast best-first kernel in
its single and paired forms, the greedy cluster kernel with the merge warp (gather4
staging by default), the sharded index.

    compute-sanitizer --tool memcheck python tools/sanitize_r2.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2204_00824_b200 import _native, datasets, search  # noqa: E402
from paper_2204_00824_b200.search import BestFirstParams, GreedyParams  # noqa: E402

base, queries = datasets.make_synthetic_split(2000, 200, 32, 8, 0.2, 11)
g = search.nn_descent(base[:1500], 16, 2, 0.5, 7)
print("nn_descent", g.ids.shape, flush=True)
gt = search.ground_truth(base, queries[:40], 10)  # exact scan, TMA row tiles
print("exact scan", gt.ids.shape, flush=True)
idx = search.GpuIndex.from_file(os.path.join(ROOT, "tests", "golden", "syn2k.tsdg"), base)
p = BestFirstParams(k=10, seed=7)
for pair in ("0", "1"):
    os.environ["TSDG_FAST_PAIR"] = pair
    r = idx.search_bestfirst(queries[:48], p, mode=_native.MODE_FAST)
    print("bf_fast pair", pair, int(r.counts.sum()), flush=True)
r = idx.search_bestfirst(queries[:16], p)
print("bf det", int(r.counts.sum()), flush=True)
for mw in ("0", "1"):
    os.environ["TSDG_GC_MERGE_WARP"] = mw
    r = idx.search_greedy(queries[:4], 10, GreedyParams(t0=4, seed=5))
    print("greedy cta merge_warp", mw, int(r.counts.sum()), flush=True)
idx.close()
print("ok", flush=True)
