"""GPU nn_descent on the first N rows of the C2 base (ncu target):
    python tools/nnd_run.py [n] [k] [iters]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2204_00824_b200 import datasets, search  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 64
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 2
base, _ = datasets.make_lowlid(n, 1, 128, latent=16, seed=1)
st = {}
t = time.time()
g = search.nn_descent(base, k, iters, 0.5, 7, stats=st)
print(json.dumps({"n": n, "k": g.k, "iters": iters, "s": time.time() - t, **st}), flush=True)
