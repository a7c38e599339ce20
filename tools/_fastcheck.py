import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2204_00824_b200 import datasets, search, _native
base, queries = datasets.make_synthetic_split(2000, 200, 32, 8, 0.2, 11)
idx = search.GpuIndex.from_file("tests/golden/syn2k.tsdg", base, device=0)
p = search.BestFirstParams(k=10, seed=7)
for v in sys.argv[1:]:
    os.environ["TSDG_FAST_VARIANT"] = v
    r = idx.search_bestfirst(queries, p, mode=_native.MODE_FAST)
    d = idx.search_bestfirst(queries, p)
    print(v, "agree", (r.ids == d.ids).mean(), flush=True)
