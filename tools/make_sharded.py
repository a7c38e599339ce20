"""Offline preparation of a SHARDED dataset (config C5 shape, scaled): the base set
is cut into S contiguous shards, each gets its own TSDG built by the reference's
CPU builder (nn_descent + build(alpha, lambda0), knn_graph.cpp:141-251,
diversify.cpp:152-209) over LOCAL ids; global id = shard offset + local id.

data/<name>/meta.json        spec + shard table + checksums
data/<name>/shard_<s>.tsdg   per-shard TSDG (plus shard_<s>.pk transport form)
data/<name>/gt.u32           exact top-gt_k over the WHOLE base (reference ground_truth)

python tools/make_sharded.py --name c5s_lowlid_2m_96 --n 2000000 --nq 10000 --d 96 \
    --latent 16 --shards 8 --knn-k 32 --iters 5
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2204_00824_b200 import datasets  # noqa: E402
from tools import graph_pack  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--name", required=True)
    ap.add_argument("--n", type=int, required=True)
    ap.add_argument("--nq", type=int, default=10000)
    ap.add_argument("--d", type=int, default=96)
    ap.add_argument("--latent", type=int, default=16)
    ap.add_argument("--clusters", type=int, default=50)
    ap.add_argument("--spread", type=float, default=0.25)
    ap.add_argument("--seed", type=int, default=5)
    ap.add_argument("--noise", type=float, default=0.01)
    ap.add_argument("--shards", type=int, default=8)
    ap.add_argument("--knn-k", type=int, default=32)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--sample-rate", type=float, default=0.5)
    ap.add_argument("--gt-k", type=int, default=100)
    ap.add_argument("--gt-queries", type=int, default=2000)
    args = ap.parse_args()
    spec = {"kind": "lowlid", "n": args.n, "nq": args.nq, "d": args.d, "latent": args.latent,
            "clusters": args.clusters, "spread": args.spread, "seed": args.seed,
            "noise": args.noise}
    out = os.path.join(ROOT, "data", args.name)
    os.makedirs(out, exist_ok=True)
    base, queries = datasets.generate(spec)
    ref = ctypes.CDLL(os.path.join(ROOT, "oracle", "_ref", "libtsdg_ref.so"))
    ref.ref_last_error.restype = ctypes.c_char_p
    S = args.shards
    bounds = [(s * args.n) // S for s in range(S + 1)]
    shards = []
    for s in range(S):
        lo, hi = bounds[s], bounds[s + 1]
        part = np.ascontiguousarray(base[lo:hi])
        path = os.path.join(out, f"shard_{s}.tsdg")
        stats = (ctypes.c_uint64 * 4)()
        t0 = time.time()
        rc = ref.ref_build_tsdg(part.ctypes.data_as(ctypes.c_void_p), ctypes.c_uint32(hi - lo),
                                ctypes.c_uint32(args.d), 0, 1, ctypes.c_uint32(args.knn_k),
                                ctypes.c_uint32(args.iters), ctypes.c_double(args.sample_rate),
                                ctypes.c_uint64(7 + s), ctypes.c_float(1.2), ctypes.c_uint32(9),
                                ctypes.c_uint32(0), path.encode(), stats)
        if rc:
            raise RuntimeError(ref.ref_last_error().decode())
        graph_pack.pack(path, os.path.join(out, f"shard_{s}.pk"))
        shards.append({"offset": lo, "n": hi - lo, "build_stats": list(stats),
                       "build_seconds": round(time.time() - t0, 1)})
        print(f"[make_sharded] shard {s}: {hi-lo} nodes in {time.time()-t0:.1f}s", flush=True)
    nq_gt = min(args.gt_queries, args.nq)
    gt = np.zeros((nq_gt, args.gt_k), np.uint32)
    t0 = time.time()
    rc = ref.ref_ground_truth(base.ctypes.data_as(ctypes.c_void_p), ctypes.c_uint32(args.n),
                              queries.ctypes.data_as(ctypes.c_void_p), ctypes.c_uint32(nq_gt),
                              ctypes.c_uint32(args.d), ctypes.c_uint32(args.gt_k), 0,
                              gt.ctypes.data_as(ctypes.c_void_p))
    if rc:
        raise RuntimeError(ref.ref_last_error().decode())
    gt.tofile(os.path.join(out, "gt.u32"))
    print(f"[make_sharded] ground truth ({nq_gt} queries) in {time.time()-t0:.1f}s", flush=True)
    meta = {"spec": spec, "shards": shards, "gt_k": args.gt_k, "gt_queries": nq_gt,
            "graph": {"builder": "nndescent", "knn_k": args.knn_k, "iters": args.iters,
                      "sample_rate": args.sample_rate, "alpha": 1.2, "lambda0": 9},
            "checksums": datasets.checksums(base, queries)}
    with open(os.path.join(out, "meta.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("[make_sharded] done", out)


if __name__ == "__main__":
    main()
