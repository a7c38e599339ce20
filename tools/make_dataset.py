"""Offline dataset preparation (NOT the search path, never timed).

Builds one benchmark/parity dataset under data/<name>/:

  meta.json      generator parameters + FNV-1a checksums of base and queries
  graph.tsdg     TSDG built by the REFERENCE's CPU builder (north star: "the
                 graph is built by the reference's CPU builder and loaded
                 unchanged"): brute_force_knn (knn_graph.cpp:64-86) or
                 nn_descent (:141-251), then build(alpha, lambda0)
                 (diversify.cpp:152-209), written by save_tsdg (:252-272).
  gt.u32         exact top-gt_k ids per query from the reference's
                 ground_truth (bench.cpp:35-57), nq x gt_k little-endian u32.

Base and query vectors are NOT stored: they are regenerated bit-identically by
paper_2204_00824_b200.datasets (tools/datagen.c) and checked against the
checksums in meta.json.  The reference library is reached through
oracle/_ref/libtsdg_ref.so (built from /root/reference by oracle/Makefile),
so this tool only runs where the reference sources were present.

Usage:
  python tools/make_dataset.py --name c2_lowlid_1m --kind lowlid --n 1000000 \
      --nq 10000 --d 128 --latent 16 --builder nndescent --knn-k 64 --iters 5
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


def _ref():
    lib = ctypes.CDLL(os.path.join(ROOT, "oracle", "_ref", "libtsdg_ref.so"))
    lib.ref_last_error.restype = ctypes.c_char_p
    return lib


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--name", required=True)
    ap.add_argument("--kind", choices=["lowlid", "synthetic"], default="lowlid")
    ap.add_argument("--n", type=int, required=True)
    ap.add_argument("--nq", type=int, required=True)
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--latent", type=int, default=16)
    ap.add_argument("--clusters", type=int, default=50)
    ap.add_argument("--spread", type=float, default=0.25)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--noise", type=float, default=0.01)
    ap.add_argument("--builder", choices=["brute", "nndescent"], default="nndescent")
    ap.add_argument("--knn-k", type=int, default=64)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--sample-rate", type=float, default=0.5)
    ap.add_argument("--knn-seed", type=int, default=7)
    ap.add_argument("--alpha", type=float, default=1.2)
    ap.add_argument("--lambda0", type=int, default=9)
    ap.add_argument("--gt-k", type=int, default=100)
    ap.add_argument("--gt", choices=["ref", "gpu"], default="ref",
                    help="ground truth by the reference (CPU) or by the GPU exact scan "
                         "(bit-identical ids, tests/test_scan.py)")
    args = ap.parse_args()

    spec = {
        "kind": args.kind, "n": args.n, "nq": args.nq, "d": args.d,
        "latent": args.latent, "clusters": args.clusters, "spread": args.spread,
        "seed": args.seed, "noise": args.noise,
    }
    out_dir = os.path.join(ROOT, "data", args.name)
    os.makedirs(out_dir, exist_ok=True)
    t0 = time.time()
    base, queries = datasets.generate(spec)
    print(f"[make_dataset] vectors {base.shape} + {queries.shape} in {time.time()-t0:.1f}s",
          flush=True)

    ref = _ref()
    graph_path = os.path.join(out_dir, "graph.tsdg")
    stats = (ctypes.c_uint64 * 4)()
    t0 = time.time()
    rc = ref.ref_build_tsdg(
        base.ctypes.data_as(ctypes.c_void_p), ctypes.c_uint32(args.n), ctypes.c_uint32(args.d),
        0, 0 if args.builder == "brute" else 1, ctypes.c_uint32(args.knn_k),
        ctypes.c_uint32(args.iters), ctypes.c_double(args.sample_rate),
        ctypes.c_uint64(args.knn_seed), ctypes.c_float(args.alpha),
        ctypes.c_uint32(args.lambda0), ctypes.c_uint32(0), graph_path.encode(), stats)
    if rc != 0:
        raise RuntimeError(ref.ref_last_error().decode())
    build_s = time.time() - t0
    print(f"[make_dataset] graph built in {build_s:.1f}s stats={list(stats)}", flush=True)

    t0 = time.time()
    gt_k = min(args.gt_k, args.n)
    if args.gt == "gpu":
        from paper_2204_00824_b200.search import ground_truth
        gt = np.ascontiguousarray(ground_truth(base, queries, gt_k).ids)
    else:
        gt = np.zeros((args.nq, gt_k), np.uint32)
        rc = ref.ref_ground_truth(
            base.ctypes.data_as(ctypes.c_void_p), ctypes.c_uint32(args.n),
            queries.ctypes.data_as(ctypes.c_void_p), ctypes.c_uint32(args.nq),
            ctypes.c_uint32(args.d), ctypes.c_uint32(gt_k), 0, gt.ctypes.data_as(ctypes.c_void_p))
        if rc != 0:
            raise RuntimeError(ref.ref_last_error().decode())
    gt.tofile(os.path.join(out_dir, "gt.u32"))
    print(f"[make_dataset] ground truth in {time.time()-t0:.1f}s", flush=True)

    meta = {
        "spec": spec,
        "graph": {
            "builder": args.builder, "knn_k": args.knn_k, "iters": args.iters,
            "sample_rate": args.sample_rate, "knn_seed": args.knn_seed,
            "alpha": args.alpha, "lambda0": args.lambda0,
            "build_stats": {"input_edges": stats[0], "stage1_edges": stats[1],
                            "augmented_edges": stats[2], "final_edges": stats[3]},
            "build_seconds": round(build_s, 1),
        },
        "gt_k": gt_k,
        "checksums": datasets.checksums(base, queries),
    }
    with open(os.path.join(out_dir, "meta.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("[make_dataset] done", out_dir)


if __name__ == "__main__":
    main()
