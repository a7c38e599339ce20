"""Graph construction on the GPU: k-NN graph (exact,
brute_force_knn, knn_graph.cpp:64-86, or nn_descent, :141-251) + two-stage
diversification (build, diversify.cpp:152-209), written in the reference's TSDG format.

    python tools/gpu_build.py <dataset> [--builder brute|nndescent|meta] [--knn-k 100]
        [--alpha 1.2] [--lambda0 9] [--out path] [--compare path.tsdg]

--builder meta takes the builder and its parameters from the dataset's meta.json (the
reference's own run that made data/<dataset>/graph.tsdg), so --compare against that
file checks the whole GPU pipeline against the reference's graph byte for byte.

Prints one JSON line: seconds per stage (host wall clock around each C-ABI call,
uploads included), BuildStats, and whether the output equals --compare byte for byte
(e.g. a graph the reference built from brute_force_knn with the same parameters)."""
import argparse
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2204_00824_b200 import datasets, search  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("dataset")
    ap.add_argument("--builder", choices=["brute", "nndescent", "meta"], default="brute")
    ap.add_argument("--knn-k", type=int, default=100)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--sample-rate", type=float, default=0.5)
    ap.add_argument("--knn-seed", type=int, default=7)
    ap.add_argument("--alpha", type=float, default=1.2)
    ap.add_argument("--lambda0", type=int, default=9)
    ap.add_argument("--max-degree", type=int, default=0)
    ap.add_argument("--out", default=None)
    ap.add_argument("--compare", default=None)
    args = ap.parse_args()
    with open(os.path.join(datasets.DATA_DIR, args.dataset, "meta.json")) as f:
        meta = json.load(f)
    base, _ = datasets.generate(meta["spec"])
    if args.builder == "meta":
        gm = meta["graph"]
        args.builder, args.knn_k, args.alpha, args.lambda0 = (gm["builder"], gm["knn_k"],
                                                              gm["alpha"], gm["lambda0"])
        if args.builder == "nndescent":
            args.iters, args.sample_rate, args.knn_seed = gm["iters"], gm["sample_rate"], gm["knn_seed"]
    nd_stats = {}
    t0 = time.perf_counter()
    if args.builder == "nndescent":
        knn = search.nn_descent(base, args.knn_k, args.iters, args.sample_rate, args.knn_seed,
                                stats=nd_stats)
    else:
        knn = search.brute_force_knn(base, args.knn_k)
    t_knn = time.perf_counter() - t0
    out = args.out or os.path.join(tempfile.mkdtemp(), "gpu.tsdg")
    st = search.BuildStats()
    t0 = time.perf_counter()
    g = search.build(base, knn, args.alpha, args.lambda0, args.max_degree, save_path=out, stats=st)
    t_build = time.perf_counter() - t0
    line = {"dataset": args.dataset, "n": int(base.shape[0]), "d": int(base.shape[1]),
            "builder": args.builder, "knn_k": knn.k, "knn_s": t_knn, "build_s": t_build,
            "stats": {"input_edges": st.input_edges, "stage1_edges": st.stage1_edges,
                      "augmented_edges": st.augmented_edges, "final_edges": st.final_edges},
            "max_degree": g.max_degree, "out": out}
    if args.builder == "nndescent":
        line["nn_descent"] = {"iters": args.iters, "sample_rate": args.sample_rate,
                              "seed": args.knn_seed, **nd_stats}
        if meta.get("graph", {}).get("builder") == "nndescent":
            line["reference_build_s"] = meta["graph"].get("build_seconds")
    if args.compare:
        with open(out, "rb") as a, open(args.compare, "rb") as b:
            line["equals_compare"] = a.read() == b.read()
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
