"""C5 at its stated shape on one B200: Deep100M-shaped 100M x 96 fp32 (low-LID
clustered generator, latent 16), cut into 8 contiguous shards of 12.5M, each with its
own TSDG (nn_descent k=32, 5 iterations, sample 0.5, seed 7; build(1.2, 9)), all 8
shards resident in HBM and searched for a 10K-query batch, the per-shard top-k merged
on the device by (dist, global id) — the sharded layout of SURVEY.md §8(e) with the
8 GPUs' shard searches run one after another on this GPU (no NCCL exchange here).

The shard graphs are built by the GPU builder (nn_descent + build), whose output equals
the reference's CPU builder byte for byte (tests/test_gpu_nndescent.py: the C2 graph);
the reference would need ~1 h per shard on 8 cores.  Ground truth: the exact scan per
shard (bit-exact with the reference's ground_truth), merged by (dist, global id).

    python tools/c5_full.py [--n 100000000] [--shards 8] [--nq 10000] [--k-sweep 16,32,...]
Prints one JSON line (times, memory, QPS, recall@10); also written to --out."""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100_000_000)
    ap.add_argument("--nq", type=int, default=10_000)
    ap.add_argument("--d", type=int, default=96)
    ap.add_argument("--shards", type=int, default=8)
    ap.add_argument("--knn-k", type=int, default=32)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--k-sweep", default="16,32,64,128,256",
                    help="k_search values tried in order until recall@10 >= 0.95")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    import torch

    from paper_2204_00824_b200 import _native, datasets, shards
    from paper_2204_00824_b200.search import BestFirstParams, build, exact_topk, nn_descent

    line = {"workload": f"Deep100M-shaped {args.n}x{args.d} fp32 L2 low-LID (latent 16) in "
                        f"{args.shards} shards, {args.nq} queries, one B200",
            "graph": f"per shard: nn_descent k={args.knn_k}, {args.iters} iterations, sample 0.5, "
                     "seed 7 + build(1.2, 9), GPU builder (== the reference's output)"}
    t = time.time()
    base, queries = datasets.make_lowlid(args.n, args.nq, args.d, latent=16, seed=1)
    line["datagen_s"] = round(time.time() - t, 1)
    table = shards.shard_bounds(args.n, args.shards)
    graphs, gts, build_s = {}, [], []
    for s, (off, ns) in enumerate(table):
        sb = base[off:off + ns]
        t = time.time()
        knn = nn_descent(sb, args.knn_k, args.iters, 0.5, 7)
        t_knn = time.time() - t
        t = time.time()
        graphs[s] = build(sb, knn, 1.2, 9)
        t_build = time.time() - t
        del knn
        t = time.time()
        gi, gd = exact_topk(sb, queries, 10)
        t_gt = time.time() - t
        gts.append((gi.astype(np.int64) + off, gd))
        build_s.append({"shard": s, "n": ns, "nn_descent_s": round(t_knn, 2), "build_s": round(t_build, 2),
                        "gt_s": round(t_gt, 2), "edges": int(graphs[s].offsets[-1])})
        print(json.dumps(build_s[-1]), file=sys.stderr, flush=True)
    line["shards"] = build_s
    # exact top-10 over the whole base: merge of the shard top-10 lists by (dist, id)
    ai = np.concatenate([g[0] for g in gts], axis=1)
    ad = np.concatenate([g[1] for g in gts], axis=1)
    order = np.lexsort((ai, ad), axis=1)
    gt = np.take_along_axis(ai, order, axis=1)[:, :10].astype(np.uint32)

    t = time.time()
    searcher = shards.ShardedSearcher(graphs, {s: base[o:o + n] for s, (o, n) in enumerate(table)},
                                      table, device=0)
    line["upload_s"] = round(time.time() - t, 1)
    line["hbm_used_gb"] = round(torch.cuda.mem_get_info()[1] / 1e9 - torch.cuda.mem_get_info()[0] / 1e9, 1)
    qd = torch.from_numpy(queries).cuda()
    from bench import recall_at_k
    def run(k, mode):
        p = BestFirstParams(k=k, seed=7)
        for _ in range(2):
            ids, dists, counts = searcher.search(qd, p, mode=mode)
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ids, dists, counts = searcher.search(qd, p, mode=mode)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = float(np.median(ts))
        ih, ch = ids.cpu().numpy().view(np.uint32), counts.cpu().numpy()
        return {"k_search": k, "ms_per_batch": round(ms, 3), "qps": args.nq / ms * 1e3,
                "recall_at_10": recall_at_k(ih, ch, gt, 10), "recall_at_1": recall_at_k(ih, ch, gt, 1)}

    sweep = []
    for k in [int(x) for x in args.k_sweep.split(",")]:
        sweep.append(run(k, _native.MODE_FAST))
        print(json.dumps(sweep[-1]), file=sys.stderr, flush=True)
        if sweep[-1]["recall_at_10"] >= 0.95:
            break
    line["fast_sweep"] = sweep
    line["fast"] = dict(sweep[-1], note="every query searched on all shards, then merged")
    line["det"] = dict(run(sweep[-1]["k_search"], _native.MODE_DETERMINISTIC),
                       note="bit-exact per-shard searches (the reference's large_batch_search per shard)")
    print(json.dumps(line), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            f.write(json.dumps(line) + "\n")


if __name__ == "__main__":
    main()
