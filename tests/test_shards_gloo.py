"""CPU, world_size 2 over gloo: the multi-GPU plumbing of shards.py with the CPU
oracle standing in for the per-GPU search (no CUDA here).

* replicated: each rank searches its query slice with query_index_base = slice
  start; the gathered slices equal the single-process batch exactly.
* sharded: each rank searches all queries on its shard block; the gathered
  per-shard lists merged by (dist, global id) equal the single-process merge over
  all shards."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import json
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle import oracle as O
    from paper_2204_00824_b200 import datasets, shards
    from paper_2204_00824_b200.search import BestFirstParams

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        meta = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))
        orc = O.Oracle()
        p = BestFirstParams(k=10, seed=21)
        # replicated
        from conftest import fixture_data
        g, b, qs = fixture_data(meta, "syn2k")
        q0, q1 = shards.query_slice(qs.shape[0], world, rank)
        r = orc.large_batch(g, b, qs[q0:q1], p, qbase=q0)
        sizes = [None] * world
        dist.all_gather_object(sizes, (q0, q1))
        parts = [None] * world
        dist.all_gather_object(parts, r.ids)
        rep_ids = np.concatenate(parts)
        # sharded
        fx = meta["fixtures"]["shards4"]
        spec = dict(fx["spec"], latent=0, noise=0.0)
        sb, sq = datasets.generate(spec)
        table = [tuple(t) for t in fx["shards"]]
        mine = shards.shards_of_rank(len(table), world, rank)
        li, ld, lc = [], [], []
        for s in mine:
            off, n = table[s]
            gs = O.parse_tsdg(os.path.join(ROOT, "tests", "golden", f"shard4_{s}.tsdg"))
            rr = orc.large_batch(gs, sb[off:off + n], sq, p)
            li.append(rr.ids.view(np.int32))
            ld.append(rr.dists)
            lc.append(rr.counts.view(np.int32))
        gi, gd, gc = shards.gather_shard_results(torch.from_numpy(np.stack(li)),
                                                 torch.from_numpy(np.stack(ld)),
                                                 torch.from_numpy(np.stack(lc)))
        merged = shards.merge_shards_host(gi.numpy().view(np.uint32), gd.numpy(),
                                          gc.numpy().view(np.uint32), [t[0] for t in table], p.k)
        if rank == 0:
            q.put((rep_ids, merged[0], merged[1], merged[2]))
    finally:
        dist.destroy_process_group()


def test_world2_gloo_replicated_and_sharded(golden_meta, golden):
    from oracle import oracle as O
    from paper_2204_00824_b200 import datasets, shards
    from paper_2204_00824_b200.search import BestFirstParams
    from conftest import fixture_data

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    rep_ids, mi, md, mc = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    orc = O.Oracle()
    p = BestFirstParams(k=10, seed=21)
    g, b, qs = fixture_data(golden_meta, "syn2k")
    np.testing.assert_array_equal(rep_ids, orc.large_batch(g, b, qs, p).ids)
    # single-process merge over all 4 shards
    fx = golden_meta["fixtures"]["shards4"]
    sb, sq = datasets.generate(dict(fx["spec"], latent=0, noise=0.0))
    res = []
    for s, (off, n) in enumerate(fx["shards"]):
        gs = O.parse_tsdg(os.path.join(ROOT, "tests", "golden", f"shard4_{s}.tsdg"))
        res.append(orc.large_batch(gs, sb[off:off + n], sq, p))
    wi, wd, wc = shards.merge_shards_host(np.stack([r.ids for r in res]),
                                          np.stack([r.dists for r in res]),
                                          np.stack([r.counts for r in res]),
                                          [t[0] for t in fx["shards"]], p.k)
    np.testing.assert_array_equal(mi, wi)
    np.testing.assert_array_equal(md, wd)
    np.testing.assert_array_equal(mc, wc)
    # merged results are real nearest neighbours of the whole base
    assert O.recall_at_k(mi, mc, golden["shards4_gt"], 10) > 0.5


def test_shard_bookkeeping():
    from paper_2204_00824_b200 import shards
    assert shards.shard_bounds(10, 4) == [(0, 2), (2, 3), (5, 2), (7, 3)]
    assert shards.shards_of_rank(8, 4, 3) == [6, 7]
    with pytest.raises(ValueError):
        shards.shards_of_rank(6, 4, 0)
    assert [shards.query_slice(10, 3, r) for r in range(3)] == [(0, 3), (3, 6), (6, 10)]
