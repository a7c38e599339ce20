"""GPU: sharded search (shards.ShardedSearcher, all shards on cuda:0) against the
oracle run per shard and merged on the host by (dist, global id)."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2204_00824_b200 import datasets, shards
from paper_2204_00824_b200.search import BestFirstParams, load_tsdg

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_sharded_search_matches_oracle_merge(golden_meta):
    import torch
    fx = golden_meta["fixtures"]["shards4"]
    sb, sq = datasets.generate(dict(fx["spec"], latent=0, noise=0.0))
    table = [tuple(t) for t in fx["shards"]]
    paths = [os.path.join(ROOT, "tests", "golden", f"shard4_{s}.tsdg") for s in range(4)]
    searcher = shards.ShardedSearcher({s: load_tsdg(paths[s]) for s in range(4)},
                                      {s: sb[o:o + n] for s, (o, n) in enumerate(table)}, table)
    orc = O.Oracle()
    for p in (BestFirstParams(k=10, seed=21), BestFirstParams(k=32, seed=3, m_segments=4)):
        qd = torch.from_numpy(sq).cuda()
        ids, dists, counts = searcher.search(qd, p)
        torch.cuda.synchronize()
        res = [orc.large_batch(O.parse_tsdg(paths[s]), sb[o:o + n], sq, p)
               for s, (o, n) in enumerate(table)]
        wi, wd, wc = shards.merge_shards_host(np.stack([r.ids for r in res]),
                                              np.stack([r.dists for r in res]),
                                              np.stack([r.counts for r in res]),
                                              [t[0] for t in table], p.k)
        np.testing.assert_array_equal(ids.cpu().numpy().view(np.uint32), wi)
        np.testing.assert_array_equal(dists.cpu().numpy().view(np.uint32), wd.view(np.uint32))
        np.testing.assert_array_equal(counts.cpu().numpy().view(np.uint32), wc)


def test_sharded_index_c_abi_matches_oracle_merge(golden_meta):
    """The in-process sharded index (C-ABI tsdg_gpu_sharded_*, peer copies + device
    merge; the four shards placed on one GPU here) equals the oracle's per-shard
    searches merged on the host."""
    from paper_2204_00824_b200.search import ShardedGpuIndex
    fx = golden_meta["fixtures"]["shards4"]
    sb, sq = datasets.generate(dict(fx["spec"], latent=0, noise=0.0))
    table = [tuple(t) for t in fx["shards"]]
    paths = [os.path.join(ROOT, "tests", "golden", f"shard4_{s}.tsdg") for s in range(4)]
    idx = ShardedGpuIndex(paths, [sb[o:o + n] for o, n in table], [o for o, _ in table],
                          devices=[0, 0, 0, 0])
    orc = O.Oracle()
    for p in (BestFirstParams(k=10, seed=21), BestFirstParams(k=32, seed=3, m_segments=4)):
        ids, dists, counts = idx.search_bestfirst(sq, p, query_index_base=7)
        res = [orc.large_batch(O.parse_tsdg(paths[s]), sb[o:o + n], sq, p, qbase=7)
               for s, (o, n) in enumerate(table)]
        wi, wd, wc = shards.merge_shards_host(np.stack([r.ids for r in res]),
                                              np.stack([r.dists for r in res]),
                                              np.stack([r.counts for r in res]),
                                              [t[0] for t in table], p.k)
        np.testing.assert_array_equal(ids, wi)
        np.testing.assert_array_equal(dists.view(np.uint32), wd.view(np.uint32))
        np.testing.assert_array_equal(counts, wc)
    idx.close()


def test_sharded_searcher_over_nccl_group(golden_meta):
    """The multi-GPU sharded path on the B200 with a real NCCL process group (one rank
    here: the box has one GPU): per-shard searches, all_gather_into_tensor over NCCL on
    the search stream, device merge — equal to the oracle's per-shard searches merged
    on the host."""
    import socket

    import torch
    import torch.distributed as dist

    if dist.is_initialized():
        pytest.skip("a process group already exists")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        fx = golden_meta["fixtures"]["shards4"]
        sb, sq = datasets.generate(dict(fx["spec"], latent=0, noise=0.0))
        table = [tuple(t) for t in fx["shards"]]
        paths = [os.path.join(ROOT, "tests", "golden", f"shard4_{s}.tsdg") for s in range(4)]
        searcher = shards.ShardedSearcher({s: load_tsdg(paths[s]) for s in range(4)},
                                          {s: sb[o:o + n] for s, (o, n) in enumerate(table)}, table,
                                          group=dist.group.WORLD)
        p = BestFirstParams(k=10, seed=21)
        ids, dists, counts = searcher.search(torch.from_numpy(sq).cuda(), p)
        torch.cuda.synchronize()
        orc = O.Oracle()
        res = [orc.large_batch(O.parse_tsdg(paths[s]), sb[o:o + n], sq, p) for s, (o, n) in enumerate(table)]
        wi, wd, wc = shards.merge_shards_host(np.stack([r.ids for r in res]), np.stack([r.dists for r in res]),
                                              np.stack([r.counts for r in res]), [t[0] for t in table], p.k)
        np.testing.assert_array_equal(ids.cpu().numpy().view(np.uint32), wi)
        np.testing.assert_array_equal(dists.cpu().numpy().view(np.uint32), wd.view(np.uint32))
    finally:
        dist.destroy_process_group()
