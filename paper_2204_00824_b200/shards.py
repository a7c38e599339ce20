"""Multi-GPU search: one process per GPU, torch.distributed for the plumbing.

Two layouts:

* replicated — the whole index on every GPU; the query batch is split into
  contiguous slices, slice r searched on rank r with query_index_base = slice
  start so query q keeps the reference's RNG stream Rng64(seed).fork(q)
  (bestfirst_search.cpp:136-143).  No collective on the data path; results are
  identical for any GPU count.
* sharded — the base set is cut into S contiguous shards, each with its own TSDG
  over local ids (global id = shard offset + local id).  Every rank searches ALL
  queries on the shards it holds, the per-shard top-k lists (ids, dists, counts)
  are exchanged with one all-gather (NCCL over NVLink on B200), and
  merge_shards_kernel merges them by (dist, global id) on the device.  The
  reference has no sharding; its per-shard searches merged on the host are the
  parity oracle (tests/test_gpu_shards.py).

The bookkeeping here (shard ownership, gather layout, id offsets) is shared by the
GPU path and the CPU gloo tests (tests/test_shards_gloo.py), which substitute the
oracle for the GPU search.
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple

import numpy as np

KINVALID = 0xFFFFFFFF


def shard_bounds(n_total: int, shards: int) -> List[Tuple[int, int]]:
    """(offset, n) of each contiguous shard."""
    b = [(s * n_total) // shards for s in range(shards + 1)]
    return [(b[s], b[s + 1] - b[s]) for s in range(shards)]


def shards_of_rank(num_shards: int, world: int, rank: int) -> List[int]:
    """Contiguous block of shard indices owned by `rank` (num_shards % world == 0)."""
    if num_shards % world:
        raise ValueError(f"{num_shards} shards cannot be split evenly over {world} ranks")
    per = num_shards // world
    return list(range(rank * per, (rank + 1) * per))


def query_slice(nq: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous query slice of `rank` in the replicated layout."""
    b = [(r * nq) // world for r in range(world + 1)]
    return b[rank], b[rank + 1]


def merge_shards_host(ids: np.ndarray, dists: np.ndarray, counts: np.ndarray,
                      shard_base: Sequence[int], k: int):
    """Host statement of the merge (the semantics merge_shards_kernel implements):
    union of every shard's first counts[s, q] entries, global id = base + local id,
    ascending by (dist, global id), first k.  ids/dists: [S, nq, k], counts [S, nq]."""
    S, nq, _ = ids.shape
    out_i = np.full((nq, k), KINVALID, np.uint32)
    out_d = np.full((nq, k), np.inf, np.float32)
    out_c = np.zeros(nq, np.uint32)
    for q in range(nq):
        cand = []
        for s in range(S):
            c = int(counts[s, q])
            for j in range(min(c, k)):
                cand.append((float(dists[s, q, j]), int(shard_base[s]) + int(ids[s, q, j])))
        cand.sort()
        cand = cand[:k]
        out_c[q] = len(cand)
        for j, (dd, ii) in enumerate(cand):
            out_i[q, j] = ii
            out_d[q, j] = dd
    return out_i, out_d, out_c


def gather_shard_results(local_ids, local_dists, local_counts, group=None):
    """All-gather the per-shard result blocks of every rank ([S_local, nq, k] each)
    into [world * S_local, nq, k] in rank order (= global shard order, since ranks
    own contiguous shard blocks).  Works on CUDA tensors over NCCL and CPU tensors
    over gloo."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    outs = []
    for t in (local_ids, local_dists, local_counts):
        full = torch.empty((world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype,
                           device=t.device)
        if t.is_cuda:
            dist.all_gather_into_tensor(full, t.contiguous(), group=group)
        else:
            parts = list(full.chunk(world, dim=0))
            dist.all_gather(parts, t.contiguous(), group=group)
            full = torch.cat(parts, dim=0)
        outs.append(full)
    return tuple(outs)


class ShardedSearcher:
    """Sharded best-first search on this rank's GPU (or all shards on one GPU when
    no process group is given)."""

    def __init__(self, shard_graphs: Dict[int, object], shard_bases: Dict[int, np.ndarray],
                 shard_table: Sequence[Tuple[int, int]], device: int = 0, group=None):
        from .search import GpuIndex

        self.table = list(shard_table)
        self.num_shards = len(self.table)
        self.local = sorted(shard_graphs)
        self.group = group
        self.device = device
        self.indexes = {s: GpuIndex(shard_graphs[s], shard_bases[s], device=device)
                        for s in self.local}

    def search(self, queries_dev, params, mode: int = 0, stream: int = 0):
        """queries_dev: CUDA float32 [nq, d].  Returns CUDA (ids int32 [nq,k] global,
        dists [nq,k], counts [nq]) merged over all shards."""
        import torch
        import torch.distributed as dist

        from .search import merge_shards_device

        nq, k = int(queries_dev.shape[0]), int(params.k)
        dev = queries_dev.device
        if not stream:  # order the searches with the collective on torch's current stream
            stream = torch.cuda.current_stream(dev).cuda_stream
        L = len(self.local)
        ids = torch.empty((L, nq, k), dtype=torch.int32, device=dev)
        dists = torch.empty((L, nq, k), dtype=torch.float32, device=dev)
        counts = torch.empty((L, nq), dtype=torch.int32, device=dev)
        for j, s in enumerate(self.local):
            self.indexes[s].search_bestfirst_device(
                queries_dev.data_ptr(), nq, params, ids[j].data_ptr(), dists[j].data_ptr(),
                counts[j].data_ptr(), 0, stream, query_index_base=0, mode=mode)
        if self.group is not None or (dist.is_available() and dist.is_initialized()
                                      and dist.get_world_size() > 1):
            g_ids, g_dists, g_counts = gather_shard_results(ids, dists, counts, self.group)
        else:
            g_ids, g_dists, g_counts = ids, dists, counts
        S = g_ids.shape[0]
        out_i = torch.empty((nq, k), dtype=torch.int32, device=dev)
        out_d = torch.empty((nq, k), dtype=torch.float32, device=dev)
        out_c = torch.empty(nq, dtype=torch.int32, device=dev)
        merge_shards_device(g_ids.data_ptr(), g_dists.data_ptr(), g_counts.data_ptr(),
                            [off for off, _ in self.table][:S], S, nq, k, out_i.data_ptr(),
                            out_d.data_ptr(), out_c.data_ptr(), stream)
        return out_i, out_d, out_c
