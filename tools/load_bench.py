"""Index load time, file -> searchable device index.

Compares, on one dataset (default C2: 1M x 128, reference-built TSDG;
LOAD_DATASET=synth: a C2-sized random graph + vectors generated in place):
  files    GpuIndex.from_files: raw .tsdg + fvecs bytes -> pinned staging -> HBM,
           decoded on the device (tsdg_gpu_index_create_from_files)
  host     our host loaders (tsdg_read_tsdg one mmap pass, tsdg_read_vectors) then
           GpuIndex(graph, base)
  ref      the reference's load_tsdg + load_vectors (oracle/_ref, host RAM only;
           no device upload) -- the loader the reference tooling uses
and checks that the two device indexes give identical search results.  The page
cache is warm for every arm after the first pass (each arm runs twice; the JSON
reports both).  Development tool; prints one JSON line per measurement.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2204_00824_b200 import datasets  # noqa: E402
from paper_2204_00824_b200.search import (BestFirstParams, GpuIndex, load_tsdg,  # noqa: E402
                                          read_vectors)


def write_fvecs(path, x):
    n, d = x.shape
    rec = np.empty((n, d + 1), np.float32)
    rec[:, 0] = np.array([d], np.int32).view(np.float32)[0]
    rec[:, 1:] = x
    rec.tofile(path)


def write_random_tsdg(path, n, seed=1, lo=30, hi=50):
    """A C2-sized TSDG with random adjacency (load timing only; format
    diversify.hpp:122-125)."""
    rng = np.random.default_rng(seed)
    deg = rng.integers(lo, hi + 1, n).astype(np.uint32)
    E = int(deg.sum())
    edge = np.zeros(E, dtype=[("t", "<u4"), ("l", "<u2"), ("d", "<f4")])
    edge["t"] = rng.integers(0, n, E, dtype=np.uint32)
    edge["l"] = rng.integers(0, 10, E).astype(np.uint16)
    edge["d"] = rng.random(E, dtype=np.float32)
    eb = edge.view(np.uint8).reshape(E, 10)
    body = np.empty(4 * n + 10 * E, np.uint8)
    starts = np.zeros(n, np.int64)
    starts[1:] = np.cumsum(4 + 10 * deg.astype(np.int64))[:-1]
    for j in range(4):
        body[starts + j] = ((deg >> (8 * j)) & 0xFF).astype(np.uint8)
    d64 = deg.astype(np.int64)
    eoff = np.repeat(starts + 4, d64) + 10 * (np.arange(E, dtype=np.int64) - np.repeat(np.cumsum(d64) - d64, d64))
    for j in range(10):
        body[eoff + j] = eb[:, j]
    hdr = b"TSDG" + np.array([1], "<u4").tobytes() + np.array([n], "<u8").tobytes() + bytes([0]) + \
        np.array([64], "<u4").tobytes() + np.array([1.2], "<f4").tobytes() + np.array([9], "<u2").tobytes()
    with open(path, "wb") as f:
        f.write(hdr)
        f.write(body.tobytes())


class _Synth:
    def __init__(self, n=1_000_000, d=128, nq=2000):
        rng = np.random.default_rng(5)
        self.base = rng.random((n, d), dtype=np.float32)
        self.queries = rng.random((nq, d), dtype=np.float32)
        self.graph_path = os.path.join(os.environ.get("TMPDIR", "/tmp"), "synth_load.tsdg")
        write_random_tsdg(self.graph_path, n)


def main():
    import torch
    name = os.environ.get("LOAD_DATASET", "c2_lowlid_1m")
    ds = _Synth() if name == "synth" else datasets.load(name)
    vpath = os.path.join(os.environ.get("TMPDIR", "/tmp"), f"{name}_base.fvecs")
    write_fvecs(vpath, ds.base)
    gpath = ds.graph_path
    sizes = {"tsdg_bytes": os.path.getsize(gpath), "fvecs_bytes": os.path.getsize(vpath)}
    out = []

    def emit(arm, rep, sec, **kw):
        line = {"dataset": name, "arm": arm, "rep": rep, "s": round(sec, 4),
                "GBps_files": round((sizes["tsdg_bytes"] + sizes["fvecs_bytes"]) / sec / 1e9, 3), **sizes, **kw}
        print(json.dumps(line), flush=True)
        out.append(line)

    torch.cuda.init()
    for rep in range(2):
        t = time.perf_counter()
        a = GpuIndex.from_files(gpath, vpath)
        torch.cuda.synchronize()
        emit("files", rep, time.perf_counter() - t)
        if rep == 0:
            keep_a = a
        else:
            a.close()
    for rep in range(2):
        t = time.perf_counter()
        g = load_tsdg(gpath)
        t1 = time.perf_counter()
        base = read_vectors(vpath)
        t2 = time.perf_counter()
        b = GpuIndex(g, base)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        emit("host", rep, t3 - t, read_tsdg_s=round(t1 - t, 4), read_vectors_s=round(t2 - t1, 4),
             upload_s=round(t3 - t2, 4))
        if rep == 0:
            keep_b = b
        else:
            b.close()
    try:
        from oracle import oracle as O  # reference loaders, timing only
        if O.ref_available():
            ref = O.Ref()
            for rep in range(2):
                t = time.perf_counter()
                base_r = ref.load_vectors(vpath)
                t1 = time.perf_counter()
                fx = ref.fixture(gpath, base_r)
                t2 = time.perf_counter()
                emit("ref", rep, t2 - t, load_vectors_s=round(t1 - t, 4), load_tsdg_s=round(t2 - t1, 4))
                del fx
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"arm": "ref", "error": str(e)}))
    p = BestFirstParams(k=14, seed=7, lambda_cut=5)
    q = ds.queries[:2000]
    ra, rb = keep_a.search_bestfirst(q, p), keep_b.search_bestfirst(q, p)
    same = bool(np.array_equal(ra.ids, rb.ids) and np.array_equal(ra.dists.view(np.uint32), rb.dists.view(np.uint32)))
    print(json.dumps({"dataset": name, "identical_search": same}), flush=True)
    if os.environ.get("LOAD_OUT"):
        with open(os.environ["LOAD_OUT"], "w") as f:
            for line in out:
                f.write(json.dumps(line) + "\n")
            f.write(json.dumps({"dataset": name, "identical_search": same}) + "\n")
    os.remove(vpath)
    if name == "synth":
        os.remove(gpath)


if __name__ == "__main__":
    main()
