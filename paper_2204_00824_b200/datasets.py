"""Deterministic synthetic datasets (inputs only — not the search path).

`generate(spec)` regenerates base/query vectors bit-identically from a spec via
tools/datagen.c (libtsdg_datagen.so):
  kind "synthetic" — the reference's make_synthetic_split (bench.cpp:114-129)
  kind "lowlid"    — SURVEY.md §8(d) recipe 2 (low-LID clustered)
`load(name)` returns a Dataset with the reference-built TSDG path and ground
truth prepared by tools/make_dataset.py under data/<name>/.
"""
from __future__ import annotations

import ctypes
import json
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(_HERE)
DATA_DIR = os.path.join(ROOT, "data")
_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "_lib", "libtsdg_datagen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        lib.tsdg_fnv1a.restype = ctypes.c_uint64
        _LIB = lib
    return _LIB


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def make_synthetic(n: int, d: int, clusters: int, spread: float, seed: int) -> np.ndarray:
    out = np.empty((n, d), np.float32)
    rc = _lib().tsdg_make_synthetic(ctypes.c_uint32(n), ctypes.c_uint32(d),
                                    ctypes.c_uint32(clusters), ctypes.c_float(spread),
                                    ctypes.c_uint64(seed), _p(out))
    if rc != 0:
        raise ValueError("make_synthetic: clusters and d must be >= 1")
    return out


def make_synthetic_split(n: int, nq: int, d: int, clusters: int, spread: float, seed: int):
    base = np.empty((n, d), np.float32)
    queries = np.empty((nq, d), np.float32)
    rc = _lib().tsdg_make_synthetic_split(ctypes.c_uint32(n), ctypes.c_uint32(nq),
                                          ctypes.c_uint32(d), ctypes.c_uint32(clusters),
                                          ctypes.c_float(spread), ctypes.c_uint64(seed),
                                          _p(base), _p(queries))
    if rc != 0:
        raise ValueError("make_synthetic_split failed")
    return base, queries


def make_lowlid(n: int, nq: int, d: int, latent: int = 16, clusters: int = 50,
                spread: float = 0.25, seed: int = 1, noise: float = 0.01):
    base = np.empty((n, d), np.float32)
    queries = np.empty((nq, d), np.float32)
    rc = _lib().tsdg_make_lowlid(ctypes.c_uint32(n), ctypes.c_uint32(nq), ctypes.c_uint32(d),
                                 ctypes.c_uint32(latent), ctypes.c_uint32(clusters),
                                 ctypes.c_float(spread), ctypes.c_uint64(seed),
                                 ctypes.c_float(noise), _p(base), _p(queries))
    if rc != 0:
        raise ValueError("make_lowlid failed")
    return base, queries


def generate(spec: dict):
    if spec["kind"] == "lowlid":
        return make_lowlid(spec["n"], spec["nq"], spec["d"], spec["latent"], spec["clusters"],
                           spec["spread"], spec["seed"], spec["noise"])
    if spec["kind"] == "synthetic":
        return make_synthetic_split(spec["n"], spec["nq"], spec["d"], spec["clusters"],
                                    spec["spread"], spec["seed"])
    raise ValueError(f"unknown dataset kind {spec['kind']!r}")


def fnv1a(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    return f"{_lib().tsdg_fnv1a(_p(a), ctypes.c_uint64(a.nbytes)):016x}"


def checksums(base: np.ndarray, queries: np.ndarray) -> dict:
    return {"base": fnv1a(base), "queries": fnv1a(queries)}


@dataclass
class Dataset:
    name: str
    base: np.ndarray
    queries: np.ndarray
    graph_path: str
    gt: np.ndarray  # nq x gt_k, u32
    meta: dict


def available(name: str) -> bool:
    d = os.path.join(DATA_DIR, name)
    have_graph = any(os.path.exists(os.path.join(d, f)) for f in ("graph.tsdg", "graph.pk"))
    return have_graph and all(os.path.exists(os.path.join(d, f)) for f in ("meta.json", "gt.u32"))


def write_fvecs(path: str, a: np.ndarray) -> None:
    """fvecs (io.cpp:58-121 format: per row an int32 dimension, then the floats)."""
    a = np.ascontiguousarray(a, np.float32)
    rec = np.empty((a.shape[0], a.shape[1] + 1), np.float32)
    rec[:, 0] = np.array([a.shape[1]], np.int32).view(np.float32)[0]
    rec[:, 1:] = a
    tmp = f"{path}.tmp{os.getpid()}"
    rec.tofile(tmp)
    os.replace(tmp, path)


def ensure_fvecs(name: str, base: np.ndarray, queries: np.ndarray):
    """data/<name>/base.fvecs and queries.fvecs (the files the reference's loaders and
    tools/prepare_inputs.c read), written from the in-memory vectors when missing."""
    d = os.path.join(DATA_DIR, name)
    bpath, qpath = os.path.join(d, "base.fvecs"), os.path.join(d, "queries.fvecs")
    if not os.path.exists(bpath):
        write_fvecs(bpath, base)
    if not os.path.exists(qpath):
        write_fvecs(qpath, queries)
    return bpath, qpath


def load(name: str, verify: bool = True) -> Dataset:
    d = os.path.join(DATA_DIR, name)
    with open(os.path.join(d, "meta.json")) as f:
        meta = json.load(f)
    base, queries = generate(meta["spec"])
    if verify:
        got = checksums(base, queries)
        if got != meta["checksums"]:
            raise RuntimeError(f"dataset {name}: regenerated vectors do not match the "
                               f"checksums the graph was built from ({got} vs {meta['checksums']})")
    gpath = os.path.join(d, "graph.tsdg")
    if not os.path.exists(gpath):
        # transport form (tools/graph_pack.py): rebuilt byte-identically, checksum-verified
        import sys
        sys.path.insert(0, ROOT)
        from tools import graph_pack

        bpath, _ = ensure_fvecs(name, base, queries)
        graph_pack.unpack(os.path.join(d, "graph.pk"), bpath, gpath)
    gt = np.fromfile(os.path.join(d, "gt.u32"), np.uint32).reshape(meta["spec"]["nq"], meta["gt_k"])
    return Dataset(name, base, queries, gpath, gt, meta)
