"""Transport encoding of a reference-built TSDG file (saves push bandwidth to the
GPU box; the search never reads this form).

pack:   graph.tsdg -> graph.pk  (header fields, degrees, and per edge the
        target and lambda packed into ceil((bits(n)+bits(lambda0))/8) bytes; the
        fp32 edge distances are dropped because they are exactly recomputable)
unpack: graph.pk + base vectors -> graph.tsdg, byte-identical to the
        original: distances recomputed in the reference's sequential fp32 order
        (tools/datagen.c tsdg_edge_distances), then the whole file's FNV-1a is
        checked against the checksum of the original recorded at pack time.
        tools/prepare_inputs.c does the same from a base.fvecs file (the
        reference arm of bench.py, which maps no library of this repository).
"""
from __future__ import annotations

import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2204_00824_b200 import datasets  # noqa: E402


def _fnv_file(path: str) -> str:
    return datasets.fnv1a(np.fromfile(path, np.uint8))


def _parse(path: str):
    raw = np.fromfile(path, np.uint8)
    assert raw[:4].tobytes() == b"TSDG"
    hdr = raw[:27].copy()
    n = int(np.frombuffer(hdr[8:16].tobytes(), "<u8")[0])
    # walk degrees with a vectorised pointer chase in chunks
    degs = np.empty(n, np.uint32)
    off = 27
    pos = np.empty(n, np.int64)
    for u in range(n):
        d = int(raw[off]) | int(raw[off + 1]) << 8 | int(raw[off + 2]) << 16 | int(raw[off + 3]) << 24
        degs[u] = d
        pos[u] = off + 4
        off += 4 + 10 * d
    E = int(degs.sum(dtype=np.uint64))
    # gather edge records
    starts = np.repeat(pos, degs) + 10 * (np.arange(E) - np.repeat(np.cumsum(degs, dtype=np.int64) - degs, degs))
    idx = starts[:, None] + np.arange(10)[None, :]
    rec = raw[idx]
    targets = rec[:, 0:4].copy().view("<u4").reshape(E)
    lambdas = rec[:, 4:6].copy().view("<u2").reshape(E)
    dists = rec[:, 6:10].copy().view("<f4").reshape(E)
    return hdr, n, degs, targets, lambdas, dists


PK_MAGIC = b"TSDGPK01"


def pack(tsdg_path: str, out_path: str) -> None:
    """graph.pk: "TSDGPK01" | u64 n | u64 E | u32 lbits | u32 nbytes | u64 fnv of the
    original file | 27-byte header | n x u32 degrees | E x nbytes (target<<lbits|lambda).
    Read by unpack() below and by the C tool tools/prepare_inputs.c."""
    hdr, n, degs, targets, lambdas, _ = _parse(tsdg_path)
    tbits = max(1, int(n - 1).bit_length())
    lbits = max(1, int(lambdas.max()).bit_length()) if lambdas.size else 1
    nbytes = (tbits + lbits + 7) // 8
    v = targets.astype(np.uint64) << np.uint64(lbits) | lambdas.astype(np.uint64)
    packed = v.view(np.uint8).reshape(-1, 8)[:, :nbytes].copy()
    fnv = int(_fnv_file(tsdg_path), 16)
    with open(out_path, "wb") as f:
        f.write(PK_MAGIC)
        f.write(np.array([n, packed.shape[0]], "<u8").tobytes())
        f.write(np.array([lbits, nbytes], "<u4").tobytes())
        f.write(np.array([fnv], "<u8").tobytes())
        f.write(hdr.tobytes())
        f.write(degs.astype("<u4").tobytes())
        f.write(packed.tobytes())


def _read_pk(pack_path: str):
    raw = np.fromfile(pack_path, np.uint8)
    if raw[:8].tobytes() != PK_MAGIC:
        raise RuntimeError(f"{pack_path}: not a graph pack")
    n, E = (int(x) for x in raw[8:24].view("<u8"))
    lbits, nbytes = (int(x) for x in raw[24:32].view("<u4"))
    fnv = int(raw[32:40].view("<u8")[0])
    hdr = raw[40:67].copy()
    degs = raw[67:67 + 4 * n].view("<u4").copy()
    packed = raw[67 + 4 * n:67 + 4 * n + E * nbytes].reshape(E, nbytes)
    return hdr, degs, packed, lbits, fnv


def unpack(pack_path: str, base: np.ndarray, out_path: str) -> None:
    hdr, degs, packed, lbits, fnv = _read_pk(pack_path)
    n = degs.shape[0]
    metric = int(hdr[16])
    E = packed.shape[0]
    full = np.zeros((E, 8), np.uint8)
    full[:, :packed.shape[1]] = packed
    v = full.view(np.uint64).reshape(E)
    targets = (v >> np.uint64(lbits)).astype(np.uint32)
    lambdas = (v & np.uint64((1 << lbits) - 1)).astype(np.uint16)
    offsets = np.zeros(n + 1, np.uint64)
    offsets[1:] = np.cumsum(degs, dtype=np.uint64)
    dists = np.empty(E, np.float32)
    lib = datasets._lib()
    b = np.ascontiguousarray(base, np.float32)
    lib.tsdg_edge_distances(b.ctypes.data_as(ctypes.c_void_p), ctypes.c_uint32(n),
                            ctypes.c_uint32(b.shape[1]), ctypes.c_int(metric),
                            offsets.ctypes.data_as(ctypes.c_void_p),
                            targets.ctypes.data_as(ctypes.c_void_p),
                            dists.ctypes.data_as(ctypes.c_void_p))
    body = np.empty(27 + 4 * n + 10 * E, np.uint8)
    body[:27] = hdr
    node_pos = 27 + 4 * np.arange(n, dtype=np.int64) + 10 * offsets[:-1].astype(np.int64)
    body[node_pos[:, None] + np.arange(4)[None, :]] = degs.astype("<u4").view(np.uint8).reshape(n, 4)
    rec = np.empty((E, 10), np.uint8)
    rec[:, 0:4] = targets.astype("<u4").view(np.uint8).reshape(E, 4)
    rec[:, 4:6] = lambdas.astype("<u2").view(np.uint8).reshape(E, 2)
    rec[:, 6:10] = dists.astype("<f4").view(np.uint8).reshape(E, 4)
    edge_node = np.repeat(np.arange(n, dtype=np.int64), degs)
    edge_pos = node_pos[edge_node] + 4 + 10 * (np.arange(E, dtype=np.int64) - offsets[:-1].astype(np.int64)[edge_node])
    body[edge_pos[:, None] + np.arange(10)[None, :]] = rec
    tmp = f"{out_path}.tmp{os.getpid()}"  # unique per process: ranks may unpack concurrently
    body.tofile(tmp)
    got = int(_fnv_file(tmp), 16)
    if got != fnv:
        os.remove(tmp)
        raise RuntimeError(f"unpacked TSDG differs from the original (fnv {got:016x} != {fnv:016x})")
    os.replace(tmp, out_path)


if __name__ == "__main__":
    name = sys.argv[1]
    d = os.path.join(datasets.DATA_DIR, name)
    pack(os.path.join(d, "graph.tsdg"), os.path.join(d, "graph.pk"))
    print("packed", os.path.getsize(os.path.join(d, "graph.pk")) / 1e6, "MB")
