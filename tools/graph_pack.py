"""Transport encoding of a reference-built TSDG file (saves push bandwidth to the
GPU box; the search never reads this form).

pack:   graph.tsdg -> graph.pack.npz  (header fields, degrees, and per edge the
        target and lambda packed into ceil((bits(n)+bits(lambda0))/8) bytes; the
        fp32 edge distances are dropped because they are exactly recomputable)
unpack: graph.pack.npz + base vectors -> graph.tsdg, byte-identical to the
        original: distances recomputed in the reference's sequential fp32 order
        (tools/datagen.c tsdg_edge_distances), then the whole file's FNV-1a is
        checked against the checksum of the original recorded at pack time.
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


def pack(tsdg_path: str, out_path: str) -> None:
    hdr, n, degs, targets, lambdas, _ = _parse(tsdg_path)
    tbits = max(1, int(n - 1).bit_length())
    lbits = max(1, int(lambdas.max()).bit_length()) if lambdas.size else 1
    nbytes = (tbits + lbits + 7) // 8
    v = targets.astype(np.uint64) << np.uint64(lbits) | lambdas.astype(np.uint64)
    packed = v.view(np.uint8).reshape(-1, 8)[:, :nbytes].copy()
    np.savez(out_path, header=hdr, degrees=degs, packed=packed,
             lbits=np.array([lbits]), fnv=np.array([_fnv_file(tsdg_path)]))


def unpack(pack_path: str, base: np.ndarray, out_path: str) -> None:
    z = np.load(pack_path)
    hdr, degs, packed, lbits = z["header"], z["degrees"], z["packed"], int(z["lbits"][0])
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
    got = _fnv_file(tmp)
    want = str(z["fnv"][0])
    if got != want:
        os.remove(tmp)
        raise RuntimeError(f"unpacked TSDG differs from the original (fnv {got} != {want})")
    os.replace(tmp, out_path)


if __name__ == "__main__":
    name = sys.argv[1]
    d = os.path.join(datasets.DATA_DIR, name)
    pack(os.path.join(d, "graph.tsdg"), os.path.join(d, "graph.pack.npz"))
    print("packed", os.path.getsize(os.path.join(d, "graph.pack.npz")) / 1e6, "MB")
