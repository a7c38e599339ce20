"""Vector-file and direct file->device loading.

CPU: tsdg_read_vectors (C-ABI, host parse) equals the reference's load_vectors
(io.cpp:58-121) on fvecs / bvecs, and every malformed-file case raises with the
reference's exact message.
GPU: GpuIndex.from_files (raw .tsdg + fvecs bytes decoded on the device) is the same
index as GpuIndex(load_tsdg(path), base): identical deterministic search results,
deg_cut and layout; device-detected bad records report the reference's message."""
import os
import struct

import numpy as np
import pytest

from oracle import oracle as O
from paper_2204_00824_b200 import _native
from paper_2204_00824_b200.search import BestFirstParams, GreedyParams, read_vectors

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def write_vecs(path, x, comp=np.float32):
    x = np.asarray(x)
    with open(path, "wb") as f:
        for row in x:
            f.write(struct.pack("<i", row.shape[0]))
            f.write(np.ascontiguousarray(row, comp).tobytes())


def both(ref, path):
    """(ours, reference) as ("ok", array) or ("err", message)."""
    out = []
    for fn in (read_vectors, ref.load_vectors):
        try:
            out.append(("ok", fn(str(path))))
        except Exception as e:  # noqa: BLE001  (comparing messages)
            out.append(("err", str(e)))
    return out


@needs_ref
def test_read_vectors_matches_reference(tmp_path):
    ref = O.Ref()
    rng = np.random.default_rng(3)
    x = rng.standard_normal((37, 13)).astype(np.float32)
    write_vecs(tmp_path / "a.fvecs", x)
    (k1, ours), (k2, theirs) = both(ref, tmp_path / "a.fvecs")
    assert k1 == k2 == "ok"
    np.testing.assert_array_equal(ours, x)
    np.testing.assert_array_equal(ours.view(np.uint32), theirs.view(np.uint32))
    b = rng.integers(0, 256, (21, 7)).astype(np.uint8)
    write_vecs(tmp_path / "b.bvecs", b, np.uint8)
    (k1, ours), (k2, theirs) = both(ref, tmp_path / "b.bvecs")
    assert k1 == k2 == "ok"
    np.testing.assert_array_equal(ours, b.astype(np.float32))
    np.testing.assert_array_equal(ours, theirs)


def _bad_files(tmp_path):
    x = np.arange(5 * 4, dtype=np.float32).reshape(5, 4)
    good = b"".join(struct.pack("<i", 4) + r.tobytes() for r in x)
    rec = 4 + 16
    cases = {
        "empty.fvecs": b"",
        "short_header.fvecs": good + b"\x04\x00",
        "short_body.fvecs": good + struct.pack("<i", 4) + b"\x00" * 7,
        "implausible.fvecs": good[:rec] + struct.pack("<i", (1 << 24) + 1) + good[rec + 4:],
        "invalid.fvecs": struct.pack("<i", 0) + good,
        "negative.fvecs": struct.pack("<i", -3) + good,
        # size stays a multiple of the record size: only a per-record check finds it
        "inconsistent.fvecs": good[:2 * rec] + struct.pack("<i", 3) + good[2 * rec + 4:],
        "nan.fvecs": good[:3 * rec + 12] + struct.pack("<f", float("nan")) + good[3 * rec + 16:],
        "inf.fvecs": good[:rec + 4] + struct.pack("<f", float("inf")) + good[rec + 8:],
        "trunc.bvecs": struct.pack("<i", 3) + b"\x01\x02\x03" + struct.pack("<i", 3) + b"\x01",
    }
    for name, data in cases.items():
        (tmp_path / name).write_bytes(data)
    return list(cases)


@needs_ref
def test_read_vectors_errors_match_reference(tmp_path):
    ref = O.Ref()
    for name in _bad_files(tmp_path):
        (k1, m1), (k2, m2) = both(ref, tmp_path / name)
        assert k1 == k2 == "err", (name, k1, k2)
        assert m1 == m2, name
    (k1, m1), (k2, m2) = both(ref, tmp_path / "missing.fvecs")
    assert k1 == k2 == "err" and m1 == m2


def test_read_vectors_shape_only_reads_first_record(tmp_path):
    x = np.ones((9, 6), np.float32)
    write_vecs(tmp_path / "s.fvecs", x)
    n, d = _native.ctypes.c_uint32(), _native.ctypes.c_uint32()
    lib = _native.lib()
    assert lib.tsdg_read_vectors_shape(str(tmp_path / "s.fvecs").encode(), _native.ctypes.byref(n),
                                       _native.ctypes.byref(d)) == 0
    assert (n.value, d.value) == (9, 6)


# ---- GPU: raw bytes decoded on the device -------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("name", ["lowlid3k", "syn2k"])
def test_index_from_files_equals_array_index(fixtures, golden_meta, name, tmp_path):
    from paper_2204_00824_b200.search import GpuIndex, load_tsdg
    _, base, queries = fixtures(name)
    gpath = os.path.join(GOLDEN, f"{name}.tsdg")
    vpath = str(tmp_path / "base.fvecs")
    write_vecs(vpath, base)
    a = GpuIndex(load_tsdg(gpath), base)
    b = GpuIndex.from_files(gpath, vpath)
    assert (a.n, a.d, a.metric, a.max_degree, a.row_stride, a.adj_stride) == \
           (b.n, b.d, b.metric, b.max_degree, b.row_stride, b.adj_stride)
    for cut in (1, 5, 10):
        np.testing.assert_array_equal(a.deg_cut(cut), b.deg_cut(cut))
    for p in (BestFirstParams(k=10, seed=7), BestFirstParams(k=48, seed=3, m_segments=16)):
        ra, rb = a.search_bestfirst(queries, p), b.search_bestfirst(queries, p)
        np.testing.assert_array_equal(ra.ids, rb.ids)
        np.testing.assert_array_equal(ra.dists.view(np.uint32), rb.dists.view(np.uint32))
        np.testing.assert_array_equal(ra.counts, rb.counts)
    ga = a.search_greedy(queries[:64], 10, GreedyParams(t0=4, seed=5))
    gb = b.search_greedy(queries[:64], 10, GreedyParams(t0=4, seed=5))
    np.testing.assert_array_equal(ga.ids, gb.ids)
    a.close()
    b.close()


@pytest.mark.gpu
def test_index_from_files_bvecs_and_padding(tmp_path, fixtures):
    """A bvecs base with d not a multiple of 4: rows widened and zero padded on the
    device; same results as the array index on the widened floats."""
    from paper_2204_00824_b200.search import GpuIndex, load_tsdg
    g, _, _ = fixtures("lowlid3k")
    rng = np.random.default_rng(11)
    b8 = rng.integers(0, 256, (g.n, 30)).astype(np.uint8)
    vpath = str(tmp_path / "base.bvecs")
    write_vecs(vpath, b8, np.uint8)
    gpath = os.path.join(GOLDEN, "lowlid3k.tsdg")
    q = rng.integers(0, 256, (200, 30)).astype(np.float32)
    a = GpuIndex(load_tsdg(gpath), b8.astype(np.float32))
    b = GpuIndex.from_files(gpath, vpath)
    p = BestFirstParams(k=10, seed=1)
    ra, rb = a.search_bestfirst(q, p), b.search_bestfirst(q, p)
    np.testing.assert_array_equal(ra.ids, rb.ids)
    np.testing.assert_array_equal(ra.dists.view(np.uint32), rb.dists.view(np.uint32))


@pytest.mark.gpu
@needs_ref
def test_index_from_files_errors(tmp_path, fixtures):
    from paper_2204_00824_b200.search import GpuIndex
    ref = O.Ref()
    g, base, _ = fixtures("lowlid3k")
    gpath = os.path.join(GOLDEN, "lowlid3k.tsdg")
    d = base.shape[1]
    rec = 4 + 4 * d
    good = b"".join(struct.pack("<i", d) + r.tobytes() for r in base)
    # bad records deep in the file, size still a multiple of the record size: found by
    # the device decode, reported with the reference's message
    for tag, data in {
        "dim": good[:1234 * rec] + struct.pack("<i", d - 1) + good[1234 * rec + 4:],
        "nan": good[:2000 * rec + 4 + 4 * 17] + struct.pack("<f", float("nan")) +
               good[2000 * rec + 4 + 4 * 18:],
    }.items():
        p = tmp_path / f"{tag}.fvecs"
        p.write_bytes(data)
        with pytest.raises(Exception) as e:
            GpuIndex.from_files(gpath, str(p))
        with pytest.raises(Exception) as e_ref:
            ref.load_vectors(str(p))
        assert str(e.value) == str(e_ref.value), tag
    # node-count mismatch
    p = tmp_path / "short.fvecs"
    p.write_bytes(good[:100 * rec])
    with pytest.raises(_native.InvalidArgument):
        GpuIndex.from_files(gpath, str(p))
    # edge target out of range (patch one target of a mid-file node)
    raw = bytearray(open(gpath, "rb").read())
    off = 4 + 4 + 8 + 1 + 4 + 4 + 2
    for _ in range(g.n // 2):
        off += 4 + 10 * struct.unpack_from("<I", raw, off)[0]
    assert struct.unpack_from("<I", raw, off)[0] > 0
    struct.pack_into("<I", raw, off + 4, g.n + 5)
    bad_g = tmp_path / "bad.tsdg"
    bad_g.write_bytes(bytes(raw))
    p = tmp_path / "base.fvecs"
    p.write_bytes(good)
    with pytest.raises(_native.InvalidArgument, match="out of range"):
        GpuIndex.from_files(str(bad_g), str(p))
    # truncated TSDG (node records run past the end): the host reader's message
    from paper_2204_00824_b200.search import load_tsdg
    cut = tmp_path / "cut.tsdg"
    cut.write_bytes(open(gpath, "rb").read()[:int(os.path.getsize(gpath) * 0.6)])
    with pytest.raises(Exception) as e_host:
        load_tsdg(str(cut))
    with pytest.raises(Exception) as e_dev:
        GpuIndex.from_files(str(cut), str(p))
    assert str(e_dev.value) == str(e_host.value) and "truncated" in str(e_dev.value)


def test_tsdg_node_count_beyond_u32_is_an_error(tmp_path):
    """A .tsdg header whose u64 node count exceeds the u32 id range is reported, not
    narrowed (diversify.cpp:286 narrows it silently)."""
    from paper_2204_00824_b200.search import InvalidArgument, TsdgRuntimeError, load_tsdg
    p = tmp_path / "big.tsdg"
    with open(p, "wb") as f:
        f.write(b"TSDG" + struct.pack("<IQBIfH", 1, (1 << 32) + 5, 0, 8, 1.2, 9))
    with pytest.raises((TsdgRuntimeError, InvalidArgument), match="32-bit id range"):
        load_tsdg(str(p))
