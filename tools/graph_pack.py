"""Transport encoding of a reference-built TSDG file (saves push bandwidth to the
GPU box; the search never reads this form).  The codec is the C tool
tools/prepare_inputs.c (built as paper_2204_00824_b200/_lib/tsdg_prepare), so the
reference arm of bench.py can rebuild its graph without loading a library of this
repository:

pack:   graph.tsdg -> graph.pk (per node: targets sorted and Rice-coded as gaps,
        lambdas at fixed width; ~20 bits per edge; the fp32 distances are dropped
        because they are exactly recomputable)
unpack: graph.pk + base.fvecs -> graph.tsdg, byte-identical to the original:
        distances recomputed in the reference's sequential fp32 order, edges put back
        in the reference's (lambda, dist, target) order (diversify.cpp:147), and the
        whole file's FNV-1a checked against the checksum recorded at pack time.

python tools/graph_pack.py <dataset>   packs data/<dataset>/graph.tsdg
"""
from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "paper_2204_00824_b200", "_lib", "tsdg_prepare")


def _tool() -> str:
    if not os.path.exists(TOOL):
        sys.path.insert(0, ROOT)
        from paper_2204_00824_b200 import _build
        _build.build_prepare()
    return TOOL


def pack(tsdg_path: str, out_path: str) -> None:
    subprocess.run([_tool(), "pack", tsdg_path, out_path], check=True)


def unpack(pack_path: str, base_fvecs: str, out_path: str, row_offset: int = 0) -> None:
    """Rebuild `out_path` from `pack_path`; the graph's nodes are rows
    [row_offset, row_offset + n) of `base_fvecs`."""
    subprocess.run([_tool(), "unpack", pack_path, base_fvecs, out_path, str(int(row_offset))],
                   check=True)


if __name__ == "__main__":
    name = sys.argv[1]
    d = os.path.join(ROOT, "data", name)
    pack(os.path.join(d, "graph.tsdg"), os.path.join(d, "graph.pk"))
    print("packed", os.path.getsize(os.path.join(d, "graph.pk")) / 1e6, "MB")
