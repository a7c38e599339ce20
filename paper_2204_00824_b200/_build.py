"""In-tree build of every native artefact (called by __graft_entry__.build()).

  _lib/libtsdg_gpu.so      CUDA kernels + C-ABI (nvcc, sm_100a only)
  _lib/libtsdg_datagen.so  synthetic input generators (gcc)
  oracle/libtsdg_oracle.so CPU oracle restatement (test infrastructure)
  oracle/_ref/*            the reference compiled from /root/reference when present
"""
from __future__ import annotations

import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "_lib")
CSRC = os.path.join(HERE, "csrc")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _run(cmd, cwd=ROOT):
    print("[build]", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=cwd)


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


GPU_SRCS = ("tsdg_gpu.cu", "bf_fast.cu", "nndescent.cu", "tsdg_io.cpp")


def _build_so(out: str, extra: list, force: bool) -> str:
    """Compile every translation unit to an object in parallel, then link."""
    os.makedirs(LIB, exist_ok=True)
    srcs = [os.path.join(CSRC, f) for f in GPU_SRCS]
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    deps.append(os.path.join(ROOT, "include", "tsdg_gpu.h"))
    if not (force or _stale(out, deps)):
        return out
    objdir = os.path.join(LIB, "obj")
    os.makedirs(objdir, exist_ok=True)
    tag = os.path.splitext(os.path.basename(out))[0]
    objs, procs = [], []
    for src in srcs:
        obj = os.path.join(objdir, f"{tag}.{os.path.basename(src)}.o")
        cmd = [NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", *extra, "-Xcompiler", "-fPIC,-O2",
               "-c", "-o", obj, src]
        print("[build]", " ".join(cmd), flush=True)
        procs.append(subprocess.Popen(cmd, cwd=ROOT))
        objs.append(obj)
    if any(p.wait() != 0 for p in procs):
        raise RuntimeError(f"nvcc failed building {out}")
    _run([NVCC, *ARCH, "-shared", "-o", out, *objs])
    return out


def build_gpu(force: bool = False) -> str:
    return _build_so(os.path.join(LIB, "libtsdg_gpu.so"), [], force)


def build_gpu_phases(force: bool = False) -> str:
    """Development variant with per-phase clock64 counters (-DTSDG_PHASES)."""
    return _build_so(os.path.join(LIB, "libtsdg_gpu_phases.so"), ["-DTSDG_PHASES"], force)


def build_datagen(force: bool = False) -> str:
    os.makedirs(LIB, exist_ok=True)
    out = os.path.join(LIB, "libtsdg_datagen.so")
    src = os.path.join(ROOT, "tools", "datagen.c")
    if force or _stale(out, [src]):
        _run(["gcc", "-std=c11", "-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
              "-o", out, src, "-lm"])
    return out


def build_prepare(force: bool = False) -> str:
    """tools/prepare_inputs.c + datagen.c -> _lib/tsdg_prepare (an executable: the
    reference arm of bench.py prepares its input files without loading a library of
    this repository into its process)."""
    os.makedirs(LIB, exist_ok=True)
    out = os.path.join(LIB, "tsdg_prepare")
    srcs = [os.path.join(ROOT, "tools", f) for f in ("prepare_inputs.c", "datagen.c")]
    if force or _stale(out, srcs):
        _run(["gcc", "-std=c11", "-D_DEFAULT_SOURCE", "-O2", "-fopenmp", "-ffp-contract=off",
              "-o", out, *srcs, "-lm"])
    return out


def build_oracle() -> None:
    _run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"])
    if os.path.isdir("/root/reference/proj/src"):
        _run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "oracle"), "ref"])


def build_cpp_tests() -> None:
    """C++ drop-in parity binary (needs the reference headers + oracle/_ref objects)."""
    if os.path.isdir("/root/reference/proj/include") and os.path.isdir(os.path.join(ROOT, "oracle", "_ref")):
        _run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")])


def build_all(force: bool = False) -> None:
    build_datagen(force)
    build_prepare(force)
    build_oracle()
    build_gpu(force)
    build_gpu_phases(force)
    build_cpp_tests()
