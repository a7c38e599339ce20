"""ctypes binding of the C-ABI in include/tsdg_gpu.h (libtsdg_gpu.so).

The library is built in-tree by __graft_entry__.build() into
paper_2204_00824_b200/_lib/.  There is no CPU fallback: if the shared object is
missing or CUDA is unavailable, every search call raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TSDG_LIB") or os.path.join(_HERE, "_lib", "libtsdg_gpu.so")

TSDG_OK, TSDG_EINVAL, TSDG_ERUNTIME, TSDG_ENCCL = 0, 1, 2, 3
MODE_DETERMINISTIC, MODE_FAST = 0, 1


class BfParamsC(ctypes.Structure):
    _fields_ = [("k", ctypes.c_uint32), ("hop_limit", ctypes.c_uint32),
                ("delta", ctypes.c_float), ("m_segments", ctypes.c_uint32),
                ("lambda_cut", ctypes.c_uint32), ("seed", ctypes.c_uint64),
                ("unbounded", ctypes.c_int32)]


class GreedyParamsC(ctypes.Structure):
    _fields_ = [("t0", ctypes.c_uint32), ("hop_limit", ctypes.c_uint32),
                ("lambda_cut", ctypes.c_uint32), ("seed", ctypes.c_uint64)]


class QueryStatsC(ctypes.Structure):
    _fields_ = [("hops", ctypes.c_uint32), ("distance_evals", ctypes.c_uint32),
                ("queue_evictions", ctypes.c_uint32), ("edges_examined", ctypes.c_uint32)]


class GraphHeaderC(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint64), ("num_edges", ctypes.c_uint64), ("k", ctypes.c_uint32),
                ("alpha", ctypes.c_float), ("lambda0", ctypes.c_uint16),
                ("metric", ctypes.c_uint8), ("max_degree", ctypes.c_uint32)]


# name -> (restype, argtypes); every symbol include/tsdg_gpu.h declares.
_VP, _U32, _U64, _I, _F = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_float
SIGNATURES = {
    "tsdg_gpu_last_error": (ctypes.c_char_p, []),
    "tsdg_gpu_abi_version": (_I, []),
    "tsdg_gpu_launch_count": (_U64, []),
    "tsdg_gpu_host_buffer_mapped": (_I, [_VP, _U64]),
    "tsdg_read_tsdg_header": (_I, [ctypes.c_char_p, _VP]),
    "tsdg_read_tsdg": (_I, [ctypes.c_char_p, _VP, _VP, _VP, _VP]),
    "tsdg_gpu_index_create": (_I, [_VP, _U32, _U32, _VP, _VP, _VP, _I, _I, _VP]),
    "tsdg_gpu_index_create_from_file": (_I, [ctypes.c_char_p, _VP, _U32, _U32, _I, _VP]),
    "tsdg_gpu_index_create_from_files": (_I, [ctypes.c_char_p, ctypes.c_char_p, _I, _VP]),
    "tsdg_read_vectors_shape": (_I, [ctypes.c_char_p, _VP, _VP]),
    "tsdg_read_vectors": (_I, [ctypes.c_char_p, _VP, _U32, _U32]),
    "tsdg_gpu_index_destroy": (_I, [_VP]),
    "tsdg_gpu_index_info": (_I, [_VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "tsdg_gpu_deg_cut": (_I, [_VP, _U32, _VP]),
    "tsdg_gpu_search_bestfirst": (_I, [_VP, _VP, _U32, _U64, _VP, _I, _VP, _VP, _VP, _VP]),
    "tsdg_gpu_search_bestfirst_device": (_I, [_VP, _VP, _U32, _U64, _VP, _I, _VP, _VP, _VP,
                                              _VP, _VP]),
    "tsdg_gpu_search_greedy": (_I, [_VP, _VP, _U32, _U32, _VP, _I, _VP, _VP, _VP, _VP]),
    "tsdg_gpu_search_greedy_device": (_I, [_VP, _VP, _U32, _U32, _VP, _I, _VP, _VP, _VP, _VP,
                                           _VP]),
    "tsdg_gpu_greedy_once": (_I, [_VP, _VP, _U32, _VP, _U32, _U32, _VP, _VP, _VP]),
    "tsdg_gpu_merge_shards_device": (_I, [_VP, _VP, _VP, _VP, _U32, _U32, _U32, _VP, _VP, _VP,
                                          _VP]),
    "tsdg_gpu_ground_truth": (_I, [_VP, _U32, _VP, _U32, _U32, _U32, _I, _I, _VP, _VP]),
    "tsdg_gpu_index_ground_truth": (_I, [_VP, _VP, _U32, _U32, _VP, _VP]),
    "tsdg_gpu_brute_force_knn": (_I, [_VP, _U32, _U32, _U32, _I, _I, _VP, _VP, _VP]),
    "tsdg_gpu_nn_descent": (_I, [_VP, _U32, _U32, _U32, _I, _U32, ctypes.c_double, _U64, _I,
                                 _VP, _VP, _VP, _VP]),
    "tsdg_gpu_exact_topk_device": (_I, [_VP, _U32, _U32, _VP, _U32, _U32, _U32, _U32, _I, _I,
                                        _U64, _VP, _VP, _VP]),
    "tsdg_gpu_build": (_I, [_VP, _U32, _U32, _VP, _VP, _U32, _F, ctypes.c_uint16, _U32, _I, _I,
                            _VP, _VP]),
    "tsdg_gpu_graph_info": (_I, [_VP, _VP, _VP, _VP]),
    "tsdg_gpu_graph_copy": (_I, [_VP, _VP, _VP, _VP, _VP]),
    "tsdg_gpu_graph_save": (_I, [_VP, ctypes.c_char_p]),
    "tsdg_gpu_graph_destroy": (_I, [_VP]),
    "tsdg_gpu_multi_create": (_I, [_VP, _U32, _U32, _VP, _VP, _VP, _I, _VP, _I, _VP]),
    "tsdg_gpu_multi_destroy": (_I, [_VP]),
    "tsdg_gpu_multi_search_bestfirst": (_I, [_VP, _VP, _U32, _U64, _VP, _I, _VP, _VP, _VP, _VP]),
    "tsdg_gpu_multi_search_greedy": (_I, [_VP, _VP, _U32, _U32, _VP, _I, _VP, _VP, _VP, _VP]),
    "tsdg_gpu_sharded_create_from_files": (_I, [_VP, _VP, _VP, _VP, _U32, _U32, _VP, _VP]),
    "tsdg_gpu_sharded_destroy": (_I, [_VP]),
    "tsdg_gpu_sharded_search_bestfirst": (_I, [_VP, _VP, _U32, _U64, _VP, _I, _VP, _VP, _VP]),
}

_lib = None


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class TsdgRuntimeError(RuntimeError):
    """std::runtime_error / CUDA failure."""


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: the CUDA extension must be built "
                "(python -c 'import __graft_entry__; __graft_entry__.build()'); "
                "there is no CPU fallback")
        so = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(so, name)
            fn.restype = res
            fn.argtypes = args
        _lib = so
    return _lib


def check(rc: int) -> None:
    if rc == TSDG_OK:
        return
    msg = lib().tsdg_gpu_last_error().decode(errors="replace")
    if rc == TSDG_EINVAL:
        raise InvalidArgument(msg)
    raise TsdgRuntimeError(msg)
