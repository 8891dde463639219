"""ctypes binding of the C-ABI library ``_lib/liblbvh_b200.so``.

This is the only route to the compute path: there is no CPU fallback.  If
the library is missing or no CUDA device is visible, every batch operation
raises immediately.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# LBVH_LIB overrides the library path (A/B builds of kernel variants).
LIB_PATH = os.environ.get("LBVH_LIB") or os.path.join(_HERE, "_lib", "liblbvh_b200.so")

STACK_CAPACITY = 64
FLAG_STACK_EXHAUSTED = 0x01
FLAG_BUFFER_OVERFLOW = 0x02
FLAG_NONFINITE = 0x04
FLAG_INVERTED_BOX = 0x08
FLAG_BAD_RADIUS = 0x10
FLAG_BAD_K = 0x20
FLAG_BAD_TREE = 0x40
NODE_BYTES = 64
BUILD_DEFER_ROWS = 0x1
KNN_SQUARED = 0x1
MAX_ITEMS = (1 << 30) - 1

_lock = threading.Lock()
_lib = None


class LbvhError(RuntimeError):
    """A non-OK return code from the C ABI."""


class CTree(ctypes.Structure):
    """Mirror of ``struct lbvh_tree`` (include/lbvh_b200.h)."""

    _fields_ = [("n", ctypes.c_int64),
                ("node_mins", ctypes.c_void_p), ("node_maxs", ctypes.c_void_p),
                ("left", ctypes.c_void_p), ("right", ctypes.c_void_p),
                ("leaf_obj", ctypes.c_void_p), ("nodes", ctypes.c_void_p),
                ("root_box", ctypes.c_void_p), ("leaf_codes", ctypes.c_void_p),
                ("leaf_dir", ctypes.c_void_p), ("leaf_dir_bits", ctypes.c_int32),
                ("flags", ctypes.c_int32)]

TREE_POINT_LEAVES = 0x1
TREE_CODES30 = 0x2
TREE_BUILT = 0x4
SPILL_CHUNK = 256


_SIGS = {
    "lbvh_strerror": ([ctypes.c_int], ctypes.c_char_p),
    "lbvh_last_cuda_error": ([], ctypes.c_char_p),
    "lbvh_abi_version": ([], ctypes.c_int),
    "lbvh_leaf_directory_bits": ([ctypes.c_int64], ctypes.c_int),
    "lbvh_leaf_directory": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                             ctypes.c_void_p], ctypes.c_int),
    "lbvh_launch_count": ([], ctypes.c_uint64),
    "lbvh_build_workspace_bytes": ([ctypes.c_int64], ctypes.c_size_t),
    "lbvh_sort_workspace_bytes": ([ctypes.c_int64], ctypes.c_size_t),
    "lbvh_topology_workspace_bytes": ([ctypes.c_int64], ctypes.c_size_t),
    "lbvh_query_workspace_bytes": ([ctypes.c_int64], ctypes.c_size_t),
    "lbvh_scan_workspace_bytes": ([ctypes.c_int64], ctypes.c_size_t),
    "lbvh_build": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                    ctypes.c_void_p, ctypes.c_size_t] + [ctypes.c_void_p] * 9
                   + [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                      ctypes.c_void_p], ctypes.c_int),
    "lbvh_finish_rows": ([ctypes.POINTER(CTree), ctypes.c_void_p, ctypes.c_void_p,
                          ctypes.c_void_p], ctypes.c_int),
    "lbvh_morton_codes": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "lbvh_sort_pairs": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                         ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p], ctypes.c_int),
    "lbvh_generate_topology": ([ctypes.c_void_p, ctypes.c_int64] + [ctypes.c_void_p] * 4 +
                               [ctypes.c_size_t, ctypes.c_void_p], ctypes.c_int),
    "lbvh_refit": ([ctypes.c_void_p] * 5 + [ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t,
                                            ctypes.c_void_p], ctypes.c_int),
    "lbvh_pack": ([ctypes.POINTER(CTree)] + [ctypes.c_void_p] * 4, ctypes.c_int),
    "lbvh_unpack_boxes": ([ctypes.POINTER(CTree)] + [ctypes.c_void_p] * 3, ctypes.c_int),
    "lbvh_query_order": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int,
                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                          ctypes.c_void_p], ctypes.c_int),
    "lbvh_check_queries": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                            ctypes.c_void_p], ctypes.c_int),
    "lbvh_spatial_count": ([ctypes.POINTER(CTree), ctypes.c_void_p, ctypes.c_void_p,
                            ctypes.c_float, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                            ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p],
                           ctypes.c_int),
    "lbvh_spatial_fill": ([ctypes.POINTER(CTree), ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.c_float, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                           ctypes.c_void_p], ctypes.c_int),
    "lbvh_exclusive_scan": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                             ctypes.c_size_t, ctypes.c_void_p], ctypes.c_int),
    "lbvh_spatial_1p": ([ctypes.POINTER(CTree), ctypes.c_void_p, ctypes.c_void_p,
                         ctypes.c_float, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                         ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p],
                        ctypes.c_int),
    "lbvh_compact": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                      ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "lbvh_knn_offsets": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                          ctypes.c_size_t, ctypes.c_void_p], ctypes.c_int),
    "lbvh_knn": ([ctypes.POINTER(CTree), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                  ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                  ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t,
                  ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "lbvh_knn_batch_workspace_bytes": ([ctypes.c_int64], ctypes.c_size_t),
    "lbvh_spatial_count_batch_workspace_bytes": ([ctypes.c_int64], ctypes.c_size_t),
    "lbvh_spatial_count_batch": ([ctypes.POINTER(CTree), ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_float, ctypes.c_int64, ctypes.c_int, ctypes.c_int64]
                                 + [ctypes.c_void_p] * 8 + [ctypes.c_int64]
                                 + [ctypes.c_void_p] * 3 + [ctypes.c_size_t]
                                 + [ctypes.c_void_p] * 4, ctypes.c_int),
    "lbvh_spill_copy": ([ctypes.c_void_p, ctypes.c_int64] + [ctypes.c_void_p] * 6
                        + [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "lbvh_knn_batch": ([ctypes.POINTER(CTree), ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                        ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                        ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p],
                       ctypes.c_int),
    "lbvh_knn_kth": ([ctypes.POINTER(CTree), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                      ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                      ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t,
                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "lbvh_knn_workspace_bytes": ([ctypes.c_int64], ctypes.c_size_t),
    "lbvh_spatial_fill_list": ([ctypes.POINTER(CTree), ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_float, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "lbvh_select_overflow": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "lbvh_unpack_knn_keys": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                              ctypes.c_void_p], ctypes.c_int),
    "lbvh_generate_cloud": ([ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_float]
                            + [ctypes.c_uint64] * 4 + [ctypes.c_void_p] * 3, ctypes.c_int),
    "lbvh_rank_forward_mask": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_float, ctypes.c_int64,
                                ctypes.c_void_p, ctypes.c_int, ctypes.c_uint32, ctypes.c_void_p,
                                ctypes.c_void_p], ctypes.c_int),
    "lbvh_knn_finalize": ([ctypes.c_int64, ctypes.c_int] + [ctypes.c_void_p] * 8, ctypes.c_int),
    "lbvh_gather_rows3": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                           ctypes.c_void_p], ctypes.c_int),
    "lbvh_scatter_result_rows": ([ctypes.c_int64, ctypes.c_int] + [ctypes.c_void_p] * 6,
                                 ctypes.c_int),
    "lbvh_morton_codes_f32": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                               ctypes.c_void_p], ctypes.c_int),
    "lbvh_forward_rows": ([ctypes.c_void_p] * 3 + [ctypes.c_int64, ctypes.c_int]
                          + [ctypes.c_void_p] * 4 + [ctypes.c_int, ctypes.c_void_p], ctypes.c_int),
    "lbvh_merge_records": ([ctypes.c_void_p] * 3 + [ctypes.c_int64, ctypes.c_void_p, ctypes.c_int]
                           + [ctypes.c_void_p] * 4 + [ctypes.c_int, ctypes.c_void_p],
                           ctypes.c_int),
    "lbvh_remap_leaves": ([ctypes.POINTER(CTree)] + [ctypes.c_void_p] * 4, ctypes.c_int),
    "lbvh_brute_knn": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                        ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p],
                       ctypes.c_int),
    "lbvh_brute_radius": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.c_float, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
}


def load_library(path: str = LIB_PATH):
    """Load and type the library (no CUDA needed; used by the CPU tests)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                f"CUDA extension {path} is missing -- build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'`; "
                "there is no CPU fallback")
        lib = ctypes.CDLL(path)
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


_CUDA_OK = False


def lib():
    """The library, after asserting a CUDA device is present (checked once:
    this sits on every query call's host path)."""
    global _CUDA_OK
    if _CUDA_OK and _lib is not None:
        return _lib
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1908_11807_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    l = load_library()
    _CUDA_OK = True
    return l


def check(rc: int) -> None:
    if rc != 0:
        l = load_library()
        msg = l.lbvh_strerror(rc).decode()
        if rc == 3:
            msg += f" ({l.lbvh_last_cuda_error().decode()})"
        raise LbvhError(f"liblbvh_b200: {msg}")


def exported_symbols():
    return sorted(_SIGS)
