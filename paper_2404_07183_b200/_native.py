"""ctypes binding of libpcfb200.so (the C ABI declared in include/pcf_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).  There is
no fallback: if the library or a CUDA device is missing, every compute entry point
raises ``BackendUnavailable``.
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
# PCF_LIB_VARIANT=name loads _lib/libpcfb200.<name>.so (tools/build_variant.py: the same
# library with one translation unit rebuilt under extra -D flags, for tuning sweeps)
LIB_PATH = os.path.join(_HERE, "_lib", "libpcfb200.so" if not os.environ.get("PCF_LIB_VARIANT")
                        else f"libpcfb200.{os.environ['PCF_LIB_VARIANT']}.so")

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p
c_i64p = ctypes.POINTER(ctypes.c_int64)
c_i32p = ctypes.POINTER(ctypes.c_int32)
c_dblp = ctypes.POINTER(ctypes.c_double)


class WorkItem(ctypes.Structure):
    _fields_ = [
        ("row0", c_i32),
        ("nrows", c_i32),
        ("col0", c_i32),
        ("col1", c_i32),
        ("logC", c_i32),
        ("log2G", c_i32),
        ("smem_mode", c_i32),
        ("cost_hi", c_i32),
    ]


# name -> (restype, argtypes).  Every symbol in include/pcf_b200.h appears here; the
# CPU test suite checks the two lists agree.
SIGNATURES = {
    "pcf_version": (ctypes.c_char_p, []),
    "pcf_last_error": (ctypes.c_char_p, []),
    "pcf_tile_threads": (c_int, []),
    "pcf_pack_sorted": (c_int, [c_vp, c_vp, c_int, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "pcf_group_offsets": (c_int, [c_vp, c_i64, c_i32, c_vp]),
    "pcf_pack_sorted32": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "pcf_plan_pairwise": (c_int, [c_vp, c_i64, c_i64, c_i64, c_i32, c_i32, c_vp, c_i64, c_i64p,
                                  c_i32p]),
    "pcf_fill_matrix": (
        c_int,
        [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, c_i32, c_i32, c_i32, c_vp, c_int, c_dbl,
         c_int, c_dbl, c_dbl, c_vp, c_int, c_i64, c_vp, c_vp],
    ),
    "pcf_fill_diagonal": (
        c_int, [c_vp, c_vp, c_vp, c_i64, c_int, c_dbl, c_dbl, c_vp, c_int, c_i64, c_vp, c_vp]
    ),
    "pcf_fill_rows": (
        c_int,
        [c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_int, c_dbl, c_int, c_int, c_dbl, c_dbl, c_vp,
         c_int, c_vp, c_vp],
    ),
    "pcf_pair_list": (c_int, [c_vp, c_vp, c_vp, c_i64, c_int, c_dbl, c_dbl, c_dbl, c_vp, c_vp]),
    "pcf_integrate_pair_host": (
        c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_dbl, c_dbl, c_int, c_dbl, c_dblp]
    ),
    "pcf_sweep_cells": (c_int, [c_vp, c_vp, c_i64, c_i64, c_dbl, c_dbl, c_vp, c_i64, c_vp,
                                c_vp]),
    "pcf_fill_block_host": (
        c_int,
        [c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_int, c_dbl, c_int, c_int, c_dbl, c_dbl, c_vp,
         c_i64, c_i64p, c_i64p],
    ),
    "pcf_matrix_host": (
        c_int,
        [c_vp, c_vp, c_int, c_vp, c_i64, c_int, c_dbl, c_int, c_int, c_dbl, c_dbl, c_i32, c_i32,
         c_vp, c_i64, c_i64p, c_i64p, c_vp],
    ),
    "pcf_release_workspace": (None, []),
    "pcf_jit_cubin": (c_int, [ctypes.c_char_p, c_vp, c_i64, c_i64p, ctypes.c_char_p, c_i64]),
    "pcf_jit_load": (c_int, [ctypes.c_char_p, ctypes.POINTER(c_vp), ctypes.c_char_p, c_i64]),
    "pcf_jit_release": (None, [c_vp]),
    "pcf_jit_tiles_cubin": (c_int, [ctypes.c_char_p, c_int, c_i64p, ctypes.c_char_p, c_i64]),
    "pcf_jit_tiles_load": (c_int, [ctypes.c_char_p, c_int, ctypes.POINTER(c_vp), ctypes.c_char_p,
                                   c_i64]),
    "pcf_jit_tiles_release": (None, [c_vp]),
    "pcf_jit_fill_tiles": (
        c_int, [c_vp, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, c_i32, c_vp,
                c_int, c_dbl, c_dbl, c_vp, c_i64, c_vp, c_vp]),
    "pcf_jit_matrix": (
        c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_int, c_dbl, c_dbl, c_vp, c_int, c_i64, c_i64,
                c_i64, c_vp, c_vp]),
    "pcf_jit_pairs": (
        c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_dbl, c_dbl, c_int, c_vp, c_vp, c_vp]),
    "pcf_jit_single": (
        c_int, [c_vp, c_vp, c_vp, c_i64, c_dbl, c_dbl, c_int, c_vp, c_vp, c_vp]),
    "pcf_probe_fp64": (c_int, [c_vp, c_int, c_int, c_vp]),
    "pcf_pow_batch": (c_int, [c_vp, c_vp, c_i64, c_vp, c_vp]),
    "pcf_collection_create": (c_int, [c_vp, c_vp, c_int, c_vp, c_i64, ctypes.POINTER(c_vp)]),
    "pcf_collection_free": (None, [c_vp]),
    "pcf_collection_fill_block": (c_int, [c_vp, c_i64, c_i64, c_int, c_dbl, c_int, c_int, c_dbl,
                                          c_dbl, c_i32, c_vp, c_int, c_i64, c_i64p, c_i64p]),
    "pcf_scan_workspace": (c_int, [c_i64, c_i64p]),
    "pcf_compact": (
        c_int, [c_int, c_vp, c_vp, c_vp, c_int, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_i64,
                c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pcf_tree_level_workspace": (c_int, [c_i64, c_i64p]),
    "pcf_tree_level": (
        c_int, [c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp,
                c_vp, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "pcf_tree_merge_level": (
        c_int, [c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp,
                c_vp, c_vp, c_vp, c_i64, c_vp]),
    "pcf_tree_dup_sample": (c_int, [c_int, c_vp, c_vp, c_i64, c_i32, c_vp, c_vp]),
    "pcf_finalize_workspace": (c_int, [c_i64, c_i64p]),
    "pcf_finalize": (c_int, [c_int, c_int, c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp,
                             c_vp, c_vp, c_vp, c_i64, c_vp]),
    "pcf_tree_merge_levels_workspace": (c_int, [c_i64, c_i64, c_i64p]),
    "pcf_tree_merge_levels": (
        c_int, [c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i32, c_i64,
                c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "pcf_scale_flag": (c_int, [c_int, c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp,
                               c_vp]),
    "pcf_std_flag": (c_int, [c_int, c_int, c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp,
                             c_vp]),
}

_lock = threading.Lock()
_lib = None
_load_error = None


def load(required=True):
    """The loaded CDLL, or raise BackendUnavailable (required=True) / return None."""
    global _lib, _load_error
    with _lock:
        if _lib is None and _load_error is None:
            try:
                lib = ctypes.CDLL(LIB_PATH)
                for name, (res, args) in SIGNATURES.items():
                    fn = getattr(lib, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = lib
            except (OSError, AttributeError) as exc:
                _load_error = f"cannot load {LIB_PATH}: {exc} (run __graft_entry__.build())"
    if _lib is None and required:
        raise errors.BackendUnavailable(_load_error)
    return _lib


def check(rc, what):
    if rc != 0:
        msg = load().pcf_last_error().decode(errors="replace")
        raise RuntimeError(f"{what} failed (code {rc}): {msg}")


def ptr(t):
    """Raw data pointer of a torch tensor or numpy array (None -> NULL)."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return ctypes.c_void_p(t.data_ptr())
    return ctypes.c_void_p(t.ctypes.data)
