"""B200 kernel plugin for the reference package (pcflib), as a maintainer would add it.

Drop-in replacement for the reference's compiled kernel module ``pcflib._sweepkern``
(pkg/src/pcflib/_sweepkern.pyx): the same three entry points with the same argument
meaning, return conventions and dtype handling, bound with ctypes to the C ABI of
libpcfb200.so (include/pcf_b200.h).  Install it as ``pcflib/_sweepkern.py`` (or import
it under that name before pcflib) and the reference's own backend selection
(pkg/src/pcflib/_backend.py:15-20,25-53: ``_COMPILED = _Backend("compiled", _sweepkern,
True)``) runs every pairwise matrix and scalar integral on the GPU unchanged:

  integrate_pair(ft, fv, gt, gv, a, b, op, p)  pyx:62-69  -> pcf_integrate_pair_host
  pack(collection)                              pyx:72-85  -> pcf_collection_create (handle)
  fill_block(packed, r0, r1, op, p, apply_root, diag, a, b, out)
                                                pyx:88-121 -> pcf_collection_fill_block

Semantics kept: raw +-inf from integrate_pair on divergence; fill_block returns None or the
block's first non-finite (i, j) in row-major order with later entries untouched; float32
collections accumulate in float64 and round at the store.  The exact plan (one lane per
pair, libm-exact pow) is used, so matrix entries equal integrate_pair bit for bit, as the
reference's tests require (tests/test_matrix.py:41-47, tests/test_backends.py:33-84).

No dependency on the B200 package's Python code: only numpy, ctypes and the .so
(PCF_B200_LIB, else the in-tree build next to this file).
"""

import ctypes
import os

import numpy as np

OP_LP = 0
OP_INNER = 1

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("PCF_B200_LIB") or os.path.join(
    _HERE, "..", "paper_2404_07183_b200", "_lib", "libpcfb200.so")
_lib = ctypes.CDLL(os.path.abspath(_LIB_PATH))
_vp, _i64, _d, _i, _i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int, \
    ctypes.c_int32
_lib.pcf_last_error.restype = ctypes.c_char_p
_lib.pcf_integrate_pair_host.argtypes = [_vp, _vp, _i64, _vp, _vp, _i64, _d, _d, _i, _d,
                                         ctypes.POINTER(_d)]
_lib.pcf_integrate_pair_host.restype = _i
_lib.pcf_collection_create.argtypes = [_vp, _vp, _i, _vp, _i64, ctypes.POINTER(_vp)]
_lib.pcf_collection_create.restype = _i
_lib.pcf_collection_free.argtypes = [_vp]
_lib.pcf_collection_free.restype = None
_lib.pcf_collection_fill_block.argtypes = [_vp, _i64, _i64, _i, _d, _i, _i, _d, _d, _i32, _vp,
                                           _i, _i64, ctypes.POINTER(_i64),
                                           ctypes.POINTER(_i64)]
_lib.pcf_collection_fill_block.restype = _i


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


def _check(rc):
    if rc:
        raise RuntimeError(_lib.pcf_last_error().decode())


def integrate_pair(ft, fv, gt, gv, a, b, op, p):
    """Raw integral over [a, b) (+-inf when the unbounded tail diverges)."""
    f = [np.ascontiguousarray(x, dtype=np.float64) for x in (ft, fv, gt, gv)]
    out = _d()
    _check(_lib.pcf_integrate_pair_host(_p(f[0]), _p(f[1]), f[0].shape[0], _p(f[2]), _p(f[3]),
                                        f[2].shape[0], float(a), float(b), int(op), float(p),
                                        ctypes.byref(out)))
    return out.value


class _Packed:
    """Device-resident, size-sorted collection (freed with the object)."""

    def __init__(self, tcat, vcat, off):
        self._lib = _lib
        self.tcat, self.vcat, self.off = tcat, vcat, off
        self.M = off.shape[0] - 1
        h = _vp()
        _check(_lib.pcf_collection_create(_p(tcat), _p(vcat), int(tcat.dtype == np.float32),
                                          _p(off), self.M, ctypes.byref(h)))
        self.handle = h

    def __del__(self):
        h, self.handle = getattr(self, "handle", None), None
        if h:
            self._lib.pcf_collection_free(h)


def pack(collection):
    """The reference's pack() layout (tcat, vcat, off), uploaded once."""
    coll = list(collection)
    kind = coll[0].dtype
    sizes = np.fromiter((f.size for f in coll), np.int64, len(coll))
    off = np.zeros(len(coll) + 1, np.int64)
    np.cumsum(sizes, out=off[1:])
    cat = np.concatenate([np.asarray(f.to_matrix() if hasattr(f, "to_matrix") else f._mat)
                          for f in coll]).astype(kind, copy=False)
    return _Packed(np.ascontiguousarray(cat[:, 0]), np.ascontiguousarray(cat[:, 1]), off)


def fill_block(packed, r0, r1, op, p, apply_root, diag, a, b, out):
    """Rows [r0, r1) of the symmetric matrix (and their mirrors) into `out`."""
    if not isinstance(packed, _Packed):
        packed = _Packed(*[np.ascontiguousarray(x) for x in packed])
    if not (out.flags.c_contiguous and out.dtype in (np.float32, np.float64)):
        raise ValueError("out must be a C-contiguous float32/float64 matrix")
    ei, ej = _i64(-1), _i64(-1)
    _check(_lib.pcf_collection_fill_block(packed.handle, int(r0), int(r1), int(op), float(p),
                                          int(bool(apply_root)), int(bool(diag)), float(a),
                                          float(b), 0, _p(out), int(out.dtype == np.float32),
                                          out.shape[1], ctypes.byref(ei), ctypes.byref(ej)))
    return None if ei.value < 0 else (int(ei.value), int(ej.value))
