"""The "cuda" kernel backend: the reference's _Backend protocol on the B200 engine.

Reference boundary: pkg/src/pcflib/_backend.py:25-91 (``_Backend.integrate_pair``,
``pack``, ``fill_block``; ``get_backend``/``set_backend``/``available_backends``;
``MASSPCF_BACKEND``).  Same method names, argument meaning and return conventions
(raw +-inf sentinel from integrate_pair, ``None`` or the first failing ``(i, j)`` from
fill_block, ``out`` mutated in place).  There is exactly one backend and no CPU
fallback: selecting anything else raises.
"""

from __future__ import annotations

import os

import numpy as np

from . import _native, errors

OP_LP = 0
OP_INNER = 1


class _Backend:
    name = "cuda"

    def integrate_pair(self, f, g, a, b, op, p):
        """Raw combination integral of one pair (float64), +-inf on divergence."""
        lib = _native.load()
        from .collection import require_cuda

        require_cuda()
        ft = np.ascontiguousarray(f.times, dtype=np.float64)
        fv = np.ascontiguousarray(f.values, dtype=np.float64)
        gt = np.ascontiguousarray(g.times, dtype=np.float64)
        gv = np.ascontiguousarray(g.values, dtype=np.float64)
        res = _native.c_dbl(0.0)
        import ctypes

        _native.check(lib.pcf_integrate_pair_host(
            _native.ptr(ft), _native.ptr(fv), ft.shape[0], _native.ptr(gt), _native.ptr(gv),
            gt.shape[0], float(a), float(b), int(op), float(p), ctypes.byref(res)),
            "pcf_integrate_pair_host")
        return res.value

    def pack(self, collection):
        """Device-resident, size-sorted copy of the collection (pcf_collection_create):
        the reference's packed tuple (_sweepkern.pack, pyx:72-85) as an opaque handle."""
        return PackedHandle(collection)

    def fill_block(self, packed, r0, r1, op, p, apply_root, diag, a, b, out, exact=True):
        """Rows [r0, r1) of the symmetric matrix into host array `out` (mirrored);
        returns None or the first non-finite (i, j) -- entries after it in the block
        are left untouched, as in the reference (pyx:88-121).  The first block of a job
        computes the whole matrix on the device (tile kernels; exact plan by default, so
        entries equal integrate_pair bit for bit) and caches it on the handle."""
        if not isinstance(packed, PackedHandle):
            packed = PackedHandle(packed)
        return packed.fill_block(r0, r1, op, p, apply_root, diag, a, b, out, exact)

    def __repr__(self):
        return f"<kernel backend: {self.name}>"


class PackedHandle:
    """pcf_collection_create handle for a list of Pcf (or an (tcat, vcat, off) tuple in
    the reference pack() layout); freed with the object."""

    def __init__(self, collection):
        import ctypes

        from .collection import require_cuda
        from .datagen import pack_matrices

        require_cuda()
        self._lib = _native.load()
        self._h = None
        if isinstance(collection, tuple) and len(collection) == 3:
            tcat, vcat, off = collection
        else:
            coll = list(collection)
            if not coll:
                raise errors.EmptyCollection("empty collection")
            kind = coll[0].dtype
            if any(f.dtype != kind for f in coll):
                raise errors.MixedPrecision("collection mixes 32- and 64-bit PCFs")
            tcat, vcat, off = pack_matrices([f.to_matrix() for f in coll], kind)
        self.tcat = np.ascontiguousarray(tcat)
        self.vcat = np.ascontiguousarray(vcat, dtype=self.tcat.dtype)
        self.off = np.ascontiguousarray(off, dtype=np.int64)
        self.M = int(self.off.shape[0] - 1)
        h = ctypes.c_void_p()
        _native.check(self._lib.pcf_collection_create(
            _native.ptr(self.tcat), _native.ptr(self.vcat), int(self.tcat.dtype == np.float32),
            _native.ptr(self.off), self.M, ctypes.byref(h)), "pcf_collection_create")
        self._h = h

    def fill_block(self, r0, r1, op, p, apply_root, diag, a, b, out, exact=True):
        import ctypes

        if not (isinstance(out, np.ndarray) and out.ndim == 2 and out.flags.c_contiguous and
                out.dtype in (np.float32, np.float64) and out.shape[0] >= self.M and
                out.shape[1] >= self.M):
            raise ValueError("out must be a C-contiguous float32/float64 M x M array")
        ei, ej = ctypes.c_int64(-1), ctypes.c_int64(-1)
        _native.check(self._lib.pcf_collection_fill_block(
            self._h, int(r0), int(r1), int(op), float(p), int(bool(apply_root)),
            int(bool(diag)), float(a), float(b), 0 if exact else 6, _native.ptr(out),
            int(out.dtype == np.float32), out.shape[1], ctypes.byref(ei), ctypes.byref(ej)),
            "pcf_collection_fill_block")
        return None if ei.value < 0 else (int(ei.value), int(ej.value))

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h is not None and getattr(self, "_lib", None) is not None:
            self._lib.pcf_collection_free(h)


_CUDA = _Backend()


def _initial():
    choice = os.environ.get("MASSPCF_BACKEND", "").strip().lower()
    if choice not in ("", "cuda"):
        # the reference's 'compiled'/'python' CPU kernels do not exist here
        raise errors.BackendUnavailable(
            f"MASSPCF_BACKEND={choice!r}: only the 'cuda' backend exists (no CPU fallback)")
    return _CUDA


_active = _initial()


def get_backend():
    return _active


def set_backend(name):
    if name == "cuda":
        return _CUDA
    if name in ("compiled", "python"):
        raise errors.BackendUnavailable(f"backend {name!r} is not part of the B200 engine")
    raise ValueError(f"unknown backend {name!r}")


def available_backends():
    return ["cuda"]
