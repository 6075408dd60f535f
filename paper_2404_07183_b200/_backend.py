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
        """Device-resident packed collection (see collection.DeviceCollection)."""
        from .collection import DeviceCollection

        return DeviceCollection.from_pcfs(collection)

    def fill_block(self, packed, r0, r1, op, p, apply_root, diag, a, b, out):
        """Rows [r0, r1) of the symmetric matrix into host array `out` (mirrored);
        returns None or the first non-finite (i, j) -- entries after it in the block
        are left untouched, as in the reference."""
        from .engine import decode_err, fill_rows

        M = packed.M
        slab, err = fill_rows(packed, r0, r1, op, p, apply_root, diag, a, b,
                              out_f32=(np.dtype(out.dtype) == np.float32))
        host = slab.cpu().numpy()
        bad = decode_err(err, M)
        for i in range(r0, r1):
            j0 = i if diag else i + 1
            if bad is not None and bad[0] == i:
                row = host[i - r0, j0:bad[1]]
                out[i, j0:bad[1]] = row
                out[j0:bad[1], i] = row
                return bad
            row = host[i - r0, j0:]
            out[i, j0:] = row
            out[j0:, i] = row
        return None

    def __repr__(self):
        return f"<kernel backend: {self.name}>"


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
