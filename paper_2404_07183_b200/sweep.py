"""Implicit common-grid sweeps (API mirror of pkg/src/pcflib/sweep.py).

``iterate_rectangles`` visits the cells of the minimal common refinement of two PCFs on
[a, b), ``iterate_segments`` the constant pieces of one PCF.  The cells are enumerated on
the device (``pcf_sweep_cells``, the same cursor walk as every integral kernel) and the
Python callback is invoked once per cell on the host, in time order -- the callback
itself is arbitrary Python and cannot run on the GPU.
"""

from __future__ import annotations

import math
from typing import Callable, NamedTuple

import numpy as np

from . import _native, errors

__all__ = ["Rectangle", "Segment", "iterate_rectangles", "iterate_segments", "rectangles",
           "segments"]

_INF = math.inf


class Rectangle(NamedTuple):
    """One cell (l, r, v_f, v_g) of the implicit common grid; r may be +inf."""

    l: float  # noqa: E741
    r: float
    v_f: float
    v_g: float


class Segment(NamedTuple):
    """One constant piece (l, r, v) of a single PCF clipped to bounds."""

    l: float  # noqa: E741
    r: float
    v: float


def _check_bounds(a, b):
    a, b = float(a), float(b)
    if math.isnan(a) or math.isnan(b) or math.isinf(a):
        raise errors.InvalidBounds(f"bad integration bounds [{a}, {b})")
    if a < 0.0 or not a < b:
        raise errors.InvalidBounds(f"bounds must satisfy 0 <= a < b, got [{a}, {b})")
    return a, b


def _cells(pcfs, a, b):
    import torch

    from .collection import DeviceCollection, current_stream_handle

    lib = _native.load()
    coll = DeviceCollection.from_pcfs(pcfs)
    inv = np.empty(coll.M, dtype=np.int64)
    inv[coll.perm_host] = np.arange(coll.M)
    s = int(inv[0])
    q = int(inv[1]) if len(pcfs) > 1 else -1
    cap = int(coll.n_points) + 1
    with torch.cuda.device(coll.device):
        cells = torch.empty(4 * cap, dtype=torch.float64, device=coll.device)
        cnt = torch.zeros(1, dtype=torch.int64, device=coll.device)
        _native.check(lib.pcf_sweep_cells(
            _native.ptr(coll.recs), _native.ptr(coll.soff), s, q, a, b, _native.ptr(cells), cap,
            _native.ptr(cnt), current_stream_handle()), "pcf_sweep_cells")
        n = int(cnt.item())
        return cells[: 4 * n].view(n, 4).cpu().numpy()


def rectangles(f, g, a=0.0, b=_INF) -> np.ndarray:
    """The cells of f and g on [a, b) as an (n, 4) float64 array (l, r, v_f, v_g)."""
    a, b = _check_bounds(a, b)
    if f.dtype != g.dtype:
        raise errors.MixedPrecision(f"cannot sweep {f.dtype.name} against {g.dtype.name}")
    return _cells([f, g], a, b)


def segments(f, a=0.0, b=_INF) -> np.ndarray:
    """The pieces of f on [a, b) as an (n, 3) float64 array (l, r, v)."""
    a, b = _check_bounds(a, b)
    return _cells([f], a, b)[:, :3]


def iterate_rectangles(f, g, a, b, visit: Callable[[Rectangle], None]):
    """Invoke ``visit`` once per cell of the minimal common refinement of f and g on
    [a, b), in increasing time order (sweep.py:67-100)."""
    for row in rectangles(f, g, a, b).tolist():
        visit(Rectangle(*row))


def iterate_segments(f, a, b, visit: Callable[[Segment], None]):
    """Invoke ``visit`` once per constant piece of f intersected with [a, b)
    (sweep.py:103-116)."""
    for row in segments(f, a, b).tolist():
        visit(Segment(*row))
