"""Generic combination integrals on the GPU.

API mirror of pkg/src/pcflib/integrate.py:51-203 (``combine_integrate``,
``combine_integrate_timedep``, ``integrate_single``, ``CombinationIntegral``) and of the
custom-integral path of matrix.py (``pairwise``, ``pairwise_job``, MatrixJob with
``integral=``, matrix.py:184-196, 273-283).  The reference calls a Python function per
rectangle; here the function is translated and compiled for the device once (jit.py)
and every entry is one device thread walking the pair in the reference's cell order.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import _native, errors, jit

_INF = math.inf

__all__ = ["CombinationIntegral", "combine_integrate", "combine_integrate_timedep",
           "integrate_single", "integrate_single_many", "combine_integrate_many"]


def _torch():
    import torch

    return torch


def _bounds(a, b):
    a, b = float(a), float(b)
    if math.isnan(a) or math.isnan(b) or math.isinf(a) or a < 0.0 or not a < b:
        raise errors.InvalidBounds(f"bounds must satisfy 0 <= a < b, got [{a}, {b})")
    return a, b


def _kind(pcfs):
    kind = pcfs[0].dtype
    for f in pcfs:
        if f.dtype != kind:
            raise errors.MixedPrecision(f"cannot combine {kind.name} with {f.dtype.name}")
    return kind


@dataclass(frozen=True)
class CombinationIntegral:
    """A functional r(integral over [a, b) of h(f, g)) (integrate.py:175-203).

    Exactly one of ``h`` (pointwise integrand) or ``H`` (antiderivative in t of a
    time-dependent integrand) must be given.  ``symmetric`` declares h(x, y) = h(y, x)
    and lets pairwise-matrix jobs compute one triangle.  The callables are compiled for
    the GPU on first use (jit.py)."""

    h: Optional[Callable] = None
    H: Optional[Callable] = None
    r: Optional[Callable] = None
    a: float = 0.0
    b: float = _INF
    symmetric: bool = False

    def __post_init__(self):
        if (self.h is None) == (self.H is None):
            raise ValueError("exactly one of h and H must be given")

    def module(self):
        return jit.JitModule.get(jit.generate(h=self.h, H=self.H, r=self.r))

    def __call__(self, f, g) -> float:
        return _pairs_values([f, g], [(0, 1)], self.module(), self.a, self.b,
                             timedep=self.H is not None)[0]


def _status_error(st, timedep, single=False):
    if st == 1:
        if single:
            return errors.DivergentIntegral("nonzero integrand on the unbounded tail")
        if timedep:
            return errors.DivergentIntegral(
                "nonzero or non-finite contribution on the unbounded tail")
        return errors.DivergentIntegral("nonzero integrand on the unbounded tail cell")
    return errors.NonFinite("integral is not finite (NaN integrand or overflow)")


def _pairs_values(pcfs, pairs, mod, a, b, timedep=False):
    """Values of explicit (i, j) pairs of `pcfs` under a loaded module; raises the
    reference's error for the first failing pair."""
    from .collection import DeviceCollection, current_stream_handle

    a, b = _bounds(a, b)
    kind = _kind(pcfs)
    torch = _torch()
    lib = _native.load()
    coll = DeviceCollection.from_pcfs(pcfs)
    inv = np.empty(coll.M, dtype=np.int64)
    inv[coll.perm_host] = np.arange(coll.M)
    sp = inv[np.asarray(pairs, dtype=np.int64).reshape(-1, 2)]
    n = sp.shape[0]
    with torch.cuda.device(coll.device):
        pd = torch.from_numpy(np.ascontiguousarray(sp.reshape(-1))).to(coll.device)
        res = torch.empty(n, dtype=torch.float64, device=coll.device)
        st = torch.empty(n, dtype=torch.int32, device=coll.device)
        _native.check(lib.pcf_jit_pairs(
            mod.handle, _native.ptr(coll.recs), _native.ptr(coll.soff), _native.ptr(pd), n,
            a, b, int(kind == np.float32), _native.ptr(res), _native.ptr(st),
            current_stream_handle()), "pcf_jit_pairs")
        vals, sts = res.cpu().numpy(), st.cpu().numpy()
    bad = np.flatnonzero(sts)
    if bad.size:
        raise _status_error(int(sts[bad[0]]), timedep)
    return [float(x) for x in vals]


def combine_integrate(f, g, h, a=0.0, b=_INF) -> float:
    """integral over [a, b) of h(f(t), g(t)) dt (integrate.py:51-78); the tail rule for
    b = inf: h(v_f, v_g) on the last cell must be 0, else DivergentIntegral."""
    _kind([f, g])
    mod = jit.JitModule.get(jit.generate(h=h))
    return _pairs_values([f, g], [(0, 1)], mod, a, b)[0]


def combine_integrate_timedep(f, g, H, a=0.0, b=_INF) -> float:
    """Time-dependent variant (integrate.py:81-111): H is an antiderivative in t of the
    integrand h(v_f, v_g, t); each cell contributes H(., ., r) - H(., ., l)."""
    _kind([f, g])
    mod = jit.JitModule.get(jit.generate(H=H))
    return _pairs_values([f, g], [(0, 1)], mod, a, b, timedep=True)[0]


def combine_integrate_many(pcfs, pairs, h=None, H=None, r=None, a=0.0, b=_INF):
    """Batched combine_integrate over explicit index pairs of one collection (one device
    launch); returns a float64 numpy array (rounded to the collection's kind)."""
    pcfs = list(pcfs)
    if not pcfs:
        raise errors.EmptyCollection("empty collection")
    mod = jit.JitModule.get(jit.generate(h=h, H=H, r=r))
    return np.asarray(_pairs_values(pcfs, pairs, mod, a, b, timedep=H is not None))


def integrate_single_many(pcfs, h, a=0.0, b=_INF):
    """integral over [a, b) of h(f(t)) dt for every PCF of a collection, one device
    thread each (integrate.py:146-171); returns a float64 numpy array."""
    from .collection import DeviceCollection, current_stream_handle

    pcfs = list(pcfs)
    if not pcfs:
        raise errors.EmptyCollection("empty collection")
    a, b = _bounds(a, b)
    kind = _kind(pcfs)
    torch = _torch()
    lib = _native.load()
    mod = jit.JitModule.get(jit.generate(u=h))
    coll = DeviceCollection.from_pcfs(pcfs)
    M = coll.M
    with torch.cuda.device(coll.device):
        res = torch.empty(M, dtype=torch.float64, device=coll.device)
        st = torch.empty(M, dtype=torch.int32, device=coll.device)
        _native.check(lib.pcf_jit_single(
            mod.handle, _native.ptr(coll.recs), _native.ptr(coll.soff), M, a, b,
            int(kind == np.float32), _native.ptr(res), _native.ptr(st),
            current_stream_handle()), "pcf_jit_single")
        vals, sts = res.cpu().numpy(), st.cpu().numpy()
    out = np.empty(M)
    out[coll.perm_host] = vals
    sto = np.empty(M, dtype=np.int32)
    sto[coll.perm_host] = sts
    bad = np.flatnonzero(sto)
    if bad.size:
        raise _status_error(int(sto[bad[0]]), False, single=True)
    return out


def integrate_single(f, h, a=0.0, b=_INF) -> float:
    """integral over [a, b) of h(f(t)) dt; same tail rule as the pairwise integrals."""
    return float(integrate_single_many([f], h, a, b)[0])


def fill_custom(coll, integral: CombinationIntegral, out, row_chunks=1, between=None):
    """Custom-integral matrix (MatrixJob with integral=, matrix.py:184-196) into the
    device tensor `out` (original order).  Symmetric integrals: q >= s, mirrored
    (diagonal included); otherwise all M^2 entries.  Returns (err, stopped) where err is
    None or (status, i, j) of the first failing entry in row-major order."""
    from .collection import current_stream_handle

    torch = _torch()
    lib = _native.load()
    a, b = _bounds(integral.a, integral.b)
    mod = integral.module()
    M = coll.M
    errs = torch.full((2,), -1, dtype=torch.int64, device=coll.device)
    out_f32 = int(out.dtype == torch.float32)
    bounds = np.linspace(0, M, max(1, int(row_chunks)) + 1).astype(np.int64)
    events = []
    for k in range(len(bounds) - 1):
        r0, r1 = int(bounds[k]), int(bounds[k + 1])
        if r1 > r0:
            _native.check(lib.pcf_jit_matrix(
                mod.handle, _native.ptr(coll.recs), _native.ptr(coll.soff),
                _native.ptr(coll.perm), M, int(bool(integral.symmetric)), a, b,
                _native.ptr(out), out_f32, out.stride(0), r0, r1, _native.ptr(errs),
                current_stream_handle()), "pcf_jit_matrix")
        if between is not None:
            ev = torch.cuda.Event()
            ev.record()
            events.append(ev)
            if len(events) >= 2:
                events[-2].synchronize()
                if between(k / (len(bounds) - 1)):
                    return None, True
    if between is not None and events:
        events[-1].synchronize()
        between(1.0)
    e = errs.cpu().numpy().view(np.uint64)
    first = None
    for st, key in ((1, int(e[0])), (2, int(e[1]))):
        if key != 2 ** 64 - 1 and (first is None or key < first[1]):
            first = (st, key)
    if first is None:
        return None, False
    st, key = first
    return (st, key // M, key % M), False
