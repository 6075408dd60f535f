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
import os
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


_PROBE = (0.0, 1.0, -1.0, 0.5, 2.5, -2.25, 1e-3, 3.75, 7.0, 1e10, -1e-7, 0.1)


def _probably_symmetric(h):
    """Does h(x, y) == h(y, x) bitwise on a fixed probe set (Python evaluation)?  Only
    then may the tile kernels, which walk a pair in either orientation, run a
    `symmetric=True` integral; otherwise the one-thread path keeps the reference's
    orientation (f = the lower original index, matrix.py:186-193)."""
    try:
        for x in _PROBE:
            for y in _PROBE:
                u, w = float(h(x, y)), float(h(y, x))
                if not (u == w or (u != u and w != w)):
                    return False
                if u == w and u == 0.0 and math.copysign(1.0, u) != math.copysign(1.0, w):
                    return False
    except Exception:
        return False
    return True


def _tiles_eligible(integral):
    return (integral.h is not None and integral.symmetric
            and os.environ.get("PCF_JIT_NO_TILES", "") in ("", "0")
            and _probably_symmetric(integral.h))


def _fill_custom_tiles(coll, integral, out, exact, chunks, between):
    """Symmetric pointwise integrands on the tile kernels (K1 / K1c / K1r / K1g / K1s compiled
    with h, pcf_jit_fill_tiles): strict upper triangle from the collection's work plan
    (exact: one lane per pair, the reference's left-to-right sum), diagonal by
    pcf_jit_pairs on (s, s).  Same return as fill_custom."""
    from .collection import current_stream_handle
    from .engine import mode_runs

    torch = _torch()
    lib = _native.load()
    a, b = _bounds(integral.a, integral.b)
    defs = jit.generate(h=integral.h, r=integral.r)
    mod = jit.JitModule.get(defs)
    tiles = jit.JitTiles.get(defs, coll.dtype == np.float32)
    M = coll.M
    out_f32 = int(out.dtype == torch.float32)
    st = current_stream_handle()
    items_dev, host_items, smem = coll.plan(exact=exact)
    err = torch.full((1,), -1, dtype=torch.int64, device=coll.device)
    counter = torch.zeros(1, dtype=torch.int32, device=coll.device)
    # diagonal: <f, f> entries through the one-thread kernel
    idx = torch.arange(M, dtype=torch.int64, device=coll.device)
    pd = torch.stack((idx, idx), 1).reshape(-1).contiguous()
    dres = torch.empty(M, dtype=torch.float64, device=coll.device)
    dst = torch.empty(M, dtype=torch.int32, device=coll.device)
    _native.check(lib.pcf_jit_pairs(
        mod.handle, _native.ptr(coll.recs), _native.ptr(coll.soff), _native.ptr(pd), M, a, b,
        out_f32, _native.ptr(dres), _native.ptr(dst), st), "pcf_jit_pairs")
    perm = coll.perm.long()
    out[perm, perm] = dres.to(out.dtype)
    segs = []
    for base, end, mode in mode_runs(host_items):
        count = end - base
        k = max(1, min(int(chunks), count))
        bnd = [base + (count * i) // k for i in range(k + 1)]
        segs += [(bnd[i], bnd[i + 1], mode) for i in range(k) if bnd[i + 1] > bnd[i]]
    events = []
    for n, (s0, s1, mode) in enumerate(segs):
        _native.check(lib.pcf_jit_fill_tiles(
            tiles.handle, mode, _native.ptr(coll.tile_recs), _native.ptr(coll.recsg),
            _native.ptr(coll.soff), _native.ptr(coll.goff), _native.ptr(coll.perm), M,
            _native.c_vp(items_dev.data_ptr() + s0 * 32), s1 - s0, smem, _native.ptr(counter),
            int(tiles.has_r), a, b, _native.ptr(out), out.stride(0), _native.ptr(err), st),
            "pcf_jit_fill_tiles")
        if between is not None:
            ev = torch.cuda.Event()
            ev.record()
            events.append(ev)
            if len(events) >= 2:
                events[-2].synchronize()
                if between(n / len(segs)):
                    return None, True
    if between is not None:
        if events:
            events[-1].synchronize()
        between(1.0)
    # first failing entry in row-major (min, max) order: the tile kernels report the
    # key only; its status comes from the one-thread kernel on the same pair
    cand = []
    bad = torch.nonzero(dst).reshape(-1)
    if bad.numel():
        o = perm[bad]
        k = int(torch.min(o).item())
        cand.append((k * M + k, k, k))
    key = int(err.item()) & 0xFFFFFFFFFFFFFFFF
    if key != 2 ** 64 - 1:
        cand.append((key, key // M, key % M))
    if not cand:
        return None, False
    _, i, j = min(cand)
    if i == j:
        stt = int(dst[int(coll.inv[i].item())].item())
    else:
        inv = coll_inv(coll)
        pair = torch.tensor([inv[i], inv[j]], dtype=torch.int64, device=coll.device)
        r1 = torch.empty(1, dtype=torch.float64, device=coll.device)
        s1_ = torch.empty(1, dtype=torch.int32, device=coll.device)
        _native.check(lib.pcf_jit_pairs(
            mod.handle, _native.ptr(coll.recs), _native.ptr(coll.soff), _native.ptr(pair), 1,
            a, b, out_f32, _native.ptr(r1), _native.ptr(s1_), st), "pcf_jit_pairs")
        stt = int(s1_.item()) or 2
    return (stt, i, j), False


def coll_inv(coll):
    inv = np.empty(coll.M, dtype=np.int64)
    inv[coll.perm_host] = np.arange(coll.M)
    return inv


def fill_custom(coll, integral: CombinationIntegral, out, row_chunks=1, between=None,
                exact=True):
    """Custom-integral matrix (MatrixJob with integral=, matrix.py:184-196) into the
    device tensor `out` (original order).  Symmetric integrals: q >= s, mirrored
    (diagonal included); otherwise all M^2 entries.  Returns (err, stopped) where err is
    None or (status, i, j) of the first failing entry in row-major order.

    Symmetric pointwise integrands run on the tile kernels (exact: one lane per pair,
    the reference's cell order; exact=False lets a warp share a long pair); the others,
    time-dependent ones, and h that fail the symmetry probe run one thread per entry."""
    from .collection import current_stream_handle

    if _tiles_eligible(integral):
        return _fill_custom_tiles(coll, integral, out, exact, row_chunks, between)
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
