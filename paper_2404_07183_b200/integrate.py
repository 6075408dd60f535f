"""Scalar pair integrals: ``lp_distance`` and ``l2_inner_product``.

Mirror of the op-coded path of pkg/src/pcflib/integrate.py:114-143: the same checks in
the same order (mixed precision, bounds, p >= 1), the backend's raw integral (+-inf
sentinel) mapped to DivergentIntegral / NonFinite, then r = raw^(1/p) rounded to the
PCFs' scalar kind.
"""

from __future__ import annotations

import math

import numpy as np

from . import errors
from ._backend import OP_INNER, OP_LP, get_backend

__all__ = ["lp_distance", "l2_inner_product"]

_INF = math.inf


def _round_to_kind(x, dtype):
    return float(np.float32(x)) if dtype == np.float32 else float(x)


def _same_kind(f, g):
    if f.dtype != g.dtype:
        raise errors.MixedPrecision(f"cannot combine {f.dtype.name} with {g.dtype.name}")
    return f.dtype


def _raw(f, g, op, p, a, b):
    _same_kind(f, g)
    a = float(a)
    b = float(b)
    if math.isnan(a) or math.isnan(b) or math.isinf(a) or a < 0.0 or not a < b:
        raise errors.InvalidBounds(f"bounds must satisfy 0 <= a < b, got [{a}, {b})")
    raw = get_backend().integrate_pair(f, g, a, b, op, float(p))
    if math.isinf(raw):
        if b == _INF:
            raise errors.DivergentIntegral("nonzero integrand on the unbounded tail cell")
        raise errors.NonFinite("integral overflowed")
    if math.isnan(raw):
        raise errors.NonFinite("integrand produced NaN")
    return raw


def lp_distance(f, g, p=1.0, a=0.0, b=_INF) -> float:
    """(integral over [a, b) of |f - g|^p)^(1/p), p >= 1."""
    p = float(p)
    if not p >= 1.0:
        raise ValueError(f"p must be >= 1, got {p}")
    raw = _raw(f, g, OP_LP, p, a, b)
    return _round_to_kind(pow(raw, 1.0 / p), _same_kind(f, g))


def l2_inner_product(f, g, a=0.0, b=_INF) -> float:
    """integral over [a, b) of f(t) g(t)."""
    return _round_to_kind(_raw(f, g, OP_INNER, 0.0, a, b), _same_kind(f, g))
