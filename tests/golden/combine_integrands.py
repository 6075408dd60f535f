"""Integrands shared by the golden generator (run against the reference pcflib) and the
GPU tests (run through the device JIT): the same Python source on both sides.

Each case: name -> (kind, callables, symmetric, bounds, exact) where kind is "h" (pointwise
h(x, y)), "H" (antiderivative H(x, y, t)) or "u" (integrate_single h(v)), and `exact`
says whether the device result must be bit-identical (IEEE + - * / abs min max sqrt
only) or within 1e-12 relative (transcendentals: CUDA libdevice vs glibc).
"""

import math

import numpy as np

W = 0.75  # a closure constant, inlined exactly


def absdiff(x, y):
    return abs(x - y)


def prod(x, y):
    return x * y


def weighted(x, y):
    d = x - W * y
    return d * d


def cond(x, y):
    return x * y if x > y else 0.5 * (x + y)


def minmax(x, y):
    return max(x, y) - min(x, y) + 0.0 * (x or y)


def asym(x, y):
    return x - 2.0 * y


def expdecay(x, y, t):
    return (y - x) * math.exp(-t)


def linear_t(x, y, t):
    return x * y * t


def square(v):
    return v * v


def softabs(v):
    return np.sqrt(v * v + 1.0) - 1.0


def sqdiff(x, y):
    return (x - y) ** 2


CASES = {
    "absdiff": ("h", dict(h=absdiff), True, (0.0, math.inf), True),
    "prod": ("h", dict(h=prod), True, (0.0, math.inf), True),
    "weighted": ("h", dict(h=weighted), False, (0.0, math.inf), True),
    "cond": ("h", dict(h=cond), False, (0.5, 7.25), True),
    "minmax": ("h", dict(h=minmax), True, (0.0, math.inf), True),
    "asym": ("h", dict(h=asym), False, (0.0, math.inf), True),
    "sqdiff_root": ("h", dict(h=sqdiff, r=math.sqrt), True, (0.0, math.inf), False),
    "expdecay": ("H", dict(H=expdecay), False, (0.0, math.inf), False),
    "linear_t": ("H", dict(H=linear_t), True, (0.25, 6.0), True),
    "square": ("u", dict(h=square), None, (0.0, math.inf), True),
    "softabs": ("u", dict(h=softabs), None, (0.5, 7.25), True),
}
