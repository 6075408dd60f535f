"""Seeded synthetic PCF collections.

``synthetic_benchmark`` and ``noisy_sin``/``noisy_cos`` restate the reference generators
(pkg/src/pcflib/datagen.py:23-139) draw for draw -- same PCG64 stream, same call order,
same redraw rules -- so a seed produces bit-identical collections here and in the
reference (pinned by tests/golden).  The ``*_packed`` variants produce the same numbers
straight into the packed SoA layout (tcat, vcat, off) without building per-PCF
objects, which is what the benchmark feeds the engine at 1e5-1e6 PCFs.

``fixed_size_collection`` and ``ecc_like_collection`` are the SURVEY.md section 8
recipes for configs c1/c2 (fixed n) and c4 (heavy-tailed, integer-valued).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import errors
from .core import Pcf

__all__ = [
    "RngSpec",
    "noisy_trig",
    "noisy_sin",
    "noisy_cos",
    "synthetic_benchmark",
    "synthetic_benchmark_packed",
    "fixed_size_collection",
    "ecc_like_collection",
    "pack_matrices",
]


@dataclass(frozen=True)
class RngSpec:
    """(seed, stream) naming one PCG64 stream."""

    seed: int
    stream: int = 0

    def generator(self) -> np.random.Generator:
        seq = np.random.SeedSequence(self.seed, spawn_key=(self.stream,))
        return np.random.Generator(np.random.PCG64(seq))


def _gen(rng) -> np.random.Generator:
    if rng is None:
        return np.random.default_rng()
    if isinstance(rng, np.random.Generator):
        return rng
    if isinstance(rng, RngSpec):
        return rng.generator()
    return RngSpec(int(rng)).generator()


def _sorted_distinct(gen, n, draw):
    """Sorted draws with exact ties re-drawn (never merged) until distinct."""
    x = np.sort(draw(gen, n))
    if n <= 1:
        return x
    while True:
        tied = np.flatnonzero(x[1:] == x[:-1])
        if tied.size == 0:
            return x
        x[tied] = draw(gen, tied.size)
        x = np.sort(x)


def _abs_normal(gen, k):
    return np.abs(gen.normal(0.0, 1.0, k))


def _uniform01(gen, k):
    return gen.uniform(0.0, 1.0, k)


def _benchmark_rows(gen, dtype):
    """One App-A PCF: n ~ U{10..1000}, times scale*|N(0,1)| sorted,
    values N(0,1), final value 0.  Returns the (n, 2) array in `dtype`."""
    n = int(gen.integers(10, 1001))
    s = abs(gen.normal())
    while True:
        t = s * _sorted_distinct(gen, n - 1, _abs_normal)
        if t[0] > 0.0 and bool((t[1:] > t[:-1]).all()):
            break
        s = abs(gen.normal())
    v = gen.normal(0.0, 1.0, n - 1)
    rows = np.empty((n, 2), dtype=np.float64)
    rows[0, 0] = 0.0
    rows[1:, 0] = t
    rows[:-1, 1] = v
    rows[-1, 1] = 0.0
    return rows.astype(dtype)


def _strictly_increasing(t):
    return t.shape[0] < 2 or bool((t[1:] > t[:-1]).all())


def _benchmark_iter(count, rng, dtype):
    if count < 1:
        raise ValueError(f"count must be >= 1, got {count}")
    gen = _gen(rng)
    dtype = np.dtype(dtype)
    for _ in range(count):
        rows = _benchmark_rows(gen, dtype)
        # narrow dtypes can merge two close times; the reference then draws a fresh
        # PCF from the same stream (datagen.py:303-307)
        while not _strictly_increasing(rows[:, 0]):
            rows = _benchmark_rows(gen, dtype)
        yield rows


def synthetic_benchmark(count, rng=None, dtype=np.float64):
    """List of ``count`` App-A benchmark PCFs."""
    return [Pcf._wrap(r) for r in _benchmark_iter(count, rng, dtype)]


def pack_matrices(mats, dtype=None):
    """(n_i, 2) arrays -> reference pack() layout: tcat, vcat, int64 off[M+1]
    (_sweepkern.pyx:72-85)."""
    mats = list(mats)
    if dtype is None:
        dtype = mats[0].dtype
    sizes = np.fromiter((m.shape[0] for m in mats), dtype=np.int64, count=len(mats))
    off = np.zeros(len(mats) + 1, dtype=np.int64)
    np.cumsum(sizes, out=off[1:])
    cat = np.concatenate(mats, axis=0).astype(dtype, copy=False)
    return np.ascontiguousarray(cat[:, 0]), np.ascontiguousarray(cat[:, 1]), off


def synthetic_benchmark_packed(count, rng=None, dtype=np.float64):
    """Same collection as synthetic_benchmark, packed (tcat, vcat, off)."""
    return pack_matrices(list(_benchmark_iter(count, rng, dtype)), np.dtype(dtype))


def _normalize_shape(shape):
    if isinstance(shape, (int, np.integer)):
        shape = (int(shape),)
    shape = tuple(int(e) for e in shape)
    if not shape or any(e < 1 for e in shape):
        raise errors.BadShape(f"bad shape {shape}")
    return shape


def _trig_rows(gen, n_points, g, sigma, dtype):
    while True:
        t = _sorted_distinct(gen, n_points, _uniform01)
        if t[0] != 0.0:
            t = np.concatenate(([0.0], t))
        v = g(2.0 * np.pi * t) + gen.normal(0.0, sigma, t.shape[0])
        rows = np.column_stack((t, v)).astype(dtype)
        if _strictly_increasing(rows[:, 0]):
            return rows


def noisy_trig_matrices(shape, n_points, kind="sin", sigma=0.1, rng=None, dtype=np.float64):
    """Row arrays of noisy sin/cos PCFs (reference datagen.py:57-94)."""
    shape = _normalize_shape(shape)
    if n_points < 1:
        raise ValueError(f"n_points must be >= 1, got {n_points}")
    if sigma < 0:
        raise ValueError(f"sigma must be >= 0, got {sigma}")
    if kind not in ("sin", "cos"):
        raise ValueError(f"kind must be 'sin' or 'cos', got {kind!r}")
    g = np.sin if kind == "sin" else np.cos
    gen = _gen(rng)
    return shape, [_trig_rows(gen, n_points, g, sigma, dtype) for _ in range(math.prod(shape))]


def noisy_trig(shape, n_points, kind="sin", sigma=0.1, rng=None, dtype=np.float64):
    from .ndarray import PcfArray

    shape, mats = noisy_trig_matrices(shape, n_points, kind, sigma, rng, dtype)
    return PcfArray([Pcf._wrap(m) for m in mats], shape=shape, dtype=dtype)


def noisy_sin(shape, n_points, sigma=0.1, rng=None, dtype=np.float64):
    return noisy_trig(shape, n_points, "sin", sigma, rng, dtype)


def noisy_cos(shape, n_points, sigma=0.1, rng=None, dtype=np.float64):
    return noisy_trig(shape, n_points, "cos", sigma, rng, dtype)


def fixed_size_collection(count, n, seed=2404, dtype=np.float64):
    """SURVEY.md section 8 c1/c2 recipe: t = 0 U sort(U(0,1) x (n-1)), v ~ N(0,1),
    v[-1] = 0; a draw whose times collide after rounding to `dtype` is redrawn."""
    gen = np.random.default_rng(seed)
    dtype = np.dtype(dtype)
    mats = []
    while len(mats) < count:
        t = np.sort(gen.uniform(0.0, 1.0, n - 1))
        v = gen.normal(0.0, 1.0, n)
        v[-1] = 0.0
        rows = np.column_stack((np.concatenate(([0.0], t)), v)).astype(dtype)
        if rows[1:, 0].size and not (rows[1, 0] > 0.0):
            continue
        if _strictly_increasing(rows[:, 0]):
            mats.append(rows)
    return mats


def ecc_like_collection(count, seed=2404, nmin_exp=1.0, nmax_exp=4.0, dtype=np.float64):
    """SURVEY.md section 8 c4 recipe (Euler-characteristic-curve-like, heavy-tailed
    sizes): n = floor(10**U(1, 4)), t = 0 U sort(U(0,1)) (n-1 points), values a +-1
    random walk offset by n//4 with final value 1 so every Lp integral converges."""
    gen = np.random.default_rng(seed)
    dtype = np.dtype(dtype)
    mats = []
    while len(mats) < count:
        n = int(math.floor(10.0 ** gen.uniform(nmin_exp, nmax_exp)))
        n = max(n, 2)
        t = np.sort(gen.uniform(0.0, 1.0, n - 1))
        steps = gen.integers(0, 2, n) * 2 - 1
        v = np.cumsum(steps).astype(np.float64) + float(n // 4)
        v[-1] = 1.0
        rows = np.column_stack((np.concatenate(([0.0], t)), v)).astype(dtype)
        if rows[1, 0] > 0.0 and _strictly_increasing(rows[:, 0]):
            mats.append(rows)
    return mats
