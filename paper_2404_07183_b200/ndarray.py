"""Shaped arrays of PCF handles and the batched mean along one dimension.

Handle bookkeeping only (the reference's pkg/src/pcflib/ndarray.py:47-265 is out of the
hot path); elements are shared references to immutable Pcf objects held in a numpy
object array, so slicing gives views exactly like the reference's PcfView.
``mean_along`` sends every fibre of the chosen dimension to the device reduction in one
batched call (reduce.mean_many) instead of a Python loop over fibres.
"""

from __future__ import annotations

import numpy as np

from . import errors
from .core import Pcf, zero_pcf

__all__ = ["Shape", "PcfArray", "PcfView", "zeros", "mean_along"]


class Shape(tuple):
    def __repr__(self):
        return "Shape(" + ", ".join(str(e) for e in self) + ")"


def _norm_shape(shape):
    if isinstance(shape, (int, np.integer)):
        shape = (int(shape),)
    shape = tuple(int(e) for e in shape)
    if not shape or any(e < 1 for e in shape):
        raise errors.ZeroExtent(f"array extents must be >= 1, got {shape}")
    return shape


def _check_index(spec, extent):
    if isinstance(spec, slice):
        if spec.step is not None and spec.step <= 0:
            raise errors.InvalidStep(f"slice step must be positive, got {spec.step}")
        return spec
    i = int(spec)
    if i < 0 or i >= extent:
        raise errors.OutOfBounds(f"index {i} out of range for extent {extent}")
    return i


class PcfArray:
    """Row-major shaped container of Pcf handles sharing one scalar kind."""

    def __init__(self, elements, shape=None, dtype=None, _store=None):
        if _store is not None:
            self._a = _store
            self.dtype = np.dtype(dtype)
            return
        elems = list(elements)
        if shape is None:
            shape = (len(elems),)
        shape = _norm_shape(shape)
        if int(np.prod(shape)) != len(elems):
            raise errors.ShapeMismatch(f"{len(elems)} elements cannot fill shape {shape}")
        if dtype is None:
            dtype = elems[0].dtype
        dtype = np.dtype(dtype)
        for f in elems:
            if f.dtype != dtype:
                raise errors.MixedPrecision(f"array holds {dtype.name}, got {f.dtype.name}")
        store = np.empty(len(elems), dtype=object)
        store[:] = elems
        self._a = store.reshape(shape)
        self.dtype = dtype

    @property
    def shape(self):
        return Shape(self._a.shape)

    @property
    def ndim(self):
        return self._a.ndim

    def __len__(self):
        return self._a.shape[0]

    def _norm(self, specs):
        if not isinstance(specs, tuple):
            specs = (specs,)
        if len(specs) > self._a.ndim:
            raise errors.BadDimension("too many indices")
        return tuple(_check_index(s, e) for s, e in zip(specs, self._a.shape))

    def __getitem__(self, specs):
        sel = self._a[self._norm(specs)]
        if isinstance(sel, Pcf):
            return sel
        return PcfView(self, sel)

    def get(self, *idx):
        return self._a[tuple(int(i) for i in idx)]

    def __setitem__(self, specs, value):
        key = self._norm(specs)
        target = self._a[key]
        if isinstance(value, Pcf):
            if value.dtype != self.dtype:
                raise errors.MixedPrecision("dtype mismatch")
            if isinstance(target, Pcf):
                self._a[key] = value
            else:
                target[...] = np.full(target.shape, None, dtype=object)
                for ix in np.ndindex(target.shape):
                    target[ix] = value
            return
        src = value._a if isinstance(value, PcfArray) else np.asarray(value, dtype=object)
        if tuple(np.shape(target)) != tuple(src.shape):
            raise errors.ShapeMismatch(f"cannot assign shape {src.shape} to {np.shape(target)}")
        for ix in np.ndindex(src.shape):
            if src[ix].dtype != self.dtype:
                raise errors.MixedPrecision("dtype mismatch")
        target[...] = src

    def to_list(self):
        return list(self._a.reshape(-1))

    def __repr__(self):
        return f"PcfArray(shape={self.shape}, dtype={self.dtype.name})"


class PcfView(PcfArray):
    """Window into a PcfArray; shares its element storage."""

    def __init__(self, parent, store):
        super().__init__(None, dtype=parent.dtype, _store=store)
        self._parent = parent


def zeros(shape, dtype=np.float64) -> PcfArray:
    shape = _norm_shape(shape)
    z = zero_pcf(dtype)
    return PcfArray([z] * int(np.prod(shape)), shape=shape, dtype=dtype)


def _fibres(array, dim):
    dim = int(dim)
    if dim < 0 or dim >= array.ndim:
        raise errors.BadDimension(f"dim {dim} out of range for rank {array.ndim}")
    moved = np.moveaxis(array._a, dim, -1)
    out_shape = moved.shape[:-1] or (1,)
    fibres = [list(moved[ix]) for ix in np.ndindex(moved.shape[:-1])] if moved.ndim > 1 \
        else [list(moved)]
    return fibres, out_shape


def mean_along(array, dim) -> PcfArray:
    """Mean PCF along `dim` (removed); a rank-1 input gives a 1-element array
    (ndarray.py:241-265); every fibre in one batched device tree."""
    from .reduce import mean_many

    fibres, out_shape = _fibres(array, dim)
    return PcfArray(mean_many(fibres), shape=out_shape, dtype=array.dtype)


def std_along(array, dim, ddof=1) -> PcfArray:
    """Pointwise sample std along `dim` (removed), pcflib.std per fibre
    (reduce.py:236-238); every fibre in one batched device moments tree."""
    from .reduce import std_many

    fibres, out_shape = _fibres(array, dim)
    return PcfArray(std_many(fibres, ddof=ddof), shape=out_shape, dtype=array.dtype)
