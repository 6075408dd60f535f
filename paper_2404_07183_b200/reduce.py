"""Reductions (mean / std) -- device implementation lands with K5 (pcf_reduce.cu)."""

from __future__ import annotations

__all__ = ["reduce_pair", "tree_reduce", "mean", "variance", "std", "mean_many"]


def _todo(*a, **k):
    raise NotImplementedError("device reductions not built yet")


reduce_pair = tree_reduce = mean = variance = std = mean_many = _todo
