"""Fused tree levels (K5w, csrc/pcf_wmerge.cu): k non-compacting merge levels in one pass
must give exactly what the level-by-level path gives (PCF_TREE_FUSE=1), which is itself
pinned to the reference tree (reduce.py:189-217) by test_gpu_reduce.py.  Covers ties
(forced merge mode on grid data), tiles that overflow shared memory (children with very
different time scales), float32, several fibres (mean_many) and the moments tree."""

import operator

import numpy as np
import pytest

from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a GPU")]

import oracle as O  # noqa: E402
import paper_2404_07183_b200 as pb  # noqa: E402
from paper_2404_07183_b200 import datagen as dg  # noqa: E402
from paper_2404_07183_b200.reduce import (DeviceLevel, mean_many, mean_packed,  # noqa: E402
                                          std_many, std_packed)


def both(monkeypatch, fn):
    monkeypatch.setenv("PCF_TREE_FUSE", "1")
    ref = fn()
    monkeypatch.setenv("PCF_TREE_FUSE", "4")
    got = fn()
    return ref, got


def mats_of(level):
    return [f.to_matrix() for f in level.to_pcfs()]


def test_c5_shape_mean_bitwise_and_oracle(monkeypatch):
    _, mats = dg.noisy_trig_matrices((10000,), 100, "sin", 0.1, dg.RngSpec(2404))
    t, v, off = dg.pack_matrices(mats)
    lvl = DeviceLevel.from_packed(t, v, off)
    ref, got = both(monkeypatch, lambda: mats_of(mean_packed(lvl)))
    assert np.array_equal(ref[0], got[0])
    assert np.array_equal(got[0], O.mean(mats))


def test_c5_shape_std_matches_unfused(monkeypatch):
    _, mats = dg.noisy_trig_matrices((2000,), 50, "cos", 0.2, dg.RngSpec(7))
    t, v, off = dg.pack_matrices(mats)
    lvl = DeviceLevel.from_packed(t, v, off)
    ref, got = both(monkeypatch, lambda: mats_of(std_packed(lvl)))
    a, b = ref[0], got[0]
    assert np.array_equal(a[:, 0], b[:, 0])
    assert np.max(np.abs(a[:, 1] - b[:, 1]) / np.maximum(np.abs(a[:, 1]), 1e-300)) < 1e-13


@pytest.mark.parametrize("op", [operator.add, max, min, operator.mul])
def test_forced_merge_with_ties(monkeypatch, op):
    """Grid times: many equal breakpoints across children (zero-width pieces at every
    level); forced non-compacting mode so every level above 0 is fused."""
    monkeypatch.setenv("PCF_TREE_MODE", "merge")
    rng = np.random.default_rng(11)
    fs = []
    for _ in range(300):
        n = int(rng.integers(1, 60))
        tt = np.concatenate(([0.0], np.sort(rng.choice(np.arange(1, 200) / 8.0, n - 1,
                                                        replace=False))))
        vv = np.round(rng.uniform(-2, 2, n), 2) if op is not operator.mul else \
            rng.choice([0.5, 1.0, 2.0, -1.0], n)
        fs.append(pb.make_pcf(np.column_stack((tt, vv))))
    ref, got = both(monkeypatch, lambda: pb.tree_reduce(fs, op).to_matrix())
    assert np.array_equal(ref, got)
    if op is operator.add:
        monkeypatch.setenv("PCF_TREE_FUSE", "4")
        assert np.array_equal(pb.mean(fs).to_matrix(), O.mean([f.to_matrix() for f in fs]))


def test_overflowing_tiles_split_inside_the_cta(monkeypatch):
    """Children with very different time scales: pivots from the largest child leave
    some tiles with far more than the shared-memory capacity of the other children's
    points, which the CTA cuts into sub-windows."""
    monkeypatch.setenv("PCF_TREE_MODE", "merge")
    rng = np.random.default_rng(5)
    mats = []
    for k in range(64):
        n = 3000 if k % 2 else 400
        scale = 1e-3 if k % 4 == 1 else 1e3
        tt = np.concatenate(([0.0], np.sort(rng.uniform(0, scale, n - 1))))
        mats.append(np.column_stack((tt, rng.normal(size=n))))
    fs = [pb.make_pcf(m) for m in mats]
    ref, got = both(monkeypatch, lambda: pb.mean(fs).to_matrix())
    assert np.array_equal(ref, got)
    assert np.array_equal(got, O.mean(mats))
    ref2, got2 = both(monkeypatch, lambda: pb.std(fs).to_matrix())
    assert np.array_equal(ref2[:, 0], got2[:, 0])
    assert np.max(np.abs(ref2[:, 1] - got2[:, 1]) / np.abs(ref2[:, 1])) < 1e-13


def test_float32_and_fibres(monkeypatch):
    monkeypatch.setenv("PCF_TREE_MODE", "merge")
    _, mats = dg.noisy_trig_matrices((700,), 40, "sin", 0.1, dg.RngSpec(3), dtype=np.float32)
    fs = [pb.make_pcf(m) for m in mats]
    ref, got = both(monkeypatch, lambda: pb.mean(fs).to_matrix())
    assert got.dtype == np.float32 and np.array_equal(ref, got)
    fibres = [fs[:1], fs[1:18], fs[18:19 + 300], fs[319:]]
    ref, got = both(monkeypatch, lambda: [m.to_matrix() for m in mean_many(fibres)])
    for a, b in zip(ref, got):
        assert np.array_equal(a, b)
    ref, got = both(monkeypatch, lambda: [m.to_matrix() for m in std_many(fibres[1:])])
    for a, b in zip(ref, got):
        assert np.array_equal(a[:, 0], b[:, 0])
        assert np.max(np.abs(a[:, 1] - b[:, 1]) / np.maximum(np.abs(a[:, 1]), 1e-30)) < 1e-6


def test_thread_tree_kernel_matches(monkeypatch):
    """K5t (PCF_TREE_KERNEL=tree: one thread per tile, a register merge tree) gives the
    same bits as the shared-memory fused kernel and the level-by-level path."""
    _, mats = dg.noisy_trig_matrices((2000,), 60, "sin", 0.1, dg.RngSpec(21))
    fs = [pb.make_pcf(m) for m in mats]
    monkeypatch.setenv("PCF_TREE_FUSE", "1")
    ref = pb.mean(fs).to_matrix()
    monkeypatch.setenv("PCF_TREE_KERNEL", "tree")
    for fz in ("2", "3"):
        monkeypatch.setenv("PCF_TREE_FUSE", fz)
        assert np.array_equal(pb.mean(fs).to_matrix(), ref)
        assert np.array_equal(pb.tree_reduce(fs, max).to_matrix(),
                              pb.tree_reduce(fs[:], max).to_matrix())


@pytest.mark.parametrize("mode", ["auto", "compact", "merge"])
def test_overflow_is_nonfinite_in_every_tree_mode(monkeypatch, mode):
    """A sum that overflows raises NonFinite like reduce_pair does (reduce.py:49-53),
    whether the levels compact, merge one by one or run fused."""
    from paper_2404_07183_b200 import errors

    monkeypatch.setenv("PCF_TREE_MODE", mode)
    rng = np.random.default_rng(2)
    fs = []
    for _ in range(64):
        tt = np.concatenate(([0.0], np.sort(rng.uniform(0, 1, 9))))
        fs.append(pb.make_pcf(np.column_stack((tt, np.full(10, 1.0e307)))))
    with pytest.raises(errors.NonFinite):
        pb.tree_reduce(fs, "add")
    assert np.isfinite(pb.tree_reduce(fs, max).to_matrix()[:, 1]).all()
