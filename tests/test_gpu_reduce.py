"""GPU reductions vs the reference: tree sums and means bit-identical (same tree, same
per-cell arithmetic, same emission rule); std/variance (parallel-moments combination)
within relative 1e-12 pointwise for float64 (1e-5 for float32), compared at the union of
both outputs' breakpoints."""

import math
import operator

import numpy as np
import pytest

from conftest import has_gpu, unpack

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a GPU")]

import oracle as O  # noqa: E402
import paper_2404_07183_b200 as pb  # noqa: E402
from paper_2404_07183_b200 import errors  # noqa: E402


def pcfs(golden, tag, dtype=None):
    return [pb.make_pcf(m, dtype=dtype) for m in unpack(golden, tag)]


def pointwise_rel(a, b, floor=0.0):
    """max relative difference of two PCF matrices at the union of their breakpoints."""
    ts = np.union1d(a[:, 0], b[:, 0])
    ia = np.searchsorted(a[:, 0], ts, side="right") - 1
    ib = np.searchsorted(b[:, 0], ts, side="right") - 1
    va, vb = a[ia, 1].astype(np.float64), b[ib, 1].astype(np.float64)
    return float(np.max(np.abs(va - vb) / np.maximum(np.maximum(np.abs(vb), floor), 1e-300)))


@pytest.mark.parametrize("k", range(5))
def test_tree_sum_and_mean_bitwise(golden, k):
    fs = pcfs(golden, f"red{k}")
    assert np.array_equal(pb.tree_reduce(fs, operator.add).to_matrix(), golden[f"red{k}_sum"])
    assert np.array_equal(pb.mean(fs).to_matrix(), golden[f"red{k}_mean"])


@pytest.mark.parametrize("k", range(5))
def test_std_variance(golden, k):
    fs = pcfs(golden, f"red{k}")
    if f"red{k}_std" not in golden:
        pytest.skip()
    s = pb.std(fs).to_matrix()
    assert pointwise_rel(s, golden[f"red{k}_std"], floor=1e-300) < 1e-12
    s0 = pb.std(fs, ddof=0).to_matrix()
    assert pointwise_rel(s0, golden[f"red{k}_std_ddof0"]) < 1e-12
    assert (s[:, 1] >= 0).all()
    # minimal discretisation
    assert (s[1:, 1] != s[:-1, 1]).all()


def test_guide_reductions(golden):
    g = pcfs(golden, "guide")
    f3, f4 = g[2], g[3]
    assert pb.mean([f3, f4]) == pb.make_pcf([(0, 3), (2, 2.5), (3, 1.5), (5, 1), (6, 0.5), (7, 0)])
    assert pb.reduce_pair(f3, f4, max) == pb.make_pcf([(0, 4), (2, 3), (3, 2), (6, 1), (7, 0)])
    s = pb.std([f3, f4])
    assert pb.evaluate(s, 0.0) == pytest.approx(math.sqrt(2.0), rel=1e-15)
    assert pb.evaluate(pb.std([f3, f4], ddof=-1), 0.0) == pytest.approx(math.sqrt(2 / 3), rel=1e-15)
    assert pb.evaluate(pb.variance([f3, f4]), 0.0) == pytest.approx(2.0, rel=1e-15)
    assert pb.std([f3, f3]) == pb.zero_pcf()
    assert pb.mean([f3, pb.scale(f3, -1)]) == pb.zero_pcf()
    assert pb.mean([f3]) == pb.minimize_discretization(f3)
    with pytest.raises(errors.InsufficientData):
        pb.std([f3])
    with pytest.raises(errors.EmptyCollection):
        pb.mean([])
    with pytest.raises(errors.MixedPrecision):
        pb.reduce_pair(f3, pb.make_pcf(np.array([[0, 1]], dtype=np.float32)), operator.add)


def test_noisy_sin_golden(golden):
    fs = pcfs(golden, "sin64")
    assert np.array_equal(pb.mean(fs).to_matrix(), golden["sin64_mean"])
    assert pointwise_rel(pb.std(fs).to_matrix(), golden["sin64_std"]) < 1e-12
    f32 = [pb.make_pcf(m.astype(np.float32)) for m in unpack(golden, "sin16f32")]
    m = pb.mean(f32).to_matrix()
    assert m.dtype == np.float32 and np.array_equal(m, golden["sin16f32_mean"])
    assert pointwise_rel(pb.std(f32).to_matrix(), golden["sin16f32_std"]) < 1e-5


def test_tree_max_min_equal_sequential_fold():
    rng = np.random.default_rng(3)
    for trial in range(20):
        mats = []
        for _ in range(int(rng.integers(1, 12))):
            n = int(rng.integers(1, 25))
            t = np.concatenate(([0.0], np.sort(rng.choice(np.arange(1, 400) / 40.0, n - 1,
                                                           replace=False))))
            mats.append(np.column_stack((t, np.round(rng.uniform(-5, 5, n), 3))))
        fs = [pb.make_pcf(m) for m in mats]
        for h in (max, min):
            seq = mats[0]
            for m in mats[1:]:
                seq = O.reduce_pair(seq, m, h)
            assert np.array_equal(pb.tree_reduce(fs, h).to_matrix(), O.minimize(seq))


def test_large_mean_matches_oracle_and_std_bruteforce():
    arr = pb.noisy_sin((700,), 60, rng=pb.RngSpec(2404))
    fs = arr.to_list()
    mats = [f.to_matrix() for f in fs]
    m = pb.mean(fs).to_matrix()
    assert np.array_equal(m, O.mean(mats))
    s = pb.std(fs).to_matrix()
    probes = np.random.default_rng(0).uniform(0, 1, 300)
    vals = np.array([[O.evaluate(x, t) for t in probes] for x in mats])
    mu = vals.sum(0) / len(mats)
    sd = np.sqrt(((vals - mu) ** 2).sum(0) / (len(mats) - 1))
    got = np.array([O.evaluate(s, t) for t in probes])
    assert np.max(np.abs(got - sd) / sd) < 1e-12
    assert np.max(np.abs(np.array([O.evaluate(m, t) for t in probes]) - mu)) < 1e-13


def test_mean_along_batched():
    A = pb.zeros((3, 9))
    A[0, :] = pb.noisy_sin((9,), 30, rng=pb.RngSpec(1))
    A[1, :] = pb.noisy_cos((9,), 12, rng=pb.RngSpec(2))
    A[2, :] = pb.noisy_sin((9,), 5, rng=pb.RngSpec(3))
    M = pb.mean_along(A, 1)
    assert tuple(M.shape) == (3,)
    for r in range(3):
        assert M[r] == pb.mean([A[r, j] for j in range(9)])
    M0 = pb.mean_along(A, 0)
    assert tuple(M0.shape) == (9,)
    for c in range(9):
        assert M0[c] == pb.mean([A[r, c] for r in range(3)])


def test_distributed_reductions_single_rank_match(tmp_path):
    """mean_distributed / std_distributed (world 1, gloo) == single-GPU results."""
    import torch
    import torch.distributed as dist

    from paper_2404_07183_b200 import datagen as dg, parallel
    from paper_2404_07183_b200.reduce import DeviceLevel, mean_packed, std_packed

    shape, mats = dg.noisy_trig_matrices((37,), 20, "sin", 0.1, dg.RngSpec(4))
    t, v, off = dg.pack_matrices(mats)
    dist.init_process_group("gloo", init_method=f"file://{tmp_path}/pg", rank=0, world_size=1)
    try:
        m = parallel.mean_distributed(t, v, off, "cuda")
        s = parallel.std_distributed(t, v, off, "cuda")
    finally:
        dist.destroy_process_group()
    lvl = DeviceLevel.from_packed(t, v, off)
    m1, s1 = mean_packed(lvl), std_packed(lvl)
    assert torch.equal(m.t[: m.ntot], m1.t[: m1.ntot]) and torch.equal(m.v[: m.ntot], m1.v[: m1.ntot])
    assert torch.equal(s.v[: s.ntot], s1.v[: s1.ntot])


def test_flag_compact_pair_matches_finalize():
    """The two-call finalisation (pcf_scale_flag + pcf_compact, tiled scan) and the
    one-call pcf_finalize give the same minimised mean."""
    import torch

    from paper_2404_07183_b200 import _native
    from paper_2404_07183_b200.reduce import DeviceLevel, _run_tree

    fs = pb.noisy_sin((300,), 40, rng=pb.RngSpec(6)).to_list()
    lvl, _ = _run_tree(DeviceLevel.from_pcfs(fs), [300], op=0)
    lib = _native.load()
    n, dev = lvl.ntot, lvl.t.device
    sc = torch.tensor([1.0 / 300], dtype=torch.float64, device=dev)
    sv = torch.empty(n, dtype=torch.float64, device=dev)
    flag = torch.empty(n, dtype=torch.int32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    _native.check(lib.pcf_scale_flag(0, _native.ptr(lvl.v), _native.ptr(lvl.t), _native.ptr(lvl.off),
                                     1, _native.ptr(sc), n, _native.ptr(sv), _native.ptr(flag),
                                     _native.ptr(status), None), "flag")
    nb = _native.c_i64(0)
    lib.pcf_scan_workspace(n, _native.ctypes.byref(nb))
    tmp = torch.empty(nb.value, dtype=torch.uint8, device=dev)
    pos = torch.empty(n, dtype=torch.int64, device=dev)
    t_out = torch.empty(n, dtype=torch.float64, device=dev)
    v_out = torch.empty(n, dtype=torch.float64, device=dev)
    off_out = torch.empty(2, dtype=torch.int64, device=dev)
    src = torch.zeros(1, dtype=torch.int64, device=dev)
    _native.check(lib.pcf_compact(0, _native.ptr(lvl.t), _native.ptr(sv), None, 8,
                                  _native.ptr(flag), n, _native.ptr(lvl.off), _native.ptr(src), 1,
                                  _native.ptr(pos), _native.ptr(tmp), tmp.numel(),
                                  _native.ptr(t_out), _native.ptr(v_out), None,
                                  _native.ptr(off_out), None), "compact")
    k = int(off_out[1].item())
    got = np.column_stack((t_out[:k].cpu().numpy(), v_out[:k].cpu().numpy()))
    assert np.array_equal(got, pb.mean(fs).to_matrix())
