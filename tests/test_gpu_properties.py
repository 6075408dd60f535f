"""Size-independent properties of the pairwise engine, checked at sizes the CPU oracle
cannot reach quickly ("through size-independent properties the domain
offers"), plus quantised-time collections (coincident breakpoints across PCFs).

* power-of-two scaling of values or times scales every L1 entry by exactly that power
  (every cell product and partial sum scales exactly): bitwise, fast mode, M = 12,000;
* repeatability: two fills are bit-identical (fixed segment order, one writer per entry);
* metric axioms: symmetry, zero diagonal, triangle inequality (1e-12 slack);
* Gram matrices are positive semi-definite (eigenvalues >= -1e-10 * max);
* quantised times: ties inside K1/K1r/K1g walks agree with the C oracle, bounded and not.
"""

import math

import numpy as np
import pytest

from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a GPU")]

import paper_2404_07183_b200 as pb  # noqa: E402
from paper_2404_07183_b200 import datagen as dg  # noqa: E402
from paper_2404_07183_b200.collection import DeviceCollection  # noqa: E402
from paper_2404_07183_b200.engine import decode_err, fill_pairwise  # noqa: E402


def _fill(t, v, off, **kw):
    coll = DeviceCollection(t, v, off)
    out, err, _ = fill_pairwise(coll, kw.pop("op", 0), kw.pop("p", 1.0),
                                kw.pop("root", True), kw.pop("diag", False), **kw)
    assert decode_err(err, coll.M) is None
    return out


def test_power_of_two_scaling_is_exact_at_scale():
    import torch

    t, v, off = dg.synthetic_benchmark_packed(12000, rng=pb.RngSpec(77))
    D = _fill(t, v, off)
    Dv = _fill(t, v * 4.0, off)          # values x 4 -> entries x 4
    Dt = _fill(t * 0.5, v, off)          # times / 2 -> entries / 2
    assert torch.equal(Dv, D * 4.0)
    assert torch.equal(Dt, D * 0.5)
    D2 = _fill(t, v, off)
    assert torch.equal(D, D2)            # repeatable bit for bit
    assert torch.equal(D, D.T) and bool((torch.diagonal(D) == 0).all())


def test_metric_axioms_and_gram_psd():
    import torch

    t, v, off = dg.synthetic_benchmark_packed(500, rng=pb.RngSpec(5))
    D = _fill(t, v, off).cpu().numpy()
    # triangle inequality d(i,k) <= d(i,j) + d(j,k) for every triple (vectorised over k)
    for j in range(0, 500, 25):
        lhs = D
        rhs = D[:, j][:, None] + D[j, :][None, :]
        assert np.all(lhs <= rhs * (1 + 1e-12) + 1e-300)
    K = _fill(t, v, off, op=1, p=0.0, root=False, diag=True).cpu().numpy()
    w = np.linalg.eigvalsh(K)
    assert w.min() >= -1e-10 * w.max()
    assert np.array_equal(K, K.T)
    del torch


def _quantised(count, seed, grid=64, nmax=3000):
    rng = np.random.default_rng(seed)
    mats = []
    for _ in range(count):
        n = int(min(nmax, 2 + rng.integers(0, 10) ** 3 + rng.integers(1, 40)))
        n = min(n, grid * 8)
        t = np.unique(rng.integers(1, grid * 8, n - 1)) / 8.0
        vals = np.round(rng.normal(0, 2, t.size + 1), 2)
        vals[-1] = 0.0
        mats.append(np.column_stack((np.concatenate(([0.0], t)), vals)))
    return mats


@pytest.mark.parametrize("bounds", [(0.0, math.inf), (1.25, 40.0)])
@pytest.mark.parametrize("exact", [False, True])
@pytest.mark.parametrize("budget_kb", [220, 40])
def test_quantised_times_against_oracle(oracle, bounds, exact, budget_kb):
    """Coincident breakpoints everywhere (times on a 1/8 grid): simultaneous jumps in all
    three tile kernels (a small shared-memory budget pushes rows to K1r/K1g)."""
    t, v, off = dg.pack_matrices(_quantised(260, 3 + budget_kb))
    coll = DeviceCollection(t, v, off)
    a, b = bounds
    plan = coll.plan(exact=exact, smem_budget=budget_kb * 1024)
    out, err, _ = fill_pairwise(coll, 0, 2.0, True, False, a=a, b=b, items=plan, exact=exact)
    assert decode_err(err, coll.M) is None
    D = out.cpu().numpy()
    for i in (0, 1, 7, 64, 130, 258):
        ref = oracle.row(t, v, off, i, p=2.0, a=a, b=b)
        rel = np.max(np.abs(D[i, i + 1:] - ref[i + 1:]) / np.maximum(np.abs(ref[i + 1:]), 1e-300))
        assert rel < 1e-12, (i, rel)
    for i in (0, 5, 200):
        ref1 = oracle.row(t, v, off, i, p=1.0, a=a, b=b)
        out1, _, _ = fill_pairwise(coll, 0, 1.0, True, False, a=a, b=b, items=plan, exact=exact)
        got = out1.cpu().numpy()[i, i + 1:]
        if exact:
            assert np.array_equal(got, ref1[i + 1:])
        else:
            assert np.max(np.abs(got - ref1[i + 1:]) / np.maximum(ref1[i + 1:], 1e-300)) < 1e-12
