"""User integrands on the tile kernels (pcf_jit_fill_tiles: K1 / K1c / K1r / K1g / K1s compiled
by NVRTC with h and r in place of |x - y|^p and the p-th root).

The one-thread-per-entry kernel (pcf_jit_matrix, bit-identical to the reference's cell
walk, tests/test_gpu_combine.py) is the checker here: exact mode must reproduce it
bitwise (one lane per pair sums the cells left to right with --fmad=false), the
warp-split plan within relative 1e-12 (float64) / the float32 rounding of it.
"""

import math

import numpy as np
import pytest

from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a GPU")]

import paper_2404_07183_b200 as pb  # noqa: E402
from paper_2404_07183_b200 import datagen as dg  # noqa: E402
from paper_2404_07183_b200 import errors  # noqa: E402

TOL64 = 1e-12


def collection(f32=False, n=300):
    t, v, off = dg.pack_matrices(dg.ecc_like_collection(n, nmax_exp=3.7))
    dt = np.float32 if f32 else np.float64
    out = []
    for i in range(off.shape[0] - 1):
        m = np.column_stack((t[off[i]:off[i + 1]], v[off[i]:off[i + 1]])).astype(dt)
        keep = np.concatenate(([True], m[1:, 0] > m[:-1, 0]))  # float32 rounding merges times
        out.append(pb.make_pcf(m[keep], dtype=dt))
    return out


def sq_diff(x, y):
    return (x - y) * (x - y)


def mixed(x, y):
    return abs(x - y) * (1.0 + x * y) + (x - y) * (x - y) * 0.25


def one_thread(monkeypatch, fs, ci):
    with monkeypatch.context() as m:
        m.setenv("PCF_JIT_NO_TILES", "1")
        return np.asarray(pb.pairwise(fs, ci))


def rel(x, ref):
    x, ref = np.asarray(x, np.float64), np.asarray(ref, np.float64)
    return float(np.max(np.abs(x - ref) / np.maximum(np.abs(ref), 1e-300)))


def test_plan_uses_every_tile_kernel():
    from paper_2404_07183_b200.collection import DeviceCollection

    coll = DeviceCollection.from_pcfs(collection())
    for exact in (False, True):
        modes = set(coll.plan(exact=exact)[1][:, 6].tolist())
        assert {1, 2, 3} <= modes, modes


@pytest.mark.parametrize("f32", [False, True])
@pytest.mark.parametrize("bounds", [(0.0, math.inf), (0.2, 0.85)])
@pytest.mark.parametrize("case", ["l1", "sq_sqrt", "mixed"])
def test_tiles_match_one_thread_kernel(monkeypatch, f32, bounds, case):
    fs = collection(f32)
    a, b = bounds
    h, r = {"l1": (lambda x, y: abs(x - y), None), "sq_sqrt": (sq_diff, math.sqrt),
            "mixed": (mixed, None)}[case]
    ci = pb.CombinationIntegral(h=h, r=r, a=a, b=b, symmetric=True)
    ref = one_thread(monkeypatch, fs, ci)
    D = np.asarray(pb.pairwise(fs, ci))  # exact by default
    assert D.dtype == ref.dtype
    assert np.array_equal(D, ref), np.max(np.abs(D - ref))
    F = np.asarray(pb.pairwise(fs, ci, exact=False))
    assert np.array_equal(F, F.T)
    assert np.array_equal(np.diag(F), np.diag(ref))
    if f32:
        assert rel(F, ref) < 2e-6
    else:
        assert rel(F, ref) < TOL64


def test_exact_l1_equals_builtin_pdist():
    fs = collection()
    D = np.asarray(pb.pairwise(fs, pb.CombinationIntegral(h=lambda x, y: abs(x - y),
                                                          symmetric=True)))
    P = np.asarray(pb.pdist(fs, p=1.0, exact=True))
    off = ~np.eye(len(fs), dtype=bool)
    assert np.array_equal(D[off], P[off])


def test_asymmetric_h_declared_symmetric_keeps_reference_orientation(monkeypatch):
    """The reference trusts `symmetric` and computes entry (i, j) with f = f_min(i, j);
    an h that fails the symmetry probe stays on the one-thread kernel, which does too."""
    fs = collection(n=60)
    ci = pb.CombinationIntegral(h=lambda x, y: x - 0.5 * y, a=0.0, b=1.0, symmetric=True)
    assert np.array_equal(np.asarray(pb.pairwise(fs, ci)), one_thread(monkeypatch, fs, ci))


def test_tile_path_errors(monkeypatch):
    """First failing entry in row-major (min, max) order and its class, as the
    one-thread kernel reports it: a divergent off-diagonal pair and a NaN tail."""
    rng = np.random.default_rng(7)
    fs = []
    for i in range(40):
        n = int(rng.integers(2, 40))
        t = np.concatenate(([0.0], np.sort(rng.random(n - 1))))
        v = rng.standard_normal(n)
        v[-1] = 0.0
        fs.append(pb.make_pcf(np.column_stack((t, v))))
    m = fs[23].to_matrix().copy()
    m[-1, 1] = 2.0
    fs[23] = pb.make_pcf(m)
    m = fs[31].to_matrix().copy()
    m[-1, 1] = 3.0
    fs[31] = pb.make_pcf(m)
    prod = pb.CombinationIntegral(h=lambda x, y: x * y, symmetric=True)
    with pytest.raises(errors.DivergentIntegral) as info:
        pb.pairwise(fs, prod)
    assert info.value.pair == (23, 23)  # the diagonal comes first in row-major order

    def cross(x, y):
        return x * y * (x - y) * (x - y)

    ci = pb.CombinationIntegral(h=cross, symmetric=True)
    with pytest.raises(errors.DivergentIntegral) as info:
        pb.pairwise(fs, ci)
    with pytest.raises(errors.DivergentIntegral) as info2:
        one_thread(monkeypatch, fs, ci)
    assert info.value.pair == info2.value.pair == (23, 31)

    nan_ci = pb.CombinationIntegral(h=lambda x, y: (x * y) / (x * y), symmetric=True)
    with pytest.raises(errors.NonFinite) as info:
        pb.pairwise(fs, nan_ci)
    with pytest.raises(errors.NonFinite) as info2:
        one_thread(monkeypatch, fs, nan_ci)
    assert info.value.pair == info2.value.pair


def test_user_h_not_evaluated_on_tie_cells(monkeypatch):
    """Simultaneous jumps: the tile walk takes them as two steps with a zero-width cell
    between, whose value pair ((5, 2) or (1, 7) here) the reference never evaluates; a
    user h that is infinite there must not leak into the sum."""
    f = pb.make_pcf(np.array([[0.0, 1.0], [1.0, 5.0], [2.0, 0.0]]))
    g = pb.make_pcf(np.array([[0.0, 2.0], [1.0, 7.0], [2.0, 0.0]]))

    def h(x, y):
        return 1.0 / ((x * y - 10.0) * (x * y - 7.0))

    ci = pb.CombinationIntegral(h=h, a=0.0, b=3.0, symmetric=True)
    ref = one_thread(monkeypatch, [f, g], ci)
    assert np.isfinite(ref).all()
    assert ref[0, 1] == (1.0 / 40.0 + 1.0 / 700.0) + 1.0 / 70.0
    assert np.array_equal(np.asarray(pb.pairwise([f, g], ci)), ref)
    assert np.array_equal(np.asarray(pb.pairwise([f, g], ci, exact=False)), ref)
    ci2 = pb.CombinationIntegral(h=h, a=0.0, b=2.0, symmetric=True)  # b on a breakpoint
    assert np.array_equal(np.asarray(pb.pairwise([f, g], ci2)), one_thread(monkeypatch, [f, g], ci2))


def test_tiny_collections_and_progress(monkeypatch):
    """M = 1 (no tile items: the diagonal alone) and M = 2; progress sinks and
    cancellation on the tile path behave as on the one-thread path."""
    f = pb.make_pcf(np.array([[0.0, 1.5], [0.5, -2.0], [1.25, 0.0]]))
    g = pb.make_pcf(np.array([[0.0, 0.25], [0.75, 0.0]]))
    ci = pb.CombinationIntegral(h=sq_diff, r=math.sqrt, symmetric=True)
    for fs in ([f], [f, g]):
        assert np.array_equal(np.asarray(pb.pairwise(fs, ci)), one_thread(monkeypatch, fs, ci))
    fs = collection(n=120)
    job = pb.pairwise_job(fs, ci)
    seen = []
    job.subscribe(seen.append)
    D = np.asarray(job.run())
    assert seen[-1] == 1.0 and all(x <= y for x, y in zip(seen, seen[1:]))
    assert np.array_equal(D, one_thread(monkeypatch, fs, ci))
    assert job.entries_computed == len(fs) * (len(fs) + 1) // 2
    job2 = pb.pairwise_job(fs, ci)
    job2.cancel()
    with pytest.raises(errors.Cancelled):
        job2.run()
