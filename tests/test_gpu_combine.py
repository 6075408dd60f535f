"""GPU parity of the generic combination integrals (pairwise / combine_integrate /
combine_integrate_timedep / integrate_single) against golden
vectors computed by the reference itself (tests/golden/make_golden_combine.py) with the
same integrand source (tests/golden/combine_integrands.py).

Bar: bit-identical for integrands of IEEE + - * / abs min max (device thread walks the
reference's cells in order, --fmad=false); relative 1e-12 where CUDA libdevice
transcendentals (exp, pow, sqrt of a non-square ...) stand in for glibc.
"""

import math
import os
import sys

import numpy as np
import pytest

from conftest import ROOT, has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a GPU")]

sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
from combine_integrands import CASES  # noqa: E402

import paper_2404_07183_b200 as pb  # noqa: E402
from paper_2404_07183_b200 import errors  # noqa: E402
from paper_2404_07183_b200.combine import integrate_single_many  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden", "reference_combine.npz")


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


def pcfs(g, tag):
    t, v, off = g[f"{tag}_tcat"], g[f"{tag}_vcat"], g[f"{tag}_off"]
    dt = np.float32 if tag.endswith("32") else np.float64
    return [pb.make_pcf(np.column_stack((t[off[i]:off[i + 1]], v[off[i]:off[i + 1]])),
                        dtype=dt) for i in range(off.shape[0] - 1)]


def close(x, ref, exact):
    x, ref = np.asarray(x, dtype=np.float64), np.asarray(ref, dtype=np.float64)
    if exact:
        return np.array_equal(x, ref, equal_nan=True)
    scale = np.maximum(np.abs(ref), 1e-300)
    d = np.abs(x - ref) / scale
    return bool(np.all((d < 1e-12) | (np.abs(x - ref) < 1e-13 * np.max(np.abs(ref)))))


@pytest.mark.parametrize("ctag", ["guide", "rnd", "rnd32", "appa"])
@pytest.mark.parametrize("name", sorted(CASES))
def test_combination_integrals_match_reference(gold, ctag, name):
    kind, fns, sym, (a, b), exact = CASES[name]
    fs = pcfs(gold, ctag)
    key = f"{ctag}_{name}"
    if kind == "u":
        got = integrate_single_many(fs, fns["h"], a, b)
        assert close(got, gold[key], exact), (got, gold[key])
        assert pb.integrate_single(fs[1], fns["h"], a, b) == got[1]
        return
    ci = pb.CombinationIntegral(h=fns.get("h"), H=fns.get("H"), r=fns.get("r"), a=a, b=b,
                                symmetric=sym)
    D = np.asarray(pb.pairwise(fs, ci))
    ref = gold[key]
    assert D.dtype == ref.dtype and D.shape == ref.shape
    assert close(D, ref, exact), np.max(np.abs(D - ref))
    if sym:
        assert np.array_equal(D, D.T)
    f, g = fs[0], fs[-1]
    val = (pb.combine_integrate(f, g, fns["h"], a, b) if kind == "h"
           else pb.combine_integrate_timedep(f, g, fns["H"], a, b))
    assert close(val, gold[key + "_scalar"], exact)
    assert close(ci(f, g), D[0, -1], True)


def test_pairwise_job_entries_progress_cancel(gold):
    fs = pcfs(gold, "rnd")
    ci = pb.CombinationIntegral(h=CASES["asym"][1]["h"], symmetric=False)
    job = pb.pairwise_job(fs, ci)
    seen = []
    job.subscribe(seen.append)
    D = job.run()
    assert job.entries_computed == len(fs) ** 2 and not D.symmetric
    assert seen[-1] == 1.0 and all(x <= y for x, y in zip(seen, seen[1:]))
    job2 = pb.pairwise_job(fs, ci)
    job2.cancel()
    with pytest.raises(errors.Cancelled):
        job2.run()
    sym = pb.pairwise_job(fs, pb.CombinationIntegral(h=CASES["prod"][1]["h"], symmetric=True))
    sym.run()
    assert sym.entries_computed == len(fs) * (len(fs) + 1) // 2


def offset(x, y):
    return x + y + 1.0


def nan_tail(x, y):
    return (x - y) / (x - y)


def test_errors(gold):
    fs = pcfs(gold, "guide")
    with pytest.raises(errors.DivergentIntegral) as info:
        pb.pairwise(fs, pb.CombinationIntegral(h=offset, symmetric=True))
    assert info.value.pair == (0, 0)
    with pytest.raises(errors.DivergentIntegral):
        pb.combine_integrate(fs[0], fs[1], offset)
    assert pb.combine_integrate(fs[0], fs[1], offset, 0.0, 2.0) == 2.0 * (5 + 2 + 1)
    with pytest.raises(errors.NonFinite):
        pb.combine_integrate(fs[0], fs[1], nan_tail)  # 0/0 on the tail cell
    with pytest.raises(errors.InvalidBounds):
        pb.combine_integrate(fs[0], fs[1], offset, 2.0, 1.0)
    f32 = pb.make_pcf(np.array([[0, 1], [1, 0]], dtype=np.float32))
    with pytest.raises(errors.MixedPrecision):
        pb.combine_integrate(fs[0], f32, offset)
    with pytest.raises(errors.UnsupportedIntegrand):
        pb.combine_integrate(fs[0], fs[1], lambda x, y: sorted([x, y])[0])
    with pytest.raises(ValueError):
        pb.CombinationIntegral()


def test_traced_integrand_without_source(gold):
    """An integrand built by exec has no source file: it is traced symbolically."""
    fs = pcfs(gold, "rnd")
    h = eval("lambda x, y: np.abs(x - y) * 0.5 + (x - y) ** 2", {"np": np})
    D = np.asarray(pb.pairwise(fs, pb.CombinationIntegral(h=h, symmetric=True)))

    def h2(x, y):
        return np.abs(x - y) * 0.5 + (x - y) ** 2

    D2 = np.asarray(pb.pairwise(fs, pb.CombinationIntegral(h=h2, symmetric=True)))
    assert np.array_equal(D, D2)


CTAGS = ["guide", "rnd", "rnd32", "appa"]


@pytest.mark.parametrize("k", range(7))
def test_sweeps_match_reference_cells(gold, k):
    """iterate_rectangles / iterate_segments: the device enumerates exactly the
    reference's cells (same edges, same values, same order)."""
    ci, i, j = (int(x) for x in gold[f"sweep{k}_which"])
    fs = pcfs(gold, CTAGS[ci])
    for bi, (a, b) in enumerate(((0.0, math.inf), (0.5, 7.25), (2.0, 3.0))):
        cells = []
        pb.iterate_rectangles(fs[i], fs[j], a, b, lambda r: cells.append(tuple(r)))
        assert np.array_equal(np.array(cells), gold[f"sweep{k}_b{bi}_rect"])
        assert isinstance(cells and pb.Rectangle(*cells[0]), pb.Rectangle)
        segs = []
        pb.iterate_segments(fs[i], a, b, lambda s: segs.append(tuple(s)))
        assert np.array_equal(np.array(segs), gold[f"sweep{k}_b{bi}_seg"])
    with pytest.raises(errors.InvalidBounds):
        pb.iterate_rectangles(fs[i], fs[j], 1.0, 1.0, lambda r: None)


@pytest.mark.parametrize("oname", ["add", "max", "min", "mul"])
@pytest.mark.parametrize("ctag", ["guide", "rnd", "rnd32"])
def test_reduction_accumulator_matches_reference(gold, oname, ctag):
    import operator

    op = {"add": operator.add, "max": max, "min": min, "mul": operator.mul}[oname]
    fs = pcfs(gold, ctag)
    acc = pb.ReductionAccumulator(op, dtype=fs[0].dtype)
    assert acc.size == 1 and acc.to_pcf().to_matrix().tolist() == [[0.0, 0.0]]
    for n, f in enumerate(fs[:9]):
        acc.combine(f)
        ref = gold[f"acc_{oname}_{ctag}_{n}"]
        got = acc.to_pcf().to_matrix()
        assert got.dtype == ref.dtype and np.array_equal(got, ref), (n, got, ref)
        assert acc.size == ref.shape[0]
    other = pb.ReductionAccumulator(op, dtype=fs[0].dtype)
    other.combine(fs[0])
    acc.combine(other)  # accumulator (op) accumulator
    with pytest.raises(errors.MixedPrecision):
        acc.combine(pb.make_pcf(np.array([[0, 1]], dtype=np.float32 if ctag != "rnd32"
                                         else np.float64)))
