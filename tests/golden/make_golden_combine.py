"""Golden vectors for the generic combination integrals (pcflib.pairwise /
combine_integrate / combine_integrate_timedep / integrate_single), computed by the
reference itself; run in the build container only:

    python tests/golden/make_golden_combine.py  ->  tests/golden/reference_combine.npz
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from combine_integrands import CASES  # noqa: E402
from make_golden import packed, random_pcf, reference_pcflib  # noqa: E402


def collections(pl):
    guide = [
        pl.make_pcf([[0.0, 5.0], [2.0, 3.0], [5.0, 0.0]]),
        pl.make_pcf([[0.0, 2.0], [4.0, 7.0], [8.0, 1.0], [9.0, 0.0]]),
        pl.make_pcf([[0.0, 4.0], [2.0, 3.0], [3.0, 1.0], [5.0, 0.0]]),
        pl.make_pcf([[0.0, 2.0], [6.0, 1.0], [7.0, 0.0]]),
    ]
    rng = np.random.default_rng(4242)
    rnd = [random_pcf(pl, rng, int(rng.integers(1, 30)), eventually_zero=True)
           for _ in range(24)]
    rnd32 = [random_pcf(pl, rng, int(rng.integers(1, 20)), dtype=np.float32,
                        eventually_zero=True) for _ in range(10)]
    appa = pl.synthetic_benchmark(16, rng=pl.RngSpec(91))
    return {"guide": guide, "rnd": rnd, "rnd32": rnd32, "appa": appa}


def main():
    pl = reference_pcflib()
    out = {}
    for ctag, fs in collections(pl).items():
        t, v, off = packed(fs)
        out[f"{ctag}_tcat"], out[f"{ctag}_vcat"], out[f"{ctag}_off"] = t, v, off
        for name, (kind, fns, sym, (a, b), _exact) in CASES.items():
            key = f"{ctag}_{name}"
            if kind == "u":
                vals = []
                for f in fs:
                    try:
                        vals.append(pl.integrate_single(f, fns["h"], a, b))
                    except (pl.errors.DivergentIntegral, pl.errors.NonFinite):
                        vals.append(np.nan)
                out[key] = np.array(vals)
                continue
            ci = pl.CombinationIntegral(h=fns.get("h"), H=fns.get("H"), r=fns.get("r"),
                                        a=a, b=b, symmetric=sym)
            try:
                out[key] = np.asarray(pl.pairwise(fs, ci, workers=1))
            except (pl.errors.DivergentIntegral, pl.errors.NonFinite) as exc:
                out[key + "_error"] = np.array(type(exc).__name__)
            # scalar API on the first pair
            f, g = fs[0], fs[-1]
            try:
                if kind == "h":
                    val = pl.combine_integrate(f, g, fns["h"], a, b)
                else:
                    val = pl.combine_integrate_timedep(f, g, fns["H"], a, b)
                out[key + "_scalar"] = np.array(val)
            except (pl.errors.DivergentIntegral, pl.errors.NonFinite) as exc:
                out[key + "_scalar_error"] = np.array(type(exc).__name__)
    # sweeps: the cells of pairs / the pieces of single PCFs (sweep.py:67-116)
    import operator

    fsets = collections(pl)
    sweep_pairs = [("guide", 0, 1), ("guide", 2, 3), ("rnd", 0, 5), ("rnd", 3, 3),
                   ("rnd", 7, 11), ("rnd32", 1, 2), ("appa", 0, 9)]
    for k, (ctag, i, j) in enumerate(sweep_pairs):
        for bi, (a, b) in enumerate(((0.0, np.inf), (0.5, 7.25), (2.0, 3.0))):
            cells = []
            pl.iterate_rectangles(fsets[ctag][i], fsets[ctag][j], a, b,
                                  lambda r: cells.append(tuple(r)))
            out[f"sweep{k}_b{bi}_rect"] = np.array(cells, dtype=np.float64)
            segs = []
            pl.iterate_segments(fsets[ctag][i], a, b, lambda sg: segs.append(tuple(sg)))
            out[f"sweep{k}_b{bi}_seg"] = np.array(segs, dtype=np.float64)
        out[f"sweep{k}_which"] = np.array([["guide", "rnd", "rnd32", "appa"].index(ctag), i, j])
    # accumulators: sequential folds (reduce.py:66-186)
    for oname, op in (("add", operator.add), ("max", max), ("min", min), ("mul", operator.mul)):
        for ctag in ("guide", "rnd", "rnd32"):
            acc = pl.ReductionAccumulator(op, dtype=fsets[ctag][0].dtype)
            snaps = []
            for f in fsets[ctag][:9]:
                acc.combine(f)
                snaps.append(acc.to_pcf().to_matrix())
            for n, m in enumerate(snaps):
                out[f"acc_{oname}_{ctag}_{n}"] = m
    path = os.path.join(HERE, "reference_combine.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path) / 1e6:.3f} MB")


if __name__ == "__main__":
    main()
