"""Generate tests/golden/*.npz from the reference implementation itself.

Run in the build container only (needs /root/reference):

    python tests/golden/make_golden.py

It builds a scratch copy of the reference package (/tmp/refbuild, `setup.py build_ext
--inplace` on a copy -- /root/reference is read-only), imports ``pcflib`` from it and
records inputs + outputs.  The GPU box never runs this; the tests read the .npz files.
"""

from __future__ import annotations

import math
import os
import shutil
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg"
BUILD = "/tmp/refbuild"


def reference_pcflib():
    if not os.path.exists(os.path.join(BUILD, "src", "pcflib", "__init__.py")):
        shutil.copytree(REF, BUILD, dirs_exist_ok=True)
        subprocess.run(["chmod", "-R", "u+w", BUILD], check=True)
    if not any(n.startswith("_sweepkern") and n.endswith(".so")
               for n in os.listdir(os.path.join(BUILD, "src", "pcflib"))):
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=BUILD,
                       check=True, capture_output=True)
    sys.path[:0] = [os.path.join(BUILD, "src"), os.path.join(BUILD, "frontend", "src")]
    import pcflib

    assert pcflib.backend_name() == "compiled"
    return pcflib


def packed(fs):
    mats = [f.to_matrix() for f in fs]
    sizes = np.array([m.shape[0] for m in mats], dtype=np.int64)
    off = np.zeros(len(mats) + 1, dtype=np.int64)
    np.cumsum(sizes, out=off[1:])
    cat = np.concatenate(mats, axis=0)
    return cat[:, 0].copy(), cat[:, 1].copy(), off


def random_pcf(pl, rng, size, dtype=np.float64, eventually_zero=False, tmax=10.0):
    """tests/conftest.py:49-58 of the reference (same draws)."""
    times = np.concatenate(
        ([0.0], np.sort(rng.choice(np.arange(1, 20 * size) * (tmax / (20 * size)),
                                   size=size - 1, replace=False)))
        if size > 1 else ([0.0],))
    values = np.round(rng.uniform(-5, 5, size), 3)
    if eventually_zero:
        values[-1] = 0.0
    return pl.make_pcf(np.column_stack((times, values)), dtype=dtype)


def main():
    pl = reference_pcflib()
    out = {}
    guide = [
        pl.make_pcf([[0.0, 5.0], [2.0, 3.0], [5.0, 0.0]]),
        pl.make_pcf([[0.0, 2.0], [4.0, 7.0], [8.0, 1.0], [9.0, 0.0]]),
        pl.make_pcf([[0.0, 4.0], [2.0, 3.0], [3.0, 1.0], [5.0, 0.0]]),
        pl.make_pcf([[0.0, 2.0], [6.0, 1.0], [7.0, 0.0]]),
    ]

    def add_matrices(tag, fs, ps=(1.0, 2.0, 3.5), gram=True, bounds=None):
        t, v, off = packed(fs)
        out[f"{tag}_tcat"], out[f"{tag}_vcat"], out[f"{tag}_off"] = t, v, off
        for p in ps:
            kw = {} if bounds is None else {"a": bounds[0], "b": bounds[1]}
            out[f"{tag}_pdist_p{p:g}"] = np.asarray(pl.pdist(fs, p=p, workers=1, **kw))
        if gram:
            kw = {} if bounds is None else {"a": bounds[0], "b": bounds[1]}
            out[f"{tag}_gram"] = np.asarray(pl.l2_kernel(fs, workers=1, **kw))

    add_matrices("guide", guide, ps=(1.0, 2.0, 3.0, 3.5))
    add_matrices("guideb", guide, ps=(1.0, 2.0), bounds=(0.5, 7.25))
    add_matrices("guideb2", guide, ps=(1.0,), bounds=(1.0, 6.0))
    add_matrices("appa30", pl.synthetic_benchmark(30, rng=pl.RngSpec(74)))
    add_matrices("appa200", pl.synthetic_benchmark(200, rng=pl.RngSpec(2026)), ps=(1.0,))
    add_matrices("appa12f32", pl.synthetic_benchmark(12, rng=pl.RngSpec(73), dtype=np.float32),
                 ps=(1.0, 3.5))
    rng = np.random.default_rng(12345)
    rnd = [random_pcf(pl, rng, int(rng.integers(1, 40)), eventually_zero=True) for _ in range(40)]
    add_matrices("rand40", rnd, ps=(1.0, 2.0, 3.0))
    add_matrices("rand40b", rnd, ps=(1.0, 3.0), bounds=(0.75, 6.5))

    # generator pins (our datagen must reproduce these bit for bit)
    for tag, fs in (("gen_appa", pl.synthetic_benchmark(25, rng=pl.RngSpec(2404))),
                    ("gen_appa32", pl.synthetic_benchmark(25, rng=pl.RngSpec(9),
                                                          dtype=np.float32))):
        t, v, off = packed(fs)
        out[f"{tag}_tcat"], out[f"{tag}_vcat"], out[f"{tag}_off"] = t, v, off
    for tag, arr in (("gen_sin", pl.noisy_sin((6,), 20, rng=pl.RngSpec(5))),
                     ("gen_cos", pl.noisy_cos((3,), 12, rng=pl.RngSpec(8))),
                     ("gen_sin32", pl.noisy_sin((4,), 30, rng=pl.RngSpec(11), dtype=np.float32))):
        t, v, off = packed(arr.to_list())
        out[f"{tag}_tcat"], out[f"{tag}_vcat"], out[f"{tag}_off"] = t, v, off

    # reductions: mean / std of small collections (the reference std is O(M*N))
    rng = np.random.default_rng(777)
    for k, (M, smax) in enumerate(((2, 10), (5, 12), (7, 20), (16, 25), (33, 8))):
        fs = [random_pcf(pl, rng, int(rng.integers(1, smax))) for _ in range(M)]
        t, v, off = packed(fs)
        out[f"red{k}_tcat"], out[f"red{k}_vcat"], out[f"red{k}_off"] = t, v, off
        out[f"red{k}_mean"] = pl.mean(fs).to_matrix()
        if M >= 2:
            out[f"red{k}_std"] = pl.std(fs).to_matrix()
            out[f"red{k}_std_ddof0"] = pl.std(fs, ddof=0).to_matrix()
        out[f"red{k}_sum"] = pl.tree_reduce(fs, lambda x, y: x + y).to_matrix()
    sins = pl.noisy_sin((64,), 100, rng=pl.RngSpec(2404)).to_list()
    t, v, off = packed(sins)
    out["sin64_tcat"], out["sin64_vcat"], out["sin64_off"] = t, v, off
    out["sin64_mean"] = pl.mean(sins).to_matrix()
    out["sin64_std"] = pl.std(sins).to_matrix()
    sins32 = pl.noisy_sin((16,), 50, rng=pl.RngSpec(31), dtype=np.float32).to_list()
    t, v, off = packed(sins32)
    out["sin16f32_tcat"], out["sin16f32_vcat"], out["sin16f32_off"] = t, v, off
    out["sin16f32_mean"] = pl.mean(sins32).to_matrix()
    out["sin16f32_std"] = pl.std(sins32).to_matrix()
    out["guide_mean34"] = pl.mean(guide[2:]).to_matrix()
    out["guide_std34"] = pl.std(guide[2:]).to_matrix()

    # scalar integrals incl. divergence sentinel (raw, un-rooted)
    bad = pl.make_pcf([(0, 1)])
    from pcflib import _sweepkern as K

    raw = []
    for f in guide + [bad]:
        for g in guide + [bad]:
            for op, p in ((0, 1.0), (0, 2.0), (1, 0.0)):
                raw.append((K.integrate_pair(f.times, f.values, g.times, g.values, 0.0,
                                             math.inf, op, p)))
    out["guide_raw"] = np.array(raw)

    path = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
