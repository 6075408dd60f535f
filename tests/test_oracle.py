"""The CPU oracle is pinned to the reference's own outputs (tests/golden, made by
tests/golden/make_golden.py from the compiled reference) before it is trusted as the
checker for the GPU engine."""

import math

import numpy as np
import pytest

from conftest import unpack

import oracle as O

TAGS_F64 = ["guide", "appa30", "appa200", "rand40"]


@pytest.mark.parametrize("tag", TAGS_F64)
def test_c_oracle_matrices_bitwise(golden, oracle, tag):
    t, v, off = golden[f"{tag}_tcat"], golden[f"{tag}_vcat"], golden[f"{tag}_off"]
    for key in golden:
        if not key.startswith(tag + "_pdist_p"):
            continue
        p = float(key.split("_p")[-1])
        D, bad = oracle.matrix(t, v, off, op=O.OP_LP, p=p, apply_root=True)
        assert bad is None
        assert np.array_equal(D, golden[key]), key
    if f"{tag}_gram" in golden:
        K, bad = oracle.matrix(t, v, off, op=O.OP_INNER, p=0.0, apply_root=False, diag=True)
        assert bad is None
        assert np.array_equal(K, golden[f"{tag}_gram"])


@pytest.mark.parametrize("tag,a,b", [("guideb", 0.5, 7.25), ("guideb2", 1.0, 6.0),
                                     ("rand40b", 0.75, 6.5)])
def test_c_oracle_bounded_bitwise(golden, oracle, tag, a, b):
    t, v, off = golden[f"{tag}_tcat"], golden[f"{tag}_vcat"], golden[f"{tag}_off"]
    for key in golden:
        if key.startswith(tag + "_pdist_p"):
            p = float(key.split("_p")[-1])
            D, _ = oracle.matrix(t, v, off, op=O.OP_LP, p=p, a=a, b=b)
            assert np.array_equal(D, golden[key]), key
    if f"{tag}_gram" in golden:
        K, _ = oracle.matrix(t, v, off, op=O.OP_INNER, p=0.0, apply_root=False, diag=True,
                             a=a, b=b)
        assert np.array_equal(K, golden[f"{tag}_gram"])


def test_c_oracle_float32(golden, oracle):
    t, v, off = golden["appa12f32_tcat"], golden["appa12f32_vcat"], golden["appa12f32_off"]
    assert t.dtype == np.float32
    for p in (1.0, 3.5):
        D, _ = oracle.matrix(t, v, off, p=p, out_dtype=np.float32)
        assert np.array_equal(D, golden[f"appa12f32_pdist_p{p:g}"])
    K, _ = oracle.matrix(t, v, off, op=O.OP_INNER, p=0.0, apply_root=False, diag=True,
                         out_dtype=np.float32)
    assert np.array_equal(K, golden["appa12f32_gram"])


def test_c_oracle_guide_raw_and_divergence(golden, oracle):
    fs = unpack(golden, "guide") + [np.array([[0.0, 1.0]])]
    raw = []
    for f in fs:
        for g in fs:
            for op, p in ((0, 1.0), (0, 2.0), (1, 0.0)):
                raw.append(oracle.accumulate(f, g, op=op, p=p))
    raw = np.array(raw)
    ref = golden["guide_raw"]
    assert np.array_equal(raw, ref)
    assert np.isinf(ref).any()  # the divergent pairs are in the vector


def test_c_oracle_matches_reference_build():
    """The restatement against the reference's own compiled _sweepkern (oracle/_ref)."""
    K = O.load_reference_kernel()
    if K is None:
        pytest.skip("oracle/_ref not built (make -C oracle ref needs /root/reference)")
    import paper_2404_07183_b200.datagen as dg

    t, v, off = dg.synthetic_benchmark_packed(60, rng=dg.RngSpec(5))
    orc = O.Oracle()
    for op, p, root, diag in ((0, 1.0, True, False), (0, 3.5, True, False),
                              (1, 0.0, False, True)):
        mine, _ = orc.matrix(t, v, off, op=op, p=p, apply_root=root, diag=diag)
        ref = np.zeros_like(mine)
        assert K.fill_block((t, v, off), 0, 60, op, p, root, diag, 0.0, math.inf, ref) is None
        assert np.array_equal(mine, ref)


@pytest.mark.parametrize("k", range(5))
def test_python_reduction_oracle(golden, k):
    fs = unpack(golden, f"red{k}")
    assert np.array_equal(O.tree_reduce(fs, lambda x, y: x + y), golden[f"red{k}_sum"])
    assert np.array_equal(O.mean(fs), golden[f"red{k}_mean"])
    if f"red{k}_std" in golden:
        assert np.array_equal(O.std(fs), golden[f"red{k}_std"])
        assert np.array_equal(O.std(fs, ddof=0), golden[f"red{k}_std_ddof0"])


def test_python_reduction_oracle_guide_and_f32(golden):
    g = unpack(golden, "guide")
    assert np.array_equal(O.mean(g[2:]), golden["guide_mean34"])
    assert np.array_equal(
        O.mean(g[2:]), np.array([(0, 3), (2, 2.5), (3, 1.5), (5, 1), (6, 0.5), (7, 0)], float))
    assert np.array_equal(O.std(g[2:]), golden["guide_std34"])
    fs = [m.astype(np.float32) for m in unpack(golden, "sin16f32")]
    assert np.array_equal(O.mean(fs, dtype=np.float32), golden["sin16f32_mean"])
