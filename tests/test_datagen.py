"""Our generators reproduce the reference's draws bit for bit (golden vectors from the
reference), so benchmark inputs are the same collections on both sides."""

import numpy as np

import paper_2404_07183_b200 as pb
from paper_2404_07183_b200 import datagen as dg


def _cat(fs):
    return dg.pack_matrices([f.to_matrix() for f in fs])


def test_synthetic_benchmark_matches_reference(golden):
    t, v, off = _cat(pb.synthetic_benchmark(25, rng=pb.RngSpec(2404)))
    assert np.array_equal(off, golden["gen_appa_off"])
    assert np.array_equal(t, golden["gen_appa_tcat"])
    assert np.array_equal(v, golden["gen_appa_vcat"])


def test_synthetic_benchmark_f32_matches_reference(golden):
    t, v, off = _cat(pb.synthetic_benchmark(25, rng=pb.RngSpec(9), dtype=np.float32))
    assert t.dtype == np.float32
    assert np.array_equal(off, golden["gen_appa32_off"])
    assert np.array_equal(t, golden["gen_appa32_tcat"])
    assert np.array_equal(v, golden["gen_appa32_vcat"])


def test_packed_variant_identical():
    a = _cat(pb.synthetic_benchmark(40, rng=pb.RngSpec(3)))
    b = dg.synthetic_benchmark_packed(40, rng=pb.RngSpec(3))
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_noisy_trig_matches_reference(golden):
    for tag, arr in (("gen_sin", pb.noisy_sin((6,), 20, rng=pb.RngSpec(5))),
                     ("gen_cos", pb.noisy_cos((3,), 12, rng=pb.RngSpec(8))),
                     ("gen_sin32", pb.noisy_sin((4,), 30, rng=pb.RngSpec(11),
                                                dtype=np.float32))):
        t, v, off = _cat(arr.to_list())
        assert np.array_equal(off, golden[f"{tag}_off"]), tag
        assert np.array_equal(t, golden[f"{tag}_tcat"]), tag
        assert np.array_equal(v, golden[f"{tag}_vcat"]), tag


def test_survey_recipes_valid():
    for rows in dg.fixed_size_collection(50, 100):
        pb.make_pcf(rows)
        assert rows.shape == (100, 2) and rows[-1, 1] == 0.0
    for rows in dg.fixed_size_collection(20, 200, dtype=np.float32):
        assert pb.make_pcf(rows).dtype == np.float32
    ecc = dg.ecc_like_collection(30)
    sizes = [r.shape[0] for r in ecc]
    assert min(sizes) >= 2 and max(sizes) <= 10000
    for rows in ecc:
        pb.make_pcf(rows)
        assert rows[-1, 1] == 1.0
