"""Collection I/O: the binary .pcfb container round-trips the
reference pack() layout bit for bit through a memory map; the reference's JSON and CSV
formats (pkg/src/pcflib/cli.py:59-150) load to the same packed arrays and our JSON writer
emits the reference's bytes; validation raises the reference's error classes."""

import json

import numpy as np
import pytest

from paper_2404_07183_b200 import datagen as dg, errors, io


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_pcfb_roundtrip_bitwise(tmp_path, dtype):
    t, v, off = dg.synthetic_benchmark_packed(300, rng=dg.RngSpec(7), dtype=dtype)
    path = tmp_path / "c.pcfb"
    io.save_packed(path, t, v, off)
    t2, v2, off2 = io.load_packed(path)
    assert t2.dtype == dtype and isinstance(t2.base, np.memmap) or t2.base is not None
    assert np.array_equal(off2, off)
    assert t2.tobytes() == t.tobytes() and v2.tobytes() == v.tobytes()
    t3, v3, off3 = io.load_collection(path)
    assert np.array_equal(t3, t) and np.array_equal(v3, v) and np.array_equal(off3, off)


def test_json_matches_reference_writer(tmp_path):
    t, v, off = dg.synthetic_benchmark_packed(25, rng=dg.RngSpec(8))
    path = tmp_path / "c.json"
    io.save_collection(path, t, v, off)
    # the reference's writer (cli.py:128-135): {"dtype", "pcfs": [[[t, v], ...]]}, compact
    doc = {"dtype": "f64", "pcfs": [[[a, b] for a, b in zip(t[off[i]:off[i + 1]].tolist(),
                                                           v[off[i]:off[i + 1]].tolist())]
                                    for i in range(len(off) - 1)]}
    assert path.read_text() == json.dumps(doc, separators=(",", ":")) + "\n"
    t2, v2, off2 = io.load_collection(path)
    assert np.array_equal(t2, t) and np.array_equal(v2, v) and np.array_equal(off2, off)


def test_csv_dir(tmp_path):
    mats = [np.array([[0.0, 1.5], [0.25, -2.0], [3.0, 0.0]]), np.array([[0.0, 7.0]])]
    for i, m in enumerate(mats):
        lines = ["t,v"] + [f"{repr(float(a))},{repr(float(b))}" for a, b in m]
        (tmp_path / f"p{i:03d}.csv").write_text("\n".join(lines) + "\n")
    t, v, off = io.load_collection(tmp_path)
    assert off.tolist() == [0, 3, 4]
    assert t.tolist() == [0.0, 0.25, 3.0, 0.0] and v.tolist() == [1.5, -2.0, 0.0, 7.0]


def test_validation_errors(tmp_path):
    ok_t, ok_v, ok_off = np.array([0.0, 1.0, 0.0]), np.array([1.0, 0.0, 2.0]), np.array([0, 2, 3])
    assert io.validate_packed(ok_t, ok_v, ok_off) == 2
    with pytest.raises(errors.NonZeroStart):
        io.validate_packed(np.array([0.0, 1.0, 0.5]), ok_v, ok_off)
    with pytest.raises(errors.NonIncreasingTimes):
        io.validate_packed(np.array([0.0, 0.0, 0.0]), ok_v, ok_off)
    with pytest.raises(errors.NonFinite):
        io.validate_packed(ok_t, np.array([1.0, np.nan, 2.0]), ok_off)
    with pytest.raises(errors.Empty):
        io.validate_packed(ok_t, ok_v, np.array([0, 2, 2, 3]))
    with pytest.raises(errors.EmptyCollection):
        io.validate_packed(ok_t[:0], ok_v[:0], np.array([0]))
    bad = tmp_path / "bad.pcfb"
    bad.write_bytes(b"PCFB\x01\x00\x00\x00" + b"\x00" * 10)
    with pytest.raises(errors.PcfError):
        io.load_packed(bad)
