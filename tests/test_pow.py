"""The libm-exact pow (csrc/pcf_pow.cuh) that every L_p kernel uses for p != 1 and for
roots: the host build of the same header must equal the C library's pow bit for bit
(glibc 2.39 pow, the reference's pow at _sweepkern.pyx:43-46,98,114 and CPython's float
pow in integrate.py), and the device build must equal the host (GPU test)."""

import math
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, has_gpu

CSRC = os.path.join(ROOT, "paper_2404_07183_b200", "csrc")


def test_host_restatement_matches_libm(tmp_path):
    import __graft_entry__ as g

    g._pow_tables()
    exe = str(tmp_path / "check_pow")
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-I", CSRC,
                    os.path.join(ROOT, "tools", "check_pow.cc"), "-o", exe, "-lm"], check=True)
    out = subprocess.run([exe, "6"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout[-3000:]
    assert "OK: 0 mismatches" in out.stdout


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a GPU")
def test_device_pow_matches_libm():
    import torch

    from paper_2404_07183_b200 import _native

    rng = np.random.default_rng(5)
    n = 200000
    ys = np.array([2.0, 3.0, 3.5, 1.5, 0.5, 1 / 3, 1 / 3.5, 1.0, 7.25])
    x = np.concatenate([rng.uniform(0, 8, n // 2), np.ldexp(rng.uniform(0.5, 1.5, n // 2),
                                                            rng.integers(-1070, 1000, n // 2)),
                        [0.0, 1.0, 5e-324, 2.0 ** -1022, 1.7976931348623157e308, math.inf]])
    y = ys[rng.integers(0, ys.shape[0], x.shape[0])]
    def libm_pow(a, b):  # CPython's float pow is the C library's pow (+ overflow check)
        try:
            return math.pow(a, b)
        except OverflowError:
            return math.inf

    want = np.array([libm_pow(a, b) for a, b in zip(x.tolist(), y.tolist())])
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    od = torch.empty_like(xd)
    lib = _native.load()
    _native.check(lib.pcf_pow_batch(_native.ptr(xd), _native.ptr(yd), x.shape[0],
                                    _native.ptr(od), None), "pcf_pow_batch")
    got = od.cpu().numpy()
    bad = np.flatnonzero(got.view(np.uint64) != want.view(np.uint64))
    assert bad.size == 0, [(x[i].hex(), y[i], got[i].hex(), want[i].hex()) for i in bad[:5]]
