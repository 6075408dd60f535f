"""CPU checks of the integrand translator (jit.py): every golden integrand translates
and NVRTC-compiles for sm_100a (no GPU needed); unsupported constructs fail loudly."""

import math
import os
import sys

import numpy as np
import pytest

from conftest import ROOT

sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
from combine_integrands import CASES  # noqa: E402

from paper_2404_07183_b200 import errors, jit  # noqa: E402


def _nvrtc_ok():
    try:
        jit.compile_only(jit.generate(h=lambda x, y: x * y))
        return True
    except Exception:
        return False


@pytest.mark.parametrize("name", sorted(CASES))
def test_golden_integrands_translate(name):
    kind, fns, *_ = CASES[name]
    src = jit.generate(u=fns["h"]) if kind == "u" else jit.generate(
        h=fns.get("h"), H=fns.get("H"), r=fns.get("r"))
    assert "pcf_" in src and "__device__" in src
    if _nvrtc_ok():
        assert jit.compile_only(src) > 0


K = 3.0


def test_semantics_of_translation():
    src = jit.generate(h=lambda x, y: max(x, y, K) % 2 if not x else -y // 4)
    assert "pcf_pymax(pcf_pymax(a_x, a_y), (0x1.8000000000000p+1))" in src
    assert "pcf_pymod" in src and "pcf_pyfloordiv(" in src
    src = jit.generate(h=lambda x, y: (x - y) ** 2 + math.pi)
    assert "pcf_sq((a_x - a_y))" in src and float.hex(math.pi) in src


def uses_list(x, y):
    return [x, y][0]


def test_unsupported_fail_loudly():
    with pytest.raises(errors.UnsupportedIntegrand):
        jit.generate(h=uses_list)
    with pytest.raises(errors.UnsupportedIntegrand):
        jit.generate(h=lambda x: x)
    h = eval("lambda x, y: x if x > y else y")  # no source and data-dependent branch
    with pytest.raises(errors.UnsupportedIntegrand):
        jit.generate(h=h)
    h = eval("lambda x, y: np.maximum(x, y) * 2 - abs(y)", {"np": np})
    assert "pcf_npmax" in jit.generate(h=h)


@pytest.mark.skipif(not _nvrtc_ok(), reason="NVRTC unavailable")
@pytest.mark.parametrize("f32", [False, True])
def test_tile_kernels_compile_for_user_integrands(f32):
    """pcf_tiles.cuh (K1 / K1c / K1r / K1g / K1s) compiles under NVRTC with a user h and r and
    exports all ten instantiations (pcf_jit_tiles_cubin)."""
    defs = jit.generate(h=lambda x, y: abs(x - y) * (1.0 + x * y), r=math.sqrt)
    assert jit.compile_tiles_only(defs, f32) > 0


def test_symmetry_probe_and_tile_eligibility(monkeypatch):
    from paper_2404_07183_b200.combine import (CombinationIntegral, _probably_symmetric,
                                               _tiles_eligible)

    assert _probably_symmetric(lambda x, y: abs(x - y))
    assert _probably_symmetric(lambda x, y: x * y + min(x, y))
    assert not _probably_symmetric(lambda x, y: x - 0.5 * y)
    assert not _probably_symmetric(lambda x, y: math.log(x - y))  # raises on the probe set
    sym = CombinationIntegral(h=lambda x, y: (x - y) ** 2, symmetric=True)
    assert _tiles_eligible(sym)
    assert not _tiles_eligible(CombinationIntegral(h=lambda x, y: (x - y) ** 2))
    assert not _tiles_eligible(CombinationIntegral(H=lambda x, y, t: x * y * t, symmetric=True))
    monkeypatch.setenv("PCF_JIT_NO_TILES", "1")
    assert not _tiles_eligible(sym)
