import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built engine")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


def unpack(g, tag):
    """(tcat, vcat, off) -> list of (n, 2) float arrays."""
    t, v, off = g[f"{tag}_tcat"], g[f"{tag}_vcat"], g[f"{tag}_off"]
    return [np.column_stack((t[off[i]:off[i + 1]], v[off[i]:off[i + 1]]))
            for i in range(off.shape[0] - 1)]


@pytest.fixture(scope="session")
def oracle():
    import oracle as _o

    return _o.Oracle()


def has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
