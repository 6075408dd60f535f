"""masspcf front-end transcripts (reference: pkg/frontend/tests/test_transcripts.py)."""

import numpy as np
import pytest

from conftest import has_gpu

import paper_2404_07183_b200 as pb
from paper_2404_07183_b200 import masspcf as mpcf
from paper_2404_07183_b200.masspcf.random import noisy_cos, noisy_sin


@pytest.fixture
def X():
    return [mpcf.Pcf(np.array([[0.0, 5.0], [2.0, 3.0], [5.0, 0.0]])),
            mpcf.Pcf(np.array([[0.0, 2.0], [4.0, 7.0], [8.0, 1.0], [9.0, 0.0]])),
            mpcf.Pcf(np.array([[0.0, 4.0], [2.0, 3.0], [3.0, 1.0], [5.0, 0.0]])),
            mpcf.Pcf(np.array([[0.0, 2.0], [6.0, 1.0], [7.0, 0.0]]))]


def test_pcf_repr_and_export(X):
    f = X[0]
    assert repr(f) == "<PCF size=3, dtype=float64>"
    m = np.asarray(f)
    assert m.shape == (3, 2) and not m.flags.writeable
    g = mpcf.Pcf(np.array([[0, 1], [1, 0]], dtype=np.float32))
    assert g.dtype == np.float32


def test_array_shapes_and_views():
    Z = mpcf.zeros((10, 5, 4))
    assert repr(Z.shape) == "Shape(10, 5, 4)"
    assert tuple(Z[2].shape) == (5, 4)
    assert tuple(Z[:, 1:3].shape) == (10, 2, 4)
    f = Z[0, 1, 2]
    assert isinstance(f, mpcf.Pcf) and repr(f) == "<PCF size=1, dtype=float64>"
    A = mpcf.zeros((2, 6))
    A[0, :] = noisy_sin((6,), n_points=10, rng=pb.RngSpec(1))
    assert all(x.size == 11 for x in A[0, :].to_list())
    V = A[0, 1:4]
    A[0, 2] = A[1, 0]
    assert V[1] == A[1, 0]  # views share elements


def test_generators_deterministic():
    a = noisy_cos((3,), n_points=12, rng=pb.RngSpec(8))
    b = noisy_cos((3,), n_points=12, rng=pb.RngSpec(8))
    for f, g in zip(a.to_list(), b.to_list()):
        assert np.array_equal(np.asarray(f), np.asarray(g))


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a GPU")
def test_frontend_matrices_and_mean(X):
    assert np.array_equal(mpcf.pdist(X), [[0, 34, 6, 12], [34, 0, 34, 24], [6, 34, 0, 10],
                                          [12, 24, 10, 0]])
    assert np.array_equal(mpcf.l2_kernel(X), [[77, 53, 55, 38], [53, 213, 31, 51],
                                              [55, 31, 43, 26], [38, 51, 26, 25]])
    want = np.array([[0.0, 9.80058139, 2.49774585, 3.81895602],
                     [9.80058139, 0.0, 10.10250875, 8.76880217],
                     [2.49774585, 10.10250875, 0.0, 2.82601424],
                     [3.81895602, 8.76880217, 2.82601424, 0.0]])
    assert np.abs(mpcf.pdist(X, p=3.5) - want).max() < 1e-7
    assert np.array_equal(mpcf.pdist(mpcf.Array(X)), mpcf.pdist(X))
    M = 10
    A = mpcf.zeros((2, M))
    A[0, :] = noisy_sin((M,), n_points=100)
    A[1, :] = noisy_cos((M,), n_points=15)
    Aavg = mpcf.mean(A, dim=1)
    assert tuple(Aavg.shape) == (2,) and isinstance(Aavg[0], mpcf.Pcf)
    S = mpcf.std(A, dim=1)
    assert tuple(S.shape) == (2,)
    B = noisy_sin((6,), n_points=20, rng=pb.RngSpec(5))
    got = mpcf.mean(B, dim=0)[0]
    assert np.array_equal(np.asarray(got), pb.mean([f._inner for f in B.to_list()]).to_matrix())
