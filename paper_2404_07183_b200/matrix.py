"""Pairwise distance / Gram matrices on the GPU.

API mirror of pkg/src/pcflib/matrix.py (``PairwiseMatrix``, ``MatrixJob``, ``pdist``,
``pdist_job``, ``l2_kernel``, ``l2_kernel_job``, ``resolve_workers``,
``progress_subscribe``).  The reference's host thread pool over row blocks
(matrix.py:146-227) is replaced by one persistent device kernel over cost-sorted tiles
(engine.fill_pairwise); ``workers`` is accepted and validated for drop-in compatibility
but the GPU decides its own parallelism.  Every entry still has exactly one writer and
a fixed summation order, so results are identical run to run and for any GPU count.
Progress is reported per completed slice of the device work queue (monotone, ending at
1.0) and cancellation is honoured between slices.
"""

from __future__ import annotations

import math
import os
import threading

import numpy as np

from . import errors
from .engine import OP_INNER, OP_LP, decode_err, fill_pairwise

__all__ = [
    "PairwiseMatrix",
    "MatrixJob",
    "pdist",
    "pdist_job",
    "l2_kernel",
    "l2_kernel_job",
    "progress_subscribe",
    "resolve_workers",
    "pairwise",
    "pairwise_job",
]

_INF = math.inf
_PROGRESS_SLICES = 8


def resolve_workers(workers=None):
    """Explicit argument, else MASSPCF_THREADS, else the CPU count (>= 1)."""
    if workers is None:
        env = os.environ.get("MASSPCF_THREADS")
        n = int(env) if env else (os.cpu_count() or 1)
    else:
        n = int(workers)
    if n < 1:
        raise ValueError(f"worker count must be >= 1, got {n}")
    return n


class PairwiseMatrix:
    """Dense M x M result (numpy on the host, or a torch tensor when the job was run
    with ``device_output=True``) plus its symmetry flag."""

    def __init__(self, data, symmetric, entries_computed=0):
        self.data = data
        self.symmetric = symmetric
        self.entries_computed = entries_computed

    @property
    def shape(self):
        return tuple(self.data.shape)

    @property
    def dtype(self):
        return self.data.dtype

    def __array__(self, dtype=None, copy=None):
        d = self.data
        if not isinstance(d, np.ndarray):
            d = d.cpu().numpy()
        return np.asarray(d, dtype=dtype)

    def __getitem__(self, idx):
        return self.data[idx]

    def __repr__(self):
        return f"PairwiseMatrix(shape={self.shape}, symmetric={self.symmetric})"


def _collection_kind(collection):
    coll = list(collection)
    if not coll:
        raise errors.EmptyCollection("pairwise matrix of an empty collection")
    kind = coll[0].dtype
    if any(f.dtype != kind for f in coll):
        raise errors.MixedPrecision("collection mixes 32- and 64-bit PCFs")
    return coll, kind


class MatrixJob:
    """A pending pairwise-matrix computation: subscribe progress sinks, keep the
    handle to cancel, then ``run``."""

    def __init__(self, collection, *, op=OP_LP, p=1.0, apply_root=False, diag=False,
                 a=0.0, b=_INF, integral=None):
        self._coll, self._dtype = _collection_kind(collection)
        self._integral = integral
        if integral is not None:  # bounds live on the integral (matrix.py:113-124)
            a, b = integral.a, integral.b
        a = float(a)
        b = float(b)
        if math.isnan(a) or math.isinf(a) or a < 0.0 or not a < b:
            raise errors.InvalidBounds(f"bounds must satisfy 0 <= a < b, got [{a}, {b})")
        self._op = op
        self._p = float(p)
        self._apply_root = bool(apply_root)
        self._diag = bool(diag)
        self._a = a
        self._b = b
        self.symmetric = True if integral is None else bool(integral.symmetric)
        self._sinks = []
        self._cancel = threading.Event()
        self.entries_computed = 0

    def subscribe(self, sink):
        """Register a callback receiving monotone fractions in (0, 1], last 1.0."""
        self._sinks.append(sink)

    def cancel(self):
        self._cancel.set()

    @property
    def cancelled(self):
        return self._cancel.is_set()

    def run(self, workers=None, device_output=False, exact=None):
        """Compute the matrix.  Default (exact, env PCF_B200_EXACT unset or 1): every entry
        is summed by one lane strictly left to right with the C library's pow, like the
        reference -- bit-identical to it and to lp_distance / l2_inner_product for every
        p (test_matrix.py:41-47,97-102).  exact=False (or PCF_B200_EXACT=0) lets up to a
        warp share a long pair and evaluates p = 2, 3 cells as products: the same cells
        summed in G runs, relative error < 1e-13.

        A host result with no progress sinks goes through the whole-matrix host-buffer
        call (pcf_matrix_host): upload, device pack, one persistent fill launch, and the
        D2H of finished rows into a pinned result while later rows compute."""
        exact_arg = exact
        if exact is None:
            exact = os.environ.get("PCF_B200_EXACT", "1").strip() not in ("0", "false", "")
        resolve_workers(workers)
        if self._cancel.is_set():
            raise errors.Cancelled("matrix job cancelled; partial work discarded")
        if (self._integral is None and not device_output and not self._sinks):
            return self._run_host(bool(exact))
        from .collection import DeviceCollection

        coll = DeviceCollection.from_pcfs(self._coll)
        M = coll.M
        last = [0.0]

        def report(frac):
            if frac > last[0]:
                last[0] = frac
                for sink in self._sinks:
                    sink(frac)
            return self._cancel.is_set()

        if self._integral is not None:
            return self._run_custom(coll, report, device_output, exact_arg)
        out, err, stopped = fill_pairwise(
            coll, self._op, self._p, self._apply_root, self._diag, self._a, self._b,
            chunks=_PROGRESS_SLICES if self._sinks else 1,
            between_chunks=report if self._sinks else None, exact=bool(exact))
        if stopped or self._cancel.is_set():
            raise errors.Cancelled("matrix job cancelled; partial work discarded")
        bad = decode_err(err, M)
        if bad is not None:
            raise self._divergence_error(bad)
        self.entries_computed = M * (M + 1) // 2 if self._diag else M * (M - 1) // 2
        data = out if device_output else out.cpu().numpy()
        return PairwiseMatrix(data, True, self.entries_computed)

    def _run_host(self, exact):
        """Host result through pcf_matrix_host (see run)."""
        from .collection import require_cuda
        from .datagen import pack_matrices
        from .engine import matrix_host

        torch = require_cuda()
        tcat, vcat, off = pack_matrices([f.to_matrix() for f in self._coll], self._dtype)
        M = int(off.shape[0] - 1)
        # pageable result (pinning an 80 GB array costs about a minute): finished rows go
        # through pcf_matrix_host's small pinned staging pool, copied into place by host
        # threads while the fill continues
        out = np.empty((M, M), dtype=np.float32 if self._dtype == np.float32 else np.float64)
        out, bad = matrix_host(tcat, vcat, off, self._op, self._p, self._apply_root,
                               self._diag, self._a, self._b, exact=exact, out=out)
        if bad is not None:
            raise self._divergence_error(bad)
        self.entries_computed = M * (M + 1) // 2 if self._diag else M * (M - 1) // 2
        return PairwiseMatrix(out, True, self.entries_computed)

    def _run_custom(self, coll, report, device_output, exact=None):
        """Arbitrary CombinationIntegral (matrix.py:184-196): the integrand is compiled
        for the device (jit.py); symmetric integrals fill one triangle incl. the
        diagonal and mirror it, asymmetric ones all M^2 entries.  Custom integrals are
        exact (the reference's per-entry sum order) unless exact=False is passed."""
        import torch

        from .combine import _status_error, fill_custom

        M = coll.M
        out = torch.zeros((M, M), dtype=coll.out_torch_dtype, device=coll.device)
        err, stopped = fill_custom(coll, self._integral, out,
                                   row_chunks=_PROGRESS_SLICES if self._sinks else 1,
                                   between=report if self._sinks else None,
                                   exact=exact is not False)
        if stopped or self._cancel.is_set():
            raise errors.Cancelled("matrix job cancelled; partial work discarded")
        if err is not None:
            exc = _status_error(err[0], self._integral.H is not None)
            exc.pair = (int(err[1]), int(err[2]))
            raise exc
        self.entries_computed = M * (M + 1) // 2 if self.symmetric else M * M
        data = out if device_output else out.cpu().numpy()
        return PairwiseMatrix(data, self.symmetric, self.entries_computed)

    def _divergence_error(self, pair):
        i, j = int(pair[0]), int(pair[1])
        if self._b == _INF:
            return errors.DivergentIntegral(
                f"integral of pair ({i}, {j}) diverges on [{self._a}, inf)", pair=(i, j))
        return errors.NonFinite(f"integral of pair ({i}, {j}) is not finite")


def pdist_job(collection, p=1.0, a=0.0, b=_INF) -> MatrixJob:
    """L_p distance matrix job: diagonal exactly 0, r = x^(1/p)."""
    p = float(p)
    if not p >= 1.0:
        raise ValueError(f"p must be >= 1, got {p}")
    return MatrixJob(collection, op=OP_LP, p=p, apply_root=True, diag=False, a=a, b=b)


def pdist(collection, p=1.0, workers=None, a=0.0, b=_INF, device_output=False, exact=None):
    """Pairwise L_p distance matrix over [a, b); L_1 by default."""
    return pdist_job(collection, p=p, a=a, b=b).run(workers, device_output=device_output,
                                                     exact=exact)


def l2_kernel_job(collection, a=0.0, b=_INF) -> MatrixJob:
    """L_2 Gram matrix job (diagonal included)."""
    return MatrixJob(collection, op=OP_INNER, p=0.0, apply_root=False, diag=True, a=a, b=b)


def l2_kernel(collection, workers=None, a=0.0, b=_INF, device_output=False, exact=None):
    """Pairwise L_2 inner product (Gram) matrix over [a, b)."""
    return l2_kernel_job(collection, a=a, b=b).run(workers, device_output=device_output,
                                                   exact=exact)


def pairwise_job(collection, integral) -> MatrixJob:
    """Job for an arbitrary combination integral (matrix.py:273-276)."""
    return MatrixJob(collection, integral=integral)


def pairwise(collection, integral, workers=None, device_output=False,
             exact=None) -> PairwiseMatrix:
    """Pairwise integrated combination matrix under an arbitrary CombinationIntegral
    (matrix.py:279-283); the integrand runs on the device (jit.py).  exact=False lets
    the tile kernels split long pairs over a warp (symmetric h only)."""
    return pairwise_job(collection, integral).run(workers, device_output=device_output,
                                                  exact=exact)


def progress_subscribe(job: MatrixJob, sink) -> None:
    job.subscribe(sink)
