"""Device-level entry points of the pairwise engine (thin wrappers over the C ABI).

``fill_pairwise`` is the on-device replacement for MatrixJob.run's block loop
(pkg/src/pcflib/matrix.py:156-234): one persistent kernel drains the cost-sorted work
queue, so scheduling, mirroring and the first-failure capture all happen on the GPU.
"""

from __future__ import annotations

import math

import numpy as np

from . import _native
from .collection import DeviceCollection, current_stream_handle

OP_LP = 0
OP_INNER = 1

_NO_ERR = np.uint64(0xFFFFFFFFFFFFFFFF)


def _torch():
    import torch

    return torch


def new_err(device):
    torch = _torch()
    return torch.full((1,), -1, dtype=torch.int64, device=device)


def decode_err(err, M):
    """None, or the (i, j) original-index pair of the first non-finite entry."""
    key = np.uint64(int(err.item()) & 0xFFFFFFFFFFFFFFFF)
    if key == _NO_ERR:
        return None
    return int(key // np.uint64(M)), int(key % np.uint64(M))


def fill_pairwise(coll: DeviceCollection, op, p, apply_root, diag, a=0.0, b=math.inf,
                  out=None, err=None, items=None, chunks=1, between_chunks=None, exact=False):
    """Write the full symmetric M x M matrix into `out` (device tensor, allocated if
    None).  Diagonal: <f,f> when `diag` (Gram), exact 0 otherwise.  Returns
    (out, err, stopped).  `items` = (items_dev, n_smem, n_global, smem_bytes) or None
    for the collection's cached plan; `exact` selects the one-lane-per-pair plan.
    `between_chunks(frac)` is called after each of `chunks` slices of the queue has
    completed on the device; returning True stops early (cancellation)."""
    torch = _torch()
    lib = _native.load()
    M = coll.M
    dev = coll.device
    with torch.cuda.device(dev):
        if out is None:
            out = torch.empty((M, M), dtype=coll.out_torch_dtype, device=dev)
        if err is None:
            err = new_err(dev)
        if items is None:
            items_dev, _, n_smem, n_glob, smem = coll.plan(exact=exact)
        else:
            items_dev, n_smem, n_glob, smem = items
        st = current_stream_handle()
        out_f32 = int(out.dtype == torch.float32)
        ld = out.stride(0)
        _native.check(lib.pcf_fill_diagonal(
            _native.ptr(coll.recs), _native.ptr(coll.soff), _native.ptr(coll.perm), M,
            int(bool(diag)), float(a), float(b), _native.ptr(out), out_f32, ld,
            _native.ptr(err), st), "pcf_fill_diagonal")
        counter = torch.zeros(1, dtype=torch.int32, device=dev)
        segs = []
        for base, count, mode in ((0, n_smem, 1), (n_smem, n_glob, 0)):
            if count <= 0:
                continue
            k = max(1, min(int(chunks), count))
            bounds = [base + (count * i) // k for i in range(k + 1)]
            segs += [(bounds[i], bounds[i + 1], mode) for i in range(k) if bounds[i + 1] > bounds[i]]
        nseg = len(segs)
        events = []
        for idx, (s0, s1, mode) in enumerate(segs):
            ptr_items = _native.ptr(items_dev) if s0 == 0 else \
                _native.c_vp(items_dev.data_ptr() + s0 * 32)
            _native.check(lib.pcf_fill_matrix(
                _native.ptr(coll.recs), _native.ptr(coll.soff), _native.ptr(coll.perm), M,
                ptr_items, s1 - s0, smem, mode, _native.ptr(counter), int(op), float(p),
                int(bool(apply_root)), float(a), float(b), _native.ptr(out), out_f32, ld,
                _native.ptr(err), st), "pcf_fill_matrix")
            if between_chunks is not None:
                ev = torch.cuda.Event()
                ev.record()
                events.append(ev)
                # keep at most one slice queued ahead of the one being reported
                if len(events) >= 2:
                    events[-2].synchronize()
                    if between_chunks((idx) / nseg):
                        return out, err, True
        if between_chunks is not None and events:
            events[-1].synchronize()
            between_chunks(1.0)
    return out, err, False


def fill_rows(coll: DeviceCollection, r0, r1, op, p, apply_root, diag, a, b, out_f32=None):
    """fill_block mirror (pyx:88-121): rows [r0, r1) of original indices, columns
    j > i (j >= i with diag), as a compact (r1-r0) x M device slab, plus err."""
    torch = _torch()
    lib = _native.load()
    M = coll.M
    with torch.cuda.device(coll.device):
        if out_f32 is None:
            out_f32 = coll.dtype == np.float32
        slab = torch.zeros((max(r1 - r0, 0), M),
                           dtype=torch.float32 if out_f32 else torch.float64, device=coll.device)
        err = new_err(coll.device)
        _native.check(lib.pcf_fill_rows(
            _native.ptr(coll.recs), _native.ptr(coll.soff), _native.ptr(coll.inv), M, int(r0),
            int(r1), int(op), float(p), int(bool(apply_root)), int(bool(diag)), float(a),
            float(b), _native.ptr(slab), int(bool(out_f32)), _native.ptr(err),
            current_stream_handle()), "pcf_fill_rows")
    return slab, err


def pair_integrals(coll: DeviceCollection, pairs_orig, op, p, a=0.0, b=math.inf):
    """Raw integrals (float64, +-inf on divergence) of original-index pairs."""
    torch = _torch()
    lib = _native.load()
    pairs = np.asarray(pairs_orig, dtype=np.int64).reshape(-1, 2)
    sorted_pairs = coll_inv_host(coll)[pairs].astype(np.int64)
    with torch.cuda.device(coll.device):
        pd = torch.from_numpy(np.ascontiguousarray(sorted_pairs.reshape(-1))).to(coll.device)
        res = torch.empty(pairs.shape[0], dtype=torch.float64, device=coll.device)
        _native.check(lib.pcf_pair_list(
            _native.ptr(coll.recs), _native.ptr(coll.soff), _native.ptr(pd), pairs.shape[0],
            int(op), float(p), float(a), float(b), _native.ptr(res), current_stream_handle()),
            "pcf_pair_list")
        return res.cpu().numpy()


def coll_inv_host(coll):
    inv = np.empty(coll.M, dtype=np.int64)
    inv[coll.perm_host] = np.arange(coll.M, dtype=np.int64)
    return inv
