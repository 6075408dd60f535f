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
# include/pcf_b200.h PCF_OP_FAST_POW: the fast plan may evaluate L_p cells (p != 1) with
# d*d / d*d*|d| / CUDA pow; without it every cell uses the C library's pow bit for bit
OP_FAST_POW = 0x10


def op_code(op, exact):
    return int(op) | (OP_FAST_POW if (not exact and int(op) == OP_LP) else 0)

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
                  out=None, err=None, items=None, chunks=1, between_chunks=None, exact=False,
                  diagonal=True):
    """Write the full symmetric M x M matrix into `out` (device tensor, allocated if
    None).  Diagonal: <f,f> when `diag` (Gram), exact 0 otherwise; `diagonal=False`
    leaves it untouched (the sharded recipe: only rank 0 owns the diagonal, so a sum
    over the ranks' zero-initialised buffers stays exact).  Returns (out, err, stopped).  `items` = (items_dev, items_host, smem_bytes) or None for the
    collection's cached plan; `exact` selects the one-lane-per-pair plan.
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
            items_dev, host_items, smem = coll.plan(exact=exact)
        else:
            items_dev, host_items, smem = items
        st = current_stream_handle()
        out_f32 = int(out.dtype == torch.float32)
        ld = out.stride(0)
        if diagonal:
            _native.check(lib.pcf_fill_diagonal(
                _native.ptr(coll.recs), _native.ptr(coll.soff), _native.ptr(coll.perm), M,
                int(bool(diag)), float(a), float(b), _native.ptr(out), out_f32, ld,
                _native.ptr(err), st), "pcf_fill_diagonal")
        counter = torch.zeros(1, dtype=torch.int32, device=dev)
        segs = []
        for base, end, mode in mode_runs(host_items):
            count = end - base
            k = max(1, min(int(chunks), count))
            bounds = [base + (count * i) // k for i in range(k + 1)]
            segs += [(bounds[i], bounds[i + 1], mode) for i in range(k) if bounds[i + 1] > bounds[i]]
        nseg = len(segs)
        events = []
        for idx, (s0, s1, mode) in enumerate(segs):
            ptr_items = _native.ptr(items_dev) if s0 == 0 else \
                _native.c_vp(items_dev.data_ptr() + s0 * 32)
            _native.check(lib.pcf_fill_matrix(
                _native.ptr(coll.tile_recs), _native.ptr(coll.recsg), _native.ptr(coll.soff),
                _native.ptr(coll.goff), _native.ptr(coll.perm), M,
                ptr_items, s1 - s0, smem, mode, coll.rec_bytes, _native.ptr(counter),
                op_code(op, exact), float(p),
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


def mode_runs(host_items):
    """Contiguous runs (lo, hi, smem_mode) of the plan: one kernel launch per run
    (the planner emits K1 items, then K1r, then K1g, each run cost-sorted)."""
    modes = np.asarray(host_items, dtype=np.int32).reshape(-1, 8)[:, 6]
    runs, lo = [], 0
    for i in range(1, modes.shape[0] + 1):
        if i == modes.shape[0] or modes[i] != modes[lo]:
            runs.append((lo, i, int(modes[lo])))
            lo = i
    return runs


def partition_items(host_items, world, rank):
    """Static cost-balanced split of the work queue over `world` GPUs.

    Items are cost-sorted (LPT order) within each kernel's run; each run is dealt out in
    snake order (0..W-1, W-1..0, ...), which keeps every rank's share cost-sorted and
    balanced to within one item.  Every pair is owned by exactly one rank, so results
    are identical for any world size.  Returns the rank's items (same run order)."""
    if world <= 1:
        return host_items
    out = []
    for lo, hi, _ in mode_runs(host_items):
        idx = np.arange(lo, hi)
        k = idx - lo
        cyc = k % (2 * world)
        owner = np.where(cyc < world, cyc, 2 * world - 1 - cyc)
        out.append(host_items[idx[owner == rank]])
    if not out:
        return host_items[:0]
    return np.concatenate(out, axis=0)


def items_to_device(host_items, device):
    torch = _torch()
    flat = np.ascontiguousarray(host_items, dtype=np.int32).reshape(-1)
    if flat.size == 0:
        flat = np.zeros(8, dtype=np.int32)
    return torch.from_numpy(flat).to(device)


def item_cells(host_items, sizes_sorted):
    """Exact cell count of the pairs covered by the items: a pair (r, c) has
    (n_r - 1) + (n_c - 1) finite steps plus the tail cell = n_r + n_c - 1 cells."""
    if host_items.shape[0] == 0:
        return 0
    sizes = np.asarray(sizes_sorted, dtype=np.int64)
    S = np.concatenate([[0], np.cumsum(sizes)])
    it = np.asarray(host_items, dtype=np.int64)
    rmax = int(it[:, 1].max())
    r = it[:, 0:1] + np.arange(rmax)[None, :]
    valid = np.arange(rmax)[None, :] < it[:, 1:2]
    r = np.where(valid, r, 0)
    c0 = np.maximum(it[:, 2:3], r + 1)
    c1 = it[:, 3:4]
    ncol = np.where(valid & (c1 > c0), c1 - c0, 0)
    colsum = np.where(ncol > 0, S[c1.repeat(rmax, 1)] - S[np.minimum(c0, c1)], 0)
    return int((ncol * (sizes[r] - 1) + colsum).sum())


def matrix_host(tcat, vcat, off, op, p, apply_root, diag, a=0.0, b=math.inf, exact=False,
                n_chunks=32, out=None, stream=None):
    """Whole matrix through the host-buffer C-ABI call ``pcf_matrix_host`` (MatrixJob.run
    over the compiled module, matrix.py:156-234, in one call): host SoA in, dense host
    M x M out (original order), device chunks drained to the host while later chunks
    compute.  `out` may be a preallocated (pinned) numpy array or torch CPU tensor;
    `stream`: a cudaStream_t handle for the compute (None: the library's own).
    Returns (out, err) with err None or the first non-finite pair (i, j)."""
    lib = _native.load()
    tcat = np.ascontiguousarray(tcat)
    vcat = np.ascontiguousarray(vcat)
    off = np.ascontiguousarray(off, dtype=np.int64)
    M = int(off.shape[0] - 1)
    f32 = tcat.dtype == np.float32
    if out is None:
        out = np.empty((M, M), dtype=np.float32 if f32 else np.float64)
    ld = out.stride(0) if hasattr(out, "stride") and callable(out.stride) else \
        out.strides[0] // out.itemsize
    import ctypes

    ei, ej = ctypes.c_int64(-1), ctypes.c_int64(-1)
    _native.check(lib.pcf_matrix_host(
        _native.ptr(tcat), _native.ptr(vcat), int(f32), _native.ptr(off), M,
        op_code(op, exact), float(p),
        int(bool(apply_root)), int(bool(diag)), float(a), float(b), 0 if exact else 6,
        int(n_chunks), _native.ptr(out), int(ld), ctypes.byref(ei), ctypes.byref(ej), stream),
        "pcf_matrix_host")
    err = None if ei.value < 0 else (int(ei.value), int(ej.value))
    return out, err
