"""Device-resident packed PCF collections (the engine's ``packed`` object).

Layout in HBM:

* ``recs``  float64[2*N]  -- N 16-byte records {t_next, v} in size-sorted order;
* ``soff``  int64[M+1]    -- record offsets of sorted PCF s;
* ``recsg`` / ``goff``    -- the K1 tile layout: the same records slot-interleaved in
  groups of GW sorted PCFs (record k of PCF s at goff[s/GW] + GW*k + s%GW), the layout K1
  stages its row blocks in; GW = 8 for float64 (16-byte records), 16 for float32
  collections, which K1 reads as 8-byte float32 records (``tile_recs``);
* ``perm``  int32[M]      -- sorted index -> original index;
* ``inv``   int32[M]      -- original index -> sorted index.

Built from the reference's pack() layout (tcat, vcat, off; _sweepkern.pyx:72-85): the
host computes the size sort (argsort of off deltas), the SoA arrays go to the device
once, and K3 (``pcf_pack_sorted``) writes the records.  float32 collections are widened
to float64 records (exact), which is how the reference computes anyway (all
arithmetic in 64-bit, pyx:38-41); results are rounded back to float32 at the end.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _native, errors

# the sm_100 opt-in dynamic shared-memory maximum (227 KB) less the tile kernels' static
# shared memory (csrc/pcf_internal.h kPlanSmemBudget); PCF_SMEM_BUDGET overrides (A/B)
_SMEM_BUDGET = int(os.environ.get("PCF_SMEM_BUDGET", str(227 * 1024 - 64)))
_MAX_COLS_PER_ITEM = int(os.environ.get("PCF_MAX_COLS", "2048"))  # columns per work item (A/B knob)


def _torch():
    import torch

    return torch


def require_cuda():
    torch = _torch()
    if not torch.cuda.is_available():
        raise errors.BackendUnavailable("no CUDA device: the B200 engine has no CPU fallback")
    return torch


def current_stream_handle():
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class DeviceCollection:
    """A packed, size-sorted collection resident on one GPU."""

    def __init__(self, tcat, vcat, off, device=None):
        torch = require_cuda()
        lib = _native.load()
        tcat = np.ascontiguousarray(tcat)
        vcat = np.ascontiguousarray(vcat)
        off = np.ascontiguousarray(off, dtype=np.int64)
        if tcat.dtype != vcat.dtype or tcat.dtype not in (np.float32, np.float64):
            raise errors.MixedPrecision("tcat/vcat must share float32 or float64")
        self.dtype = np.dtype(tcat.dtype)
        self.M = int(off.shape[0] - 1)
        if self.M < 1:
            raise errors.EmptyCollection("empty collection")
        self.device = torch.device(device if device is not None else "cuda")
        sizes = np.diff(off)
        perm = np.argsort(-sizes, kind="stable").astype(np.int32)
        ssizes = sizes[perm].astype(np.int64)
        soff = np.zeros(self.M + 1, dtype=np.int64)
        np.cumsum(ssizes, out=soff[1:])
        inv = np.empty(self.M, dtype=np.int32)
        inv[perm] = np.arange(self.M, dtype=np.int32)
        self.sizes_sorted = ssizes
        self.perm_host = perm
        self.n_points = int(soff[-1])
        # K1 tile layout: float64 -> 16-byte records, 8-row interleaved groups;
        # float32 -> 8-byte records, 16-row interleaved groups (half the shared-memory bytes)
        self.rec_bytes = 8 if self.dtype == np.float32 else 16
        gw = 128 // self.rec_bytes
        goff = np.zeros((self.M + gw - 1) // gw + 1, dtype=np.int64)
        goff[1:] = np.cumsum(gw * ssizes[0::gw])
        self.goff_host = goff
        with torch.cuda.device(self.device):
            dev = self.device
            t_d = torch.from_numpy(tcat).to(dev, non_blocking=False)
            v_d = torch.from_numpy(vcat).to(dev, non_blocking=False)
            off_d = torch.from_numpy(off).to(dev)
            self.perm = torch.from_numpy(perm).to(dev)
            self.inv = torch.from_numpy(inv).to(dev)
            self.soff = torch.from_numpy(soff).to(dev)
            self.recs = torch.empty(2 * max(self.n_points, 1), dtype=torch.float64, device=dev)
            self.goff = torch.from_numpy(goff).to(dev)
            st = current_stream_handle()
            if self.rec_bytes == 16:
                self.recsg = torch.empty(2 * max(int(goff[-1]), 1), dtype=torch.float64,
                                         device=dev)
                rc = lib.pcf_pack_sorted(
                    _native.ptr(t_d), _native.ptr(v_d), 0, _native.ptr(off_d),
                    _native.ptr(self.perm), _native.ptr(self.soff), self.M,
                    _native.ptr(self.recs), _native.ptr(self.goff), _native.ptr(self.recsg), st)
                _native.check(rc, "pcf_pack_sorted")
                self.tile_recs = self.recs
            else:
                rc = lib.pcf_pack_sorted(
                    _native.ptr(t_d), _native.ptr(v_d), 1, _native.ptr(off_d),
                    _native.ptr(self.perm), _native.ptr(self.soff), self.M,
                    _native.ptr(self.recs), None, None, st)
                _native.check(rc, "pcf_pack_sorted")
                # +2 records: column chunks are copied in whole 16-byte units
                self.tile_recs = torch.zeros(2 * (self.n_points + 2), dtype=torch.float32,
                                             device=dev)
                self.recsg = torch.empty(2 * max(int(goff[-1]), 1), dtype=torch.float32,
                                         device=dev)
                rc = lib.pcf_pack_sorted32(
                    _native.ptr(t_d), _native.ptr(v_d), _native.ptr(off_d),
                    _native.ptr(self.perm), _native.ptr(self.soff), self.M,
                    _native.ptr(self.tile_recs), _native.ptr(self.goff),
                    _native.ptr(self.recsg), st)
                _native.check(rc, "pcf_pack_sorted32")
            del t_d, v_d, off_d
        self._plans = {}

    @classmethod
    def from_pcfs(cls, collection, device=None):
        from .datagen import pack_matrices

        coll = list(collection)
        if not coll:
            raise errors.EmptyCollection("empty collection")
        dtype = coll[0].dtype
        for f in coll:
            if f.dtype != dtype:
                raise errors.MixedPrecision("collection mixes 32- and 64-bit PCFs")
        tcat, vcat, off = pack_matrices([f.to_matrix() for f in coll], dtype)
        return cls(tcat, vcat, off, device=device)

    # -- work plan ------------------------------------------------------------------
    def plan(self, exact=False, smem_budget=_SMEM_BUDGET, max_cols=_MAX_COLS_PER_ITEM):
        """Tile work items (cached): (items_dev, items_host, smem_bytes).

        exact=True restricts every pair to one lane (the reference's left-to-right
        sum, bitwise for p=1 and inner products); otherwise up to a warp per pair."""
        max_log2g = 0 if exact else 6
        key = (max_log2g, smem_budget, max_cols)
        rb = self.rec_bytes
        if key in self._plans:
            return self._plans[key]
        torch = _torch()
        lib = _native.load()
        sizes = np.ascontiguousarray(self.sizes_sorted, dtype=np.int64)
        n = ctypes.c_int64(0)
        smem = ctypes.c_int32(0)
        _native.check(lib.pcf_plan_pairwise(_native.ptr(sizes), self.M, smem_budget, max_cols,
                                            max_log2g, rb, None, 0, ctypes.byref(n),
                                            ctypes.byref(smem)),
                      "pcf_plan_pairwise")
        items = (_native.WorkItem * max(n.value, 1))()
        _native.check(lib.pcf_plan_pairwise(_native.ptr(sizes), self.M, smem_budget, max_cols,
                                            max_log2g, rb, ctypes.cast(items, ctypes.c_void_p),
                                            n.value,
                                            ctypes.byref(n), ctypes.byref(smem)),
                      "pcf_plan_pairwise")
        host = np.frombuffer(items, dtype=np.int32).reshape(-1, 8)[: n.value].copy()
        dev = torch.from_numpy(host.reshape(-1)).to(self.device)
        res = (dev, host, int(smem.value))
        self._plans[key] = res
        return res

    @property
    def out_torch_dtype(self):
        torch = _torch()
        return torch.float32 if self.dtype == np.float32 else torch.float64
