"""Reductions of PCF collections on the GPU: reduce_pair, tree_reduce, mean, variance,
std (API mirror of pkg/src/pcflib/reduce.py:31-238).

* ``tree_reduce`` / ``mean`` run the reference's exact tree -- level pairs (0,1)(2,3)...,
  an odd last node passing through (reduce.py:189-208) -- one device launch pair per
  level (K5 merge + compaction), with the same per-cell arithmetic and the same
  emission rule as reduce_pair (reduce.py:47-57).  The mean is therefore bit-identical
  to the reference's.
* ``variance`` / ``std`` use the parallel-moments combination (Chan et al.) on the same
  tree shape: each node carries (mean, M2) per cell, merged pointwise as a
  rectangle-iteration combination.  This is O(N log M) instead of the reference's
  O(M * |mean|) (reduce.py:231 builds (f_i - mean)^2 for every i), and matches it within
  floating-point tolerance (not bitwise); see DESIGN.md.

Arbitrary Python callables cannot run on the device; the associative ops the engine
implements are add, max, min and mul (given as ``operator.add``, ``max``, ``min``,
``operator.mul`` or their names).
"""

from __future__ import annotations

import math
import operator
import os
import threading

import numpy as np

from . import _native, errors
from .collection import current_stream_handle, require_cuda
from .core import Pcf

__all__ = ["reduce_pair", "tree_reduce", "mean", "variance", "std", "mean_many",
           "ReductionAccumulator",
           "DeviceLevel", "mean_packed", "std_packed"]

_OPS = {"add": 0, "max": 1, "min": 2, "mul": 3}


def _op_code(h):
    if isinstance(h, str):
        key = h
    elif h is operator.add or h is np.add:
        key = "add"
    elif h is max or h is np.maximum:
        key = "max"
    elif h is min or h is np.minimum:
        key = "min"
    elif h is operator.mul or h is np.multiply:
        key = "mul"
    else:
        key = None
    if key not in _OPS:
        raise NotImplementedError(
            f"combination map {h!r} has no device kernel; supported: add, max, min, mul")
    return _OPS[key]


def _torch():
    import torch

    return torch


class DeviceLevel:
    """Nodes of one tree level on the device: SoA times/values (+ optional M2 for the
    moments tree) with int64 node offsets."""

    def __init__(self, t, v, off, nnodes, ntot, is_f32, m2=None):
        self.t, self.v, self.off, self.m2 = t, v, off, m2
        self.nnodes, self.ntot, self.is_f32 = int(nnodes), int(ntot), bool(is_f32)

    @classmethod
    def from_packed(cls, tcat, vcat, off, device="cuda"):
        torch = require_cuda()
        tcat = np.ascontiguousarray(tcat)
        is_f32 = tcat.dtype == np.float32
        t = torch.from_numpy(tcat).to(device)
        v = torch.from_numpy(np.ascontiguousarray(vcat, dtype=tcat.dtype)).to(device)
        o = torch.from_numpy(np.ascontiguousarray(off, dtype=np.int64)).to(device)
        return cls(t, v, o, len(off) - 1, int(off[-1]), is_f32)

    @classmethod
    def from_pcfs(cls, collection, device="cuda"):
        from .datagen import pack_matrices

        coll = list(collection)
        kind = coll[0].dtype
        for f in coll:
            if f.dtype != kind:
                raise errors.MixedPrecision(f"cannot combine {kind.name} with {f.dtype.name}")
        return cls.from_packed(*pack_matrices([f.to_matrix() for f in coll], kind), device=device)

    def to_pcfs(self, values=None):
        """Host Pcf objects, one per node."""
        n = self.ntot  # buffers may be scratch capacity: copy only the live points
        t = self.t[:n].cpu().numpy()
        v = (self.v if values is None else values)[:n].cpu().numpy()
        off = self.off[: self.nnodes + 1].cpu().numpy()
        out = []
        for k in range(self.nnodes):
            mat = np.empty((off[k + 1] - off[k], 2), dtype=t.dtype)
            mat[:, 0] = t[off[k]:off[k + 1]]
            mat[:, 1] = v[off[k]:off[k + 1]]
            out.append(Pcf._wrap(mat))
        return out


def _pairing(seg_nodes):
    """(src, cnt, next_seg_nodes) for one level over fibres with seg_nodes nodes each."""
    seg_nodes = np.asarray(seg_nodes, dtype=np.int64)
    nxt = (seg_nodes + 1) // 2
    base = np.concatenate([[0], np.cumsum(seg_nodes)[:-1]])
    obase = np.concatenate([[0], np.cumsum(nxt)[:-1]])
    nout = int(nxt.sum())
    fib = np.repeat(np.arange(seg_nodes.shape[0]), nxt)
    local = np.arange(nout, dtype=np.int64) - obase[fib]
    src = base[fib] + 2 * local
    cnt = np.where(2 * local + 1 < seg_nodes[fib], 2, 1).astype(np.int32)
    return src, cnt, nxt


def _check_status(status, what):
    if int(status.item()) != 0:
        raise errors.NonFinite(f"{what} produced a non-finite value")


def _plan_levels(seg_nodes, leaves0=None, moments=False):
    """All levels' (src, cnt[, leaves]) for fibres of seg_nodes nodes (host, once)."""
    seg_nodes = np.asarray(seg_nodes, dtype=np.int64)
    leaves = None
    if moments:
        leaves = (np.asarray(leaves0, dtype=np.int64).copy() if leaves0 is not None
                  else np.ones(int(seg_nodes.sum()), dtype=np.int64))
    plan = []
    while (seg_nodes > 1).any():
        src, cnt, nxt = _pairing(seg_nodes)
        plan.append((src, cnt, leaves))
        if moments:
            merged = leaves[src].copy()
            two = cnt == 2
            merged[two] += leaves[src[two] + 1]
            leaves = merged
        seg_nodes = nxt
    return plan, leaves


_PLAN_CACHE = {}
_SCRATCH_TLS = threading.local()  # per thread: a tree's output lives here until consumed


def _scratch_dict():
    d = getattr(_SCRATCH_TLS, "bufs", None)
    if d is None:
        d = _SCRATCH_TLS.bufs = {}
    return d


def _in_scratch(x):
    if x is None:
        return False
    p = x.data_ptr()
    for buf in _scratch_dict().values():
        b = buf.data_ptr()
        if b <= p < b + buf.numel() * buf.element_size():
            return True
    return False


def _scratch(name, numel, dtype, dev):
    """A cached device buffer of at least `numel` elements (grow-only, per name / dtype /
    device); the caller uses the first `numel`.  Results never alias scratch: the tree's
    output level is copied out by _finalize / to_pcfs before the next tree runs."""
    torch = _torch()
    key = (name, dtype, str(dev))
    cache = _scratch_dict()
    buf = cache.get(key)
    if buf is None or buf.numel() < numel:
        cache.pop(key, None)
        buf = torch.empty(max(int(numel), 1), dtype=dtype, device=dev)
        cache[key] = buf
    return buf[:numel]


def _device_plan(seg_nodes, leaves0, moments, dev):
    """Host pairing plan + one device upload of every level's src / cnt (/ leaves),
    cached per tree shape (the plan depends only on the fibre sizes)."""
    torch = _torch()
    seg_nodes = np.asarray(seg_nodes, dtype=np.int64)
    key = None
    if leaves0 is None and seg_nodes.size <= 64:
        key = (tuple(int(x) for x in seg_nodes), bool(moments), str(dev))
        if key in _PLAN_CACHE:
            return _PLAN_CACHE[key]
    plan, leaves_final = _plan_levels(seg_nodes, leaves0, moments)
    src_d = cnt_d = lv_d = None
    if plan:
        src_d = torch.from_numpy(np.concatenate([p[0] for p in plan])).to(dev)
        cnt_d = torch.from_numpy(np.concatenate([p[1] for p in plan])).to(dev)
        if moments:
            lv_d = torch.from_numpy(np.concatenate([p[2] for p in plan])).to(dev)
    res = (plan, leaves_final, src_d, cnt_d, lv_d)
    if key is not None:
        if len(_PLAN_CACHE) > 16:
            _PLAN_CACHE.clear()
        _PLAN_CACHE[key] = res
    return res


_FUSED_CACHE = {}


def _fused_tables(plan, l0, l1, pkey, dev):
    """Node tables of levels [l0, l1) run as one fused pass: for every output node of level
    l1 - 1 the first input node of level l0 and the number of input nodes its subtree
    covers (the level pairings composed downwards; device int64 / int32 arrays)."""
    key = None if pkey is None else pkey + (l0, l1)
    if key is not None and key in _FUSED_CACHE:
        return _FUSED_CACHE[key]
    torch = _torch()
    src, cnt = plan[l1 - 1][0], plan[l1 - 1][1]
    first = np.asarray(src, dtype=np.int64)
    last = first + np.asarray(cnt, dtype=np.int64)
    for lvl in range(l1 - 2, l0 - 1, -1):
        s_, c_ = np.asarray(plan[lvl][0], dtype=np.int64), np.asarray(plan[lvl][1], dtype=np.int64)
        first, last = s_[first], s_[last - 1] + c_[last - 1]
    res = (torch.from_numpy(first).to(dev),
           torch.from_numpy((last - first).astype(np.int32)).to(dev))
    if key is not None:
        if len(_FUSED_CACHE) > 64:
            _FUSED_CACHE.clear()
        _FUSED_CACHE[key] = res
    return res


def _run_tree(level: DeviceLevel, seg_nodes, op=None, moments=False, leaves0=None):
    """Reduce each fibre (seg_nodes[i] consecutive nodes) to one node: one tiled level
    kernel per tree level -- compacting (pcf_tree_level) for level 0, and for the upper
    levels too unless level 0 kept >= 90% of its candidates, in which case they run as
    non-compacting merges (pcf_tree_merge_level; zero-width pieces are dropped by
    _finalize).  The pairing plan is uploaded once (cached per tree shape) and the levels
    run back to back; the only host synchronisation is the level-0 kept count in auto
    mode (each level's point count is read on the device; the host passes an upper bound).
    The returned level lives in cached scratch: consume or copy it before the next tree."""
    torch = _torch()
    lib = _native.load()
    dev = level.t.device
    st = current_stream_handle()
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    plan, leaves_final, src_d, cnt_d, lv_d = _device_plan(seg_nodes, leaves0, moments, dev)
    if not plan:
        return level, leaves_final
    if _in_scratch(level.t) or _in_scratch(level.v) or _in_scratch(level.m2):
        # the input is a previous tree's output (scratch): copy it out before reuse
        level = DeviceLevel(level.t.clone(), level.v.clone(), level.off.clone(), level.nnodes,
                            level.ntot, level.is_f32,
                            None if level.m2 is None else level.m2.clone())
    bound = max(level.ntot, 1)
    nb = _native.c_i64(0)
    lib.pcf_tree_level_workspace(bound, _native.ctypes.byref(nb))
    ws = _scratch("ws", max(nb.value, 256), torch.uint8, dev)
    kind = 4 if moments else int(op)
    # the level ping-pong buffers and the workspace come from a grow-only cache: a tree of
    # 1e8 points needs ~5 GB of scratch, and re-allocating it per call from a fragmented
    # caching allocator costs synchronising cudaFree/cudaMalloc rounds
    bufs = [(_scratch(f"t{k}", bound, level.t.dtype, dev),
             _scratch(f"v{k}", bound, level.v.dtype, dev),
             _scratch(f"m{k}", bound, torch.float64, dev) if moments else None)
            for k in range(2)]
    so = lo = 0
    cur_t, cur_v, cur_m2, cur_off = level.t, level.v, level.m2, level.off
    nout = level.nnodes
    mode = os.environ.get("PCF_TREE_MODE", "auto")  # auto | compact | merge
    merge = mode == "merge"
    # levels per fused pass (pcf_tree_merge_levels, K5w): 4 (c5 mean 26 -> 14.1 ms, c5 std
    # 26.5 -> 22.4 ms against one launch per level)
    fuse_env = os.environ.get("PCF_TREE_FUSE")
    fuse = max(1, min(4, int(fuse_env))) if fuse_env else 4
    pkey = (None if leaves0 is not None or np.asarray(seg_nodes).size > 64 else
            (tuple(int(x) for x in np.asarray(seg_nodes)), bool(moments), str(dev)))
    merge0 = False  # level 0 too runs non-compacting (fused with the levels above it, if any)
    if mode == "auto" and len(plan) > 1 and level.nnodes >= 2:
        # a sample of neighbouring leaf pairs: nearly distinct breakpoints mean compaction
        # would drop (almost) nothing, so every level can be a fused merge
        counts = _scratch("dup", 2, torch.int64, dev)
        _native.check(lib.pcf_tree_dup_sample(int(level.is_f32), _native.ptr(cur_t),
                                              _native.ptr(cur_off), level.nnodes,
                                              min(4096, level.nnodes // 2), _native.ptr(counts),
                                              st), "pcf_tree_dup_sample")
        dup, seen = (int(x) for x in counts.cpu())
        merge0 = merge = seen > 0 and dup <= 0.02 * seen
    elif mode == "merge":
        merge0 = True
    li = 0
    nbuf = 0
    while li < len(plan):
        src, cnt, _ = plan[li]
        if merge and (li > 0 or merge0) and fuse > 1 and len(plan) - li > 1:
            # several non-compacting levels in one pass (pcf_tree_merge_levels, K5w)
            g = min(fuse, len(plan) - li)
            nfirst, ncnt = _fused_tables(plan, li, li + g, pkey, dev)
            nout = int(plan[li + g - 1][0].shape[0])
            t_out, v_out, m2_out = bufs[nbuf % 2]
            off_out = torch.empty(nout + 1, dtype=torch.int64, device=dev)
            nbw = _native.c_i64(0)
            lib.pcf_tree_merge_levels_workspace(bound, nout, _native.ctypes.byref(nbw))
            wsw = _scratch("wsw", max(nbw.value, 256), torch.uint8, dev)
            _native.check(lib.pcf_tree_merge_levels(
                kind, int(level.is_f32), _native.ptr(cur_t), _native.ptr(cur_v),
                _native.ptr(cur_m2) if moments else None, _native.ptr(cur_off),
                _native.ptr(nfirst), _native.ptr(ncnt),
                _native.c_vp(lv_d.data_ptr() + 8 * lo) if moments else None,
                nout, g, bound, _native.ptr(t_out), _native.ptr(v_out),
                _native.ptr(m2_out) if moments else None, _native.ptr(off_out), _native.ptr(wsw),
                wsw.numel(), st), "pcf_tree_merge_levels")
            for k in range(g):
                so += plan[li + k][0].shape[0]
                if moments:
                    lo += plan[li + k][2].shape[0]
            cur_t, cur_v, cur_m2, cur_off = t_out, v_out, m2_out, off_out
            li += g
            nbuf += 1
            continue
        nout = src.shape[0]
        t_out, v_out, m2_out = bufs[nbuf % 2]
        off_out = torch.empty(nout + 1, dtype=torch.int64, device=dev)
        args = (int(level.is_f32), _native.ptr(cur_t), _native.ptr(cur_v),
                _native.ptr(cur_m2) if moments else None, _native.ptr(cur_off),
                _native.c_vp(src_d.data_ptr() + 8 * so), _native.c_vp(cnt_d.data_ptr() + 4 * so),
                _native.c_vp(lv_d.data_ptr() + 8 * lo) if moments else None,
                nout, bound, _native.ptr(t_out), _native.ptr(v_out),
                _native.ptr(m2_out) if moments else None, _native.ptr(off_out), _native.ptr(ws),
                ws.numel())
        if merge and (li > 0 or merge0):
            # non-compacting merge (zero-width pieces are dropped by _finalize)
            _native.check(lib.pcf_tree_merge_level(kind, *args, st), "pcf_tree_merge_level")
        else:
            _native.check(lib.pcf_tree_level(kind, *args, _native.ptr(status), st),
                          "pcf_tree_level")
        if li == 0 and len(plan) > 1 and mode == "auto" and not merge0:
            # nearly distinct breakpoints (compaction kept >= 90% of level 0): the upper
            # levels would drop almost nothing, so they run without compaction
            kept = int(off_out[-1].item())
            merge = kept >= 0.9 * level.ntot
        so += nout
        if moments:
            lo += plan[li][2].shape[0]
        cur_t, cur_v, cur_m2, cur_off = t_out, v_out, m2_out, off_out
        li += 1
        nbuf += 1
    ntot = int(cur_off[-1].item())
    if not moments:
        _check_status(status, "reduction")
    out = DeviceLevel(cur_t, cur_v, cur_off, nout, ntot, level.is_f32, cur_m2)
    return out, leaves_final


def _finalize(level: DeviceLevel, scales, kind, take_sqrt=False):
    """kind 'scale': T(v * T(scale)) + minimise; kind 'm2': T(M2*scale) [sqrt] + minimise.
    One pcf_finalize call (two tiled passes; zero-width pieces dropped first)."""
    torch = _torch()
    lib = _native.load()
    dev = level.t.device
    st = current_stream_handle()
    n = level.ntot
    tdt = torch.float32 if level.is_f32 else torch.float64
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    sc = torch.tensor(np.asarray(scales, dtype=np.float64), device=dev)
    nb = _native.c_i64(0)
    lib.pcf_finalize_workspace(n, _native.ctypes.byref(nb))
    ws = _scratch("fin", max(nb.value, 16), torch.uint8, dev)
    t_out = torch.empty(max(n, 1), dtype=level.t.dtype, device=dev)
    v_out = torch.empty(max(n, 1), dtype=tdt, device=dev)
    off_out = torch.empty(level.nnodes + 1, dtype=torch.int64, device=dev)
    code = 0 if kind == "scale" else (2 if take_sqrt else 1)
    src = level.v if kind == "scale" else level.m2
    _native.check(lib.pcf_finalize(code, int(level.is_f32), _native.ptr(src), _native.ptr(level.t),
                                   _native.ptr(level.off), level.nnodes, _native.ptr(sc), n,
                                   _native.ptr(t_out), _native.ptr(v_out), _native.ptr(off_out),
                                   _native.ptr(status), _native.ptr(ws), ws.numel(), st),
                  "pcf_finalize")
    _check_status(status, "scaling")
    return DeviceLevel(t_out, v_out, off_out, level.nnodes, int(off_out[-1].item()),
                       level.is_f32)


def _as_list(collection, what):
    coll = list(collection)
    if not coll:
        raise errors.EmptyCollection(f"{what} of an empty collection")
    return coll


# ------------------------------------------------------------------------ public API
def reduce_pair(f: Pcf, g: Pcf, h) -> Pcf:
    """The induced combination h_*(f, g), minimally discretised (reduce.py:31-63)."""
    if f.dtype != g.dtype:
        raise errors.MixedPrecision(f"cannot combine {f.dtype.name} with {g.dtype.name}")
    level, _ = _run_tree(DeviceLevel.from_pcfs([f, g]), [2], op=_op_code(h))
    return level.to_pcfs()[0]


def tree_reduce(collection, h) -> Pcf:
    """Fixed-shape binary tree fold (reduce.py:189-208); final minimise."""
    coll = _as_list(collection, "tree_reduce")
    level, _ = _run_tree(DeviceLevel.from_pcfs(coll), [len(coll)], op=_op_code(h))
    # the final minimise (reduce.py:208) = a scale by exactly 1 with change flags
    return _finalize(level, [1.0], "scale").to_pcfs()[0]


def mean_packed(level: DeviceLevel, seg_nodes=None):
    """Device-level mean(s): one per fibre of seg_nodes (default: all nodes one fibre)."""
    if seg_nodes is None:
        seg_nodes = [level.nnodes]
    seg_nodes = np.asarray(seg_nodes, dtype=np.int64)
    out, _ = _run_tree(level, seg_nodes, op=0)
    return _finalize(out, 1.0 / seg_nodes.astype(np.float64), "scale")


def mean(collection) -> Pcf:
    """(1/n) sum of the collection (reduce.py:211-217), bit-identical to the reference."""
    coll = _as_list(collection, "mean")
    return mean_packed(DeviceLevel.from_pcfs(coll)).to_pcfs()[0]


def mean_many(fibres):
    """Means of several independent collections in one batched device tree."""
    fibres = [list(f) for f in fibres]
    for f in fibres:
        if not f:
            raise errors.EmptyCollection("mean of an empty collection")
    flat = [g for f in fibres for g in f]
    level = DeviceLevel.from_pcfs(flat)
    return mean_packed(level, [len(f) for f in fibres]).to_pcfs()


def std_many(fibres, ddof=1, take_sqrt=True):
    """Stds (or variances) of several independent collections in one batched device
    moments tree (segmented by fibre, like mean_many)."""
    fibres = [list(f) for f in fibres]
    for f in fibres:
        if len(f) < 2:
            raise errors.InsufficientData("variance needs at least two PCFs")
    flat = [g for f in fibres for g in f]
    level = DeviceLevel.from_pcfs(flat)
    return std_packed(level, ddof, take_sqrt=take_sqrt,
                      seg_nodes=[len(f) for f in fibres]).to_pcfs()


def _moments_level(level: DeviceLevel):
    torch = _torch()
    m2 = torch.zeros(max(level.ntot, 1), dtype=torch.float64, device=level.t.device)
    mu = level.v.to(torch.float64)
    return DeviceLevel(level.t, mu, level.off, level.nnodes, level.ntot, level.is_f32, m2)


def std_packed(level: DeviceLevel, ddof=1, take_sqrt=True, seg_nodes=None):
    if seg_nodes is None:
        seg_nodes = [level.nnodes]
    seg_nodes = np.asarray(seg_nodes, dtype=np.int64)
    denom = seg_nodes - ddof
    if (denom == 0).any():
        raise ZeroDivisionError("float division by zero")
    if take_sqrt and (denom < 0).any():
        raise ValueError("math domain error")  # negative variance, as math.sqrt raises
    out, _ = _run_tree(_moments_level(level), seg_nodes, moments=True)
    return _finalize(out, 1.0 / denom.astype(np.float64), "m2", take_sqrt=take_sqrt)


def variance(collection, ddof=1) -> Pcf:
    """Pointwise sample variance (1/(n-ddof)) sum (f_i - mean)^2 (reduce.py:220-233)."""
    coll = list(collection)
    if len(coll) < 2:
        raise errors.InsufficientData("variance needs at least two PCFs")
    return std_packed(DeviceLevel.from_pcfs(coll), ddof, take_sqrt=False).to_pcfs()[0]


def std(collection, ddof=1) -> Pcf:
    """Pointwise sample standard deviation (reduce.py:236-238)."""
    coll = list(collection)
    if len(coll) < 2:
        raise errors.InsufficientData("variance needs at least two PCFs")
    return std_packed(DeviceLevel.from_pcfs(coll), ddof, take_sqrt=True).to_pcfs()[0]


class ReductionAccumulator:
    """Mutable PCF state for in-place associative folds (reduce.py:66-186), held on the
    device: ``combine(other)`` sets state <- state (op) other with reduce_pair's emission
    rule (one pcf_tree_level launch merging the two), so the state is always minimally
    discretised.  A fresh accumulator is the canonical zero PCF; the first combine
    replaces it by a minimised copy of ``other`` (correct for ops without an identity at
    0, and equal to 0 (+) f for addition).  ``capacity`` is accepted for API
    compatibility; device buffers are sized per combine."""

    def __init__(self, op, dtype=np.float64, capacity=16):
        self.op = op
        self._code = _op_code(op)
        self.dtype = np.dtype(dtype)
        if self.dtype not in (np.float32, np.float64):
            raise errors.MixedPrecision(f"unsupported PCF kind {self.dtype}")
        self._state = None  # DeviceLevel with one node, None = fresh zero PCF
        self._fresh = True

    @property
    def size(self):
        return 1 if self._state is None else self._state.ntot

    def _as_level(self, other):
        if isinstance(other, ReductionAccumulator):
            if other.dtype != self.dtype:
                raise errors.MixedPrecision(
                    f"cannot combine {self.dtype.name} with {other.dtype.name}")
            if other._state is not None:
                return other._state
            return DeviceLevel.from_pcfs([other.to_pcf()])
        if other.dtype != self.dtype:
            raise errors.MixedPrecision(
                f"cannot combine {self.dtype.name} with {other.dtype.name}")
        return DeviceLevel.from_pcfs([other])

    def combine(self, other) -> None:
        """state <- state (op) other, where other is a Pcf or another accumulator."""
        torch = _torch()
        lvl = self._as_level(other)
        if self._fresh:
            self._state = _finalize(lvl, [1.0], "scale")  # minimised copy (exact x1)
            self._fresh = False
            return
        st = self._state
        t = torch.cat([st.t[: st.ntot], lvl.t[: lvl.ntot]])
        v = torch.cat([st.v[: st.ntot], lvl.v[: lvl.ntot]])
        off = torch.tensor([0, st.ntot, st.ntot + lvl.ntot], dtype=torch.int64,
                           device=t.device)
        pair = DeviceLevel(t, v, off, 2, st.ntot + lvl.ntot, self.dtype == np.float32)
        out, _ = _run_tree(pair, [2], op=self._code)
        # the tree's output lives in shared scratch: the state keeps its own copy
        self._state = DeviceLevel(out.t[: out.ntot].clone(), out.v[: out.ntot].clone(),
                                  out.off.clone(), 1, out.ntot, out.is_f32)

    def to_pcf(self) -> Pcf:
        """Snapshot the state as an immutable Pcf."""
        if self._state is None:
            return Pcf._wrap(np.zeros((1, 2), dtype=self.dtype))
        return self._state.to_pcfs()[0]
