"""CPU oracle for the B200 engine -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this module, and only as the checker or the CPU baseline.  The product path
(paper_2404_07183_b200) never imports it.

Three layers:

1. ``Oracle`` -- ctypes wrapper of oracle/_build/libpcforacle.so, a C restatement of the
   reference kernel module (pcf_oracle.c restates _sweepkern.pyx:24-59 and 88-121).
2. ``load_reference_kernel()`` -- the reference's own _sweepkern.pyx compiled from its
   source into oracle/_ref/ (oracle/Makefile ``ref``), when present.
3. Pure-Python restatements of the reduction path (reduce_pair, tree_reduce, mean,
   variance, std; pkg/src/pcflib/reduce.py:31-63, 189-238 and core.py:165-214), for the
   small sizes the tests use.

Parity is pinned: tests/test_oracle.py checks 1 and 3 against golden vectors produced by
the reference itself (tests/golden/make_golden.py) and 1 against 2 bit for bit.
"""

from __future__ import annotations

import ctypes
import importlib.machinery
import importlib.util
import math
import os
import subprocess
import sysconfig

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libpcforacle.so")
REF_SO = os.path.join(HERE, "_ref", "_sweepkern" + sysconfig.get_config_var("EXT_SUFFIX"))

OP_LP = 0
OP_INNER = 1


def build(ref=True):
    """make -C oracle [ref]; the ref target needs /root/reference (this container)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref and os.path.exists("/root/reference/pkg/src/pcflib/_sweepkern.pyx"):
        subprocess.run(["make", "-s", "-C", HERE, "ref", "refpkg"], check=True)


class Oracle:
    """C restatement of the reference kernel module."""

    def __init__(self):
        if not os.path.exists(LIB):
            build(ref=False)
        lib = ctypes.CDLL(LIB)
        d, i64, vp, ci = ctypes.c_double, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
        lib.pcf_oracle_accumulate.restype = d
        lib.pcf_oracle_accumulate.argtypes = [vp, vp, i64, vp, vp, i64, d, d, ci, d]
        lib.pcf_oracle_fill_block.restype = ci
        lib.pcf_oracle_fill_block.argtypes = [vp, vp, vp, i64, i64, i64, ci, d, ci, ci, d, d, vp,
                                              i64, ctypes.POINTER(i64), ctypes.POINTER(i64)]
        lib.pcf_oracle_row.restype = ci
        lib.pcf_oracle_row.argtypes = [vp, vp, vp, i64, i64, ci, d, ci, d, d, vp]
        lib.pcf_oracle_rows_threaded.restype = d
        lib.pcf_oracle_rows_threaded.argtypes = [vp, vp, vp, i64, vp, i64, ci, d, ci, ci]
        self.lib = lib

    @staticmethod
    def _p(a):
        return ctypes.c_void_p(a.ctypes.data)

    def accumulate(self, f, g, a=0.0, b=math.inf, op=OP_LP, p=1.0):
        """Raw integral of two (n, 2) row arrays; +-inf on divergence (pyx:24-59)."""
        f = np.asarray(f, dtype=np.float64)
        g = np.asarray(g, dtype=np.float64)
        ft, fv = np.ascontiguousarray(f[:, 0]), np.ascontiguousarray(f[:, 1])
        gt, gv = np.ascontiguousarray(g[:, 0]), np.ascontiguousarray(g[:, 1])
        return self.lib.pcf_oracle_accumulate(self._p(ft), self._p(fv), ft.shape[0], self._p(gt),
                                              self._p(gv), gt.shape[0], float(a), float(b),
                                              int(op), float(p))

    def matrix(self, tcat, vcat, off, op=OP_LP, p=1.0, apply_root=True, diag=False, a=0.0,
               b=math.inf, out_dtype=np.float64):
        """Whole matrix via fill_block(0, M) (pyx:88-121).  Returns (out, err_pair)."""
        tcat = np.ascontiguousarray(tcat, dtype=np.float64)
        vcat = np.ascontiguousarray(vcat, dtype=np.float64)
        off = np.ascontiguousarray(off, dtype=np.int64)
        M = off.shape[0] - 1
        out = np.zeros((M, M), dtype=np.float64)
        ei, ej = ctypes.c_int64(-1), ctypes.c_int64(-1)
        bad = self.lib.pcf_oracle_fill_block(self._p(tcat), self._p(vcat), self._p(off), M, 0, M,
                                             int(op), float(p), int(apply_root), int(diag),
                                             float(a), float(b), self._p(out), M,
                                             ctypes.byref(ei), ctypes.byref(ej))
        # the reference stores (floating)acc into a T-typed matrix: round once
        return out.astype(out_dtype), ((ei.value, ej.value) if bad else None)

    def row(self, tcat, vcat, off, i, op=OP_LP, p=1.0, apply_root=True, a=0.0, b=math.inf):
        """Entries D[i, j] for j > i (O(M) memory row sample) on [a, b)."""
        M = off.shape[0] - 1
        row = np.zeros(M, dtype=np.float64)
        self.lib.pcf_oracle_row(self._p(tcat), self._p(vcat), self._p(off), M, int(i), int(op),
                                float(p), int(apply_root), float(a), float(b), self._p(row))
        return row

    def rows_threaded(self, tcat, vcat, off, rows, op=OP_LP, p=1.0, apply_root=True,
                      threads=1):
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        return self.lib.pcf_oracle_rows_threaded(self._p(tcat), self._p(vcat), self._p(off),
                                                 off.shape[0] - 1, self._p(rows), rows.shape[0],
                                                 int(op), float(p), int(apply_root), int(threads))


def load_reference_kernel():
    """The reference's compiled _sweepkern (built from its own .pyx), or None."""
    if not os.path.exists(REF_SO):
        return None
    loader = importlib.machinery.ExtensionFileLoader("_sweepkern", REF_SO)
    spec = importlib.util.spec_from_file_location("_sweepkern", REF_SO, loader=loader)
    mod = importlib.util.module_from_spec(spec)
    loader.exec_module(mod)
    return mod


# ---------------------------------------------------------------- reduction restatement
def _cells(f, g):
    """Cells (left edge, v_f, v_g) of the common refinement on [0, inf); simultaneous
    jumps advance both cursors (sweep.py:67-100)."""
    ft, fv = f[:, 0].tolist(), f[:, 1].tolist()
    gt, gv = g[:, 0].tolist(), g[:, 1].tolist()
    k = m = 0
    t = 0.0
    out = []
    while True:
        out.append((t, fv[k], gv[m]))
        tnf = ft[k + 1] if k + 1 < len(ft) else math.inf
        tng = gt[m + 1] if m + 1 < len(gt) else math.inf
        tn = tnf if tnf < tng else tng
        if tn == math.inf:
            return out
        if tnf == tn:
            k += 1
        if tng == tn:
            m += 1
        t = tn


def reduce_pair(f, g, h, dtype=np.float64):
    """reduce.py:31-63: emit (l, v) where v = h(v_f, v_g) (float64, cast to float32 for
    float32 PCFs) differs from the last emitted value."""
    ts, vs = [], []
    for l, a, b in _cells(f, g):
        v = float(h(a, b))
        if dtype == np.float32:
            v = float(np.float32(v))
        if not math.isfinite(v):
            raise ArithmeticError("non-finite")
        if not vs or v != vs[-1]:
            ts.append(l)
            vs.append(v)
    out = np.empty((len(ts), 2), dtype=dtype)
    out[:, 0] = ts
    out[:, 1] = vs
    return out


def minimize(f):
    """core.py:189-203"""
    if f.shape[0] == 1:
        return f
    keep = np.ones(f.shape[0], dtype=bool)
    keep[1:] = f[1:, 1] != f[:-1, 1]
    return np.ascontiguousarray(f[keep])


def tree_reduce(mats, h, dtype=np.float64):
    """reduce.py:189-208: level pairs (0,1)(2,3)...; odd last passes through."""
    level = list(mats)
    if len(level) == 1:
        return minimize(level[0])
    while len(level) > 1:
        nxt = [reduce_pair(level[i], level[i + 1], h, dtype) for i in range(0, len(level) - 1, 2)]
        if len(level) % 2:
            nxt.append(level[-1])
        level = nxt
    return minimize(level[0])


def scale(f, a, dtype=np.float64):
    """core.py:165-178 (multiply by T(a) in T arithmetic)."""
    if a == 0.0:
        return np.zeros((1, 2), dtype=dtype)
    out = f.copy()
    out[:, 1] = f[:, 1] * np.dtype(dtype).type(a)
    return out


def mean(mats, dtype=np.float64):
    """reduce.py:211-217"""
    total = tree_reduce(mats, lambda x, y: x + y, dtype)
    return minimize(scale(total, 1.0 / len(mats), dtype))


def variance(mats, ddof=1, dtype=np.float64):
    """reduce.py:220-233 (O(M * |mean|): small collections only)."""
    n = len(mats)
    fbar = mean(mats, dtype)
    sq = [reduce_pair(f, fbar, lambda x, y: (x - y) * (x - y), dtype) for f in mats]
    total = tree_reduce(sq, lambda x, y: x + y, dtype)
    return minimize(scale(total, 1.0 / (n - ddof), dtype))


def std(mats, ddof=1, dtype=np.float64):
    """reduce.py:236-238 with core.apply_unary(math.sqrt)."""
    v = variance(mats, ddof, dtype)
    out = v.copy()
    out[:, 1] = [float(math.sqrt(x)) for x in v[:, 1].tolist()]
    return minimize(out)


def evaluate(f, t):
    k = int(np.searchsorted(f[:, 0], t, side="right")) - 1
    return float(f[k, 1])
