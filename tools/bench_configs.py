"""Secondary configurations of BASELINE.json (parity + device timing + CPU reference
beside), one JSON line each.  bench.py carries the headline (c3) contract; this covers

  c1  L1 distance matrix, 1,000 PCFs x 100 breakpoints, float64 (full CPU reference run)
  c2  L2 Gram matrix, 10,000 PCFs x 200 breakpoints, float64 and float32
  c4  L_p (p = 2, 3) distance matrix, 10,000 heavy-tailed PCFs (10..10,000 breakpoints)
  c5  mean / std of 1,000,000 noisy-sine PCFs (101 points each)

    python tools/bench_configs.py [c1 c2 c4 c5] [--quick]

Parity is checked in every run (bitwise where the design promises it, else the north-star
tolerance); the CPU reference is the reference's compiled kernel (oracle/_ref) for the
matrices and the Python restatement of reduce.py (oracle/oracle.py) for the reductions.
"""

from __future__ import annotations

import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import torch  # noqa: E402

import oracle as O  # noqa: E402
from paper_2404_07183_b200 import datagen as dg  # noqa: E402
from paper_2404_07183_b200.collection import DeviceCollection  # noqa: E402
from paper_2404_07183_b200.engine import decode_err, fill_pairwise, item_cells  # noqa: E402

QUICK = "--quick" in sys.argv


def dev_time(fn, reps=3):
    fn()
    fn()  # second warm-up: first-call allocations and plan caching settle
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    out = None
    for _ in range(reps):
        out = None  # the previous result is released before the next call allocates
        out = fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, out


def cpu_rows(t, v, off, rows, op, p, root, diag=False, threads=None):
    """Reference kernel (oracle/_ref) on the given rows, all threads; returns
    (values per row dict, seconds)."""
    import threading

    from numpy.lib.stride_tricks import as_strided

    K = O.load_reference_kernel()
    t64 = np.ascontiguousarray(t, dtype=t.dtype)
    packed = (t64, np.ascontiguousarray(v), np.ascontiguousarray(off))
    M = off.shape[0] - 1
    threads = threads or os.cpu_count()
    res = {}
    lock = threading.Lock()
    todo = list(rows)

    def work():
        buf = np.zeros(M, dtype=t.dtype)
        sink = as_strided(buf, shape=(M, M), strides=(0, buf.itemsize))
        while True:
            with lock:
                if not todo:
                    return
                i = todo.pop()
            K.fill_block(packed, i, i + 1, op, p, root, diag, 0.0, math.inf, sink)
            with lock:
                res[i] = buf.copy()

    t0 = time.perf_counter()
    ths = [threading.Thread(target=work) for _ in range(threads)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    return res, time.perf_counter() - t0


def rel(x, ref):
    return float(np.max(np.abs(x.astype(np.float64) - ref) /
                        np.maximum(np.abs(ref.astype(np.float64)), 1e-300)))


def matrix_case(name, t, v, off, op, p, root, diag, exact_ok, tol, sample_rows):
    M = off.shape[0] - 1
    n = np.diff(off)
    pairs = M * (M + 1) // 2 if diag else M * (M - 1) // 2
    coll = DeviceCollection(t, v, off)
    res = {"config": name, "M": M, "pairs": pairs}
    # one output buffer for every timed call: a fresh M x M allocation inside the timed
    # region would time the allocator, not the kernels
    buf = torch.empty((M, M), dtype=coll.out_torch_dtype, device=coll.device)
    for exact in ([False, True] if exact_ok else [False]):
        ms, (out, err, _) = dev_time(lambda: fill_pairwise(coll, op, p, root, diag, out=buf,
                                                           exact=exact))
        D = out.cpu().numpy()
        key = "exact" if exact else "fast"
        res[key] = {"ms": ms, "pairs_per_s": pairs / ms * 1e3, "err": decode_err(err, M)}
        res[key]["cells_per_s"] = ((M - 1) * int(n.sum()) - M * (M - 1) // 2
                                   + (int(n.sum()) if diag else 0)) / ms * 1e3
        rows = sample_rows
        vals, secs = cpu_rows(t, v, off, rows, op, p, root, diag)
        worst = 0.0
        bitwise = True
        for i in rows:
            # the aliasing row sink also receives the mirrored writes: its slot i (the
            # diagonal) is overwritten, so rows are compared strictly above the diagonal
            j0 = i + 1
            got = D[i, j0:]
            ref = vals[i][j0:]
            if op == 1 and not exact:
                K = np.sqrt(np.abs(np.diag(D).astype(np.float64)))
                worst = max(worst, float(np.max(np.abs(got - ref) /
                                                np.maximum(K[i] * K[j0:], 1e-300))))
            else:
                worst = max(worst, rel(got, ref))
            bitwise &= bool(np.array_equal(got, ref))
        res[key]["parity"] = {"rows_checked": len(rows), "max_rel": worst, "bitwise": bitwise,
                              "tol": tol, "ok": bool(bitwise or worst < tol)}
        cpu_pairs = sum(M - (i if diag else i + 1) for i in rows)
        res["cpu_reference"] = {"pairs_per_s": cpu_pairs / secs, "cores": os.cpu_count(),
                                "kind": "reference" if O.load_reference_kernel() else "port",
                                "sample_rows": len(rows), "seconds": secs}
    print(json.dumps(res), flush=True)
    return res


def c1():
    mats = dg.fixed_size_collection(1000, 100)
    t, v, off = dg.pack_matrices(mats)
    matrix_case("c1: L1 distance, 1000 PCFs x 100 bps, f64", t, v, off, 0, 1.0, True, False,
                True, 1e-12, list(range(999)))


def c2():
    M = 2000 if QUICK else 10000
    for dt in (np.float64, np.float32):
        t, v, off = dg.pack_matrices(dg.fixed_size_collection(M, 200, dtype=dt))
        rows = list(np.linspace(0, M - 2, 24).astype(int))
        matrix_case(f"c2: L2 Gram, {M} PCFs x 200 bps, {np.dtype(dt).name}", t, v, off, 1, 0.0,
                    False, True, True, 1e-12 if dt == np.float64 else 1e-5, rows)


def c4():
    M = 2000 if QUICK else 10000
    t, v, off = dg.pack_matrices(dg.ecc_like_collection(M))
    rows = list(np.linspace(0, M - 2, 12).astype(int))
    for p in (2.0, 3.0):
        matrix_case(f"c4: L{p:g} distance, {M} heavy-tailed PCFs (10..10^4 bps), f64", t, v,
                    off, 0, p, True, False, False, 1e-12, rows)


def c5():
    from paper_2404_07183_b200.reduce import DeviceLevel, mean_packed, std_packed

    M = 100000 if QUICK else 1000000
    shape, mats = dg.noisy_trig_matrices((M,), 100, "sin", 0.1, dg.RngSpec(2404))
    t, v, off = dg.pack_matrices(mats)
    N = int(off[-1])
    lvl = DeviceLevel.from_packed(t, v, off)
    ms_mean, m = dev_time(lambda: mean_packed(lvl), reps=2)
    ms_std, s = dev_time(lambda: std_packed(lvl), reps=2)
    levels = math.ceil(math.log2(M))
    algo_bytes = 2 * 16 * N * levels  # read + write (t, v) per level, float64
    # parity: pointwise at probe times vs brute force over all M PCFs (vectorised)
    K = 48
    probes = np.sort(np.random.default_rng(0).uniform(0, 1, K))
    vals = np.empty((M, K))
    starts = off[:-1]
    for k, pr in enumerate(probes):  # exact: count breakpoints <= probe per PCF
        cnt = np.add.reduceat((t <= pr).astype(np.int64), starts)
        vals[:, k] = v[starts + cnt - 1]
    mu = vals.sum(0) / M
    sd = np.sqrt(((vals - vals.mean(0)) ** 2).sum(0) / (M - 1))
    mt, mv = m.t.cpu().numpy()[: m.ntot], m.v.cpu().numpy()[: m.ntot]
    st_, sv = s.t.cpu().numpy()[: s.ntot], s.v.cpu().numpy()[: s.ntot]
    gm = mv[np.searchsorted(mt, probes, side="right") - 1]
    gs = sv[np.searchsorted(st_, probes, side="right") - 1]
    # CPU reference (Python restatement of reduce.mean) on a bounded sample
    Ms = 2048 if QUICK else 8192
    t0 = time.perf_counter()
    O.mean(mats[:Ms])
    cpu_s = time.perf_counter() - t0
    pts_levels = sum(m_.shape[0] for m_ in mats[:Ms]) * math.ceil(math.log2(Ms))
    res = {
        "config": f"c5: mean/std of {M} noisy-sine PCFs (101 pts), f64", "M": M, "points": N,
        "mean_ms": ms_mean, "std_ms": ms_std,
        "mean_points_levels_per_s": N * levels / ms_mean * 1e3,
        "mean_hbm_gbs_algorithmic": algo_bytes / ms_mean * 1e-6,
        "mean_points_out": m.ntot, "std_points_out": s.ntot,
        "parity": {"probes": K, "mean_max_abs": float(np.max(np.abs(gm - mu))),
                   "mean_max_rel": float(np.max(np.abs(gm - mu) / np.abs(mu))),
                   "std_max_rel": float(np.max(np.abs(gs - sd) / sd))},
        "cpu_reference": {"kind": "port (oracle/oracle.py restates reduce.py in Python)",
                          "sample_pcfs": Ms, "seconds": cpu_s,
                          "points_levels_per_s": pts_levels / cpu_s, "cores": 1},
    }
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    which = [a for a in sys.argv[1:] if not a.startswith("--")] or ["c1", "c2", "c4", "c5"]
    for w in which:
        torch.cuda.empty_cache()  # each config starts from a clean caching allocator
        globals()[w]()
