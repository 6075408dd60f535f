"""Device timing of the pairwise fill on config-like collections (development aid; the
bench contract is bench.py / tools/bench_configs.py).

    python tools/time_cfg.py c1 c1x c2f64 c2f64x c2f32 c3:20000 c4:4000
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_07183_b200 import datagen as dg  # noqa: E402
from paper_2404_07183_b200.collection import DeviceCollection  # noqa: E402
from paper_2404_07183_b200.engine import decode_err, fill_pairwise  # noqa: E402


def case(name):
    key, _, m = name.partition(":")
    exact = key.endswith("x")
    key = key.rstrip("x")
    if key == "c1":
        mats, op, p, root, diag = dg.fixed_size_collection(int(m or 1000), 100), 0, 1.0, True, False
    elif key in ("c2f64", "c2f32"):
        dt = np.float32 if key == "c2f32" else np.float64
        mats = dg.fixed_size_collection(int(m or 10000), 200, dtype=dt)
        op, p, root, diag = 1, 0.0, False, True
    elif key == "c3":
        mats = dg.synthetic_benchmark(int(m or 20000), rng=dg.RngSpec(2404))
        mats = [f.to_matrix() for f in mats]
        op, p, root, diag = 0, 1.0, True, False
    elif key == "c4":
        mats, op, p, root, diag = dg.ecc_like_collection(int(m or 4000)), 0, 2.0, True, False
    else:
        raise SystemExit(f"unknown case {name}")
    return mats, op, p, root, diag, exact


for name in sys.argv[1:]:
    mats, op, p, root, diag, exact = case(name)
    t, v, off = dg.pack_matrices(mats)
    n = np.diff(off)
    M = len(n)
    cells = (M - 1) * int(n.sum()) - M * (M - 1) // 2
    coll = DeviceCollection(t, v, off)
    pl = coll.plan(exact=exact)
    host, smem = pl[1], pl[-1]
    modes = np.bincount(host[:, 6], minlength=3).tolist()
    g = np.bincount(host[:, 5], minlength=7).tolist()
    out = torch.empty((M, M), dtype=coll.out_torch_dtype, device="cuda")
    for _ in range(2):
        fill_pairwise(coll, op, p, root, diag, out=out, exact=exact)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    s.record()
    for _ in range(reps):
        _, err, _ = fill_pairwise(coll, op, p, root, diag, out=out, exact=exact)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    print(f"{name:10s} M={M} {ms:9.3f} ms  cells/s={cells / ms * 1e3:.3e} "
          f"items={len(host)} modes(K1g,K1,K1r)={modes} log2G={g} smem={smem} "
          f"err={decode_err(err, M)}", flush=True)
