"""Fused tree levels vs level by level (PCF_TREE_FUSE=4 vs 1) on c5-shaped collections
of growing size: the t = 0 tie run at the top of the tree grows with M (GPU)."""
import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2404_07183_b200 import reduce as R
from paper_2404_07183_b200 import datagen as dg
for M in [3000, 10000, 30000, 60000, 100000]:
    _, mats = dg.noisy_trig_matrices((M,), 100, "sin", 0.1, dg.RngSpec(2404))
    t, v, off = dg.pack_matrices(mats)
    lvl = R.DeviceLevel.from_packed(t, v, off)
    res = {}
    for fz in ("1", "4"):
        os.environ["PCF_TREE_FUSE"] = fz
        out = R.mean_packed(lvl)  # finalised: fused and level-by-level trees differ only in
        res[fz] = (out.t[:out.ntot].cpu().numpy().copy(),  # which zero-width pieces exist
                   out.v[:out.ntot].cpu().numpy().copy())
    a, b = res["1"], res["4"]
    d = np.flatnonzero(a[0] != b[0])
    print(M, "same t", np.array_equal(a[0], b[0]), "same v", np.array_equal(a[1], b[1]),
          "nt diffs", d.size, d[:5], flush=True)
