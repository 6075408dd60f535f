"""Single fills of config-like collections for ncu (c2 f32/f64 Gram, c4 ECC L2)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2404_07183_b200 import datagen as dg
from paper_2404_07183_b200.collection import DeviceCollection
from paper_2404_07183_b200.engine import fill_pairwise
which = sys.argv[1]
M = int(sys.argv[2]) if len(sys.argv) > 2 else 4000
if which in ("c2f32", "c2f64"):
    dt = np.float32 if which == "c2f32" else np.float64
    t, v, off = dg.pack_matrices(dg.fixed_size_collection(M, 200, dtype=dt))
    op, p, root, diag = 1, 0.0, False, True
else:
    t, v, off = dg.pack_matrices(dg.ecc_like_collection(M))
    op, p, root, diag = 0, 2.0, True, False
coll = DeviceCollection(t, v, off)
for _ in range(2):
    fill_pairwise(coll, op, p, root, diag)
torch.cuda.synchronize()
