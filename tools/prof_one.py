"""One pdist fill for profiling (ncu -k regex:k_fill_tiles)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2404_07183_b200 import datagen as dg
from paper_2404_07183_b200.collection import DeviceCollection
from paper_2404_07183_b200.engine import fill_pairwise
M = int(sys.argv[1]) if len(sys.argv) > 1 else 6000
exact = len(sys.argv) > 2 and sys.argv[2] == "exact"
t, v, off = dg.synthetic_benchmark_packed(M, rng=dg.RngSpec(2404))
coll = DeviceCollection(t, v, off)
for _ in range(2):
    fill_pairwise(coll, 0, 1.0, True, False, exact=exact)
torch.cuda.synchronize()
