"""One fast-plan JIT tile fill (h = |x - y|, App-A M PCFs) for an ncu capture of the
NVRTC-compiled K1 (HK = H_USER)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2404_07183_b200 import datagen as dg  # noqa: E402
from paper_2404_07183_b200.collection import DeviceCollection  # noqa: E402
from paper_2404_07183_b200.combine import CombinationIntegral, fill_custom  # noqa: E402


def absdiff(x, y):
    return abs(x - y)


M = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
t, v, off = dg.synthetic_benchmark_packed(M, rng=dg.RngSpec(2404))
coll = DeviceCollection(t, v, off)
out = torch.empty((M, M), dtype=torch.float64, device="cuda")
fill_custom(coll, CombinationIntegral(h=absdiff, symmetric=True), out, exact=False)
torch.cuda.synchronize()
