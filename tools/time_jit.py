"""Device timing of a JIT-compiled pairwise integrand vs the op-coded L1 kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_07183_b200 import datagen as dg  # noqa: E402
from paper_2404_07183_b200.collection import DeviceCollection  # noqa: E402
from paper_2404_07183_b200.combine import CombinationIntegral, fill_custom  # noqa: E402
from paper_2404_07183_b200.engine import fill_pairwise  # noqa: E402


def absdiff(x, y):
    return abs(x - y)


M = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
t, v, off = dg.synthetic_benchmark_packed(M, rng=dg.RngSpec(2404))
n = np.diff(off)
cells = (M - 1) * int(n.sum()) - M * (M - 1) // 2
coll = DeviceCollection(t, v, off)
out = torch.empty((M, M), dtype=torch.float64, device="cuda")
ci = CombinationIntegral(h=absdiff, symmetric=True)


def one_thread():
    os.environ["PCF_JIT_NO_TILES"] = "1"
    try:
        return fill_custom(coll, ci, out)
    finally:
        del os.environ["PCF_JIT_NO_TILES"]


for name, fn in (("op-coded L1 (K1)", lambda: fill_pairwise(coll, 0, 1.0, False, False, out=out)),
                 ("op-coded L1 exact", lambda: fill_pairwise(coll, 0, 1.0, False, False, out=out,
                                                             exact=True)),
                 ("JIT tiles", lambda: fill_custom(coll, ci, out, exact=False)),
                 ("JIT tiles exact", lambda: fill_custom(coll, ci, out, exact=True)),
                 ("JIT one thread", one_thread)):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    print(f"{name:20s} {ms:9.1f} ms  {cells / ms * 1e3:.3e} cells/s", flush=True)
