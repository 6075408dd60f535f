"""pcf_matrix_host timing on the c3 workload (development aid): host-buffer whole matrix,
pinned in/out, for several chunk counts."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PCF_HOST_TIMING"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_07183_b200 import datagen as dg  # noqa: E402
from paper_2404_07183_b200.engine import matrix_host  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
chunks = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1", "32"])]
t, v, off = dg.synthetic_benchmark_packed(M, rng=dg.RngSpec(2404))
ht = torch.from_numpy(t).pin_memory()
hv = torch.from_numpy(v).pin_memory()
ho = torch.from_numpy(off).pin_memory()
# PCF_E2E_PAGEABLE=1: a plain numpy result (rows through pcf_matrix_host's staging pool)
if os.environ.get("PCF_E2E_PAGEABLE"):
    out = np.empty((M, M), dtype=np.float64)
else:
    out = torch.empty((M, M), dtype=torch.float64, pin_memory=True)
for nc in chunks:
    for rep in range(2):
        t0 = time.perf_counter()
        matrix_host(ht.numpy(), hv.numpy(), ho.numpy(), 0, 1.0, True, False, n_chunks=nc, out=out)
        if rep == 0 and os.environ.get("PCF_E2E_PAGEABLE"):
            print("  (first call: includes first-touch page faults of the result)", flush=True)
        print(f"chunks={nc} rep={rep} wall {time.perf_counter() - t0:.3f} s", flush=True)
