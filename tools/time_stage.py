"""pcf_matrix_host staging-pool A/B on the c3 workload (development aid): pageable numpy
result, PCF_STAGE_WORKERS / PCF_STAGE_SLOTS / PCF_STAGE_MB per configuration."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PCF_HOST_TIMING"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_07183_b200 import datagen as dg  # noqa: E402
from paper_2404_07183_b200.engine import matrix_host  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
cfgs = sys.argv[2:] or ["8,8,128", "16,8,128", "16,16,64", "16,16,128"]
t, v, off = dg.synthetic_benchmark_packed(M, rng=dg.RngSpec(2404))
ht = torch.from_numpy(t).pin_memory()
hv = torch.from_numpy(v).pin_memory()
ho = torch.from_numpy(off).pin_memory()
out = np.empty((M, M), dtype=np.float64)
matrix_host(ht.numpy(), hv.numpy(), ho.numpy(), 0, 1.0, True, False, n_chunks=32, out=out)
for rep in range(2):
    for c in cfgs:
        w, s, mb = c.split(",")
        os.environ["PCF_STAGE_WORKERS"], os.environ["PCF_STAGE_SLOTS"], os.environ["PCF_STAGE_MB"] = w, s, mb
        print(f"cfg workers={w} slots={s} MB={mb}", file=sys.stderr, flush=True)
        matrix_host(ht.numpy(), hv.numpy(), ho.numpy(), 0, 1.0, True, False, n_chunks=32, out=out)
