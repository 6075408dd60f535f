"""K1 throughput per merge-path split class (items grouped by log2 G) on App-A M PCFs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_07183_b200 import datagen as dg  # noqa: E402
from paper_2404_07183_b200.collection import DeviceCollection  # noqa: E402
from paper_2404_07183_b200.engine import fill_pairwise, item_cells, items_to_device  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
t, v, off = dg.synthetic_benchmark_packed(M, rng=dg.RngSpec(2404))
coll = DeviceCollection(t, v, off)
dev_items, host, smem = coll.plan()
out = torch.empty((M, M), dtype=torch.float64, device="cuda")
tot_ms = 0
for g in range(7):
    sel = host[host[:, 5] == g]
    if sel.shape[0] == 0:
        continue
    cells = item_cells(sel, coll.sizes_sorted)
    items = (items_to_device(sel, coll.device), sel, smem)
    fill_pairwise(coll, 0, 1.0, True, False, out=out, items=items)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    fill_pairwise(coll, 0, 1.0, True, False, out=out, items=items)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    tot_ms += ms
    rows = np.unique(sel[:, 0])
    print(f"log2G={g}: {sel.shape[0]:6d} items, rows n~{coll.sizes_sorted[rows].mean():6.0f}, "
          f"{cells:.3e} cells, {ms:8.2f} ms, {cells / ms * 1e3:.3e} cells/s", flush=True)
print(f"sum {tot_ms:.1f} ms")
