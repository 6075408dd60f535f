"""c4 (heavy-tailed ECC-like, L2) device time per tile kernel (K1 / K1r / K1g)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_07183_b200 import datagen as dg  # noqa: E402
from paper_2404_07183_b200.collection import DeviceCollection  # noqa: E402
from paper_2404_07183_b200.engine import fill_pairwise, item_cells, items_to_device  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
t, v, off = dg.pack_matrices(dg.ecc_like_collection(M))
coll = DeviceCollection(t, v, off)
dev_items, host, smem = coll.plan()
out = torch.empty((M, M), dtype=torch.float64, device="cuda")
for mode, name in ((1, "K1"), (3, "K1c"), (2, "K1r"), (0, "K1g")):
    sel = host[host[:, 6] == mode]
    if sel.shape[0] == 0:
        continue
    cells = item_cells(sel, coll.sizes_sorted)
    items = (items_to_device(sel, coll.device), sel, smem)
    fill_pairwise(coll, 0, 2.0, True, False, out=out, items=items)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    fill_pairwise(coll, 0, 2.0, True, False, out=out, items=items)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    rows = np.unique(sel[:, 0])
    print(f"{name}: {sel.shape[0]:6d} items, {rows.size} row blocks, rows n {coll.sizes_sorted[rows].min()}.."
          f"{coll.sizes_sorted[rows].max()}, {cells:.3e} cells, {ms:8.2f} ms, "
          f"{cells / ms * 1e3:.3e} cells/s, log2G hist {np.bincount(sel[:, 5]).tolist()}", flush=True)
