"""Quick device timing of the pairwise fill (development aid, not the bench contract)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2404_07183_b200 import datagen as dg
from paper_2404_07183_b200.collection import DeviceCollection
from paper_2404_07183_b200.engine import fill_pairwise, decode_err

M = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["fast"]
t0 = time.time()
t, v, off = dg.synthetic_benchmark_packed(M, rng=dg.RngSpec(2404))
n = np.diff(off)
W = (M - 1) * int(n.sum()) - M * (M - 1) // 2
print(f"gen {time.time()-t0:.1f}s M={M} N={off[-1]} cells={W:.4e}", flush=True)
coll = DeviceCollection(t, v, off)
out = torch.empty((M, M), dtype=torch.float64, device="cuda")
for mode in modes:
    exact = mode == "exact"
    _, host, smem = coll.plan(exact=exact)
    g = np.bincount(host[:, 5], minlength=6)
    m = np.bincount(host[:, 6], minlength=3)
    print(f"[{mode}] items={len(host)} per mode(K1g,K1,K1r)={m.tolist()} smem={smem} log2G hist={g.tolist()}", flush=True)
    fill_pairwise(coll, 0, 1.0, True, False, out=out, exact=exact)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 2
    s.record()
    for _ in range(reps):
        _, err, _ = fill_pairwise(coll, 0, 1.0, True, False, out=out, exact=exact)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    print(f"[{mode}] {ms:.1f} ms/step  pairs/s={M*(M-1)/2/ms*1e3:.4e}  cells/s={W/ms*1e3:.4e}  err={decode_err(err, M)}", flush=True)
