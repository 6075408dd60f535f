"""Repeated c5 mean/std timings (allocator / warm-up sensitivity check)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2404_07183_b200 import datagen as dg
from paper_2404_07183_b200.reduce import DeviceLevel, mean_packed, std_packed
M = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
shape, mats = dg.noisy_trig_matrices((M,), 100, "sin", 0.1, dg.RngSpec(2404))
t, v, off = dg.pack_matrices(mats)
lvl = DeviceLevel.from_packed(t, v, off)
if len(sys.argv) > 2:  # fragment the allocator like a preceding c2 run
    junk = [torch.empty(10000 * 10000, dtype=torch.float64, device="cuda") for _ in range(3)]
    del junk
for name, fn in (("mean", lambda: mean_packed(lvl)), ("std", lambda: std_packed(lvl))):
    for r in range(4):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter(); a.record(); fn(); b.record(); torch.cuda.synchronize()
        print(name, r, f"dev {a.elapsed_time(b):.1f} ms wall {1e3*(time.perf_counter()-t0):.1f} ms", flush=True)
