"""Host-side costs behind a host-buffer M x M result (development aid): pinning 80 GB,
and pageable device-to-host copy rates into fresh / touched pages."""
import time
import numpy as np
import torch

c = np.empty(80_000_000_000 // 8, dtype=np.float64)
d = torch.empty(1_000_000_000 // 8, dtype=torch.float64, device="cuda")
for label in ("fresh", "touched"):
    t0 = time.perf_counter()
    for k in range(8):  # 8 GB pageable D2H
        torch.from_numpy(c[k * d.numel():(k + 1) * d.numel()]).copy_(d)
    torch.cuda.synchronize()
    print(f"pageable D2H into {label} pages: {8 / (time.perf_counter() - t0):.2f} GB/s", flush=True)
t0 = time.perf_counter()
src = np.ones(d.numel(), dtype=np.float64)
for k in range(8, 16):  # host memcpy into fresh pages, one thread
    c[k * d.numel():(k + 1) * d.numel()] = src
print(f"host memcpy into fresh pages (1 thread): {8 / (time.perf_counter() - t0):.2f} GB/s", flush=True)
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
t0 = time.perf_counter()
p = torch.empty(1_000_000_000 // 8, dtype=torch.float64, pin_memory=True)
print(f"pin 1 GB: {time.perf_counter() - t0:.3f} s", flush=True)
