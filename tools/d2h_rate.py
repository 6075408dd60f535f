"""D2H bandwidth into pinned host memory (development aid): one contiguous copy vs the
row-sized copies pcf_matrix_host issues, on one and on two streams."""
import time

import torch

M = 100000
rows = 10000
dev = torch.empty((rows, M), dtype=torch.float64, device="cuda")
host = torch.empty((rows, M), dtype=torch.float64, pin_memory=True)
nbytes = dev.numel() * 8


def timed(fn, label):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{label:32s} {nbytes / dt / 1e9:6.1f} GB/s", flush=True)


timed(lambda: host.copy_(dev, non_blocking=True), "one 8 GB copy")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def rows_on(streams, step=1):
    for i in range(rows):
        with torch.cuda.stream(streams[(i // 256) % len(streams)]):
            host[i].copy_(dev[i], non_blocking=True)
    for s in streams:
        s.synchronize()


timed(lambda: rows_on([s1]), "800 KB rows, one stream")
timed(lambda: rows_on([s1, s2]), "800 KB rows, two streams")
