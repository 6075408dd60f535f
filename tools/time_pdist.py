"""The drop-in call at c3: paper_2404_07183_b200.pdist(fs) on 100,000 App-A Pcf objects
(reference entry point pkg/src/pcflib/matrix.py:246-270), wall time per call in the
default exact mode and in fast mode, next to the bench's e2e (pcf_matrix_host on packed
arrays).  Includes packing the Pcf objects and the pinned 80 GB result.

    python tools/time_pdist.py [M] [reps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2404_07183_b200 as pb  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
t0 = time.perf_counter()
fs = pb.synthetic_benchmark(M, rng=pb.RngSpec(2404))
print(f"generated {M} Pcf objects in {time.perf_counter() - t0:.1f} s", flush=True)
pairs = M * (M - 1) // 2
for exact in (True, False):
    for r in range(reps):
        t0 = time.perf_counter()
        D = pb.pdist(fs, p=1.0, exact=exact)
        dt = time.perf_counter() - t0
        arr = np.asarray(D)
        print(f"pdist exact={exact} rep={r}: {dt:.3f} s = {pairs / dt:.4e} pairs/s "
              f"(D[0,1]={arr[0, 1]!r}, D[{M - 2},{M - 1}]={arr[M - 2, M - 1]!r})", flush=True)
        del D, arr
