"""The reference's OWN pdist (pkg/src/pcflib/matrix.py:256-258: MatrixJob, its thread pool
and row blocks of <= 64 MB) with the B200 plugin installed as its compiled kernel module
(integration/pcflib_cuda_kernels.py -> oracle/_ref/refpkg), timed at M PCFs; compared with
this package's pdist on the same collection.  Run on the GPU box:

    python tools/time_ref_plugin.py [M]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
M = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
REFPKG = os.path.join(ROOT, "oracle", "_ref", "refpkg")
code = f"""
import time, numpy as np, pcflib
print('backend', pcflib.backend_name(), flush=True)
fs = pcflib.synthetic_benchmark({M}, rng=pcflib.RngSpec(2404))
for r in range(2):
    t0 = time.perf_counter(); D = pcflib.pdist(fs); dt = time.perf_counter() - t0
    print(f'reference pdist + B200 plugin M={M} rep={{r}}: {{dt:.3f}} s = {{{M}*({M}-1)/2/dt:.4e}} pairs/s', flush=True)
np.save('/tmp/ref_plugin_D.npy', np.asarray(D)[:4])
"""
env = dict(os.environ, PYTHONPATH=os.path.join(REFPKG, "src"), MASSPCF_BACKEND="compiled",
           PCF_B200_LIB=os.path.join(ROOT, "paper_2404_07183_b200", "_lib", "libpcfb200.so"))
subprocess.run([sys.executable, "-c", code], env=env, check=True)
sys.path.insert(0, ROOT)
import time  # noqa: E402

import numpy as np  # noqa: E402

import paper_2404_07183_b200 as pb  # noqa: E402

fs = pb.synthetic_benchmark(M, rng=pb.RngSpec(2404))
for r in range(2):
    t0 = time.perf_counter()
    D = pb.pdist(fs)
    dt = time.perf_counter() - t0
    print(f"paper_2404_07183_b200.pdist M={M} rep={r}: {dt:.3f} s = "
          f"{M * (M - 1) / 2 / dt:.4e} pairs/s", flush=True)
ref = np.load("/tmp/ref_plugin_D.npy")
print("first 4 rows bitwise equal:", bool(np.array_equal(ref, np.asarray(D)[:4])))
