"""The reference's OWN test suites run against the B200 kernel plugin.

oracle/_ref/refpkg (built by `make -C oracle refpkg` from /root/reference, git-ignored,
shipped to the GPU box with the tree) is the reference's pure-Python package and tests
with integration/pcflib_cuda_kernels.py installed as pcflib._sweepkern: the reference's
"compiled" backend (pkg/src/pcflib/_backend.py:15-20,52) then runs every integral and
matrix on the B200 through the C ABI.  Run unmodified:

* tests/test_backends.py  -- python twin vs compiled(=B200): bitwise for L_p (p = 1, 2,
  3.5), inner products, bounded domains, float32, pdist / l2_kernel matrices, 4 workers;
* tests/test_matrix.py    -- golden matrices, matrix == scalar path bitwise (p = 1, 2,
  3.5), divergence identification, workers invariance, progress, cancellation;
* tests/test_integrate.py -- the scalar API (lp_distance, l2_inner_product, float32
  accumulate-in-float64 KAT, p = 3.5 golden).
"""

import os
import subprocess
import sys

import pytest

from conftest import ROOT, has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a GPU")]

REFPKG = os.path.join(ROOT, "oracle", "_ref", "refpkg")


@pytest.mark.parametrize("suite", ["test_backends.py", "test_matrix.py", "test_integrate.py"])
def test_reference_suite_on_b200_plugin(suite):
    if not os.path.exists(os.path.join(REFPKG, ".stamp")):
        pytest.fail("oracle/_ref/refpkg missing: run `make -C oracle refpkg` where "
                    "/root/reference exists (build() does)")
    env = dict(os.environ, PYTHONPATH=os.path.join(REFPKG, "src"), MASSPCF_BACKEND="compiled",
               PCF_B200_LIB=os.path.join(ROOT, "paper_2404_07183_b200", "_lib",
                                         "libpcfb200.so"))
    # test_env_forces_python starts `python -c "import pcflib"` with an env scrubbed to
    # PATH, so it needs pcflib installed in site-packages; it fails the same way for the
    # unmodified reference here and exercises no kernel
    out = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--rootdir", REFPKG,
         "--deselect", "tests/test_backends.py::TestSelection::test_env_forces_python",
         os.path.join(REFPKG, "tests", suite)],
        capture_output=True, text=True, env=env, cwd=REFPKG, timeout=1200)
    tail = out.stdout[-4000:] + out.stderr[-2000:]
    assert out.returncode == 0, tail
    # the plugin really is the compiled backend in that process
    probe = subprocess.run(
        [sys.executable, "-c", "import pcflib, pcflib._sweepkern as k; "
         "print(pcflib.backend_name(), k.__file__)"],
        capture_output=True, text=True, env=env, cwd=REFPKG, timeout=300)
    assert probe.stdout.split()[0] == "compiled" and probe.stdout.strip().endswith("_sweepkern.py")
