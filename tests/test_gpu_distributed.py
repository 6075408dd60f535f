"""N > 1 device paths with two ranks sharing the one B200 (gloo collectives, every
kernel on cuda:0): the sharded pairwise matrix (work queue dealt across ranks, the
diagonal owned by rank 0) and the aligned-subtree mean/std must equal the single-GPU
results bit for bit; `bench.py --gpus 2` must launch two ranks itself and assemble the
same host matrix as `--gpus 1` (reference tree reduce.py:189-238,
paper's 8-GPU run PAPER.md:790-792)."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a GPU")]

import paper_2404_07183_b200 as pb  # noqa: E402
from paper_2404_07183_b200 import datagen as dg  # noqa: E402


def _spawn(fn, *args, world=2):
    import torch.multiprocessing as mp

    import _dist_workers as W

    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=getattr(W, fn), args=(r, world, *args)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]


@pytest.mark.parametrize("M", [1000, 777])
def test_mean_std_two_ranks_bitwise(tmp_path, M):
    import torch

    from paper_2404_07183_b200.reduce import DeviceLevel, mean_packed, std_packed

    _spawn("reductions", str(tmp_path / "pg"), str(tmp_path), M, 40)
    got = np.load(tmp_path / "red.npz")
    _, mats = dg.noisy_trig_matrices((M,), 40, "sin", 0.1, dg.RngSpec(2404))
    lvl = DeviceLevel.from_packed(*dg.pack_matrices(mats))
    m, s = mean_packed(lvl), std_packed(lvl)
    torch.cuda.synchronize()
    assert np.array_equal(got["mt"], m.t[: m.ntot].cpu().numpy())
    assert np.array_equal(got["mv"], m.v[: m.ntot].cpu().numpy())
    assert np.array_equal(got["st"], s.t[: s.ntot].cpu().numpy())
    assert np.array_equal(got["sv"], s.v[: s.ntot].cpu().numpy())


def test_sharded_matrices_two_ranks_bitwise(tmp_path):
    M = 300
    _spawn("matrices", str(tmp_path / "pg"), str(tmp_path), M)
    got = np.load(tmp_path / "mat.npz")
    fs = pb.synthetic_benchmark(M, rng=pb.RngSpec(2404))
    want = {
        "l1_fast": pb.pdist(fs, p=1.0, exact=False),
        "l1_exact": pb.pdist(fs, p=1.0, exact=True),
        "l2_fast": pb.pdist(fs, p=2.0, exact=False),
        "gram_fast": pb.l2_kernel(fs, exact=False),
        "gram_exact": pb.l2_kernel(fs, exact=True),
    }
    for k, w in want.items():
        assert np.array_equal(got[k], np.asarray(w)), k
    # the Gram diagonal is written once (rank 0), not world x <f,f>
    assert np.array_equal(np.diag(got["gram_fast"]), np.diag(np.asarray(want["gram_exact"])))
    assert tuple(got["bad_err"]) == (0, M)


def _bench(gpus, M):
    env = dict(os.environ, PCF_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus),
                          "--M", str(M), "--steps", "1", "--warmup", "1", "--no-cpu"],
                         capture_output=True, text=True, env=env, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-3000:]
    return json.loads(lines[0])


def test_bench_self_launches_two_ranks():
    one = _bench(1, 6000)
    two = _bench(2, 6000)
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["e2e"]["row_digest"] == one["e2e"]["row_digest"]
    assert two["e2e"]["d2h_bytes_per_step"] == 6000 * 6000 * 8
