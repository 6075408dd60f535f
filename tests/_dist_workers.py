"""Rank bodies of tests/test_gpu_distributed.py (spawned processes; importable by name).
Two gloo ranks share cuda:0: the device kernels run in every rank, the collectives go
through host memory (NCCL refuses two ranks on one GPU)."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _init(rank, world, initfile):
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"file://{initfile}", rank=rank,
                            world_size=world)
    return dist


def reductions(rank, world, initfile, outdir, M, npts):
    import torch

    from paper_2404_07183_b200 import datagen as dg, parallel

    dist = _init(rank, world, initfile)
    try:
        _, mats = dg.noisy_trig_matrices((M,), npts, "sin", 0.1, dg.RngSpec(2404))
        t, v, off = dg.pack_matrices(mats)
        m = parallel.mean_distributed(t, v, off, "cuda:0")
        s = parallel.std_distributed(t, v, off, "cuda:0")
        if rank == 0:
            np.savez(os.path.join(outdir, "red.npz"),
                     mt=m.t[: m.ntot].cpu().numpy(), mv=m.v[: m.ntot].cpu().numpy(),
                     st=s.t[: s.ntot].cpu().numpy(), sv=s.v[: s.ntot].cpu().numpy())
        else:
            assert m is None and s is None
        torch.cuda.synchronize()
    finally:
        dist.destroy_process_group()


def matrices(rank, world, initfile, outdir, M):
    import torch

    from paper_2404_07183_b200 import datagen as dg, parallel

    dist = _init(rank, world, initfile)
    try:
        t, v, off = dg.synthetic_benchmark_packed(M, rng=dg.RngSpec(2404))
        res = {}
        for name, (op, p, root, diag, exact) in {
                "l1_fast": (0, 1.0, True, False, False),
                "l1_exact": (0, 1.0, True, False, True),
                "l2_fast": (0, 2.0, True, False, False),
                "gram_fast": (1, 0.0, False, True, False),
                "gram_exact": (1, 0.0, False, True, True)}.items():
            out, err = parallel.matrix_distributed(t, v, off, op, p, root, diag, exact=exact,
                                                   device="cuda:0")
            if rank == 0:
                assert err is None
                res[name] = out.cpu().numpy()
            else:
                assert out is None
        # a divergent pair is reported as the row-major first over both ranks
        bad = dg.pack_matrices([np.column_stack((t[off[i]:off[i + 1]], v[off[i]:off[i + 1]]))
                                for i in range(M)] + [np.array([[0.0, 1.0]])])
        out, err = parallel.matrix_distributed(*bad, 0, 1.0, True, False, device="cuda:0")
        if rank == 0:
            res["bad_err"] = np.array(err)
            np.savez(os.path.join(outdir, "mat.npz"), **res)
        torch.cuda.synchronize()
    finally:
        dist.destroy_process_group()
