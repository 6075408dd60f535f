"""Small invocations of every device kernel family, for compute-sanitizer
(racecheck / synccheck / memcheck / initcheck).  Each case prints the work-plan modes it
ran so the log shows which kernels were covered:

  K1  k_fill_tiles_smem   (fast plan, App-A rows < ~1000 records, double/single buffer)
  K1c k_fill_colgroups    (heavy tail: one resident long row, interleaved column groups)
  K1r k_fill_rowres       (long x long pairs)
  K1s k_fill_rows_staged  (exact plan, App-A rows)
  K1g k_fill_tiles_global (exact plan, rows too long to stage)
  K3  k_pack_sorted(32), diagonal, pair list
  K5  k_level_tiled (compacting level), K5m k_merge_level, moments tree, finalisers
  K5w k_wmerge (fused levels: ties, overflowing tiles cut into sub-windows), k_fin_*

usage: python tools/sanitize_cases.py [case ...]   (default: all)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_07183_b200 as pb  # noqa: E402
from paper_2404_07183_b200 import datagen as dg  # noqa: E402
from paper_2404_07183_b200.collection import DeviceCollection  # noqa: E402
from paper_2404_07183_b200.engine import fill_pairwise, mode_runs  # noqa: E402

NAMES = {1: "K1", 3: "K1c", 2: "K1r", 4: "K1s", 0: "K1g"}


def run_pairwise(tag, t, v, off, exact, op=0, p=1.0, root=True, diag=False):
    coll = DeviceCollection(t, v, off)
    _, host, _ = coll.plan(exact=exact)
    modes = [NAMES[m] for _, _, m in mode_runs(host)]
    out, err, _ = fill_pairwise(coll, op, p, root, diag, exact=exact)
    torch.cuda.synchronize()
    print(f"[{tag}] M={coll.M} exact={exact} kernels={modes} "
          f"finite={bool(torch.isfinite(out).all())}", flush=True)


def case_k1():
    t, v, off = dg.synthetic_benchmark_packed(160, rng=dg.RngSpec(7))
    run_pairwise("K1 fast f64", t, v, off, exact=False)
    run_pairwise("K1 fast gram", t, v, off, exact=False, op=1, p=0.0, root=False, diag=True)
    t32, v32, off32 = dg.pack_matrices(dg.fixed_size_collection(96, 40, dtype=np.float32))
    run_pairwise("K1 fast f32", t32, v32, off32, exact=False)


def case_k1s():
    t, v, off = dg.synthetic_benchmark_packed(160, rng=dg.RngSpec(8))
    run_pairwise("K1s exact", t, v, off, exact=True)
    fs = pb.synthetic_benchmark(40, rng=pb.RngSpec(9))
    pb.pdist(fs, p=1.0, a=0.25, b=1.5, exact=True)  # bounded walk
    print("[K1s bounded] ok", flush=True)


def case_tail():
    mats = dg.ecc_like_collection(48, seed=11)
    t, v, off = dg.pack_matrices(mats)
    run_pairwise("K1c/K1r fast p=2", t, v, off, exact=False, p=2.0)
    run_pairwise("K1g exact p=2", t, v, off, exact=True, p=2.0)


def case_reduce():
    arr = pb.noisy_sin((300,), 40, rng=pb.RngSpec(3))
    fs = arr.to_list()
    for mode in ("compact", "merge"):
        os.environ["PCF_TREE_MODE"] = mode
        m = pb.mean(fs)
        s = pb.std(fs)
        print(f"[reduce {mode}] mean {m.size} pts, std {s.size} pts", flush=True)
    os.environ.pop("PCF_TREE_MODE", None)
    import operator

    g = [pb.make_pcf(np.column_stack((np.arange(5.0), np.arange(5.0) % 3))) for _ in range(9)]
    pb.tree_reduce(g, max)
    pb.tree_reduce(g, operator.mul)
    print("[reduce max/mul] ok", flush=True)


def case_fused():
    os.environ["PCF_TREE_MODE"] = "merge"
    os.environ["PCF_TREE_FUSE"] = "4"
    rng = np.random.default_rng(5)
    mats = []
    for k in range(48):  # different time scales: tiles overflow and split in the CTA
        n = 1200 if k % 2 else 150
        scale = 1e-3 if k % 4 == 1 else 1e3
        tt = np.concatenate(([0.0], np.sort(rng.uniform(0, scale, n - 1))))
        mats.append(np.column_stack((tt, rng.normal(size=n))))
    fs = [pb.make_pcf(m) for m in mats]
    m = pb.mean(fs)
    s = pb.std(fs)
    g = [pb.make_pcf(np.column_stack((np.arange(6.0), np.arange(6.0) % 4))) for _ in range(40)]
    pb.tree_reduce(g, max)  # grid times: ties at every level
    os.environ.pop("PCF_TREE_MODE", None)
    os.environ.pop("PCF_TREE_FUSE", None)
    print(f"[K5w fused] mean {m.size} pts, std {s.size} pts, ties ok", flush=True)


CASES = {"k1": case_k1, "k1s": case_k1s, "tail": case_tail, "reduce": case_reduce,
         "fused": case_fused}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
    print("sanitize cases done", flush=True)
