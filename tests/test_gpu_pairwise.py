"""GPU parity of the pairwise engine against the reference (golden vectors from the
reference build) and the CPU oracle (same seeded inputs).

Tolerances (BASELINE.json north star): float64 relative 1e-12, float32 relative 1e-5.
Bitwise where the algorithm allows it: exact mode (one lane per pair) reproduces the
reference's left-to-right sum, so p=1 and Gram entries are bit-identical.
Gram entries use the condition-aware bound |d| <= tol * sqrt(K_ii K_jj) (Cauchy-Schwarz
bound on sum |f g| dt), because random-sign values make some inner products ~0.
"""

import math

import numpy as np
import pytest

from conftest import has_gpu, unpack

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a GPU")]

import oracle as O  # noqa: E402
import paper_2404_07183_b200 as pb  # noqa: E402
from paper_2404_07183_b200 import datagen as dg  # noqa: E402
from paper_2404_07183_b200 import errors  # noqa: E402

TOL64 = 1e-12
TOL32 = 1e-5


def pcfs(golden, tag, dtype=None):
    return [pb.make_pcf(m, dtype=dtype) for m in unpack(golden, tag)]


def rel_err(x, ref):
    scale = np.maximum(np.abs(ref), np.finfo(np.float64).tiny)
    return float(np.max(np.abs(x.astype(np.float64) - ref) / scale))


def gram_err(K, Kref):
    d = np.sqrt(np.abs(np.outer(np.diag(Kref), np.diag(Kref)))) + np.finfo(float).tiny
    return float(np.max(np.abs(K.astype(np.float64) - Kref) / d))


@pytest.mark.parametrize("tag", ["guide", "appa30", "appa200", "rand40"])
@pytest.mark.parametrize("exact", [True, False])
def test_pdist_against_reference(golden, tag, exact):
    fs = pcfs(golden, tag)
    for key in golden:
        if not key.startswith(tag + "_pdist_p"):
            continue
        p = float(key.split("_p")[-1])
        D = np.asarray(pb.pdist(fs, p=p, exact=exact))
        ref = golden[key]
        assert D.dtype == np.float64 and D.shape == ref.shape
        assert np.array_equal(D, D.T)
        assert (np.diag(D) == 0).all()
        if exact:  # one lane per pair + the C library's pow: every p is bitwise
            assert np.array_equal(D, ref), key
        else:
            assert rel_err(D, ref) < TOL64, key


@pytest.mark.parametrize("tag", ["guide", "appa30", "appa200", "rand40"])
def test_gram_against_reference(golden, tag):
    fs = pcfs(golden, tag)
    ref = golden[f"{tag}_gram"] if f"{tag}_gram" in golden else None
    if ref is None:
        pytest.skip("no gram golden")
    K = np.asarray(pb.l2_kernel(fs, exact=True))
    assert np.array_equal(K, ref)
    Kf = np.asarray(pb.l2_kernel(fs))
    assert gram_err(Kf, ref) < TOL64
    assert np.array_equal(np.diag(Kf), np.diag(ref))  # diagonal walk is always sequential


def test_guide_golden_exact(golden):
    fs = pcfs(golden, "guide")
    assert np.array_equal(np.asarray(pb.pdist(fs)), [[0, 34, 6, 12], [34, 0, 34, 24],
                                                      [6, 34, 0, 10], [12, 24, 10, 0]])
    assert np.array_equal(np.asarray(pb.l2_kernel(fs)), [[77, 53, 55, 38], [53, 213, 31, 51],
                                                          [55, 31, 43, 26], [38, 51, 26, 25]])
    p35 = np.array([[0.0, 9.80058139, 2.49774585, 3.81895602],
                    [9.80058139, 0.0, 10.10250875, 8.76880217],
                    [2.49774585, 10.10250875, 0.0, 2.82601424],
                    [3.81895602, 8.76880217, 2.82601424, 0.0]])
    assert np.abs(np.asarray(pb.pdist(fs, p=3.5)) - p35).max() < 1e-7


@pytest.mark.parametrize("tag,a,b", [("guideb", 0.5, 7.25), ("guideb2", 1.0, 6.0),
                                     ("rand40b", 0.75, 6.5)])
def test_bounded_domain(golden, tag, a, b):
    fs = pcfs(golden, tag)
    for key in golden:
        if key.startswith(tag + "_pdist_p"):
            p = float(key.split("_p")[-1])
            for exact in (True, False):
                D = np.asarray(pb.pdist(fs, p=p, a=a, b=b, exact=exact))
                if exact and p == 1.0:
                    assert np.array_equal(D, golden[key]), key
                else:
                    assert rel_err(D, golden[key]) < TOL64, key
    if f"{tag}_gram" in golden:
        K = np.asarray(pb.l2_kernel(fs, a=a, b=b, exact=True))
        assert np.array_equal(K, golden[f"{tag}_gram"])


def test_float32(golden):
    fs = pcfs(golden, "appa12f32")
    assert fs[0].dtype == np.float32
    for p in (1.0, 3.5):
        D = np.asarray(pb.pdist(fs, p=p))
        assert D.dtype == np.float32
        ref = golden[f"appa12f32_pdist_p{p:g}"]
        assert rel_err(D, ref.astype(np.float64)) < TOL32
        if p == 1.0:
            assert np.array_equal(np.asarray(pb.pdist(fs, p=p, exact=True)), ref)
    K = np.asarray(pb.l2_kernel(fs, exact=True))
    assert K.dtype == np.float32 and np.array_equal(K, golden["appa12f32_gram"])


def test_scalar_api_matches_reference(golden):
    fs = pcfs(golden, "guide") + [pb.make_pcf([[0.0, 1.0]])]
    raw = golden["guide_raw"]
    k = 0
    for f in fs:
        for g in fs:
            for op, p in ((0, 1.0), (0, 2.0), (1, 0.0)):
                got = pb.get_backend().integrate_pair(f, g, 0.0, math.inf, op, p)
                if op == 0 and p == 2.0:
                    assert got == pytest.approx(raw[k], rel=TOL64)
                else:
                    assert got == raw[k] or (math.isinf(got) and got == raw[k])
                k += 1
    f1, f2 = fs[0], fs[1]
    assert pb.lp_distance(f1, f2) == 34.0
    assert pb.l2_inner_product(f1, f2) == 53.0
    with pytest.raises(errors.DivergentIntegral):
        pb.lp_distance(f1, fs[-1])
    with pytest.raises(errors.InvalidBounds):
        pb.lp_distance(f1, f2, a=2.0, b=1.0)
    with pytest.raises(ValueError):
        pb.lp_distance(f1, f2, p=0.5)


def test_divergent_entry_identified(golden):
    fs = pcfs(golden, "guide") + [pb.make_pcf([(0, 1)])]
    with pytest.raises(errors.DivergentIntegral) as info:
        pb.pdist(fs)
    assert info.value.pair == (0, 4)
    with pytest.raises(errors.DivergentIntegral) as info:
        pb.l2_kernel(fs)
    assert info.value.pair == (4, 4)  # <bad, bad> diverges; (0..3, 4) do not (tails are 0)


def test_errors_before_kernels():
    f = pb.make_pcf([[0, 1], [1, 0]])
    g = pb.make_pcf(np.array([[0, 1], [1, 0]], dtype=np.float32))
    with pytest.raises(errors.EmptyCollection):
        pb.pdist([])
    with pytest.raises(errors.MixedPrecision):
        pb.pdist([f, g])
    with pytest.raises(ValueError):
        pb.pdist([f, f], p=0.5)
    with pytest.raises(errors.InvalidBounds):
        pb.pdist([f, f], a=-1.0)
    with pytest.raises(ValueError):
        pb.pdist([f, f], workers=0)


def test_single_and_tiny_collections():
    f = pb.make_pcf([[0, 1], [1, 0]])
    assert np.array_equal(np.asarray(pb.pdist([f])), [[0.0]])
    assert np.array_equal(np.asarray(pb.l2_kernel([f])), [[1.0]])
    z = pb.make_pcf([[0, 0]])
    D = np.asarray(pb.pdist([z, z, f]))
    assert np.array_equal(D, [[0, 0, 1], [0, 0, 1], [1, 1, 0]])


def test_fill_block_backend_mirror(golden, oracle):
    fs = pcfs(golden, "appa30")
    be = pb.get_backend()
    packed = be.pack(fs)
    out = np.zeros((30, 30))
    assert be.fill_block(packed, 3, 11, 0, 1.0, True, False, 0.0, math.inf, out) is None
    ref = golden["appa30_pdist_p1"]
    mask = np.zeros_like(out, dtype=bool)
    for i in range(3, 11):
        mask[i, i + 1:] = True
    mask |= mask.T
    assert np.array_equal(out[mask], ref[mask])
    assert (out[~mask] == 0).all()
    # first failing entry of the block, later entries untouched
    bad = fs + [pb.make_pcf([(0, 1)])]
    out = np.zeros((31, 31))
    assert be.fill_block(be.pack(bad), 0, 31, 0, 1.0, True, False, 0.0, math.inf, out) == (0, 30)


def test_progress_and_cancel():
    fs = pb.synthetic_benchmark(64, rng=pb.RngSpec(48))
    job = pb.pdist_job(fs)
    seen = []
    pb.progress_subscribe(job, seen.append)
    job.run()
    assert seen and seen[-1] == 1.0
    assert all(b >= a for a, b in zip(seen, seen[1:]))
    job = pb.pdist_job(fs)
    job.subscribe(lambda frac: job.cancel())
    with pytest.raises(errors.Cancelled):
        job.run()
    assert job.entries_computed == 0
    job = pb.l2_kernel_job(fs)
    job.run()
    assert job.entries_computed == 64 * 65 // 2


@pytest.mark.parametrize("recipe", ["appa", "fixed100", "ecc"])
def test_against_oracle_rows(oracle, recipe):
    """Larger seeded collections: sampled rows vs the C oracle."""
    if recipe == "appa":
        t, v, off = dg.synthetic_benchmark_packed(1500, rng=pb.RngSpec(2404))
        ps = (1.0,)
    elif recipe == "fixed100":
        t, v, off = dg.pack_matrices(dg.fixed_size_collection(1200, 100))
        ps = (1.0, 2.0)
    else:
        t, v, off = dg.pack_matrices(dg.ecc_like_collection(300, nmax_exp=3.7))
        ps = (2.0, 3.0)
    from paper_2404_07183_b200.collection import DeviceCollection
    from paper_2404_07183_b200.engine import decode_err, fill_pairwise

    coll = DeviceCollection(t, v, off)
    M = coll.M
    rows = np.unique(np.linspace(0, M - 2, 12).astype(int))
    for p in ps:
        out, err, _ = fill_pairwise(coll, 0, p, True, False)
        assert decode_err(err, M) is None
        D = out.cpu().numpy()
        for i in rows:
            ref = oracle.row(t, v, off, i, p=p)
            assert rel_err(D[i, i + 1:], ref[i + 1:]) < TOL64
        assert np.array_equal(D, D.T)
        out2, _, _ = fill_pairwise(coll, 0, p, True, False)
        assert np.array_equal(out2.cpu().numpy(), D)  # deterministic
    K, err, _ = fill_pairwise(coll, 1, 0.0, False, True)
    if recipe == "ecc":  # final values are 1: every inner product diverges on [0, inf)
        assert decode_err(err, M) == (0, 0)
        assert np.isinf(K.cpu().numpy()).all()
        return
    K = K.cpu().numpy()
    for i in rows[:4]:
        f = np.column_stack((t[off[i]:off[i + 1]], v[off[i]:off[i + 1]]))
        for j in range(0, M, max(1, M // 50)):
            g = np.column_stack((t[off[j]:off[j + 1]], v[off[j]:off[j + 1]]))
            ref = oracle.accumulate(f, g, op=1, p=0.0)
            bound = math.sqrt(abs(K[i, i] * K[j, j])) * TOL64
            assert abs(K[i, j] - ref) <= bound + 1e-300


def test_exact_mode_bitwise_large(oracle):
    t, v, off = dg.synthetic_benchmark_packed(400, rng=pb.RngSpec(7))
    fs = [pb.make_pcf(np.column_stack((t[off[i]:off[i + 1]], v[off[i]:off[i + 1]])))
          for i in range(400)]
    D = np.asarray(pb.pdist(fs, exact=True))
    ref, _ = oracle.matrix(t, v, off)
    assert np.array_equal(D, ref)
    Df = np.asarray(pb.pdist(fs))
    assert rel_err(Df + np.eye(400), ref + np.eye(400)) < TOL64


def _rank_fill(rank, world, port, q):
    import os

    import torch
    import torch.distributed as dist

    from paper_2404_07183_b200 import datagen as dg
    from paper_2404_07183_b200.collection import DeviceCollection
    from paper_2404_07183_b200.engine import fill_pairwise, items_to_device, partition_items
    from paper_2404_07183_b200 import parallel

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t, v, off = dg.synthetic_benchmark_packed(700, rng=dg.RngSpec(99))
        coll = DeviceCollection(t, v, off)
        _, host, smem = coll.plan()
        mine = partition_items(host, world, rank)
        M = coll.M
        out = torch.zeros((M, M), dtype=torch.float64, device="cuda")
        fill_pairwise(coll, 0, 1.0, True, False, out=out,
                      items=(items_to_device(mine, "cuda"), mine, smem))
        cpu = out.cpu()
        parallel.assemble_matrix(cpu, dst=0)
        if rank == 0:
            full, _, _ = fill_pairwise(coll, 0, 1.0, True, False)
            q.put(bool(torch.equal(cpu, full.cpu())))
    finally:
        dist.destroy_process_group()


def test_sharded_fill_bitwise_equal_single_gpu():
    """Two ranks (sharing this GPU, gloo for the assembly) fill disjoint halves of the
    tile queue; the assembled matrix equals the single-GPU matrix bit for bit."""
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_fill, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    assert q.get(timeout=10)


@pytest.mark.parametrize("recipe,f32,bounds", [("ecc", False, (0.0, math.inf)),
                                               ("ecc", False, (0.3, 2.5)),
                                               ("appa", False, (0.0, math.inf)),
                                               ("ecc", True, (0.0, math.inf))])
def test_streamed_long_pairs(oracle, recipe, f32, bounds):
    """K2 (mode-2 items: one pair per CTA through 1024-record windows) against the C
    oracle, forced onto most rows by a small shared-memory budget."""
    from paper_2404_07183_b200.collection import DeviceCollection
    from paper_2404_07183_b200.engine import decode_err, fill_pairwise

    if recipe == "ecc":
        t, v, off = dg.pack_matrices(dg.ecc_like_collection(160, nmax_exp=3.7))
    else:
        t, v, off = dg.synthetic_benchmark_packed(300, rng=pb.RngSpec(5))
    if f32:
        t, v = t.astype(np.float32), v.astype(np.float32)
    coll = DeviceCollection(t, v, off)
    M = coll.M
    # ECC: 80 KB leaves room for K1r's 4-slot column rings next to rows of 1024..~3000
    # records (longer rows go to K1g); App-A rows (< 1024 records) that miss K1 go to K1g
    dev, host, smem = coll.plan(smem_budget=(80 if recipe == "ecc" else 48) * 1024)
    assert (host[:, 6] == (2 if recipe == "ecc" else 0)).sum() > 0
    a, b = bounds
    rows = np.unique(np.linspace(0, M - 2, 10).astype(int))
    tol = 1e-5 if f32 else TOL64
    for p in (1.0, 2.0):
        out, err, _ = fill_pairwise(coll, 0, p, True, False, a=a, b=b,
                                    items=(dev, host, smem))
        assert decode_err(err, M) is None
        D = out.cpu().numpy().astype(np.float64)
        tt, vv = t.astype(np.float64), v.astype(np.float64)
        for i in rows:
            ref = oracle.row(tt, vv, off, i, p=p, a=a, b=b)
            assert rel_err(D[i, i + 1:], ref[i + 1:]) < tol
        assert np.array_equal(D, D.T)
        out2, _, _ = fill_pairwise(coll, 0, p, True, False, a=a, b=b,
                                   items=(dev, host, smem))
        assert np.array_equal(out2.cpu().numpy(), out.cpu().numpy())  # deterministic


@pytest.mark.parametrize("case", ["appa_l1", "gram64", "gram32", "ecc_l2", "bounded",
                                  "exact_l1", "divergent", "one"])
def test_matrix_host_equals_device_fill(case, oracle):
    """pcf_matrix_host (host buffers in/out, chunked fill with the D2H of finished rows
    overlapping later chunks) writes exactly the matrix of the device-resident fill: the
    same plan, every pair computed by the same lanes, only the item order differs."""
    from paper_2404_07183_b200.collection import DeviceCollection
    from paper_2404_07183_b200.engine import decode_err, fill_pairwise, matrix_host

    op, p, root, diag, a, b, exact = 0, 1.0, True, False, 0.0, math.inf, False
    if case in ("appa_l1", "exact_l1", "bounded"):
        t, v, off = dg.synthetic_benchmark_packed(700, rng=pb.RngSpec(11))
        exact = case == "exact_l1"
        if case == "bounded":
            a, b, p = 0.2, 1.7, 2.0
    elif case in ("gram64", "gram32"):
        dt = np.float32 if case == "gram32" else np.float64
        t, v, off = dg.pack_matrices(dg.fixed_size_collection(600, 50, dtype=dt))
        op, p, root, diag = 1, 0.0, False, True
    elif case == "ecc_l2":
        t, v, off = dg.pack_matrices(dg.ecc_like_collection(150, nmax_exp=3.5))
        p = 2.0
    elif case == "divergent":
        mats = [f.to_matrix() for f in pb.synthetic_benchmark(40, rng=pb.RngSpec(3))]
        mats[17] = np.array([[0.0, 1.0], [0.5, 2.0]])  # final value 2 != 0: diverges vs all
        t, v, off = dg.pack_matrices(mats)
    else:
        t, v, off = dg.pack_matrices([np.array([[0.0, 1.0], [1.0, 0.0]])])
    M = off.shape[0] - 1
    for n_chunks in (1, 7):
        H, herr = matrix_host(t, v, off, op, p, root, diag, a, b, exact=exact,
                              n_chunks=n_chunks)
        coll = DeviceCollection(t, v, off)
        D, err, _ = fill_pairwise(coll, op, p, root, diag, a=a, b=b, exact=exact)
        derr = decode_err(err, M)
        assert herr == derr
        if case == "divergent":
            assert herr == (0, 17)
            continue
        assert herr is None
        D = D.cpu().numpy()
        assert H.dtype == D.dtype and np.array_equal(H, D), case
    if case in ("appa_l1", "exact_l1"):
        ref = oracle.row(t, v, off, 5)
        if exact:
            assert np.array_equal(H[5, 6:], ref[6:])
        assert rel_err(H[5, 6:], ref[6:]) < TOL64


@pytest.mark.parametrize("f32", [False, True])
@pytest.mark.parametrize("exact", [False, True])
@pytest.mark.parametrize("bounds", [(0.0, math.inf), (0.2, 0.85)])
def test_all_tile_kernels_against_oracle(oracle, f32, exact, bounds):
    """A heavy-tailed collection whose plan uses every tile kernel (K1, K1c for long rows
    against short column groups, K1r for long x long pairs, K1g in exact mode) at the
    default shared-memory budget; rows against the C oracle (p = 1 bitwise in exact mode)."""
    from paper_2404_07183_b200.collection import DeviceCollection
    from paper_2404_07183_b200.engine import decode_err, fill_pairwise

    t, v, off = dg.pack_matrices(dg.ecc_like_collection(300, nmax_exp=3.7))
    if f32:
        t, v = t.astype(np.float32), v.astype(np.float32)
    coll = DeviceCollection(t, v, off)
    _, host, _ = coll.plan(exact=exact)
    modes = set(host[:, 6].tolist())
    assert {1, 2, 3} <= modes, modes
    a, b = bounds
    tt, vv = t.astype(np.float64), v.astype(np.float64)
    rows = [0, 3, 40, 150, 298]
    for p in (1.0, 2.0):
        out, err, _ = fill_pairwise(coll, 0, p, True, False, a=a, b=b, exact=exact)
        assert decode_err(err, coll.M) is None
        D = out.cpu().numpy().astype(np.float64)
        assert np.array_equal(D, D.T)
        for i in rows:
            ref = oracle.row(tt, vv, off, i, p=p, a=a, b=b)
            got, want = D[i, i + 1:], ref[i + 1:]
            if f32:
                want = want.astype(np.float32).astype(np.float64)
                assert rel_err(got, want) < TOL32
            elif exact and p == 1.0:
                assert np.array_equal(got, want), i
            else:
                assert rel_err(got, want) < TOL64, i


@pytest.mark.parametrize("exact", [False, True])
def test_matrix_host_pinned_and_pageable_results_agree(exact):
    """pcf_matrix_host writes a pinned result directly and a pageable one through its
    pinned staging pool (host threads copy the rows into place); both, and a strided
    (ld > M) pageable result, hold the same bits."""
    import torch

    from paper_2404_07183_b200.engine import matrix_host

    t, v, off = dg.synthetic_benchmark_packed(900, rng=pb.RngSpec(17))
    M = len(off) - 1
    pinned = torch.empty((M, M), dtype=torch.float64, pin_memory=True).numpy()
    a, bad_a = matrix_host(t, v, off, 0, 1.0, True, False, exact=exact, out=pinned)
    b, bad_b = matrix_host(t, v, off, 0, 1.0, True, False, exact=exact,
                           out=np.empty((M, M)))
    wide = np.full((M, M + 37), -1.0)
    c, bad_c = matrix_host(t, v, off, 0, 1.0, True, False, exact=exact, out=wide[:, :M])
    assert bad_a is None and bad_b is None and bad_c is None
    assert np.array_equal(a, b) and np.array_equal(a, c)
    assert (wide[:, M:] == -1.0).all()  # the padding columns untouched
