"""Multi-GPU host logic on CPU (gloo, world_size 2): work sharding covers every pair once
and C1 assembly reproduces the single-process matrix bit for bit; C2 gathers
variable-length payloads in rank order; the aligned-subtree decomposition of the
reduction tree equals the full tree bit for bit.  The per-pair compute inside these
tests is the CPU oracle standing in for the device kernels (test-only)."""

import ctypes
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2404_07183_b200 import _native, datagen as dg, engine, parallel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _plan(sizes_sorted):
    lib = _native.load()
    n = ctypes.c_int64()
    smem = ctypes.c_int32()
    s = np.ascontiguousarray(sizes_sorted, dtype=np.int64)
    lib.pcf_plan_pairwise(_native.ptr(s), s.shape[0], 220 * 1024, 16, 6, 16, None, 0,
                          ctypes.byref(n), ctypes.byref(smem))
    items = (_native.WorkItem * max(n.value, 1))()
    lib.pcf_plan_pairwise(_native.ptr(s), s.shape[0], 220 * 1024, 16, 6, 16,
                          ctypes.cast(items, ctypes.c_void_p), n.value, ctypes.byref(n),
                          ctypes.byref(smem))
    host = np.frombuffer(items, dtype=np.int32).reshape(-1, 8)[: n.value].copy()
    return host, int((host[:, 6] == 1).sum())


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t, v, off = dg.synthetic_benchmark_packed(90, rng=dg.RngSpec(11))
        M = off.shape[0] - 1
        sizes = np.diff(off)
        perm = np.argsort(-sizes, kind="stable")
        items, n_smem = _plan(sizes[perm])
        mine = engine.partition_items(items, world, rank)
        orc = O.Oracle()
        out = torch.zeros((M, M), dtype=torch.float64)
        owned = 0
        for row0, nrows, col0, col1, *_ in mine:
            for ps in range(row0, row0 + nrows):
                for qs in range(max(col0, ps + 1), col1):
                    i, j = int(perm[ps]), int(perm[qs])
                    f = np.column_stack((t[off[i]:off[i + 1]], v[off[i]:off[i + 1]]))
                    g = np.column_stack((t[off[j]:off[j + 1]], v[off[j]:off[j + 1]]))
                    val = orc.accumulate(f, g, op=0, p=1.0)
                    out[i, j] = val
                    out[j, i] = val
                    owned += 1
        parallel.assemble_matrix(out, dst=0)
        cnt = torch.tensor([owned], dtype=torch.int64)
        dist.all_reduce(cnt)
        # C2: variable-length gather
        payload = torch.arange(rank * 3 + 1, dtype=torch.float64) + 100 * rank
        got = parallel.gather_varlen((payload, payload * 2), dst=0)
        if rank == 0:
            ref, _ = orc.matrix(t, v, off)
            q.put(("matrix", bool(np.array_equal(out.numpy(), ref)), int(cnt.item()),
                   M * (M - 1) // 2))
            q.put(("gather", [x.tolist() for x in got[0]], [x.tolist() for x in got[1]]))
    finally:
        dist.destroy_process_group()


def test_sharded_fill_and_gathers_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    res = dict((x[0], x[1:]) for x in (q.get(timeout=10), q.get(timeout=10)))
    ok, owned, total = res["matrix"]
    assert ok and owned == total
    g0, g1 = res["gather"]
    assert g0 == [[0.0], [100.0, 101.0, 102.0, 103.0]]
    assert g1 == [[0.0], [200.0, 202.0, 204.0, 206.0]]


@pytest.mark.parametrize("M,world", [(1, 2), (7, 2), (64, 8), (100, 8), (1000, 3), (5, 8)])
def test_subtree_blocks_aligned(M, world):
    blocks = parallel.subtree_blocks(M, world)
    assert len(blocks) == world
    assert blocks[0][0] == 0 and max(b for _, b in blocks) == M
    size = blocks[0][1] - blocks[0][0]
    assert size & (size - 1) == 0  # power of two
    for (lo, hi), (lo2, _) in zip(blocks, blocks[1:]):
        assert hi == lo2 or hi == M
        if hi > lo:
            assert lo % size == 0


def _tree_raw(mats):
    """reduce.tree_reduce without the final minimise (oracle restatement)."""
    level = list(mats)
    while len(level) > 1:
        nxt = [O.reduce_pair(level[i], level[i + 1], lambda x, y: x + y)
               for i in range(0, len(level) - 1, 2)]
        if len(level) % 2:
            nxt.append(level[-1])
        level = nxt
    return level[0]


@pytest.mark.parametrize("M,world", [(13, 2), (37, 4), (64, 8), (50, 3)])
def test_aligned_subtrees_reproduce_full_tree(M, world):
    rng = np.random.default_rng(M)
    mats = []
    for _ in range(M):
        n = int(rng.integers(1, 12))
        tt = np.concatenate(([0.0], np.sort(rng.choice(np.arange(1, 200) / 20.0, n - 1,
                                                        replace=False))))
        mats.append(np.column_stack((tt, np.round(rng.uniform(-5, 5, n), 2))))
    full = O.minimize(_tree_raw(mats))
    parts = [_tree_raw(mats[lo:hi]) for lo, hi in parallel.subtree_blocks(M, world) if hi > lo]
    assert np.array_equal(O.minimize(_tree_raw(parts)), full)


def test_c3_partition_cost_balanced():
    """The snake deal of the c3 plan (100k App-A PCFs, RngSpec(2404)) gives every one of
    2/4/8 ranks the same number of rectangle cells to within 2% (max/min), in both the
    fast and the exact plan."""
    t, v, off = dg.synthetic_benchmark_packed(100000, rng=dg.RngSpec(2404))
    sizes = np.diff(off)
    ss = np.ascontiguousarray(sizes[np.argsort(-sizes, kind="stable")], dtype=np.int64)
    lib = _native.load()
    total = (len(ss) - 1) * int(ss.sum()) - len(ss) * (len(ss) - 1) // 2
    for log2g in (6, 0):
        n, smem = ctypes.c_int64(), ctypes.c_int32()
        lib.pcf_plan_pairwise(_native.ptr(ss), ss.shape[0], 220 * 1024, 2048, log2g, 16, None,
                              0, ctypes.byref(n), ctypes.byref(smem))
        items = (_native.WorkItem * n.value)()
        lib.pcf_plan_pairwise(_native.ptr(ss), ss.shape[0], 220 * 1024, 2048, log2g, 16,
                              ctypes.cast(items, ctypes.c_void_p), n.value, ctypes.byref(n),
                              ctypes.byref(smem))
        host = np.frombuffer(items, dtype=np.int32).reshape(-1, 8)[: n.value].copy()
        for world in (2, 4, 8):
            costs = parallel.partition_costs(host, ss, world)
            assert sum(costs) == total  # every pair exactly once
            assert max(costs) / min(costs) <= 1.02, (log2g, world, costs)
