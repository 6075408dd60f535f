"""Multi-GPU sharding and the two collectives of the engine.

One process per GPU (torch.distributed, NCCL over NVLink on the GPU box; gloo works for
the host-side logic).  The path shards with no collective on the data path:

* Pairwise matrices: the cost-sorted tile queue is dealt across ranks
  (engine.partition_items); every pair has exactly one owner and one fixed summation
  order, so the matrix is bit-identical for any world size.  C1 assembles the result on
  rank 0 with one sum-reduce of zero-initialised buffers whose written entries are
  disjoint (x + 0 = x exactly).
* Mean / std: the reference tree (reduce.py:189-208) pairs node 2k with 2k+1 at every
  level, so a power-of-two-aligned block of 2^L leaves is an independent subtree whose
  internal pairing (odd passthrough included, for the last block) equals a standalone
  tree on those leaves.  Rank r reduces block r to one node; C2 gathers the G partial
  PCFs (variable length: sizes first, then padded payloads) onto rank 0, which runs the
  remaining log2(G) levels -- bit-identical to the single-GPU tree.
"""

from __future__ import annotations

import math

import numpy as np

__all__ = ["subtree_blocks", "assemble_matrix", "gather_varlen", "mean_distributed",
           "std_distributed", "fill_pairwise_sharded", "matrix_distributed",
           "partition_costs"]


def subtree_blocks(M, world):
    """Leaf ranges [lo, hi) of the power-of-two-aligned subtrees, one per rank (trailing
    ranks may get empty ranges when M is small)."""
    if M < 1:
        raise ValueError("empty collection")
    per = max(1, math.ceil(M / world))
    size = 1 << max(0, math.ceil(math.log2(per)))
    out = []
    for r in range(world):
        lo = min(M, r * size)
        hi = min(M, (r + 1) * size)
        out.append((lo, hi))
    return out


def assemble_matrix(out, group=None, dst=0):
    """C1: sum-reduce the ranks' zero-initialised M x M buffers onto `dst` (in place)."""
    import torch.distributed as dist

    dist.reduce(out, dst=dst, op=dist.ReduceOp.SUM, group=group)
    return out


def gather_varlen(tensors, dst=0, group=None):
    """C2: gather a tuple of equal-length 1-D tensors of per-rank variable length onto
    `dst`.  Returns, on dst, one list per input tensor with every rank's payload in rank
    order (None elsewhere)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    # NCCL moves device tensors; gloo (host-side test plumbing) only host tensors
    dev = torch.device("cpu") if dist.get_backend(group) == "gloo" else tensors[0].device
    n = torch.tensor([tensors[0].numel()], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    cap = max(max(sizes), 1)
    result = []
    for x in tensors:
        pad = torch.zeros(cap, dtype=x.dtype, device=dev)
        pad[: x.numel()] = x.to(dev)
        # only dst receives payloads (the sizes went to everyone: 8 bytes per rank)
        bufs = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
        dist.gather(pad, bufs, dst=dst, group=group)
        result.append([b[:s] for b, s in zip(bufs, sizes)] if rank == dst else None)
    return result


def partition_costs(host_items, sizes_sorted, world):
    """Cells each rank computes under engine.partition_items (balance check)."""
    from .engine import item_cells, partition_items

    return [item_cells(partition_items(host_items, world, r), sizes_sorted)
            for r in range(world)]


def fill_pairwise_sharded(coll, op, p, apply_root, diag, a=0.0, b=math.inf, exact=False,
                          group=None, out=None):
    """This rank's share of the pairwise matrix: the collection's
    cost-sorted work queue is dealt in snake order (engine.partition_items) and only
    this rank's items run; rank 0 alone writes the diagonal (Gram <f,f> or the distance
    zeros), so every entry of the M x M matrix has exactly one writer across the ranks.
    `out` (device, zero-initialised if None) receives only the rank's entries; summing
    the ranks' buffers (assemble_matrix, or a reduce-scatter) gives the single-GPU
    matrix bit for bit.  Returns (out, err) with err the engine's first-failure word."""
    import torch
    import torch.distributed as dist

    from .engine import fill_pairwise, items_to_device, partition_items

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    _, host_items, smem = coll.plan(exact=exact)
    mine = partition_items(host_items, world, rank)
    if out is None:
        out = torch.zeros((coll.M, coll.M), dtype=coll.out_torch_dtype, device=coll.device)
    out, err, _ = fill_pairwise(coll, op, p, apply_root, diag, a, b, out=out,
                                items=(items_to_device(mine, coll.device), mine, smem),
                                exact=exact, diagonal=(rank == 0))
    return out, err


def _min_err_word(err, group):
    """Minimum over ranks of the engine's unsigned first-failure words (UINT64_MAX =
    none): flip the sign bit so a signed MIN orders them as unsigned."""
    import torch
    import torch.distributed as dist

    flip = -(1 << 63)
    key = err.to(torch.int64) ^ flip
    on_host = dist.get_backend(group) == "gloo"
    buf = key.cpu() if on_host else key
    dist.all_reduce(buf, op=dist.ReduceOp.MIN, group=group)
    return buf.to(err.device) ^ flip


def matrix_distributed(tcat, vcat, off, op, p, apply_root, diag, a=0.0, b=math.inf,
                       exact=False, device=None, group=None, dst=0):
    """Whole pairwise matrix over all ranks of `group`: every rank packs the collection,
    computes its share (fill_pairwise_sharded) and C1 sum-reduces the buffers onto
    `dst`.  Returns (matrix, first_failing_pair) on dst, (None, None) elsewhere; the
    failing pair is the minimum over the ranks (the row-major first, as the reference
    reports it)."""
    import torch.distributed as dist

    from .collection import DeviceCollection
    from .engine import decode_err

    coll = DeviceCollection(tcat, vcat, off, device=device)
    out, err = fill_pairwise_sharded(coll, op, p, apply_root, diag, a, b, exact, group)
    err_min = _min_err_word(err, group)
    if dist.get_backend(group) == "gloo":  # gloo reduces host tensors only
        host = out.cpu()
        dist.reduce(host, dst=dst, group=group)
        if dist.get_rank(group) == dst:
            out.copy_(host)
    else:
        assemble_matrix(out, group=group, dst=dst)
    if dist.get_rank(group) != dst:
        return None, None
    return out, decode_err(err_min, coll.M)


def _local_level(tcat, vcat, off, lo, hi, device):
    from .reduce import DeviceLevel

    o = off[lo:hi + 1] - off[lo]
    return DeviceLevel.from_packed(tcat[off[lo]:off[hi]], vcat[off[lo]:off[hi]], o, device)


def _stack_partials(parts_t, parts_v, parts_m2, is_f32, device):
    import torch

    from .reduce import DeviceLevel

    t = torch.cat(parts_t).to(device)
    v = torch.cat(parts_v).to(device)
    m2 = torch.cat(parts_m2).to(device) if parts_m2 is not None else None
    sizes = [p.numel() for p in parts_t]
    off = torch.tensor(np.concatenate([[0], np.cumsum(sizes)]), dtype=torch.int64,
                       device=device)
    return DeviceLevel(t, v, off, len(sizes), int(sum(sizes)), is_f32, m2)


def mean_distributed(tcat, vcat, off, device, group=None):
    """Mean of a packed collection over all ranks of `group`; the result (a
    DeviceLevel with one node) on rank 0, None elsewhere.  Bit-identical to
    reduce.mean_packed on one GPU."""
    import torch.distributed as dist

    from .reduce import _finalize, _run_tree

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    M = off.shape[0] - 1
    blocks = subtree_blocks(M, world)
    lo, hi = blocks[rank]
    import torch

    if hi > lo:
        level, _ = _run_tree(_local_level(tcat, vcat, off, lo, hi, device), [hi - lo], op=0)
        t_loc, v_loc = level.t[: level.ntot], level.v[: level.ntot]
    else:
        dt = torch.float32 if tcat.dtype == np.float32 else torch.float64
        t_loc = torch.empty(0, dtype=dt, device=device)
        v_loc = torch.empty(0, dtype=dt, device=device)
    parts = gather_varlen((t_loc, v_loc), dst=0, group=group)
    if rank != 0:
        return None
    pt = [p for p, (a, b) in zip(parts[0], blocks) if b > a]
    pv = [p for p, (a, b) in zip(parts[1], blocks) if b > a]
    top = _stack_partials(pt, pv, None, tcat.dtype == np.float32, device)
    out, _ = _run_tree(top, [top.nnodes], op=0)
    return _finalize(out, [1.0 / M], "scale")


def std_distributed(tcat, vcat, off, device, ddof=1, take_sqrt=True, group=None):
    """Pointwise std (parallel-moments tree) over all ranks; result on rank 0."""
    import torch
    import torch.distributed as dist

    from .reduce import _finalize, _moments_level, _run_tree

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    M = off.shape[0] - 1
    if M - ddof == 0:
        raise ZeroDivisionError("float division by zero")
    blocks = subtree_blocks(M, world)
    lo, hi = blocks[rank]
    if hi > lo:
        level, _ = _run_tree(_moments_level(_local_level(tcat, vcat, off, lo, hi, device)),
                             [hi - lo], moments=True)
        loc = (level.t[: level.ntot], level.v[: level.ntot], level.m2[: level.ntot])
    else:
        dt = torch.float32 if tcat.dtype == np.float32 else torch.float64
        loc = (torch.empty(0, dtype=dt, device=device),
               torch.empty(0, dtype=torch.float64, device=device),
               torch.empty(0, dtype=torch.float64, device=device))
    parts = gather_varlen(loc, dst=0, group=group)
    if rank != 0:
        return None
    keep = [b > a for (a, b) in blocks]
    pt = [p for p, k in zip(parts[0], keep) if k]
    pm = [p for p, k in zip(parts[1], keep) if k]
    p2 = [p for p, k in zip(parts[2], keep) if k]
    top = _stack_partials(pt, pm, p2, tcat.dtype == np.float32, device)
    leaves = np.array([b - a for (a, b) in blocks if b > a], dtype=np.int64)
    out, _ = _run_tree(top, [top.nnodes], moments=True, leaves0=leaves)
    return _finalize(out, [1.0 / (M - ddof)], "m2", take_sqrt=take_sqrt)
