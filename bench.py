"""Benchmark: PCF pair-integrals/s of the 100k-PCF L1 distance matrix (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1)

One step = the full upper triangle of the pairwise L1 distance matrix of M = 100,000
App-A synthetic PCFs (pcflib.synthetic_benchmark(100000, RngSpec(2404)), float64;
5.0585e12 rectangle cells, 4.99995e9 pair-integrals) written as the dense M x M result in
original order.  With N GPUs the cost-sorted tile queue is dealt across ranks (strong
scaling: the same matrix, 1/N of the pairs per GPU, no collective on the data path).

Printed JSON (rank 0, one line): value = pairs / (max over ranks of the device time of
K steps) with inputs resident in HBM; e2e = the same metric through the host-buffer
path (pinned host inputs -> H2D -> device pack -> fill -> D2H of the whole matrix);
roofline of the dominant kernel (k_fill_tiles_smem) against the FP64 peak measured
live by a DFMA probe; cpu_baseline = the reference's own compiled kernel
(oracle/_ref, built from _sweepkern.pyx) on a row sample on all host cores.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PCF pair-integrals/sec (100k-PCF L1 distance matrix)"
# collectives backend: nccl (one GPU per rank); PCF_BENCH_BACKEND=gloo runs the same
# multi-rank logic with host-side collectives, e.g. two ranks on one GPU for testing
BACKEND = os.environ.get("PCF_BENCH_BACKEND", "nccl")
UNIT = "pair-integrals/s"
FLOPS_PER_CELL_L1 = 4  # |vf - vg|, tn - t, mul, add
# planner smem_mode -> kernel (csrc/pcf_tiles.cuh)
KERNEL_NAMES = {1: "k_fill_tiles_smem", 3: "k_fill_colgroups", 4: "k_fill_rows_staged",
                2: "k_fill_rowres", 0: "k_fill_tiles_global"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--M", type=int, default=100000)
    ap.add_argument("--exact", action="store_true", help="one lane per pair (bitwise mode)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-other", action="store_true",
                    help="skip the second (exact when the headline is fast) device timing")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload(M):
    from paper_2404_07183_b200 import datagen as dg

    t, v, off = dg.synthetic_benchmark_packed(M, rng=dg.RngSpec(2404))
    n = np.diff(off)
    pairs = M * (M - 1) // 2
    cells = (M - 1) * int(n.sum()) - pairs
    return t, v, off, pairs, cells


# ------------------------------------------------------------------ clocks sampling
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ CPU reference leg
def cpu_reference_sample(t, v, off, seconds, threads=None):
    """Time the reference's compiled kernel (oracle/_ref, else the C port) on contiguous
    row blocks spread over [0, M) with an O(M) aliasing sink, on all host
    cores.  Returns (pairs/s, cells/s, kind, cores, sample description)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    from numpy.lib.stride_tricks import as_strided

    M = off.shape[0] - 1
    threads = threads or os.cpu_count() or 1
    n = np.diff(off)
    K = O.load_reference_kernel()
    kind = "reference" if K is not None else "port"
    packed = (np.ascontiguousarray(t), np.ascontiguousarray(v), np.ascontiguousarray(off))
    orc = None if K is not None else O.Oracle()
    # calibrate: rows spread over [0, M), one row per task
    rng = np.random.default_rng(0)
    order = rng.permutation(M - 1)
    lock = threading.Lock()
    state = {"next": 0, "pairs": 0, "cells": 0, "stop": False}

    def worker():
        buf = np.zeros(M)
        sink = as_strided(buf, shape=(M, M), strides=(0, 8))
        while True:
            with lock:
                if state["stop"] or state["next"] >= order.shape[0]:
                    return
                i = int(order[state["next"]])
                state["next"] += 1
            if K is not None:
                K.fill_block(packed, i, i + 1, 0, 1.0, True, False, 0.0, math.inf, sink)
            else:
                orc.row(packed[0], packed[1], packed[2], i)
            np_ = M - 1 - i
            cl = np_ * (int(n[i]) - 1) + int(off[M] - off[i + 1])
            with lock:
                state["pairs"] += np_
                state["cells"] += cl

    ths = [threading.Thread(target=worker, daemon=True) for _ in range(threads)]
    t0 = time.perf_counter()
    for th in ths:
        th.start()
    time.sleep(seconds)
    with lock:
        state["stop"] = True
    for th in ths:
        th.join()
    dt = time.perf_counter() - t0
    desc = (f"{state['next']} random rows i of the same {M}-PCF collection, all j > i "
            f"({state['pairs']} pair-integrals, {state['cells']:.3e} cells) via "
            f"{'reference _sweepkern.fill_block (oracle/_ref)' if K is not None else 'C port'}"
            f" on {threads} threads, {dt:.1f} s")
    return state["pairs"] / dt, state["cells"] / dt, kind, threads, desc


def reference_rows_parity(t, v, off, gpu_rows):
    """The e2e (host) result's sampled rows against the reference's own kernel
    (oracle/_ref; the C port if the reference could not be built), one row per call:
    fill_block(i, i + 1) into an O(M) aliasing sink leaves D[i, i+1:] in buf[i+1:]
    (SURVEY.md 8d).  North-star tolerance: relative 1e-12."""
    import concurrent.futures

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    from numpy.lib.stride_tricks import as_strided

    M = off.shape[0] - 1
    K = O.load_reference_kernel()
    packed = (np.ascontiguousarray(t), np.ascontiguousarray(v), np.ascontiguousarray(off))

    def ref_row(i):
        if K is None:
            return O.Oracle().row(packed[0], packed[1], packed[2], i)
        buf = np.zeros(M)
        K.fill_block(packed, i, i + 1, 0, 1.0, True, False, 0.0, math.inf,
                     as_strided(buf, shape=(M, M), strides=(0, 8)))
        return buf

    worst, rows = 0.0, sorted(gpu_rows)
    with concurrent.futures.ThreadPoolExecutor(len(rows)) as ex:
        for i, ref in zip(rows, ex.map(ref_row, rows)):
            got, want = gpu_rows[i][i + 1:], ref[i + 1:]
            worst = max(worst, float(np.max(np.abs(got - want) /
                                            np.maximum(np.abs(want), 1e-300))))
    return {"rows": rows, "columns_per_row": "all j > i", "max_rel": worst, "tol": 1e-12,
            "ok": worst < 1e-12, "checked": "e2e host result (pcf_matrix_host)",
            "against": "reference _sweepkern.fill_block" if K is not None else "C port"}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    M = args.M
    t, v, off, pairs, cells = workload(M)
    secs = max(5.0, min(args.cpu_seconds, 120.0 / max(1, args.steps + args.warmup)))
    vals = []
    desc = kind = cores = None
    for step in range(args.warmup + args.steps):
        pps, cps, kind, cores, desc = cpu_reference_sample(t, v, off, secs)
        if step >= args.warmup:
            vals.append(pps)
    val = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": pairs / val * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: App-A PCFs (pcflib.synthetic_benchmark, RngSpec(2404))",
        "config": {"workload": f"c3: L1 distance matrix of {M} App-A PCFs, float64",
                   "M": M, "pairs": pairs, "cells": cells},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": desc},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our GPU leg
def fp64_peak_tflops(lib, torch, stream):
    from paper_2404_07183_b200 import _native

    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    iters, bps = 4096, 8
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    for _ in range(2):
        lib.pcf_probe_fp64(_native.ptr(out), iters, bps, stream)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    lib.pcf_probe_fp64(_native.ptr(out), iters, bps, stream)
    e.record()
    torch.cuda.synchronize()
    flops = nsm * bps * 256 * 8 * iters * 2.0
    return flops / (s.elapsed_time(e) * 1e-3) / 1e12


def run_ours(args):
    import torch
    import torch.distributed as tdist

    from paper_2404_07183_b200 import _native
    from paper_2404_07183_b200.collection import DeviceCollection, current_stream_handle
    from paper_2404_07183_b200.engine import (decode_err, item_cells, items_to_device,
                                              mode_runs, new_err, partition_items)

    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if BACKEND != "nccl":  # ranks may share a GPU
        local = local % max(1, torch.cuda.device_count())
    if world > 1:
        torch.cuda.set_device(local)
        if BACKEND == "nccl":
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:  # test plumbing: several ranks sharing one GPU (NCCL refuses that)
            tdist.init_process_group("gloo")
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    lib = _native.load()
    M = args.M
    t, v, off, pairs, cells = workload(M)

    coll = DeviceCollection(t, v, off, device=dev)
    out = torch.empty((M, M), dtype=torch.float64, device=dev)
    err = new_err(dev)
    counter = torch.zeros(1, dtype=torch.int32, device=dev)
    st = current_stream_handle()
    stream = torch.cuda.current_stream()

    def timed_fill(exact, steps, warmup, sample_clocks):
        """Plan (exact or fast), then `warmup` untimed and `steps` timed whole-matrix
        fills bracketed by barrier + synchronize; returns the max-over-ranks time, the
        per-kernel-mode CUDA-event averages (each launch timed on the stream it runs on)
        and the cells each mode covers."""
        _, host_items, smem = coll.plan(exact=exact)
        my_items = partition_items(host_items, world, rank)
        items_dev = items_to_device(my_items, dev)
        runs = mode_runs(my_items)
        ev = {mode: [] for _, _, mode in runs}

        def step(record=False):
            launches = 0
            if rank == 0:  # one writer per entry across ranks: the diagonal is rank 0's
                lib.pcf_fill_diagonal(_native.ptr(coll.recs), _native.ptr(coll.soff),
                                      _native.ptr(coll.perm), M, 0, 0.0, math.inf,
                                      _native.ptr(out), 0, M, _native.ptr(err), st)
                launches = 1
            for lo, hi, mode in runs:
                if record:
                    a, b = (torch.cuda.Event(enable_timing=True),
                            torch.cuda.Event(enable_timing=True))
                    a.record(stream)
                rc = lib.pcf_fill_matrix(
                    _native.ptr(coll.tile_recs), _native.ptr(coll.recsg),
                    _native.ptr(coll.soff), _native.ptr(coll.goff), _native.ptr(coll.perm), M,
                    _native.c_vp(items_dev.data_ptr() + lo * 32), hi - lo, smem, mode,
                    coll.rec_bytes, _native.ptr(counter), 0, 1.0, 1, 0.0, math.inf,
                    _native.ptr(out), 0, M, _native.ptr(err), st)
                _native.check(rc, "pcf_fill_matrix")
                launches += 1
                if record:
                    b.record(stream)
                    ev[mode].append((a, b))
            return launches

        for _ in range(max(warmup, 0)):
            step()
        torch.cuda.synchronize()
        if world > 1:
            tdist.barrier()
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        launches = 0
        with ClockSampler(local) as clk:
            t0.record(stream)
            for _ in range(steps):
                launches += step(record=True)
            t1.record(stream)
            torch.cuda.synchronize()
        ms = t0.elapsed_time(t1)
        if world > 1:
            tt = torch.tensor([ms], dtype=torch.float64,
                              device=dev if BACKEND == "nccl" else "cpu")
            tdist.all_reduce(tt, op=tdist.ReduceOp.MAX)
            tdist.barrier()
            ms = float(tt.item())
        bad = decode_err(err, M)
        if bad is not None:
            raise RuntimeError(f"non-finite entry {bad}")
        kms = {mode: float(np.mean([a.elapsed_time(b) for a, b in e])) for mode, e in ev.items()}
        mcells = {mode: item_cells(my_items[my_items[:, 6] == mode], coll.sizes_sorted)
                  for mode in kms}
        return {"ms": ms, "launches": launches, "kms": kms, "mcells": mcells,
                "items": int(host_items.shape[0]), "smem": smem, "clk": clk}

    def dominant(res):
        """The kernel mode with the largest share of the step, its name, time and cells."""
        mode = max(res["kms"], key=lambda m: res["kms"][m])
        return mode, KERNEL_NAMES.get(mode, str(mode)), res["kms"][mode], res["mcells"][mode]

    peak = fp64_peak_tflops(lib, torch, st)
    main = timed_fill(args.exact, args.steps, args.warmup, True)
    ms = main["ms"]
    clk = main["clk"]
    value = pairs * args.steps / (ms * 1e-3)
    dmode, dname, k_avg, smem_cells = dominant(main)
    achieved = FLOPS_PER_CELL_L1 * smem_cells / (k_avg * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "k1_traffic.json")
    if os.path.exists(tpath):
        try:
            tr = json.load(open(tpath))
            if tr.get("M") == M and tr.get("exact") == bool(args.exact):
                traffic = tr.get("bytes_per_launch")
        except (OSError, ValueError):
            traffic = None
    launches = main["launches"]
    host_items_n, smem = main["items"], main["smem"]
    # the other mode (exact when the headline is fast), measured the same way on the same
    # buffers: exact = one lane per pair summed left to right, bitwise equal to the
    # reference kernel; it is what pdist()/l2_kernel() run by default
    other = None
    if not args.no_other:
        o_steps = max(1, min(args.steps, 2))
        o = timed_fill(not args.exact, o_steps, 1, False)
        om, oname, oms, ocells = dominant(o)
        other = {"mode": "fast (merge-path G lanes/pair)" if args.exact
                 else "exact (1 lane/pair, bitwise vs the reference kernel)",
                 "value": pairs * o_steps / (o["ms"] * 1e-3), "unit": UNIT,
                 "ms_per_step": o["ms"] / o_steps, "steps": o_steps, "warmup": 1,
                 "gpu_launches": o["launches"], "work_items": o["items"],
                 "clocks": o["clk"].summary(),
                 "dominant_kernel": {"name": oname, "kernel_ms": oms, "cells": ocells,
                                     "cells_per_s_per_gpu": ocells / (oms * 1e-3),
                                     "fp64_frac": FLOPS_PER_CELL_L1 * ocells
                                     / (oms * 1e-3) / 1e12 / peak},
                 "kernel_ms_by_mode": {KERNEL_NAMES.get(k, str(k)): v
                                       for k, v in o["kms"].items()}}
    del out

    # ---- end-to-end through the host-buffer path
    e2e = None
    if not args.no_e2e:
        del coll  # the e2e path holds its own 80 GB result buffer
        torch.cuda.empty_cache()
        e2e = run_e2e(args, t, v, off, pairs, world, rank, dev)
        lib.pcf_release_workspace()

    cpu = None
    gpu_rows = e2e.pop("_rows", None) if e2e else None
    if rank == 0 and world == 1 and not args.no_cpu:
        pps, cps, kind, cores, desc = cpu_reference_sample(t, v, off, args.cpu_seconds)
        cpu = {"value": pps, "unit": UNIT, "cores": cores, "kind": kind, "sample": desc,
               "cells_per_s": cps, "extrapolated_full_matrix_s": cells / cps}
        if gpu_rows:
            cpu["parity"] = reference_rows_parity(t, v, off, gpu_rows)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: App-A PCFs (pcflib.synthetic_benchmark(100000, RngSpec(2404)))",
            "config": {
                "workload": f"c3: L1 distance matrix of {M} App-A PCFs, float64, full M x M "
                            "output in original order",
                "M": M, "pairs": pairs, "cells": cells,
                "mode": "exact (1 lane/pair)" if args.exact else "fast (merge-path G lanes/pair)",
                "parallelism": f"tile-queue split over {world} GPU(s)",
                "l2": f"no flush needed: {16 * int(off[-1]) / 1e9:.2f} GB input records + "
                      f"{8 * M * M / 1e9:.1f} GB output per step >> 126 MB L2",
                "work_items": host_items_n, "smem_bytes": smem,
            },
            "clocks": clk.summary(),
            "gpu_launches": launches,
            "roofline": {
                "bound": "fp64", "kernel": dname,
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic,
                "peak_source": "measured live: DFMA probe (pcf_probe_fp64); MEASURED_PEAKS.json "
                               "has no FP64 figure",
                "algorithmic": f"{FLOPS_PER_CELL_L1} flop/cell x {smem_cells:.4e} cells per launch",
                "kernel_ms_by_mode": {KERNEL_NAMES.get(k, str(k)): v
                                      for k, v in main["kms"].items()},
                "kernel_ms": k_avg,
                "cells_per_s_per_gpu": smem_cells / (k_avg * 1e-3),
                "traffic_note": "ncu dram read+write per launch (profiles/k1_traffic.json); "
                                "above the 81 GB algorithmic because every 8-byte scattered "
                                "output store costs a 32-byte sector read + write",
                # the resource that actually binds this kernel: the SM's shared-memory
                # data pipe (128 B/clk/SM); algorithmically one 16-byte record load/cell
                "limiter": smem_limiter(smem_cells / (k_avg * 1e-3), clk.summary()),
            },
            "e2e": e2e,
            "exact" if not args.exact else "fast": other,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        tdist.destroy_process_group()


def smem_limiter(cells_per_s, clocks):
    """Shared-memory data-pipe roofline of K1 (16 algorithmic bytes per cell against
    128 B/clk/SM x 148 SMs at the measured SM clock) plus the ncu evidence committed
    under profiles/."""
    mhz = clocks.get("sm_mhz") or 1965.0
    peak = 128.0 * 148 * mhz * 1e6
    out = {"resource": "shared-memory data pipe (LSU wavefronts, 128 B/clk/SM)",
           "algorithmic_bytes_per_cell": 16, "achieved_GBs": cells_per_s * 16 / 1e9,
           "peak_GBs": peak / 1e9, "frac": cells_per_s * 16 / peak}
    path = os.path.join(ROOT, "profiles", "k1_limiter.json")
    if os.path.exists(path):
        try:
            out["ncu"] = json.load(open(path))
        except (OSError, ValueError):
            pass
    return out


def run_e2e(args, t, v, off, pairs, world, rank, dev):
    """Host-buffer path: pinned inputs -> H2D -> K3 pack -> K1 fill -> D2H of the whole
    matrix (rank 0 gathers with an NCCL sum-reduce when N > 1; ranks write disjoint
    entries into zero-initialised buffers, so the sum is exact)."""
    import torch
    import torch.distributed as tdist

    from paper_2404_07183_b200 import _native
    from paper_2404_07183_b200.collection import DeviceCollection
    from paper_2404_07183_b200.engine import fill_pairwise, partition_items, items_to_device

    M = off.shape[0] - 1
    host_t = torch.from_numpy(t).pin_memory()
    host_v = torch.from_numpy(v).pin_memory()
    host_off = torch.from_numpy(off).pin_memory()
    shm = _shared_host_matrix(M, rank, world, dev) if world > 1 else None
    if shm is not None:
        host_out = shm[1]  # one host matrix (shared memory) that every rank fills
    else:
        # a plain (pageable) numpy result, as pdist returns it: pcf_matrix_host drains the
        # finished rows through its pinned staging pool (pinning an 80 GB result instead
        # costs ~56 s of host time; the staged path measures within 1% of a pinned one)
        host_out = np.empty((M, M), dtype=np.float64) if world == 1 else (
            torch.empty((M, M), dtype=torch.float64, pin_memory=True) if rank == 0 else None)
    band = -(-M // world)
    # world 1: pcf_matrix_host owns its device buffers (workspace cached between calls);
    # N ranks: zeroed M x M buffers (rows padded to N bands for the reduce-scatter)
    out_full = torch.zeros((band * world, M), dtype=torch.float64, device=dev) \
        if world > 1 else None
    out = out_full[:M] if world > 1 else None
    recv = torch.empty((band, M), dtype=torch.float64, device=dev) \
        if shm is not None else None
    stream = torch.cuda.current_stream()
    bi = host_t.numel() * 8 + host_v.numel() * 8 + host_off.numel() * 8
    bo = M * M * 8 if rank == 0 else 0

    if world == 1:
        # the reference-facing host-buffer C-ABI call: pinned SoA in, pageable M x M out
        from paper_2404_07183_b200.engine import matrix_host

        st_handle = ctypes.c_void_p(stream.cuda_stream)
        tn, vn, on = host_t.numpy(), host_v.numpy(), host_off.numpy()

        def e2e_step():
            _, bad = matrix_host(tn, vn, on, 0, 1.0, True, False, exact=args.exact,
                                 n_chunks=32, out=host_out, stream=st_handle)
            if bad is not None:
                raise RuntimeError(f"non-finite entry {bad}")
        path = ("pcf_matrix_host (one C-ABI call): pinned host SoA (reference pack() layout) "
                "-> H2D (overlapped with the host size sort + plan) -> pcf_pack_sorted -> "
                "diagonal -> one persistent K1 launch over a column-sweep queue in 512 "
                "cost-balanced chunks; the rows each chunk finishes are D2H'd through a pinned "
                "staging pool into the (pageable numpy) M x M float64 result on two copy "
                "streams while later chunks compute")
    elif shm is not None:
        path = ("pinned host SoA (reference pack() layout) -> H2D -> pcf_pack_sorted -> "
                "pcf_fill_diagonal + pcf_fill_matrix (rank's share of the tile queue) -> "
                "reduce-scatter of row bands over NVLink -> every rank D2Hs its band into one "
                "shared (registered) host M x M float64 matrix")
    else:
        path = ("pinned host SoA (reference pack() layout) -> H2D -> pcf_pack_sorted -> "
                "pcf_fill_diagonal + pcf_fill_matrix (rank's share) -> NCCL reduce to rank 0 "
                "-> D2H of the M x M float64 matrix")

    def e2e_step_multi():
        coll = DeviceCollection.__new__(DeviceCollection)
        # same construction as DeviceCollection.__init__, but from pinned host tensors
        dt = host_t.to(dev, non_blocking=True)
        dv = host_v.to(dev, non_blocking=True)
        do = host_off.to(dev, non_blocking=True)
        _build_collection(coll, dt, dv, do, off, dev)
        items_dev, host_items, smem = coll.plan(exact=args.exact)
        if world > 1:
            mine = partition_items(host_items, world, rank)
            items = (items_to_device(mine, dev), mine, smem)
        else:
            items = (items_dev, host_items, smem)
        fill_pairwise(coll, 0, 1.0, True, False, out=out, items=items,
                      diagonal=(rank == 0))
        if shm is not None:
            # every entry has exactly one writer and the buffers start at zero, so the
            # sum-reduce-scatter assembles each band exactly; each rank then drains its
            # band over its own PCIe link
            if BACKEND == "nccl":
                tdist.reduce_scatter_tensor(recv, out_full)
            else:  # gloo has no reduce-scatter: same result through an all-reduce
                host = out_full.cpu()
                tdist.all_reduce(host)
                recv.copy_(host[rank * band:(rank + 1) * band])
            r0, r1 = rank * band, min(M, (rank + 1) * band)
            if r1 > r0:
                host_out[r0:r1].copy_(recv[: r1 - r0], non_blocking=True)
            return
        if world > 1:
            if BACKEND == "nccl":
                tdist.reduce(out, dst=0)
            else:
                host = out.cpu()
                tdist.reduce(host, dst=0)
                if rank == 0:
                    out.copy_(host)
        if rank == 0:
            host_out.copy_(out, non_blocking=True)

    if world > 1:
        e2e_step = e2e_step_multi
    for _ in range(1):
        e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        tdist.barrier()
    k = max(1, min(args.steps, 2))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(k):
        e2e_step()
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device=dev if BACKEND == "nccl" else "cpu")
        tdist.all_reduce(tt, op=tdist.ReduceOp.MAX)
        ms = float(tt.item())
    if shm is not None:
        bo = M * M * 8  # the whole matrix reaches host memory, one band per rank
        tdist.barrier()
    res = {"value": pairs * k / (ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": bi,
           "d2h_bytes_per_step": bo, "ms_per_step": ms / k, "steps": k, "path": path}
    if rank == 0:
        # a few rows of the host result, checked against the reference kernel by the CPU
        # leg (the only place bench.py runs oracle/), and their digest (identical for
        # every GPU count: one writer and one summation order per entry)
        res["_rows"] = {int(i): np.array(host_out[int(i)], dtype=np.float64, copy=True)
                        for i in sorted({1, M // 3, (2 * M) // 3, M - 2}) if 0 <= i < M - 1}
        res["row_digest"] = float(sum(float(np.sum(r)) for r in res["_rows"].values()))
    if shm is not None:
        _release_shared(shm, rank, world)
    return res


def _shared_host_matrix(M, rank, world, dev):
    """One M x M float64 host matrix in /dev/shm mapped by every rank and registered
    (pinned) with CUDA, so each rank can DMA its row band straight into the final result.
    Returns (memmap, tensor, path, registered) or None (then rank 0 gathers)."""
    import torch
    import torch.distributed as tdist

    path = f"/dev/shm/pcf_b200_e2e_{os.environ.get('MASTER_PORT', '0')}_{M}.bin"
    ok = torch.tensor([1], dtype=torch.int32, device=dev if BACKEND == "nccl" else "cpu")
    mm = None
    try:
        if rank == 0:
            # a sparse file larger than the tmpfs would SIGBUS on first touch (the default
            # container /dev/shm is 64 MB): check the free space first, fall back if short
            st = os.statvfs("/dev/shm")
            if st.f_bavail * st.f_frsize < M * M * 8 + (1 << 30):
                raise OSError("not enough free space in /dev/shm")
            mm = np.memmap(path, dtype=np.float64, mode="w+", shape=(M, M))
    except (OSError, ValueError):
        ok[0] = 0
    tdist.broadcast(ok, src=0)
    if not int(ok[0]):
        return None
    tdist.barrier()
    try:
        if rank != 0:
            mm = np.memmap(path, dtype=np.float64, mode="r+", shape=(M, M))
        ten = torch.from_numpy(mm)
        rc = torch.cuda.cudart().cudaHostRegister(ten.data_ptr(), M * M * 8, 0)
        reg = int(rc) == 0
    except (OSError, ValueError, RuntimeError):
        ok[0] = 0
        ten, reg = None, False
    tdist.all_reduce(ok, op=tdist.ReduceOp.MIN)
    if not int(ok[0]):
        return None
    return mm, ten, path, reg


def _release_shared(shm, rank, world):
    import torch
    import torch.distributed as tdist

    mm, ten, path, reg = shm
    if reg:
        torch.cuda.cudart().cudaHostUnregister(ten.data_ptr())
    tdist.barrier()
    if rank == 0:
        try:
            os.unlink(path)
        except OSError:
            pass


def _build_collection(coll, dt, dv, do, off_host, dev):
    """DeviceCollection from device-resident SoA arrays (the e2e path)."""
    import torch

    from paper_2404_07183_b200 import _native
    from paper_2404_07183_b200.collection import current_stream_handle

    M = off_host.shape[0] - 1
    sizes = np.diff(off_host)
    perm = np.argsort(-sizes, kind="stable").astype(np.int32)
    ssizes = sizes[perm].astype(np.int64)
    soff = np.zeros(M + 1, dtype=np.int64)
    np.cumsum(ssizes, out=soff[1:])
    coll.dtype = np.dtype(np.float64)
    coll.M = M
    coll.device = dev
    coll.sizes_sorted = ssizes
    coll.perm_host = perm
    coll.n_points = int(soff[-1])
    coll.perm = torch.from_numpy(perm).to(dev, non_blocking=True)
    coll.soff = torch.from_numpy(soff).to(dev, non_blocking=True)
    coll.inv = None
    coll.recs = torch.empty(2 * coll.n_points, dtype=torch.float64, device=dev)
    goff = np.zeros((M + 7) // 8 + 1, dtype=np.int64)
    goff[1:] = np.cumsum(8 * ssizes[0::8])
    coll.rec_bytes = 16
    coll.goff_host = goff
    coll.goff = torch.from_numpy(goff).to(dev, non_blocking=True)
    coll.recsg = torch.empty(2 * int(goff[-1]), dtype=torch.float64, device=dev)
    coll.tile_recs = coll.recs
    coll._plans = {}
    _native.check(_native.load().pcf_pack_sorted(
        _native.ptr(dt), _native.ptr(dv), 0, _native.ptr(do), _native.ptr(coll.perm),
        _native.ptr(coll.soff), M, _native.ptr(coll.recs), _native.ptr(coll.goff),
        _native.ptr(coll.recsg), current_stream_handle()), "pcf_pack_sorted")


def _free_port():
    import socket

    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def self_launch(args):
    """`bench.py --gpus N` without a torchrun environment: re-run this script as N ranks
    (one process per GPU) under torch.distributed.run on 127.0.0.1 and pass its exit
    status through; rank 0 prints the JSON line."""
    if args.impl == "ours" and BACKEND == "nccl":
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.stderr.write(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) "
                             "visible (NCCL needs one GPU per rank)\n")
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)  # host cores only: rank 0 works, other ranks exit
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
