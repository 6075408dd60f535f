"""C-ABI boundary checks that need no GPU: the library loads, exports exactly what
include/pcf_b200.h declares, and the host-side tile planner covers the upper triangle
exactly once within the shared-memory budget."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT

from paper_2404_07183_b200 import _native

HEADER = os.path.join(ROOT, "include", "pcf_b200.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(pcf_[a-z0-9_]+)\s*\(", src))


def test_library_loads_and_exports_header():
    lib = _native.load()
    declared = header_functions()
    assert declared == set(_native.SIGNATURES), declared ^ set(_native.SIGNATURES)
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (pcf_[a-z0-9_]+)$", out, flags=re.M))
    assert declared <= exported, declared - exported
    for name in declared:
        assert getattr(lib, name) is not None
    assert lib.pcf_version().startswith(b"pcfb200")
    assert lib.pcf_tile_threads() == 512


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def plan(sizes, budget=220 * 1024, max_cols=64, max_log2g=6, rec_bytes=16):
    lib = _native.load()
    sizes = np.ascontiguousarray(sizes, dtype=np.int64)
    n = ctypes.c_int64()
    smem = ctypes.c_int32()
    assert lib.pcf_plan_pairwise(_native.ptr(sizes), sizes.shape[0], budget, max_cols, max_log2g,
                                 rec_bytes, None, 0, ctypes.byref(n), ctypes.byref(smem)) == 0
    items = (_native.WorkItem * max(n.value, 1))()
    assert lib.pcf_plan_pairwise(_native.ptr(sizes), sizes.shape[0], budget, max_cols, max_log2g,
                                 rec_bytes, ctypes.cast(items, ctypes.c_void_p), n.value,
                                 ctypes.byref(n), ctypes.byref(smem)) == 0
    return np.frombuffer(items, dtype=np.int32).reshape(-1, 8)[: n.value].copy(), smem.value


@pytest.mark.parametrize("dist", ["appa", "small", "huge", "beyond", "one", "two"])
@pytest.mark.parametrize("max_log2g", [0, 6])
@pytest.mark.parametrize("rec_bytes", [16, 8])
def test_planner_covers_upper_triangle_once(dist, max_log2g, rec_bytes):
    rng = np.random.default_rng(1)
    sizes = {
        "appa": rng.integers(10, 1001, 700),
        "small": rng.integers(1, 30, 900),
        "huge": np.concatenate([rng.integers(2000, 12000, 20), rng.integers(10, 500, 80)]),
        "beyond": np.concatenate([rng.integers(14000, 30000, 12), rng.integers(10, 3000, 60)]),
        "one": np.array([5]),
        "two": np.array([3, 9]),
    }[dist]
    sizes = np.sort(sizes)[::-1].copy()
    M = sizes.shape[0]
    items, smem = plan(sizes, max_log2g=max_log2g, rec_bytes=rec_bytes)
    gw = 128 // rec_bytes
    units = 512 // gw
    seen = np.zeros((M, M), dtype=np.int32)
    S = np.concatenate([[0], np.cumsum(sizes)])
    threads = 512
    for row0, nrows, col0, col1, logc, log2g, mode, cost in items:
        single = bool(logc >> 8)  # K1 single-buffered columns
        logc &= 0xFF
        C, G = 1 << logc, 1 << log2g
        assert log2g <= max_log2g
        assert col0 > row0 and col1 <= M and nrows >= 1
        if mode == 1:  # K1: GW-row interleaved groups, 512/GW smem-phase units = RG x C x G
            assert row0 % gw == 0 and nrows <= 2 * gw
            RG = 2 if nrows > gw else 1
            partial = RG * C * G < units  # exact-mode K1 with idle quarters
            assert RG * C * G == units or (partial and G == 1 and RG * C * gw >= 256)
            rows_b = sum(gw * sizes[row0 + gw * k] * rec_bytes for k in range(RG))
            col_b = (S[min(col0 + C, col1)] - S[col0]) * rec_bytes + 32
            al = lambda x: (x + 127) // 128 * 128  # noqa: E731
            nbuf = 1 if single else 2
            # segment partials [2][512] + tails [2][512 / G]: only split pairs use them
            red = (2 * 512 + 2 * (512 // G)) * 8 if G > 1 else 0
            assert al(rows_b) + nbuf * al(col_b) + red <= smem <= 220 * 1024
            if single and G > 1:
                # one buffer of 2C columns replaces two of C / 2 (split 2G), which fit
                half_c = (S[min(col0 + C // 2, col1)] - S[col0]) * rec_bytes + 32
                assert al(rows_b) + 2 * al(half_c) + (2 * 512 + 2 * (512 // (2 * G))) * 8 <= 220 * 1024
        elif mode == 3:  # K1c: one resident row x interleaved column groups (CG x G units)
            assert nrows == 1 and C * G == units
            gs = [gw * sizes[gw * k] * rec_bytes for k in range(col0 // gw,
                                                               min((col0 // gw) + C, (M + gw - 1) // gw))]
            al = lambda x: (x + 127) // 128 * 128  # noqa: E731
            nbuf = 1 if single else 2
            red = (2 * 512 + 2 * (512 // G)) * 8 if G > 1 else 0
            assert al((sizes[row0] + 4) * rec_bytes + 16) + nbuf * al(sum(gs) + 16) + red \
                <= smem <= 220 * 1024
        elif mode == 2:  # K1r: one resident row, C columns x G segments
            assert nrows == 1 and C * G == threads and G <= 32
            assert (sizes[row0] * rec_bytes + 127) // 128 * 128 <= smem <= 220 * 1024
        elif mode == 4:  # K1s (exact mode): staged GW-row groups, columns through L1
            assert max_log2g == 0 and G == 1 and row0 % gw == 0 and nrows <= 2 * gw
            RG = 2 if nrows > gw else 1
            assert RG * C == units
            rows_b = sum(gw * sizes[row0 + gw * k] * rec_bytes for k in range(RG))
            assert (rows_b + 127) // 128 * 128 <= smem <= 220 * 1024
        else:  # K1g: R x C pairs x G lanes in-warp (rows beyond shared memory)
            assert mode == 0 and nrows * C * G <= threads and G <= 32
            # rows beyond shared memory, or short rows that miss K1 (K1r is for >= 1024)
            assert sizes[row0] * rec_bytes > 220 * 1024 or sizes[row0] < 1024
        if mode != 1 and row0 % gw:  # outside K1, blocks stop at the next group boundary
            assert (row0 + nrows - 1) // gw == row0 // gw
        for r in range(row0, row0 + nrows):
            for q in range(col0, col1):
                if q > r:
                    seen[r, q] += 1
    iu = np.triu_indices(M, 1)
    assert (seen[iu] == 1).all()
    assert seen.sum() == M * (M - 1) // 2
    for m in (1, 3, 4, 2, 0):
        costs = items[items[:, 6] == m][:, 7]
        assert (np.diff(costs) <= 0).all()  # LPT order within each kernel's run
    runs = [m for k, m in enumerate(items[:, 6]) if k == 0 or items[k - 1, 6] != m]
    assert runs == [m for m in (1, 3, 4, 2, 0) if m in runs]  # one contiguous run per kernel


def test_planner_rejects_unsorted():
    lib = _native.load()
    sizes = np.array([3, 5], dtype=np.int64)
    n = ctypes.c_int64()
    assert lib.pcf_plan_pairwise(_native.ptr(sizes), 2, 1 << 16, 64, 5, 16, None, 0,
                                 ctypes.byref(n), None) == 1
    assert b"sorted" in lib.pcf_last_error()


def test_no_cuda_means_loud_failure():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2404_07183_b200 as pb
    from paper_2404_07183_b200 import errors

    fs = [pb.make_pcf([[0, 1], [1, 0]]), pb.make_pcf([[0, 2], [2, 0]])]
    with pytest.raises(errors.BackendUnavailable):
        pb.pdist(fs)
    with pytest.raises(errors.BackendUnavailable):
        pb.lp_distance(fs[0], fs[1])


def test_jit_tile_prelude_matches_host_layout():
    """The NVRTC prelude of the user-integrand tile module (csrc/pcf_jit.cu) restates
    PcfWorkItem and kTileThreads; both must match the host definitions the planner fills
    (include/pcf_b200.h, csrc/pcf_internal.h)."""
    import re

    hdr = open(os.path.join(ROOT, "include", "pcf_b200.h")).read()
    body = re.search(r"typedef struct pcf_work_item \{(.*?)\} pcf_work_item;", hdr, re.S).group(1)
    host_fields = re.findall(r"int32_t\s+(\w+);", body)
    src = open(os.path.join(ROOT, "paper_2404_07183_b200", "csrc", "pcf_jit.cu")).read()
    pre = re.search(r"struct PcfWorkItem \{ int ([^;]*); \};", src).group(1)
    assert [f.strip() for f in pre.split(",")] == host_fields
    internal = open(os.path.join(ROOT, "paper_2404_07183_b200", "csrc", "pcf_internal.h")).read()
    n_host = re.search(r"constexpr int kTileThreads = (\d+);", internal).group(1)
    n_rtc = re.search(r"constexpr int kTileThreads = (\d+);", src).group(1)
    assert n_host == n_rtc
