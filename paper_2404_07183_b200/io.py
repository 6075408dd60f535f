"""Collection I/O for large collections.

The reference reads and writes collections as JSON ({"dtype": "f32"|"f64", "pcfs":
[[[t, v], ...], ...]}) or a directory of two-column CSV files (pkg/src/pcflib/cli.py:59-150),
one Python Pcf object per PCF -- at 1e5-1e6 PCFs the parsing and the per-PCF objects
dominate end to end.  Here:

* ``save_packed`` / ``load_packed`` -- a binary container of the reference pack() layout
  (tcat, vcat, int64 off; _sweepkern.pyx:72-85): a 64-byte header (magic, dtype tag,
  M, N), then off[M+1], tcat[N], vcat[N], little-endian.  ``load_packed`` memory-maps
  the file, so loading is O(1) and the arrays go straight to ``pcf_matrix_host`` /
  ``DeviceCollection`` without Pcf objects.
* ``load_collection`` / ``save_collection`` -- the reference's JSON and CSV-directory
  formats, returned packed (the same values, bit for bit: shortest round-trip decimals,
  cli.py:39-41), plus .pcfb files.
* ``validate_packed`` -- the Pcf invariants (core.py:114-136: t0 == 0, strictly increasing
  finite times, finite values, >= 1 row) checked vectorised over a whole packed collection,
  with the reference's error classes.
"""

from __future__ import annotations

import json
import struct
from pathlib import Path

import numpy as np

from . import errors

__all__ = ["save_packed", "load_packed", "load_collection", "save_collection",
           "validate_packed", "MAGIC"]

MAGIC = b"PCFB\x01\x00\x00\x00"
_HEADER = struct.Struct("<8s4sxxxxqq32x")  # magic, dtype tag, M, N; 64 bytes


def _tag(dtype):
    return b"f32\x00" if np.dtype(dtype) == np.float32 else b"f64\x00"


def validate_packed(tcat, vcat, off):
    """Raise the reference's errors for any PCF of the packed collection that violates
    the Pcf invariants (core.py:114-136); returns the number of PCFs."""
    off = np.asarray(off, dtype=np.int64)
    M = off.shape[0] - 1
    if M < 1:
        raise errors.EmptyCollection("collection is empty")
    sizes = np.diff(off)
    if (sizes < 1).any():
        i = int(np.flatnonzero(sizes < 1)[0])
        raise errors.Empty(f"pcf #{i} has no rows")
    t = np.asarray(tcat)
    v = np.asarray(vcat)
    if not np.isfinite(t).all() or not np.isfinite(v).all():
        bad = np.flatnonzero(~(np.isfinite(t) & np.isfinite(v)))[0]
        i = int(np.searchsorted(off, bad, side="right") - 1)
        raise errors.NonFinite(f"pcf #{i} has a non-finite entry")
    starts = off[:-1]
    if (t[starts] != 0).any():
        i = int(np.flatnonzero(t[starts] != 0)[0])
        raise errors.NonZeroStart(f"pcf #{i}: first time must be 0, got {t[starts[i]]!r}")
    inc = np.ones(t.shape[0], dtype=bool)
    inc[1:] = t[1:] > t[:-1]
    inc[starts] = True  # each PCF's first point has no predecessor
    if not inc.all():
        bad = int(np.flatnonzero(~inc)[0])
        i = int(np.searchsorted(off, bad, side="right") - 1)
        raise errors.NonIncreasingTimes(f"pcf #{i}: times must be strictly increasing")
    return M


def save_packed(path, tcat, vcat, off):
    """Write a packed collection as one .pcfb file."""
    tcat = np.ascontiguousarray(tcat)
    vcat = np.ascontiguousarray(vcat, dtype=tcat.dtype)
    off = np.ascontiguousarray(off, dtype=np.int64)
    if tcat.dtype not in (np.float32, np.float64):
        raise errors.MixedPrecision("times/values must be float32 or float64")
    off0 = off - off[0]
    M, N = off.shape[0] - 1, int(off0[-1])
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(MAGIC, _tag(tcat.dtype), M, N))
        fh.write(off0.astype("<i8").tobytes())
        fh.write(tcat[off[0]:off[0] + N].astype(tcat.dtype.newbyteorder("<")).tobytes())
        fh.write(vcat[off[0]:off[0] + N].astype(tcat.dtype.newbyteorder("<")).tobytes())


def load_packed(path, validate=True):
    """(tcat, vcat, off) memory-mapped from a .pcfb file (read-only views)."""
    path = Path(path)
    with open(path, "rb") as fh:
        head = fh.read(_HEADER.size)
    if len(head) < _HEADER.size:
        raise errors.PcfError(f"{path}: truncated header")
    magic, tag, M, N = _HEADER.unpack(head)
    if magic != MAGIC:
        raise errors.PcfError(f"{path}: not a .pcfb file")
    if tag not in (b"f32\x00", b"f64\x00"):
        raise errors.PcfError(f"{path}: unknown dtype tag {tag!r}")
    dt = np.dtype("<f4" if tag == b"f32\x00" else "<f8")
    need = _HEADER.size + 8 * (M + 1) + 2 * dt.itemsize * N
    if path.stat().st_size < need:
        raise errors.PcfError(f"{path}: truncated ({path.stat().st_size} < {need} bytes)")
    mm = np.memmap(path, dtype=np.uint8, mode="r")
    o = _HEADER.size
    off = mm[o:o + 8 * (M + 1)].view("<i8")
    o += 8 * (M + 1)
    tcat = mm[o:o + dt.itemsize * N].view(dt)
    o += dt.itemsize * N
    vcat = mm[o:o + dt.itemsize * N].view(dt)
    if validate:
        if int(off[0]) != 0 or int(off[-1]) != N or (np.diff(off) < 0).any():
            raise errors.PcfError(f"{path}: corrupt offsets")
        validate_packed(tcat, vcat, off)
    return tcat, vcat, off


def _load_json(p):
    doc = json.loads(Path(p).read_text())
    if not isinstance(doc, dict) or "pcfs" not in doc:
        raise errors.PcfError(f"{p}: expected an object with 'dtype' and 'pcfs'")
    tag = doc.get("dtype", "f64")
    if tag not in ("f32", "f64"):
        raise errors.PcfError(f"unknown dtype tag {tag!r} (expected 'f32' or 'f64')")
    dt = np.float32 if tag == "f32" else np.float64
    rows = doc["pcfs"]
    sizes = np.fromiter((len(r) for r in rows), dtype=np.int64, count=len(rows))
    off = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum(sizes, out=off[1:])
    flat = np.asarray([x for r in rows for pt in r for x in pt], dtype=np.float64)
    flat = flat.reshape(-1, 2).astype(dt)
    return np.ascontiguousarray(flat[:, 0]), np.ascontiguousarray(flat[:, 1]), off


def _load_csv_dir(p):
    files = sorted(f for f in Path(p).iterdir() if f.suffix == ".csv")
    if not files:
        raise errors.PcfError(f"{p}: no .csv files found")
    ts, vs, sizes = [], [], []
    for f in files:
        lines = f.read_text().splitlines()
        if not lines or lines[0].replace(" ", "") != "t,v":
            raise errors.PcfError(f"{f}: row 1: expected header 't,v'")
        body = [ln for ln in lines[1:] if ln.strip()]
        arr = np.asarray([[float(x) for x in ln.split(",")] for ln in body], dtype=np.float64)
        arr = arr.reshape(-1, 2)
        ts.append(arr[:, 0])
        vs.append(arr[:, 1])
        sizes.append(arr.shape[0])
    off = np.zeros(len(sizes) + 1, dtype=np.int64)
    np.cumsum(sizes, out=off[1:])
    return np.concatenate(ts), np.concatenate(vs), off


def load_collection(path, validate=True):
    """Packed (tcat, vcat, off) from a .pcfb file, a reference JSON document or a
    directory of reference CSV files (cli.py:59-109)."""
    p = Path(path)
    if p.is_dir():
        res = _load_csv_dir(p)
    else:
        with open(p, "rb") as fh:
            head = fh.read(8)
        if head == MAGIC:
            return load_packed(p, validate=validate)
        res = _load_json(p)
    if validate:
        validate_packed(*res)
    return res


def _fmt(x):
    return repr(float(x))  # shortest round-trip decimal, as cli.py:39-41


def save_collection(path, tcat, vcat, off, fmt=None):
    """Write a packed collection as .pcfb (fmt 'pcfb' or a .pcfb suffix) or as the
    reference's compact JSON document (cli.py:128-135)."""
    path = Path(path)
    fmt = fmt or ("pcfb" if path.suffix == ".pcfb" else "json")
    if fmt == "pcfb":
        return save_packed(path, tcat, vcat, off)
    tcat, vcat = np.asarray(tcat), np.asarray(vcat)
    tag = "f32" if tcat.dtype == np.float32 else "f64"
    parts = []
    for i in range(len(off) - 1):
        a, b = int(off[i]), int(off[i + 1])
        parts.append("[" + ",".join(f"[{_fmt(t)},{_fmt(v)}]" for t, v in
                                    zip(tcat[a:b].tolist(), vcat[a:b].tolist())) + "]")
    text = '{"dtype":"' + tag + '","pcfs":[' + ",".join(parts) + "]}\n"
    path.write_text(text)
    return None

