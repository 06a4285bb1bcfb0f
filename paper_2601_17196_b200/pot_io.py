"""File formats of the reference (io.hpp) plus the binary instance / plan
format; the layouts match include/pot/io.hpp.

  trace_to_csv / write_trace_csv   io.hpp:116-135 ("t,E,phi,rounded_cost,elapsed_s")
  read_ppm / write_ppm             io.hpp:159-218 (binary P6)
  read_xyz / write_xyz             io.hpp:220-258
  read/write_instance_json         io.hpp:37-114 (keys r, c, C (flat or rows), s)
  read/write_instance_bin          "POTINST1" | int64 n | f64 s | r[n] | c[n] | C[n*n] row-major
  write_plan_bin / read_plan_bin   "POTPLAN1" | int64 rows, cols | f64 mass | X | row_slack | col_slack
"""
from __future__ import annotations

import json
import math
import struct
from typing import Iterable

import numpy as np

from .pot import ErrorCode, Instance, PotError, TraceRecord, TransportPlan


def _fmt(x: float) -> str:  # "%.17g", io.hpp:21-25
    return "%.17g" % x


def trace_to_csv(records: Iterable[TraceRecord]) -> str:
    out = ["t,E,phi,rounded_cost,elapsed_s\n"]
    for r in records:
        rc = "" if r.rounded_cost is None or (isinstance(r.rounded_cost, float) and math.isnan(r.rounded_cost)) \
            else _fmt(r.rounded_cost)
        out.append(f"{r.t},{_fmt(r.error)},{_fmt(r.phi)},{rc},{_fmt(r.elapsed_s)}\n")
    return "".join(out)


def write_trace_csv(path: str, records) -> None:
    _write(path, trace_to_csv(records).encode())


def _write(path: str, data: bytes) -> None:
    try:
        with open(path, "wb") as f:
            f.write(data)
    except OSError as e:
        raise PotError(ErrorCode.IoFailure, f"cannot write {path}: {e}")


def _read(path: str) -> bytes:
    try:
        with open(path, "rb") as f:
            return f.read()
    except OSError as e:
        raise PotError(ErrorCode.IoFailure, f"cannot open {path}: {e}")


def instance_from_json(doc: dict) -> Instance:
    if not all(k in doc for k in ("r", "c", "C", "s")):
        raise PotError(ErrorCode.IoFailure, "instance needs keys r, c, C, s")
    r = np.asarray(doc["r"], dtype=np.float64)
    c = np.asarray(doc["c"], dtype=np.float64)
    n = r.size
    if c.size != n:
        raise PotError(ErrorCode.IoFailure, "r and c lengths differ")
    C = doc["C"]
    if len(C) and isinstance(C[0], list):
        if len(C) != n or any(len(row) != n for row in C):
            raise PotError(ErrorCode.IoFailure, "cost row / column count mismatch")
        C = np.asarray(C, dtype=np.float64)
    else:
        if len(C) != n * n:
            raise PotError(ErrorCode.IoFailure, "flat cost must have n^2 entries")
        C = np.asarray(C, dtype=np.float64).reshape(n, n)
    return Instance(r=r, c=c, s=float(doc["s"]), C=C)


def read_instance_json(path: str) -> Instance:
    try:
        doc = json.loads(_read(path))
    except ValueError as e:
        raise PotError(ErrorCode.IoFailure, f"{path}: {e}")
    return instance_from_json(doc)


def write_instance_json(path: str, inst: Instance) -> None:
    doc = {"C": [float(x) for x in np.asarray(inst.C).ravel()], "c": [float(x) for x in inst.c],
           "r": [float(x) for x in inst.r], "s": float(inst.s)}
    _write(path, (json.dumps(doc, indent=2) + "\n").encode())


def write_instance_bin(path: str, inst: Instance) -> None:
    n = inst.size()
    C = np.ascontiguousarray(inst.C, dtype="<f8")
    _write(path, b"POTINST1" + struct.pack("<qd", n, float(inst.s)) + np.asarray(inst.r, "<f8").tobytes() +
           np.asarray(inst.c, "<f8").tobytes() + C.tobytes())


def read_instance_bin(path: str) -> Instance:
    b = _read(path)
    if len(b) < 24 or b[:8] != b"POTINST1":
        raise PotError(ErrorCode.IoFailure, f"{path}: not a POTINST1 file")
    n, s = struct.unpack("<qd", b[8:24])
    need = 24 + 8 * (2 * n + n * n)
    if n < 0 or len(b) < need:
        raise PotError(ErrorCode.IoFailure, f"{path}: truncated")
    a = np.frombuffer(b, dtype="<f8", count=2 * n + n * n, offset=24)
    return Instance(r=a[:n].copy(), c=a[n:2 * n].copy(), s=s, C=a[2 * n:].reshape(n, n).copy())


def write_plan_bin(path: str, plan: TransportPlan) -> None:
    X = np.ascontiguousarray(plan.X, dtype="<f8")
    rows, cols = X.shape
    _write(path, b"POTPLAN1" + struct.pack("<qqd", rows, cols, float(plan.mass)) + X.tobytes() +
           np.asarray(plan.row_slack, "<f8").tobytes() + np.asarray(plan.col_slack, "<f8").tobytes())


def read_plan_bin(path: str) -> TransportPlan:
    b = _read(path)
    if len(b) < 32 or b[:8] != b"POTPLAN1":
        raise PotError(ErrorCode.IoFailure, f"{path}: not a POTPLAN1 file")
    rows, cols, mass = struct.unpack("<qqd", b[8:32])
    a = np.frombuffer(b, dtype="<f8", offset=32)
    if a.size < rows * cols + rows + cols:
        raise PotError(ErrorCode.IoFailure, f"{path}: truncated")
    X = a[:rows * cols].reshape(rows, cols).copy()
    return TransportPlan(X=X, mass=mass, row_slack=a[rows * cols:rows * cols + rows].copy(),
                         col_slack=a[rows * cols + rows:rows * cols + rows + cols].copy())


def read_ppm(path: str) -> np.ndarray:
    """Binary P6 (maxval 255) -> uint8 array (height, width, 3)."""
    b = _read(path)
    pos = 0

    def token():
        nonlocal pos
        while True:
            while pos < len(b) and chr(b[pos]).isspace():
                pos += 1
            if pos < len(b) and b[pos:pos + 1] == b"#":
                while pos < len(b) and b[pos:pos + 1] != b"\n":
                    pos += 1
                continue
            break
        start = pos
        while pos < len(b) and not chr(b[pos]).isspace():
            pos += 1
        return b[start:pos]

    if token() != b"P6":
        raise PotError(ErrorCode.IoFailure, f"{path}: expected binary PPM (P6)")
    try:
        w, h, mx = int(token()), int(token()), int(token())
    except ValueError:
        raise PotError(ErrorCode.IoFailure, f"{path}: malformed PPM header")
    if w <= 0 or h <= 0 or mx != 255:
        raise PotError(ErrorCode.IoFailure, f"{path}: unsupported PPM header")
    pos += 1
    data = b[pos:pos + 3 * w * h]
    if len(data) != 3 * w * h:
        raise PotError(ErrorCode.IoFailure, f"{path}: truncated pixel data")
    return np.frombuffer(data, dtype=np.uint8).reshape(h, w, 3).copy()


def write_ppm(path: str, rgb: np.ndarray) -> None:
    rgb = np.ascontiguousarray(rgb, dtype=np.uint8)
    h, w = rgb.shape[:2]
    _write(path, f"P6\n{w} {h}\n255\n".encode() + rgb.tobytes())


def read_xyz(path: str) -> np.ndarray:
    vals = _read(path).split()
    try:
        a = np.array([float(v) for v in vals[: len(vals) // 3 * 3]], dtype=np.float64)
    except ValueError:
        raise PotError(ErrorCode.IoFailure, f"{path}: malformed point")
    if a.size == 0:
        raise PotError(ErrorCode.IoFailure, f"{path}: no points")
    return a.reshape(-1, 3)


def write_xyz(path: str, pts: np.ndarray) -> None:
    pts = np.asarray(pts, dtype=np.float64)
    if pts.ndim != 2 or pts.shape[1] != 3:
        raise PotError(ErrorCode.DimensionMismatch, "point cloud must be N x 3")
    _write(path, "".join(f"{_fmt(x)} {_fmt(y)} {_fmt(z)}\n" for x, y, z in pts).encode())
