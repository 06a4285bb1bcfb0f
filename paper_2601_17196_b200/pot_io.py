"""Host file formats around the solver path; the
layouts match include/pot/io.hpp. Kept from the reference are only the
contracts a drop-in user depends on:

  trace_to_csv / write_trace_csv   io.hpp:116-135 ("t,E,phi,rounded_cost,elapsed_s")
  read/write_instance_json         io.hpp:37-114 (keys r, c, C (flat or rows), s)
  summary_json                     tools/pot_main.cpp:78-97 (the CLI's summary.json fields)
  EXIT_OK / EXIT_FAILURE / EXIT_USAGE, run_command   pot_main.cpp:337-386 (0 / 1 / 2)
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


_STATUS_NAMES = ("converged", "max-iterations-exceeded", "step-size-underflow")  # core.hpp:286-293


def summary_json(inst: Instance, res, solver: str) -> dict:
    """The CLI's summary.json document (tools/pot_main.cpp:78-97): solver,
    status, iterations, cost, final_error, tolerance, gamma, wall_seconds,
    feasibility_gap and, when the solver computed them, theory_bounds."""
    doc = {"solver": solver, "status": _STATUS_NAMES[int(res.status)],
           "iterations": int(res.iterations), "cost": float(res.cost), "final_error": float(res.final_error),
           "tolerance": float(res.tolerance), "gamma": float(res.gamma), "wall_seconds": float(res.wall_seconds),
           "feasibility_gap": float(res.feasibility_gap)}
    if getattr(res, "bounds", None) is not None:
        b = res.bounds
        doc["theory_bounds"] = {"R": b.R, "L": b.L, "mu_f": b.mu_f, "iteration_bound": b.iteration_bound}
    return doc


def write_summary_json(path: str, inst: Instance, res, solver: str) -> None:
    _write(path, (json.dumps(summary_json(inst, res, solver), indent=2, sort_keys=True) + "\n").encode())


EXIT_OK, EXIT_FAILURE, EXIT_USAGE = 0, 1, 2  # pot_main.cpp:337-386


def run_command(fn, *args, **kwargs) -> int:
    """Exit code of the reference CLI for running `fn`: 0 on success, 1 when
    it raises (PotError or any other exception; the message goes to stderr)."""
    import sys
    try:
        fn(*args, **kwargs)
        return EXIT_OK
    except Exception as e:  # the CLI catches PotError and std::exception alike
        print(f"error: {e}", file=sys.stderr)
        return EXIT_FAILURE
