"""ctypes binding of oracle/_build/libpotoracle.so — TEST INFRASTRUCTURE.

Restates the reference solvers on the CPU (fp64, single thread) so tests can
compare the CUDA path against them on identical inputs."""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libpotoracle.so")
KAT = os.path.join(HERE, "_build", "kat_main")

_lib = None


def build():
    subprocess.run(["make", "-C", HERE, "-j4"], check=True, stdout=subprocess.DEVNULL)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        _lib = ctypes.CDLL(LIB)
    return _lib


def _dp(a):
    if a is None:
        return ctypes.POINTER(ctypes.c_double)()
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code  # pot::ErrorCode ordinal


@dataclass
class OracleResult:
    status: int
    iterations: int
    gamma: float
    tolerance: float
    final_error: float
    wall_seconds: float
    cost: float
    feasibility_gap: float
    mass: float
    phi: float
    bounds: Optional[tuple]
    plan: Optional[np.ndarray]
    log: np.ndarray      # rows: t, halvings, block_hat, zbest_is_check, block_check, error, phi_check, phi_hat, theta
    trace: np.ndarray    # rows: t, error, phi, rounded_cost, elapsed


def solve(kind: int, r, c, s, C=None, X=None, Y=None, scale=1.0, epsilon=0.1, gamma_override=None,
          max_iterations=50000, block_rule=0, p=1.0, log_every=1000000, record_rounded_cost=False,
          want_plan=True, skip_plan=False, log_cap=200000, trace_cap=100000) -> OracleResult:
    L = lib()
    n = len(r)
    r = np.ascontiguousarray(r, dtype=np.float64)
    c = np.ascontiguousarray(c, dtype=np.float64)
    Cc = None if C is None else np.ascontiguousarray(C, dtype=np.float64)
    Xc = None if X is None else np.ascontiguousarray(X, dtype=np.float64)
    Yc = None if Y is None else np.ascontiguousarray(Y, dtype=np.float64)
    d = 0 if Xc is None else Xc.shape[1]
    cfg = np.array([epsilon, gamma_override or 0.0, max_iterations, block_rule, p, log_every,
                    1.0 if record_rounded_cost else 0.0], dtype=np.float64)
    summary = np.zeros(16)
    plan = np.empty((n, n)) if (want_plan and not skip_plan and Xc is None) else None
    log = np.zeros((log_cap, 9))
    trace = np.zeros((trace_cap, 5))
    log_len = ctypes.c_long(0)
    err = ctypes.create_string_buffer(512)
    fn = L.oracle_solve
    fn.argtypes = [ctypes.c_int, ctypes.c_long] + [ctypes.POINTER(ctypes.c_double)] * 3 + [ctypes.c_double] + \
        [ctypes.POINTER(ctypes.c_double)] * 3 + [ctypes.c_int, ctypes.c_double, ctypes.c_int] + \
        [ctypes.POINTER(ctypes.c_double)] * 3 + [ctypes.c_long, ctypes.POINTER(ctypes.c_long),
                                                ctypes.POINTER(ctypes.c_double), ctypes.c_long, ctypes.c_char_p,
                                                ctypes.c_int]
    rc = fn(kind, n, _dp(Cc), _dp(r), _dp(c), float(s), _dp(cfg), _dp(Xc), _dp(Yc), d, float(scale),
            1 if skip_plan else 0, _dp(summary), _dp(plan), _dp(log), log_cap, ctypes.byref(log_len), _dp(trace),
            trace_cap, err, 512)
    if rc:
        raise OracleError(rc - 1, err.value.decode())
    k = min(log_len.value, log_cap)
    tl = min(int(summary[15]), trace_cap)
    return OracleResult(int(summary[0]), int(summary[1]), summary[2], summary[3], summary[4], summary[5], summary[6],
                        summary[7], summary[8], summary[9],
                        tuple(summary[11:15]) if summary[10] else None, plan, log[:k].copy(), trace[:tl].copy())


def config_points(config_id: int, n: int, seed: int = 1):
    """BASELINE.json configs[config_id - 1] as points through the fixture
    generator linked into the oracle library (the same synthetic.cpp as
    pot.make_config_points, without loading libpotgpu.so): returns
    (r, c, X, Y, s, cost_scale)."""
    L = lib()
    r, c = np.empty(n), np.empty(n)
    X, Y = np.empty((n, 3)), np.empty((n, 3))
    d = ctypes.c_int(0)
    s, sc = np.empty(1), np.empty(1)
    fn = L.potgpu_make_config
    fn.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_uint64] + [ctypes.POINTER(ctypes.c_double)] * 4 + \
        [ctypes.POINTER(ctypes.c_int)] + [ctypes.POINTER(ctypes.c_double)] * 2
    rc = fn(config_id, n, seed, _dp(r), _dp(c), _dp(X), _dp(Y), ctypes.byref(d), _dp(s), _dp(sc))
    if rc:
        raise OracleError(rc - 1, "invalid config id / size")
    dd = d.value
    X = X.reshape(-1)[: n * dd].reshape(n, dd).copy()
    Y = Y.reshape(-1)[: n * dd].reshape(n, dd).copy()
    return r, c, X, Y, float(s[0]), float(sc[0])


def sweep(C, gamma, u, v, w):
    """Row/col sums, total and max exponent of B(z) at logK = -C/gamma."""
    L = lib()
    n = C.shape[0]
    C = np.ascontiguousarray(C, dtype=np.float64)
    u = np.ascontiguousarray(u, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    row, col = np.empty(n), np.empty(n)
    tot, mx = ctypes.c_double(0), ctypes.c_double(0)
    err = ctypes.create_string_buffer(256)
    fn = L.oracle_sweep
    fn.argtypes = [ctypes.c_long, ctypes.POINTER(ctypes.c_double), ctypes.c_double] + \
        [ctypes.POINTER(ctypes.c_double)] * 2 + [ctypes.c_double] + [ctypes.POINTER(ctypes.c_double)] * 4 + \
        [ctypes.c_char_p, ctypes.c_int]
    rc = fn(n, _dp(C), gamma, _dp(u), _dp(v), w, _dp(row), _dp(col), ctypes.byref(tot), ctypes.byref(mx), err, 256)
    return rc, row, col, tot.value, mx.value


def random_instance(seed, n):
    """test_util.hpp:12-30 with a fresh mt19937_64(seed)."""
    L = lib()
    r, c, C, s = np.empty(n), np.empty(n), np.empty((n, n)), np.empty(1)
    fn = L.oracle_random_instance
    fn.argtypes = [ctypes.c_ulonglong, ctypes.c_long] + [ctypes.POINTER(ctypes.c_double)] * 4
    fn(seed, n, _dp(r), _dp(c), _dp(C), _dp(s))
    return r, c, C, float(s[0])


def make_synthetic(n, seed, mass_r, mass_c, s_frac):
    L = lib()
    r, c, C, s = np.empty(n), np.empty(n), np.empty((n, n)), np.empty(1)
    fn = L.oracle_make_synthetic
    fn.argtypes = [ctypes.c_long, ctypes.c_ulonglong, ctypes.c_double, ctypes.c_double, ctypes.c_double] + \
        [ctypes.POINTER(ctypes.c_double)] * 4
    fn(n, seed, mass_r, mass_c, s_frac, _dp(r), _dp(c), _dp(C), _dp(s))
    return r, c, C, float(s[0])


def run_kats():
    if not os.path.exists(KAT):
        build()
    return subprocess.run([KAT], capture_output=True, text=True)


def kmeans(points, k, seed):
    """kmeans_quantize (color_transfer.hpp:34-118) in the oracle."""
    L = lib()
    pts = np.ascontiguousarray(points, dtype=np.float64)
    n = pts.shape[0]
    C, W = np.zeros((max(k, 1), 3)), np.zeros(max(k, 1))
    A = np.zeros(max(n, 1), dtype=np.int32)
    rounds = ctypes.c_int(0)
    err = ctypes.create_string_buffer(256)
    fn = L.oracle_kmeans
    fn.argtypes = [ctypes.c_long, ctypes.POINTER(ctypes.c_double), ctypes.c_int, ctypes.c_ulonglong,
                   ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int),
                   ctypes.POINTER(ctypes.c_int), ctypes.c_char_p, ctypes.c_int]
    rc = fn(n, _dp(pts) if n else None, int(k), int(seed), _dp(C), _dp(W), A.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
            ctypes.byref(rounds), err, 256)
    if rc:
        raise OracleError(rc - 1, err.value.decode())
    return C[:k], W[:k], A[:n], rounds.value


def round_pot(X, C, r, c, s):
    """round_pot (rounding.hpp:46-77) in the oracle; returns (X_out, cost, gap, mass)."""
    L = lib()
    X = np.ascontiguousarray(X, dtype=np.float64)
    n = X.shape[0]
    C = np.ascontiguousarray(C if C is not None else np.zeros((n, n)), dtype=np.float64)
    out, cgm = np.empty_like(X), np.zeros(3)
    err = ctypes.create_string_buffer(256)
    fn = L.oracle_round_pot
    fn.argtypes = [ctypes.c_long] + [ctypes.POINTER(ctypes.c_double)] * 4 + [ctypes.c_double] + \
        [ctypes.POINTER(ctypes.c_double)] * 2 + [ctypes.c_char_p, ctypes.c_int]
    rc = fn(n, _dp(X), _dp(C), _dp(np.ascontiguousarray(r, dtype=np.float64)),
            _dp(np.ascontiguousarray(c, dtype=np.float64)), float(s), _dp(out), _dp(cgm), err, 256)
    if rc:
        raise OracleError(rc - 1, err.value.decode())
    return out


def round_balanced(X, r, c):
    L = lib()
    X = np.ascontiguousarray(X, dtype=np.float64)
    out = np.empty_like(X)
    err = ctypes.create_string_buffer(256)
    fn = L.oracle_round_balanced
    fn.argtypes = [ctypes.c_long, ctypes.c_long] + [ctypes.POINTER(ctypes.c_double)] * 4 + [ctypes.c_char_p, ctypes.c_int]
    rc = fn(X.shape[0], X.shape[1], _dp(X), _dp(np.ascontiguousarray(r, dtype=np.float64)),
            _dp(np.ascontiguousarray(c, dtype=np.float64)), _dp(out), err, 256)
    if rc:
        raise OracleError(rc - 1, err.value.decode())
    return out
