"""CPU restatement of rigid point-cloud registration — TEST INFRASTRUCTURE ONLY.

Follows /root/reference/proj/include/pot/registration.hpp:
  RigidTransform::apply_all / compose   :21-32
  fit_rigid                             :40-71  (numpy SVD for Eigen's JacobiSVD)
  register_point_clouds                 :127-199
Each round's transport solve runs in the C++ oracle (binding.solve, the
restatement of solvers.hpp); cost build, Procrustes fit and the outer loop
are numpy in the reference's order. Pinned by the reference's own
registration tests (test_apps.cpp FitRigid*, Registration*;
test_acceptance.cpp C11), ported in tests/test_oracle_registration.py.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List

import numpy as np

from . import binding

ZERO_MASS_PLAN = 12  # pot::ErrorCode ordinals (core.hpp:21-39)
DEGENERATE_SVD = 13
DIMENSION_MISMATCH = 0
EMPTY_INPUT = 14
INVALID_ARGUMENT = 15


def apply_all(R, t, pts):
    """(pts * R^T).rowwise() + t^T, three-term dot products in order."""
    out = np.empty_like(pts)
    for d in range(3):
        out[:, d] = ((pts[:, 0] * R[d, 0] + pts[:, 1] * R[d, 1]) + pts[:, 2] * R[d, 2]) + t[d]
    return out


def _matmul3(a, b):
    o = np.empty((3, 3))
    for i in range(3):
        for j in range(3):
            o[i, j] = (a[i, 0] * b[0, j] + a[i, 1] * b[1, j]) + a[i, 2] * b[2, j]
    return o


def _matvec3(a, x):
    return np.array([(a[i, 0] * x[0] + a[i, 1] * x[1]) + a[i, 2] * x[2] for i in range(3)])


def compose(a, b):
    """(a o b)(y) = a(b(y)) (registration.hpp:27-32)."""
    Ra, ta = a
    Rb, tb = b
    return _matmul3(Ra, Rb), _matvec3(Ra, tb) + ta


def fit_rigid(pi, x, y):
    """Weighted Procrustes fit of y onto x under the coupling pi."""
    if x.shape[1] != 3 or y.shape[1] != 3:
        raise binding.OracleError(DIMENSION_MISMATCH, "point clouds must be N x 3")
    if pi.shape != (x.shape[0], y.shape[0]):
        raise binding.OracleError(DIMENSION_MISMATCH, "coupling shape does not match the clouds")
    mass = pi.sum()
    if not mass > 0:
        raise binding.OracleError(ZERO_MASS_PLAN, "coupling carries no mass")
    mean_x = (x.T @ pi.sum(axis=1)) / mass
    mean_y = (y.T @ pi.sum(axis=0)) / mass
    cov = (x - mean_x).T @ pi @ (y - mean_y)
    U, S, Vt = np.linalg.svd(cov)
    if not S[1] > 1e-12 * max(S[0], 1e-300):
        raise binding.OracleError(DEGENERATE_SVD, "cross-covariance has rank < 2; rotation is not determined")
    orient = 1.0 if np.linalg.det(U @ Vt) > 0 else -1.0
    R = U @ np.diag([1.0, 1.0, orient]) @ Vt
    return R, mean_x - R @ mean_y


@dataclass
class Record:
    round: int
    inner_iterations: int
    accumulated_iterations: int
    cost: float
    increment: float
    gamma: float


@dataclass
class Result:
    R: np.ndarray
    t: np.ndarray
    converged: bool
    rounds: List[Record] = field(default_factory=list)


def register_point_clouds(reference, moving, kind=0, alpha=0.4, gamma0=4.4e-3, anneal_rate=0.83,
                          transform_threshold=1e-5, max_registrations=60, epsilon=0.1, max_iterations=50000,
                          log_every=10 ** 9, p=1.0, block_rule=0) -> Result:
    reference = np.ascontiguousarray(reference, dtype=np.float64)
    moving = np.ascontiguousarray(moving, dtype=np.float64)
    if reference.shape[1] != 3 or moving.shape[1] != 3:
        raise binding.OracleError(DIMENSION_MISMATCH, "point clouds must be N x 3")
    if reference.shape[0] < 3 or moving.shape[0] < 3:
        raise binding.OracleError(EMPTY_INPUT, "need at least 3 points per cloud")
    m, n = reference.shape[0], moving.shape[0]
    side = max(m, n)
    r = np.zeros(side)
    r[:m] = 1.0 / side
    c = np.zeros(side)
    c[:n] = 1.0 / side
    s = alpha * min(m, n) / side
    C = np.ones((side, side))
    R, t = np.eye(3), np.zeros(3)
    gamma = gamma0
    acc = 0
    res = Result(R, t, False)
    for rnd in range(1, max_registrations + 1):
        cur = apply_all(R, t, moving)
        d = reference[:, None, :] - cur[None, :, :]
        D2 = (d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2]
        cmax = D2.max()
        if not cmax > 0:
            res.converged = True
            break
        C[:m, :n] = D2 / cmax
        C[:, n:] = 1.0
        C[m:, :] = 1.0
        sol = binding.solve(kind, r, c, s, C=C, epsilon=epsilon, gamma_override=gamma, max_iterations=max_iterations,
                            log_every=log_every, p=p, block_rule=block_rule)
        inc = fit_rigid(sol.plan[:m, :n], reference, cur)
        Rn, tn = compose(inc, (R, t))
        delta = np.sqrt(((Rn - R) ** 2).sum()) + np.sqrt(((tn - t) ** 2).sum())
        R, t = Rn, tn
        acc += sol.iterations
        res.rounds.append(Record(rnd, sol.iterations, acc, sol.cost, delta, gamma))
        gamma *= anneal_rate
        if delta < transform_threshold:
            res.converged = True
            break
    res.R, res.t = R, t
    return res
