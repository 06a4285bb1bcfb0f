"""Exact partial-OT value by LP (the reference's oracle.hpp:181-199 solves the
same LP with a dense simplex; here scipy's HiGHS). Test infrastructure."""
import numpy as np
from scipy.optimize import linprog


def solve_exact(r, c, C, s):
    n = len(r)
    A_ub = np.zeros((2 * n, n * n))
    for i in range(n):
        A_ub[i, i * n:(i + 1) * n] = 1.0          # row sums <= r
        A_ub[n + i, i::n] = 1.0                   # col sums <= c
    b_ub = np.concatenate([r, c])
    A_eq = np.ones((1, n * n))
    res = linprog(C.reshape(-1), A_ub=A_ub, b_ub=b_ub, A_eq=A_eq, b_eq=[s], bounds=(0, None), method="highs")
    assert res.status == 0, res.message
    return res.fun, res.x.reshape(n, n)
