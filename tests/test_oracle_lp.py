"""C01 (test_acceptance.cpp:104-146; test_solvers.cpp:209-223, 356-371,
431-444, 463-478): every solver is an eps-approximation of the exact POT
value, feasible to 1e-9, and the three solvers agree within 2 eps —
checked on the CPU oracle against an exact LP."""
import numpy as np
import pytest

from oracle import binding
from tests.lp import solve_exact


@pytest.mark.parametrize("seed", range(1000, 1012))
def test_oracle_eps_approximation(seed):
    n = 3 + (seed % 6)
    r, c, C, s = binding.random_instance(seed, n)
    opt, _ = solve_exact(r, c, C, s)
    eps = 0.1
    costs = []
    for kind, p in ((0, 1.0), (1, 1.0), (2, 2.0)):
        res = binding.solve(kind, r, c, s, C=C, epsilon=eps, p=p, max_iterations=200000)
        assert res.status == 0
        assert res.feasibility_gap <= 1e-9 * max(1.0, r.sum())
        assert res.cost <= opt + eps + 1e-9
        assert res.cost >= opt - 1e-9
        costs.append(res.cost)
    for a in range(3):
        for b in range(a + 1, 3):
            assert abs(costs[a] - costs[b]) <= 2 * eps + 1e-9
