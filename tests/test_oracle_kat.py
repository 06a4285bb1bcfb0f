"""Pins the CPU oracle against every known-answer test the reference's own
suites hold for this path (proj/tests/test_{dual,solvers,extend_rounding,
core}.cpp hand values), ported GTest-free in oracle/kat_main.cpp."""
from oracle import binding


def test_oracle_known_answer_tests():
    res = binding.run_kats()
    assert res.returncode == 0, res.stdout[-4000:]
    assert " 0 failures" in res.stdout
    # every ported reference case ran
    assert res.stdout.count("PASS ") >= 60, res.stdout


def test_synthetic_generator_matches_oracle_restatement():
    """The library's make_synthetic_instance draws exactly like the
    oracle's restatement of synthetic.hpp:15-54 (bit-exact)."""
    import numpy as np
    from paper_2601_17196_b200 import pot
    for n, seed in ((1, 3), (7, 5), (40, 5)):
        inst = pot.make_synthetic_instance(n, seed, 5.0, 3.0, 0.2)
        r, c, C, s = binding.make_synthetic(n, seed, 5.0, 3.0, 0.2)
        assert np.array_equal(inst.r, r) and np.array_equal(inst.c, c)
        assert np.array_equal(inst.C, C) and inst.s == s
