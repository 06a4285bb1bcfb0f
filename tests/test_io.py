"""File formats (paper_2601_17196_b200/pot_io.py, include/pot/io.hpp):
round trips, the trace CSV header contract (io.hpp:117), error codes."""
import math

import numpy as np
import pytest

from paper_2601_17196_b200 import pot, pot_io


def test_instance_json_and_binary_round_trip(tmp_path):
    inst = pot.make_synthetic_instance(9, 4, 1.0, 1.3, 0.6)
    for name, w, r in (("a.json", pot_io.write_instance_json, pot_io.read_instance_json),
                       ("a.potb", pot_io.write_instance_bin, pot_io.read_instance_bin)):
        w(str(tmp_path / name), inst)
        back = r(str(tmp_path / name))
        assert np.array_equal(back.C, inst.C) and np.array_equal(back.r, inst.r) and np.array_equal(back.c, inst.c)
        assert back.s == inst.s


def test_instance_json_row_form_and_errors(tmp_path):
    p = tmp_path / "rows.json"
    p.write_text('{"r": [0.5, 0.5], "c": [0.5, 0.5], "C": [[0, 1], [1, 0]], "s": 0.5}')
    inst = pot_io.read_instance_json(str(p))
    assert inst.C.tolist() == [[0, 1], [1, 0]]
    p.write_text('{"r": [0.5], "c": [0.5], "s": 0.5}')
    with pytest.raises(pot.PotError) as e:
        pot_io.read_instance_json(str(p))
    assert e.value.code == pot.ErrorCode.IoFailure
    with pytest.raises(pot.PotError) as e:
        pot_io.read_instance_bin(str(tmp_path / "missing.potb"))
    assert e.value.code == pot.ErrorCode.IoFailure


def test_trace_csv_contract():
    recs = [pot.TraceRecord(0, 1.5, -2.0, 0.25, 0.0), pot.TraceRecord(10, 0.125, -1.0, math.nan, 0.5)]
    csv = pot_io.trace_to_csv(recs)
    assert csv.splitlines()[0] == "t,E,phi,rounded_cost,elapsed_s"
    assert csv.splitlines()[1] == "0,1.5,-2,0.25,0"
    assert csv.splitlines()[2] == "10,0.125,-1,,0.5"  # absent rounded cost = empty field


def test_plan_round_trip(tmp_path):
    plan = pot.TransportPlan(X=np.arange(6.0).reshape(2, 3), mass=15.0, row_slack=np.array([0.1, 0.2]),
                             col_slack=np.array([0.3, 0.4, 0.5]))
    pot_io.write_plan_bin(str(tmp_path / "p.bin"), plan)
    back = pot_io.read_plan_bin(str(tmp_path / "p.bin"))
    assert np.array_equal(back.X, plan.X) and back.mass == 15.0 and np.array_equal(back.col_slack, plan.col_slack)


def test_summary_fields_and_exit_codes(tmp_path):
    """summary.json field set (tools/pot_main.cpp:78-97) and exit codes (:337-386)."""
    import json
    from types import SimpleNamespace
    inst = pot.make_synthetic_instance(3, 2, 1.0, 1.0, 0.5)
    res = SimpleNamespace(status=pot.SolveStatus.MaxIterationsExceeded, iterations=4, cost=0.5, final_error=1e-3,
                          tolerance=1e-4, gamma=0.01, wall_seconds=0.1, feasibility_gap=0.0,
                          bounds=pot.TheoryBounds(1.0, 2.0, 0.5, 10.0) if hasattr(pot, "TheoryBounds") else None)
    pot_io.write_summary_json(str(tmp_path / "summary.json"), inst, res, "aspot")
    doc = json.loads((tmp_path / "summary.json").read_text())
    assert set(doc) >= {"solver", "status", "iterations", "cost", "final_error", "tolerance", "gamma", "wall_seconds",
                        "feasibility_gap"}
    assert doc["status"] == "max-iterations-exceeded" and doc["iterations"] == 4
    if res.bounds is not None:
        assert set(doc["theory_bounds"]) == {"R", "L", "mu_f", "iteration_bound"}
    assert pot_io.run_command(lambda: None) == pot_io.EXIT_OK == 0
    assert pot_io.run_command(lambda: pot.validate(pot.Instance(r=np.array([-1.0]), c=np.array([1.0]), s=0.5,
                                                                C=np.zeros((1, 1))))) == pot_io.EXIT_FAILURE == 1
    assert pot_io.EXIT_USAGE == 2


def test_io_header_cpu(tmp_path):
    """include/pot/io.hpp compiled on the host alone (no solve, no GPU)."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "tio")
    subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-I", os.path.join(root, "include"),
                    os.path.join(root, "tests", "cpp", "test_io_cpu.cpp"), "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0 and out.stdout.strip().endswith("OK"), out.stdout + out.stderr
