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


def test_plan_ppm_xyz_round_trips(tmp_path):
    plan = pot.TransportPlan(X=np.arange(6.0).reshape(2, 3), mass=15.0, row_slack=np.array([0.1, 0.2]),
                             col_slack=np.array([0.3, 0.4, 0.5]))
    pot_io.write_plan_bin(str(tmp_path / "p.bin"), plan)
    back = pot_io.read_plan_bin(str(tmp_path / "p.bin"))
    assert np.array_equal(back.X, plan.X) and back.mass == 15.0 and np.array_equal(back.col_slack, plan.col_slack)
    rgb = np.random.default_rng(1).integers(0, 256, (4, 5, 3), dtype=np.uint8)
    pot_io.write_ppm(str(tmp_path / "i.ppm"), rgb)
    assert np.array_equal(pot_io.read_ppm(str(tmp_path / "i.ppm")), rgb)
    (tmp_path / "c.ppm").write_bytes(b"P6\n# comment\n2 1\n255\n" + bytes(range(6)))
    assert pot_io.read_ppm(str(tmp_path / "c.ppm")).shape == (1, 2, 3)
    pts = np.array([[0.1, 0.2, 0.3], [-1e-300, 5.0, 7.25]])
    pot_io.write_xyz(str(tmp_path / "p.xyz"), pts)
    assert np.array_equal(pot_io.read_xyz(str(tmp_path / "p.xyz")), pts)
