"""bench.py --impl reference (the CPU arm the driver times beside ours): it
runs the oracle port only and never maps libpotgpu.so into the process, and
its `steps` is the number of iterations it actually ran."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROBE = r"""
import io, json, sys, contextlib
sys.argv = ["bench.py", "--impl", "reference", "--n", "512", "--steps", "3", "--ref-budget", "5", "--no-cpu"]
sys.path.insert(0, ".")
import bench
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    bench.main()
maps = open("/proc/self/maps").read()
print(json.dumps({"line": json.loads(buf.getvalue().strip().splitlines()[-1]),
                  "potgpu_mapped": "libpotgpu" in maps, "oracle_mapped": "libpotoracle" in maps}))
"""


def test_reference_arm_is_oracle_only():
    out = subprocess.run([sys.executable, "-c", PROBE], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["oracle_mapped"] and not res["potgpu_mapped"]
    line = res["line"]
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "port"
    assert 1 <= line["steps"] <= 3 and line["steps"] == line["cpu_baseline"]["iterations"]
    assert abs(line["ms_per_step"] - 1000.0 * line["cpu_baseline"]["seconds"] / line["steps"]) < 1e-6


def test_reference_fixture_generator_matches_product():
    """binding.config_points (oracle library) == pot.make_config_points (libpotgpu) bit for bit."""
    import numpy as np
    from oracle import binding
    from paper_2601_17196_b200 import pot
    for cfg in (1, 2, 3, 4, 5):
        a = binding.config_points(cfg, 300, 7)
        b = pot.make_config_points(cfg, 300, 7)
        assert all(np.array_equal(x, y) for x, y in zip(a[:4], b[:4])) and a[4:] == b[4:]
