"""The row-sharded product path (csrc/shard.cuh) in TWO processes.

Each process is one rank of a torch.distributed job (gloo) with its own
libpotgpu context on the same GPU; the cross-process reduction of every
sweep goes through the host collective backend (potgpu_comm_init_host,
pot.init_distributed_host: device -> pinned -> torch.distributed.all_reduce
-> device). Everything else is the multi-GPU path exactly: each rank sweeps
its own rows, gathers [rows | cols | max slots], reduces, and runs the
replicated decisions. A SUM of two operands is order independent, so the
two-process job must reproduce the one-process two-shard run
(potgpu_comm_init_local, the same gather + fixed-order device sum) BIT FOR
BIT, and both ranks must return identical results; against the unsharded
oracle the fp64 bars hold (identical decisions, objective 1e-6).
Reference loop being sharded: solvers.hpp:323-369 (ASPOT), :415-481
(extended Sinkhorn: the column LSE's MAX then SUM reduction)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from oracle import binding
from paper_2601_17196_b200 import pot

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import json, os, sys
sys.path.insert(0, %r)
import numpy as np
import torch.distributed as dist
from paper_2601_17196_b200 import pot
from tests.mp_cases import CASES, run_case
dist.init_process_group("gloo")
ctx = pot.Context(0)
pot.init_distributed_host(ctx)
out = {"comm": list(ctx.comm_info())}
for name in CASES:
    out[name] = run_case(name, ctx)
with open(sys.argv[1] + ".%%d.json" %% dist.get_rank(), "w") as f:
    json.dump(out, f)
dist.destroy_process_group()
""" % ROOT


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def two_ranks(tmp_path_factory):
    base = str(tmp_path_factory.mktemp("mp") / "res")
    port = free_port()
    procs = []
    for rank in range(2):
        env = dict(os.environ, RANK=str(rank), WORLD_SIZE="2", LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, "-c", WORKER, base], env=env, cwd=ROOT,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = []
    for p in procs:
        try:
            o, _ = p.communicate(timeout=900)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        outs.append(o)
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o[-4000:]
    return [json.load(open(f"{base}.{r}.json")) for r in range(2)]


def test_both_ranks_identical(two_ranks):
    a, b = two_ranks
    assert a["comm"] == [0, 2, 1] and b["comm"] == [1, 2, 1]
    for name in a:
        if name != "comm":
            assert a[name] == b[name], name


@pytest.mark.parametrize("name", ["aspot_f64", "feasible_f64", "tuned_f64", "aspot_f32_points"])
def test_two_processes_match_two_local_shards_bitwise(two_ranks, name):
    from tests.mp_cases import run_case
    local = run_case(name, pot.Context(0).shard_local(2))
    got = dict(two_ranks[0][name])
    # the plan cost is summed per rank and then across ranks (a scalar
    # host sum), so only it may differ, in its last bits
    gc, lc = got.pop("cost"), local.pop("cost")
    assert abs(gc - lc) <= 1e-14 * abs(lc)
    assert got == local, {k: (got[k], local[k]) for k in got if got[k] != local[k]}


@pytest.mark.parametrize("name", ["aspot_f64", "feasible_f64", "tuned_f64"])
def test_two_processes_match_oracle(two_ranks, name):
    from tests.mp_cases import CASES, oracle_case
    got = two_ranks[0][name]
    o = oracle_case(name)
    assert got["status"] == o.status and got["iterations"] == o.iterations
    if name == "aspot_f64":
        assert np.array_equal(np.array(got["log"])[:, 1:5], o.log[:, 1:5])
    assert abs(got["cost"] - o.cost) <= 1e-6 * abs(o.cost)
    assert got["gap"] <= 1e-7
