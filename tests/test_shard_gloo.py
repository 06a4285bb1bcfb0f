"""The multi-GPU decomposition (csrc/shard.cuh) checked on CPU with two
`gloo` ranks: each rank evaluates its row block of B(z) with the CPU oracle,
folds it into the all-reduce layout [rows (own; 0 elsewhere) | cols | max
slot per shard], and one SUM all-reduce must reproduce the unsharded
evaluation — row sums and max exponent bit for bit, column sums to
reassociation. The Sinkhorn column LSE (MAX all-reduce, rescale, SUM
all-reduce) must equal the full log-sum-exp. Also the NCCL-id broadcast the
GPU ranks use (pot.init_distributed) and the shard split."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import binding
from paper_2601_17196_b200 import pot

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, port, n, out_dir):
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        # the NCCL id travels exactly as in pot.init_distributed
        box = [pot.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        ids = [None] * WORLD
        dist.all_gather_object(ids, box[0])
        assert len(ids[0]) == 128 and ids[0] == ids[1]

        r, c, C, s = binding.random_instance(4242, n)
        rng = np.random.default_rng(7)
        u, v, w = rng.uniform(-3, 1, n), rng.uniform(-3, 1, n), float(rng.uniform(-1, 1))
        gamma = 0.05
        lo, hi = pot.shard_rows(n, WORLD)[rank]
        # this rank's rows of B(z): the oracle's own sweep with the other
        # rows masked (u = -inf: their entries hit the exp clamp floor,
        # ~1e-308, far below the column sums' last bit)
        um = np.full(n, -np.inf)
        um[lo:hi] = u[lo:hi]
        rc, row, col, tot, mx = binding.sweep(C, gamma, um, v, w)
        assert rc == 0
        vec = np.zeros(2 * n + WORLD)
        vec[lo:hi] = row[lo:hi]
        vec[n:2 * n] = col
        vec[2 * n + rank] = mx
        t = torch.from_numpy(vec)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        red = t.numpy()
        # Sinkhorn column LSE of x_ij = logK_ij + u_i over this rank's rows
        x = (-C[lo:hi]) / gamma + u[lo:hi, None]
        m = x.max(axis=0)
        S = np.exp(x - m).sum(axis=0)
        tm = torch.from_numpy(m.copy())
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        M = tm.numpy()
        tS = torch.from_numpy(S * np.exp(m - M))
        dist.all_reduce(tS, op=dist.ReduceOp.SUM)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), red=red, lse=M + np.log(tS.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [7, 130])
def test_two_rank_reduction_reproduces_unsharded(tmp_path, n):
    mp.start_processes(_rank_main, args=(_free_port(), n, str(tmp_path)), nprocs=WORLD, join=True, start_method="spawn")
    a, b = (np.load(tmp_path / f"rank{k}.npz") for k in range(WORLD))
    np.testing.assert_array_equal(a["red"], b["red"])  # every rank sees the same vector
    np.testing.assert_array_equal(a["lse"], b["lse"])
    r, c, C, s = binding.random_instance(4242, n)
    rng = np.random.default_rng(7)
    u, v, w = rng.uniform(-3, 1, n), rng.uniform(-3, 1, n), float(rng.uniform(-1, 1))
    rc, row, col, tot, mx = binding.sweep(C, 0.05, u, v, w)
    red = a["red"]
    np.testing.assert_array_equal(red[:n], row)  # own rows + exact zeros
    np.testing.assert_allclose(red[n:2 * n], col, rtol=1e-14)
    assert red[2 * n:].max() == mx
    x = (-C) / 0.05 + u[:, None]
    full = x.max(axis=0) + np.log(np.exp(x - x.max(axis=0)).sum(axis=0))
    np.testing.assert_allclose(a["lse"], full, rtol=1e-14)


@pytest.mark.parametrize("n,world,per", [(10, 3, 1), (5, 4, 2), (16384, 8, 1), (1, 2, 1)])
def test_shard_rows_partition(n, world, per):
    rows = pot.shard_rows(n, world, per)
    assert len(rows) == world * per
    assert rows[0][0] == 0 and rows[-1][1] == n
    for (a, b), (c, d) in zip(rows, rows[1:]):
        assert b == c and a <= b
    sizes = [b - a for a, b in rows]
    assert max(sizes) - min(sizes) <= 1
