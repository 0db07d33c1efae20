"""CPU, world_size 2 (gloo): the row-sharding decomposition of DESIGN.md §6.
Each rank takes its rows from the library's own partition (pcal_partition, a
host function) and computes the per-iteration partials of C1–C4 on its rows;
the gloo allreduce of the partials must equal the unsharded quantities, and
the slabs must tile the rows exactly."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    import paper_1810_03930_b200 as P
    try:
        grid, p = (8, 8, 6), 5
        n = grid[0] * grid[1] * grid[2]
        rng = np.random.default_rng(0)
        x = np.asfortranarray(rng.standard_normal((n, p)))
        xp = np.asfortranarray(rng.standard_normal((n, p)))
        g = np.asfortranarray(rng.standard_normal((n, p)))
        gp = np.asfortranarray(rng.standard_normal((n, p)))
        d, dp = rng.standard_normal(p), rng.standard_normal(p)
        m = P.StencilModel(grid, np.zeros(n), p, 1.0)
        r0, nr = P.partition(m, world, rank)
        sl = slice(r0, r0 + nr)
        # C1: [GᵀX; XᵀX] partials; C2: column f / kkt² / d partials; C3: ss, sy, yy; C4: ‖z_j‖²
        gl, gpl = g - d * x, gp - dp * xp
        parts = np.concatenate([
            (g[sl].T @ x[sl]).ravel(), (x[sl].T @ x[sl]).ravel(),
            np.sum(x[sl] * g[sl], axis=0), np.sum((g[sl] - x[sl]) ** 2, axis=0),
            [np.sum((x[sl] - xp[sl]) ** 2), np.sum((x[sl] - xp[sl]) * (gl[sl] - gpl[sl])),
             np.sum((gl[sl] - gpl[sl]) ** 2)],
            np.sum((x[sl] - 0.25 * gl[sl]) ** 2, axis=0)])
        t = torch.from_numpy(parts.copy())
        dist.all_reduce(t)
        full = np.concatenate([
            (g.T @ x).ravel(), (x.T @ x).ravel(), np.sum(x * g, axis=0),
            np.sum((g - x) ** 2, axis=0),
            [np.sum((x - xp) ** 2), np.sum((x - xp) * (gl - gpl)), np.sum((gl - gpl) ** 2)],
            np.sum((x - 0.25 * gl) ** 2, axis=0)])
        rows = torch.tensor([r0, nr], dtype=torch.int64)
        allrows = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allrows, rows)
        out[rank] = (float(np.max(np.abs(t.numpy() - full) / (1 + np.abs(full)))),
                     [tuple(r.tolist()) for r in allrows], nr % (grid[0] * grid[1]))
    finally:
        dist.destroy_process_group()


def test_row_sharded_partials_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for rank in range(world):
        err, rows, rem = res[rank]
        assert err <= 1e-12
        assert rem == 0  # whole z-planes
        assert rows[0][0] == 0 and rows[0][0] + rows[0][1] == rows[1][0]
        assert rows[1][0] + rows[1][1] == 8 * 8 * 6
