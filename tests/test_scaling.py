"""CPU: the GPU scaling harness (run_scaling, harness.cpp:106-138) — report
format (report_io.cpp:138-162), argument checks, the case files the worker
processes load, and the rank-count invariance of the chunk-ordered reduction
the sharded path uses (world size 1 vs 2 over gloo, bitwise)."""
import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1810_03930_b200 as P
from paper_1810_03930_b200 import scaling as S


def test_to_json_matches_reference_keys():
    r = S.ScalingReport(gpus=[1, 2], wall_times=[2.0, 1.0], speedups=[1.0, 2.0],
                        categories=[P.CategoryTimers(0.5, 1.0, 0.1), P.CategoryTimers()],
                        identical_results=True, mode="nccl")
    j = json.loads(S.to_json(r))
    assert set(j) == {"threads", "wall_times", "speedups", "categories", "identical_results",
                      "hardware_oversubscribed", "mode"}
    assert j["threads"] == [1, 2] and j["identical_results"] is True
    assert j["categories"][0] == {"blas3_s": 0.5, "func_s": 1.0, "orth_s": 0.1, "blas3_pct": 25.0,
                                  "func_pct": 50.0, "orth_pct": 5.0}
    assert set(j["categories"][1]) >= {"blas3_s", "func_s", "orth_s"}


def test_gpu_list_must_start_at_one():
    with pytest.raises(P.ParameterError):
        S.run_scaling(None, P.SolverConfig(), None, gpus=[2, 4])
    with pytest.raises(P.ParameterError):
        S.run_scaling(None, P.SolverConfig(), None, gpus=[])


def test_case_file_roundtrip(tmp_path):
    rng = np.random.default_rng(3)
    a = rng.standard_normal((40, 40))
    a = a + a.T
    m = P.QuadraticModel(a, 3, 7.5, g0=rng.standard_normal((40, 3)))
    cfg = P.SolverConfig(max_iter=17, algorithm="plam-da", eta_rule=P.StepsizeRule(kind=2))
    x0 = rng.standard_normal((40, 3))
    path = str(tmp_path / "case.npz")
    S._save_case(path, m, cfg, x0)
    m2, cfg2, x2 = S._load_case(path)
    assert np.array_equal(m2.a, m.a) and np.array_equal(m2.g0, m.g0) and m2.s == 7.5
    assert cfg2 == cfg and np.array_equal(x2, x0)
    st = P.KohnShamModel((8, 8, 4), rng.standard_normal(256), 2, 3.0)
    S._save_case(path, st, cfg, x0)
    st2, _, _ = S._load_case(path)
    assert st2.kind == P.MODEL_KOHN_SHAM and st2.grid == (8, 8, 4) and np.array_equal(st2.v, st.v)


def test_row_chunks_cover_partition():
    """Every rank owns whole chunks (pcal_row_chunks / pcal_partition)."""
    m = P.QuadraticModel(np.zeros((1000, 1000)), 20, 1.0)
    q, nc = P.row_chunks(m)
    assert q % 32 == 0 and (nc - 1) * q < 1000 <= nc * q
    for R in (1, 2, 3, nc):
        parts = [P.partition(m, R, r) for r in range(R)]
        assert sum(nr for _, nr in parts) == 1000
        assert all(r0 % q == 0 for r0, _ in parts)
    with pytest.raises(P.ParameterError):
        P.partition(m, nc + 1, 0)
    g = P.StencilModel((16, 16, 128), np.zeros(16 * 16 * 128), 4, 1.0)
    q, nc = P.row_chunks(g)
    assert q == 2 * 256 and nc == 64  # ⌈128/64⌉ = 2 planes per chunk


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _chunk_ordered_sums(x, g, q, r0, nr):
    """Per-chunk partials of the owned rows: [GᵀX | Σ x∘g per column | Σ x²] (W values)."""
    out = []
    for c0 in range(r0, r0 + nr, q):
        sl = slice(c0, min(c0 + q, r0 + nr))
        out.append(np.concatenate([(g[sl].T @ x[sl]).ravel(), np.sum(x[sl] * g[sl], axis=0),
                                   [np.sum(x[sl] ** 2)]]))
    return np.array(out)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, p = 1000, 6
        rng = np.random.default_rng(11)
        x = rng.standard_normal((n, p)) * np.exp(rng.uniform(-20, 20, (n, 1)))
        g = rng.standard_normal((n, p)) * np.exp(rng.uniform(-20, 20, (n, 1)))
        m = P.QuadraticModel(np.zeros((n, n)), p, 1.0)
        q, nc = P.row_chunks(m)
        r0, nr = P.partition(m, world, rank)
        mine = _chunk_ordered_sums(x, g, q, r0, nr)
        # all-gather with per-rank padding to the largest chunk count, as on the device
        cmax = max(P.partition(m, world, r)[1] for r in range(world))
        cmax = -(-cmax // q)
        pad = np.zeros((cmax, mine.shape[1]))
        pad[: mine.shape[0]] = mine
        bufs = [torch.zeros_like(torch.from_numpy(pad)) for _ in range(world)]
        dist.all_gather(bufs, torch.from_numpy(pad))
        counts = [-(-P.partition(m, world, r)[1] // q) for r in range(world)]
        total = np.zeros(mine.shape[1])
        for r in range(world):  # sequential, global chunk order
            for c in range(counts[r]):
                total = total + bufs[r].numpy()[c]
        ref = np.zeros(mine.shape[1])
        for row in _chunk_ordered_sums(x, g, q, 0, n):  # one rank owning every chunk
            ref = ref + row
        out[rank] = (total.tobytes() == ref.tobytes(), sum(counts) == nc)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_chunk_ordered_reduction_is_rank_count_invariant_gloo(world):
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert all(res[r] == (True, True) for r in range(world))
