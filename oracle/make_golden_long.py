"""Long parity windows and the config-5 shape (tests/golden/long_*.npz).

Run in the build container (where /root/reference exists), in the background:
    python -m oracle.make_golden_long cfg5s cfg2 grids40 gridsfull ens2

Two generators are used, and each fixture says which:
  * ``reference`` — the UNMODIFIED reference solve() (oracle/_ref), driving the
    restated grid operator for the stencil / Kohn–Sham models.  Used for the
    config-5 shape (p = 1024) and the 40-iteration windows of configs 3 and 4.
  * ``port`` — the C restatement (oracle/pcal_oracle.c + orc_blas.c), bitwise
    equal to the reference (tests/test_oracle_golden.py; each long run below
    also re-checks its first iterations against a reference-generated trace
    before it is written).  Used where the reference itself needs hours: config
    2's full 500 iterations (≈80 min in the reference) and its 1-ulp ensemble
    (K = 8 more runs), the full runs of configs 3 and 4.

Large matrices are stored as row samples (every ``ROW_STRIDE``-th row plus the
first 8), never whole.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

from oracle.oracle import Config, Model, Reference, Restatement, MODEL_STENCIL, MODEL_KOHN_SHAM
from oracle.oracle import MODEL_DENSE

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
TINY = float(np.finfo(float).tiny)
INIT_SALT = 0x1235713
TH = int(os.environ.get("GOLDEN_THREADS", os.cpu_count() or 8))


def rows_of(x: np.ndarray, stride: int) -> np.ndarray:
    """First 8 rows + every stride-th row (the sample the GPU tests compare)."""
    idx = np.unique(np.concatenate([np.arange(min(8, x.shape[0])), np.arange(0, x.shape[0], stride)]))
    return idx, np.ascontiguousarray(x[idx])


def grid_instance(O: Restatement, kind: int, grid, seed: int = 1):
    from paper_1810_03930_b200.problems import ks_potential
    n = grid[0] * grid[1] * grid[2]
    if kind == MODEL_STENCIL:
        v = O.random_uniform(n, seed)
        s = 12.0 + float(np.max(v))
    else:
        v = ks_potential(grid, seed, O)
        s = 6.0 + float(np.max(np.abs(v)))
    return n, v, s


def save(name: str, g: dict) -> None:
    path = os.path.join(OUT, name)
    np.savez_compressed(path, **g)
    print("wrote", path, flush=True)


def pack(prefix: str, rep, g: dict, stride: int) -> None:
    g[prefix + "trace"] = rep.trace[:, :6]
    g[prefix + "final_pre"] = rep.final_pre
    g[prefix + "final_post"] = rep.final_post if rep.final_post is not None else np.full(4, np.nan)
    g[prefix + "iterations"] = rep.iterations
    g[prefix + "status"] = rep.status
    g[prefix + "degenerate_steps"] = rep.degenerate_steps
    if rep.stop_x is not None:
        idx, g[prefix + "stop_x_rows"] = rows_of(rep.stop_x, stride)
        _, g[prefix + "final_x_rows"] = rows_of(rep.final_x, stride)
        g[prefix + "row_idx"] = idx


def cfg5_shape() -> None:
    """Config 5's operator and p = 1024 on grids the reference finishes in
    minutes: 32³ (n = 32768) and 16³ (n = 4096 = 4p: ragged GEMM edges), 5 PCAL
    iterations + the final CholeskyQR2, by the unmodified reference solve()."""
    R, O = Reference(), Restatement()
    g = {"generator": "reference"}
    for name, grid, iters in [("g16", (16, 16, 16), 5), ("g32", (32, 32, 32), 5)]:
        n, v, s = grid_instance(O, MODEL_STENCIL, grid)
        x0 = O.initial_point_qr(n, 1024, 1 ^ INIT_SALT, threads=TH)
        t = time.time()
        rep = R.solve(Model(MODEL_STENCIL, n, 1024, s, grid=grid, v=v),
                      Config(tol_rel_kkt=TINY, max_iter=iters, threads=TH, final_orth=True), x0)
        print(name, "reference", iters, "iterations:", time.time() - t, flush=True)
        g[name + "_s"] = s
        pack(name + "_", rep, g, 512)
        # the port on the same instance must agree bitwise (pins it for the GPU
        # tests, which rebuild the oracle states with the fast port)
        t = time.time()
        rp = O.solve(Model(MODEL_STENCIL, n, 1024, s, grid=grid, v=v),
                     Config(tol_rel_kkt=TINY, max_iter=iters, threads=TH, final_orth=True), x0)
        print(name, "port:", time.time() - t, flush=True)
        assert np.array_equal(rp.trace[:, :6], rep.trace[:, :6]), name
        assert np.array_equal(rp.final_x, rep.final_x), name
    save("long_cfg5_shape.npz", g)


def cfg2_full() -> None:
    """Config 2: the full 500 iterations + final orthonormalisation (port)."""
    from paper_1810_03930_b200.problems import REFERENCE_S
    O = Restatement()
    pre = np.load(os.path.join(OUT, "reference_cfg2.npz"))
    m = O.dense_trace_min(16384, 128, 1, s=REFERENCE_S[(16384, 1)], threads=TH)
    x0 = O.initial_point_qr(16384, 128, 1 ^ INIT_SALT, threads=TH)
    t = time.time()
    rep = O.solve(m, Config(tol_rel_kkt=TINY, max_iter=500, threads=TH, final_orth=True), x0)
    print("cfg2 port 500:", time.time() - t, flush=True)
    ref_tr = pre["cfg2_trace"]
    assert np.array_equal(rep.trace[: ref_tr.shape[0], :6], ref_tr), "port != reference prefix"
    g = {"generator": "port", "s": m.s}
    pack("base_", rep, g, 64)
    save("long_cfg2.npz", g)


def ensemble2(k: int = 8) -> None:
    """Config 2: K runs from X0 with one entry moved by one ulp (probe 3's
    perturbation), the spread the end-of-run KKT / feasibility / X must sit in."""
    from paper_1810_03930_b200.problems import REFERENCE_S
    O = Restatement()
    path = os.path.join(OUT, "long_cfg2.npz")
    g = dict(np.load(path))
    m = O.dense_trace_min(16384, 128, 1, s=REFERENCE_S[(16384, 1)], threads=TH)
    x0 = O.initial_point_qr(16384, 128, 1 ^ INIT_SALT, threads=TH)
    rows = []
    for q in range(int(g.get("ens_done", 0)), k):
        xp = x0.copy(order="F")
        flat = xp.reshape(-1, order="F")
        e = (q * 2654435761) % flat.size
        flat[e] = np.nextafter(flat[e], np.inf if q % 2 == 0 else -np.inf)
        xp = flat.reshape(x0.shape, order="F")
        t = time.time()
        rep = O.solve(m, Config(tol_rel_kkt=TINY, max_iter=500, threads=TH, final_orth=True), xp)
        print("ens", q, time.time() - t, rep.final_pre, rep.final_post, flush=True)
        g[f"ens{q}_final_pre"] = rep.final_pre
        g[f"ens{q}_final_post"] = rep.final_post
        _, g[f"ens{q}_final_x_rows"] = rows_of(rep.final_x, 64)
        _, g[f"ens{q}_stop_x_rows"] = rows_of(rep.stop_x, 64)
        g[f"ens{q}_trace"] = rep.trace[:, :6]
        g["ens_done"] = q + 1
        save("long_cfg2.npz", g)  # after every member: partial ensembles survive


def grids40() -> None:
    """Configs 3 and 4 at full size: 40 iterations of the unmodified reference
    solve() driving the restated operators (SURVEY §8(c) trace window)."""
    R, O = Reference(), Restatement()
    g = {"generator": "reference"}
    for name, kind, grid, p in [("cfg3", MODEL_STENCIL, (64, 64, 64), 256),
                                ("cfg4", MODEL_KOHN_SHAM, (48, 48, 48), 512)]:
        n, v, s = grid_instance(O, kind, grid)
        x0 = O.initial_point_qr(n, p, 1 ^ INIT_SALT, threads=TH)
        t = time.time()
        rep = R.solve(Model(kind, n, p, s, grid=grid, v=v),
                      Config(tol_rel_kkt=TINY, max_iter=40, threads=TH, final_orth=False), x0)
        print(name, "reference 40:", time.time() - t, flush=True)
        g[name + "_s"] = s
        pack(name + "_", rep, g, 1024)
        save("long_grids40.npz", g)


def grids_full() -> None:
    """Configs 3 (300 iterations) and 4 (200) end to end with the port, after
    checking its first 40 iterations bitwise against long_grids40.npz."""
    O = Restatement()
    w = np.load(os.path.join(OUT, "long_grids40.npz"))
    g = {"generator": "port"}
    for name, kind, grid, p, iters in [("cfg3", MODEL_STENCIL, (64, 64, 64), 256, 300),
                                       ("cfg4", MODEL_KOHN_SHAM, (48, 48, 48), 512, 200)]:
        n, v, s = grid_instance(O, kind, grid)
        x0 = O.initial_point_qr(n, p, 1 ^ INIT_SALT, threads=TH)
        t = time.time()
        rep = O.solve(Model(kind, n, p, s, grid=grid, v=v),
                      Config(tol_rel_kkt=TINY, max_iter=iters, threads=TH, final_orth=True), x0)
        print(name, "port", iters, time.time() - t, flush=True)
        ref = w[name + "_trace"]
        assert np.array_equal(rep.trace[: ref.shape[0], :6], ref), name + ": port != reference"
        pack(name + "_", rep, g, 1024)
        save("long_grids_full.npz", g)


def ensemble_grids(k: int = 4) -> None:
    """Configs 3 and 4: K runs of the port from X0 with one entry moved by one
    ulp (the spread the end of run must sit in), appended to long_grids_full.npz."""
    O = Restatement()
    path = os.path.join(OUT, "long_grids_full.npz")
    g = dict(np.load(path))
    for name, kind, grid, p, iters in [("cfg3", MODEL_STENCIL, (64, 64, 64), 256, 300),
                                       ("cfg4", MODEL_KOHN_SHAM, (48, 48, 48), 512, 200)]:
        n, v, s = grid_instance(O, kind, grid)
        x0 = O.initial_point_qr(n, p, 1 ^ INIT_SALT, threads=TH)
        for q in range(int(g.get(name + "_ens_done", 0)), k):
            flat = x0.reshape(-1, order="F").copy()
            e = (q * 2654435761) % flat.size
            flat[e] = np.nextafter(flat[e], np.inf if q % 2 == 0 else -np.inf)
            xp = flat.reshape(x0.shape, order="F")
            t = time.time()
            rep = O.solve(Model(kind, n, p, s, grid=grid, v=v),
                          Config(tol_rel_kkt=TINY, max_iter=iters, threads=TH, final_orth=True), xp)
            print(name, "ens", q, time.time() - t, rep.final_pre, rep.final_post, flush=True)
            g[f"{name}_ens{q}_final_pre"] = rep.final_pre
            g[f"{name}_ens{q}_final_post"] = rep.final_post
            _, g[f"{name}_ens{q}_final_x_rows"] = rows_of(rep.final_x, 1024)
            g[name + "_ens_done"] = q + 1
            save("long_grids_full.npz", g)


JOBS = {"cfg5s": cfg5_shape, "cfg2": cfg2_full, "grids40": grids40, "gridsfull": grids_full,
        "ens2": ensemble2, "ensgrids": ensemble_grids}

if __name__ == "__main__":
    for job in sys.argv[1:]:
        t0 = time.time()
        JOBS[job]()
        print(f"== {job} done in {time.time() - t0:.0f} s", flush=True)
