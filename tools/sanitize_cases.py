"""Small solves touching every kernel family, for compute-sanitizer runs
(memcheck / racecheck / synccheck / initcheck) where the GPU pool allows them
(the round-1 pool refuses compute-sanitizer):

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py

Covers: the persistent small-problem kernel, the graph path (GEMM configs for
p ≤ 32 and p = 64/128, stream-K fixup), the z-marching stencil and the
Kohn–Sham pipeline, the bilinear and density models, MOptQR / dual ascent,
the final CholeskyQR2 + MGS2 fallback, the emulated sharded path (chunk
partials, fixed-tree Gram reduction, halo exchange)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_03930_b200 as P  # noqa: E402
from paper_1810_03930_b200 import harness as H  # noqa: E402

ITERS = int(os.environ.get("SAN_ITERS", "4"))


def cfg(**kw):
    return P.SolverConfig(tol_rel_kkt=np.finfo(float).tiny, max_iter=ITERS, **kw)


def run(name, fn):
    fn()
    print("ok", name, flush=True)


def main():
    dense = lambda n, p, seed: P.QuadraticModel(P.gen_dense_operator(n, seed), p, 2.0 * np.sqrt(n))
    x0 = lambda n, p, seed: P.initial_point(n, p, seed)
    run("dense small kernel", lambda: P.solve(dense(200, 10, 1), cfg(), x0(200, 10, 2)))
    os.environ["PCAL_NO_SMALL_KERNEL"] = "1"
    run("dense graph p=10", lambda: P.solve(dense(200, 10, 1), cfg(), x0(200, 10, 2)))
    run("dense graph p=64", lambda: P.solve(dense(600, 64, 3), cfg(), x0(600, 64, 4)))
    run("dense graph p=128", lambda: P.solve(dense(1100, 128, 5), cfg(), x0(1100, 128, 6)))
    del os.environ["PCAL_NO_SMALL_KERNEL"]
    run("moptqr", lambda: P.solve(dense(300, 8, 7), cfg(algorithm="moptqr"), x0(300, 8, 8)))
    run("pcal-da", lambda: P.solve(dense(300, 8, 7), cfg(algorithm="pcal-da"), x0(300, 8, 8)))
    grid = (16, 16, 8)
    n = 16 * 16 * 8
    v = P.random_uniform(n, 3)
    run("stencil", lambda: P.solve(P.StencilModel(grid, v, 6, 12.0 + v.max()), cfg(), x0(n, 6, 9)))
    run("kohn-sham", lambda: P.solve(P.KohnShamModel(grid, -v, 6, 6.0 + v.max()), cfg(),
                                     x0(n, 6, 10)))
    for kind in ("p4", "p1", "p6"):
        m = H.make_problem(H.ProblemSpec(kind=kind, n=120, p=6, seed=11))
        run(kind, lambda m=m: P.solve(m, cfg(), x0(120, 6, 12)))
    rank_def = np.zeros((64, 4), order="F")
    rank_def[:, 0] = 1.0
    rank_def[:, 1] = 1.0
    rank_def[:, 2] = np.arange(64.0)
    rank_def[:, 3] = 1e-9 * np.arange(64.0) ** 2
    def rank_deficient():
        try:
            P.orthonormalize(rank_def)  # CholeskyQR2 fails, MGS2 runs, rank_error
        except P.RankError:
            return
        raise AssertionError("expected rank_error")
    run("orthonormalize (MGS2 fallback)", rank_deficient)
    run("sharded dense R=2", lambda: P.solve_emulated(dense(700, 20, 13), cfg(), x0(700, 20, 14),
                                                      2))
    run("sharded stencil R=2", lambda: P.solve_emulated(
        P.StencilModel(grid, v, 6, 12.0 + v.max()), cfg(), x0(n, 6, 9), 2))
    m = H.make_problem(H.ProblemSpec(kind="p6", n=300, p=8, seed=15))
    run("sharded p6 R=3", lambda: P.solve_emulated(m, cfg(), x0(300, 8, 16), 3))
    print("all cases ran")


if __name__ == "__main__":
    main()
