"""Run-to-run determinism: the same solve three times in one process, traces compared bitwise.

    python tools/determinism_probe.py 5:6 3:300   (config:iterations ...)
"""
import sys, time, os
sys.path.insert(0, ".")
import numpy as np
import paper_1810_03930_b200 as P
from paper_1810_03930_b200.problems import make_instance
for spec in sys.argv[1:]:
    cfg, iters = (int(v) for v in spec.split(":"))
    inst = make_instance(cfg, P, threads=16)
    m = inst.model(P)
    x0 = P.initial_point(inst.n, inst.p, 1 ^ 0x1235713)
    tr = []
    for rep in range(3):
        r = P.solve(m, P.SolverConfig(tol_rel_kkt=1e-300, max_iter=iters, final_orth=False), x0)
        tr.append(r.trace[:, :6].copy())
    for rep in (1, 2):
        a, b = tr[0], tr[rep]
        same = a.shape == b.shape and np.array_equal(a, b)
        first = None
        if not same:
            k = min(a.shape[0], b.shape[0])
            bad = np.nonzero(~np.all(a[:k] == b[:k], axis=1))[0]
            first = int(bad[0]) if len(bad) else k
        print(f"cfg {cfg} iters {iters} run0 vs run{rep}: identical={same} first_diff_row={first}",
              flush=True)
        if first is not None:
            print("   ", a[first].tolist(), "\n   ", b[first].tolist(), flush=True)
