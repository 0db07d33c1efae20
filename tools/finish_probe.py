import numpy as np, torch
import paper_1810_03930_b200 as P
from paper_1810_03930_b200.problems import make_instance
n = 16384
inst = make_instance(2, P, threads=16)
x0 = P.initial_point(n, 128, inst.seed ^ 0x1235713)
r = P.solve(inst.model(P), P.SolverConfig(tol_rel_kkt=np.finfo(float).tiny, max_iter=2), x0)
print(r.status)
