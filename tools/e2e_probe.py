"""Breakdown of the fixed per-solve overhead of the drop-in call (config 2)."""
import time, numpy as np, torch
import paper_1810_03930_b200 as P
from paper_1810_03930_b200.problems import make_instance
n = 16384
a_t = torch.empty((n, n), dtype=torch.float64).pin_memory()
inst = make_instance(2, P, threads=16, a_out=a_t.numpy().T)
x0 = P.initial_point(n, 128, inst.seed ^ 0x1235713)
m = inst.model(P)
cfg = P.SolverConfig(tol_rel_kkt=np.finfo(float).tiny, max_iter=50)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    s = P.Session(m, cfg, x0); s.sync(); t1 = time.perf_counter()
    s.run(50); s.sync(); t2 = time.perf_counter()
    r = s.finish(); t3 = time.perf_counter()
    s.close(); t4 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms  run50 {1e3*(t2-t1):.1f} ms  finish {1e3*(t3-t2):.1f} ms  destroy {1e3*(t4-t3):.1f} ms")
t0 = time.perf_counter(); torch.cuda.synchronize()
buf = torch.empty((n, n), dtype=torch.float64, device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter(); buf.copy_(a_t, non_blocking=True); torch.cuda.synchronize()
print(f"H2D 2 GiB pinned: {1e3*(time.perf_counter()-t0):.1f} ms")
