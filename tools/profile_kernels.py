"""Per-kernel CUDA-event breakdown of one PCAL iteration for a BASELINE config.
usage: python tools/profile_kernels.py [--config C] [--iters K]"""
import argparse, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_03930_b200 as P
from paper_1810_03930_b200.problems import make_instance

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--sharded", action="store_true", help="the row-sharded path on one NCCL rank")
a = ap.parse_args()
t = time.time()
inst = make_instance(a.config, P, threads=os.cpu_count() or 8)
x0 = P.initial_point(inst.n, inst.p, inst.seed ^ 0x1235713)
print(f"config {a.config}: n={inst.n} p={inst.p} setup {time.time()-t:.1f}s", flush=True)
cfg = P.SolverConfig(tol_rel_kkt=float(np.finfo(float).tiny), max_iter=a.iters * 3 + 10,
                     final_orth=False)
if a.sharded:
    comm = P.Comm(1, 0, P.nccl_unique_id(), 0)
    ses = P.ShardedSession(inst.model(P), cfg, x0, comm, inst.n)
else:
    ses = P.Session(inst.model(P), cfg, x0)
with ses as s:
    s.run(3); s.sync()
    prof = s.profile_kernels(a.iters)
    ph = s.profile(a.iters)
tot = sum(prof.values())
for k, v in sorted(prof.items(), key=lambda kv: -kv[1]):
    print(f"  {k:22s} {v*1e3:10.1f} us  {100*v/tot:5.1f}%")
print(f"  {'TOTAL':22s} {tot*1e3:10.1f} us   phases(ms): " + ", ".join(f"{k}={v:.4f}" for k, v in ph.items()))
