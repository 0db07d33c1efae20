import sys, json
sys.path.insert(0, ".")
import paper_1810_03930_b200 as P
from paper_1810_03930_b200.problems import make_instance
for cfg in (3, 4, 5):
    inst = make_instance(cfg, P, threads=16)
    ses = P.Session(inst.model(P), P.SolverConfig(tol_rel_kkt=1e-300, max_iter=20, final_orth=False), 1 ^ 0x1235713)
    ses.run(3); ses.sync()
    kp = ses.profile_kernels(3 if cfg == 5 else 5)
    print(cfg, json.dumps({k: round(v, 4) for k, v in sorted(kp.items(), key=lambda kv: -kv[1])}), flush=True)
    ses.close()
