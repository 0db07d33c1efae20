"""GPU scaling harness: ``run_scaling`` over GPU counts.

The reference's ``run_scaling`` (harness.cpp:106-138) re-runs one cell at
thread counts 1, m₂, m₃, …, records wall time, speedup and the blas3 / func /
orth categories per count, and asserts that every run is bitwise identical to
the first (``same_numerics``).  Its report is ``ScalingReport``
(report.hpp:74-82) written by ``to_json(ScalingReport)`` (report_io.cpp:138-162).

Here the axis is the number of GPUs (ranks) of the row-sharded path.  Its
reductions are taken per fixed global row chunk and summed in chunk order
(DESIGN.md §6), so ``identical_results`` holds across GPU counts exactly as
it holds across thread counts in the reference.  Two launch modes:

* ``"nccl"`` — one process per GPU: for every count, ``torch.distributed.run``
  starts ``python -m paper_1810_03930_b200.scaling --worker`` on that many
  GPUs; each rank solves its row slab (``solve_sharded``) over NCCL.
* ``"emulated"`` — the R ranks run as host threads on one GPU with loopback
  collectives (``solve_emulated``): the same kernels and the same reduction
  order, so ``identical_results`` is meaningful; wall times are not (every
  rank shares the GPU), which ``hardware_oversubscribed`` records, like the
  reference's flag for more threads than hardware threads (harness.cpp:113-118).

CLI (the reference's scaling study on a BASELINE config):
    python -m paper_1810_03930_b200.scaling --config 3 --gpus 1,2,4,8 --iters 50 \
        [--mode nccl|emulated] [--out scaling.json]
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import tempfile
from dataclasses import asdict, dataclass, field
from typing import List, Optional

import numpy as np

import paper_1810_03930_b200 as P
from paper_1810_03930_b200 import report_io

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@dataclass
class ScalingReport:
    """ScalingReport (report.hpp:74-82); ``gpus`` replaces ``threads``."""
    gpus: List[int] = field(default_factory=list)
    wall_times: List[float] = field(default_factory=list)
    speedups: List[float] = field(default_factory=list)
    categories: List[P.CategoryTimers] = field(default_factory=list)
    runs: List[P.RunReport] = field(default_factory=list)
    identical_results: bool = False
    hardware_oversubscribed: bool = False
    mode: str = "emulated"


def visible_gpus() -> int:
    return P.device_count()


# ---- case files: the model / config / start point every worker process loads ----
def _save_case(path: str, model, config: P.SolverConfig, x0) -> None:
    d = {"kind": model.kind, "n": model.n, "p": model.p, "s": model.s,
         "x0": np.asfortranarray(x0, dtype=np.float64),
         "config": json.dumps(asdict(config))}
    if model.kind in (P.MODEL_DENSE, P.MODEL_BILINEAR, P.MODEL_DENSITY):
        if model.location != P.HOST:
            raise P.ParameterError("run_scaling: the model must live in host memory")
        d["a"] = model.a
        if model.kind == P.MODEL_DENSE and model.g0 is not None:
            d["g0"] = model.g0
        if model.kind == P.MODEL_BILINEAR:
            d["b"] = model.b
        if model.kind == P.MODEL_DENSITY:
            d["linv"] = model.linv
            d["coeff"] = model.coeff
            d["variant"] = model.variant
            d["mode"] = model.mode
    elif model.kind in (P.MODEL_STENCIL, P.MODEL_KOHN_SHAM):
        d["grid"] = np.array(model.grid)
        d["v"] = model.v
    else:
        raise P.ParameterError("run_scaling: device-callback models are single-GPU")
    np.savez(path, **d)


def _load_case(path: str):
    z = np.load(path)
    kind = int(z["kind"])
    p, s = int(z["p"]), float(z["s"])
    if kind == P.MODEL_DENSE:
        model = P.QuadraticModel(z["a"], p, s, g0=z["g0"] if "g0" in z else None)
    elif kind == P.MODEL_BILINEAR:
        model = P.BilinearModel(z["a"], z["b"], s)
    elif kind == P.MODEL_DENSITY:
        model = P.DensityModel(z["a"], p, float(z["coeff"]), s, variant=str(z["variant"]),
                               linv=z["linv"], mode=str(z["mode"]))
    elif kind == P.MODEL_STENCIL:
        model = P.StencilModel(tuple(z["grid"]), z["v"], p, s)
    else:
        model = P.KohnShamModel(tuple(z["grid"]), z["v"], p, s)
    c = json.loads(str(z["config"]))
    c["eta_rule"] = P.StepsizeRule(**c["eta_rule"])
    c["alm"] = P.AlmOptions(**c["alm"])
    return model, P.SolverConfig(**c), np.asfortranarray(z["x0"])


def _local_model(model, r0: int, nr: int):
    """The LOCAL slab of the model a sharded session takes (pcal_b200.h)."""
    if model.kind == P.MODEL_DENSE:
        g0 = None if model.g0 is None else np.asfortranarray(model.g0[r0:r0 + nr])
        return P.QuadraticModel(np.asfortranarray(model.a[r0:r0 + nr, :]), model.p, model.s,
                                g0=g0, n=model.n)
    if model.kind == P.MODEL_BILINEAR:
        return P.BilinearModel(np.asfortranarray(model.a[r0:r0 + nr, :]), model.b, model.s,
                               n=model.n)
    if model.kind == P.MODEL_DENSITY:
        return P.DensityModel(np.asfortranarray(model.a[r0:r0 + nr, :]), model.p, model.coeff,
                              model.s, variant=model.variant,
                              linv=np.asfortranarray(model.linv[r0:r0 + nr, :]), n=model.n)
    cls = P.KohnShamModel if model.kind == P.MODEL_KOHN_SHAM else P.StencilModel
    return cls(model.grid, model.v[r0:r0 + nr], model.p, model.s)


def _worker(case: str, out: str) -> None:
    """One rank of one scaling run (launched by torch.distributed.run)."""
    import torch
    import torch.distributed as dist
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")  # only to broadcast the NCCL id and gather rows
    model, config, x0 = _load_case(case)
    config.device = local
    obj = [P.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    comm = P.Comm(world, rank, obj[0], local)
    r0, nr = P.partition(model, world, rank)
    timers = P.CategoryTimers()
    rep = P.solve_sharded(_local_model(model, r0, nr), config, x0[r0:r0 + nr], comm, nr,
                          timers=timers)
    comm.close()
    # every rank writes its rows; rank 0 adds the replicated report
    d = {"row0": r0}
    if rep.stop_iterate is not None:
        d["stop_x"] = rep.stop_iterate
    if rep.final_x is not None:
        d["final_x"] = rep.final_x
    np.savez(f"{out}.rank{rank}.npz", **d)
    if rank == 0:
        f = rep.final_pre_orth
        d = {"trace": rep.trace, "iterations": rep.iterations, "world": world,
             "degenerate_steps": rep.degenerate_steps, "wall_time": rep.wall_time,
             "status": rep.status, "beta": rep.beta, "eta0": rep.eta0,
             "pre": np.array([f.fval, f.kkt_abs, f.kkt_rel, f.feas]),
             "timers": np.array([timers.blas3, timers.func, timers.orth]), "n": model.n}
        if rep.final_post_orth is not None:
            f = rep.final_post_orth
            d["post"] = np.array([f.fval, f.kkt_abs, f.kkt_rel, f.feas])
        np.savez(out, **d)
    dist.barrier()
    dist.destroy_process_group()


def _read_run(path: str, p: int):
    z = np.load(path, allow_pickle=False)
    n, world = int(z["n"]), int(z["world"])
    xs = {}
    for r in range(world):
        zr = np.load(f"{path}.rank{r}.npz")
        for key in ("stop_x", "final_x"):
            if key in zr:
                m = xs.setdefault(key, np.zeros((n, p), order="F"))
                r0 = int(zr["row0"])
                m[r0:r0 + zr[key].shape[0]] = zr[key]
    post = P.FinalMetrics(*z["post"]) if "post" in z else None
    rep = P.RunReport(trace=z["trace"], final_pre_orth=P.FinalMetrics(*z["pre"]),
                      final_post_orth=post, stop_iterate=xs.get("stop_x"),
                      final_x=xs.get("final_x"), iterations=int(z["iterations"]),
                      degenerate_steps=int(z["degenerate_steps"]),
                      wall_time=float(z["wall_time"]), status=str(z["status"]),
                      beta=float(z["beta"]), eta0=float(z["eta0"]))
    t = z["timers"]
    return rep, P.CategoryTimers(float(t[0]), float(t[1]), float(t[2]))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run_nccl(model, config, x0, g: int, workdir: str, timeout: float):
    case = os.path.join(workdir, "case.npz")
    if not os.path.exists(case):
        _save_case(case, model, config, x0)
    out = os.path.join(workdir, f"run_{g}.npz")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={g}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           "-m", "paper_1810_03930_b200.scaling", "--worker", case, out]
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    subprocess.run(cmd, check=True, env=env, timeout=timeout, cwd=ROOT)
    return _read_run(out, model.p)


def run_scaling(model, config: P.SolverConfig, x0, gpus=(1, 2, 4), mode: Optional[str] = None,
                timeout: float = 1800.0) -> ScalingReport:
    """run_scaling (harness.cpp:106-138) over GPU counts ``gpus`` (must start at 1)."""
    gpus = [int(g) for g in gpus]
    if not gpus or gpus[0] != 1:
        raise P.ParameterError("run_scaling: GPU list must start at 1")
    if any(g < 1 for g in gpus):
        raise P.ParameterError("run_scaling: GPU counts must be positive")
    have = visible_gpus()
    if mode is None:
        mode = "nccl" if have >= max(gpus) and max(gpus) > 1 else "emulated"
    if mode not in ("nccl", "emulated"):
        raise P.ParameterError(f"run_scaling: unknown mode {mode!r}")
    rep = ScalingReport(mode=mode)
    with tempfile.TemporaryDirectory() as work:
        for g in gpus:
            if mode == "nccl" and g > have:
                raise P.ParameterError(f"run_scaling: {g} GPUs requested, {have} visible")
            if mode == "emulated" and g > 1:
                if not rep.hardware_oversubscribed:
                    print(f"warning: {g} ranks on {max(have, 1)} GPU(s)", file=sys.stderr)
                rep.hardware_oversubscribed = True
            if mode == "emulated":
                t = P.CategoryTimers()
                run = P.solve_emulated(model, config, x0, g, timers=t)
            else:
                run, t = _run_nccl(model, config, x0, g, work, timeout)
            rep.gpus.append(g)
            rep.wall_times.append(run.wall_time)
            rep.categories.append(t)
            rep.runs.append(run)
    rep.identical_results = all(report_io.same_numerics(rep.runs[0], r) for r in rep.runs[1:])
    rep.speedups = [rep.wall_times[0] / t if t > 0.0 else 0.0 for t in rep.wall_times]
    if rep.speedups:
        rep.speedups[0] = 1.0  # by definition
    return rep


def to_json(r: ScalingReport) -> str:
    """to_json(ScalingReport) (report_io.cpp:138-162); the thread axis is named
    ``threads`` as in the reference (it counts GPUs here) and ``mode`` is added."""
    cats = []
    for i, c in enumerate(r.categories):
        total = r.wall_times[i] if i < len(r.wall_times) and r.wall_times[i] > 0.0 else 0.0
        row = {"blas3_s": c.blas3, "func_s": c.func, "orth_s": c.orth}
        if total > 0.0:
            row.update({"blas3_pct": 100.0 * c.blas3 / total, "func_pct": 100.0 * c.func / total,
                        "orth_pct": 100.0 * c.orth / total})
        cats.append(row)
    j = {"threads": r.gpus, "wall_times": r.wall_times, "speedups": r.speedups,
         "categories": cats, "identical_results": r.identical_results,
         "hardware_oversubscribed": r.hardware_oversubscribed, "mode": r.mode}
    if r.runs:
        j["iterations"] = r.runs[0].iterations
        j["status"] = report_io.STATUS_TEXT[r.runs[0].status]
    return json.dumps(j, indent=2, sort_keys=True)


def write_scaling_file(r: ScalingReport, path: str) -> None:
    """write_scaling_file (report_io.cpp:218-224)."""
    with open(path, "w") as f:
        f.write(to_json(r) + "\n")


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--worker", nargs=2, metavar=("CASE", "OUT"), help=argparse.SUPPRESS)
    ap.add_argument("--config", type=int, default=3, help="BASELINE config (problems.CONFIGS)")
    ap.add_argument("--gpus", default="1,2,4,8")
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--mode", choices=("nccl", "emulated"), default=None)
    ap.add_argument("--out", default=None)
    args = ap.parse_args(argv)
    if args.worker:
        _worker(*args.worker)
        return 0
    from paper_1810_03930_b200.problems import make_instance
    inst = make_instance(args.config, P)
    x0 = P.initial_point(inst.n, inst.p, inst.seed ^ 0x1235713)
    cfg = P.SolverConfig(tol_rel_kkt=np.finfo(float).tiny, max_iter=args.iters)
    rep = run_scaling(inst.model(P), cfg, x0, [int(g) for g in args.gpus.split(",")], args.mode)
    text = to_json(rep)
    print(text)
    if args.out:
        write_scaling_file(rep, args.out)
    return 0 if rep.identical_results else 1


if __name__ == "__main__":
    sys.exit(main())
