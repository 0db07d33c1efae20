#!/usr/bin/env python
"""PCAL iterations/s on B200 (BASELINE.json metric), one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]

A "step" is one PCAL iteration (solver.cpp:369-439) of config C (default 5:
the 7-point Laplacian + diagonal potential on a 128³ periodic grid, p = 1024,
FP64 — BASELINE configs[4], the 1/2/4/8-GPU sweep the metric is quoted on and
the largest configuration that fits one GPU).
  value : iterations/s with the instance resident in HBM, K iterations timed
          with CUDA events on the session stream (graphs, no host sync), max
          over ranks; the working set (X, P, X_prev, P_prev: 64 GiB at config 5;
          the 2 GiB dense A at config 2) is far larger than L2, so every
          iteration streams it from HBM (no L2 flush needed).
  e2e   : the public drop-in call pcal_solve() (host buffers: H2D of the operator
          and X0 from pinned memory, D2H of the report and X) for the config's
          full iteration count + final orthonormalization, wall clock.
  roofline : dominant kernel, achieved = algorithmic flops (or bytes) per launch
          ÷ its mean CUDA-event duration measured in this run; peak = measured
          FP64 DMMA rate (profiles/fp64_peaks_r02.json; MEASURED_PEAKS.json has
          no FP64 entry) or MEASURED_PEAKS.json hbm_gbs for HBM-bound kernels.
  cpu_baseline : the UNMODIFIED reference solve() (oracle/_ref) on the host
          cores, per-iteration time from its own trace clock, bounded sample
          (config 5: a z-slab of the grid, time scaled by n / n_slab — the
          reference needs ≈190 GiB and ≈30 min per full-size iteration).
--impl reference times that CPU implementation alone (rank 0; others exit 0).
N > 1: one process per GPU (torchrun; `--gpus N` without torchrun spawns the N
ranks itself); the instance is ROW-SHARDED over the ranks (z-slabs / row
blocks, NCCL collectives): strong scaling, value = K /
max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
TINY = float(np.finfo(float).tiny)
INIT_SALT = 0x1235713


def load_peaks() -> dict:
    peaks = {"fp64_tflops": 37.15, "fp64_src": "fallback (DMMA microbenchmark, round 1)",
             "hbm_gbs": 6544.3, "hbm_src": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        peaks["hbm_gbs"] = float(m["hbm_gbs"])
        peaks["hbm_src"] = "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        pass
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peaks_r02.json")) as f:
            m = json.load(f)
        peaks["fp64_tflops"] = float(m["dmma_tflops"])
        peaks["fp64_src"] = "measured DMMA.8x8x4 peak at 1965 MHz, profiles/fp64_peaks_r02.json"
    except Exception:
        pass
    return peaks


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""
    NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
             0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
             0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device: int):
        self.samples, self.reasons, self.ok = [], 0, False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self) -> dict:
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": ["unavailable"]}
        names = [n for bit, n in self.NAMES.items() if self.reasons & bit and bit != 0x1]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max,
                "reasons": names, "samples": len(self.samples)}


def dist_setup(ngpus: int):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # the log shows the real rank count
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def pinned_f64(n_rows: int, n_cols: int):
    """Column-major FP64 host matrix in pinned memory (for the e2e H2D copies)."""
    import torch
    t = torch.empty(n_rows * n_cols, dtype=torch.float64, pin_memory=True)
    arr = t.numpy().reshape((n_cols, n_rows)).T  # Fortran-ordered view
    return t, arr


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# Per-iteration reference work is linear in n at fixed p (every term is O(np²)
# or O(np)), so a configuration too large for the reference on one host is
# timed on a z-slab of its own grid and scaled by n / n_slab.  Config 5 needs
# ≈ 12 live n×p matrices in the reference's solve() — ≈ 190 GiB of host RAM
# against the box's 196 GB — and ≈ 20–35 min per iteration, so its reference
# sample is the 128×128×SLAB_NZ slab with p = 1024.
SLAB_NZ = {"reference": 16, "cpu_baseline": 2}


def cpu_reference_rate(inst, x0=None, budget_s: float = 15.0, threads: int = None, min_iters=1,
                       max_iters=None, slab_nz: int = None):
    """Time the reference CPU solve() on a bounded sample; returns (iters/s, info).

    slab_nz: time the grid model on the nx×ny×slab_nz bottom slab of the same
    grid (V = the slab's rows of the config's potential, the config's s, the
    slab's own seeded QR start point) and scale the per-iteration time by
    n / n_slab."""
    from oracle.oracle import Config, Model, MODEL_DENSE, MODEL_KOHN_SHAM, MODEL_STENCIL
    from oracle.oracle import Reference, Restatement, available_reference
    threads = threads or os.cpu_count() or 1
    R = Reference() if available_reference() else Restatement()
    kind = {"dense": MODEL_DENSE, "stencil": MODEL_STENCIL, "kohn_sham": MODEL_KOHN_SHAM}[inst.kind]
    n, grid, v, scale = inst.n, inst.grid or (0, 0, 0), inst.v, 1.0
    t_setup = time.perf_counter()
    if slab_nz is not None and inst.kind == "stencil" and slab_nz < grid[2]:
        grid = (grid[0], grid[1], slab_nz)
        n = grid[0] * grid[1] * grid[2]
        v = np.ascontiguousarray(inst.v[:n])
        scale = inst.n / n
        x0 = None
    if x0 is None:  # the threaded C restatement of initial_point (bitwise the reference's)
        x0 = Restatement().initial_point_qr(n, inst.p, inst.seed ^ INIT_SALT, threads=threads)
    t_setup = time.perf_counter() - t_setup
    m = Model(kind, n, inst.p, inst.s, a=inst.a, grid=grid, v=v)
    t0 = time.perf_counter()
    # probe: one iteration, per-iteration time from the reference's own trace clock
    probe = R.solve(m, Config(tol_rel_kkt=TINY, max_iter=1, threads=threads, final_orth=False), x0)
    t_it = max(probe.trace[1, 6] - probe.trace[0, 6], 1e-6)
    iters = int(max(min_iters, min(inst.iters, max_iters or inst.iters, budget_s / t_it)))
    if iters <= 1 and budget_s <= 2 * t_it:  # one iteration already spent the budget
        rep, iters = probe, 1
    else:
        rep = R.solve(m, Config(tol_rel_kkt=TINY, max_iter=iters, threads=threads,
                                final_orth=False), x0)
    wall = time.perf_counter() - t0
    per = (rep.trace[iters, 6] - rep.trace[0, 6]) / iters * scale
    what = "reference solve() (oracle/_ref)" if R.kind == "reference" else "C restatement (oracle)"
    if inst.kind != "dense":
        what += " driving the restated grid operator (no reference operator exists)"
    where = (f"the {grid[0]}x{grid[1]}x{grid[2]} z-slab (n={n}) of config {inst.cfg}'s grid, "
             f"p={inst.p}, per-iteration time x n/n_slab = {scale:g}" if scale != 1.0
             else f"config {inst.cfg} (n={n}, p={inst.p})")
    info = {"kind": R.kind, "cores": threads, "iters": iters, "cpu_model": cpu_model(),
            "sample": f"{what}: {iters} PCAL iteration(s) of {where}, timed by its trace "
                      f"clock, setup excluded",
            "sample_n": n, "scale": scale, "setup_s": round(t_setup, 2), "solve_wall_s": round(wall, 2),
            "host_rss_gib": round(peak_rss_gib(), 2)}
    return 1.0 / per, info


def peak_rss_gib() -> float:
    try:
        import resource
        return resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2 ** 20
    except Exception:
        return float("nan")


WORKLOADS = {1: "config 1: dense trace-min n=1000 p=20 (A=sym(randn), seed 1)",
             2: "config 2: dense trace-min n=16384 p=128 (A=sym(randn), seed 1)",
             3: "config 3: 7-pt periodic Laplacian + diag V, 64^3, p=256, seed 1",
             4: "config 4: Kohn-Sham-like 48^3, p=512, seed 1",
             5: "config 5: 7-pt Laplacian + diag V, 128^3, p=1024, seed 1 (scaling sweep)"}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    # the instance comes from the oracle's restatement of the reference RNG
    # (bitwise the reference's data): nothing of the B200 library on this path
    from paper_1810_03930_b200.problems import CONFIGS, REFERENCE_S, Instance, ks_potential
    from oracle.oracle import Restatement
    O = Restatement()
    c = CONFIGS[args.config]
    th = os.cpu_count() or 8
    slab = None
    if c["kind"] == "dense":
        m = O.dense_trace_min(c["n"], c["p"], 1, s=REFERENCE_S.get((c["n"], 1)), threads=th)
        inst = Instance(args.config, "dense", m.n, m.p, c["iters"], m.s, a=m.a)
    else:
        g = c["grid"]
        nn = g[0] * g[1] * g[2]
        v = O.random_uniform(nn, 1) if c["kind"] == "stencil" else ks_potential(g, 1, O)
        s = 12.0 + float(v.max()) if c["kind"] == "stencil" else 6.0 + float(np.abs(v).max())
        inst = Instance(args.config, c["kind"], nn, c["p"], c["iters"], s, v=v, grid=g)
        if args.config == 5:
            slab = SLAB_NZ["reference"]
    budget = float(os.environ.get("PCAL_REF_BUDGET_S", "60"))
    rate, info = cpu_reference_rate(inst, None, budget_s=budget, min_iters=1, max_iters=args.steps,
                                    slab_nz=slab)
    line = {"metric": "PCAL iterations/sec", "impl": "reference", "value": rate,
            "unit": "iterations/s", "n_gpus": args.gpus, "steps": info["iters"],
            "warmup": 1, "ms_per_step": 1e3 / rate, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOADS[args.config], "n": inst.n, "p": inst.p,
                       "kind": inst.kind, "s": inst.s},
            "cpu_baseline": {"value": rate, "unit": "iterations/s", "cores": info["cores"],
                             "kind": info["kind"], "sample": info["sample"],
                             "cpu_model": info["cpu_model"], "sample_n": info["sample_n"],
                             "scale": info["scale"], "setup_s": info["setup_s"],
                             "solve_wall_s": info["solve_wall_s"],
                             "host_rss_gib": info["host_rss_gib"]},
            "e2e": {"value": rate, "unit": "iterations/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_emulated(args) -> int:
    """`--gpus N --emulate`: the row-sharded algorithm with N ranks emulated on
    one GPU (host threads, loopback collectives) against the same
    algorithm with one rank: the reports must be bitwise identical
    (same_numerics, report_io.cpp:259-283).  A correctness check of the N-GPU
    path on a one-GPU box, not a timing."""
    import paper_1810_03930_b200 as P
    from paper_1810_03930_b200 import report_io
    from paper_1810_03930_b200.problems import make_instance
    inst = make_instance(args.config, P, threads=os.cpu_count() or 8)
    x0 = P.initial_point(inst.n, inst.p, inst.seed ^ INIT_SALT)
    model = inst.model(P)
    cfg = P.SolverConfig(tol_rel_kkt=TINY, max_iter=args.steps)
    t0 = time.perf_counter()
    r1 = P.solve_emulated(model, cfg, x0, 1)
    t1 = time.perf_counter()
    rn = P.solve_emulated(model, cfg, x0, args.gpus)
    t2 = time.perf_counter()
    rows = [P.partition(model, args.gpus, r)[1] for r in range(args.gpus)]
    line = {"mode": "emulated", "config": {"workload": WORKLOADS[args.config], "n": inst.n,
                                           "p": inst.p},
            "n_ranks": args.gpus, "iterations": args.steps,
            "same_numerics": bool(report_io.same_numerics(r1, rn)),
            "rows_per_rank": rows,
            "device_bytes_per_rank_nxp": [4 * 8 * r * inst.p for r in rows],
            "wall_s": {"ranks_1": round(t1 - t0, 2), f"ranks_{args.gpus}": round(t2 - t1, 2)},
            "final_post_f": [r1.final_post_orth.fval if r1.final_post_orth else None,
                             rn.final_post_orth.fval if rn.final_post_orth else None]}
    print(json.dumps(line), flush=True)
    return 0 if line["same_numerics"] else 1


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` without torchrun: launch N ranks (one per GPU) of this
    same command through torch.distributed.run and return its exit code."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5,
                    help="BASELINE config (default 5: the 1/2/4/8-GPU sweep the metric names)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-calls", type=int, default=3)
    ap.add_argument("--sharded", action="store_true",
                    help="use the NCCL row-sharded path even on one GPU (testing)")
    ap.add_argument("--emulate", action="store_true",
                    help="with --gpus N: N ranks emulated on one GPU, same_numerics vs 1 rank")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.emulate:
        return run_emulated(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # NCCL's own log shows the rank count the communicator really has
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        return spawn_ranks(args)

    import torch
    import paper_1810_03930_b200 as P
    from paper_1810_03930_b200.problems import make_instance

    rank, world, local = dist_setup(args.gpus)
    if args.gpus > 1 and world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = local
    K, W = args.steps, max(args.warmup, 3)
    peaks = load_peaks()
    hostthreads = max(1, (os.cpu_count() or 8) // world)

    # ---- setup (not timed): instance in pinned host memory; X0 = initial_point
    # ({Qr}, seed) built by the library on the device (PCAL_X0_SEED) — sharded,
    # each rank draws and orthonormalises only its own rows
    t_setup = time.perf_counter()
    a_pin = None
    if args.config in (1, 2):
        n = {1: 1000, 2: 16384}[args.config]
        a_t, a_pin = pinned_f64(n, n)
    inst = make_instance(args.config, P, threads=hostthreads, a_out=a_pin, device=dev)
    x0_seed = inst.seed ^ INIT_SALT
    prof_iters = 10 if args.config < 5 else 4
    cfg = P.SolverConfig(tol_rel_kkt=TINY, max_iter=W + K + prof_iters + 2, final_orth=False,
                         device=dev)
    comm = None
    if world > 1 or args.sharded:
        # row sharding over NCCL: this rank's slab of the instance
        obj = [P.nccl_unique_id() if rank == 0 else None]
        if world > 1:
            import torch.distributed as dist
            dist.broadcast_object_list(obj, src=0)
        comm = P.Comm(world, rank, obj[0], dev)
        gm = inst.model(P)
        r0, nr = P.partition(gm, world, rank)
        if inst.kind == "dense":
            a_loc = np.asfortranarray(inst.a[r0:r0 + nr, :])
            model = P.QuadraticModel(a_loc, inst.p, inst.s, n=inst.n)
        elif inst.kind == "stencil":
            model = P.StencilModel(inst.grid, inst.v[r0:r0 + nr], inst.p, inst.s)
        else:
            model = P.KohnShamModel(inst.grid, inst.v[r0:r0 + nr], inst.p, inst.s)
        ses = P.ShardedSession(model, cfg, x0_seed, comm, nr)
    else:
        model = inst.model(P)
        r0, nr = 0, inst.n
        ses = P.Session(model, cfg, x0_seed)
    # this rank's rows of X0 in pinned host memory: the e2e call's input
    x0_t, x0h = pinned_f64(nr, inst.p)
    ses.get_x(out=x0h)
    t_setup = time.perf_counter() - t_setup

    # ---- value: device-resident iterations, CUDA events on the session stream
    stream = torch.cuda.ExternalStream(ses.stream, device=dev)
    ses.run(W)
    ses.sync()
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = ses.kernel_launches
    with ClockSampler(dev) as clk:
        e0.record(stream)
        ses.run(K)
        e1.record(stream)
        e1.synchronize()
    launches = ses.kernel_launches - l0
    kpi = ses.kernels_per_iteration
    ms = e0.elapsed_time(e1)
    torch.cuda.synchronize()
    ms = max_over_ranks(ms, world)
    barrier(world)
    phases = ses.profile(prof_iters)      # per-phase CUDA-event durations (same session)
    # X·[W|C] as one block (P = G − X·M1, 2np² flop) or two (4np²), and how
    # often the kkt identity's gated fallback ran
    xm_form, xm_fallbacks = ses.xm_mode() if hasattr(ses, "xm_mode") else ("two_block", 0)
    rep = ses.finish(want_x=False)
    ses.close()
    del ses
    assert rep.status == "max_iter", rep.status
    ms_per = ms / K
    # sharded: the ranks advance ONE iteration of the problem together (strong
    # scaling); N = 1 is the same formula
    value = K / (ms * 1e-3)

    # ---- roofline of the dominant kernel + whole-iteration roofline
    n, p = inst.n, inst.p
    P64 = peaks["fp64_tflops"] * 1e12
    BW = peaks["hbm_gbs"] * 1e9
    nl = nr  # this rank's rows: per-launch work of its kernels
    gram_flops = (2.0 if inst.kind != "dense" else 3.0) * nl * p * p
    work = {"gradient": (inst.grad_flops() * nl / n, "tensor") if inst.kind == "dense"
            else ((16.0 * nl * p + inst.op_bytes() * nl / n), "hbm"),
            "gram": (gram_flops, "tensor"),
            "xm": ((2.0 if xm_form == "single_block" else 4.0) * nl * p * p, "tensor")}
    dom = max(("gradient", "gram", "xm"), key=lambda k: phases[k])
    amount, bound = work[dom]
    t = phases[dom] * 1e-3
    if bound == "tensor":
        ach, peak, unit = amount / t / 1e12, peaks["fp64_tflops"], "TFLOP/s"
        src = peaks["fp64_src"]
    else:
        ach, peak, unit = amount / t / 1e9, peaks["hbm_gbs"], "GB/s"
        src = peaks["hbm_src"]
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", f"ncu_cfg{args.config}_summary.json")) as f:
            traffic = json.load(f).get("dram_bytes_per_launch", {}).get(dom)
    except Exception:
        pass
    # flops the iteration's GEMMs must do in the formulation executed: Gram
    # (3np², grid models 2np²: symmetric GᵀX), X·M1 (2np²) or X·[W|C] (4np²)
    F = (gram_flops + work["xm"][0]) * n / nl + inst.grad_flops()
    F_two_block = 7.0 * n * p * p + inst.grad_flops()  # round-1 definition (3np² + 4np²)
    B = 80.0 * n * p + inst.op_bytes()
    t_star = max(F / P64, B / BW) / world
    t_star_two = max(F_two_block / P64, B / BW) / world
    roof = {"bound": bound, "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak,
            "traffic": traffic, "kernel": dom, "kernel_ms": phases[dom], "peak_src": src,
            "work_per_launch": amount,
            "work_def": ("2np^2 (upper tiles of the symmetric G^TX + X^TX)" if dom == "gram"
                         and inst.kind != "dense" else
                         {"gram": "3np^2", "xm": "2np^2 (X·M1, M1 = W - beta C)"
                          if xm_form == "single_block" else "4np^2 (X·[W|C])", "gradient":
                          "2n^2p" if inst.kind == "dense" else "16np+8n bytes"}[dom])}
    iter_roof = {"flops": F, "bytes": B, "t_star_ms": t_star * 1e3, "frac": t_star * 1e3 / ms_per,
                 "bound": "fp64" if F / P64 >= B / BW else "hbm",
                 "def": "T* = max((F_gram + F_xm + F_grad) / P_fp64, (80np+B_op) / BW) / n_gpus; "
                        "F_gram = 3np^2 (grid models 2np^2), F_xm = 2np^2 single block / 4np^2 two",
                 "xm_form": xm_form, "xm_identity_fallbacks": xm_fallbacks,
                 "t_star_two_block_ms": t_star_two * 1e3,
                 "frac_vs_two_block": t_star_two * 1e3 / ms_per,
                 "phase_ms": {k: round(v, 5) for k, v in phases.items()}}

    # ---- e2e: the public drop-in call with host buffers
    e2e = None
    if not args.no_e2e:
        iters = inst.iters
        # one untimed 1-iteration call first: module loading and first-use setup
        # of the final-orthonormalisation kernels are not part of a steady call
        warm = P.SolverConfig(tol_rel_kkt=TINY, max_iter=1, device=dev)
        emodel = model if comm is not None else inst.model(P, a=inst.a if inst.kind == "dense"
                                                           else None)
        if comm is not None:
            P.solve_sharded(emodel, warm, x0h, comm, nr)
        else:
            P.solve(emodel, warm, x0h)
        # the report's stop / final iterates land in pinned host buffers (the
        # step's result read-back is then a DMA, not a page-faulting pageable copy)
        o1_t, o1 = pinned_f64(nr, p)
        o2_t, o2 = pinned_f64(nr, p)
        # timed calls, the median reported: the host↔device copies of one call
        # vary from run to run on this pool (measured 1.16–1.69 s for config 2)
        walls = []
        for _ in range(max(1, args.e2e_calls)):
            barrier(world)
            t0 = time.perf_counter()
            ecfg = P.SolverConfig(tol_rel_kkt=TINY, max_iter=iters, device=dev)
            if comm is not None:
                r = P.solve_sharded(emodel, ecfg, x0h, comm, nr, out=(o1, o2))
            else:
                r = P.solve(emodel, ecfg, x0h, out=(o1, o2))
            walls.append(max_over_ranks(time.perf_counter() - t0, world))
            post = r.final_post_orth.feas if r.final_post_orth else None
        wall = statistics.median(walls)
        h2d = inst.op_bytes() + 8 * n * p
        d2h = 8 * 2 * n * p + 8 * 7 * (iters + 1)
        e2e = {"value": iters / wall, "unit": "iterations/s",
               "h2d_bytes_per_step": h2d / iters, "d2h_bytes_per_step": d2h / iters,
               "iterations": iters, "wall_s": wall, "walls_s": walls, "status": r.status,
               "final_post_feas": post,
               "includes": "H2D operator+X0 (pinned), all iterations, final CholeskyQR2, "
                           "D2H trace + stop/final X; median of the timed calls after one "
                           "untimed 1-iteration call"}

    # ---- CPU baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            rate, info = cpu_reference_rate(
                inst, np.asfortranarray(x0h) if args.config < 5 else None, budget_s=15.0,
                slab_nz=SLAB_NZ["cpu_baseline"] if args.config == 5 else None)
            cpu = {"value": rate, "unit": "iterations/s", "cores": info["cores"],
                   "kind": info["kind"], "sample": info["sample"], "cpu_model": info["cpu_model"]}
        except Exception as e:  # reported, never silently substituted
            cpu = {"value": None, "unit": "iterations/s", "cores": 0, "kind": "unavailable",
                   "sample": f"failed: {e}"}

    if rank == 0:
        wl = WORKLOADS[args.config]
        line = {
            "metric": "PCAL iterations/sec", "value": value, "unit": "iterations/s",
            "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": ms_per,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference RNG stream, seed 1; no dataset)",
            "config": {"workload": wl, "n": n, "p": p, "kind": inst.kind, "s": inst.s,
                       "iterations_per_solve": inst.iters,
                       "parallelism": "single-gpu" if comm is None
                       else f"row-sharded x{world} (NCCL: Gram/partials allreduce, "
                            f"{'X allgather' if inst.kind == 'dense' else 'z-halo planes'})",
                       "l2": ("inputs larger than L2: A = %.1f GiB streamed every iteration"
                              % (inst.op_bytes() / 2 ** 30)) if inst.kind == "dense"
                       else "inputs larger than L2: working set (X, P, X_prev, P_prev) = "
                            "%.1f GiB" % (4 * 8 * n * p / world / 2 ** 30),
                       "iteration_graph_kernels": kpi, "setup_s": round(t_setup, 2)},
            "roofline": roof, "iteration_roofline": iter_roof, "cpu_baseline": cpu,
            "e2e": e2e, "clocks": clk.summary(), "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
