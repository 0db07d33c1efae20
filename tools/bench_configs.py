"""Run bench.py for every BASELINE config and collect profiles/bench_<tag>_configs.json.
usage (GPU box): python tools/bench_configs.py [--tag r01] [--configs 1 2 3 4 5]"""
import argparse, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("--tag", default="r01")
ap.add_argument("--configs", type=int, nargs="*", default=[1, 2, 3, 4, 5])
ap.add_argument("--out", default=None, help="default profiles/bench_<tag>_configs.json")
a = ap.parse_args()
rows = []
for c in a.configs:
    steps = {1: 2000, 2: 200, 3: 60, 4: 40, 5: 4}[c]
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", str(c),
                          "--steps", str(steps), "--warmup", "5", "--no-cpu-baseline"],
                         capture_output=True, text=True, timeout=1200)
    line = [l for l in out.stdout.splitlines() if l.startswith("{")]
    if out.returncode or not line:
        print(f"config {c} failed: {out.stderr[-500:]}", flush=True)
        continue
    d = json.loads(line[-1])
    ir = d["iteration_roofline"]
    rows.append({"config": c, "workload": d["config"]["workload"], "ms_per_iteration": d["ms_per_step"],
                 "iterations_per_s": d["value"], "t_star_ms": ir["t_star_ms"], "roofline_frac": ir["frac"],
                 "phase_ms": ir["phase_ms"], "dominant_kernel": d["roofline"]["kernel"],
                 "dominant_frac_of_peak": d["roofline"]["frac"],
                 "e2e_iterations_per_s": (d.get("e2e") or {}).get("value"), "clocks": d["clocks"]})
    print(c, d["ms_per_step"], ir["frac"], flush=True)
json.dump({"source": "python tools/bench_configs.py (bench.py --config C --no-cpu-baseline; B200, one GPU)",
           "rows": rows,
           "note": "e2e = the drop-in pcal_solve() with host buffers after one untimed 1-iteration call"},
          open(a.out or os.path.join(ROOT, "profiles", f"bench_{a.tag}_configs.json"), "w"), indent=1)
