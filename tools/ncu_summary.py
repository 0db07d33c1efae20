"""Summarise ncu outputs into profiles/ (launch list + one --set full capture).

usage: python tools/ncu_summary.py --launches L.csv --full R.ncu-rep --config 2 --tag r01
Writes profiles/<tag>_cfg<C>_launches.txt, profiles/<tag>_cfg<C>_full.txt and
profiles/ncu_cfg<C>_summary.json (dram bytes per launch, consumed by bench.py).
"""
import argparse
import collections
import csv
import io
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name: str) -> str:
    nm = name.replace("pcal::", "").replace("(int)", "")
    if "gemm_xm_tmem" in nm:
        return "gemm_xm_tmem<128x128,MC,XM>"
    if "gemm_xm_staged" in nm:
        return "gemm_xm_staged<128x64,MC,XM>"
    if "gemm_xm1_staged" in nm:
        return "gemm_xm1_staged<64x64,MC,XM>"
    if "k_stencil_tma" in nm:
        return "k_stencil_tma"
    m = re.search(r"gemm_(streamk|fixup|fixup_store)<GemmCfg<(\d+), (\d+), \d+, \d+, \d+, (\d)(?:, \d+)?>(?:, (\d))?(?:, (\d))?", nm)
    if m:
        kind = {"0": "STORE", "1": "GRAD", "2": "XM", None: "STORE"}[m.group(5)]
        mode = "MC" if m.group(4) == "0" else "KC"
        prod = f",P{m.group(6)}" if m.group(6) else ""
        return f"gemm_{m.group(1)}<{m.group(2)}x{m.group(3)},{mode},{kind}{prod}>"
    m = re.search(r"(k_[a-z0-9_]+)", name)
    return m.group(1) if m else name[:60]


def phase_of(s: str) -> str:
    if "GRAD" in s or "stencil" in s or s.startswith(("k_row_sq", "k_axis", "k_spectral", "k_ks")):
        return "gradient"
    if "KC,STORE" in s or s == "k_small_pxp":
        return "gram"
    if "XM" in s or "MC,STORE" in s or s in ("k_sum_rows", "k_finish_eval", "k_zero_i32",
                                               "k_colsum3", "k_kkt_corr", "k_kkt_gate"):
        return "xm"
    if s in ("k_bb_partials", "k_eta", "k_update", "k_normalize", "k_step_fused", "k_bb_cols",
             "k_bb_cols_sum", "k_colscale", "k_update_norm"):
        return "step"
    return "other"


def launches(path: str, out, kpi: int):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    data = []
    for r in rows[hdr + 1:]:
        if len(r) <= vi or r[h.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        us = v / 1e3 if unit in ("ns", "nsecond") else v * 1e3 if unit in ("ms", "msecond") else v
        data.append((short(r[ki]), us))
    # the last `kpi` launches of the run are one full iteration graph
    it = data[-kpi:] if kpi and len(data) >= kpi else data
    tot = sum(u for _, u in it)
    print(f"# ncu launch list (gpu__time_duration.sum, --clock-control none): {len(data)} launches;"
          f" last iteration = {len(it)} kernels, {tot:.1f} us (cold-cache, serialised)", file=out)
    by = collections.OrderedDict()
    for k, u in it:
        by.setdefault(k, [0, 0.0])
        by[k][0] += 1
        by[k][1] += u
    print(f"{'kernel':45s} {'n':>3s} {'us':>10s} {'share':>7s} phase", file=out)
    for k, (c, u) in sorted(by.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:45s} {c:3d} {u:10.1f} {100 * u / tot:6.1f}% {phase_of(k)}", file=out)
    ph = collections.Counter()
    for k, u in it:
        ph[phase_of(k)] += u
    print("phase shares:", {k: round(100 * v / tot, 1) for k, v in ph.most_common()}, file=out)


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed"]


def to_base(v: str, unit: str) -> float:
    x = float(v.replace(",", ""))
    scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "KB": 1e3, "MB": 1e6,
             "GB": 1e9, "B": 1, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9, "second": 1,
             "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1}
    return x * scale.get(unit, 1)


def full(path: str, out, summary: dict):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    print(f"# ncu --set full --clock-control none ({os.path.basename(path)})", file=out)
    for r in rows[2:]:
        name = short(r[h.index("Kernel Name")])
        print(f"## {name}", file=out)
        vals = {}
        for m in METRICS:
            if m in h:
                i = h.index(m)
                vals[m] = (r[i], units[i])
                print(f"  {m:80s} {r[i]:>14s} {units[i]}", file=out)
        t = to_base(*vals["gpu__time_duration.sum"])
        rb = to_base(*vals["dram__bytes_read.sum"])
        wb = to_base(*vals["dram__bytes_write.sum"])
        print(f"  dram read+write per launch: {(rb + wb) / 1e9:.4f} GB; "
              f"effective {(rb + wb) / t / 1e9:.1f} GB/s", file=out)
        ph = phase_of(name)
        kern = ("streamk" in name or "xm_tmem" in name or "xm_staged" in name or "xm1_staged" in name
                or "stencil" in name)
        # per phase: the longest capture (the iteration's launch, not a smaller
        # set-up launch of the same kernel, e.g. the initial point's Gram)
        if kern and ph in ("gradient", "gram", "xm") and rb + wb == rb + wb:
            if ph not in summary or t > summary[ph][1]:
                summary[ph] = (rb + wb, t)


def app_csv(path: str, out, summary: dict):
    """`ncu --replay-mode application --csv` output (one row per launch and
    metric): config 5's 64 GiB working set defeats kernel replay."""
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Name" in r)
    h = rows[hdr]
    ii, ki, mi, ui, vi = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit",
                                                "Metric Value"))
    launches = {}
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        d = launches.setdefault(r[ii], {"name": r[ki]})
        d[r[mi]] = to_base(r[vi], r[ui]) if r[ui] not in ("%", "") else float(r[vi].replace(",", ""))
    print(f"# ncu --replay-mode application --clock-control none ({os.path.basename(path)})",
          file=out)
    for lid in sorted(launches, key=int):
        d = launches[lid]
        name = short(d["name"])
        t = d.get("gpu__time_duration.sum", float("nan"))
        rb, wb = d.get("dram__bytes_read.sum", 0.0), d.get("dram__bytes_write.sum", 0.0)
        pipe = d.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", float("nan"))
        print(f"{lid:>4s} {name:45s} {t * 1e3:10.3f} ms  DRAM {(rb + wb) / 1e9:8.3f} GB "
              f"({(rb + wb) / t / 1e9 if t == t and t > 0 else 0:7.1f} GB/s)  tensor pipe {pipe:5.1f} %",
              file=out)
        ph = phase_of(name)
        kern = ("streamk" in d["name"] or "xm1_staged" in d["name"] or "xm_staged" in d["name"]
                or "stencil" in d["name"])
        if kern and ph in ("gradient", "gram", "xm") and t == t:
            if ph not in summary or t > summary[ph][1]:
                summary[ph] = (rb + wb, t)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--kpi", type=int, default=19, help="kernels per iteration graph")
    ap.add_argument("--outdir", default=os.path.join(ROOT, "profiles"),
                    help="where the summaries go (on a GPU box: under gpurun_out/)")
    ap.add_argument("--app-csv", help="application-replay CSV (config 5)")
    a = ap.parse_args()
    prof = a.outdir
    os.makedirs(prof, exist_ok=True)
    if a.launches:
        with open(os.path.join(prof, f"{a.tag}_cfg{a.config}_launches.txt"), "w") as f:
            launches(a.launches, f, a.kpi)
    if a.full or a.app_csv:
        summ = {}
        with open(os.path.join(prof, f"{a.tag}_cfg{a.config}_full.txt"), "w") as f:
            if a.full:
                full(a.full, f, summ)
            else:
                app_csv(a.app_csv, f, summ)
        with open(os.path.join(prof, f"ncu_cfg{a.config}_summary.json"), "w") as f:
            json.dump({"source": os.path.basename(a.full or a.app_csv), "tag": a.tag,
                       "dram_bytes_per_launch": {k: v[0] for k, v in summ.items()},
                       "duration_s_per_launch": {k: v[1] for k, v in summ.items()}},
                      f, indent=1)


if __name__ == "__main__":
    main()
