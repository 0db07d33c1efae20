"""Summarise per-instruction warp-stall samples of one kernel from an ncu report.
usage: python tools/ncu_stalls.py REPORT.ncu-rep KERNEL_SUBSTRING [top]"""
import csv, io, subprocess, sys, collections
rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks, cur = [], None
for line in out.splitlines():
    if line.startswith('"Kernel Name"'):
        cur = [line]; blocks.append(cur)
    elif cur is not None:
        cur.append(line)
for b in blocks:
    name = next(csv.reader([b[0]]))[1]
    if pat not in name:
        continue
    rows = list(csv.reader(io.StringIO("\n".join(b[1:]))))
    hdr = rows[0]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = collections.Counter(); byop = collections.Counter(); total = 0
    insts = []
    for r in rows[1:]:
        if len(r) < len(hdr): continue
        s = int(float(r[si] or 0)); total += s
        op = r[1].strip().split()[0] if r[1].strip() else "?"
        if op.startswith("@"): op = r[1].strip().split()[1]
        byop[op.split(".")[0]] += s
        for i in stall_cols:
            tot[hdr[i]] += int(float(r[i] or 0))
        insts.append((s, r[0][-5:], r[1].strip()[:70], {hdr[i]: r[i] for i in stall_cols if r[i] not in ("0", "")}))
    print("kernel:", name, "samples:", total)
    print("stall reasons:", [(k, v) for k, v in tot.most_common(10)])
    print("by opcode:", byop.most_common(12))
    for s, a, t, d in sorted(insts, reverse=True)[:top]:
        print(f"{s:7d} {a} {t:70s} {d}")
    break
