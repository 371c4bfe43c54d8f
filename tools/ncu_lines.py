#!/usr/bin/env python3
"""Per-source-line instruction counts and stall samples of an ncu report (run here).

    python tools/ncu_lines.py report.ncu-rep|page.csv[.gz] [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
if rep.endswith(".csv.gz"):  # a source page exported on the GPU box (tools/_prof*.sh)
    import gzip

    out = gzip.open(rep, "rt").read()
elif rep.endswith(".csv"):
    out = open(rep).read()
else:
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
rows = []
fname = ""
total_i = total_s = 0
hdr = None
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr) or not r[0].isdigit():
        continue
    d = {}
    for k, v in zip(hdr, r):  # "Source" appears twice (cuda, sass): keep the first
        d.setdefault(k, v)
    try:
        ins = int(d.get("Instructions Executed", "0") or 0)
        smp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    if ins == 0 and smp == 0:
        continue
    total_i += ins
    total_s += smp
    rows.append((ins, smp, f"{fname}:{r[0]}", r[1].strip()[:70]))
rows.sort(key=lambda x: -x[0])
print(f"total warp-instr {total_i:.4g}  samples {total_s}")
for ins, smp, loc, src in rows[:top]:
    print(f"{ins / total_i * 100:6.2f}% instr {smp / max(total_s, 1) * 100:6.2f}% stall  {loc:22s} {src}")
