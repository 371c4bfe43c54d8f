#!/usr/bin/env python3
"""One-line summaries of ncu raw-page CSV exports (tools/_prof*.sh): time, instructions,
warps, issue, pipe utilisation and the top stall reasons.

    python tools/ncu_brief.py gpurun_out/NAME.raw.csv ...
"""
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    d = dict(zip(rows[0], rows[2]))

    def g(k):
        try:
            return float(d.get(k, "nan").replace(",", ""))
        except ValueError:
            return float("nan")

    pipes = {p: g(f"sm__inst_executed_pipe_{p}.avg.pct_of_peak_sustained_active")
             for p in ("alu", "fma", "fp64", "xu", "lsu", "adu")}
    st = [(k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], g(k)) for k in d
          if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
    st.sort(key=lambda kv: -kv[1])
    print(f"{path.split('/')[-1]}: {d.get('Kernel Name', '?')[:60]}")
    print(f"  {g('gpu__time_duration.sum'):.3f} {rows[1][rows[0].index('gpu__time_duration.sum')]}  "
          f"inst {g('smsp__inst_executed.sum'):.4g}  regs {g('launch__registers_per_thread'):.0f}  "
          f"warps/SM {g('sm__warps_active.avg.per_cycle_active'):.1f}  issue {g('smsp__issue_active.avg.per_cycle_active'):.2f}  "
          f"dram {g('dram__bytes_read.sum') + g('dram__bytes_write.sum'):.4g}")
    print("  pipes % " + " ".join(f"{k}={v:.1f}" for k, v in pipes.items()))
    print("  stalls/issue " + " ".join(f"{k}={v:.2f}" for k, v in st[:7]))
