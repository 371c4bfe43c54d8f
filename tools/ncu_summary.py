#!/usr/bin/env python3
"""Summarise ncu reports (run here, no GPU needed) into profiles/.

    python tools/ncu_summary.py OUT_PREFIX report1.ncu-rep [report2.ncu-rep ...]

Writes OUT_PREFIX.md (one table row per report: time, issue, pipe utilisation,
warp-execution efficiency, branch uniformity, occupancy, DRAM bytes) and updates
profiles/ncu_summary.json (per kernel label: the per-launch DRAM traffic that bench.py
reports as roofline.traffic).
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
METRICS = [
    ("time_ms", "gpu__time_duration.sum", 1e-6),
    ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    ("ipc_per_sm", "sm__inst_executed.avg.per_cycle_active", 1),
    ("alu_pct", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1),
    ("fma_pct", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 1),
    ("fp64_pct", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 1),
    ("xu_pct", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1),
    ("lsu_pct", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", 1),
    ("adu_pct", "sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active", 1),
    ("warp_exec_eff_threads", "smsp__thread_inst_executed_per_inst_executed.ratio", 1),
    ("branch_uniform_pct", "smsp__sass_average_branch_targets_threads_uniform.pct", 1),
    ("divergent_branches", "smsp__sass_branch_targets_threads_divergent.sum", 1),
    ("warps_active_per_sm", "sm__warps_active.avg.per_cycle_active", 1),
    ("regs", "launch__registers_per_thread", 1),
    ("warp_instr", "smsp__inst_executed.sum", 1),
    ("dram_read_bytes", "dram__bytes_read.sum", 1),
    ("dram_write_bytes", "dram__bytes_write.sum", 1),
    ("stall_math_throttle", "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", 1),
    ("stall_not_selected", "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", 1),
    ("stall_wait", "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", 1),
    ("stall_short_scoreboard", "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", 1),
]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "usecond": 1e3,
              "msecond": 1e6, "nsecond": 1}


def read(rep: Path) -> dict:
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    res = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""}
    for key, name, scale in METRICS:
        if name not in hdr:
            continue
        i = hdr.index(name)
        try:
            v = float(vals[i].replace(",", ""))
        except ValueError:
            continue
        u = units[i]
        if key == "time_ms":
            v = v * UNIT_SCALE.get(u, 1) * 1e-6
        elif key.startswith("dram"):
            v = v * UNIT_SCALE.get(u, 1)
        res[key] = v
    return res


def main():
    prefix = Path(sys.argv[1])
    reps = [Path(p) for p in sys.argv[2:]]
    cols = ["time_ms", "issue_active_pct", "alu_pct", "fma_pct", "fp64_pct", "xu_pct", "lsu_pct",
            "warp_exec_eff_threads", "branch_uniform_pct", "warps_active_per_sm", "regs", "dram_read_bytes",
            "dram_write_bytes"]
    lines = ["| report | kernel | " + " | ".join(cols) + " |", "|" + "---|" * (len(cols) + 2)]
    summary_path = ROOT / "profiles" / "ncu_summary.json"
    summary = json.loads(summary_path.read_text()) if summary_path.exists() else {}
    allres = {}
    for rep in reps:
        r = read(rep)
        allres[rep.stem] = r
        kname = r["kernel"].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        lines.append(f"| {rep.stem} | `{kname}` | " + " | ".join(
            (f"{r[c]:.4g}" if isinstance(r.get(c), float) else str(r.get(c, ""))) for c in cols) + " |")
        summary.setdefault(kname, {})
        summary[kname][rep.stem] = {"dram_bytes_per_launch": r.get("dram_read_bytes", 0) + r.get("dram_write_bytes", 0),
                                    "time_ms": r.get("time_ms")}
    prefix.parent.mkdir(parents=True, exist_ok=True)
    prefix.with_suffix(".md").write_text("\n".join(lines) + "\n")
    prefix.with_suffix(".json").write_text(json.dumps(allres, indent=1))
    summary_path.write_text(json.dumps(summary, indent=1))
    print("\n".join(lines))


if __name__ == "__main__":
    main()
