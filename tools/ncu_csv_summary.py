#!/usr/bin/env python3
"""Summarise the CSV exports of tools/prof_round2.sh (run here, no GPU needed).

    python tools/ncu_csv_summary.py DIR OUT_PREFIX

Writes OUT_PREFIX.md (one row per capture: time, issue, pipes, warp-execution
efficiency, branch uniformity, occupancy, DRAM bytes, top stalls), OUT_PREFIX.json (the
same numbers) and adds each capture's per-launch DRAM traffic to profiles/ncu_summary.json
under the kernel name the run reported (wlp_last_kernel, from the driver's stdout), which
is where bench.py looks up roofline.traffic.
"""
import csv
import json
import re
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
M = [("time_ms", "gpu__time_duration.sum"), ("issue_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
     ("alu_pct", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
     ("fma_pct", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
     ("fp64_pct", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
     ("xu_pct", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
     ("lsu_pct", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
     ("threads_per_warp_instr", "smsp__thread_inst_executed_per_inst_executed.ratio"),
     ("branch_uniform_pct", "smsp__sass_average_branch_targets_threads_uniform.pct"),
     ("warps_per_sm", "sm__warps_active.avg.per_cycle_active"), ("regs", "launch__registers_per_thread"),
     ("warp_instr", "smsp__inst_executed.sum"), ("dram_read", "dram__bytes_read.sum"),
     ("dram_write", "dram__bytes_write.sum")]
SCALE = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def load(path: Path) -> dict:
    rows = [r for r in csv.reader(open(path)) if r]
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"kernel_demangled": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""}
    for key, name in M:
        if name not in hdr:
            continue
        i = hdr.index(name)
        try:
            v = float(vals[i].replace(",", ""))
        except ValueError:
            continue
        d[key] = v * SCALE.get(units[i], 1.0)
    st = []
    for i, name in enumerate(hdr):
        m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio$", name)
        if m:
            try:
                st.append((m.group(1), float(vals[i])))
            except ValueError:
                pass
    st.sort(key=lambda kv: -kv[1])
    d["top_stalls"] = {k: round(v, 2) for k, v in st[:4]}
    return d


def main():
    src, prefix = Path(sys.argv[1]), Path(sys.argv[2])
    res = {}
    for raw in sorted(src.glob("*.raw.csv")):
        label = raw.name[: -len(".raw.csv")]
        try:
            d = load(raw)
        except Exception as e:  # noqa: BLE001
            print("skip", raw, e)
            continue
        out = (src / f"{label}.stdout")
        m = re.search(r"\bkernel (k_\S+)", out.read_text()) if out.exists() else None
        d["kernel"] = m.group(1) if m else d["kernel_demangled"]
        if "k_seed" in d["kernel_demangled"] or not m:  # (the seeding, or a plan: the name ncu reports)
            d["kernel"] = re.sub(r"^(?:void )?(?:\w+>)?::(k_\w+(<[^>]*>)?).*$", r"\1", d["kernel_demangled"])
        res[label] = d
    lines = ["| capture | kernel (wlp_last_kernel) | ms | issue % | ALU % | FMA % | FP64 % | XU % | threads/warp-instr | "
             "branch uniform % | warps/SM | regs | warp-instr | DRAM MB | top stalls (per issue) |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for label, d in res.items():
        dram = (d.get("dram_read", 0) + d.get("dram_write", 0)) / 1e6
        lines.append(f"| {label} | `{d['kernel']}` | {d.get('time_ms', 0):.3f} | {d.get('issue_pct', 0):.1f} | "
                     f"{d.get('alu_pct', 0):.1f} | {d.get('fma_pct', 0):.1f} | {d.get('fp64_pct', 0):.1f} | "
                     f"{d.get('xu_pct', 0):.1f} | {d.get('threads_per_warp_instr', 0):.2f} | "
                     f"{d.get('branch_uniform_pct', 0):.1f} | {d.get('warps_per_sm', 0):.1f} | {d.get('regs', 0):.0f} | "
                     f"{d.get('warp_instr', 0):.4g} | {dram:.1f} | "
                     + ", ".join(f"{k} {v}" for k, v in d["top_stalls"].items()) + " |")
    prefix.with_suffix(".md").write_text("\n".join(lines) + "\n")
    prefix.with_suffix(".json").write_text(json.dumps(res, indent=1) + "\n")
    summ_path = ROOT / "profiles" / "ncu_summary.json"
    summ = json.loads(summ_path.read_text()) if summ_path.exists() else {}
    for label, d in res.items():
        summ.setdefault(d["kernel"], {})[f"{prefix.name}_{label}"] = {
            "dram_bytes_per_launch": d.get("dram_read", 0) + d.get("dram_write", 0), "time_ms": d.get("time_ms")}
    summ_path.write_text(json.dumps(summ, indent=1) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
