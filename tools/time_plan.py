#!/usr/bin/env python3
"""Time BASELINE config 5 (mm1 plan: 64 sets x 30 replications x 10^4 clients, one
launch) on the GPU box: model-kernel ms, min over repeats.  python tools/time_plan.py [wlp|tlp]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1501_01405_b200 as w  # noqa: E402

mode = w.mode_from_name(sys.argv[1] if len(sys.argv) > 1 else "wlp")
sets = [w.ModelParams(replications=30, clients=10_000, lambda_=0.1 + 0.8 * k / 63, mu=1.0) for k in range(64)]
seeds = [42 + k for k in range(64)]
outs = [torch.empty(64 * 30, dtype=torch.float64, device="cuda") for _ in range(3)]
plan = w.PlanSets(sets, seeds)
ms = []
for i in range(6):
    rep = w.SimReport()
    w.run_plan(w.ModelKind.Mm1, plan, None, mode, outs, on_device=True, report=rep)
    torch.cuda.synchronize()
    if i:
        ms.append(rep.kernel_ms)
print(f"plan {w.mode_name(mode)} kernel_ms min {min(ms):.4f}")
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for i in range(20):
    w.run_plan(w.ModelKind.Mm1, plan, None, mode, outs, on_device=True, report=w.SimReport())
e1.record(s)
torch.cuda.synchronize()
print(f"plan {w.mode_name(mode)} ms_per_run {e0.elapsed_time(e1) / 20:.4f}")
