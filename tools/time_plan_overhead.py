#!/usr/bin/env python3
"""Per-call cost of BASELINE config 5 plans on the GPU box (device-resident outputs),
with and without a SimReport, against the plan kernel alone.

    python tools/time_plan_overhead.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1501_01405_b200 as w  # noqa: E402

SEEDS = [42 + k for k in range(64)]
CASES = {
    "mm1_64x30x1e4": (w.ModelKind.Mm1, [w.ModelParams(replications=30, clients=10_000, lambda_=0.1 + 0.8 * k / 63,
                                                      mu=1.0) for k in range(64)], 3),
    "walk_hetero_64x30": (w.ModelKind.Walk, [w.ModelParams(replications=30, steps=100 + 30 * k, chunks=30)
                                             for k in range(64)], 1),
}
s = torch.cuda.current_stream()
for name, (m, sets, nout) in CASES.items():
    plan = w.PlanSets(sets, SEEDS)
    outs = [torch.empty(64 * 30, dtype=torch.float64, device="cuda") for _ in range(nout)]
    kms = []
    for i in range(8):
        rep = w.SimReport()
        w.run_plan(m, plan, None, w.ExecutionMode.Wlp, outs, on_device=True, report=rep)
        kms.append(rep.kernel_ms)
    res = {"kernel_ms": min(kms[2:])}
    for label, mk in (("run_ms", lambda: None), ("run_ms_report", w.SimReport)):
        for _ in range(3):
            w.run_plan(m, plan, None, w.ExecutionMode.Wlp, outs, on_device=True, report=mk())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(50):
            w.run_plan(m, plan, None, w.ExecutionMode.Wlp, outs, on_device=True, report=mk())
        e1.record(s)
        torch.cuda.synchronize()
        res[label] = e0.elapsed_time(e1) / 50
    print(name, " ".join(f"{k} {v:.4f}" for k, v in res.items()), f"run/kernel {res['run_ms'] / res['kernel_ms']:.2f}")
