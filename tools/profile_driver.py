#!/usr/bin/env python3
"""Launch one configuration of the replication kernels for ncu (run on the GPU box).

    python tools/profile_driver.py MODEL MODE R N [--repeat K]
    ncu --set full --clock-control none --import-source on -k regex:k_wlp -s 1 -c 1 \
        -o gpurun_out/prof_pi_wlp python tools/profile_driver.py pi wlp 1000000 10000 --repeat 2
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_1501_01405_b200 as w  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("model", choices=["pi", "mm1", "walk"])
ap.add_argument("mode", choices=["sequential", "tlp", "wlp"])
ap.add_argument("R", type=int)
ap.add_argument("N", type=int)
ap.add_argument("--repeat", type=int, default=2)
ap.add_argument("--counters", action="store_true", help="instrumented kernels; print the SimReport tallies")
ap.add_argument("--ir", action="store_true", help="run the reference's IR kernel on the GPU IR interpreter")
ap.add_argument("--lambda", dest="lam", type=float, default=0.5)
ap.add_argument("--wlp-variant", type=int, default=0)
ap.add_argument("--tlp-variant", type=int, default=0)
ap.add_argument("--pipe-lanes", type=int, default=0)
a = ap.parse_args()
m = w.model_from_name(a.model)
p = w.ModelParams(replications=a.R, draws=a.N, clients=a.N, steps=a.N, lambda_=a.lam)
if a.ir:
    from paper_1501_01405_b200 import ir

    for _ in range(a.repeat):
        run = ir.run_model(m, p, w.mode_from_name(a.mode), 42)
    print(a.model, a.mode, a.R, a.N, "IR", "mean", float(run.primary.mean()), "report", run.report)
    sys.exit(0)
outs = [torch.empty(a.R, dtype=torch.float64, device="cuda") for _ in w.OUTPUT_NAMES[m]]
rep = w.SimReport()
ctx = w.hw_counters() if a.counters else None
if ctx:
    ctx.__enter__()
with w.wlp_variant(a.wlp_variant), w.tlp_variant(a.tlp_variant), w.pipe_lanes(a.pipe_lanes):
    for _ in range(a.repeat):
        w.run_shard(m, p, w.mode_from_name(a.mode), 42, 0, a.R, outs, on_device=True, report=rep)
if ctx:
    ctx.__exit__(None, None, None)
torch.cuda.synchronize()
print(a.model, a.mode, a.R, a.N, "mean", float(outs[0].mean()), "kernel", w.last_kernel(), "report", rep)
