#!/usr/bin/env python3
"""Cost curves over the replication count on the B200 (the paper's Fig. 5-7 experiment,
PAPER.md:427-477, with measured kernel time instead of Fermi cycles): for each model and
mapping, the model-kernel time (CUDA events, min of 3) at R = 2^k.

    python tools/sweep_curves.py > profiles/round1_sweep_curves.csv
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1501_01405_b200 as w  # noqa: E402

print("model,mode,replications,units,kernel_ms,reps_per_s")
for model, units in ((w.ModelKind.Pi, 1000), (w.ModelKind.Mm1, 1000), (w.ModelKind.Walk, 1000)):
    for k in range(0, 24, 1):
        R = 1 << k
        p = w.ModelParams(replications=R, draws=units, clients=units, steps=units)
        outs = [torch.empty(R, dtype=torch.float64, device="cuda") for _ in w.OUTPUT_NAMES[model]]
        for mode in (w.ExecutionMode.Wlp, w.ExecutionMode.Tlp):
            ms = []
            for i in range(4):
                rep = w.SimReport()
                w.run_shard(model, p, mode, 42, 0, R, outs, on_device=True, report=rep)
                if i:
                    ms.append(rep.kernel_ms)
            best = min(ms)
            print(f"{w.model_name(model)},{w.mode_name(mode)},{R},{units},{best:.5f},{R / (best * 1e-3):.6g}",
                  flush=True)
