#!/usr/bin/env python3
"""Three mappings of the same replications on the B200 (model-kernel ms, best of 3):
  * paper WLP  — the reference's own wrap_wlp IR kernel (one replication per warp, lane 0
                 alone), compiled by the IR JIT;
  * paper TLP  — the reference's wrap_tlp IR kernel, compiled the same way;
  * engine WLP / TLP — the hand-written kernels (lane-cooperative WLP).
The IR bodies keep the reference's per-unit global memory traffic (models.cpp:146-150,
233-237), so only the two IR columns compare mappings like for like.

    python tools/mapping_compare.py > profiles/round1_mapping_compare.txt
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1501_01405_b200 as w  # noqa: E402
from paper_1501_01405_b200 import ir  # noqa: E402

print(f"{'model':5} {'R':>6} {'IR wlp (paper)':>15} {'IR tlp':>8} {'engine wlp':>11} {'engine tlp':>11}")
for model in (w.ModelKind.Pi, w.ModelKind.Mm1, w.ModelKind.Walk):
    for R in (32, 1024, 8192, 65535):
        p = w.ModelParams(replications=R, draws=1000, clients=1000, steps=1000)
        row = []
        for mode in (w.ExecutionMode.Wlp, w.ExecutionMode.Tlp):
            ms = min(ir.run_model(model, p, mode, 42, jit=True).report.kernel_ms for _ in range(3))
            row.append(ms)
        outs = [torch.empty(R, dtype=torch.float64, device="cuda") for _ in w.OUTPUT_NAMES[model]]
        for mode in (w.ExecutionMode.Wlp, w.ExecutionMode.Tlp):
            best = 1e30
            for _ in range(3):
                rep = w.SimReport()
                w.run_shard(model, p, mode, 42, 0, R, outs, on_device=True, report=rep)
                best = min(best, rep.kernel_ms)
            row.append(best)
        print(f"{w.model_name(model):5} {R:>6} {row[0]:15.4f} {row[1]:8.4f} {row[2]:11.4f} {row[3]:11.4f}", flush=True)
