#!/usr/bin/env python3
"""GPU timeline of a few back-to-back runs (CUPTI through torch.profiler; run on the GPU
box): every kernel / memset / memcpy with its start, duration and the gap before it.

    python tools/timeline.py walk 100000 1000 [--report]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1501_01405_b200 as w  # noqa: E402

model = w.model_from_name(sys.argv[1])
R, N = int(sys.argv[2]), int(sys.argv[3])
report = "--report" in sys.argv
p = w.ModelParams(replications=R, draws=N, clients=N, steps=N)
outs = [torch.empty(R, dtype=torch.float64, device="cuda") for _ in w.OUTPUT_NAMES[model]]


def run():
    w.run_shard(model, p, w.ExecutionMode.Wlp, 42, 0, R, outs, on_device=True,
                report=w.SimReport() if report else None)


for _ in range(5):
    run()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(4):
        run()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ev.sort(key=lambda e: e.time_range.start)
prev = None
for e in ev:
    s, d = e.time_range.start, e.time_range.end - e.time_range.start
    gap = s - prev if prev is not None else 0
    print(f"{s:12.1f} us  dur {d:8.2f}  gap {gap:7.2f}  {e.name[:70]}")
    prev = e.time_range.end
