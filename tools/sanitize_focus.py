"""Focused compute-sanitizer driver for one round-2 kernel family (run on the GPU box):

    compute-sanitizer --tool racecheck python tools/sanitize_focus.py pipe|mm1|bs|seed|seed128|planes|plan
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_1501_01405_b200 as w  # noqa: E402
M, E = w.ModelKind, w.ExecutionMode
which = sys.argv[1]
if which == "pipe":
    for lanes in (2, 4, 32):
        with w.wlp_variant(2), w.pipe_lanes(lanes):
            w.run_model(M.Pi, w.ModelParams(replications=1100, draws=999), E.Wlp, master_seed=11)
elif which == "mm1":
    for lanes in (2, 8):
        with w.wlp_variant(2), w.pipe_lanes(lanes), w.near_cap(4):
            w.run_model(M.Mm1, w.ModelParams(replications=1100, clients=512), E.Wlp, master_seed=11)
elif which == "bs":
    with w.wlp_variant(3), w.pipe_lanes(4):
        w.run_model(M.Walk, w.ModelParams(replications=70_000, steps=300), E.Wlp, master_seed=13)
elif which == "seed":
    w.run_model(M.Walk, w.ModelParams(replications=20_000, steps=100), E.Tlp, master_seed=5)
elif which == "seed128":  # 128 slots per thread, batched swizzled staging, rejections, a ragged end
    R = (1 << 22) + 1_017
    w.seed_streams(9, 0, R, rejected=[3, 31, 32, 33, 127, 128, 4_096, R - 40, R - 1])
    w.seed_streams(9, 77, R - 500)
elif which == "planes":  # the seeding writes bit planes only; the pipeline's wrap groups read them
    with w.wlp_variant(3):
        w.run_model(M.Walk, w.ModelParams(replications=(1 << 22) + 37, steps=16, chunks=7), E.Wlp, master_seed=7)
elif which == "plan":  # PDL-chained plan seeding + model, asynchronous return into device buffers
    import torch

    for m, sets in ((M.Walk, [w.ModelParams(replications=30, steps=100 + 30 * k, chunks=30) for k in range(16)]),
                    (M.Mm1, [w.ModelParams(replications=30, clients=300, lambda_=0.1 + 0.05 * k, mu=1.0)
                             for k in range(16)])):
        outs = [torch.empty(16 * 30, dtype=torch.float64, device="cuda") for _ in range(3)]
        ps = w.PlanSets(sets, [42 + k for k in range(16)])
        for _ in range(3):
            w.run_plan(m, ps, None, E.Wlp, outs, on_device=True)
        torch.cuda.synchronize()
print("done", which)
