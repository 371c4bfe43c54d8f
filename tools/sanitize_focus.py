"""Focused compute-sanitizer driver for one round-2 kernel family (run on the GPU box):

    compute-sanitizer --tool racecheck python tools/sanitize_focus.py pipe|mm1|bs|seed
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
print("done", which)
