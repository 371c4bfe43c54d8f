#!/usr/bin/env python3
"""Small runs of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool racecheck python tools/sanitize_driver.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402

import paper_1501_01405_b200 as w  # noqa: E402

M, E = w.ModelKind, w.ExecutionMode
for model in (M.Pi, M.Mm1, M.Walk):
    for R, N in ((5, 77), (70, 300), (40, 4000)):
        p = w.ModelParams(replications=R, draws=N, clients=N, steps=N, lambda_=0.3, mu=0.9)
        for mode in (E.Tlp, E.Wlp):
            for variant in (0, 1, 2):
                with w.wlp_variant(variant):
                    w.run_model(model, p, mode, master_seed=7)
# the warp pipelines at a size where auto selection picks them, and the instrumented kernels
for model in (M.Pi, M.Mm1, M.Walk):
    w.run_model(model, w.ModelParams(replications=150_000, draws=40, clients=40, steps=40), E.Wlp, master_seed=5)
# the walk's bitsliced kernels: lane chunks (auto), the pipeline with seeding-written planes
# (auto at large R) and with its own plane pass (forced at small R), the bitsliced TLP
w.run_model(M.Walk, w.ModelParams(replications=20_000, steps=100), E.Wlp, master_seed=5)
w.run_model(M.Walk, w.ModelParams(replications=500_000, steps=20), E.Wlp, master_seed=5)
with w.wlp_variant(3):
    w.run_model(M.Walk, w.ModelParams(replications=3_000, steps=70), E.Wlp, master_seed=5)
with w.tlp_variant(2):
    w.run_model(M.Walk, w.ModelParams(replications=3_001, steps=70), E.Tlp, master_seed=5)
    with w.hw_counters():
        for mode in (E.Tlp, E.Wlp):
            w.run_model(model, w.ModelParams(replications=100, draws=300, clients=300, steps=300), mode, master_seed=5)
sets = [w.ModelParams(replications=3 + k, clients=100 + 37 * k, lambda_=0.2 + 0.1 * k, mu=1.0) for k in range(6)]
for mode in (E.Tlp, E.Wlp):
    w.run_plan(M.Mm1, sets, list(range(6)), mode)
    w.run_plan(M.Walk, [w.ModelParams(replications=4, steps=50 + 90 * k) for k in range(5)], list(range(5)), mode)
# round 2: the wrapped pipelines at every lanes-per-replication S (forced at small R: fewer
# warps, each with its wrap replications), the single-pass mm1 pipeline (mu = 1 and a
# general rate; its near-one overflow redo forced by a small list capacity), the bitsliced
# walk pipeline with wrap groups at S = 4 / 8 / 32; the two-lane pipelines (S = 2)
for lanes in (2, 4, 8, 16, 32):
    with w.wlp_variant(2), w.pipe_lanes(lanes):
        for model in (M.Pi, M.Walk):
            w.run_model(model, w.ModelParams(replications=1100, draws=999, steps=999), E.Wlp, master_seed=11)
for lanes in (2, 8, 32):
    for cap in (128, 4):
        with w.wlp_variant(2), w.pipe_lanes(lanes), w.near_cap(cap):
            w.run_model(M.Mm1, w.ModelParams(replications=1100, clients=512), E.Wlp, master_seed=11)
            w.run_model(M.Mm1, w.ModelParams(replications=1100, clients=520, lambda_=0.3, mu=0.9), E.Wlp,
                        master_seed=12)
for lanes in (4, 8, 32):
    with w.wlp_variant(3), w.pipe_lanes(lanes):
        w.run_model(M.Walk, w.ModelParams(replications=70_000, steps=300), E.Wlp, master_seed=13)
w.confidence_interval(list(np.linspace(0.0, 1.0, 1000)), 0.95)
for jit in (False, True):
    w.run_model(M.Walk, w.ModelParams(replications=64, steps=100), E.Tlp, master_seed=3,
                opts=w.SimOptions(irInterpreter=True, irJit=jit))
print("sanitize driver done")
