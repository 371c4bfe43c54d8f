#!/usr/bin/env python3
"""Randomised stress of every model x mode x kernel variant against the oracle port
(one-off, longer than the pytest suite's 150 configurations):

    python tools/stress_random.py [seconds] [seed] [large_share]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_1501_01405_b200 as w  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
LARGE = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0  # share of large-R configurations
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
port = oracle.Oracle("port")
t0, n, bad = time.time(), 0, 0
while time.time() - t0 < budget:
    model = int(rng.integers(0, 3))
    if rng.random() < LARGE:  # large R with few units: the walk's pipeline / lane-chunk switch
        R = int(rng.choice([100_000, 150_001, 400_000, 700_003, 1_000_000, 4_194_305, 5_000_003]))
        N = int(rng.choice([1, 16, 17, 33, 64, 100]))
    else:
        R = int(rng.choice([1, 7, 31, 32, 33, 63, 64, 65, 97, 128, 500, 1000, 4097, 6000]))
        N = int(rng.choice([1, 2, 15, 16, 17, 31, 32, 33, 100, 255, 256, 257, 999, 1000, 2049, 4096, 5000]))
    chunks = int(rng.choice([1, 2, 3, 30, 97, 1 << 20, (1 << 31) + 5, (1 << 53) + 3]))
    lam = float(rng.choice([0.125, 0.3, 0.5, 0.7, 0.9, 0.99, 1.5, 2.0]))
    mu = float(rng.choice([0.5, 1.0, 1.3, 0.9]))
    p = w.ModelParams(replications=R, draws=N, clients=N, steps=N, chunks=chunks, lambda_=lam, mu=mu)
    seed = int(rng.integers(0, 2**63))
    mode = w.ExecutionMode(int(rng.integers(0, 3)))
    wv, tv = int(rng.integers(0, 5)), int(rng.integers(0, 3))
    try:
        want = port.run_model(model, oracle.params_from(p), seed)
    except oracle.OracleError:  # invalid parameters: the engine must refuse them too
        want = None
    try:
        with w.wlp_variant(wv), w.tlp_variant(tv):
            run = w.run_model(w.ModelKind(model), p, mode, master_seed=seed,
                              tlp_block_size=int(rng.choice([32, 50, 256])))
    except w.DomainError:
        run = None
    if want is None or run is None:
        ok = want is None and run is None
    else:
        ok = all(np.array_equal(run.outputs[k], want[k]) for k in oracle.OUTPUTS[model])
    n += 1
    if not ok:
        bad += 1
        print("MISMATCH", model, R, N, chunks, lam, mu, mode, wv, tv, seed, w.last_kernel(), flush=True)
print(f"stress: {n} configurations, {bad} mismatches, {time.time() - t0:.0f} s")
sys.exit(1 if bad else 0)
