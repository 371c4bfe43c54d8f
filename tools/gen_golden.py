#!/usr/bin/env python3
"""Generate tests/golden/* from the reference itself (run in the build container).

Sources:
  * /root/reference/proj/taus88.golden and tests/golden/sweep_pi.golden — the
    reference's own golden vectors, re-checked against oracle/_ref and stored as
    fixtures (the GPU box has no /root/reference).
  * oracle/_ref/libwarpsim_ref.so — the reference sources compiled unmodified
    (oracle/Makefile): per-replication outputs of run_model(Sequential) for the seeds,
    models and replication counts the reference's tests use (acceptance_test.cpp:250-277,
    test_models.cpp:276-326), -log(1-u) values from the host glibc, CI values.

Doubles are stored as float.hex strings (bit-exact round trip).

    make -C oracle && python tools/gen_golden.py
"""
from __future__ import annotations

import hashlib
import json
import platform
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402

GOLD = ROOT / "tests" / "golden"
REF = Path("/root/reference/proj")


def hexs(a) -> list:
    return [float(x).hex() for x in np.asarray(a, dtype=np.float64)]


def keys_digest(k: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(k, dtype="<u4").tobytes()).hexdigest()


def main() -> None:
    GOLD.mkdir(parents=True, exist_ok=True)
    ref = oracle.Oracle("reference")

    # 1. taus88.golden (proj/taus88.golden): seed line + 100 outputs
    lines = (REF / "taus88.golden").read_text().split()
    seed = [int(x) for x in lines[:3]]
    outs = [int(x) for x in lines[3:]]
    assert len(outs) == 100
    assert list(ref.taus_stream(*seed, 100)) == outs
    (GOLD / "taus88.json").write_text(json.dumps({"source": "proj/taus88.golden", "seed": seed, "outputs": outs}))

    # 2. sweep_pi.golden (proj/tests/golden/sweep_pi.golden): byte-stable CSV
    csv = (REF / "tests" / "golden" / "sweep_pi.golden").read_text()
    assert ref.sweep_csv(0, 7, 1, 2, 1, oracle.params(draws=100), 42) == csv
    (GOLD / "sweep_pi.csv").write_text(csv)

    # 3. per-replication outputs of run_model(Sequential)
    cases = []
    small = dict(draws=200, clients=150, steps=120, chunks=7)  # acceptance_test.cpp:256-259
    for seed_ in (42, 9001, 20260201):
        for model in (0, 1, 2):
            for R in (1, 7, 32, 33):
                p = oracle.params(replications=R, **small)
                res = ref.run_model(model, p, seed_)
                cases.append({"seed": seed_, "model": model, "params": dict(replications=R, **small),
                              "outputs": {k: hexs(v) for k, v in res.items() if not k.startswith("_")}})
            # default ModelParams (models.hpp:24-30), one warp's worth of replications
            p = oracle.params(replications=32)
            res = ref.run_model(model, p, seed_)
            cases.append({"seed": seed_, "model": model, "params": dict(replications=32),
                          "outputs": {k: hexs(v) for k, v in res.items() if not k.startswith("_")}})
    # ragged / edge shapes: N below a warp, N not a multiple of 32, tiny chunks, lambda >= mu
    edge = [(0, dict(replications=5, draws=1)), (0, dict(replications=3, draws=31)),
            (0, dict(replications=3, draws=33)), (2, dict(replications=4, steps=1, chunks=2)),
            (2, dict(replications=4, steps=63, chunks=2)), (1, dict(replications=3, clients=1)),
            (1, dict(replications=3, clients=257, lambda_=1.0, mu=0.5)),
            (1, dict(replications=2, clients=300, lambda_=0.3, mu=0.7)),
            # extreme rates: overflow to inf / underflow, non power-of-two and 2^k rates
            (1, dict(replications=3, clients=50, lambda_=1e-300, mu=1e300)),
            (1, dict(replications=3, clients=50, lambda_=2.0**-600, mu=2.0**700)),
            (1, dict(replications=3, clients=50, lambda_=3.0, mu=0.1)),
            # chunks beyond 2^53: the reference folds in double with c rounded
            (2, dict(replications=3, steps=101, chunks=2**60 + 1)),
            (2, dict(replications=3, steps=101, chunks=2**53 + 1)),
            (0, dict(replications=2, draws=2**20 + 3))]
    for model, kw in edge:
        res = ref.run_model(model, oracle.params(**kw), 7)
        cases.append({"seed": 7, "model": model, "params": kw,
                      "outputs": {k: hexs(v) for k, v in res.items() if not k.startswith("_")}})
    (GOLD / "replications.json").write_text(json.dumps({"generator": "oracle/_ref run_model Sequential",
                                                        "cases": cases}))

    # 4. random_spacing keys
    sp = {}
    for seed_, R in ((42, 1000), (9001, 4096), (20260201, 100000)):
        k = ref.random_spacing(seed_, R)
        sp[str(seed_)] = {"count": R, "sha256": keys_digest(k), "head": k[:, :4].T.tolist(),
                          "master": list(ref.master_from_seed(seed_))}
    (GOLD / "spacing.json").write_text(json.dumps(sp))

    # 5. -log(1-u) through the reference's exponential_from_u (host glibc log)
    rng = np.random.default_rng(1501)
    ks = np.concatenate([np.arange(0, 64), 2**32 - 1 - np.arange(0, 64),
                         (1 << 28) + np.arange(-64, 64),  # near-one window edge (u = 1/16)
                         rng.integers(0, 2**32, 4096)]).astype(np.uint64)
    u = ks.astype(np.float64) * 2.0**-32
    v = ref.exponential_from_u(u, 1.0)
    (GOLD / "log_pairs.json").write_text(json.dumps({
        "glibc": platform.libc_ver(), "host_log_variant": oracle.host_log_variant(),
        "k": [int(x) for x in ks], "neg_log1m": hexs(v)}))

    # 6. statistics
    cis = []
    for vec, level in (([1.0, 2.0, 3.0, 4.0, 5.0], 0.95), ([2.5] * 4, 0.95), ([float(i % 2) for i in range(30)], 0.99),
                       (list(rng.normal(3.0, 2.0, 300)), 0.95), (list(rng.normal(-1.0, 0.1, 257)), 0.9)):
        m, hw, n, w = ref.confidence_interval(vec, level)
        cis.append({"x": hexs(vec), "level": level, "mean": float(m).hex(), "half_width": float(hw).hex(),
                    "n": n, "warn": w})
    zs = {str(p): float(ref.inverse_normal_cdf(p)).hex() for p in (0.005, 0.025, 0.1, 0.4, 0.5, 0.6, 0.9, 0.975,
                                                                    0.9995)}
    (GOLD / "stats.json").write_text(json.dumps({"ci": cis, "z": zs}))

    # 7. statistical pins at seed 42 (acceptance criteria 6-8) as digests of full outputs
    pins = {}
    r = ref.run_model(0, oracle.params(replications=1, draws=1_000_000), 42)
    pins["pi_1x1e6"] = {"out": hexs(r["out"])}
    r = ref.run_model(1, oracle.params(replications=30, clients=100_000), 42)
    pins["mm1_30x1e5"] = {k: hexs(v) for k, v in r.items() if not k.startswith("_")}
    r = ref.run_model(2, oracle.params(replications=3000, steps=1000, chunks=30), 42)
    pins["walk_3000x1000"] = {"sha256": hashlib.sha256(r["out"].astype("<f8").tobytes()).hexdigest(),
                              "head": hexs(r["out"][:8])}
    (GOLD / "pins.json").write_text(json.dumps(pins))
    print("golden fixtures written to", GOLD)


if __name__ == "__main__":
    main()
