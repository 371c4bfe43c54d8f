"""Experimental plan (BASELINE config 5): many factor-level sets in one launch, each set
bit-identical to its own run_model (the oracle loops run_model(Sequential) per set)."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _check_plan(gpu, port, model, sets, seeds):
    for mode in (gpu.ExecutionMode.Wlp, gpu.ExecutionMode.Tlp):
        got = gpu.run_plan(model, sets, seeds, mode)
        for k, (p, s) in enumerate(zip(sets, seeds)):
            want = port.run_model(int(model), oracle.params_from(p), s)
            for name in gpu.OUTPUT_NAMES[model]:
                assert np.array_equal(got[k][name], want[name]), (mode, k, name)


def test_config5_mm1_lambda_sweep(gpu, port):
    # 64 factor levels x 30 replications, lambda_k = mu * (0.1 + 0.8 k / 63), seed 42 + k
    sets = [gpu.ModelParams(replications=30, clients=10_000, lambda_=1.0 * (0.1 + 0.8 * k / 63), mu=1.0)
            for k in range(64)]
    _check_plan(gpu, port, gpu.ModelKind.Mm1, sets, [42 + k for k in range(64)])


def test_plan_heterogeneous_trip_counts(gpu, port):
    pi_sets = [gpu.ModelParams(replications=1 + (k * 7) % 40, draws=1 + 137 * k) for k in range(24)]
    _check_plan(gpu, port, gpu.ModelKind.Pi, pi_sets, [1000 + k for k in range(24)])
    walk_sets = [gpu.ModelParams(replications=3 + k, steps=50 + 211 * k, chunks=2 + k) for k in range(16)]
    _check_plan(gpu, port, gpu.ModelKind.Walk, walk_sets, [7 * k for k in range(16)])
    mm1_sets = [gpu.ModelParams(replications=1 + k % 5, clients=1 + 97 * k, lambda_=0.25 + 0.05 * k, mu=1.0 + 0.5 * (k % 3))
                for k in range(12)]
    _check_plan(gpu, port, gpu.ModelKind.Mm1, mm1_sets, [99 + k for k in range(12)])


def test_plan_mm1_mixed_division_modes(gpu, port):
    # sets whose rates take the 2^k multiply, the reciprocal form and IEEE division in one
    # launch (the TLP plan falls back to division for every lane when any set needs it)
    rates = [(0.5, 1.0), (0.3, 0.9), (0.25, 2.0), (1.3e-290, 1.7e-290), (0.7, 0.75), (4.0, 3.0)]
    for pick in (rates, [r for r in rates if r[0] > 1e-100]):
        sets = [gpu.ModelParams(replications=7 + k, clients=200 + 31 * k, lambda_=lam, mu=mu)
                for k, (lam, mu) in enumerate(pick)]
        _check_plan(gpu, port, gpu.ModelKind.Mm1, sets, [5 + k for k in range(len(pick))])


def test_plan_errors(gpu):
    with pytest.raises(gpu.DomainError):
        gpu.run_plan(gpu.ModelKind.Pi, [gpu.ModelParams(draws=0)], [1], gpu.ExecutionMode.Wlp)
    with pytest.raises(gpu.DomainError):
        gpu.run_plan(gpu.ModelKind.Pi, [gpu.ModelParams()], [1, 2], gpu.ExecutionMode.Wlp)
