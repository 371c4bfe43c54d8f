"""Full-size parity at BASELINE configs 2-4 against the reference itself (oracle/_ref, the
reference sources compiled unmodified, on every host core):

  * config 2 (pi, 10^6 x 10^4) and config 3 (walk, 10^5 x 10^3): EVERY replication of
    the WLP and TLP runs bit for bit against the reference's random_spacing +
    pi_/walk_replication (models.cpp:46-59, rng.cpp:67-87);
  * config 4 (10^7 x 10^3 per model): the device's 10^7 stream keys equal the reference's
    random_spacing, and 10^5 random replications per model (plus the first and last)
    equal the reference's replication functions bit for bit;
  * every config: over the same full output array, the reference-order device confidence
    interval (wlp_set_stats_order(1)) bit-identical to the reference's confidence_interval
    (models.cpp:99-119); the default accurate one (wlp_run) and the merged multi-slice one
    (wlp_run_devices) within 1e-13 of the exactly rounded statistics, and within the
    reference's own rounding drift (n * 2^-53, at least 1e-12) of the reference's.
"""
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

NTH = os.cpu_count() or 1
SEED = 42


def _rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def _device_outputs(gpu, model, p, mode, ci=False):
    import torch

    outs = [torch.empty(p.replications, dtype=torch.float64, device="cuda") for _ in oracle.OUTPUTS[model]]
    cis = gpu.run_model_into(gpu.ModelKind(model), p, mode, SEED, outs, on_device=True, ci_level=0.95 if ci else None)
    torch.cuda.synchronize()
    return [o.cpu().numpy() for o in outs], cis


def _exact_ci(x, level=0.95):
    """The confidence interval with exactly rounded sums (math.fsum) and the reference's
    quantile: what the accurate device statistics approximate to a few ulps."""
    import math

    import paper_1501_01405_b200 as w

    n = len(x)
    mean = math.fsum(x) / n
    d = x - mean
    ss = math.fsum(d * d)
    z = w.inverse_normal_cdf(0.5 + level / 2)
    return mean, z * math.sqrt(ss / (n - 1)) / math.sqrt(n)


def _check_cis(gpu, ref, model, p, outs, device_cis):
    """Device CI (accurate order) and the 3-slice merged CI within 1e-13 of the exactly
    rounded statistics and within the reference's own rounding error of its naive loop
    (n * 2^-53 relative, at least 1e-12); the reference-order CI bit-identical to the
    reference's confidence_interval (models.cpp:99-119)."""
    _, merged = gpu.run_devices(gpu.ModelKind(model), p, gpu.ExecutionMode.Wlp, SEED, [0, 0, 0], ci_level=0.95)
    with gpu.stats_order(1):
        _, seq = _device_outputs(gpu, model, p, gpu.ExecutionMode.Wlp, ci=True)
    naive_tol = max(1e-12, p.replications * 2.0**-53)
    for k, name in enumerate(oracle.OUTPUTS[model]):
        mean, hw, n, warn = ref.confidence_interval(outs[k])
        emean, ehw = _exact_ci(outs[k])
        for c in (device_cis[k], merged[k]):
            assert c.n == n == p.replications
            assert _rel(c.mean, emean) <= 1e-13 and _rel(c.halfWidth, ehw) <= 1e-13, (name, c, emean, ehw)
            assert _rel(c.mean, mean) <= naive_tol, (name, c.mean, mean)
            assert _rel(c.halfWidth, hw) <= naive_tol, (name, c.halfWidth, hw)
            assert c.warnSmallSample == warn
        assert (seq[k].mean, seq[k].halfWidth, seq[k].n, seq[k].warnSmallSample) == (mean, hw, n, warn), name


@pytest.mark.parametrize("model,kw", [(0, dict(replications=1_000_000, draws=10_000)),
                                      (2, dict(replications=100_000, steps=1000, chunks=30))],
                         ids=["cfg2-pi-1e6x1e4", "cfg3-walk-1e5x1e3"])
def test_every_replication_equals_reference(gpu, ref, model, kw):
    p = gpu.ModelParams(**kw)
    keys = ref.random_spacing(SEED, p.replications)
    assert np.array_equal(gpu.random_spacing_seed(SEED, p.replications), keys)
    want = ref.replications(model, oracle.params_from(p), keys, nthreads=NTH)
    for mode in (gpu.ExecutionMode.Wlp, gpu.ExecutionMode.Tlp):
        outs, cis = _device_outputs(gpu, model, p, mode, ci=True)
        for a, name in zip(outs, oracle.OUTPUTS[model]):
            assert np.array_equal(a.view(np.uint64), want[name].view(np.uint64)), (mode, name)
    _check_cis(gpu, ref, model, p, outs, cis)


@pytest.fixture(scope="module")
def ref_keys_1e7(ref):
    return ref.random_spacing(SEED, 10_000_000)  # the reference's own sequential loop (~15 s)


def test_cfg4_stream_keys_equal_reference(gpu, ref_keys_1e7):
    assert np.array_equal(gpu.random_spacing_seed(SEED, 10_000_000), ref_keys_1e7)


@pytest.mark.parametrize("model,kw", [(0, dict(draws=1000)), (1, dict(clients=1000)),
                                      (2, dict(steps=1000, chunks=30))], ids=["pi", "mm1", "walk"])
def test_cfg4_sampled_replications_and_ci(gpu, ref, ref_keys_1e7, model, kw):
    p = gpu.ModelParams(replications=10_000_000, **kw)
    outs, cis = _device_outputs(gpu, model, p, gpu.ExecutionMode.Wlp, ci=True)
    rng = np.random.default_rng(4 + model)
    idx = np.unique(np.concatenate([rng.choice(p.replications, 100_000, replace=False), [0, p.replications - 1]]))
    want = ref.replications(model, oracle.params_from(p), np.ascontiguousarray(ref_keys_1e7[:, idx]), nthreads=NTH)
    for a, name in zip(outs, oracle.OUTPUTS[model]):
        assert np.array_equal(a[idx].view(np.uint64), want[name].view(np.uint64)), name
    _check_cis(gpu, ref, model, p, outs, cis)
