"""The rest of the reference's rng / models header API on the device path (VERDICT r1
"complete the boundary"): the *_replication_u templates over caller-given uniforms
(wlp_run_uniforms) with the reference's scripted KATs and against the reference's own
templates (oracle/_ref ref_replications_u); exponential_from_u in bulk (wlp_exponentials)
and scalar; taus_next / uniform01 / TausStream; and run_model over several devices
(wlp_run_devices) — on a one-GPU box the same device listed twice, which runs the
multi-slice machinery (threads, barriers, global spacing check, merged statistics)."""
import math

import numpy as np
import pytest

import oracle
import paper_1501_01405_b200 as w
from conftest import golden

pytestmark = pytest.mark.gpu

REF = oracle.optional("reference")
need_ref = pytest.mark.skipif(REF is None, reason="oracle/_ref not built")


class ScriptedU:
    """test_models.cpp:16-24: a scripted uniform sequence, cycling when exhausted."""

    def __init__(self, us):
        self.us, self.i = list(us), 0

    def __call__(self):
        u = self.us[self.i % len(self.us)]
        self.i += 1
        return u


def u_for_exponential(x, rate):  # test_models.cpp:28
    return 1.0 - math.exp(-rate * x)


def test_pi_scripted(gpu):  # test_models.cpp:36-43
    assert w.pi_replication_u(10, ScriptedU([0.5, 0.5])) == 4.0
    assert w.pi_replication_u(10, ScriptedU([0.9, 0.9])) == 0.0
    assert w.pi_replication_u(2, ScriptedU([0.5, 0.5, 0.9, 0.9])) == 2.0
    assert w.pi_replication_u(1, ScriptedU([0.6, 0.8])) == 4.0  # x^2+y^2 == 1 exactly: inside
    with pytest.raises(w.DomainError, match="pi: draws must be >= 1"):
        w.pi_replication_u(0, ScriptedU([0.5]))


def test_mm1_hand_trace(gpu):  # test_models.cpp:58-65
    u = ScriptedU([u_for_exponential(1.0, 1.0), u_for_exponential(2.0, 1.0)])
    idle, wait, sys_ = w.mm1_replication_u(3, 1.0, 1.0, u)
    assert wait == pytest.approx(1.0, rel=1e-12)
    assert sys_ == pytest.approx(3.0, rel=1e-12)
    assert idle == pytest.approx(1.0 / 3.0, rel=1e-12)
    assert u.i == 6  # two draws per client, in order
    for bad in [(0, 1.0, 1.0), (3, 0.0, 1.0), (3, 1.0, -1.0)]:
        with pytest.raises(w.DomainError):
            w.mm1_replication_u(*bad, ScriptedU([0.5]))


def test_walk_scripted(gpu):  # test_models.cpp:123-137
    assert w.walk_replication_u(30, 30, ScriptedU([0.1, 0.9])) == 0.0
    assert w.walk_replication_u(31, 30, ScriptedU([0.1, 0.9])) == 1.0
    assert w.walk_replication_u(17, 30, ScriptedU([0.6, 0.6])) == 0.0
    assert w.walk_replication_u(1, 30, ScriptedU([0.3, 0.3])) == 29.0
    assert w.walk_replication_u(2, 30, ScriptedU([0.3, 0.3])) == 28.0
    assert w.walk_replication_u(1, 5, ScriptedU([0.25, 0.0])) == 4.0  # 4u = 1: second quarter
    assert w.walk_replication_u(1, 5, ScriptedU([0.999, 0.0])) == 0.0
    with pytest.raises(w.DomainError, match="walk: steps must be >= 1"):
        w.walk_replication_u(0, 30, ScriptedU([0.1]))
    with pytest.raises(w.DomainError, match="walk: chunks must be >= 2"):
        w.walk_replication_u(5, 1, ScriptedU([0.1]))


def _uniforms(rng, count, n):
    """Random doubles in [0,1) with the edges mixed in: 0, the walk's cut points, the
    pi circle's exact (0.6, 0.8), the largest double below 1, tiny and near-one values."""
    u = rng.random((count, 2 * n))
    edges = np.array([0.0, 0.25, 0.5, 0.75, 0.6, 0.8, np.nextafter(1.0, 0.0), 5e-324, 1e-300, 1 - 2**-30,
                      2**-4, 1 - 2**-4, 0.9375, 0.0625])
    mask = rng.random(u.shape) < 0.2
    u[mask] = rng.choice(edges, size=int(mask.sum()))
    return u


@need_ref
@pytest.mark.parametrize("model", [0, 1, 2])
def test_uniform_bodies_match_reference_templates(gpu, model):
    rng = np.random.default_rng(100 + model)
    for n, lam, mu, chunks in [(1, 0.5, 1.0, 2), (7, 0.3, 1.7, 5), (64, 0.9, 1.0, 30), (333, 3.0, 2.5, 7)]:
        p = w.ModelParams(draws=n, clients=n, steps=n, lambda_=lam, mu=mu, chunks=chunks)
        u = _uniforms(rng, 97, n)
        got = w.run_uniforms(model, p, u)
        want = REF.replications_u(model, oracle.params_from(p), u)
        for k in want:
            assert np.array_equal(got[k].view(np.uint64), want[k].view(np.uint64)), (model, n, k)


@need_ref
def test_exponentials_match_reference(gpu):
    rng = np.random.default_rng(7)
    u = np.concatenate([rng.random(50000), [0.0, np.nextafter(1.0, 0.0), 1e-300, 0.5, 1 - 2**-53, 2**-4]])
    for rate in (1.0, 0.5, 3.0, 1e-3, 7.25):
        got = w.exponentials(u, rate)
        want = REF.exponential_from_u(u, rate)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), rate
    with pytest.raises(w.DomainError, match=r"u outside \[0,1\)"):
        w.exponentials(np.array([0.5, 1.0]), 1.0)
    with pytest.raises(w.DomainError, match="rate must be > 0"):
        w.exponentials(np.array([0.5]), 0.0)


@need_ref
def test_scalar_rng_utilities(gpu):
    g = golden("taus88.json")
    st = w.make_rng_state(*g["seed"])
    assert [w.taus_next(st) for _ in range(100)] == g["outputs"]  # test_rng.cpp:43-57
    st = w.rng_state_from_seed(5150)
    probe = w.RngState(st.s1, st.s2, st.s3)
    u1 = w.uniform01(probe)
    assert u1 == w.taus_stream(st, 1)[0] * 2.0**-32
    for u, rate in [(0.0, 1.0), (1.0 - math.exp(-1.0), 1.0), (0.5, 2.0), (0.999, 0.3)]:
        assert w.exponential_from_u(u, rate) == REF.exponential_from_u([u], rate)[0]
    for u, rate in [(0.5, 0.0), (0.5, -1.0), (1.0, 1.0), (-0.1, 1.0)]:
        with pytest.raises(w.DomainError):
            w.exponential_from_u(u, rate)
    # TausStream through the template equals the stream form (same draws, same body)
    s = w.rng_state_from_seed(923)
    assert w.pi_replication_u(500, w.TausStream(s)) == w.pi_replication(500, s)
    assert w.walk_replication_u(57, 7, w.TausStream(s)) == w.walk_replication(57, 7, s)
    assert w.mm1_replication_u(90, 0.5, 1.0, w.TausStream(s)) == w.mm1_replication(90, 0.5, 1.0, s)


@pytest.mark.parametrize("model", [w.ModelKind.Pi, w.ModelKind.Mm1, w.ModelKind.Walk])
@pytest.mark.parametrize("mode", [w.ExecutionMode.Wlp, w.ExecutionMode.Tlp])
def test_run_devices_slices_equal_single_device(gpu, model, mode):
    p = w.ModelParams(replications=100_003, draws=50, clients=40, steps=60, chunks=7)
    one = w.run_model(model, p, mode, master_seed=42)
    ci_one = [w.confidence_interval(one.outputs[k]) for k in w.OUTPUT_NAMES[model]]
    for devs in ([0], [0, 0], [0, 0, 0]):
        rep = w.SimReport()
        outs, cis = w.run_devices(model, p, mode, 42, devs, ci_level=0.95, report=rep)
        for k, o in zip(w.OUTPUT_NAMES[model], outs):
            assert np.array_equal(o, one.outputs[k]), (devs, k)
        for a, b in zip(cis, ci_one):
            assert a.n == b.n == p.replications
            assert a.mean == pytest.approx(b.mean, rel=1e-12, abs=1e-15)
            assert a.halfWidth == pytest.approx(b.halfWidth, rel=1e-12)
        assert rep.kernel_ms > 0


def test_run_devices_through_run_model_options(gpu):
    p = w.ModelParams(replications=70_000, draws=20)
    a = w.run_model(w.ModelKind.Pi, p, w.ExecutionMode.Wlp, master_seed=9)
    n = w.device_count()
    b = w.run_model(w.ModelKind.Pi, p, w.ExecutionMode.Wlp, master_seed=9, opts=w.SimOptions(devices=n))
    assert np.array_equal(a.primary, b.primary)


def test_run_devices_errors(gpu):
    p = w.ModelParams(replications=10, draws=5)
    with pytest.raises(w.DomainError, match="does not exist"):
        w.run_devices(w.ModelKind.Pi, p, w.ExecutionMode.Wlp, 1, [0, 999])
    with pytest.raises(w.DomainError, match="at least one device"):
        w.run_devices(w.ModelKind.Pi, p, w.ExecutionMode.Wlp, 1, [])
    with pytest.raises(w.DomainError):
        w.run_devices(w.ModelKind.Pi, w.ModelParams(replications=0), w.ExecutionMode.Wlp, 1, [0])
