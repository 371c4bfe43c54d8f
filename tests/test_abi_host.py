"""The C ABI without a GPU: the library loads, exports every symbol include/wlp_b200.h
declares, and its host-side logic (reference utilities, GF(2) jump-ahead, spacing
rejection bookkeeping, statistics merge) matches the reference. CPU only."""
import re
import subprocess

import numpy as np
import pytest

import oracle
import paper_1501_01405_b200 as w
from conftest import ROOT, golden, unhex


def declared_symbols():
    text = (ROOT / "include" / "wlp_b200.h").read_text()
    return set(re.findall(r"^\s*(?:int|const char\*)\s+(wlp_\w+)\s*\(", text, re.M))


def test_exports_every_declared_symbol():
    decl = declared_symbols()
    assert len(decl) >= 20
    nm = subprocess.run(["nm", "-D", "--defined-only", str(w.LIB_PATH)], capture_output=True, text=True,
                        check=True).stdout
    exported = set(re.findall(r"\bT (wlp_\w+)", nm))
    assert decl <= exported, decl - exported
    assert set(w.EXPORTS) == decl  # the Python mirror binds exactly the header


def test_library_links_cuda_runtime_and_has_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", str(w.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_compute_without_gpu_fails_loudly():
    try:
        n = w.device_count()
    except w.Error:
        n = 0
    if n:
        pytest.skip("a GPU is present")
    with pytest.raises(w.Error):
        w.run_model(w.ModelKind.Pi, w.ModelParams(replications=2, draws=10), w.ExecutionMode.Wlp, master_seed=1)


def test_kernel_variant_knobs_and_last_kernel():
    # host-side setters: ranges checked, reset by the context managers; no run yet on this
    # thread, so no kernel name
    for bad in (-1, 5):
        with pytest.raises(w.DomainError):
            with w.wlp_variant(bad):
                pass
    for bad in (-1, 3):
        with pytest.raises(w.DomainError):
            with w.tlp_variant(bad):
                pass
    for bad in (-1, 1, 3, 12, 64):
        with pytest.raises(w.DomainError):
            with w.pipe_lanes(bad):
                pass
    for bad in (0, 3, 256):
        with pytest.raises(w.DomainError):
            with w.near_cap(bad):
                pass
    with w.wlp_variant(4), w.tlp_variant(2), w.pipe_lanes(8), w.near_cap(16):
        pass
    assert isinstance(w.last_kernel(), str)


def test_validate_params_matches_reference_semantics():
    P = w.ModelParams
    assert w.validate_params(w.ModelKind.Pi, P()) is None
    for model, p in [(w.ModelKind.Pi, P(draws=0)), (w.ModelKind.Pi, P(replications=0)),
                     (w.ModelKind.Mm1, P(clients=0)), (w.ModelKind.Mm1, P(lambda_=0.0)),
                     (w.ModelKind.Mm1, P(mu=-1.0)), (w.ModelKind.Walk, P(steps=0)),
                     (w.ModelKind.Walk, P(chunks=1))]:
        with pytest.raises(w.DomainError):
            w.validate_params(model, p)
    assert "unstable" in w.validate_params(w.ModelKind.Mm1, P(lambda_=1.0, mu=0.5))


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_plan_launch_matches_reference(ref, mode):
    for R in [1, 7, 31, 32, 33, 50, 64, 255, 256, 257, 1000, 65535]:
        for block in [32, 50, 128, 256, 1024]:
            dims, warn = ref.plan_launch(R, mode, block)
            plan = w.plan_launch(R, w.ExecutionMode(mode), tlp_block_size=block)
            assert (plan.cfg.blockDim[0], plan.cfg.gridDim[0], plan.cfg.warpSize) == dims
            assert plan.warning == warn
    with pytest.raises(w.PlanError):
        w.plan_launch(65536, w.ExecutionMode.Wlp)  # test_wlp.cpp:130 — the reference's grid cap
    with pytest.raises(w.PlanError):
        w.plan_launch(10, w.ExecutionMode.Tlp, tlp_block_size=2048)
    with pytest.raises(w.PlanError):
        w.plan_launch(0, w.ExecutionMode.Tlp)


def test_plan_launch_check_order():
    """wlp.cpp:73-76: replications, then the block's lower bound, then the profile limit."""
    with pytest.raises(w.PlanError, match="at least one replication"):
        w.plan_launch(0, w.ExecutionMode.Tlp, tlp_block_size=4096)
    with pytest.raises(w.PlanError, match=">= 1"):
        w.plan_launch(5, w.ExecutionMode.Tlp, w.DeviceProfile(maxThreadsPerBlock=16), tlp_block_size=0)
    with pytest.raises(w.PlanError, match="maxThreadsPerBlock"):
        w.plan_launch(5, w.ExecutionMode.Tlp, w.DeviceProfile(maxThreadsPerBlock=64), tlp_block_size=128)
    # a profile above CUDA's limit: the device limit, reported as such
    with pytest.raises(w.PlanError, match="device limit"):
        w.plan_launch(5, w.ExecutionMode.Tlp, w.DeviceProfile(maxThreadsPerBlock=4096), tlp_block_size=2048)


def test_master_from_seed_and_make_state(port):
    for seed in [0, 1, 42, 9001, 20260201, 2**64 - 1]:
        assert tuple(vars(w.rng_state_from_seed(seed)).values()) == port.master_from_seed(seed)
    assert w.make_rng_state(0, 0, 0) == w.RngState(2, 8, 16)
    assert w.make_rng_state(1, 7, 15) == w.RngState(3, 15, 31)
    assert w.make_rng_state(2, 8, 16) == w.RngState(2, 8, 16)


def test_host_jump_ahead_equals_sequential_steps(port):
    rng = np.random.default_rng(5)
    for _ in range(6):
        s = [int(x) for x in rng.integers(0, 2**32, 3)]
        st = w.make_rng_state(*s)
        n = int(rng.integers(1, 3000))
        seq = port.taus_stream(st.s1, st.s2, st.s3, n + 1)
        j = w.jump_state(st, n)
        # the next output after jumping n steps equals output n+1 of the sequential stream
        nxt = port.taus_stream(j.s1, j.s2, j.s3, 1)[0]
        assert nxt == seq[n]


def test_inverse_normal_cdf_bit_exact():
    for p, z in golden("stats.json")["z"].items():
        assert w.inverse_normal_cdf(float(p)).hex() == z
    with pytest.raises(w.DomainError):
        w.inverse_normal_cdf(1.0)


def _sp(index, key):
    return w.Special(index, *key, 0)


def test_spacing_rejections_bookkeeping():
    # no specials / distinct specials: nothing rejected
    assert w.spacing_rejections([]) == []
    assert w.spacing_rejections([_sp(3, (2, 9, 40)), _sp(10, (3, 9, 40))]) == []
    # equal keys: every later occurrence is rejected, in any input order
    sp = [_sp(40, (2, 8, 16)), _sp(5, (2, 8, 16)), _sp(17, (2, 8, 16)), _sp(9, (3, 8, 16))]
    assert w.spacing_rejections(sp) == [17, 40]
    # merged with an earlier list
    assert w.spacing_rejections(sp, prev=[1, 50]) == [1, 17, 40, 50]
    # 1000 consecutive rejections of one stream is the reference's Error (rng.cpp:80-82)
    with pytest.raises(w.Error):
        w.spacing_rejections([], prev=list(range(100, 1100)))
    assert len(w.spacing_rejections([], prev=list(range(100, 1099)))) == 999


def test_stats_merge_and_ci_match_reference(ref):
    x = np.random.default_rng(3).normal(2.0, 0.5, 1001)
    # build exact shard statistics on the host (sum, then centred SS about the mean)
    parts = np.array_split(x, 3)
    tot = w.Stats()
    for p in parts:
        tot = w.stats_merge(tot, w.Stats(len(p), float(np.sum(p)), 0.0, 0.0, 0.0, 0.0))
    mean = (tot.sum_hi + tot.sum_lo) / tot.n
    ss = w.Stats()
    for p in parts:
        ss = w.stats_merge(ss, w.Stats(0, 0.0, 0.0, 0.0, float(np.sum((p - mean) ** 2)), 0.0))
    tot.ss_hi, tot.ss_lo = ss.ss_hi, ss.ss_lo
    ci = w.ci_from_stats(tot, 0.95)
    m, hw, n, warn = ref.confidence_interval(x, 0.95)
    assert ci.n == n and ci.warnSmallSample == warn
    assert ci.mean == pytest.approx(m, rel=1e-12) and ci.halfWidth == pytest.approx(hw, rel=1e-12)
    with pytest.raises(w.DomainError):
        w.ci_from_stats(w.Stats(1, 1.0, 0, 0, 0, 0))
