"""Parity of the sm_100a path (through the C ABI) with the CPU oracle: bit-exact raw
streams, stream seeds and per-replication outputs; aggregate statistics within 1e-12
relative (bit-exact for R <= 256, where the device sums sequentially like the
reference, models.cpp:104-109). Run on the B200 box: pytest -m gpu."""
import hashlib

import numpy as np
import pytest

import oracle
from conftest import GOLD, golden, unhex

pytestmark = pytest.mark.gpu

MODES = ("Sequential", "Tlp", "Wlp")


def P(w, **kw):
    return w.ModelParams(**kw)


def hexes(a):
    return [float(x).hex() for x in a]


def test_native_library_is_the_cuda_build(gpu):
    lib = gpu.native_library()
    assert lib._name.endswith("libwlp_b200.so")
    assert gpu.device_count() >= 1


# ---- raw streams and seeding ------------------------------------------------------------


def test_taus88_golden(gpu):
    g = golden("taus88.json")  # proj/taus88.golden
    got = gpu.taus_stream(gpu.RngState(*g["seed"]), 100)
    assert got.tolist() == g["outputs"]


def test_taus_stream_long_jump_ahead(gpu, port):
    # 64-output chunks per thread start by GF(2) jump-ahead: every chunk boundary checked
    for seed in [(1, 2, 3), (2, 8, 16), (0xFFFFFFFF, 0xFFFFFFF0, 0x80000000), (123456789, 362436069, 521288629)]:
        st = gpu.make_rng_state(*seed)
        got = gpu.taus_stream(st, 200_003)
        assert np.array_equal(got, port.taus_stream(*seed, 200_003))


def test_random_spacing_digests(gpu):
    for seed, want in golden("spacing.json").items():
        k = gpu.random_spacing_seed(int(seed), want["count"])
        assert k[:, :4].T.tolist() == want["head"]
        assert hashlib.sha256(np.ascontiguousarray(k, dtype="<u4").tobytes()).hexdigest() == want["sha256"]


def test_random_spacing_large_vs_port(gpu, port):
    k = gpu.random_spacing_seed(77, 1_000_003)
    assert np.array_equal(k, port.random_spacing(77, 1_000_003))


def test_seed_shards_and_rejection_remap(gpu, port):
    R = 20_000
    whole = port.random_spacing(5, R + 3)
    # shards of the same run concatenate to the whole run
    parts = [gpu.seed_streams(5, b, c)[0] for b, c in ((0, 7000), (7000, 1), (7001, R - 7001))]
    assert np.array_equal(np.concatenate(parts, axis=1), whole[:, :R])
    # a rejection list (as produced by a key collision) skips those candidates, exactly
    # like random_spacing's redraw loop (rng.cpp:74-84)
    rej = [0, 4, 5, 19_999]
    keys, _ = gpu.seed_streams(5, 0, R - 1, rejected=rej)
    keep = np.array([i for i in range(R + 3) if i not in rej][: R - 1])
    assert np.array_equal(keys, whole[:, keep])
    keys2, _ = gpu.seed_streams(5, 12_345, 100, rejected=rej)
    assert np.array_equal(keys2, whole[:, keep[12_345:12_445]])


def test_seed_batches_large_ragged(gpu, port):
    # runs of >= 2^22 streams seed 128 slots per thread in batches of 32 (swizzled staging):
    # a ragged count, a shard offset and rejections in the first and last batches
    R = (1 << 22) + 1_000 + 17
    whole = port.random_spacing(9, R + 520)
    keys, _ = gpu.seed_streams(9, 0, R)
    assert np.array_equal(keys, whole[:, :R])
    rej = [3, 31, 32, 33, 127, 128, 4_096, R - 40, R - 1]
    keep = np.array([i for i in range(R + 520) if i not in set(rej)])
    keys, _ = gpu.seed_streams(9, 0, R, rejected=rej)
    assert np.array_equal(keys, whole[:, keep[:R]])
    keys, _ = gpu.seed_streams(9, 77, R - 500, rejected=rej)
    assert np.array_equal(keys, whole[:, keep[77:77 + R - 500]])


def test_walk_planes_from_batched_seeding(gpu, port):
    # the bitsliced walk pipeline reads the bit planes the 128-slot seeding writes, one
    # group per batch; a ragged last group (37 of 32 * k + 37 replications)
    p = gpu.ModelParams(replications=(1 << 22) + 37, steps=48, chunks=7)
    run = gpu.run_model(gpu.ModelKind.Walk, p, gpu.ExecutionMode.Wlp, master_seed=31337)
    want = port.run_model(2, oracle.params_from(p), 31337)
    assert np.array_equal(run.outputs["out"], want["out"]), \
        gpu.last_kernel()


def test_special_candidates_reported(gpu):
    # over many candidates some key component falls below twice its minimum
    keys, specials = gpu.seed_streams(11, 0, 3_000_000)
    s1, s2, s3 = keys.astype(np.int64)
    mask = (s1 < 4) | (s2 < 16) | (s3 < 32)
    assert sorted(s.index for s in specials) == np.nonzero(mask)[0].tolist()


# ---- per-replication outputs --------------------------------------------------------------


@pytest.mark.parametrize("case", golden("replications.json")["cases"],
                         ids=lambda c: f"m{c['model']}-s{c['seed']}-{c['params']}")
def test_run_model_golden_all_modes(gpu, case):
    kw = dict(case["params"])
    p = gpu.ModelParams(**kw)
    for mode in MODES:
        run = gpu.run_model(gpu.ModelKind(case["model"]), p, gpu.ExecutionMode[mode], master_seed=case["seed"])
        for name, want in case["outputs"].items():
            assert hexes(run.outputs[name]) == want, (mode, name)


@pytest.mark.parametrize("model", [0, 1, 2])
def test_medium_runs_vs_port(gpu, port, model):
    kw = {0: dict(replications=4099, draws=1000), 1: dict(replications=1500, clients=999, lambda_=0.6, mu=0.9),
          2: dict(replications=5003, steps=1000, chunks=30)}[model]
    p = gpu.ModelParams(**kw)
    want = port.run_model(model, oracle.params_from(p), 20260201)
    for mode in MODES:
        run = gpu.run_model(gpu.ModelKind(model), p, gpu.ExecutionMode[mode], master_seed=20260201)
        for name in oracle.OUTPUTS[model]:
            assert np.array_equal(run.outputs[name], want[name]), (mode, name)


@pytest.mark.parametrize("lam,mu", [(0.5, 1.0), (0.95, 1.0), (0.999, 1.0), (2.0, 1.0), (0.05, 1.0), (0.3, 0.7)])
@pytest.mark.parametrize("clients", [1, 7, 255, 256, 257, 511, 1234])
def test_mm1_wlp_segment_chaining_all_loads(gpu, port, lam, mu, clients):
    # WLP mm1 chains the Lindley recursion across 32 lane segments of a 256-client panel by
    # fixed-point rounds: light load (regenerates within a segment), heavy and overloaded
    # queues (the waiting time never returns to 0: up to 32 rounds), ragged last panels
    p = gpu.ModelParams(replications=97, clients=clients, lambda_=lam, mu=mu)
    want = port.run_model(1, oracle.params_from(p), 31337)
    run = gpu.run_model(gpu.ModelKind.Mm1, p, gpu.ExecutionMode.Wlp, master_seed=31337)
    for name in oracle.OUTPUTS[1]:
        assert np.array_equal(run.outputs[name], want[name]), name


@pytest.mark.parametrize("lam,mu", [(float.fromhex("0x1.fffffffffffffp-1"), float.fromhex("0x1.0000000000001p0")),
                                    (0.1, 1e-3), (1.3e-290, 1.7e-290), (0.3, 1e300), (2.0**-950, 2.0**-949),
                                    (3.0, 7.0)])
def test_mm1_rate_division_modes_all_mappings(gpu, port, lam, mu):
    # -log(1-u)/rate is a multiply for 2^k rates, a reciprocal + Markstein correction inside
    # [2^-900, 2^900] (tools/div_check.cu) and IEEE division outside: same bits either way
    p = gpu.ModelParams(replications=70, clients=300, lambda_=lam, mu=mu)
    want = port.run_model(1, oracle.params_from(p), 99)
    for mode in (gpu.ExecutionMode.Tlp, gpu.ExecutionMode.Wlp):
        for variant in (0, 1, 2):
            with gpu.wlp_variant(variant):
                run = gpu.run_model(gpu.ModelKind.Mm1, p, mode, master_seed=99)
            for name in oracle.OUTPUTS[1]:
                assert np.array_equal(run.outputs[name], want[name]), (mode, variant, name)


@pytest.mark.parametrize("R,steps", [(1, 1), (31, 15), (32, 16), (33, 17), (100, 1000), (4097, 333), (45, 70_000)])
def test_walk_bitsliced_tlp_matches_oracle(gpu, port, R, steps):
    # thread per 32 replications, state bits of 32 streams per word (bitslice.cuh): ragged
    # last group, step counts around the 16-step carry-save blocks, and a walk past 65520
    # steps (the int32 shared-memory flush)
    p = gpu.ModelParams(replications=R, steps=steps, chunks=7 + R % 23)
    want = port.run_model(2, oracle.params_from(p), 1234 + R)
    with gpu.tlp_variant(2):
        run = gpu.run_model(gpu.ModelKind.Walk, p, gpu.ExecutionMode.Tlp, master_seed=1234 + R)
    assert np.array_equal(run.outputs["out"], want["out"])


@pytest.mark.parametrize("variant", [3, 4], ids=["pipeline", "lane-chunks"])
@pytest.mark.parametrize("R,steps", [(1, 1), (33, 17), (64, 16), (100, 1000), (5000, 333), (70, 40_000),
                                     (40, 65_535), (3000, 511), (50, 100_000)])
def test_walk_bitsliced_wlp_matches_oracle(gpu, port, R, steps, variant):
    # 3: groups of 32 replications move lane to lane as bit planes, lane chunks of whole
    # 16-step blocks with the steps past a group's end masked out of the counts;
    # 4: a warp per group, every lane jumps the 32 streams to its chunk and the counts are
    # summed over lanes by a transpose-reduce (n = 100000: the pipeline's fallback)
    p = gpu.ModelParams(replications=R, steps=steps, chunks=3 + R % 29)
    want = port.run_model(2, oracle.params_from(p), 4321 + R)
    with gpu.wlp_variant(variant):
        run = gpu.run_model(gpu.ModelKind.Walk, p, gpu.ExecutionMode.Wlp, master_seed=4321 + R)
    assert np.array_equal(run.outputs["out"], want["out"])


@pytest.mark.parametrize("lanes", [4, 8, 16, 32])
@pytest.mark.parametrize("R,steps", [(2000, 1), (2048, 37), (5000, 1000), (70_000, 999), (3000, 5003), (2100, 16)])
def test_walk_bitsliced_pipeline_lanes_wrap_vs_oracle(gpu, port, R, steps, lanes):
    # S lanes per group of 32 replications (32/S pipelines per warp), rotating chunks not
    # tied to 16-step blocks, wrap groups (jumped seeds as planes at step 0, early and late
    # counters summed), the rotation feed; ragged last group
    p = gpu.ModelParams(replications=R, steps=steps, chunks=3 + R % 31)
    want = port.run_model(2, oracle.params_from(p), 99 + R)
    with gpu.wlp_variant(3), gpu.pipe_lanes(lanes):
        run = gpu.run_model(gpu.ModelKind.Walk, p, gpu.ExecutionMode.Wlp, master_seed=99 + R)
    assert gpu.last_kernel() == "k_wlp_walk_bs_pipe"
    assert np.array_equal(run.outputs["out"], want["out"])


def test_walk_wlp_auto_picks_the_bitsliced_pipeline_at_large_R(gpu, port):
    # R = 6e5: above the automatic threshold; the result is still the reference's
    p = gpu.ModelParams(replications=600_000, steps=100, chunks=30)
    want = port.run_model(2, oracle.params_from(p), 42)
    run = gpu.run_model(gpu.ModelKind.Walk, p, gpu.ExecutionMode.Wlp, master_seed=42)
    assert gpu.last_kernel() == "k_wlp_walk_bs_pipe"
    assert np.array_equal(run.outputs["out"], want["out"])
    small = gpu.ModelParams(replications=1000, steps=100, chunks=30)
    gpu.run_model(gpu.ModelKind.Walk, small, gpu.ExecutionMode.Wlp, master_seed=42)
    assert gpu.last_kernel() in ("k_wlp_lanes<walk>", "k_wlp_pipe<walk>")
    mid = gpu.ModelParams(replications=100_000, steps=1000, chunks=30)
    gpu.run_model(gpu.ModelKind.Walk, mid, gpu.ExecutionMode.Wlp, master_seed=42)
    assert gpu.last_kernel() == "k_wlp_walk_bs_lanes"
    gpu.run_model(gpu.ModelKind.Walk, small, gpu.ExecutionMode.Tlp, master_seed=42)
    assert gpu.last_kernel() == "k_tlp<walk>"


def test_run_streams_pi_mm1_walk_replication(gpu, port):
    keys = port.random_spacing(3, 50)
    st = gpu.RngState(*[int(x) for x in keys[:, 7]])
    seed = keys[:, 7:8]
    assert gpu.pi_replication(777, st) == port.replications(0, oracle.params(draws=777), seed)["out"][0]
    m = port.replications(1, oracle.params(clients=321, lambda_=0.25, mu=2.0), seed)
    assert gpu.mm1_replication(321, 0.25, 2.0, st) == (m["outIdle"][0], m["outWait"][0], m["outSys"][0])
    assert gpu.walk_replication(99, 4, st) == port.replications(2, oracle.params(steps=99, chunks=4), seed)["out"][0]


def test_statistical_pins(gpu):
    pins = golden("pins.json")
    r = gpu.run_model(gpu.ModelKind.Pi, P(gpu, replications=1, draws=1_000_000), gpu.ExecutionMode.Wlp,
                      master_seed=42)
    assert hexes(r.primary) == pins["pi_1x1e6"]["out"]
    for mode in ("Wlp", "Tlp"):
        r = gpu.run_model(gpu.ModelKind.Mm1, P(gpu, replications=30, clients=100_000), gpu.ExecutionMode[mode],
                          master_seed=42)
        for k in ("outIdle", "outWait", "outSys"):
            assert hexes(r.outputs[k]) == pins["mm1_30x1e5"][k]
    r = gpu.run_model(gpu.ModelKind.Walk, P(gpu, replications=3000, steps=1000, chunks=30), gpu.ExecutionMode.Wlp,
                      master_seed=42)
    assert hashlib.sha256(r.primary.astype("<f8").tobytes()).hexdigest() == pins["walk_3000x1000"]["sha256"]


def test_device_log_port_vs_glibc_fixture(gpu):
    g = golden("log_pairs.json")
    got = gpu.debug_neg_log1m(np.asarray(g["k"], dtype=np.uint32))
    assert hexes(got) == g["neg_log1m"]


def test_device_log_port_vs_host_libm_dense(gpu, port):
    # 2^24 evenly spread model inputs + the whole near-one window edge region
    k = np.concatenate([np.arange(0, 2**32, 256, dtype=np.uint64), np.arange(2**28 - 4096, 2**28 + 4096)])
    k = k.astype(np.uint32)
    got = gpu.debug_neg_log1m(k)
    if oracle.host_log_variant() != "fma":
        pytest.skip("this host's libm is not the FMA variant the fixtures were made with")
    want = port.exponential_from_u(k.astype(np.float64) * 2.0**-32, 1.0)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


# ---- statistics ---------------------------------------------------------------------------


def test_confidence_interval_golden(gpu):
    g = golden("stats.json")
    for c in g["ci"]:
        ci = gpu.confidence_interval(unhex(c["x"]), c["level"])
        assert ci.n == c["n"] and ci.warnSmallSample == c["warn"]
        if c["n"] <= 256:  # sequential device sum: bit-exact
            assert ci.mean.hex() == c["mean"] and ci.halfWidth.hex() == c["half_width"]
        else:
            assert ci.mean == pytest.approx(float.fromhex(c["mean"]), rel=1e-12)
            assert ci.halfWidth == pytest.approx(float.fromhex(c["half_width"]), rel=1e-12)
    with pytest.raises(gpu.DomainError):
        gpu.confidence_interval([1.0])
    with pytest.raises(gpu.DomainError):
        gpu.confidence_interval([1.0, 2.0], 1.0)


def test_device_ci_of_run_matches_reference(gpu, ref):
    for model, kw in [(0, dict(replications=100_000, draws=100)), (1, dict(replications=20_000, clients=200)),
                      (2, dict(replications=50_000, steps=200, chunks=30))]:
        p = gpu.ModelParams(**kw)
        outs = [np.empty(p.replications) for _ in oracle.OUTPUTS[model]]
        cis = gpu.run_model_into(gpu.ModelKind(model), p, gpu.ExecutionMode.Wlp, 42, outs, on_device=False,
                                 ci_level=0.95)
        for o, ci in zip(outs, cis):
            m, hw, n, warn = ref.confidence_interval(o, 0.95)
            assert ci.n == n and ci.mean == pytest.approx(m, rel=1e-12, abs=1e-300)
            assert ci.halfWidth == pytest.approx(hw, rel=1e-12)


def test_sweep_golden_means(gpu):
    # proj/tests/golden/sweep_pi.golden: seed 42, draws 100, R = 1, 2 — mean / CI columns
    rows = [r.split(",") for r in (GOLD / "sweep_pi.csv").read_text().splitlines()[1:]]
    for R, mode, _, *_, mean, lo, hi in rows:
        run = gpu.run_model(gpu.ModelKind.Pi, P(gpu, replications=int(R), draws=100), gpu.mode_from_name(mode),
                            master_seed=42)
        if int(R) == 1:
            assert repr(float(run.primary[0])) == mean
        else:
            ci = gpu.confidence_interval(run.primary)
            assert (repr(float(ci.mean)), repr(float(ci.low())), repr(float(ci.high()))) == (mean, lo, hi)


# ---- shards, errors, warnings ---------------------------------------------------------------


def test_shards_concatenate_to_whole_run(gpu):
    p = P(gpu, replications=10_007, clients=300)
    whole = gpu.run_model(gpu.ModelKind.Mm1, p, gpu.ExecutionMode.Wlp, master_seed=9)
    parts = {k: [] for k in ("outIdle", "outWait", "outSys")}
    for b, c in ((0, 3000), (3000, 5000), (8000, 2007)):
        outs = [np.empty(c) for _ in range(3)]
        sp = gpu.run_shard(gpu.ModelKind.Mm1, p, gpu.ExecutionMode.Tlp, 9, b, c, outs, on_device=False)
        assert isinstance(sp, list)
        for k, o in zip(parts, outs):
            parts[k].append(o)
    for k in parts:
        assert np.array_equal(np.concatenate(parts[k]), whole.outputs[k])


def test_errors_and_warnings(gpu):
    with pytest.raises(gpu.DomainError):
        gpu.run_model(gpu.ModelKind.Pi, P(gpu, replications=3, draws=0), gpu.ExecutionMode.Wlp)
    with pytest.raises(gpu.DomainError):
        gpu.run_model(gpu.ModelKind.Mm1, P(gpu, replications=3, mu=0.0), gpu.ExecutionMode.Tlp)
    with pytest.raises(gpu.PlanError):
        gpu.run_model(gpu.ModelKind.Walk, P(gpu, replications=3), gpu.ExecutionMode.Tlp, tlp_block_size=4096)
    # test_models.cpp:350-366
    run = gpu.run_model(gpu.ModelKind.Mm1, P(gpu, replications=50, clients=20, lambda_=1.0, mu=0.5),
                        gpu.ExecutionMode.Tlp, master_seed=1)
    assert "unstable" in run.warning and "warp" in run.warning
    run = gpu.run_model(gpu.ModelKind.Mm1, P(gpu, replications=64, clients=20), gpu.ExecutionMode.Tlp, master_seed=1)
    assert run.warning is None
    assert run.report.kernel_ms > 0 and run.report.totalCycles > 0


# ---- full-size properties (BASELINE configs 2-4) --------------------------------------------


def _device_run(gpu, model, p, mode, seed):
    import torch

    outs = [torch.empty(p.replications, dtype=torch.float64, device="cuda") for _ in oracle.OUTPUTS[model]]
    gpu.run_model_into(gpu.ModelKind(model), p, mode, seed, outs, on_device=True)
    torch.cuda.synchronize()
    return [o.cpu().numpy() for o in outs]


@pytest.mark.parametrize("model,kw", [(0, dict(replications=1_000_000, draws=10_000)),
                                      (2, dict(replications=100_000, steps=1000, chunks=30)),
                                      (0, dict(replications=10_000_000, draws=1000)),
                                      (1, dict(replications=10_000_000, clients=1000)),
                                      (2, dict(replications=10_000_000, steps=1000, chunks=30))],
                         ids=["cfg2-pi", "cfg3-walk", "cfg4-pi", "cfg4-mm1", "cfg4-walk"])
def test_full_size_wlp_equals_tlp_and_sampled_oracle(gpu, ref, model, kw):
    p = gpu.ModelParams(**kw)
    wlp = _device_run(gpu, model, p, gpu.ExecutionMode.Wlp, 42)
    tlp = _device_run(gpu, model, p, gpu.ExecutionMode.Tlp, 42)
    for a, b in zip(wlp, tlp):
        assert np.array_equal(a, b)
    # a random sample of replications re-computed by the reference on the host
    idx = np.sort(np.random.default_rng(0).choice(p.replications, 512, replace=False))
    keys = gpu.random_spacing_seed(42, p.replications)[:, idx]
    want = ref.replications(model, oracle.params_from(p), keys, nthreads=8)
    for a, name in zip(wlp, oracle.OUTPUTS[model]):
        assert np.array_equal(a[idx], want[name])
    # integer-valued outputs stay in range; pi mean near pi
    if model == 0:
        assert abs(wlp[0].mean() - np.pi) < 1e-3
    if model == 2:
        assert wlp[0].min() >= 0 and wlp[0].max() < kw["chunks"] and np.all(wlp[0] == np.floor(wlp[0]))


@pytest.mark.parametrize("variant", [1, 2])
@pytest.mark.parametrize("model,kw", [(0, dict(replications=5000, draws=1000)), (0, dict(replications=777, draws=31)),
                                      (0, dict(replications=3, draws=5000)), (0, dict(replications=2000, draws=1)),
                                      (2, dict(replications=4099, steps=1000, chunks=30)),
                                      (2, dict(replications=100, steps=33, chunks=7)),
                                      (2, dict(replications=1, steps=70, chunks=4)),
                                      (1, dict(replications=3000, clients=1000)),
                                      (1, dict(replications=500, clients=37, lambda_=0.9, mu=1.0)),
                                      (1, dict(replications=64, clients=5, lambda_=2.0, mu=1.0)),
                                      (1, dict(replications=2, clients=3000, lambda_=0.7, mu=0.75))])
def test_wlp_lane_jump_and_pipeline_kernels_agree_with_oracle(gpu, port, variant, model, kw):
    # the two WLP kernels of each model (pi / walk: lane jumps or warp pipeline; mm1:
    # segment chaining or warp pipeline) give the reference's bits
    p = gpu.ModelParams(**kw)
    want = port.run_model(model, oracle.params_from(p), 777)
    with gpu.wlp_variant(variant):
        run = gpu.run_model(gpu.ModelKind(model), p, gpu.ExecutionMode.Wlp, master_seed=777)
    for name in oracle.OUTPUTS[model]:
        assert np.array_equal(run.outputs[name], want[name]), name


@pytest.mark.parametrize("cap", [1, 4, 16, 32, 128])
@pytest.mark.parametrize("lanes", [8, 32])
def test_mm1_pipeline_near_list_overflow_redo(gpu, port, cap, lanes):
    # the single-pass mm1 pipeline lists a panel's near-one draws (~32 of 512) with a
    # shared-memory atomic; more than `cap` entries (never at the real cap of 128 with
    # random draws) redo the panel from the saved stream state: force it with small caps
    p = gpu.ModelParams(replications=3000, clients=1024, lambda_=0.5, mu=1.0)
    want = port.run_model(1, oracle.params_from(p), 555)
    with gpu.wlp_variant(2), gpu.pipe_lanes(lanes), gpu.near_cap(cap):
        run = gpu.run_model(gpu.ModelKind.Mm1, p, gpu.ExecutionMode.Wlp, master_seed=555)
    assert gpu.last_kernel() == "k_wlp_mm1_pipe"
    for name in oracle.OUTPUTS[1]:
        assert np.array_equal(run.outputs[name], want[name]), name


@pytest.mark.parametrize("lanes", [2, 4, 8, 16, 32])
@pytest.mark.parametrize("lam,mu,n", [(0.5, 1.0, 1000), (0.3, 0.9, 512), (0.9, 1.0, 2048), (1.7, 1.0, 64),
                                      (0.4, 0.4, 800), (0.1, 1e-3, 96)])
def test_mm1_pipeline_lanes_and_division_modes(gpu, port, lanes, lam, mu, n):
    # S = 8 / 16 / 32 lanes per replication, rotating whole-panel chunks, the interleaved
    # recursion, every division mode (mu = 1 services skip the division)
    p = gpu.ModelParams(replications=2500, clients=n, lambda_=lam, mu=mu)
    want = port.run_model(1, oracle.params_from(p), 8080 + n)
    with gpu.wlp_variant(2), gpu.pipe_lanes(lanes):
        run = gpu.run_model(gpu.ModelKind.Mm1, p, gpu.ExecutionMode.Wlp, master_seed=8080 + n)
    for name in oracle.OUTPUTS[1]:
        assert np.array_equal(run.outputs[name], want[name]), name


@pytest.mark.parametrize("model,kw", [(0, dict(replications=300_000, draws=100)),
                                      (1, dict(replications=200_000, clients=64)),
                                      (2, dict(replications=500_000, steps=100, chunks=9)),
                                      (2, dict(replications=50_000, steps=100, chunks=9)),
                                      (1, dict(replications=700, clients=300))])
@pytest.mark.parametrize("mode", [1, 2])
def test_host_outputs_pinned_mirrors_and_pageable_copies(gpu, port, model, kw, mode):
    # outputs into pinned host memory are stored there by the model kernel as they are
    # produced (no copy after the run); pageable host arrays keep the device buffer and the
    # copy. Both equal the reference, through run_model (wlp_run) and run_shard.
    import torch

    p = gpu.ModelParams(**kw)
    want = port.run_model(model, oracle.params_from(p), 404)
    names = oracle.OUTPUTS[model]
    pinned = [torch.zeros(p.replications, dtype=torch.float64, pin_memory=True) for _ in names]
    gpu.run_model_into(gpu.ModelKind(model), p, gpu.ExecutionMode(mode), 404, [t.numpy() for t in pinned],
                       on_device=False)
    pageable = [np.zeros(p.replications) for _ in names]
    gpu.run_model_into(gpu.ModelKind(model), p, gpu.ExecutionMode(mode), 404, pageable, on_device=False)
    shard = [torch.zeros(p.replications, dtype=torch.float64, pin_memory=True) for _ in names]
    gpu.run_shard(gpu.ModelKind(model), p, gpu.ExecutionMode(mode), 404, 0, p.replications,
                  [t.numpy() for t in shard], on_device=False)
    for k, name in enumerate(names):
        assert np.array_equal(pinned[k].numpy(), want[name]), ("pinned", name)
        assert np.array_equal(pageable[k], want[name]), ("pageable", name)
        assert np.array_equal(shard[k].numpy(), want[name]), ("shard", name)


@pytest.mark.parametrize("model", [0, 2])
@pytest.mark.parametrize("R,n", [(992, 1), (1000, 5), (2500, 257), (2500, 999), (3001, 1000), (1500, 10_000),
                                 (4000, 63), (993, 2049)])
@pytest.mark.parametrize("lanes", [32, 16, 8, 4, 2])
def test_wrapped_pipeline_rotating_chunks_vs_oracle(gpu, port, model, R, n, lanes):
    # the pi / walk warp pipeline with rotating chunk lengths (PipeSched: G-unit blocks, a
    # remainder of blocks spread over the phases, a sub-block tail at phase 31) and the wrap
    # (lanes 1..31 start kWrap replications per warp at their chunk by a lane-table jump,
    # whose early chunks then run in the drain): every replication bit-exact, including the
    # wrap ones, which sit at the front of the array (warp w owns [31w, 31w + 31)); with
    # 16 or 8 lanes per replication, 2 or 4 pipelines per warp, each with its own wrap set
    kw = dict(replications=R, draws=n) if model == 0 else dict(replications=R, steps=n, chunks=5 + R % 17)
    p = gpu.ModelParams(**kw)
    want = port.run_model(model, oracle.params_from(p), 2024 + R)
    with gpu.wlp_variant(2), gpu.pipe_lanes(lanes):
        run = gpu.run_model(gpu.ModelKind(model), p, gpu.ExecutionMode.Wlp, master_seed=2024 + R)
    assert gpu.last_kernel().startswith("k_wlp_pipe")
    for name in oracle.OUTPUTS[model]:
        assert np.array_equal(run.outputs[name], want[name]), name


@pytest.mark.parametrize("model,kw", [(0, dict(replications=10_000_000, draws=1000)),
                                      (2, dict(replications=10_000_000, steps=1000, chunks=30)),
                                      (1, dict(replications=2_000_000, clients=1000))])
def test_pipeline_full_size_equals_lane_jumps(gpu, model, kw):
    p = gpu.ModelParams(**kw)
    outs = {}
    for v in (1, 2):
        with gpu.wlp_variant(v):
            outs[v] = _device_run(gpu, model, p, gpu.ExecutionMode.Wlp, 42)
    for a, b in zip(outs[1], outs[2]):
        assert np.array_equal(a, b)


def test_walk_full_size_all_five_kernels_agree(gpu):
    # config 4 walk through the per-replication WLP pipeline, the bitsliced WLP pipeline and
    # lane chunks, the per-replication TLP and the bitsliced TLP: one array, bit for bit
    p = gpu.ModelParams(replications=10_000_000, steps=1000, chunks=30)
    runs = []
    for wv, tv, mode in ((2, 0, gpu.ExecutionMode.Wlp), (3, 0, gpu.ExecutionMode.Wlp), (4, 0, gpu.ExecutionMode.Wlp),
                         (0, 1, gpu.ExecutionMode.Tlp), (0, 2, gpu.ExecutionMode.Tlp)):
        with gpu.wlp_variant(wv), gpu.tlp_variant(tv):
            runs.append(_device_run(gpu, 2, p, mode, 42)[0])
    for r in runs[1:]:
        assert np.array_equal(r, runs[0])


def test_randomized_configurations_all_kernels_vs_oracle(gpu, port):
    # 150 random small configurations: every model, mode and WLP kernel variant, ragged
    # unit counts, rates that are / are not powers of two, light to overloaded queues
    rng = np.random.default_rng(20261017)
    for it in range(150):
        model = int(rng.integers(0, 3))
        R = int(rng.choice([1, 2, 31, 32, 33, 64, 65, 100, 257, 1000, 3000]))
        N = int(rng.choice([1, 2, 3, 7, 31, 32, 33, 63, 64, 65, 127, 128, 129, 255, 256, 257, 500, 1000, 2049]))
        lam = float(rng.choice([0.125, 0.25, 0.5, 0.3, 0.7, 0.9, 1.0, 1.7]))
        mu = float(rng.choice([0.5, 1.0, 2.0, 0.8, 1.3]))
        p = gpu.ModelParams(replications=R, draws=N, clients=N, steps=N, chunks=int(rng.integers(2, 40)),
                            lambda_=lam, mu=mu)
        seed = int(rng.integers(0, 2**63))
        want = port.run_model(model, oracle.params_from(p), seed)
        mode = gpu.ExecutionMode(int(rng.integers(0, 3)))
        variant = int(rng.integers(0, 5))
        with gpu.wlp_variant(variant), gpu.tlp_variant(min(variant, 2)):
            run = gpu.run_model(gpu.ModelKind(model), p, mode, master_seed=seed,
                                tlp_block_size=int(rng.choice([32, 50, 128, 256])))
        for name in oracle.OUTPUTS[model]:
            assert np.array_equal(run.outputs[name], want[name]), (it, model, R, N, lam, mu, mode, variant, name)
