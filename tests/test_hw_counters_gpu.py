"""SimReport from hardware: instrumented kernels count divergence events
with the reference's definition and the global memory warp-instructions (paper Table 1).
The TLP divergence counts must equal the reference simulator's on the same streams: the
same replication->lane mapping meets the same data in every warp."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("model", [0, 1, 2])
@pytest.mark.parametrize("R,block", [(64, 256), (50, 256), (100, 50), (33, 32)])
def test_tlp_divergence_equals_reference_simulator(gpu, ref, model, R, block):
    kw = dict(replications=R, draws=60, clients=70, steps=80, chunks=7)
    p = gpu.ModelParams(**kw)
    want = ref.run_model_report(model, oracle.params(**kw), 42, 1, block)
    plain = gpu.run_model(gpu.ModelKind(model), p, gpu.ExecutionMode.Tlp, master_seed=42, tlp_block_size=block)
    with gpu.hw_counters():
        run = gpu.run_model(gpu.ModelKind(model), p, gpu.ExecutionMode.Tlp, master_seed=42, tlp_block_size=block)
    assert run.report.divergenceEvents == want["divergenceEvents"]
    if model != 0:
        assert run.report.divergenceEvents > 0
    # the instrumented kernel computes the same outputs
    for name in gpu.OUTPUT_NAMES[gpu.ModelKind(model)]:
        assert np.array_equal(run.outputs[name], plain.outputs[name])
    # TLP memory warp-instructions: 3 seed loads and one store per output per live warp
    block = min(R, block)  # plan_launch geometry (wlp.cpp:88-92)
    live_warps = sum(-(-min(block, R - b0) // 32) for b0 in range(0, R, block))
    n_out = 3 if model == 1 else 1
    staged = 0
    seed_warps = live_warps
    if model == 1:  # the log table staged per warp (256 doubles over `block` threads)
        nb = -(-R // block)
        for w in range(-(-block // 32)):
            first = 32 * w
            staged += nb * (-(-(256 - first) // block) if first < 256 else 0)
        seed_warps = nb * (-(-block // 32))  # predicated seed loads issue in every warp
    assert run.report.memReads == 3 * seed_warps + staged
    assert run.report.memWrites == n_out * live_warps


@pytest.mark.parametrize("model", [0, 1, 2])
def test_wlp_has_no_divergence(gpu, ref, model):
    kw = dict(replications=64, draws=200, clients=200, steps=200, chunks=7)
    with gpu.hw_counters():
        run = gpu.run_model(gpu.ModelKind(model), gpu.ModelParams(**kw), gpu.ExecutionMode.Wlp, master_seed=7)
    assert run.report.divergenceEvents == 0 == ref.run_model_report(model, oracle.params(**kw), 7, 2)["divergenceEvents"]
    assert run.report.memReads >= 3 * 64 and run.report.memWrites >= (3 if model == 1 else 1)
    # counters are per call and off again outside the context
    run2 = gpu.run_model(gpu.ModelKind(model), gpu.ModelParams(**kw), gpu.ExecutionMode.Wlp, master_seed=7)
    assert run2.report.memReads == 0 and run2.report.divergenceEvents == 0


def test_walk_table1_direction(gpu):
    # paper Table 1 / Fig. 7 direction: TLP diverges on the walk, WLP does not
    p = gpu.ModelParams(replications=64, steps=1000, chunks=30)
    with gpu.hw_counters():
        tlp = gpu.run_model(gpu.ModelKind.Walk, p, gpu.ExecutionMode.Tlp, master_seed=42)
        wlp = gpu.run_model(gpu.ModelKind.Walk, p, gpu.ExecutionMode.Wlp, master_seed=42)
    assert tlp.report.divergenceEvents > 1000 and wlp.report.divergenceEvents == 0


@pytest.mark.parametrize("model,expect", [(0, 128), (2, 128), (1, None)])
def test_wlp_warp_splits_measured(gpu, model, expect):
    # The WLP kernels run the model's ifs as arithmetic (divergenceEvents 0, as the
    # reference), but their own lane-divergent loops are counted: 200 units over 32 lanes
    # (K = 7) leave lanes 0-27 with 7, lane 28 with 4 and lanes 29-31 with none, so pi's
    # tail loop (7 / 4 / 0 trips) and the walk's 4-step loop (1 / 1 / 0) and tail (3 / 0 / 0)
    # split twice per replication; mm1 splits in its near-one log lists.
    kw = dict(replications=64, draws=200, clients=200, steps=200, chunks=7)
    with gpu.hw_counters():
        run = gpu.run_model(gpu.ModelKind(model), gpu.ModelParams(**kw), gpu.ExecutionMode.Wlp, master_seed=7)
    assert run.report.divergenceEvents == 0
    if expect is not None:
        assert run.report.warpSplits == expect
    else:
        assert run.report.warpSplits > 0


def test_tlp_warp_splits_include_model_events(gpu):
    p = gpu.ModelParams(replications=256, clients=300)
    with gpu.hw_counters():
        run = gpu.run_model(gpu.ModelKind.Mm1, p, gpu.ExecutionMode.Tlp, master_seed=3)
    assert run.report.divergenceEvents > 0
    assert run.report.warpSplits > run.report.divergenceEvents  # + the near-one list loops


@pytest.mark.parametrize("mode", ["wlp", "tlp"])
def test_total_cycles_from_clock64(gpu, mode):
    p = gpu.ModelParams(replications=20000, steps=2000, chunks=30)
    with gpu.hw_counters():
        run = gpu.run_model(gpu.ModelKind.Walk, p, gpu.mode_from_name(mode), master_seed=1)
    rep = run.report
    assert rep.kernel_ms > 0 and rep.totalCycles > 0
    # the makespan on one SM's clock fits inside the event-timed launch (<= ~2.1 GHz)
    assert rep.totalCycles <= rep.kernel_ms * 2.2e6
    assert rep.totalCycles >= rep.kernel_ms * 0.3e6
