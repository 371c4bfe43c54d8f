"""The reference's kernel IR executed by the B200 SIMT interpreter:
memory contents and the SimReport counters must equal the reference simulator's
(simulate, device.cpp:140-226) — fixtures tests/golden/ir/*.json made by the reference
(tools/gen_ir_golden.py) — and run_model through the IR path must reproduce the engine's
bit-exact outputs."""
import json

import numpy as np
import pytest

import oracle
import paper_1501_01405_b200 as w
from conftest import GOLD
from ir_corpus import CASES, FAULTS, fresh_arrays, streams_for
from paper_1501_01405_b200 import ir

pytestmark = pytest.mark.gpu

KEYS = ("issues", "aluIssues", "memReads", "memWrites", "divergenceEvents")
CORPUS = json.loads((GOLD / "ir" / "corpus.json").read_text())
MODELS = json.loads((GOLD / "ir" / "models.json").read_text())


def cfg_of(c):
    bx, by, bz, gx, gy, ws = c
    return w.LaunchConfig((bx, by, bz), (gx, gy), ws)


@pytest.mark.parametrize("name", sorted(CASES))
def test_corpus_matches_reference_simulator(gpu, name):
    c = CASES[name]
    arrays = fresh_arrays(c)
    rep = ir.simulate(c["text"], cfg_of(c["cfg"]), c["scalars"], arrays, streams_for(c),
                      w.SimOptions(maskStackDepth=c["mask_depth"]))
    want = CORPUS["cases"][name]
    for k, v in arrays.items():
        assert [float(x).hex() for x in v] == want["arrays"][k], k
    assert {k: getattr(rep, k) for k in KEYS} == want["report"]
    assert rep.kernel_ms > 0


@pytest.mark.parametrize("name", sorted(FAULTS))
def test_faults_raise_fault_error_with_the_reference_message(gpu, name):
    text, _ = FAULTS[name]
    depth = 3 if name == "mask_stack" else 32
    with pytest.raises(w.FaultError) as e:
        ir.simulate(text, w.LaunchConfig((32, 1, 1), (1, 1), 32), {}, {"o": np.zeros(4)}, None,
                    w.SimOptions(maskStackDepth=depth))
    assert str(e.value) == CORPUS["faults"][name]["message"]


def test_issue_budget_stops_a_kernel_that_never_ends(gpu):
    text = "(kernel (local x int) (body (while (ge x 0) (assign x (add x 1)))))"
    with pytest.raises(w.FaultError, match="issue budget"):
        ir.simulate(text, w.LaunchConfig((64, 1, 1), (4, 1), 32), {}, {}, None, w.SimOptions(maxIssuesPerWarp=5000))


def test_launch_and_binding_errors(gpu):
    text = "(kernel (param n int) (param o array) (body (store o 0 n)))"
    L = w.LaunchConfig((32, 1, 1), (1, 1), 32)
    with pytest.raises(w.DomainError):  # unbound scalar
        ir.simulate(text, L, {}, {"o": np.zeros(1)})
    with pytest.raises(w.DomainError):  # int param given a real
        ir.simulate(text, L, {"n": 1.5}, {"o": np.zeros(1)})
    with pytest.raises(w.DomainError):  # unbound array
        ir.simulate(text, L, {"n": 1}, {})
    with pytest.raises(w.PlanError):  # maxThreadsPerBlock
        ir.simulate(text, w.LaunchConfig((64, 1, 1), (1, 1), 32), {"n": 1}, {"o": np.zeros(1)},
                    max_threads_per_block=32)
    with pytest.raises(w.DomainError):  # warpSize > 32: one IR warp per hardware warp
        ir.simulate(text, w.LaunchConfig((64, 1, 1), (1, 1), 64), {"n": 1}, {"o": np.zeros(1)})
    o = np.zeros(1)
    ir.simulate(text, L, {"n": 7}, {"o": o})
    assert o[0] == 7.0


@pytest.mark.parametrize("run", MODELS, ids=lambda r: f"m{r['model']}-mode{r['mode']}-R{r['params']['replications']}"
                         f"-b{r['tlp_block']}")
def test_run_model_through_ir_matches_engine_and_reference_counters(gpu, port, run):
    p = w.ModelParams(**run["params"])
    mode = w.ExecutionMode(run["mode"])
    got = w.run_model(w.ModelKind(run["model"]), p, mode, master_seed=run["seed"], tlp_block_size=run["tlp_block"],
                      opts=w.SimOptions(irInterpreter=True))
    want = port.run_model(run["model"], oracle.params_from(p), run["seed"])
    for name in oracle.OUTPUTS[run["model"]]:
        assert np.array_equal(got.outputs[name], want[name]), name
    assert {k: getattr(got.report, k) for k in KEYS} == run["report"]


def test_walk_tlp_divergence_matches_hand_written_kernel_counters(gpu, ref):
    # the IR walk (reference body) and the hand-written TLP walk count the same
    # divergence events: same lanes, same draws, same branch structure
    p = w.ModelParams(replications=256, steps=300, chunks=30)
    via_ir = w.run_model(w.ModelKind.Walk, p, w.ExecutionMode.Tlp, master_seed=3, opts=w.SimOptions(irInterpreter=True))
    with w.hw_counters():
        hand = w.run_model(w.ModelKind.Walk, p, w.ExecutionMode.Tlp, master_seed=3)
    assert np.array_equal(via_ir.primary, hand.primary)
    assert via_ir.report.divergenceEvents == hand.report.divergenceEvents > 0
    assert via_ir.report.divergenceEvents == ref.run_model_report(2, oracle.params_from(p), 3, 1)["divergenceEvents"]


def test_user_defined_kernel_runs_a_model_without_recompiling(gpu, port):
    # the user-style pi kernel of the corpus equals pi_replication on the same streams
    c = CASES["user_pi_tlp_counts_in_registers"]
    keys = port.random_spacing(99, 150)
    out = np.zeros(150)
    ir.simulate(c["text"], cfg_of(c["cfg"]), {"replications": 150, "draws": 200}, {"out": out}, keys)
    want = port.replications(0, oracle.params(draws=200), keys)["out"]
    assert np.array_equal(out, want)


# ---- the same kernels compiled (IR -> CUDA C++ -> NVRTC -> sm_100a) ---------------------------


@pytest.mark.parametrize("name", sorted(CASES))
def test_jit_corpus_memory_matches_reference_simulator(gpu, name):
    c = CASES[name]
    arrays = fresh_arrays(c)
    rep = ir.simulate(c["text"], cfg_of(c["cfg"]), c["scalars"], arrays, streams_for(c), jit=True)
    want = CORPUS["cases"][name]
    for k, v in arrays.items():
        assert [float(x).hex() for x in v] == want["arrays"][k], k
    assert rep.kernel_ms > 0 and rep.issues == 0  # no lockstep accounting when compiled


@pytest.mark.parametrize("name", sorted(set(FAULTS) - {"mask_stack"}))  # no mask stack when compiled
def test_jit_faults_raise_fault_error(gpu, name):
    text, _ = FAULTS[name]
    with pytest.raises(w.FaultError) as e:
        ir.simulate(text, w.LaunchConfig((32, 1, 1), (1, 1), 32), {}, {"o": np.zeros(4)}, None, jit=True)
    want = CORPUS["faults"][name]["message"]
    assert str(e.value).split(":")[0] == want.split(":")[0]


def test_jit_loop_guard_stops_a_kernel_that_never_ends(gpu):
    text = "(kernel (local x int) (body (while (ge x 0) (assign x (add x 1)))))"
    with pytest.raises(w.FaultError, match="issue budget"):
        ir.simulate(text, w.LaunchConfig((64, 1, 1), (4, 1), 32), {}, {}, None, w.SimOptions(maxIssuesPerWarp=5000),
                    jit=True)


@pytest.mark.parametrize("model", [0, 1, 2])
@pytest.mark.parametrize("mode", [w.ExecutionMode.Tlp, w.ExecutionMode.Wlp])
def test_jit_run_model_equals_engine(gpu, port, model, mode):
    p = w.ModelParams(replications=300, draws=200, clients=150, steps=170, chunks=9, lambda_=0.8, mu=1.1)
    run = w.run_model(w.ModelKind(model), p, mode, master_seed=5, opts=w.SimOptions(irInterpreter=True, irJit=True))
    want = port.run_model(model, oracle.params_from(p), 5)
    for name in oracle.OUTPUTS[model]:
        assert np.array_equal(run.outputs[name], want[name]), name


@pytest.mark.parametrize("model", [0, 1, 2])
def test_sequential_report_is_the_reference_unit_cost_accounting(gpu, ref, model):
    # models.cpp:377-389: Sequential charges R x the issues of ONE body execution (rid 0,
    # stream 0, one thread of warpSize 1); the IR path reproduces those numbers exactly
    kw = dict(replications=23, draws=70, clients=60, steps=50, chunks=7)
    p = w.ModelParams(**kw)
    run = w.run_model(w.ModelKind(model), p, w.ExecutionMode.Sequential, master_seed=11,
                      opts=w.SimOptions(irInterpreter=True))
    want = ref.run_model_report(model, oracle.params(**kw), 11, 0)
    for k in ("totalCycles", "issues", "aluIssues", "memReads", "memWrites", "divergenceEvents", "peakResidentWarps"):
        assert getattr(run.report, k) == want[k], k
    plain = w.run_model(w.ModelKind(model), p, w.ExecutionMode.Sequential, master_seed=11)
    for name in oracle.OUTPUTS[model]:
        assert np.array_equal(run.outputs[name], plain.outputs[name])


@pytest.mark.parametrize("jit", [False, True])
def test_readme_user_model_example(gpu, port, jit):
    text = """(kernel (param n int) (param draws int) (param out array)
  (local r int) (local i int) (local x real) (local c real)
  (body (assign r (add tid.x (mul bdim.x bid.x)))
        (if (lt r n) (then
          (while (lt i draws) (assign x (draw)) (assign c (add c (lt x 0.25))) (assign i (add i 1)))
          (store out r (div c draws))))))"""
    out = np.zeros(1000)
    keys = w.random_spacing_seed(7, 1000)
    ir.simulate(text, w.LaunchConfig((256, 1, 1), (4, 1), 32), {"n": 1000, "draws": 500}, {"out": out}, keys, jit=jit)
    want = [np.count_nonzero(port.taus_stream(*map(int, keys[:, r]), 500) < 2**30) / 500 for r in range(1000)]
    assert np.array_equal(out, np.array(want))
