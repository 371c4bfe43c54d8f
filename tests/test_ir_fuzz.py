"""Differential fuzzing of the kernel-IR path against the reference:
random programs (tests/ir_fuzz.py) through the reference simulator (simulate,
device.cpp:140-226, built into oracle/_ref) and through the B200 interpreter and JIT.

Host: the text form round-trips to the reference's canonical dump, and every program's
JIT source compiles for sm_100a. GPU: memory bit-identical and SimReport counters equal
to the reference's (interpreter), memory bit-identical (JIT), faults on both sides or on
neither."""
import numpy as np
import pytest

import oracle
import paper_1501_01405_b200 as w
from ir_fuzz import Gen
from paper_1501_01405_b200 import ir
from test_ir_host import _nvrtc_compile

KEYS = ("issues", "aluIssues", "memReads", "memWrites", "divergenceEvents")
N_INTERP = 2000
N_JIT = 160


def _ref_run(ref, c):
    arrays = {k: v.copy() for k, v in c["arrays"].items()}
    try:
        rep = ref.ir_simulate(c["text"], c["cfg"], c["scalars"], arrays, c["streams"])
    except oracle.OracleError as e:
        if "[3]" not in str(e):  # a fault; anything else is a broken test program
            raise
        return None, None
    return arrays, rep


def _ours(c, jit):
    arrays = {k: v.copy() for k, v in c["arrays"].items()}
    bx, by, bz, gx, gy, ws = c["cfg"]
    try:
        rep = ir.simulate(c["text"], w.LaunchConfig((bx, by, bz), (gx, gy), ws), c["scalars"], arrays, c["streams"],
                          jit=jit)
    except w.FaultError:
        return None, None
    return arrays, rep


def _hex(arrays):
    return {k: [float(x).hex() for x in v] for k, v in arrays.items()}


@pytest.mark.parametrize("block", range(4))
def test_fuzz_text_round_trips_to_the_reference_dump(ref, block):
    for s in range(block * 100, block * 100 + 100):
        text = Gen(s).case()["text"]
        assert ir.canonical(text) == ref.ir_canonical(text), s


def test_fuzz_jit_sources_compile_for_sm100a():
    for s in range(0, N_JIT, 4):
        assert _nvrtc_compile(ir.jit_source(Gen(s).case()["text"])) == "", s


@pytest.mark.gpu
@pytest.mark.parametrize("block", range(8))
def test_fuzz_interpreter_matches_reference_simulator(gpu, ref, block):
    faults = 0
    for s in range(block * N_INTERP // 8, (block + 1) * N_INTERP // 8):
        c = Gen(s).case()
        want, wrep = _ref_run(ref, c)
        got, grep_ = _ours(c, jit=False)
        assert (want is None) == (got is None), f"seed {s}: fault on one side only"
        if want is None:
            faults += 1
            continue
        assert _hex(got) == _hex(want), f"seed {s}"
        assert {k: getattr(grep_, k) for k in KEYS} == {k: wrep[k] for k in KEYS}, f"seed {s}"
    assert faults < N_INTERP // 8 // 2  # most programs run to the end


@pytest.mark.gpu
def test_fuzz_jit_matches_reference_simulator(gpu, ref):
    for s in range(N_JIT):
        c = Gen(s).case()
        want, _ = _ref_run(ref, c)
        got, _ = _ours(c, jit=True)
        assert (want is None) == (got is None), f"seed {s}: fault on one side only"
        if want is not None:
            assert _hex(got) == _hex(want), f"seed {s}"
