"""Kernel IR front end without a GPU: the model kernels' text, the
s-expression parser / printer and its errors, against the reference (kernel_text.cpp,
models.cpp:124-268, wlp.cpp:107-138) and its committed dumps (tests/golden/ir)."""
import pytest

import paper_1501_01405_b200 as w
from conftest import GOLD
from ir_corpus import CASES, FAULTS
from paper_1501_01405_b200 import ir

NAMES = {0: "pi", 1: "mm1", 2: "walk"}


@pytest.mark.parametrize("model", [0, 1, 2])
@pytest.mark.parametrize("mode,tag", [(None, "body"), (w.ExecutionMode.Tlp, "tlp"), (w.ExecutionMode.Wlp, "wlp")])
def test_model_kernels_print_as_the_reference(model, mode, tag):
    want = (GOLD / "ir" / f"{NAMES[model]}_{tag}.sexp").read_text()  # dump_kernel of the reference's programs
    assert ir.model_text(w.ModelKind(model), mode) == want


@pytest.mark.parametrize("name", sorted(CASES) + sorted(FAULTS))
def test_canonical_text_is_a_fixpoint_and_matches_reference(ref, name):
    text = CASES[name]["text"] if name in CASES else FAULTS[name][0]
    once = ir.canonical(text)
    assert ir.canonical(once) == once
    assert once == ref.ir_canonical(text)


def test_literals_comments_and_registers():
    t = ir.canonical("""; header comment
    (kernel (param o array) (local a real) (local k int)
      (body
        (assign a 1e5)   ; real: exponent
        (assign a -0.0)
        (assign a 3.)
        (assign k -7)
        (store o 0 (add warpsize (mul bdim.z gdim.y)))))""")
    assert "(assign a 1e+05)" in t and "(assign a -0.0)" in t and "(assign a 3.0)" in t
    assert "(assign k -7)" in t and "(add warpsize (mul bdim.z gdim.y))" in t


BAD = [
    "", "(kernel", "(kernel))", "(kernel (body (assign x 1)))", "(kernel (param x int) (param x real) (body))",
    "(kernel (local tid.x int) (body))", "(kernel (param a array) (body (assign a 1)))",
    "(kernel (param a array) (local x real) (body (assign x a)))", "(kernel (local x int) (body (assign x (pow 2 3))))",
    "(kernel (local x int) (body (assign x (add 1))))", "(kernel (local x int) (body (frob x)))",
    "(kernel (local x int) (body (if x (else (halt)))))", "(kernel (local x int) (body (halt 1)))",
    "(kernel (local x int) (param p array) (body (load x p 0)))", "(kernel (local x int) (body) (body))",
    "(kernel (local x float) (body))", "(kernel (param x vector) (body))", "(foo)", "(kernel) (kernel)",
    "(kernel (local x int) (body (assign x (draw 1))))",
]


@pytest.mark.parametrize("text", BAD)
def test_malformed_text_is_a_parse_error_in_both(ref, text):
    with pytest.raises(w.ParseError):
        ir.canonical(text)
    with pytest.raises(Exception):
        ref.ir_canonical(text)


def test_parse_error_carries_a_line_reference():
    with pytest.raises(w.ParseError, match=r"line 3"):
        ir.canonical("(kernel (local x int)\n (body\n  (assign y 1)))")


def _nvrtc_compile(src: str) -> str:
    """Compile a JIT source for sm_100a with NVRTC (no GPU needed); returns '' or the log."""
    import ctypes as C

    from conftest import ROOT

    lib = C.CDLL("libnvrtc.so.12")
    csrc = ROOT / "paper_1501_01405_b200" / "csrc"
    names = ["taus88.cuh", "glibc_log.cuh", "glibc_log_data.h", "stdint.h"]
    texts = [(csrc / n).read_text() for n in names[:3]] + [
        "#pragma once\ntypedef unsigned int uint32_t; typedef int int32_t; typedef unsigned long long uint64_t;\n"
        "typedef long long int64_t;\n"]
    prog = C.c_void_p()
    arr = C.c_char_p * 4
    assert lib.nvrtcCreateProgram(C.byref(prog), src.encode(), b"k.cu", 4, arr(*[t.encode() for t in texts]),
                                  arr(*[n.encode() for n in names])) == 0
    opts = (C.c_char_p * 4)(b"--gpu-architecture=sm_100a", b"--fmad=false", b"--std=c++17", b"-default-device")
    rc = lib.nvrtcCompileProgram(prog, 4, opts)
    size = C.c_size_t()
    lib.nvrtcGetProgramLogSize(prog, C.byref(size))
    log = C.create_string_buffer(size.value)
    lib.nvrtcGetProgramLog(prog, log)
    lib.nvrtcDestroyProgram(C.byref(prog))
    return "" if rc == 0 else log.value.decode()


@pytest.mark.parametrize("which", ["models"] + sorted(CASES))
def test_jit_sources_compile_for_sm100a(which):
    # the IR JIT's generated CUDA C++ compiles with NVRTC (the compiler the library dlopens)
    texts = ([ir.model_text(w.ModelKind(m), w.ExecutionMode(md)) for m in range(3) for md in (1, 2)]
             if which == "models" else [CASES[which]["text"]])
    for t in texts:
        src = ir.jit_source(t)
        assert "extern \"C\" __global__" in src
        assert _nvrtc_compile(src) == ""


def test_c_abi_rejects_malformed_flattened_programs():
    # wlp_ir_simulate / wlp_ir_jit_source check every index and every expression of a
    # flattened program on the host before anything reaches a device (include/wlp_b200.h)
    import ctypes as C

    lib = w.native_library()

    class Stmt(C.Structure):
        _fields_ = [(n, C.c_int32) for n in ("kind", "slot", "arr", "code_a", "code_b", "b1_begin", "b1_end",
                                              "b2_begin", "b2_end", "flags")]

    class Prog(C.Structure):
        _fields_ = [("stmts", C.POINTER(Stmt)), ("n_stmts", C.c_int32), ("top_begin", C.c_int32),
                    ("top_end", C.c_int32), ("code", C.POINTER(C.c_int32)), ("n_code", C.c_int32),
                    ("n_locals", C.c_int32), ("local_init", C.POINTER(C.c_int64)), ("n_params", C.c_int32),
                    ("param_bits", C.POINTER(C.c_int64)), ("param_is_array", C.POINTER(C.c_int32))]

    def prog(stmts, code, n_locals=1, top=None):
        S = (Stmt * max(len(stmts), 1))(*[Stmt(*s) for s in stmts])
        K = (C.c_int32 * len(code))(*code)
        L = (C.c_int64 * max(n_locals, 1))()
        P = (C.c_int64 * 1)()
        A = (C.c_int32 * 1)(0)
        t = top or (0, len(stmts))
        return Prog(S, len(stmts), t[0], t[1], K, len(code), n_locals, L, 1, P, A), (S, K, L, P, A)

    OP_CONST, OP_LOCAL, OP_END, OP_ADD_I = 1, 2, 0, 10
    good = ([(0, 0, -1, 0, -1, 0, 0, 0, 0, 0)], [OP_CONST, 5, 0, OP_END])
    bad = [
        ([(0, 3, -1, 0, -1, 0, 0, 0, 0, 0)], [OP_CONST, 5, 0, OP_END]),          # local slot out of range
        ([(0, 0, -1, 9, -1, 0, 0, 0, 0, 0)], [OP_CONST, 5, 0, OP_END]),          # code offset out of range
        ([(0, 0, -1, 1, -1, 0, 0, 0, 0, 0)], [OP_CONST, 5, 0, OP_END]),          # offset inside an expression
        ([(0, 0, -1, 0, -1, 0, 0, 0, 0, 0)], [OP_ADD_I, OP_END]),                 # stack underflow
        ([(0, 0, -1, 0, -1, 0, 0, 0, 0, 0)], [OP_CONST, 5, 0, OP_CONST, 1, 0, OP_END]),  # two values left
        ([(0, 0, -1, 0, -1, 0, 0, 0, 0, 0)], [OP_LOCAL, 7, OP_END]),              # bad local in code
        ([(0, 0, -1, 0, -1, 0, 0, 0, 0, 0)], [99, OP_END]),                       # unknown opcode
        ([(0, 0, -1, 0, -1, 0, 0, 0, 0, 0)], [OP_CONST, 5]),                      # unterminated
        ([(3, -1, -1, 0, -1, 0, 5, 0, 0, 0)], [OP_CONST, 1, 0, OP_END]),          # body range past the end
        ([(2, 0, -1, 0, 0, 0, 0, 0, 0, 0)], [OP_CONST, 1, 0, OP_END]),            # store to a scalar param
        ([(7, 0, -1, 0, -1, 0, 0, 0, 0, 0)], [OP_CONST, 1, 0, OP_END]),           # unknown statement kind
        ([(4, -1, -1, 0, -1, 0, 1, 0, 0, 0)], [OP_CONST, 1, 0, OP_END]),          # WHILE whose body holds itself
        ([(3, -1, -1, 0, -1, 1, 2, 1, 2, 0), (5, -1, -1, -1, -1, 0, 0, 0, 0, 0)],  # then and else overlap
         [OP_CONST, 1, 0, OP_END]),
        ([(3, -1, -1, 0, -1, 1, 2, 0, 0, 0), (4, -1, -1, 0, -1, 0, 1, 0, 0, 0)],  # IF -> WHILE -> IF cycle
         [OP_CONST, 1, 0, OP_END]),
    ]
    need = C.c_int(0)
    p, keep = prog(*good)
    assert lib.wlp_ir_jit_source(C.byref(p), None, 0, C.byref(need)) == 0 and need.value > 100
    for stmts, code in bad:
        p, keep = prog(stmts, code)
        assert lib.wlp_ir_jit_source(C.byref(p), None, 0, C.byref(need)) == w.EDOMAIN, (stmts, code)
        cfg = w._Cfg(32, 1, 1, 1, 1, 32)
        rc = lib.wlp_ir_simulate(C.byref(p), C.byref(cfg), 1024, None, None, 0, None, 0, 0, 32, 1000, None, None)
        assert rc == w.EDOMAIN, (stmts, code)
