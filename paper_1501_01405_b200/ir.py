"""The reference's kernel IR on the B200: Python mirror of
include/warpsim_ir_b200.hpp over libwarpsim_b200.so (the C++ front end: parser, builder
rules, flattening) and libwlp_b200.so (wlp_ir_simulate: the SIMT interpreter kernel).

    text = model_text(ModelKind.Walk, ExecutionMode.Tlp)      # dump_kernel(wrap_tlp(...))
    rep = simulate(text, LaunchConfig((64, 1, 1), (2, 1), 32),
                   scalars={"replications": 100, "steps": 50, "chunks": 7},
                   arrays={"posX": np.zeros(100), "posY": np.zeros(100), "out": np.zeros(100)},
                   streams=keys)                              # device.hpp:91-93, on the GPU

Kernel text follows kernel_text.hpp (s-expressions, ';' comments). Arrays are updated in
place; the returned SimReport carries the reference simulator's exact issue / memory /
divergence counters and the measured kernel time.
"""
from __future__ import annotations

import ctypes as C
from typing import Mapping, Optional, Sequence

import numpy as np

from . import (OUTPUT_NAMES, PRIMARY, DomainError, Error, ExecutionMode, FaultError, LaunchConfig, ModelKind,
               ModelParams, ModelRun, ParseError, PlanError, RngState, SimOptions, SimReport, _Cfg, _params, _Params,
               _Report, _report, _PKG, plan_launch)

CXX_PATH = _PKG / "libwarpsim_b200.so"
_EXC = {1: DomainError, 2: PlanError, 3: FaultError, 6: ParseError}

_P = C.c_void_p
_SIGS = {
    "warpsim_ir_last_error": (C.c_char_p, []),
    "warpsim_ir_canonical": (C.c_int, [C.c_char_p, C.c_char_p, C.c_int, C.POINTER(C.c_int)]),
    "warpsim_ir_model_text": (C.c_int, [C.c_int, C.c_int, C.c_char_p, C.c_int, C.POINTER(C.c_int)]),
    "warpsim_ir_simulate_text": (C.c_int, [C.c_char_p, C.POINTER(_Cfg), C.c_int, C.c_int, _P, _P, _P, _P, C.c_int, _P,
                                           _P, _P, _P, C.c_int64, C.c_int, C.c_int64, C.c_int, C.POINTER(_Report)]),
    "warpsim_ir_run_model": (C.c_int, [C.c_int, C.POINTER(_Params), C.c_int, C.c_uint64, C.c_int, _P, _P, _P,
                                       C.POINTER(_Report), C.c_char_p, C.c_int, C.c_int]),
    "warpsim_ir_jit_source_text": (C.c_int, [C.c_char_p, C.c_char_p, C.c_int, C.POINTER(C.c_int)]),
}
_lib: Optional[C.CDLL] = None


def _cxx() -> C.CDLL:
    global _lib
    if _lib is None:
        if not CXX_PATH.exists():
            raise ImportError(f"{CXX_PATH.name} is not built; run `python -m paper_1501_01405_b200.build`")
        lib = C.CDLL(str(CXX_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def _check(status: int) -> None:
    if status:
        msg = (_cxx().warpsim_ir_last_error() or b"").decode(errors="replace")
        raise _EXC.get(status, Error)(msg)


def _text(fn, *args) -> str:
    need = C.c_int(0)
    _check(fn(*args, None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value)
    _check(fn(*args, buf, need.value, None))
    return buf.value.decode()


def canonical(text: str) -> str:
    """dump_kernel(parse_kernel(text)) (kernel_text.hpp); ParseError on malformed text."""
    return _text(_cxx().warpsim_ir_canonical, text.encode())


def model_text(model: ModelKind, mode: Optional[ExecutionMode] = None) -> str:
    """Text of build_model_body(model) (models.cpp:124-268), wrapped for Tlp / Wlp
    (wlp.cpp:107-138) when a mode is given."""
    m = 0 if mode is None or ExecutionMode(mode) == ExecutionMode.Sequential else int(mode)
    return _text(_cxx().warpsim_ir_model_text, int(model), m)


def _streams_soa(streams) -> np.ndarray:
    if streams is None:
        return np.zeros((3, 0), dtype=np.uint32)
    if isinstance(streams, np.ndarray):
        a = np.ascontiguousarray(streams, dtype=np.uint32)
        if a.ndim != 2 or a.shape[0] != 3:
            raise DomainError("streams must be a (3, n) uint32 array (SoA s1, s2, s3)")
        return a
    return np.ascontiguousarray(np.array([[s.s1 for s in streams], [s.s2 for s in streams],
                                          [s.s3 for s in streams]], dtype=np.uint32).reshape(3, -1))


def jit_source(text: str) -> str:
    """The CUDA C++ the IR JIT generates for a kernel text (compiled by NVRTC on use)."""
    return _text(_cxx().warpsim_ir_jit_source_text, text.encode())


def simulate(text: str, cfg: LaunchConfig, scalars: Mapping[str, object], arrays: Mapping[str, np.ndarray],
             streams=None, opts: Optional[SimOptions] = None, max_threads_per_block: int = 1024,
             jit: bool = False) -> SimReport:
    """simulate (device.cpp:140-226) of a kernel given as text, on the GPU interpreter
    (jit=True: compiled to sm_100a through NVRTC instead; same memory results, time only).
    `scalars`: name -> int (Int params) or float; `arrays`: name -> float64 numpy array,
    updated in place; `streams`: lane streams by global thread id ((3, n) uint32 or a
    sequence of RngState)."""
    opts = opts or SimOptions()
    names = list(scalars)
    is_int = (C.c_int * max(len(names), 1))(*[isinstance(scalars[k], (int, np.integer)) and
                                              not isinstance(scalars[k], bool) for k in names])
    ivals = (C.c_int64 * max(len(names), 1))(*[int(scalars[k]) if is_int[i] else 0 for i, k in enumerate(names)])
    rvals = (C.c_double * max(len(names), 1))(*[0.0 if is_int[i] else float(scalars[k]) for i, k in enumerate(names)])
    cnames = (C.c_char_p * max(len(names), 1))(*[k.encode() for k in names])
    anames = list(arrays)
    for k in anames:
        a = arrays[k]
        if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous):
            raise DomainError(f"array '{k}' must be a C-contiguous float64 numpy array")
    canames = (C.c_char_p * max(len(anames), 1))(*[k.encode() for k in anames])
    aptrs = (C.c_void_p * max(len(anames), 1))(*[arrays[k].ctypes.data for k in anames])
    alen = (C.c_int64 * max(len(anames), 1))(*[arrays[k].size for k in anames])
    st = _streams_soa(streams)
    bd, gd = tuple(cfg.blockDim), tuple(cfg.gridDim)
    c = _Cfg(int(bd[0]), int(bd[1]), int(bd[2]), int(gd[0]), int(gd[1]), int(cfg.warpSize))
    rep = _Report()
    _check(_cxx().warpsim_ir_simulate_text(text.encode(), C.byref(c), int(max_threads_per_block), len(names), cnames,
                                           is_int, ivals, rvals, len(anames), canames, aptrs, alen,
                                           st.ctypes.data if st.size else None, st.shape[1],
                                           int(opts.maskStackDepth), int(opts.maxIssuesPerWarp), int(bool(jit)),
                                           C.byref(rep)))
    return _report(rep)


def run_model(model: ModelKind, p: ModelParams, mode: ExecutionMode, master_seed: int = 1,
              tlp_block_size: int = 256, jit: bool = False) -> ModelRun:
    """run_model (models.cpp:329-397) through the reference's IR path, on the GPU
    interpreter (or compiled, jit=True): build_kernel -> random_spacing ->
    assign_lane_streams -> simulate."""
    model, mode = ModelKind(model), ExecutionMode(mode)
    names = OUTPUT_NAMES[model]
    R = int(p.replications)
    outs = [np.empty(R) for _ in names]
    o = [x.ctypes.data for x in outs] + [None] * (3 - len(outs))
    rep = _Report()
    warn = C.create_string_buffer(512)
    _check(_cxx().warpsim_ir_run_model(int(model), C.byref(_params(p)), int(mode), master_seed & (2**64 - 1),
                                       int(tlp_block_size), o[0], o[1], o[2], C.byref(rep), warn, 512,
                                       int(bool(jit))))
    outputs = dict(zip(names, outs))
    plan = plan_launch(R, mode, None, tlp_block_size)
    return ModelRun(outputs, outputs[PRIMARY[model]], _report(rep), plan.cfg, mode, warn.value.decode() or None)
