"""B200-native Multiple-Replications-in-Parallel engine (Warp-Level Parallelism, arXiv 1501.01405).

Python mirror of the reference's replication-runner API (proj/include/warpsim/models.hpp,
rng.hpp, wlp.hpp, error.hpp) over the C ABI of ``libwlp_b200.so`` (include/wlp_b200.h).
Names, argument meaning and error types follow the reference:

    run_model(ModelKind.Pi, ModelParams(replications=32, draws=100), ExecutionMode.Wlp,
              DeviceProfile(), master_seed=42)                          # models.hpp:173-175
    confidence_interval(run.primary)                                    # models.hpp:132

Every model computation runs in the sm_100a kernels; there is no CPU path. Importing
works without a GPU (host utilities such as plan_launch / validate_params run on the
host, as in the reference); compute calls raise ``Error`` when no device is usable, and
importing raises if the native library has not been built (``build.build_all()``).
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from pathlib import Path
from typing import Optional, Sequence

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libwlp_b200.so"

# ---- errors (error.hpp:8-36) ------------------------------------------------------------


class Error(RuntimeError):
    """warpsim::Error"""


class DomainError(Error):
    """Invalid arguments (warpsim::DomainError)."""


class PlanError(Error):
    """Launch planning failure (warpsim::PlanError)."""


class FaultError(Error):
    """A lane hit a runtime fault (warpsim::FaultError)."""


class ParseError(Error):
    """warpsim::ParseError"""


class AnalysisError(Error):
    """warpsim::AnalysisError"""


OK, EDOMAIN, EPLAN, EFAULT, ESPACING, ECUDA, EPARSE, EINTERNAL = 0, 1, 2, 3, 4, 5, 6, 7
_EXC = {EDOMAIN: DomainError, EPLAN: PlanError, EFAULT: FaultError, ESPACING: Error, ECUDA: Error,
        EPARSE: ParseError, EINTERNAL: Error}

# ---- enums and records --------------------------------------------------------------------


class ModelKind(enum.IntEnum):  # models.hpp:18
    Pi = 0
    Mm1 = 1
    Walk = 2


class ExecutionMode(enum.IntEnum):  # wlp.hpp:16
    Sequential = 0
    Tlp = 1
    Wlp = 2


_MODEL_NAMES = {ModelKind.Pi: "pi", ModelKind.Mm1: "mm1", ModelKind.Walk: "walk"}
_MODE_NAMES = {ExecutionMode.Sequential: "sequential", ExecutionMode.Tlp: "tlp", ExecutionMode.Wlp: "wlp"}
OUTPUT_NAMES = {ModelKind.Pi: ("out",), ModelKind.Mm1: ("outIdle", "outWait", "outSys"), ModelKind.Walk: ("out",)}
PRIMARY = {ModelKind.Pi: "out", ModelKind.Mm1: "outWait", ModelKind.Walk: "out"}  # models.cpp:304-324


def model_name(m: ModelKind) -> str:
    return _MODEL_NAMES[ModelKind(m)]


def model_from_name(name: str) -> ModelKind:
    for k, v in _MODEL_NAMES.items():
        if v == name:
            return k
    raise DomainError(f"unknown model '{name}' (pi|mm1|walk)")


def mode_name(m: ExecutionMode) -> str:
    return _MODE_NAMES[ExecutionMode(m)]


def mode_from_name(name: str) -> ExecutionMode:
    for k, v in _MODE_NAMES.items():
        if v == name:
            return k
    raise DomainError(f"unknown execution mode '{name}' (sequential|tlp|wlp)")


@dataclass
class ModelParams:  # models.hpp:23-31 (`lambda` is spelled lambda_ in Python)
    replications: int = 1
    draws: int = 1000
    clients: int = 1000
    lambda_: float = 0.5
    mu: float = 1.0
    steps: int = 1000
    chunks: int = 30

    def units(self, model: ModelKind) -> int:
        return {ModelKind.Pi: self.draws, ModelKind.Mm1: self.clients, ModelKind.Walk: self.steps}[ModelKind(model)]


@dataclass
class RngState:  # rng.hpp:11-17
    s1: int = 2
    s2: int = 8
    s3: int = 16


@dataclass
class DeviceProfile:  # device.hpp:19-28 — accepted for signature compatibility, ignored
    numSMs: int = 14
    warpSchedulersPerSM: int = 2
    maxResidentBlocksPerSM: int = 8
    maxResidentWarpsPerSM: int = 48
    deviceResidentBlockCap: int = 64
    aluIssueCycles: int = 1
    memLatencyCycles: int = 400
    maxThreadsPerBlock: int = 1024


@dataclass
class SimOptions:  # device.hpp:53-60
    smPermutationSeed: Optional[int] = None  # accepted, ignored (real hardware)
    maskStackDepth: int = 32  # IR interpreter mask-stack bound
    # B200 extensions: run Tlp / Wlp through the reference's IR kernels on the GPU IR
    # interpreter (paper_1501_01405_b200.ir), and its per-IR-warp issue guard
    irInterpreter: bool = False
    maxIssuesPerWarp: int = 1 << 50
    irJit: bool = False  # with irInterpreter: compile the IR kernel (NVRTC) instead
    # B200 extension: shard run_model over GPUs 0..devices-1 of this process (wlp_run_devices)
    devices: int = 1


@dataclass
class SimReport:  # device.hpp:62-71; measured on the GPU (see wlp_report in wlp_b200.h)
    totalCycles: int = 0
    wavesExecuted: int = 0
    peakResidentWarps: int = 0
    issues: int = 0
    aluIssues: int = 0
    memReads: int = 0
    memWrites: int = 0
    divergenceEvents: int = 0
    kernel_ms: float = 0.0
    warpSplits: int = 0  # instrumented runs: every warp split of the kernel (wlp_report.warp_splits)


@dataclass
class LaunchConfig:  # kernel_ir.hpp:35-45
    blockDim: tuple = (1, 1, 1)
    gridDim: tuple = (1, 1)
    warpSize: int = 32


@dataclass
class LaunchPlan:  # wlp.hpp:38-43
    cfg: LaunchConfig
    replications: int
    mode: ExecutionMode
    warning: Optional[str]


@dataclass
class ModelRun:  # models.hpp:160-167
    outputs: dict
    primary: np.ndarray
    report: SimReport
    cfg: LaunchConfig
    mode: ExecutionMode
    warning: Optional[str]


@dataclass
class ConfidenceInterval:  # models.hpp:118-127
    mean: float = 0.0
    halfWidth: float = 0.0
    level: float = 0.95
    n: int = 0
    warnSmallSample: bool = False

    def low(self) -> float:
        return self.mean - self.halfWidth

    def high(self) -> float:
        return self.mean + self.halfWidth


# ---- C ABI --------------------------------------------------------------------------------


class _Params(C.Structure):
    _fields_ = [("replications", C.c_int64), ("draws", C.c_int64), ("clients", C.c_int64),
                ("lambda_", C.c_double), ("mu", C.c_double), ("steps", C.c_int64), ("chunks", C.c_int64)]


class _Cfg(C.Structure):
    _fields_ = [("block_x", C.c_int64), ("block_y", C.c_int64), ("block_z", C.c_int64),
                ("grid_x", C.c_int64), ("grid_y", C.c_int64), ("warp_size", C.c_int32)]


class _Report(C.Structure):
    _fields_ = [("total_cycles", C.c_int64), ("waves_executed", C.c_int64), ("peak_resident_warps", C.c_int64),
                ("issues", C.c_uint64), ("alu_issues", C.c_uint64), ("mem_reads", C.c_uint64),
                ("mem_writes", C.c_uint64), ("divergence_events", C.c_uint64), ("kernel_ms", C.c_double),
                ("warp_splits", C.c_uint64)]


class _CI(C.Structure):
    _fields_ = [("mean", C.c_double), ("half_width", C.c_double), ("level", C.c_double), ("n", C.c_int64),
                ("warn_small_sample", C.c_int32)]


class Stats(C.Structure):
    """wlp_stats: shard sufficient statistics (count, double-double sums)."""
    _fields_ = [("n", C.c_int64), ("sum_hi", C.c_double), ("sum_lo", C.c_double), ("center", C.c_double),
                ("ss_hi", C.c_double), ("ss_lo", C.c_double)]


class Special(C.Structure):
    """wlp_special: a seeding candidate whose key could collide."""
    _fields_ = [("index", C.c_int64), ("s1", C.c_uint32), ("s2", C.c_uint32), ("s3", C.c_uint32),
                ("pad", C.c_uint32)]


_P = C.c_void_p
_I64 = C.c_int64
_SIGS = {
    "wlp_last_error": (C.c_char_p, []),
    "wlp_version": (C.c_int, []),
    "wlp_set_hw_counters": (C.c_int, [C.c_int]),
    "wlp_set_wlp_variant": (C.c_int, [C.c_int]),
    "wlp_set_tlp_variant": (C.c_int, [C.c_int]),
    "wlp_set_pipe_lanes": (C.c_int, [C.c_int]),
    "wlp_debug_set_near_cap": (C.c_int, [C.c_int]),
    "wlp_last_kernel": (C.c_char_p, []),
    "wlp_validate_params": (C.c_int, [C.c_int, C.POINTER(_Params), C.c_char_p, C.c_int]),
    "wlp_plan_launch": (C.c_int, [_I64, C.c_int, C.c_int, _I64, C.POINTER(_Cfg), C.c_char_p, C.c_int]),
    "wlp_master_from_seed": (C.c_int, [C.c_uint64, _P]),
    "wlp_make_state": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, _P]),
    "wlp_jump_host": (C.c_int, [_P, C.c_uint64, _P]),
    "wlp_inverse_normal_cdf": (C.c_int, [C.c_double, C.POINTER(C.c_double)]),
    "wlp_spacing_rejections": (C.c_int, [_P, _I64, _P, _I64, _P, _I64, C.POINTER(_I64)]),
    "wlp_stats_merge": (C.c_int, [C.POINTER(Stats), C.POINTER(Stats)]),
    "wlp_ci_from_stats": (C.c_int, [C.POINTER(Stats), C.c_double, C.POINTER(_CI)]),
    "wlp_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "wlp_taus_stream": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, _I64, _P, C.c_int, _P]),
    "wlp_seed_streams": (C.c_int, [C.c_uint64, _I64, _I64, _P, _I64, _P, C.c_int, _P, _P, _I64, C.POINTER(_I64)]),
    "wlp_seed_streams_exact": (C.c_int, [C.c_uint64, _I64, _P, C.c_int, _P]),
    "wlp_seed_streams_state": (C.c_int, [_P, _I64, _P, C.c_int, _P, _P]),
    "wlp_run_streams": (C.c_int, [C.c_int, C.POINTER(_Params), C.c_int, _P, _I64, C.c_int, _P, _P, _P, C.c_int, _P,
                                  C.POINTER(_Report)]),
    "wlp_run_shard": (C.c_int, [C.c_int, C.POINTER(_Params), C.c_int, C.c_uint64, C.c_int, _I64, _I64, _P, _I64,
                                _P, _P, _P, C.c_int, _P, _P, _I64, C.POINTER(_I64), C.POINTER(_Report)]),
    "wlp_run": (C.c_int, [C.c_int, C.POINTER(_Params), C.c_int, C.c_uint64, C.c_int, _P, _P, _P, C.c_int, _P,
                          C.POINTER(_Report), C.POINTER(_CI), C.c_double, C.c_char_p, C.c_int]),
    "wlp_run_plan": (C.c_int, [C.c_int, _P, _P, C.c_int, C.c_int, C.c_int, _P, _P, _P, C.c_int, _P,
                               C.POINTER(_Report)]),
    "wlp_stats_device": (C.c_int, [_P, _I64, C.c_int, C.POINTER(Stats), _P]),
    "wlp_confidence_interval": (C.c_int, [_P, _I64, C.c_double, C.POINTER(_CI)]),
    "wlp_debug_neg_log1m": (C.c_int, [_P, _I64, _P]),
    "wlp_ir_simulate": (C.c_int, [_P, C.POINTER(_Cfg), _I64, _P, _P, C.c_int, _P, _I64, C.c_int, C.c_int, _I64, _P,
                                  C.POINTER(_Report)]),
    "wlp_ir_jit_simulate": (C.c_int, [_P, C.POINTER(_Cfg), _I64, _P, _P, C.c_int, _P, _I64, C.c_int, _I64, _P,
                                      C.POINTER(_Report)]),
    "wlp_ir_jit_source": (C.c_int, [_P, C.c_char_p, C.c_int, C.POINTER(C.c_int)]),
    "wlp_shutdown": (C.c_int, []),
    "wlp_taus_next": (C.c_int, [_P, C.POINTER(C.c_uint32)]),
    "wlp_set_stats_order": (C.c_int, [C.c_int]),
    "wlp_uniform01": (C.c_int, [_P, C.POINTER(C.c_double)]),
    "wlp_exponential_from_u": (C.c_int, [C.c_double, C.c_double, C.POINTER(C.c_double)]),
    "wlp_run_devices": (C.c_int, [C.c_int, C.POINTER(_Params), C.c_int, C.c_uint64, C.c_int, _P, C.c_int, _P, _P,
                                  _P, C.POINTER(_Report), C.POINTER(_CI), C.c_double, C.c_char_p, C.c_int]),
    "wlp_run_uniforms": (C.c_int, [C.c_int, C.POINTER(_Params), _P, _I64, C.c_int, _P, _P, _P, C.c_int, _P]),
    "wlp_exponentials": (C.c_int, [_P, _I64, C.c_double, _P, C.c_int, _P]),
}
EXPORTS = tuple(_SIGS)


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH.name} is not built; run `python -m paper_1501_01405_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


class _LazyLib:
    """Loads libwlp_b200.so on first use (so `python -m paper_1501_01405_b200.build` can run
    before the library exists); any call without the library raises ImportError."""

    _cdll: Optional[C.CDLL] = None

    def __getattr__(self, name: str):
        if _LazyLib._cdll is None:
            _LazyLib._cdll = _load()
        return getattr(_LazyLib._cdll, name)


_lib = _LazyLib()


def native_library() -> C.CDLL:
    """The loaded libwlp_b200.so (loads it)."""
    _lib.wlp_version
    return _LazyLib._cdll


def _check(status: int) -> None:
    if status != OK:
        msg = (_lib.wlp_last_error() or b"").decode(errors="replace")
        raise _EXC.get(status, Error)(msg)


def _params(p: ModelParams) -> _Params:
    return _Params(int(p.replications), int(p.draws), int(p.clients), float(p.lambda_), float(p.mu),
                   int(p.steps), int(p.chunks))


def _ptr(a) -> Optional[int]:
    """Data pointer of a numpy array / torch tensor / int / None."""
    if a is None:
        return None
    if isinstance(a, int):
        return a
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise DomainError("array must be C-contiguous")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    raise DomainError(f"unsupported buffer type {type(a)!r}")


def _report(r: _Report) -> SimReport:
    return SimReport(r.total_cycles, r.waves_executed, r.peak_resident_warps, r.issues, r.alu_issues, r.mem_reads,
                     r.mem_writes, r.divergence_events, r.kernel_ms, r.warp_splits)


# ---- host utilities (reference host functions) ----------------------------------------------


def validate_params(model: ModelKind, p: ModelParams) -> Optional[str]:
    """validate_params (models.cpp:26-44): DomainError, or the lambda >= mu warning."""
    buf = C.create_string_buffer(512)
    _check(_lib.wlp_validate_params(int(model), C.byref(_params(p)), buf, 512))
    return buf.value.decode() or None


def plan_launch(replications: int, mode: ExecutionMode, prof: Optional[DeviceProfile] = None,
                tlp_block_size: int = 256, grid_limit: int = 65535) -> LaunchPlan:
    """plan_launch (wlp.cpp:71-105), reference geometry and PlanError semantics."""
    prof = prof or DeviceProfile()
    # the reference's check order (wlp.cpp:73-76); the C layer adds CUDA's 1024-thread limit
    if replications < 1:
        raise PlanError("plan_launch: need at least one replication")
    if tlp_block_size < 1:
        raise PlanError("plan_launch: tlp_block_size must be >= 1")
    if tlp_block_size > prof.maxThreadsPerBlock:
        raise PlanError("plan_launch: tlp_block_size exceeds maxThreadsPerBlock")
    cfg = _Cfg()
    buf = C.create_string_buffer(512)
    _check(_lib.wlp_plan_launch(int(replications), int(mode), int(tlp_block_size), int(grid_limit), C.byref(cfg),
                                buf, 512))
    lc = LaunchConfig((cfg.block_x, cfg.block_y, cfg.block_z), (cfg.grid_x, cfg.grid_y), cfg.warp_size)
    return LaunchPlan(lc, int(replications), ExecutionMode(mode), buf.value.decode() or None)


def make_rng_state(s1: int, s2: int, s3: int) -> RngState:
    """make_rng_state (rng.cpp:29-34)."""
    out = (C.c_uint32 * 3)()
    _check(_lib.wlp_make_state(s1 & 0xFFFFFFFF, s2 & 0xFFFFFFFF, s3 & 0xFFFFFFFF, out))
    return RngState(*out)


def rng_state_from_seed(seed: int) -> RngState:
    """rng_state_from_seed (rng.cpp:36-40)."""
    out = (C.c_uint32 * 3)()
    _check(_lib.wlp_master_from_seed(seed & (2**64 - 1), out))
    return RngState(*out)


def jump_state(state: RngState, n: int) -> RngState:
    """State after n taus_next calls, by GF(2) jump-ahead (host)."""
    s = (C.c_uint32 * 3)(state.s1, state.s2, state.s3)
    out = (C.c_uint32 * 3)()
    _check(_lib.wlp_jump_host(s, n, out))
    return RngState(*out)


def inverse_normal_cdf(p: float) -> float:
    """inverse_normal_cdf (models.cpp:61-97)."""
    z = C.c_double()
    _check(_lib.wlp_inverse_normal_cdf(float(p), C.byref(z)))
    return z.value


def spacing_rejections(specials: Sequence[Special], prev: Sequence[int] = ()) -> list:
    """Rejected candidate indices of random_spacing given all special candidates."""
    n = len(specials)
    arr = (Special * max(n, 1))(*specials)
    pv = (C.c_int64 * max(len(prev), 1))(*prev)
    out = (C.c_int64 * (n + len(prev) + 1))()
    nout = C.c_int64()
    _check(_lib.wlp_spacing_rejections(arr, n, pv, len(prev), out, n + len(prev) + 1, C.byref(nout)))
    return list(out[: nout.value])


def stats_merge(a: Stats, b: Stats) -> Stats:
    r = Stats(a.n, a.sum_hi, a.sum_lo, a.center, a.ss_hi, a.ss_lo)
    _check(_lib.wlp_stats_merge(C.byref(r), C.byref(b)))
    return r


def ci_from_stats(s: Stats, level: float = 0.95) -> ConfidenceInterval:
    ci = _CI()
    _check(_lib.wlp_ci_from_stats(C.byref(s), float(level), C.byref(ci)))
    return ConfidenceInterval(ci.mean, ci.half_width, ci.level, ci.n, bool(ci.warn_small_sample))


# ---- device entry points ----------------------------------------------------------------------


def device_count() -> int:
    n = C.c_int()
    _check(_lib.wlp_device_count(C.byref(n)))
    return n.value


def taus_stream(state: RngState, n: int) -> np.ndarray:
    """make_rng_state(state) then n taus_next outputs (rng.cpp:29-51), on the GPU."""
    out = np.empty(n, dtype=np.uint32)
    _check(_lib.wlp_taus_stream(state.s1, state.s2, state.s3, n, _ptr(out), 0, None))
    return out


def random_spacing_seed(master_seed: int, count: int) -> np.ndarray:
    """random_spacing(rng_state_from_seed(master_seed), count) (rng.cpp:67-87) on the GPU.
    Returns a (3, count) uint32 array (rows s1, s2, s3)."""
    out = np.empty((3, count), dtype=np.uint32)
    _check(_lib.wlp_seed_streams_exact(master_seed & (2**64 - 1), count, _ptr(out), 0, None))
    return out


def random_spacing(master: RngState, count: int):
    """random_spacing(master, count) (rng.cpp:67-87) on the GPU from a master state.
    Returns (streams as a (3, count) uint32 array, the master after the consumed draws)."""
    out = np.empty((3, count), dtype=np.uint32)
    m = (C.c_uint32 * 3)(master.s1, master.s2, master.s3)
    after = (C.c_uint32 * 3)()
    _check(_lib.wlp_seed_streams_state(m, count, _ptr(out) if count else None, 0, None, after))
    return out, RngState(*after)


def seed_streams(master_seed: int, slot_begin: int, count: int, rejected: Sequence[int] = (),
                 special_cap: int = 4096):
    """Shard form of random_spacing: stream slots [slot_begin, slot_begin+count) given a
    global rejection list; returns (keys (3,count), specials list)."""
    out = np.empty((3, count), dtype=np.uint32)
    rej = np.asarray(sorted(rejected), dtype=np.int64)
    sp = (Special * special_cap)()
    nsp = C.c_int64()
    _check(_lib.wlp_seed_streams(master_seed & (2**64 - 1), slot_begin, count, _ptr(rej) if len(rej) else None,
                                 len(rej), _ptr(out), 0, None, sp, special_cap, C.byref(nsp)))
    return out, list(sp[: min(nsp.value, special_cap)])


def run_streams(model: ModelKind, p: ModelParams, mode: ExecutionMode, streams: np.ndarray):
    """Replications over explicit streams ((3,R) uint32): pi_/mm1_/walk_replication
    (models.cpp:46-59) of every stream, on the GPU. Returns a dict of output arrays."""
    streams = np.ascontiguousarray(streams, dtype=np.uint32)
    R = streams.shape[1]
    outs = [np.empty(R) for _ in OUTPUT_NAMES[ModelKind(model)]]
    o = [_ptr(x) for x in outs] + [None] * (3 - len(outs))
    _check(_lib.wlp_run_streams(int(model), C.byref(_params(p)), int(mode), _ptr(streams), R, 0, o[0], o[1], o[2], 0,
                                None, None))
    return dict(zip(OUTPUT_NAMES[ModelKind(model)], outs))


def pi_replication(draws: int, stream: RngState) -> float:
    """pi_replication (models.cpp:46-49), one replication on the GPU."""
    s = np.array([[stream.s1], [stream.s2], [stream.s3]], dtype=np.uint32)
    return float(run_streams(ModelKind.Pi, ModelParams(draws=draws), ExecutionMode.Wlp, s)["out"][0])


def mm1_replication(clients: int, lambda_: float, mu: float, stream: RngState):
    """mm1_replication (models.cpp:51-54) -> (avgIdle, avgWaitQueue, avgSystem)."""
    s = np.array([[stream.s1], [stream.s2], [stream.s3]], dtype=np.uint32)
    o = run_streams(ModelKind.Mm1, ModelParams(clients=clients, lambda_=lambda_, mu=mu), ExecutionMode.Wlp, s)
    return float(o["outIdle"][0]), float(o["outWait"][0]), float(o["outSys"][0])


def taus_next(state: RngState) -> int:
    """taus_next (rng.cpp:42-51): advances `state` in place, returns the output (host utility)."""
    s = (C.c_uint32 * 3)(state.s1, state.s2, state.s3)
    out = C.c_uint32()
    _check(_lib.wlp_taus_next(s, C.byref(out)))
    state.s1, state.s2, state.s3 = s
    return out.value


def uniform01(state: RngState) -> float:
    """uniform01 (rng.cpp:53-55) = taus_next * 2^-32."""
    return taus_next(state) * 2.0**-32


def exponential_from_u(u: float, rate: float) -> float:
    """exponential_from_u (rng.cpp:58-61): -log(1-u)/rate through the glibc-log port."""
    out = C.c_double()
    _check(_lib.wlp_exponential_from_u(float(u), float(rate), C.byref(out)))
    return out.value


def exponential(state: RngState, rate: float) -> float:
    """exponential (rng.cpp:63-65)."""
    return exponential_from_u(uniform01(state), rate)


class TausStream:
    """Callable uniform source over an owned state (rng.hpp:42-45)."""

    def __init__(self, state: RngState):
        self.state = RngState(state.s1, state.s2, state.s3)

    def __call__(self) -> float:
        return uniform01(self.state)


def exponentials(u, rate: float) -> np.ndarray:
    """exponential_from_u over an array, on the GPU (glibc-log port)."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.empty(len(u))
    _check(_lib.wlp_exponentials(_ptr(u) if len(u) else None, len(u), float(rate), _ptr(out) if len(u) else None, 0,
                                 None))
    return out


def run_uniforms(model: ModelKind, p: ModelParams, u) -> dict:
    """The reference's *_replication_u bodies (models.hpp:49-108) on the GPU over explicit
    uniforms: u is (count, 2*units) — row r is replication r's source, consumed in order."""
    model = ModelKind(model)
    n = p.units(model)
    u = np.ascontiguousarray(u, dtype=np.float64)
    if u.ndim == 1:
        u = u.reshape(1, -1)
    count = u.shape[0]
    if count and u.shape[1] != 2 * n:
        raise DomainError(f"run_uniforms: need {2 * n} uniforms per replication, got {u.shape[1]}")
    outs = [np.empty(count) for _ in OUTPUT_NAMES[model]]
    o = [_ptr(x) if count else None for x in outs] + [None] * (3 - len(outs))
    _check(_lib.wlp_run_uniforms(int(model), C.byref(_params(p)), _ptr(u) if count else None, count, 0, o[0], o[1],
                                 o[2], 0, None))
    return dict(zip(OUTPUT_NAMES[model], outs))


def _draw(units: int, nxt) -> np.ndarray:
    return np.array([nxt() for _ in range(2 * units)], dtype=np.float64)


def pi_replication_u(draws: int, nxt) -> float:
    """pi_replication_u (models.hpp:49-59): `nxt` is called 2*draws times on the host, the
    body runs on the GPU."""
    p = ModelParams(draws=draws)
    validate_params(ModelKind.Pi, p)
    return float(run_uniforms(ModelKind.Pi, p, _draw(draws, nxt))["out"][0])


def mm1_replication_u(clients: int, lambda_: float, mu: float, nxt):
    """mm1_replication_u (models.hpp:61-84) -> (avgIdle, avgWaitQueue, avgSystem)."""
    p = ModelParams(clients=clients, lambda_=lambda_, mu=mu)
    validate_params(ModelKind.Mm1, p)
    o = run_uniforms(ModelKind.Mm1, p, _draw(clients, nxt))
    return float(o["outIdle"][0]), float(o["outWait"][0]), float(o["outSys"][0])


def walk_replication_u(steps: int, chunks: int, nxt) -> float:
    """walk_replication_u (models.hpp:86-108)."""
    p = ModelParams(steps=steps, chunks=chunks)
    validate_params(ModelKind.Walk, p)
    return float(run_uniforms(ModelKind.Walk, p, _draw(steps, nxt))["out"][0])


def walk_replication(steps: int, chunks: int, stream: RngState) -> float:
    """walk_replication (models.cpp:56-59)."""
    s = np.array([[stream.s1], [stream.s2], [stream.s3]], dtype=np.uint32)
    return float(run_streams(ModelKind.Walk, ModelParams(steps=steps, chunks=chunks), ExecutionMode.Wlp, s)["out"][0])


class wlp_variant:
    """Context manager selecting the WLP kernel for calls on this thread: 0 automatic,
    1 lane jumps, 2 warp pipeline, 3 walk bitsliced warp pipeline, 4 walk bitsliced lane
    chunks (outputs identical; wlp_set_wlp_variant)."""

    def __init__(self, variant: int):
        self.variant = int(variant)

    def __enter__(self):
        _check(_lib.wlp_set_wlp_variant(self.variant))
        return self

    def __exit__(self, *exc):
        _check(_lib.wlp_set_wlp_variant(0))


class pipe_lanes:
    """Context manager: lanes per replication of the warp pipelines (2, 4, 8, 16, 32;
    0 automatic) for calls on this thread (wlp_set_pipe_lanes)."""

    def __init__(self, lanes: int):
        self.lanes = int(lanes)

    def __enter__(self):
        _check(_lib.wlp_set_pipe_lanes(self.lanes))
        return self

    def __exit__(self, *exc):
        _check(_lib.wlp_set_pipe_lanes(0))


class near_cap:
    """Test hook: near-one list capacity of the mm1 warp pipeline (power of two <= 128) for
    calls on this thread (wlp_debug_set_near_cap); small values exercise the overflow redo."""

    def __init__(self, cap: int):
        self.cap = int(cap)

    def __enter__(self):
        _check(_lib.wlp_debug_set_near_cap(self.cap))
        return self

    def __exit__(self, *exc):
        _check(_lib.wlp_debug_set_near_cap(128))


def last_kernel() -> str:
    """Name of the model kernel the last run on this thread launched (wlp_last_kernel)."""
    return _lib.wlp_last_kernel().decode()


class tlp_variant:
    """Context manager selecting the TLP kernel for calls on this thread: 0 automatic,
    1 thread per replication, 2 bitsliced walk (thread per 32 replications; outputs
    identical; wlp_set_tlp_variant)."""

    def __init__(self, variant: int):
        self.variant = int(variant)

    def __enter__(self):
        _check(_lib.wlp_set_tlp_variant(self.variant))
        return self

    def __exit__(self, *exc):
        _check(_lib.wlp_set_tlp_variant(0))


class stats_order:
    """Context manager: summation order of the device statistics on this thread
    (wlp_set_stats_order): 0 accurate double-double (default), 1 the reference's
    sequential order (confidence_interval bit for bit at any n)."""

    def __init__(self, order: int):
        self.order = order

    def __enter__(self):
        _check(_lib.wlp_set_stats_order(self.order))
        return self

    def __exit__(self, *exc):
        _lib.wlp_set_stats_order(0)


class hw_counters:
    """Context manager: SimReports of run_model inside carry hardware counters
    (divergenceEvents with the reference's definition, memReads/memWrites as global
    load/store warp-instructions) from instrumented kernels. See wlp_set_hw_counters."""

    def __enter__(self):
        _check(_lib.wlp_set_hw_counters(1))
        return self

    def __exit__(self, *exc):
        _check(_lib.wlp_set_hw_counters(0))
        return False


def run_model(model: ModelKind, p: ModelParams, mode: ExecutionMode, prof: Optional[DeviceProfile] = None,
              master_seed: int = 1, tlp_block_size: int = 256, opts: Optional[SimOptions] = None,
              *, timed: bool = True) -> ModelRun:
    """run_model (models.cpp:329-397): seeds R streams by random spacing from master_seed,
    runs the model in `mode` on the GPU, returns per-replication outputs (host arrays).

    Outputs are bit-identical to the reference's Sequential mode. `prof`/`opts` are
    accepted for signature compatibility and ignored (the hardware is real). The
    SEQUENTIAL mode runs the warp-per-replication kernel too (there is no host path);
    its `cfg` is the reference's single-thread geometry.
    """
    model, mode = ModelKind(model), ExecutionMode(mode)
    if opts is not None and opts.irInterpreter:
        from . import ir  # the reference's IR kernels on the GPU interpreter (or compiled)

        return ir.run_model(model, p, mode, master_seed, tlp_block_size, jit=opts.irJit)
    plan = plan_launch(p.replications, mode, prof, tlp_block_size, grid_limit=0x7FFFFFFF)
    R = int(p.replications)
    names = OUTPUT_NAMES[model]
    outs = [np.empty(R) for _ in names]
    o = [_ptr(x) for x in outs] + [None] * (3 - len(outs))
    rep = _Report()
    warn = C.create_string_buffer(512)
    devices = opts.devices if opts is not None else 1
    if devices > 1:  # contiguous slices over GPUs 0..devices-1, one host thread each
        devs = (C.c_int * devices)(*range(devices))
        _check(_lib.wlp_run_devices(int(model), C.byref(_params(p)), int(mode), master_seed & (2**64 - 1),
                                    int(tlp_block_size), devs, devices, o[0], o[1], o[2],
                                    C.byref(rep) if timed else None, None, 0.95, warn, 512))
        outputs = dict(zip(names, outs))
        return ModelRun(outputs, outputs[PRIMARY[model]], _report(rep), plan.cfg, mode, warn.value.decode() or None)
    _check(_lib.wlp_run(int(model), C.byref(_params(p)), int(mode), master_seed & (2**64 - 1), int(tlp_block_size),
                        o[0], o[1], o[2], 0, None, C.byref(rep) if timed else None, None, 0.95, warn, 512))
    outputs = dict(zip(names, outs))
    return ModelRun(outputs, outputs[PRIMARY[model]], _report(rep), plan.cfg, mode, warn.value.decode() or None)


def run_devices(model: ModelKind, p: ModelParams, mode: ExecutionMode, master_seed: int, devices: Sequence[int],
                outs=None, *, ci_level: Optional[float] = None, tlp_block_size: int = 256,
                report: Optional[SimReport] = None):
    """run_model over several GPUs of this process (wlp_run_devices): host output arrays
    (allocated when outs is None), bit-identical to run_model; returns (outs, CIs or None)."""
    model = ModelKind(model)
    names = OUTPUT_NAMES[model]
    if outs is None:
        outs = [np.empty(int(p.replications)) for _ in names]
    o = [_ptr(x) for x in outs] + [None] * (3 - len(outs))
    devs = (C.c_int * max(len(devices), 1))(*devices)
    cis = (_CI * len(names))() if ci_level is not None else None
    rep = _Report() if report is not None else None
    _check(_lib.wlp_run_devices(int(model), C.byref(_params(p)), int(mode), master_seed & (2**64 - 1),
                                int(tlp_block_size), devs, len(devices), o[0], o[1], o[2],
                                C.byref(rep) if rep is not None else None, cis, float(ci_level or 0.95), None, 0))
    if rep is not None:
        report.__dict__.update(vars(_report(rep)))
    ci = None if cis is None else [ConfidenceInterval(c.mean, c.half_width, c.level, c.n,
                                                      bool(c.warn_small_sample)) for c in cis]
    return outs, ci


def run_model_into(model: ModelKind, p: ModelParams, mode: ExecutionMode, master_seed: int, outs, *,
                   on_device: bool, stream: Optional[int] = None, tlp_block_size: int = 256,
                   ci_level: Optional[float] = None, report: Optional[SimReport] = None):
    """Low-level run_model writing into caller buffers (device pointers / torch CUDA tensors
    when on_device, else host arrays; pinned host arrays are written by the kernels
    directly). Returns the list of ConfidenceIntervals when ci_level is given (device
    reduction, one synchronisation for the run and every CI), else None."""
    o = [_ptr(x) for x in outs] + [None] * (3 - len(outs))
    nci = len(OUTPUT_NAMES[ModelKind(model)])
    cis = (_CI * nci)() if ci_level is not None else None
    rep = _Report() if report is not None else None
    _check(_lib.wlp_run(int(model), C.byref(_params(p)), int(mode), master_seed & (2**64 - 1), int(tlp_block_size),
                        o[0], o[1], o[2], 1 if on_device else 0, stream, C.byref(rep) if rep is not None else None,
                        cis, float(ci_level or 0.95), None, 0))
    if rep is not None:
        report.__dict__.update(vars(_report(rep)))
    if cis is None:
        return None
    return [ConfidenceInterval(c.mean, c.half_width, c.level, c.n, bool(c.warn_small_sample)) for c in cis]


_SPECIAL_BUFS: dict = {}


def _special_buffer(cap: int):
    """A reused ctypes array for the specials a shard run reports (allocating and zeroing
    ~100 KB per call showed up in small runs' host time)."""
    b = _SPECIAL_BUFS.get(cap)
    if b is None:
        b = _SPECIAL_BUFS[cap] = (Special * cap)()
    return b


def run_shard(model: ModelKind, p: ModelParams, mode: ExecutionMode, master_seed: int, r_begin: int, r_count: int,
              outs, *, on_device: bool, rejected: Sequence[int] = (), stream: Optional[int] = None,
              tlp_block_size: int = 256, special_cap: int = 4096, report: Optional[SimReport] = None):
    """Shard [r_begin, r_begin + r_count) of a run of p.replications; returns the shard's
    special seeding candidates. If `report` is given it is filled
    with the model kernel's measured time (CUDA events on the launching stream). With
    on_device and no report the call returns once the seeding has reported, the model
    still running on `stream` (None: the legacy default stream, torch's default)."""
    o = [_ptr(x) for x in outs] + [None] * (3 - len(outs))
    rej = np.asarray(sorted(rejected), dtype=np.int64) if len(rejected) else None  # (usually empty)
    sp = _special_buffer(special_cap)
    nsp = C.c_int64()
    rep = _Report() if report is not None else None
    _check(_lib.wlp_run_shard(int(model), C.byref(_params(p)), int(mode), master_seed & (2**64 - 1),
                              int(tlp_block_size), r_begin, r_count, _ptr(rej) if rej is not None else None,
                              len(rej) if rej is not None else 0,
                              o[0], o[1], o[2], 1 if on_device else 0, stream, sp, special_cap, C.byref(nsp),
                              C.byref(rep) if rep is not None else None))
    if rep is not None:
        report.__dict__.update(vars(_report(rep)))
    if nsp.value > special_cap:
        raise Error("too many special seeding candidates")
    return [Special.from_buffer_copy(x) for x in sp[: nsp.value]]  # (the buffer is reused)


class PlanSets:
    """A plan's factor-level sets and master seeds marshalled once for the C ABI (the
    per-set ctypes conversion costs ~2 us a set, 150 us for BASELINE config 5's 64 sets —
    more than a third of the run). Pass it to run_plan in place of (sets, master_seeds)."""

    def __init__(self, sets: Sequence[ModelParams], master_seeds: Sequence[int]):
        if len(sets) != len(master_seeds):
            raise DomainError("plan: one master seed per set")
        n = len(sets)
        self.sets = list(sets)
        self.params = (_Params * max(n, 1))(*[_params(p) for p in sets])
        self.seeds = (C.c_uint64 * max(n, 1))(*[s & (2**64 - 1) for s in master_seeds])
        self.replications = [int(p.replications) for p in sets]
        self.total = sum(self.replications)

    def __len__(self) -> int:
        return len(self.sets)


def run_plan(model: ModelKind, sets, master_seeds: Optional[Sequence[int]], mode: ExecutionMode,
             outs=None, *, on_device: bool = False, stream: Optional[int] = None, tlp_block_size: int = 256,
             report: Optional[SimReport] = None):
    """Experimental plan (BASELINE config 5): every factor-level set k is
    run_model(model, sets[k], mode, master_seeds[k]), all in one launch. `sets` is a list of
    ModelParams (with `master_seeds`) or a PlanSets (master_seeds None). Returns a list (per
    set) of output dicts when outs is None (host), else fills `outs` (concatenated)."""
    model = ModelKind(model)
    ps = sets if isinstance(sets, PlanSets) else PlanSets(sets, master_seeds)
    n = len(ps)
    arr, seeds, R = ps.params, ps.seeds, ps.total
    sets = ps.sets
    names = OUTPUT_NAMES[model]
    host = outs is None
    if host:
        outs = [np.empty(R) for _ in names]
    o = [_ptr(x) for x in outs] + [None] * (3 - len(outs))
    rep = _Report() if report is not None else None
    _check(_lib.wlp_run_plan(int(model), arr, seeds, n, int(mode), int(tlp_block_size), o[0], o[1], o[2],
                             1 if on_device else 0, stream, C.byref(rep) if rep is not None else None))
    if rep is not None:
        report.__dict__.update(vars(_report(rep)))
    if not host:
        return None
    res, off = [], 0
    for p in sets:
        r = int(p.replications)
        res.append({nm: o_[off:off + r] for nm, o_ in zip(names, outs)})
        off += r
    return res


def stats_device(x, n: int, pass_: int, stats: Optional[Stats] = None, stream: Optional[int] = None) -> Stats:
    """Device sufficient statistics of a device array (pass 1: sum; pass 2: centred SS)."""
    s = stats if stats is not None else Stats()
    _check(_lib.wlp_stats_device(_ptr(x), n, pass_, C.byref(s), stream))
    return s


def confidence_interval(samples, level: float = 0.95) -> ConfidenceInterval:
    """confidence_interval (models.cpp:99-119) through the device reduction. For n <= 256
    the sums are the reference's sequential loop, bit for bit."""
    x = np.ascontiguousarray(samples, dtype=np.float64)
    ci = _CI()
    _check(_lib.wlp_confidence_interval(_ptr(x) if len(x) else None, len(x), float(level), C.byref(ci)))
    return ConfidenceInterval(ci.mean, ci.half_width, ci.level, ci.n, bool(ci.warn_small_sample))


def debug_neg_log1m(k) -> np.ndarray:
    """-log(1 - k*2^-32) through the device glibc-log port (test hook)."""
    k = np.ascontiguousarray(k, dtype=np.uint32)
    out = np.empty(len(k))
    _check(_lib.wlp_debug_neg_log1m(_ptr(k) if len(k) else None, len(k), _ptr(out) if len(k) else None))
    return out


def shutdown() -> None:
    _check(_lib.wlp_shutdown())
