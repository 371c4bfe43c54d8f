"""TEST INFRASTRUCTURE ONLY — the CPU oracle.

Python bindings (ctypes) for
  * ``oracle/_ref/libwarpsim_ref.so`` — the reference sources compiled unmodified
    (oracle/Makefile) behind oracle/ref_shim.cpp: ``Oracle("reference")``;
  * ``oracle/liboracle.so`` — the plain-C restatement (oracle/oracle.c): ``Oracle("port")``.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) may
import this package, and only as the checker / CPU baseline. The product
(paper_1501_01405_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path
from typing import Optional

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SO = HERE / "_ref" / "libwarpsim_ref.so"
PORT_SO = HERE / "liboracle.so"
OUTPUTS = {0: ("out",), 1: ("outIdle", "outWait", "outSys"), 2: ("out",)}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class _Params(C.Structure):
    _fields_ = [("replications", C.c_int64), ("draws", C.c_int64), ("clients", C.c_int64),
                ("lambda_", C.c_double), ("mu", C.c_double), ("steps", C.c_int64), ("chunks", C.c_int64)]


def params(replications=1, draws=1000, clients=1000, lambda_=0.5, mu=1.0, steps=1000, chunks=30) -> _Params:
    return _Params(replications, draws, clients, lambda_, mu, steps, chunks)


def params_from(p) -> _Params:
    """From a paper_1501_01405_b200.ModelParams-like object."""
    return _Params(int(p.replications), int(p.draws), int(p.clients), float(p.lambda_), float(p.mu), int(p.steps),
                   int(p.chunks))


def build() -> None:
    """Build liboracle.so and, when /root/reference is present, _ref/libwarpsim_ref.so."""
    targets = ["liboracle.so"] if not Path("/root/reference/proj/src").is_dir() else ["all"]
    subprocess.run(["make", "-s", "-C", str(HERE), *[str(HERE / t) if t.endswith(".so") else t for t in targets]],
                   check=True)


def available(kind: str) -> bool:
    return (REF_SO if kind == "reference" else PORT_SO).exists()


class Oracle:
    def __init__(self, kind: str = "reference"):
        self.kind = kind
        path = REF_SO if kind == "reference" else PORT_SO
        if not path.exists():
            raise FileNotFoundError(f"oracle library {path} not built (make -C oracle)")
        self.lib = C.CDLL(str(path))
        self.p = "ref_" if kind == "reference" else "oracle_"

    def _fn(self, name: str):
        return getattr(self.lib, self.p + name)

    def _check(self, st: int) -> None:
        if st:
            msg = ""
            if self.kind == "reference":
                f = self.lib.ref_last_error
                f.restype = C.c_char_p
                msg = f().decode()
            raise OracleError(st, msg)

    def taus_stream(self, s1: int, s2: int, s3: int, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint32)
        f = self._fn("taus_stream")
        f.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_int64, C.c_void_p]
        self._check(f(s1, s2, s3, n, out.ctypes.data))
        return out

    def master_from_seed(self, seed: int):
        out = (C.c_uint32 * 3)()
        f = self._fn("master_from_seed")
        f.argtypes = [C.c_uint64, C.c_void_p]
        self._check(f(seed, out) or 0)
        return tuple(out)

    def random_spacing(self, seed: int, count: int) -> np.ndarray:
        out = np.empty((3, count), dtype=np.uint32)
        f = self._fn("random_spacing")
        f.argtypes = [C.c_uint64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        self._check(f(seed, count, out[0].ctypes.data, out[1].ctypes.data, out[2].ctypes.data))
        return out

    def replications(self, model: int, p: _Params, streams: np.ndarray, nthreads: int = 1) -> dict:
        streams = np.ascontiguousarray(streams, dtype=np.uint32)
        R = streams.shape[1]
        outs = [np.empty(R) for _ in OUTPUTS[model]]
        ptrs = [o.ctypes.data for o in outs] + [None] * (3 - len(outs))
        f = self._fn("replications")
        if self.kind == "reference":
            f.argtypes = [C.c_int, C.POINTER(_Params), C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                          C.c_void_p, C.c_void_p, C.c_int]
            self._check(f(model, C.byref(p), streams[0].ctypes.data, streams[1].ctypes.data,
                          streams[2].ctypes.data, R, *ptrs, nthreads))
        else:
            f.argtypes = [C.c_int, C.POINTER(_Params), C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                          C.c_void_p, C.c_void_p]
            self._check(f(model, C.byref(p), streams[0].ctypes.data, streams[1].ctypes.data,
                          streams[2].ctypes.data, R, *ptrs))
        return dict(zip(OUTPUTS[model], outs))

    def run_model(self, model: int, p: _Params, seed: int, mode: int = 0, tlp_block: int = 256) -> dict:
        """run_model outputs (+ '_warning', '_cycles' for the reference)."""
        R = p.replications
        outs = [np.empty(R) for _ in OUTPUTS[model]]
        ptrs = [o.ctypes.data for o in outs] + [None] * (3 - len(outs))
        f = self._fn("run_model")
        res = dict(zip(OUTPUTS[model], outs))
        if self.kind == "reference":
            warn = C.create_string_buffer(512)
            cyc = C.c_int64()
            f.argtypes = [C.c_int, C.POINTER(_Params), C.c_int, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p,
                          C.c_void_p, C.c_char_p, C.c_int, C.POINTER(C.c_int64)]
            self._check(f(model, C.byref(p), mode, seed, tlp_block, *ptrs, warn, 512, C.byref(cyc)))
            res["_warning"] = warn.value.decode() or None
            res["_cycles"] = cyc.value
        else:
            if mode != 0:
                raise ValueError("the C port implements the Sequential path only")
            f.argtypes = [C.c_int, C.POINTER(_Params), C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]
            self._check(f(model, C.byref(p), seed, *ptrs))
        return res

    def confidence_interval(self, x, level: float = 0.95):
        x = np.ascontiguousarray(x, dtype=np.float64)
        mean, hw = C.c_double(), C.c_double()
        warn = C.c_int()
        f = self._fn("confidence_interval")
        if self.kind == "reference":
            n = C.c_int64()
            f.argtypes = [C.c_void_p, C.c_int64, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double),
                          C.POINTER(C.c_int64), C.POINTER(C.c_int)]
            self._check(f(x.ctypes.data if len(x) else None, len(x), level, C.byref(mean), C.byref(hw), C.byref(n),
                          C.byref(warn)))
        else:
            f.argtypes = [C.c_void_p, C.c_int64, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double),
                          C.POINTER(C.c_int)]
            self._check(f(x.ctypes.data if len(x) else None, len(x), level, C.byref(mean), C.byref(hw),
                          C.byref(warn)))
        return mean.value, hw.value, len(x), bool(warn.value)

    def inverse_normal_cdf(self, p: float) -> float:
        z = C.c_double()
        f = self._fn("inverse_normal_cdf")
        f.argtypes = [C.c_double, C.POINTER(C.c_double)]
        self._check(f(p, C.byref(z)))
        return z.value

    def replications_u(self, model: int, p: _Params, u) -> dict:
        """The reference's *_replication_u templates over rows of explicit uniforms
        (reference only)."""
        u = np.ascontiguousarray(u, dtype=np.float64)
        R = u.shape[0]
        outs = [np.empty(R) for _ in OUTPUTS[model]]
        ptrs = [o.ctypes.data for o in outs] + [None] * (3 - len(outs))
        f = self._fn("replications_u")
        f.argtypes = [C.c_int, C.POINTER(_Params), C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        self._check(f(model, C.byref(p), u.ctypes.data, R, *ptrs))
        return dict(zip(OUTPUTS[model], outs))

    def exponential_from_u(self, u, rate: float) -> np.ndarray:
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.empty_like(u)
        f = self._fn("exponential_from_u")
        f.argtypes = [C.c_void_p, C.c_int64, C.c_double, C.c_void_p]
        self._check(f(u.ctypes.data, len(u), rate, out.ctypes.data))
        return out

    # reference-only helpers
    def run_model_report(self, model: int, p: _Params, seed: int, mode: int, tlp_block: int = 256) -> dict:
        """The reference's SimReport (simulated Fermi counters) of run_model."""
        out = (C.c_int64 * 8)()
        f = self.lib.ref_run_model_report
        f.argtypes = [C.c_int, C.POINTER(_Params), C.c_int, C.c_uint64, C.c_int, C.c_void_p]
        self._check(f(model, C.byref(p), mode, seed, tlp_block, out))
        keys = ("totalCycles", "wavesExecuted", "peakResidentWarps", "issues", "aluIssues", "memReads", "memWrites",
                "divergenceEvents")
        return dict(zip(keys, list(out)))

    # kernel IR (reference-only): the checker of the GPU IR interpreter
    def _ir_text(self, fn, *args) -> str:
        need = C.c_int(0)
        self._check(fn(*args, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        self._check(fn(*args, buf, need.value, None))
        return buf.value.decode()

    def ir_model_text(self, model: int, mode: int = 0) -> str:
        """dump_kernel of build_model_body(model), wrap_tlp (mode 1) / wrap_wlp (mode 2)."""
        f = self.lib.ref_ir_model_text
        f.argtypes = [C.c_int, C.c_int, C.c_char_p, C.c_int, C.POINTER(C.c_int)]
        return self._ir_text(f, model, mode)

    def ir_canonical(self, text: str) -> str:
        f = self.lib.ref_ir_canonical
        f.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.POINTER(C.c_int)]
        return self._ir_text(f, text.encode())

    def ir_simulate(self, text: str, cfg: tuple, scalars: dict, arrays: dict, streams: Optional[np.ndarray] = None,
                    mask_depth: int = 32, max_threads_per_block: int = 1024) -> dict:
        """The reference simulator (simulate, device.cpp:140-226) on a kernel text.
        cfg = (bx, by, bz, gx, gy, warpSize); arrays (float64) are updated in place;
        streams (3, n) uint32. Returns the SimReport fields."""
        names = list(scalars)
        n = max(len(names), 1)
        is_int = (C.c_int * n)(*[isinstance(scalars[k], (int, np.integer)) for k in names])
        ivals = (C.c_int64 * n)(*[int(scalars[k]) if is_int[i] else 0 for i, k in enumerate(names)])
        rvals = (C.c_double * n)(*[0.0 if is_int[i] else float(scalars[k]) for i, k in enumerate(names)])
        cn = (C.c_char_p * n)(*[k.encode() for k in names])
        an = list(arrays)
        m = max(len(an), 1)
        can = (C.c_char_p * m)(*[k.encode() for k in an])
        ap = (C.c_void_p * m)(*[arrays[k].ctypes.data for k in an])
        al = (C.c_int64 * m)(*[arrays[k].size for k in an])
        st = np.zeros((3, 0), dtype=np.uint32) if streams is None else np.ascontiguousarray(streams, dtype=np.uint32)
        c6 = (C.c_int64 * 6)(*cfg)
        out = (C.c_int64 * 8)()
        f = self.lib.ref_ir_simulate_text
        f.argtypes = [C.c_char_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                      C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_void_p]
        self._check(f(text.encode(), c6, max_threads_per_block, len(names), cn, is_int, ivals, rvals, len(an), can, ap,
                      al, st.ctypes.data if st.size else None, st.shape[1], mask_depth, out))
        keys = ("totalCycles", "wavesExecuted", "peakResidentWarps", "issues", "aluIssues", "memReads", "memWrites",
                "divergenceEvents")
        return dict(zip(keys, list(out)))

    def plan_launch(self, R: int, mode: int, tlp_block: int = 256):
        dims = (C.c_int64 * 3)()
        warn = C.create_string_buffer(512)
        f = self.lib.ref_plan_launch
        f.argtypes = [C.c_int64, C.c_int, C.c_int, C.c_void_p, C.c_char_p, C.c_int]
        self._check(f(R, mode, tlp_block, dims, warn, 512))
        return tuple(dims), warn.value.decode() or None

    def sweep_csv(self, model: int, modes_mask: int, rmin: int, rmax: int, rstep: int, p: _Params, seed: int,
                  tlp_block: int = 256) -> str:
        buf = C.create_string_buffer(1 << 20)
        f = self.lib.ref_sweep_csv
        f.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.POINTER(_Params), C.c_uint64, C.c_int,
                      C.c_char_p, C.c_int64]
        self._check(f(model, modes_mask, rmin, rmax, rstep, C.byref(p), seed, tlp_block, buf, 1 << 20))
        return buf.value.decode()


def host_log_variant() -> str:
    """Which glibc `log` the host's ifunc selects (the mm1 port reproduces the FMA one)."""
    try:
        flags = Path("/proc/cpuinfo").read_text().split("flags", 1)[1].split("\n", 1)[0].split()
    except Exception:  # pragma: no cover
        return "unknown"
    return "fma" if ("fma" in flags and "avx2" in flags) else "non-fma"


def optional(kind: str) -> Optional[Oracle]:
    return Oracle(kind) if available(kind) else None
