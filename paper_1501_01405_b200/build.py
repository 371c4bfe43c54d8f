"""Build the native libraries in-tree (sm_100a only).

    python -m paper_1501_01405_b200.build          # or __graft_entry__.build()

Outputs (git-ignored, shipped to the GPU box with the gpurun snapshot):
    paper_1501_01405_b200/libwlp_b200.so       CUDA kernels + C ABI (include/wlp_b200.h)
    paper_1501_01405_b200/libwarpsim_b200.so   C++ drop-in API (include/warpsim_b200.hpp)

Device code is compiled with --fmad=false: the reference is built with
-ffp-contract=off (proj/CMakeLists.txt:12-13), so no a*b+c may be fused except the
explicit fma() steps of the glibc log port.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
HOST = PKG / "host"
LIB = PKG / "libwlp_b200.so"
CXXLIB = PKG / "libwarpsim_b200.so"
CLI = PKG / "warpsim"

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
           "-Xptxas", "-warn-spills"]


def _run(cmd: list[str]) -> None:
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _stale(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_cuda(force: bool = False) -> Path:
    srcs = [CSRC / "kernels.cu", CSRC / "ir_interp.cu", CSRC / "runtime.cu"]
    deps = srcs + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.hpp")) + sorted(CSRC.glob("*.h")) + [
        ROOT / "include" / "wlp_b200.h"]
    if force or _stale(LIB, deps):
        _run([NVCC, *ARCH, *NVFLAGS, "-shared", *map(str, srcs), "-o", str(LIB)])
    return LIB


def build_cxx(force: bool = False) -> Path:
    srcs = [HOST / "warpsim_api.cpp", HOST / "ir.cpp"]
    deps = srcs + [ROOT / "include" / "warpsim_b200.hpp", ROOT / "include" / "warpsim_ir_b200.hpp",
                   ROOT / "include" / "wlp_b200.h", LIB]
    if force or _stale(CXXLIB, deps):
        _run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-fPIC", "-shared", f"-I{ROOT / 'include'}",
              *map(str, srcs), "-o", str(CXXLIB), f"-L{PKG}", "-lwlp_b200", "-Wl,-rpath,$ORIGIN"])
    return CXXLIB


def build_cli(force: bool = False) -> Path:
    src = HOST / "cli.cpp"
    if force or _stale(CLI, [src, ROOT / "include" / "warpsim_b200.hpp", ROOT / "include" / "warpsim_ir_b200.hpp",
                             CXXLIB]):
        _run(["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", str(src), "-o", str(CLI), f"-L{PKG}",
              "-lwarpsim_b200", "-lwlp_b200", "-Wl,-rpath,$ORIGIN"])
    return CLI


def build_all(force: bool = False) -> None:
    build_cuda(force)
    build_cxx(force)
    build_cli(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
