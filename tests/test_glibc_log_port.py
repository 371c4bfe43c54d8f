"""The glibc-log port (csrc/glibc_log.cuh, host build) against this host's libm `log`.
CPU only; the device build of the same source is pinned in test_parity_gpu.py."""
import subprocess

import pytest

import oracle
from conftest import ROOT, golden


def test_port_matches_libm_sampled(tmp_path):
    if oracle.host_log_variant() != "fma":
        pytest.skip("host glibc selects the non-FMA log; the port reproduces __log_fma")
    exe = tmp_path / "chk"
    subprocess.run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-pthread",
                    str(ROOT / "tools" / "check_glibc_log.cpp"), "-o", str(exe), "-lm"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0, out.stdout
    assert "mismatches 0" in out.stdout


def test_fixture_records_fma_variant():
    assert golden("log_pairs.json")["host_log_variant"] == "fma"
