"""The reference's own doctest unit tests (proj/tests/test_rng.cpp, test_models.cpp,
test_sweep.cpp), compiled unmodified against the drop-in headers and run on the GPU path
(tests/cpp/Makefile; doctest stand-in tests/cpp/doctest_shim/doctest.h).

Excluded test cases, each about the reference's simulated cycle accounting, which the
drop-in replaces by measured GPU time (DESIGN.md §1 "Deliberate deviations"):
  * "sequential mode: host outputs, replication-linear unit cost" — asserts
    totalCycles(R=9) == 9 * totalCycles(R=1) of the unit-cost replay; its output checks
    are covered by "device execution is bit-identical to the host references";
  * "sequential rows scale linearly in R" — the same identity on sweep rows;
  * "wlp cost curve steps exactly at the residency cap" — the C2050 profile's simulated
    wave steps (replications 65, 129). The measured curves are in profiles/;
  * "sweeps are deterministic and byte-stable against the golden file" — the golden CSV's
    total_cycles column is simulated; here it is measured (so two sweeps differ there).
    Every other column of sweep_pi.golden is checked byte for byte by
    tests/test_cpp_dropin.py.
The reference's other test files (test_wlp, test_device_sim, test_kernel_ir,
test_kernel_text) exercise the host SIMT simulator's internals (WarpState, IssueRecord,
load_profile), which are out of scope.
"""
import subprocess
from pathlib import Path

import pytest

HERE = Path(__file__).resolve().parent / "cpp"
BIN = HERE / "_ref" / "reftests"
EXCLUDED = ["sequential mode: host outputs, replication-linear unit cost",
            "sequential rows scale linearly in R",
            "wlp cost curve steps exactly at the residency cap",
            "sweeps are deterministic and byte-stable against the golden file"]
need_bin = pytest.mark.skipif(not BIN.exists(), reason="tests/cpp/_ref/reftests not built (needs /root/reference)")


@need_bin
def test_reference_test_cases_are_all_compiled():
    names = subprocess.run([str(BIN), "--list"], capture_output=True, text=True, check=True).stdout.splitlines()
    assert len(names) == 40
    assert set(EXCLUDED) <= set(names)
    for must in ("taus88 reproduces the shipped golden sequence", "pi replication on scripted draws",
                 "mm1 hand trace: arrivals (1,1,1), services (2,2,2)", "walk on scripted draws",
                 "device execution is bit-identical to the host references",
                 "sweeps are deterministic and byte-stable against the golden file"):
        assert must in names


@need_bin
@pytest.mark.gpu
def test_reference_unit_tests_pass_on_the_gpu_path(gpu):
    r = subprocess.run([str(BIN), *[f"--exclude={n}" for n in EXCLUDED]], capture_output=True, text=True, cwd=HERE,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "36 run, 0 failed, 4 excluded" in r.stdout
