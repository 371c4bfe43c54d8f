"""The C++ drop-in API (include/warpsim_b200.hpp) and the warpsim CLI, driven by the C++
harness tests/cpp/test_dropin.cpp (the reference's test cases, oracle as host reference)."""
import subprocess

import pytest

import oracle
from conftest import ROOT

PKG = ROOT / "paper_1501_01405_b200"


@pytest.fixture(scope="module")
def harness(tmp_path_factory):
    if not (PKG / "libwarpsim_b200.so").exists():
        from paper_1501_01405_b200 import build

        build.build_all()
    if not oracle.available("port"):
        oracle.build()
    exe = tmp_path_factory.mktemp("cpp") / "test_dropin"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT / 'include'}", str(ROOT / "tests" / "cpp" / "test_dropin.cpp"),
                    "-o", str(exe), f"-L{PKG}", "-lwarpsim_b200", "-lwlp_b200", str(oracle.PORT_SO),
                    f"-Wl,-rpath,{PKG}:{oracle.HERE}"], check=True)
    return exe


def _run(cmd):
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    print(out.stdout[-4000:], out.stderr[-2000:])
    return out


def test_cpp_host_api(harness):
    out = _run([str(harness), "--cpu", str(ROOT)])
    assert out.returncode == 0 and "0 failures" in out.stdout


def test_cli_usage_exit_codes():
    cli = PKG / "warpsim"
    assert _run([str(cli)]).returncode == 2
    assert _run([str(cli), "frobnicate"]).returncode == 2


@pytest.mark.gpu
def test_cpp_full_api_on_gpu(harness):
    out = _run([str(harness), "--gpu", str(ROOT)])
    assert out.returncode == 0 and "0 failures" in out.stdout


@pytest.mark.gpu
def test_cli_sweep_steps_ci(tmp_path):
    cli = PKG / "warpsim"
    csv = tmp_path / "pi.csv"
    r = _run([str(cli), "sweep", "--model", "pi", "--modes", "sequential,tlp,wlp", "--r-min", "1", "--r-max", "2",
              "--draws", "100", "--seed", "42", "--out", str(csv)])
    assert r.returncode == 0
    got = [l.split(",") for l in csv.read_text().splitlines()[1:]]
    want = [l.split(",") for l in (ROOT / "tests" / "golden" / "sweep_pi.csv").read_text().splitlines()[1:]]
    assert [g[:3] + g[8:] for g in got] == [w[:3] + w[8:] for w in want]
    # steps on the reference's (simulated, monotone) cost curves
    r = _run([str(cli), "steps", str(ROOT / "tests" / "golden" / "sweep_pi.csv")])
    assert r.returncode == 0 and "wlp" in r.stdout and "plateau=81408" in r.stdout
    # measured GPU cycles are not monotone in R: detect_steps keeps the reference's
    # AnalysisError (exit 1) rather than inventing steps
    r = _run([str(cli), "steps", str(csv)])
    assert r.returncode in (0, 1)
    r = _run([str(cli), "ci", "--model", "mm1", "--replications", "30", "--clients", "100000", "--seed", "42"])
    assert r.returncode == 0 and "wait" in r.stdout and "n=30" in r.stdout
    r = _run([str(cli), "ci", "--model", "pi", "--draws", "0"])
    assert r.returncode == 2  # DomainError


def test_cli_dump_kernel_prints_the_reference_ir():
    # warpsim_main.cpp:101-110: `sweep --dump-kernel` prints each mode's kernel text
    out = _run([str(PKG / "warpsim"), "sweep", "--model", "mm1", "--modes", "tlp,wlp", "--r-max", "9",
                "--dump-kernel"])
    assert out.returncode == 0
    want = "".join(f"; mm1, {m}, R=9\n" + (ROOT / "tests" / "golden" / "ir" / f"mm1_{m}.sexp").read_text() + "\n"
                   for m in ("tlp", "wlp"))
    assert out.stdout == want


@pytest.mark.gpu
def test_cli_sweep_with_ir_counters_matches_reference_golden_csv():
    # proj/tests/golden/sweep_pi.golden through `warpsim sweep --ir-counters`: every column
    # of the sequential rows (the unit-cost accounting) and every column but the
    # Fermi-modelled total_cycles of the tlp / wlp rows equal the reference's CSV
    out = _run([str(PKG / "warpsim"), "sweep", "--model", "pi", "--modes", "sequential,tlp,wlp", "--r-min", "1",
                "--r-max", "2", "--draws", "100", "--seed", "42", "--ir-counters"])
    assert out.returncode == 0
    got = [r.split(",") for r in out.stdout.strip().splitlines()]
    want = [r.split(",") for r in (ROOT / "tests" / "golden" / "sweep_pi.csv").read_text().strip().splitlines()]
    assert got[0] == want[0] and len(got) == len(want)
    for g, r in zip(got[1:], want[1:]):
        if g[1] == "sequential":
            assert g == r
        else:
            assert g[:3] + g[4:] == r[:3] + r[4:] and int(g[3]) > 0
