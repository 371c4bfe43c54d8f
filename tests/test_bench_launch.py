"""bench.py's launch plumbing on CPU: --gpus N outside torchrun re-launches N ranks
(torch.distributed.run, 127.0.0.1), the ranks come up, WORLD_SIZE must equal --gpus, and
timings are maxed over ranks. The GPU work itself is covered by the -m gpu suite."""
import json
import os
import subprocess
import sys

from conftest import ROOT


def _bench(*args, env=None):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True, env=e,
                          timeout=300)


def _line(out: str) -> dict:
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out
    return json.loads(lines[0])


def test_self_launch_two_ranks():
    r = _bench("--gpus", "2", "--dry-run")
    assert r.returncode == 0, r.stderr
    d = _line(r.stdout)
    assert (d["n_gpus"], d["world"], d["backend"], d["max_over_ranks"]) == (2, 2, "gloo", 2.0)


def test_reference_arm_self_launch_prints_once():
    r = _bench("--gpus", "3", "--dry-run", "--impl", "reference")
    assert r.returncode == 0, r.stderr
    assert _line(r.stdout)["n_gpus"] == 3


def test_single_gpu_does_not_relaunch():
    r = _bench("--dry-run")
    assert r.returncode == 0, r.stderr
    d = _line(r.stdout)
    assert (d["n_gpus"], d["backend"]) == (1, None)


def test_world_size_must_match_gpus():
    r = _bench("--gpus", "4", "--dry-run", env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0
    assert "--gpus 4 but torchrun started 2 ranks" in r.stderr
