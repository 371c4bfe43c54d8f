"""Test configuration.

Markers:
  gpu — needs a CUDA device (run on the B200 box: pytest -m gpu). Everything else runs on
        CPU: the oracle against the reference's golden vectors, the host-side logic of the
        C ABI, the glibc-log port, the GF(2) seeding algebra and the multi-rank (gloo) path.
"""
import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLD = Path(__file__).resolve().parent / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200)")


def golden(name: str):
    return json.loads((GOLD / name).read_text())


def unhex(xs):
    return [float.fromhex(x) for x in xs]


@pytest.fixture(scope="session")
def gpu():
    import paper_1501_01405_b200 as w

    try:
        n = w.device_count()
    except w.Error as e:  # pragma: no cover - only on a box without a usable GPU
        pytest.fail(f"no usable CUDA device: {e}")
    assert n >= 1
    return w


@pytest.fixture(scope="session")
def ref():
    import oracle

    if not oracle.available("reference"):
        pytest.skip("oracle/_ref not built")
    return oracle.Oracle("reference")


@pytest.fixture(scope="session")
def port():
    import oracle

    if not oracle.available("port"):
        oracle.build()
    return oracle.Oracle("port")
