"""Shared fixtures. `-m "not gpu"` runs here (no GPU); `-m gpu` runs on a B200."""
from __future__ import annotations

import os
import sys

import pytest

TESTS = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(TESTS)
for p in (ROOT, TESTS):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running full-size case")


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle():
    """The C restatement (built on demand; a few seconds)."""
    from oracle.pyoracle import LIBS, Checker, build
    if not os.path.exists(LIBS["orc"]):
        build()
    return Checker("orc")


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference headers (oracle/_ref); only where it was built."""
    from oracle.pyoracle import LIBS, Checker
    if not os.path.exists(LIBS["ref"]):
        pytest.skip("oracle/_ref not built (reference tree absent)")
    return Checker("ref")


@pytest.fixture(scope="session")
def srla_lib():
    """libsrla_b200.so, built with nvcc if missing or stale."""
    from paper_1803_10369_b200 import build as b
    b.build()
    from paper_1803_10369_b200.srla import load_library
    return load_library()


@pytest.fixture(scope="session")
def gpu(srla_lib):
    if not gpu_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    return 0
