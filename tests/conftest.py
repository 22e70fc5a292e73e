"""Shared pytest configuration.

`-m gpu` tests need a B200 (run under gpurun); everything else runs on CPU.
The CPU oracle (oracle/, test infrastructure only) is loaded from
oracle/build/ and built on demand with `make -C oracle`.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_BUILD = os.path.join(ROOT, "oracle", "build")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def load_oracle():
    if ORACLE_BUILD not in sys.path:
        sys.path.insert(0, ORACLE_BUILD)
    try:
        import _oracle  # noqa: F401
    except ImportError:
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
        import _oracle  # noqa: F401
    return sys.modules["_oracle"]


@pytest.fixture(scope="session")
def oracle():
    return load_oracle()
