"""Test configuration.

Markers: ``gpu`` tests need a B200 (run on the GPU box with ``-m gpu``); the
rest run on CPU (``-m "not gpu"``).  The CPU oracles in oracle/ are test
infrastructure: tests use them as the checker, never as the thing tested.
"""
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 (B200) GPU")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Port
    return Port()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Reference, available_reference
    if not available_reference():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Reference()


@pytest.fixture(scope="session")
def golden():
    import json
    return json.loads((GOLDEN / "shift_golden.json").read_text())


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test collected without a CUDA device")
    return torch.device("cuda:0")
