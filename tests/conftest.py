"""Shared fixtures.  `-m gpu` tests need a B200 and the built libbsg.so; the
rest run on CPU (oracle pinning, C-ABI symbol table, host logic, gloo)."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

LIB = os.path.join(ROOT, "paper_2106_06161_b200", "lib", "libbsg.so")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libbsg.so")
    config.addinivalue_line("markers", "slow: long-running (full-size) parity checks")


def ensure_lib() -> str:
    """Build libbsg.so if it is missing (nvcc cross-compiles without a GPU)."""
    if not os.path.exists(LIB):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2106_06161_b200", "csrc"), "-j8"], check=True,
                       stdout=subprocess.DEVNULL)
    return LIB


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(ROOT, "tests", "golden", "golden_ref.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle


@pytest.fixture(scope="session")
def bsg():
    ensure_lib()
    import paper_2106_06161_b200 as b
    return b


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a CUDA device (run with -m 'not gpu' on CPU hosts)")
    return torch
