"""The C++ drop-in shim (include/bijshuf_gpu/shuffle.hpp): compiles on CPU hosts;
runs the reference's unit-test cases on the GPU."""
from __future__ import annotations

import os
import subprocess

import pytest

from conftest import ROOT, ensure_lib

SRC = os.path.join(ROOT, "tests", "cpp", "test_shim.cpp")
BIN = os.path.join(ROOT, "build", "test_shim")
SRC_BIJ = os.path.join(ROOT, "tests", "cpp", "test_shim_bijection.cpp")
BIN_BIJ = os.path.join(ROOT, "build", "test_shim_bijection")


def build_shim(src: str = SRC, binary: str = BIN) -> str:
    lib = ensure_lib()
    os.makedirs(os.path.dirname(binary), exist_ok=True)
    libdir = os.path.dirname(lib)
    subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), src, "-L",
                    libdir, "-lbsg", f"-Wl,-rpath,{libdir}", "-o", binary], check=True)
    return binary


def test_shim_compiles():
    build_shim()
    assert os.path.exists(BIN)


def test_shim_reference_unit_bijection_cases():
    """Every case of the reference's unit_bijection.cpp through the shim (host scalar entry points, no GPU)."""
    b = build_shim(SRC_BIJ, BIN_BIJ)
    r = subprocess.run([b], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "all checks passed" in r.stdout


@pytest.mark.gpu
def test_shim_reference_unit_cases_on_gpu():
    b = build_shim()
    r = subprocess.run([b], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "all checks passed" in r.stdout
