"""The C++ drop-in shim (include/bijshuf_gpu/shuffle.hpp): compiles on CPU hosts;
runs the reference's unit-test cases on the GPU."""
from __future__ import annotations

import os
import subprocess

import pytest

from conftest import ROOT, ensure_lib

SRC = os.path.join(ROOT, "tests", "cpp", "test_shim.cpp")
BIN = os.path.join(ROOT, "build", "test_shim")


def build_shim() -> str:
    lib = ensure_lib()
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    libdir = os.path.dirname(lib)
    subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"), SRC, "-L", libdir,
                    "-lbsg", f"-Wl,-rpath,{libdir}", "-o", BIN], check=True)
    return BIN


def test_shim_compiles():
    build_shim()
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_shim_reference_unit_cases_on_gpu():
    b = build_shim()
    r = subprocess.run([b], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "all checks passed" in r.stdout
