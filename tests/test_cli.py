"""bijshuf-cli-compatible front end (proj/tools/bijshuf_cli.cpp): exit codes,
JSON report and the bench CSV schema (bench.hpp:209-241); mirrors
acceptance.cpp:310-371."""
from __future__ import annotations

import io
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
from conftest import ROOT, ensure_lib


def cli(*args, inp=None):
    ensure_lib()
    return subprocess.run([sys.executable, "-m", "paper_2106_06161_b200.cli", *args], cwd=ROOT, capture_output=True,
                          text=True, input=inp, timeout=600)


def test_usage_errors_exit_2():
    assert cli().returncode == 2
    assert cli("test").returncode == 2  # --kind required
    assert cli("test", "--kind", "nope").returncode == 2
    assert cli("shuffle").returncode == 2
    assert cli("bench", "--format", "xml").returncode == 2


def test_csv_writer_roundtrip():
    from paper_2106_06161_b200 import cli as C
    recs = [{"algorithm": "bijective", "input_size": 257, "trials": 5, "runtime_s": 1.25e-05,
             "throughput_mitems_s": 20.56}]
    f = io.StringIO()
    C.write_csv(f, recs)
    lines = f.getvalue().splitlines()
    assert lines[0] == "algorithm,input_size,trials,runtime_s,throughput_mitems_s"
    alg, size, trials, rt, tp = lines[1].split(",")
    assert (alg, int(size), int(trials), float(rt), float(tp)) == ("bijective", 257, 5, 1.25e-05, 20.56)
    assert C.default_bench_sizes()[0] == 257 and C.default_bench_sizes()[-1] == (1 << 26) + 1


@pytest.mark.gpu
def test_cli_shuffle_and_test_and_bench():
    r = cli("shuffle", "--indices", "1000", "--seed", "7")
    assert r.returncode == 0
    assert [int(x) for x in r.stdout.split()] == [int(v) for v in O.shuffle_indices(1000, 7)]
    r = cli("shuffle", "-", "--seed", "3", inp="".join(f"line{i}\n" for i in range(100)))
    assert r.returncode == 0 and sorted(r.stdout.split()) == sorted(f"line{i}" for i in range(100))
    assert r.stdout.split() == [f"line{int(i)}" for i in O.shuffle_indices(100, 3)]
    good = cli("test", "--kind", "chi2", "--gen", "philox", "--rounds", "24", "--samples", "100000")
    assert good.returncode == 0 and json.loads(good.stdout)["pass"] is True
    bad = cli("test", "--kind", "chi2", "--gen", "lcg", "--samples", "100000")
    assert bad.returncode == 1 and json.loads(bad.stdout)["pass"] is False
    fy = cli("test", "--kind", "mmd-normal", "--gen", "fisher-yates", "--n", "100", "--samples", "10000")  # acceptance.cpp:347-349
    assert fy.returncode == 0, fy.stdout + fy.stderr
    b = cli("bench", "--sizes", "1025,65537", "--trials", "2")
    assert b.returncode == 0
    lines = b.stdout.splitlines()
    assert lines[0] == "algorithm,input_size,trials,runtime_s,throughput_mitems_s" and len(lines) == 7
