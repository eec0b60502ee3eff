"""C ABI checks that need no GPU: the library loads, exports every symbol of
include/bsg.h, and its host-side logic (key schedule, parameter derivation,
scalar bijections, partitioning, error semantics) matches the reference."""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, ensure_lib

HEADER = os.path.join(ROOT, "include", "bsg.h")


@pytest.fixture(scope="module")
def so():
    ensure_lib()
    from paper_2106_06161_b200 import _lib
    return _lib


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*[\w\s\*]+?\b(bsg_\w+)\s*\(", text, flags=re.M)) - {"bsg_allgather_u64_fn"})


def test_exports_every_declared_symbol(so):
    syms = declared_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(so.lib, s), s
    assert set(syms) == set(so.SIGNATURES), set(syms) ^ set(so.SIGNATURES)


def test_exports_only_the_abi(so):
    out = os.popen(f"nm -D --defined-only {so.LIB_PATH}").read().split()
    names = [w for w in out if w.startswith("bsg_")]
    assert set(names) == set(declared_symbols())


def test_key_schedule_and_mix(so, golden):
    for case in golden["round_keys"]:
        k = (ctypes.c_uint32 * case["rounds"])()
        assert so.lib.bsg_derive_round_keys(case["seed"], case["rounds"], k) == 0
        assert list(k) == case["keys"]
    assert so.lib.bsg_derive_round_keys(1, 0, (ctypes.c_uint32 * 1)()) == so.EINVAL
    import oracle as O
    for z in [0, 1, 42, 2**63, 2**64 - 1]:
        assert so.lib.bsg_mix64(z) == O.C.orc_mix64(z)


def test_make_lcg_and_apply(so, golden):
    a, c = ctypes.c_uint64(), ctypes.c_uint64()
    for case in golden["make_lcg"]:
        assert so.lib.bsg_make_lcg(case["bits"], case["seed"], ctypes.byref(a), ctypes.byref(c)) == 0
        assert (a.value, c.value) == (case["a"], case["c"])
    for bad in (0, 64):
        assert so.lib.bsg_make_lcg(bad, 1, ctypes.byref(a), ctypes.byref(c)) == so.EINVAL
    y = ctypes.c_uint64()
    assert so.lib.bsg_lcg_apply(3, 3, 1, 5, ctypes.byref(y)) == 0 and y.value == 0  # unit_bijection.cpp:67-70
    assert so.lib.bsg_lcg_apply(3, 3, 0, 8, ctypes.byref(y)) == so.ERANGE


def test_host_philox_matches_reference_fixtures(so, golden):
    y = ctypes.c_uint64()
    for bits, seed, rounds, x, yy in golden["philox_apply"]:
        assert so.lib.bsg_philox_apply(bits, seed, rounds, x, ctypes.byref(y)) == 0
        assert y.value == yy, (bits, seed, rounds, x)
    for bits, seed, rounds, yy, x in golden["philox_invert"]:
        assert so.lib.bsg_philox_invert(bits, seed, rounds, yy, ctypes.byref(y)) == 0
        assert y.value == x


def test_host_philox_errors(so):  # bijection.hpp:75-78, 96-97
    y = ctypes.c_uint64()
    assert so.lib.bsg_philox_apply(1, 0, 24, 0, ctypes.byref(y)) == so.EINVAL
    assert so.lib.bsg_philox_apply(64, 0, 24, 0, ctypes.byref(y)) == so.EINVAL
    assert so.lib.bsg_philox_apply(8, 0, 2, 0, ctypes.byref(y)) == so.EINVAL
    assert so.lib.bsg_philox_apply(8, 7, 24, 256, ctypes.byref(y)) == so.ERANGE
    assert so.lib.bsg_philox_invert(8, 7, 24, 256, ctypes.byref(y)) == so.ERANGE


def test_domain_bits(so):
    for m, b in [(2, 4), (3, 4), (16, 4), (17, 5), (1000, 10), (1024, 10), (1025, 11), (2**33, 33), (2**33 + 1, 34)]:
        assert so.lib.bsg_domain_bits(m) == b


def test_counter_partition_covers_domain(so):
    b, e = ctypes.c_uint64(), ctypes.c_uint64()
    for m in (5, 1000, 2**29, 2**29 + 1, 2**33):
        n = 1 << so.lib.bsg_domain_bits(m)
        for world in (1, 2, 3, 7, 8):
            prev = 0
            for r in range(world):
                assert so.lib.bsg_dist_counter_range(m, r, world, ctypes.byref(b), ctypes.byref(e)) == 0
                assert b.value == prev and e.value >= b.value
                prev = e.value
            assert prev == n
    assert so.lib.bsg_dist_counter_range(1000, 3, 3, ctypes.byref(b), ctypes.byref(e)) == so.EINVAL


def test_status_strings(so):
    for s in range(8):
        assert so.lib.bsg_status_string(s)
    assert so.lib.bsg_config_default().num_rounds == 24 and so.lib.bsg_config_default().variant == 1


def test_no_cpu_fallback_without_gpu(so):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2106_06161_b200 as bsg
    with pytest.raises(bsg.CudaError):
        bsg.shuffle_indices(1000)
    with pytest.raises(bsg.CudaError):
        bsg.shuffle_values(np.arange(100, dtype=np.uint64))
    with pytest.raises(bsg.CudaError):
        bsg.gather(np.arange(10, dtype=np.uint64), np.zeros(3, dtype=np.uint64))
