"""Pin the C oracle (oracle/bijshuf_oracle.c) to the reference.

Sources of truth, in order:
  * the reference's own frozen values (proj/tests/unit_bijection.cpp:32-37
    round keys, :52-84 LCG arithmetic, unit_shuffle.cpp:14-46 compaction and
    domain bits);
  * tests/golden/golden_ref.json, produced by running the reference itself
    (oracle/_ref, see tests/golden/make_golden.py);
  * when oracle/_ref is present, a live comparison on fresh random cases.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import pytest

import oracle as O

PHILOX, LCG = O.PHILOX, O.LCG


def test_round_keys_golden_seed42():  # unit_bijection.cpp:32-37
    assert list(O.keys(42, 4)) == [0x2FEB6E95, 0xB266F103, 0x130F9F52, 0x0E4AE394]


def test_round_keys_fixtures(golden):
    for case in golden["round_keys"]:
        assert list(O.keys(case["seed"], case["rounds"])) == case["keys"]


def test_derive_round_keys_rejects_zero():  # unit_bijection.cpp:39-41
    k = (ctypes.c_uint32 * 1)()
    assert O.C.orc_derive_round_keys(1, 0, k) == -1


def test_mix64_reference_points():  # unit_bijection.cpp:13-16 against oracles.hpp ref_mix64
    def ref(z):
        M = (1 << 64) - 1
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)
    for z in [0, 1, 42, 0xDEADBEEF, (1 << 64) - 1]:
        assert O.C.orc_mix64(z) == ref(z)


def test_lcg_known_answers():  # unit_bijection.cpp:43-84
    y = ctypes.c_uint64()
    assert O.C.orc_lcg_apply(3, 3, 0, 1, ctypes.byref(y)) == 0 and y.value == 3
    assert O.C.orc_lcg_apply(4, 1, 0, 9, ctypes.byref(y)) == 0 and y.value == 9
    assert O.C.orc_lcg_apply(3, 3, 1, 5, ctypes.byref(y)) == 0 and y.value == 0
    assert O.C.orc_lcg_apply(3, 3, 0, 8, ctypes.byref(y)) == -2
    img = set()
    for x in range(8):
        O.C.orc_lcg_apply(3, 3, 0, x, ctypes.byref(y))
        img.add(y.value)
    assert img == set(range(8))
    for seed in range(200):
        a, c = O.make_lcg(16, seed)
        assert a & 1 and a < (1 << 16) and c < (1 << 16)
    for bad in (0, 64):
        with pytest.raises(ValueError):
            O.make_lcg(bad, 1)


def test_make_lcg_fixtures(golden):
    for case in golden["make_lcg"]:
        assert O.make_lcg(case["bits"], case["seed"]) == (case["a"], case["c"])


def test_philox_apply_fixtures(golden):
    for bits, seed, rounds, x, y in golden["philox_apply"]:
        assert O.philox_apply(bits, seed, rounds, x) == y, (bits, seed, rounds, x)


def test_philox_invert_fixtures(golden):
    for bits, seed, rounds, y, x in golden["philox_invert"]:
        assert O.philox_invert(bits, seed, rounds, y) == x, (bits, seed, rounds, y)


def test_philox_bijective_and_invertible_small():  # unit_bijection.cpp:86-135
    for bits in range(2, 13):
        seed = 1234 + bits
        img = [O.philox_apply(bits, seed, 24, x) for x in range(1 << bits)]
        assert sorted(img) == list(range(1 << bits))
        assert all(O.philox_invert(bits, seed, 24, y) == x for x, y in enumerate(img))


def test_philox_rejects_bad_parameters():  # unit_bijection.cpp:171-175
    k = O.keys(0, 24)
    y = ctypes.c_uint64()
    assert O.C.orc_philox_apply(8, k, 24, 256, ctypes.byref(y)) == -2  # out of domain
    for bits, rounds in [(1, 24), (64, 24), (8, 2)]:
        m = 1 << min(bits, 4) | 3
        out = np.empty(m, dtype=np.uint64)  # room for every survivor the call may write
        assert O.C.orc_shuffle_indices(m, 0, PHILOX, rounds, out.ctypes.data) in (0, -1)
    out = np.empty(100, dtype=np.uint64)
    assert O.C.orc_shuffle_indices(100, 0, PHILOX, 2, out.ctypes.data) == -1


def test_domain_bits_table():  # unit_shuffle.cpp:39-46
    for m, bits in [(3, 4), (16, 4), (17, 5), (1000, 10), (1024, 10), (1025, 11)]:
        assert O.C.orc_domain_bits(m) == bits


def test_trivial_sizes():  # unit_shuffle.cpp:48-65
    assert list(O.shuffle_indices(1)) == [0]
    assert len(O.shuffle_indices(0)) == 0
    seen = set()
    for seed in range(32):
        p = tuple(O.shuffle_indices(2, seed))
        assert p in ((0, 1), (1, 0))
        assert p[0] == O.C.orc_mix64(seed) & 1
        seen.add(p)
    assert len(seen) == 2


def test_indices_full_fixtures(golden):
    for case in golden["indices_full"]:
        p = O.shuffle_indices(case["m"], case["seed"], case["variant"], case["rounds"])
        assert [int(v) for v in p] == case["perm"], case["m"]


def test_indices_hash_fixtures(golden):
    for case in golden["indices_hash"]:
        p = O.shuffle_indices(case["m"], case["seed"], case["variant"], case["rounds"])
        assert f"{O.fnv1a64(p):016x}" == case["fnv"], case
        assert [int(v) for v in p[:8]] == case["head"]


def _values_input(m, eb):
    raw = (np.arange(m * eb, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)).astype(np.uint8)
    return raw.reshape(m, eb)


def _fnv_bytes(a):
    b = np.ascontiguousarray(a).tobytes()
    b += bytes((-len(b)) % 8)
    return f"{O.fnv1a64(np.frombuffer(b, dtype=np.uint64)):016x}"


def test_values_hash_fixtures(golden):
    for case in golden["values_hash"]:
        raw = _values_input(case["m"], case["elem_bytes"])
        out = O.shuffle_values(raw, case["seed"], case["variant"], case["rounds"])
        assert _fnv_bytes(out) == case["fnv_bytes"], case


def test_batched_fixtures(golden):
    for case in golden["batched"]:
        for row in case["rows"]:
            p = O.shuffle_indices(case["m"], case["seed"] + row["b"], case["variant"], case["rounds"])
            assert f"{O.fnv1a64(p):016x}" == row["fnv"]


def test_range_concatenation_is_the_shuffle():
    m = 5000
    full = O.shuffle_indices(m, 9)
    n = 1 << O.C.orc_domain_bits(m)
    cuts = [0, 1, 777, 4096, 4097, n]
    parts = [O.shuffle_indices_range(m, 9, PHILOX, 24, a, b) for a, b in zip(cuts, cuts[1:])]
    assert np.array_equal(np.concatenate(parts), full)


@pytest.mark.skipif(O.REF is None, reason="oracle/_ref not built (needs /root/reference)")
def test_live_against_reference():
    rng = np.random.default_rng(7)
    for _ in range(40):
        m = int(rng.integers(3, 200000))
        seed = int(rng.integers(0, 2**64, dtype=np.uint64))
        variant = int(rng.integers(0, 2))
        rounds = int(rng.choice([3, 7, 12, 24, 40]))
        assert np.array_equal(O.shuffle_indices(m, seed, variant, rounds),
                              O.ref_shuffle_indices(m, seed, variant, rounds)), (m, seed, variant, rounds)


@pytest.mark.skipif(O.REF is None, reason="oracle/_ref not built (needs /root/reference)")
def test_reference_worker_independence():  # unit_shuffle.cpp:96-107 via the reference itself
    m = (1 << 18) + 12345
    base = O.ref_shuffle_indices(m, 17, PHILOX, 24, workers=1)
    for w in (2, 8, 0):
        assert np.array_equal(O.ref_shuffle_indices(m, 17, PHILOX, 24, workers=w), base)
    assert np.array_equal(O.shuffle_indices(m, 17), base)


@pytest.mark.slow
@pytest.mark.skipif(not os.environ.get("BSG_SLOW"), reason="set BSG_SLOW=1 (needs ~20 GB RAM, minutes)")
def test_values_full_hash_fixtures(golden):
    for case in golden["values_full_hash"]:
        vals = np.arange(case["m"], dtype=np.uint64)
        out = O.shuffle_values(vals, case["seed"], case["variant"], case["rounds"])
        assert f"{O.fnv1a64(out):016x}" == case["fnv"]
