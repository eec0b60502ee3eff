"""Host-side logic of the Python mirror (no GPU): argument semantics that the
reference enforces before any compute, config mirroring, planning helpers."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import ensure_lib

ensure_lib()
import paper_2106_06161_b200 as bsg  # noqa: E402
from paper_2106_06161_b200 import distributed as D  # noqa: E402


def test_config_defaults_mirror_reference():  # shuffle.hpp:25-30
    c = bsg.ShuffleConfig()
    assert (c.seed, c.variant, c.num_rounds, c.workers) == (0, bsg.BijectionVariant.VariablePhilox, 24, 0)
    assert int(bsg.BijectionVariant.Lcg) == 0 and int(bsg.BijectionVariant.VariablePhilox) == 1
    raw = c._c()
    assert raw.num_rounds == 24 and raw.variant == 1


def test_make_philox_params():  # bijection.hpp:73-88
    p = bsg.make_philox(7, 11)
    assert (p.left_side_bits, p.right_side_bits) == (3, 4)  # unit_bijection.cpp:94-99
    assert p.round_keys == bsg.derive_round_keys(11, 24)
    with pytest.raises(bsg.InvalidArgument):
        bsg.make_philox(1, 0)
    with pytest.raises(bsg.InvalidArgument):
        bsg.make_philox(64, 0)
    with pytest.raises(bsg.InvalidArgument):
        bsg.make_philox(8, 0, 2)


def test_scalar_bijections_roundtrip():  # unit_bijection.cpp:121-156 (host scalar path)
    for bits in range(2, 11):
        p = bsg.make_philox(bits, 1234 + bits)
        img = [bsg.philox_apply(p, x) for x in range(1 << bits)]
        assert sorted(img) == list(range(1 << bits))
        assert all(bsg.philox_invert(p, y) == x for x, y in enumerate(img))
    p = bsg.make_philox(63, 5)
    rng = np.random.default_rng(777)
    for x in rng.integers(0, 2**63, size=2000, dtype=np.uint64):
        assert bsg.philox_invert(p, bsg.philox_apply(p, int(x))) == int(x)
    with pytest.raises(bsg.OutOfRange):
        bsg.philox_apply(bsg.make_philox(8, 7), 256)
    lp = bsg.LcgParams(3, 3, 0)
    assert sorted(bsg.lcg_apply(lp, x) for x in range(8)) == list(range(8))
    with pytest.raises(bsg.OutOfRange):
        bsg.lcg_apply(lp, 8)


def test_compact_permutation():  # unit_shuffle.cpp:14-37
    assert list(bsg.compact_permutation([6, 3, 0, 7, 5, 1, 4, 2], 5)) == [3, 0, 1, 4, 2]
    assert list(bsg.compact_permutation([2, 0, 3, 1], 4)) == [2, 0, 3, 1]
    with pytest.raises(bsg.InvalidArgument):
        bsg.compact_permutation([0, 1], 3)


def test_alias_rejected_before_compute():  # shuffle.hpp:311-312, 356-358
    v = np.arange(5, dtype=np.uint64)
    with pytest.raises(bsg.InvalidArgument):
        bsg.shuffle_values_into(v, bsg.ShuffleConfig(), v)
    with pytest.raises(bsg.InvalidArgument):
        bsg.gather_into(v, np.zeros(2, dtype=np.uint64), v)


def test_transfer_plan_moves_only_boundaries():
    m, world = 1000, 4
    counts = [240, 260, 255, 245]
    plan = D.transfer_plan(counts, m, world)
    for src in range(world):
        assert sum(plan[src]) == counts[src]
    shards = D.equal_shards(m, world)
    for dst in range(world):
        assert sum(plan[src][dst] for src in range(world)) == shards[dst][1] - shards[dst][0]
    moved = sum(plan[s][d] for s in range(world) for d in range(world) if s != d)
    assert moved == 10 + 5  # only the boundary slack crosses ranks
    assert D.offsets_from_counts(counts, 2) == 500


def test_philox_params_path_matches_reference_kats(golden):
    """philox_apply/philox_invert over caller-held params (bsg_philox_*_params) reproduce every reference KAT
    (widths 2..63, rounds 3..100) -- the path the C++ shim and this mirror use."""
    cache = {}
    for bits, seed, rounds, x, y in golden["philox_apply"]:
        p = cache.setdefault((bits, seed, rounds), bsg.make_philox(bits, seed, rounds))
        assert bsg.philox_apply(p, x) == y
    for bits, seed, rounds, y, x in golden["philox_invert"]:
        p = cache.setdefault((bits, seed, rounds), bsg.make_philox(bits, seed, rounds))
        assert bsg.philox_invert(p, y) == x


def test_caller_built_philox_params():  # unit_bijection.cpp:106-115, 138-147
    p = bsg.VariablePhiloxParams(total_bits=8, left_side_bits=4, right_side_bits=4, num_rounds=0,
                                 left_side_mask=0xF, right_side_mask=0xF)
    assert bsg.philox_apply(p, 0b10110011) == 0b10110011
    q = bsg.VariablePhiloxParams(6, 3, 3, 0, 0x7, 0x7)
    assert bsg.philox_invert(q, 0b101101) == 0b101101
    r = bsg.make_philox(20, 99)
    y = bsg.philox_apply(r, 12345)
    r.round_keys[3] ^= 1
    y2 = bsg.philox_apply(r, 12345)
    assert y2 != y and bsg.philox_invert(r, y2) == 12345
    r.num_rounds = 40  # more rounds than keys
    with pytest.raises(bsg.InvalidArgument):
        bsg.philox_apply(r, 1)


def test_bijection_spec_and_splitmix():  # bijection.hpp:146-169, splitmix.hpp:35-63
    lcg = bsg.make_bijection(bsg.LcgParams(4, 1, 0))
    assert lcg.domain_bits == 4 and bsg.bijection_apply(lcg, 9) == 9
    with pytest.raises(bsg.OutOfRange):
        bsg.bijection_apply(lcg, 16)
    ph = bsg.make_bijection(bsg.make_philox(8, 7))
    assert ph.domain_bits == 8 and sorted(bsg.bijection_apply(ph, x) for x in range(256)) == list(range(256))
    g = bsg.SplitMix64(777)
    assert g() == bsg.mix64((777 + 0x9E3779B97F4A7C15) & (2**64 - 1))
    assert all(g.below(7) < 7 for _ in range(100))
    with pytest.raises(bsg.InvalidArgument):
        g.below(0)


def test_bench_checksum_matches_fixture_definition():
    """bench.py's GPU-side output checksum (run here on CPU tensors) equals the generator's numpy definition,
    for u64 indices, u32 rows and 16-byte records (tests/golden/make_bench_checksums.py)."""
    import json
    import os
    import sys

    import torch
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "tests", "golden"))
    import bench
    import make_bench_checksums as G
    perm = np.random.default_rng(5).permutation(1 << 16).astype(np.uint64)
    s, ws = bench.output_checksum(torch, torch.from_numpy(perm.view(np.int64)), first_word=0)
    assert (int(s) & (2**64 - 1), int(ws) & (2**64 - 1)) == G.checksum_words(lambda lo, hi: perm[lo:hi], perm.size)
    rows = perm.astype(np.uint32).reshape(64, -1)
    s, ws = bench.output_checksum(torch, torch.from_numpy(rows.view(np.int32)))
    flat = rows.reshape(-1).astype(np.uint64)
    assert (int(s) & (2**64 - 1), int(ws) & (2**64 - 1)) == G.checksum_words(lambda lo, hi: flat[lo:hi], flat.size)
    rec = np.stack([perm * np.uint64(2), perm * np.uint64(2) + np.uint64(1)], axis=1).reshape(-1)
    s, ws = bench.output_checksum(torch, torch.from_numpy(rec.view(np.int64)).view(torch.complex128))
    assert (int(s) & (2**64 - 1), int(ws) & (2**64 - 1)) == G.checksum_words(lambda lo, hi: rec[lo:hi], rec.size)
    cfgs = json.load(open(os.path.join(root, "tests", "golden", "bench_checksums.json")))["configs"]
    for k in ("c1@1", "c2@1", "c2@8", "c3@1", "c3@8", "c2lcg@1", "c3lcg@1", "c5@1", "c4@rank0", "c4@rank7"):
        assert k in cfgs and len(cfgs[k]["wsum"]) == 16
