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
