"""GPU parity: the sm_100a kernels through the C ABI against the oracle and the
reference-generated fixtures.  Bit-exact throughout (integer/index work)."""
from __future__ import annotations

import ctypes

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

PHILOX, LCG = O.PHILOX, O.LCG


def cfg_of(bsg, seed=0, variant=PHILOX, rounds=24, workers=0):
    return bsg.ShuffleConfig(seed=seed, variant=bsg.BijectionVariant(variant), num_rounds=rounds, workers=workers)


def gpu_indices(bsg, cuda, m, **kw):
    t = bsg.shuffle_indices(m, cfg_of(bsg, **kw), device="cuda")
    return t.cpu().numpy().view(np.uint64)


# ------------------------------------------------------------ bijections --
def test_bijection_apply_matches_fixtures(bsg, cuda, golden):
    by = {}
    for bits, seed, rounds, x, y in golden["philox_apply"]:
        by.setdefault((bits, seed, rounds), []).append((x, y))
    for (bits, seed, rounds), xy in by.items():
        xs = np.array([a for a, _ in xy], dtype=np.uint64)
        ys = np.array([b for _, b in xy], dtype=np.uint64)
        got = bsg.bijection_apply(bsg.BijectionVariant.VariablePhilox, bits, seed, rounds, xs)
        assert np.array_equal(got, ys), (bits, seed, rounds)
        back = bsg.bijection_apply(bsg.BijectionVariant.VariablePhilox, bits, seed, rounds, ys, inverse=True)
        assert np.array_equal(back, xs), (bits, seed, rounds)


def test_bijection_apply_exhaustive_widths(bsg, cuda):
    for bits in range(2, 23):
        for variant in (PHILOX, LCG):
            n = 1 << bits
            x = cuda.arange(n, dtype=cuda.int64, device="cuda")
            y = bsg.bijection_apply(bsg.BijectionVariant(variant), bits, 0xABC + bits, 24, x)
            yn = y.cpu().numpy().view(np.uint64)
            assert np.array_equal(np.sort(yn), np.arange(n, dtype=np.uint64)), (bits, variant)
            if variant == PHILOX:
                idx = np.linspace(0, n - 1, 64).astype(np.uint64)
                exp = [O.philox_apply(bits, 0xABC + bits, 24, int(i)) for i in idx]
                assert np.array_equal(yn[idx.astype(np.int64)], np.array(exp, dtype=np.uint64))
            inv = bsg.bijection_apply(bsg.BijectionVariant(variant), bits, 0xABC + bits, 24, y, inverse=True)
            assert cuda.equal(inv, x)


def test_bijection_apply_counter_mode_wide(bsg, cuda):
    for bits in (33, 40, 47, 63):
        start = (1 << bits) - 5000
        y = bsg.bijection_apply(bsg.BijectionVariant.VariablePhilox, bits, 77, 24, None, start=start, n=5000)
        exp = np.array([O.philox_apply(bits, 77, 24, start + i) for i in range(0, 5000, 97)], dtype=np.uint64)
        assert np.array_equal(y[::97], exp)


def test_bijection_apply_rejects_out_of_domain(bsg, cuda):
    with pytest.raises(bsg.OutOfRange):
        bsg.bijection_apply(bsg.BijectionVariant.VariablePhilox, 8, 7, 24, np.array([256], dtype=np.uint64))


# -------------------------------------------------------------- indices --
def test_indices_full_fixtures(bsg, cuda, golden):
    for case in golden["indices_full"]:
        got = gpu_indices(bsg, cuda, case["m"], seed=case["seed"], variant=case["variant"], rounds=case["rounds"])
        assert [int(v) for v in got] == case["perm"], case["m"]


def test_indices_hash_fixtures(bsg, cuda, golden):
    for case in golden["indices_hash"]:
        got = gpu_indices(bsg, cuda, case["m"], seed=case["seed"], variant=case["variant"], rounds=case["rounds"])
        assert f"{O.fnv1a64(got):016x}" == case["fnv"], case
        assert [int(v) for v in got[:8]] == case["head"]


def test_indices_exhaustive_small_sizes(bsg, cuda):
    for m in range(0, 2200):
        for variant, seed in ((PHILOX, m * 31 + 1), (LCG, m)):
            got = gpu_indices(bsg, cuda, m, seed=seed, variant=variant)
            exp = O.shuffle_indices(m, seed, variant, 24)
            assert np.array_equal(got, exp), (m, variant)


def test_indices_pow2_boundaries(bsg, cuda):
    for k in range(4, 25):
        for m in ((1 << k) - 1, 1 << k, (1 << k) + 1):
            for variant in (PHILOX, LCG):
                got = gpu_indices(bsg, cuda, m, seed=k, variant=variant)
                assert np.array_equal(got, O.shuffle_indices(m, k, variant, 24)), (m, variant)


def test_generic_round_counts(bsg, cuda):
    for rounds in (3, 4, 7, 12, 23, 25, 31, 32, 33, 64, 100):
        for m in (1000, 4096, 70001):
            got = gpu_indices(bsg, cuda, m, seed=rounds, rounds=rounds)
            assert np.array_equal(got, O.shuffle_indices(m, rounds, PHILOX, rounds)), (m, rounds)


def test_force_compact_equals_pow2_path(bsg, cuda):
    for m in (16, 1 << 12, 1 << 20, 1 << 23):
        base = gpu_indices(bsg, cuda, m, seed=3)
        old = bsg.set_force_compact(True)
        try:
            comp = gpu_indices(bsg, cuda, m, seed=3)
        finally:
            bsg.set_force_compact(old)
        assert np.array_equal(base, comp), m


def test_host_pointer_path_and_workers(bsg, cuda):
    m = (1 << 18) + 12345  # unit_shuffle.cpp:96-107
    exp = O.shuffle_indices(m, 17)
    for w in (1, 2, 8, 0):
        got = bsg.shuffle_indices(m, cfg_of(bsg, seed=17, workers=w))  # numpy (host) output
        assert np.array_equal(got, exp)


def test_determinism_acceptance_case(bsg, cuda):  # acceptance.cpp:232-244
    a = gpu_indices(bsg, cuda, 1000001, seed=7)
    b = gpu_indices(bsg, cuda, 1000001, seed=7)
    assert np.array_equal(a, b) and O.is_valid_permutation(a)
    assert np.array_equal(a, O.shuffle_indices(1000001, 7))


def test_invalid_arguments(bsg, cuda):
    with pytest.raises(bsg.InvalidArgument):
        bsg.shuffle_indices(100, cfg_of(bsg, rounds=2))
    # m <= 2 never validates (shuffle.hpp:228-240)
    assert list(bsg.shuffle_indices(2, cfg_of(bsg, rounds=0, seed=5))) == [O.C.orc_mix64(5) & 1,
                                                                           (O.C.orc_mix64(5) & 1) ^ 1]
    v = np.arange(10, dtype=np.uint64)
    with pytest.raises(bsg.InvalidArgument):
        bsg.shuffle_values_into(v, cfg_of(bsg), v)
    t = cuda.arange(10, device="cuda")
    with pytest.raises(bsg.InvalidArgument):
        bsg.shuffle_values_into(t, cfg_of(bsg), t)


# --------------------------------------------------------------- values --
def _values_input(m, eb):
    raw = (np.arange(m * eb, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)).astype(np.uint8)
    return raw.reshape(m, eb)


def _fnv_bytes(a):
    b = np.ascontiguousarray(a).tobytes()
    b += bytes((-len(b)) % 8)
    return f"{O.fnv1a64(np.frombuffer(b, dtype=np.uint64)):016x}"


def test_values_fixtures_all_element_sizes(bsg, cuda, golden):
    for case in golden["values_hash"]:
        raw = _values_input(case["m"], case["elem_bytes"])
        eb = case["elem_bytes"]
        dt = {1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}.get(eb)
        if dt is not None:
            arr = raw.view(dt).reshape(case["m"])
        else:
            arr = raw.view(np.dtype((np.void, eb))).reshape(case["m"])
        cfg = cfg_of(bsg, seed=case["seed"], variant=case["variant"], rounds=case["rounds"])
        out = bsg.shuffle_values(arr, cfg)  # host path
        assert _fnv_bytes(out) == case["fnv_bytes"], case
        if dt is not None or eb == 16:
            td = cuda.from_numpy(raw.copy()).cuda()  # (m, eb) uint8 device tensor
            if eb in (2, 4, 8):
                td = td.view({2: cuda.int16, 4: cuda.int32, 8: cuda.int64}[eb]).reshape(case["m"])
            elif eb == 16:
                td = td.view(cuda.int64).reshape(case["m"], 2)
            else:
                td = td.reshape(case["m"])
            od = cuda.empty_like(td)
            bsg.shuffle_values_into(td, cfg, od) if eb != 16 else _values16(bsg, td, od, cfg)
            cuda.cuda.synchronize()
            assert _fnv_bytes(od.cpu().numpy()) == case["fnv_bytes"], case


def _values16(bsg, td, od, cfg):
    from paper_2106_06161_b200 import _lib
    _lib.check(_lib.lib.bsg_shuffle_values(td.data_ptr(), od.data_ptr(), td.shape[0], 16,
                                           ctypes.byref(cfg._c()), None), "values16")


def test_values_match_indices(bsg, cuda):  # unit_shuffle.cpp:137-148
    m = 70000
    vals = cuda.arange(m, dtype=cuda.int64, device="cuda") * 3 + 1
    out = bsg.shuffle_values(vals, cfg_of(bsg, seed=31))
    perm = bsg.shuffle_indices(m, cfg_of(bsg, seed=31), device="cuda")
    assert cuda.equal(out, vals[perm])


def test_values_into_reuse_and_trivial(bsg, cuda):  # unit_shuffle.cpp:205-221
    for m in (1000, 70000, 17, 2, 1, 0):
        vals = (np.arange(m, dtype=np.uint64) * 7 + 3)
        out = bsg.shuffle_values(vals, cfg_of(bsg, seed=21))
        assert np.array_equal(out, O.shuffle_values(vals, 21)) if m else len(out) == 0


def test_values_full_size_hashes(bsg, cuda, golden):
    """The bench workload itself (2^29 u64) and the worst-case padding sizes, vs the reference run."""
    for case in golden["values_full_hash"]:
        m = case["m"]
        vals = cuda.arange(m, dtype=cuda.int64, device="cuda")
        out = bsg.shuffle_values(vals, cfg_of(bsg, seed=case["seed"], variant=case["variant"],
                                              rounds=case["rounds"]))
        host = out.cpu().numpy().view(np.uint64)
        del vals, out
        assert f"{O.fnv1a64(host):016x}" == case["fnv"], case
        cuda.cuda.empty_cache()


# --------------------------------------------------------------- ranges --
def test_range_concatenation(bsg, cuda):
    from paper_2106_06161_b200 import _lib
    for m, variant in ((5000, PHILOX), ((1 << 20) + 3, PHILOX), ((1 << 20) + 3, LCG), (1 << 16, PHILOX)):
        cfg = cfg_of(bsg, seed=9, variant=variant)._c()
        n = 1 << O.C.orc_domain_bits(m)
        cuts = [0, 1, 777, 4096, 4097, n // 2 + 13, n]
        pieces = []
        for a, b in zip(cuts, cuts[1:]):
            out = cuda.empty(max(b - a, 1), dtype=cuda.int64, device="cuda")
            cnt = ctypes.c_uint64()
            _lib.check(_lib.lib.bsg_shuffle_range(m, ctypes.byref(cfg), a, b, None, None, out.data_ptr(), 8,
                                                  ctypes.addressof(cnt), None), "range")
            c2 = ctypes.c_uint64()
            _lib.check(_lib.lib.bsg_range_count(m, ctypes.byref(cfg), a, b, ctypes.byref(c2), None), "count")
            assert cnt.value == c2.value
            pieces.append(out[:cnt.value].cpu().numpy().view(np.uint64))
        assert np.array_equal(np.concatenate(pieces), O.shuffle_indices(m, 9, variant, 24)), m


def test_wide_domain_ranges(bsg, cuda):
    """bits > 32 (64-bit counters): indices and u8 payload on slices of the 2^33 domain."""
    from paper_2106_06161_b200 import _lib
    m = (1 << 32) + 5
    cfg = cfg_of(bsg, seed=0x5EED)._c()
    payload = (cuda.arange(m, dtype=cuda.int64, device="cuda") % 251).to(cuda.uint8)
    for a, b in (((1 << 32) - 3000, (1 << 32) + 5000), (0, 6000), ((1 << 33) - 4096, 1 << 33)):
        exp = O.shuffle_indices_range(m, 0x5EED, PHILOX, 24, a, b)
        out = cuda.empty(b - a, dtype=cuda.int64, device="cuda")
        cnt = ctypes.c_uint64()
        _lib.check(_lib.lib.bsg_shuffle_range(m, ctypes.byref(cfg), a, b, None, None, out.data_ptr(), 8,
                                              ctypes.addressof(cnt), None), "range")
        assert cnt.value == len(exp)
        assert np.array_equal(out[:cnt.value].cpu().numpy().view(np.uint64), exp)
        outv = cuda.empty(b - a, dtype=cuda.uint8, device="cuda")
        _lib.check(_lib.lib.bsg_shuffle_range(m, ctypes.byref(cfg), a, b, payload.data_ptr(), None,
                                              outv.data_ptr(), 1, ctypes.addressof(cnt), None), "range u8")
        assert np.array_equal(outv[:cnt.value].cpu().numpy(), (exp % 251).astype(np.uint8))
    del payload
    cuda.cuda.empty_cache()


def test_sharded_input_equals_contiguous(bsg, cuda):
    from paper_2106_06161_b200 import _lib
    m, G = (1 << 20) + 777, 4
    S = (m + G - 1) // G
    vals = cuda.arange(G * S, dtype=cuda.int64, device="cuda") * 5 + 2
    shards = [vals[g * S:(g + 1) * S].clone() for g in range(G)]
    sh = _lib.bsg_shards()
    for g in range(G):
        sh.ptrs[g] = shards[g].data_ptr()
    sh.count, sh.shard_elems = G, S
    cfg = cfg_of(bsg, seed=4)._c()
    n = 1 << O.C.orc_domain_bits(m)
    out = cuda.empty(m, dtype=cuda.int64, device="cuda")
    cnt = ctypes.c_uint64()
    _lib.check(_lib.lib.bsg_shuffle_range(m, ctypes.byref(cfg), 0, n, None, ctypes.byref(sh), out.data_ptr(), 8,
                                          ctypes.addressof(cnt), None), "sharded")
    assert cnt.value == m
    exp = bsg.shuffle_values(vals[:m].contiguous(), cfg_of(bsg, seed=4))
    assert cuda.equal(out, exp)


def test_dist_shuffle_single_process_ranks(bsg, cuda):
    """Every rank of a simulated world, with the allgather answered from the count pass."""
    from paper_2106_06161_b200 import _lib
    m, W = (1 << 19) + 9, 3
    cfg = cfg_of(bsg, seed=12)._c()
    counts = []
    for r in range(W):
        b, e = ctypes.c_uint64(), ctypes.c_uint64()
        _lib.check(_lib.lib.bsg_dist_counter_range(m, r, W, ctypes.byref(b), ctypes.byref(e)), "range")
        c = ctypes.c_uint64()
        _lib.check(_lib.lib.bsg_range_count(m, ctypes.byref(cfg), b.value, e.value, ctypes.byref(c), None), "cnt")
        counts.append(c.value)

    @_lib.ALLGATHER_FN
    def ag(send, recv, user):
        for i, c in enumerate(counts):
            recv[i] = c
        return 0

    vals = cuda.arange(m, dtype=cuda.int64, device="cuda")
    full = cuda.empty(m, dtype=cuda.int64, device="cuda")
    for r in range(W):
        out = cuda.empty(m, dtype=cuda.int64, device="cuda")
        off, cnt = ctypes.c_uint64(), ctypes.c_uint64()
        _lib.check(_lib.lib.bsg_dist_shuffle_values(m, ctypes.byref(cfg), r, W, vals.data_ptr(), None,
                                                    out.data_ptr(), 8, ag, None, ctypes.byref(off),
                                                    ctypes.byref(cnt), None), "dist")
        assert cnt.value == counts[r]
        full[off.value:off.value + cnt.value] = out[:cnt.value]
    assert np.array_equal(full.cpu().numpy().view(np.uint64), O.shuffle_indices(m, 12))


# ------------------------------------------------------------- batched --
def test_batched_fixtures(bsg, cuda, golden):
    for case in golden["batched"]:
        m = case["m"]
        batch = 4
        vals = cuda.arange(m, dtype=cuda.int32, device="cuda").repeat(batch, 1)
        out = bsg.shuffle_values_batched(vals, cfg_of(bsg, seed=case["seed"], variant=case["variant"],
                                                      rounds=case["rounds"]))
        for row in case["rows"]:
            got = out[row["b"]].cpu().numpy().astype(np.uint64)
            assert f"{O.fnv1a64(got):016x}" == row["fnv"], (m, row["b"])


def test_batched_vs_oracle_many(bsg, cuda):
    rng = np.random.default_rng(3)
    for m, dt, rounds, variant in ((1024, np.uint32, 24, PHILOX), (1000, np.uint64, 24, PHILOX),
                                   (4096, np.uint16, 24, LCG), (3, np.uint8, 24, PHILOX), (777, np.uint32, 12, PHILOX),
                                   (1 << 14, np.uint64, 24, PHILOX), (5000, np.uint32, 31, PHILOX),
                                   (2, np.uint32, 24, PHILOX), (1 << 17, np.uint32, 24, PHILOX),
                                   # shared-memory table rounds (L == R <= 5): odd and generic round counts
                                   (1000, np.uint32, 25, PHILOX), (64, np.uint32, 3, PHILOX),
                                   (256, np.uint64, 7, PHILOX), (16, np.uint8, 24, PHILOX),
                                   (1023, np.uint16, 100, PHILOX)):
        batch = 37
        vals = rng.integers(0, np.iinfo(dt).max, size=(batch, m), dtype=dt)
        got = bsg.shuffle_values_batched(vals, cfg_of(bsg, seed=123, variant=variant, rounds=rounds))
        exp = O.shuffle_values_batched(vals, 123, variant, rounds)
        assert np.array_equal(got, exp), (m, dt, rounds)


def test_batched_c4_shape(bsg, cuda):
    """C4: 65536 shuffles of 1024 u32 (one GPU's share of 8192 checked against the oracle)."""
    batch, m = 8192, 1024
    vals = cuda.randint(0, 2**31 - 1, (batch, m), dtype=cuda.int32, device="cuda")
    out = bsg.shuffle_values_batched(vals, cfg_of(bsg, seed=1000))
    vh, oh = vals.cpu().numpy().view(np.uint32), out.cpu().numpy().view(np.uint32)
    for b in (0, 1, 2, 4095, 8191):
        perm = O.shuffle_indices(m, 1000 + b)
        assert np.array_equal(oh[b], vh[b][perm.astype(np.int64)])


# --------------------------------------------------------------- gather --
def test_gather(bsg, cuda):  # unit_shuffle.cpp:422-442
    src = np.array([10, 20, 30], dtype=np.uint64)
    idx = np.array([2, 2, 0, 1], dtype=np.uint64)
    assert list(bsg.gather(src, idx)) == [30, 30, 10, 20]
    with pytest.raises(bsg.InvalidArgument):
        bsg.gather_into(src, idx, src)
    big = cuda.arange(1 << 22, dtype=cuda.int64, device="cuda") * 3
    ix = cuda.randint(0, 1 << 22, (1 << 21,), device="cuda")
    assert cuda.equal(bsg.gather(big, ix), big[ix])
    for dt in (cuda.uint8, cuda.int16, cuda.int32):
        s = (cuda.arange(1000, device="cuda") % 100).to(dt)
        i = cuda.randint(0, 1000, (5000,), device="cuda")
        assert cuda.equal(bsg.gather(s, i), s[i])


def test_sort_shuffle_baseline_is_permutation(bsg, cuda):
    n = 1 << 20
    v = cuda.arange(n, dtype=cuda.int64, device="cuda")
    out = bsg.sort_shuffle_u64(v, 1)
    assert cuda.equal(out.sort().values, v) and not cuda.equal(out, v)


def test_kernel_launch_counter_moves(bsg, cuda):
    before = bsg.kernel_launches()
    bsg.shuffle_indices(1 << 20, cfg_of(bsg), device="cuda")
    cuda.cuda.synchronize()
    assert bsg.kernel_launches() > before


def test_pipeline_streams_match_oracle(bsg, cuda):
    m = (1 << 20) + 3
    pairs = [(cuda.arange(m, dtype=cuda.int64).pin_memory(), cuda.empty(m, dtype=cuda.int64).pin_memory())
             for _ in range(3)]
    with bsg.Pipeline(m, 8, depth=2) as pipe:
        tickets = [pipe.submit(pairs[i][0], pairs[i][1], cfg_of(bsg, seed=40 + i)) for i in range(3)]
        for t in tickets:
            pipe.wait(t)
    for i in range(3):
        assert np.array_equal(pairs[i][1].numpy().view(np.uint64), O.shuffle_indices(m, 40 + i)), i
    with pytest.raises(bsg.InvalidArgument):
        with bsg.Pipeline(16, 8) as pipe:
            pipe.submit(pairs[0][0], pairs[0][1])  # m exceeds capacity


def test_pipeline_batched_rows_match_oracle(bsg, cuda):
    """bsg_pipeline_submit_batched: rows of pinned host buffers, row b shuffled with seed + b, streamed through
    two slots (the C4 e2e path)."""
    batch, m = 64, 1024
    ins = [cuda.arange(m, dtype=cuda.int32).repeat(batch, 1).contiguous().pin_memory() for _ in range(3)]
    outs = [cuda.empty(batch, m, dtype=cuda.int32).pin_memory() for _ in range(3)]
    with bsg.Pipeline(batch * m, 4, depth=2) as pipe:
        tickets = [pipe.submit_batched(ins[i], outs[i], cfg_of(bsg, seed=900 + 100 * i)) for i in range(3)]
        for t in tickets:
            pipe.wait(t)
        with pytest.raises(bsg.InvalidArgument):
            pipe.submit_batched(cuda.zeros(batch + 1, m, dtype=cuda.int32).pin_memory(),
                                cuda.zeros(batch + 1, m, dtype=cuda.int32).pin_memory())  # exceeds capacity
    for i in range(3):
        for b in (0, 1, batch - 1):
            exp = O.shuffle_indices(m, 900 + 100 * i + b)
            assert np.array_equal(outs[i][b].numpy().astype(np.uint64), exp), (i, b)


def test_partitioned_path_matches_single_pass(bsg, cuda, golden):
    """The three-pass partitioned kernel (pow2, large) is bit-identical to the fused single pass."""
    old = bsg.set_path(2)
    try:
        for m, dt, variant, rounds in (((1 << 16), cuda.int64, PHILOX, 24), ((1 << 20), cuda.int32, PHILOX, 24),
                                       ((1 << 21), cuda.int64, LCG, 24), ((1 << 22), cuda.int64, PHILOX, 12),
                                       ((1 << 23), cuda.int32, PHILOX, 24), ((1 << 19), cuda.int64, PHILOX, 24)):
            vals = cuda.arange(m, dtype=dt, device="cuda")
            got = bsg.shuffle_values(vals, cfg_of(bsg, seed=m + rounds, variant=variant, rounds=rounds))
            exp = O.shuffle_indices(m, m + rounds, variant, rounds)
            assert np.array_equal(got.cpu().numpy().astype(np.uint64), exp), (m, dt, variant, rounds)
        for case in golden["values_full_hash"]:
            if case["m"] & (case["m"] - 1):
                continue
            vals = cuda.arange(case["m"], dtype=cuda.int64, device="cuda")
            out = bsg.shuffle_values(vals, cfg_of(bsg, seed=case["seed"], variant=case["variant"]))
            host = out.cpu().numpy().view(np.uint64)
            del vals, out
            assert f"{O.fnv1a64(host):016x}" == case["fnv"], case
    finally:
        bsg.set_path(old)
        cuda.cuda.empty_cache()


def test_route_and_scatter_sharded_simulation(bsg, cuda):
    """Sharded pow2 shuffle by destination routing, every rank simulated in one process:
    route (bsg_route_by_dest) -> exchange (slicing, as the all-to-all would) -> place (bsg_scatter_permutation)."""
    from paper_2106_06161_b200 import distributed as D
    for m, W, dt in (((1 << 20), 4, cuda.int64), ((1 << 22), 8, cuda.int32), ((1 << 16), 2, cuda.int64)):
        cfg = cfg_of(bsg, seed=m + W)
        S = m // W
        full_in = cuda.arange(m, dtype=dt, device="cuda") * 5 + 1
        routed = [D._gpu_route(full_in[r * S:(r + 1) * S].contiguous(), m, cfg, r, W) for r in range(W)]
        out = []
        for dst in range(W):
            vs, ds = [], []
            for src in range(W):
                vals, dl, counts = routed[src]
                off = sum(counts[:dst])
                vs.append(vals[off:off + counts[dst]])
                ds.append(dl[off:off + counts[dst]])
            out.append(D._gpu_scatter(cuda.cat(vs), cuda.cat(ds), S))
        got = cuda.cat(out).cpu().numpy().astype(np.int64).view(np.uint64)
        exp = O.shuffle_indices(m, m + W) * np.uint64(5) + np.uint64(1)  # the oracle's permutation of the payload
        assert np.array_equal(got, exp), (m, W)


def test_scatter_permutation_paths(bsg, cuda):
    from paper_2106_06161_b200 import distributed as D
    for n, path in ((1 << 12, 0), (1 << 21, 2), (1 << 21, 1)):
        old = bsg.set_path(path)
        try:
            perm = bsg.shuffle_indices(n, cfg_of(bsg, seed=n), device="cuda")
            vals = cuda.arange(n, dtype=cuda.int64, device="cuda")
            out = D._gpu_scatter(vals, perm.to(cuda.int32), n)
            ref = cuda.empty_like(vals)
            ref[perm] = vals
            assert cuda.equal(out, ref), (n, path)
        finally:
            bsg.set_path(old)


def test_partitioned_16_byte_payload(bsg, cuda):
    """16-byte records through the partitioned path and the single pass, via the C ABI."""
    from paper_2106_06161_b200 import _lib
    m = 1 << 20
    rec = cuda.arange(2 * m, dtype=cuda.int64, device="cuda").view(m, 2)
    exp = O.shuffle_indices(m, 44)
    for path in (1, 2):
        old = bsg.set_path(path)
        try:
            out = cuda.empty_like(rec)
            _lib.check(_lib.lib.bsg_shuffle_values(rec.data_ptr(), out.data_ptr(), m, 16,
                                                   ctypes.byref(cfg_of(bsg, seed=44)._c()), None), "u128")
            cuda.cuda.synchronize()
            got = out.cpu().numpy()
            assert np.array_equal(got[:, 0].astype(np.uint64), 2 * exp), path
            assert np.array_equal(got[:, 1].astype(np.uint64), 2 * exp + 1), path
        finally:
            bsg.set_path(old)


def test_concurrent_callers_on_separate_streams(bsg, cuda):
    """Host threads on their own CUDA streams share one device context (look-back workspace,
    key buffer, partition workspace): results must stay exact."""
    import threading
    sizes = [(1 << 20) + 7, 1 << 21, 5000, (1 << 18) + 1, 1 << 16, 123457]
    errors = []

    def worker(tid):
        try:
            s = cuda.cuda.Stream()
            with cuda.cuda.stream(s):
                for it in range(4):
                    m = sizes[(tid + it) % len(sizes)]
                    seed = tid * 100 + it
                    vals = cuda.arange(m, dtype=cuda.int64, device="cuda")
                    out = bsg.shuffle_values(vals, cfg_of(bsg, seed=seed, rounds=24 if it % 2 else 12))
                    s.synchronize()
                    exp = O.shuffle_indices(m, seed, PHILOX, 24 if it % 2 else 12)
                    if not np.array_equal(out.cpu().numpy().view(np.uint64), exp):
                        errors.append((tid, it, m))
        except Exception as e:  # noqa: BLE001
            errors.append((tid, repr(e)))

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors


def test_pipeline_with_pageable_buffers(bsg, cuda):
    m = 70001
    a = np.arange(m, dtype=np.uint64)
    b = np.empty_like(a)
    with bsg.Pipeline(m, 8) as pipe:
        pipe.wait(pipe.submit(a, b, cfg_of(bsg, seed=31)))
    assert np.array_equal(b, O.shuffle_indices(m, 31))


def test_pow2_wide_counters(bsg, cuda):
    """m = 2^33 (64-bit counters on the all-survive path) on counter slices, both variants."""
    from paper_2106_06161_b200 import _lib
    m = 1 << 33
    for variant in (PHILOX, LCG):
        cfg = cfg_of(bsg, seed=0xC0FFEE, variant=variant)._c()
        for a, b in ((0, 5000), ((1 << 32) - 2500, (1 << 32) + 2500), (m - 5000, m)):
            out = cuda.empty(b - a, dtype=cuda.int64, device="cuda")
            cnt = ctypes.c_uint64()
            _lib.check(_lib.lib.bsg_shuffle_range(m, ctypes.byref(cfg), a, b, None, None, out.data_ptr(), 8,
                                                  ctypes.addressof(cnt), None), "range")
            assert cnt.value == b - a
            exp = O.shuffle_indices_range(m, 0xC0FFEE, variant, 24, a, b)
            assert np.array_equal(out.cpu().numpy().view(np.uint64), exp), (variant, a)


def test_partitioned_512_coarse_buckets(bsg, cuda):
    """2^30 u64 takes 512 coarse buckets (two bins per thread in P1's scan); equal to the single pass."""
    m = 1 << 30
    vals = cuda.arange(m, dtype=cuda.int64, device="cuda")
    outs = []
    for path in (2, 1):
        old = bsg.set_path(path)
        try:
            outs.append(bsg.shuffle_values(vals, cfg_of(bsg, seed=30)))
        finally:
            bsg.set_path(old)
    assert cuda.equal(outs[0], outs[1])
    assert np.array_equal(outs[0][:4096].cpu().numpy().view(np.uint64), O.shuffle_indices_range(m, 30, PHILOX, 24, 0, 4096))
    del vals, outs
    cuda.cuda.empty_cache()


def test_partitioned_512_fine_windows_16_byte(bsg, cuda):
    """C5's per-GPU unit: 2^30 16-byte records take 512 coarse buckets x 512 fine windows (two bins per
    thread in both scans).  The keys of the output must be the permutation itself (single pass), and the
    first entries the oracle's."""
    m = 1 << 30
    rec = cuda.arange(2 * m, dtype=cuda.int64, device="cuda").view(cuda.complex128)
    old = bsg.set_path(2)
    try:
        out = bsg.shuffle_values(rec, cfg_of(bsg, seed=55))
    finally:
        bsg.set_path(old)
    del rec
    keys = out.view(cuda.int64).view(m, 2)[:, 0] // 2
    vals_ok = cuda.equal(out.view(cuda.int64).view(m, 2)[:, 1], out.view(cuda.int64).view(m, 2)[:, 0] + 1)
    del out
    cuda.cuda.empty_cache()
    perm = bsg.shuffle_indices(m, cfg_of(bsg, seed=55), device="cuda")
    assert vals_ok
    assert cuda.equal(keys, perm)
    assert np.array_equal(perm[:4096].cpu().numpy().view(np.uint64), O.shuffle_indices_range(m, 55, PHILOX, 24, 0, 4096))
    del keys, perm
    cuda.cuda.empty_cache()


def test_cuda_graph_capture_and_replay(bsg, cuda):
    """Device-pointer calls are capturable into a CUDA graph (after one uncaptured call sizes the workspaces);
    every replay recomputes the shuffle of the input's current contents -- including the look-back path,
    whose status words a replay cannot re-epoch, and generic round counts, whose keys a replay re-uploads."""
    cases = [((1 << 20), 24, cuda.int64, "pow2"), ((1 << 20) + 7, 24, cuda.int64, "lookback"),
             ((1 << 16) + 1, 9, cuda.int32, "generic rounds"), ((1 << 25), 24, cuda.int64, "partitioned"),
             ((1 << 25) + 3, 24, cuda.int64, "partitioned")]  # padded: window scan + compaction in the graph
    for m, rounds, dt, what in cases:
        cfg = cfg_of(bsg, seed=77, rounds=rounds)
        vals = cuda.arange(m, dtype=dt, device="cuda")
        out = cuda.empty_like(vals)
        old = bsg.set_path(2 if what == "partitioned" else 0)
        try:
            bsg.shuffle_values_into(vals, cfg, out)  # sizes the workspaces outside the capture
            s = cuda.cuda.Stream()
            g = cuda.cuda.CUDAGraph()
            with cuda.cuda.stream(s):
                cuda.cuda.synchronize()
                with cuda.cuda.graph(g, stream=s):
                    bsg.shuffle_values_into(vals, cfg, out)
            for k in range(3):
                vals.copy_(cuda.arange(m, dtype=dt, device="cuda") * (k + 2) + k)
                out.zero_()
                g.replay()
                cuda.cuda.synchronize()
                exp = bsg.shuffle_values(vals, cfg)
                assert cuda.equal(out, exp), (what, k)
        finally:
            bsg.set_path(old)
    rows = cuda.arange(1024, dtype=cuda.int32, device="cuda").repeat(64, 1)
    outb = cuda.empty_like(rows)
    bsg.shuffle_values_batched(rows, bsg.ShuffleConfig(seed=5), out=outb)
    g = cuda.cuda.CUDAGraph()
    s = cuda.cuda.Stream()
    with cuda.cuda.stream(s):
        cuda.cuda.synchronize()
        with cuda.cuda.graph(g, stream=s):
            bsg.shuffle_values_batched(rows, bsg.ShuffleConfig(seed=5), out=outb)
    outb.zero_()
    g.replay()
    cuda.cuda.synchronize()
    assert cuda.equal(outb, bsg.shuffle_values_batched(rows, bsg.ShuffleConfig(seed=5)))


def test_partitioned_full_32_bit_domain(bsg, cuda):
    """The largest partitioned shape: 2^32 u32 (bits = 32, 512 x 512 fan-out, write-back positions that use all
    32 bits of the position tables).  Equal to the single pass; head and tail against the oracle."""
    m = 1 << 32
    vals = cuda.arange(m, dtype=cuda.int64, device="cuda").to(cuda.int32)  # low 32 bits of the index
    outs = []
    for path in (2, 1):
        old = bsg.set_path(path)
        try:
            outs.append(bsg.shuffle_values(vals, cfg_of(bsg, seed=32)))
        finally:
            bsg.set_path(old)
    del vals
    cuda.cuda.empty_cache()
    assert cuda.equal(outs[0], outs[1])
    head = outs[0][:2048].cpu().numpy().view(np.uint32).astype(np.uint64)
    tail = outs[0][-2048:].cpu().numpy().view(np.uint32).astype(np.uint64)
    assert np.array_equal(head, O.shuffle_indices_range(m, 32, PHILOX, 24, 0, 2048))
    assert np.array_equal(tail, O.shuffle_indices_range(m, 32, PHILOX, 24, m - 2048, m))
    del outs
    cuda.cuda.empty_cache()


def test_partitioned_non_power_of_two(bsg, cuda):
    """Non-power-of-two domains through the partitioned path (inputs routed by counter f^-1(j), windows compacted by
    counter rank): equal to the oracle for both bijections, u64 and u32 payloads, ragged last tiles."""
    for m, variant, dt in [((1 << 20) + 1, PHILOX, cuda.int64), ((1 << 20) + 1, LCG, cuda.int64),
                           (3 * (1 << 18) + 17, PHILOX, cuda.int32), ((1 << 16) + 4097, PHILOX, cuda.int64),
                           ((1 << 15) - 3, LCG, cuda.int32), ((1 << 21) - 1, PHILOX, cuda.int64)]:
        vals = cuda.arange(m, dtype=dt, device="cuda")
        old = bsg.set_path(2)
        try:
            out = bsg.shuffle_values(vals, cfg_of(bsg, seed=m, variant=variant))
        finally:
            bsg.set_path(old)
        got = out.cpu().numpy().astype(np.int64).view(np.uint64) if dt == cuda.int32 else out.cpu().numpy().view(np.uint64)
        assert np.array_equal(got, O.shuffle_indices(m, m, variant, 24)), (m, variant, dt)


def test_partitioned_non_power_of_two_overflow_windows(bsg, cuda):
    """The persistent last pass stages at most `cap` survivors per 2^14-counter window; windows above it go to
    the round-based pass through a device list.  Lowering the cap (8192: about half the windows; 0: all of them;
    8300: a few) must not change the output, for u32/u64, both bijections, and outputs at odd offsets (the bulk
    store's unaligned head and tail)."""
    old_path = bsg.set_path(2)
    old_cap = bsg.set_rank_stage_cap(9216)
    try:
        for cap in (8192, 0, 8300, 9216):
            bsg.set_rank_stage_cap(cap)
            for m, variant, dt in [((1 << 20) + 1, PHILOX, cuda.int64), ((1 << 19) + 5, LCG, cuda.int32),
                                   ((1 << 21) - 7, LCG, cuda.int64), (3 * (1 << 17) + 1, PHILOX, cuda.int32)]:
                vals = cuda.arange(m, dtype=dt, device="cuda")
                buf = cuda.full((m + 3,), -1, dtype=dt, device="cuda")
                out = buf[1:m + 1]  # element-aligned, not 16-byte aligned
                bsg.shuffle_values_into(vals, cfg_of(bsg, seed=m + cap, variant=variant), out)
                got = out.cpu().numpy().astype(np.int64).view(np.uint64) if dt == cuda.int32 else \
                    out.cpu().numpy().view(np.uint64)
                assert np.array_equal(got, O.shuffle_indices(m, m + cap, variant, 24)), (cap, m, variant, dt)
                assert int(buf[0]) == -1 and int(buf[m + 1]) == -1 and int(buf[m + 2]) == -1, (cap, m)
    finally:
        bsg.set_rank_stage_cap(old_cap)
        bsg.set_path(old_path)


def test_partitioned_host_buffers_staged(bsg, cuda):
    """Host input and output through the partitioned path: the H2D is chunked under P1 and (power of two) the D2H
    under P3 (StageIO in bsg_shuffle_values); pinned and pageable buffers, both bijections, padded domains."""
    old = bsg.set_path(2)
    try:
        for m, variant, dt, pinned in [((1 << 20), PHILOX, cuda.int64, True), ((1 << 20) + 3, PHILOX, cuda.int64, True),
                                       ((1 << 21), LCG, cuda.int32, False), ((1 << 19) + 77, LCG, cuda.int32, True),
                                       (12345, PHILOX, cuda.int64, False)]:
            vals = cuda.arange(m, dtype=dt) * 3 + 1
            out = cuda.empty_like(vals)
            if pinned:
                vals, out = vals.pin_memory(), out.pin_memory()
            bsg.shuffle_values_into(vals, cfg_of(bsg, seed=m, variant=variant), out)
            got = out.numpy().astype(np.int64).view(np.uint64)
            exp = O.shuffle_indices(m, m, variant, 24) * np.uint64(3) + np.uint64(1)
            assert np.array_equal(got, exp), (m, variant, dt, pinned)
    finally:
        bsg.set_path(old)


def test_partitioned_bulk_and_plain_stores_agree(bsg, cuda):
    """The last passes write placed windows by bulk shared->global copies (default) or plain stores
    (bsg_set_bulk_stores(0)): both equal the oracle, power of two or padded, aligned or not."""
    old_path = bsg.set_path(2)
    old_bulk = bsg.set_bulk_stores(True)
    try:
        for bulk in (True, False):
            bsg.set_bulk_stores(bulk)
            for m, variant, dt, off in [((1 << 20), PHILOX, cuda.int64, 0), ((1 << 20), LCG, cuda.int32, 1),
                                        ((1 << 20) + 3, PHILOX, cuda.int64, 1), ((1 << 18) + 9, LCG, cuda.int32, 0)]:
                vals = cuda.arange(m, dtype=dt, device="cuda")
                buf = cuda.full((m + 2,), -1, dtype=dt, device="cuda")
                out = buf[off:off + m]
                bsg.shuffle_values_into(vals, cfg_of(bsg, seed=m + off, variant=variant), out)
                got = out.cpu().numpy().astype(np.int64).view(np.uint64) if dt == cuda.int32 else \
                    out.cpu().numpy().view(np.uint64)
                assert np.array_equal(got, O.shuffle_indices(m, m + off, variant, 24)), (bulk, m, variant, dt, off)
    finally:
        bsg.set_bulk_stores(old_bulk)
        bsg.set_path(old_path)


def test_partitioned_non_power_of_two_full_size(bsg, cuda):
    """C3 itself (2^29+1 u64, 2^30 counters): the partitioned and single-pass paths agree bit for bit, for the
    Feistel and the LCG; the head matches the oracle."""
    m = (1 << 29) + 1
    vals = cuda.arange(m, dtype=cuda.int64, device="cuda")
    for variant in (PHILOX, LCG):
        outs = []
        for path in (2, 1):
            old = bsg.set_path(path)
            try:
                outs.append(bsg.shuffle_values(vals, cfg_of(bsg, seed=0x5EED, variant=variant)))
            finally:
                bsg.set_path(old)
        assert cuda.equal(outs[0], outs[1]), variant
        exp = O.shuffle_indices_range(m, 0x5EED, variant, 24, 0, 8192)  # survivors of the first 8192 counters
        assert np.array_equal(outs[0][:len(exp)].cpu().numpy().view(np.uint64), exp), variant
        del outs
    del vals
    cuda.cuda.empty_cache()


def test_cuda_graph_survives_workspace_growth(bsg, cuda):
    """A graph captured with the partition workspace sized for 2^22 stays valid after an uncaptured 2^24 call
    grows the workspace (the captured allocation is retired, not freed)."""
    m = (1 << 22) + 1
    cfg = cfg_of(bsg, seed=3)
    vals = cuda.arange(m, dtype=cuda.int64, device="cuda")
    out = cuda.empty_like(vals)
    old = bsg.set_path(2)
    try:
        bsg.shuffle_values_into(vals, cfg, out)
        g = cuda.cuda.CUDAGraph()
        s = cuda.cuda.Stream()
        with cuda.cuda.stream(s):
            cuda.cuda.synchronize()
            with cuda.cuda.graph(g, stream=s):
                bsg.shuffle_values_into(vals, cfg, out)
        big = cuda.arange((1 << 24) + 1, dtype=cuda.int64, device="cuda")
        bsg.shuffle_values(big, cfg)  # grows the cached workspace
        del big
        out.zero_()
        g.replay()
        cuda.cuda.synchronize()
        assert cuda.equal(out, bsg.shuffle_values(vals, cfg))
    finally:
        bsg.set_path(old)


def test_partitioned_random_shapes(bsg, cuda):
    """Randomised parity of the forced partitioned path (power of two or not, both bijections, u32/u64, generic
    round counts) against the oracle."""
    rng = np.random.default_rng(2106)
    old = bsg.set_path(2)
    try:
        for _ in range(24):
            m = int(rng.integers(1 << 14, 1 << 21))
            if rng.random() < 0.25:
                m = 1 << int(m.bit_length() - 1)
            variant = int(rng.integers(0, 2))
            rounds = int(rng.choice([24, 24, 7, 30]))
            seed = int(rng.integers(0, 2**63))
            dt = cuda.int64 if rng.random() < 0.5 else cuda.int32
            vals = cuda.arange(m, dtype=dt, device="cuda")
            out = bsg.shuffle_values(vals, cfg_of(bsg, seed=seed, variant=variant, rounds=rounds))
            got = out.cpu().numpy().astype(np.int64).view(np.uint64)
            assert np.array_equal(got, O.shuffle_indices(m, seed, variant, rounds)), (m, seed, variant, rounds, dt)
    finally:
        bsg.set_path(old)


def test_c5_kernel_sharded_16byte_wide_counters(bsg, cuda):
    """The C5 per-rank kernel: m = 2^33 16-byte {key, value} records read through an 8-entry shard table
    (k_pow2 with 64-bit counters, uint4 payload, sharded source), on counter slices of three ranks' ranges.
    The 8 shards of 2^30 records alias two 16 GiB buffers A/B (shard g -> A if g even), so the record read
    for image j is {key = j mod 2^30, value = tag(j >> 30)}: both the in-shard index and the shard choice are
    checked against the oracle's images."""
    from paper_2106_06161_b200 import _lib
    m, S, G = 1 << 33, 1 << 30, 8
    tags = (0xAAAA0000, 0xBBBB0000)
    bufs = []
    for t in tags:
        rec = cuda.empty((S, 2), dtype=cuda.int64, device="cuda")
        rec[:, 0] = cuda.arange(S, dtype=cuda.int64, device="cuda")
        rec[:, 1] = t
        bufs.append(rec)
    sh = _lib.bsg_shards()
    for g in range(G):
        sh.ptrs[g] = bufs[g & 1].data_ptr()
    sh.count, sh.shard_elems = G, S
    try:
        for variant in (PHILOX, LCG):
            cfg = cfg_of(bsg, seed=0x5EED, variant=variant)._c()
            for a, b in ((0, 1 << 16), ((3 << 30) - 7000, (3 << 30) + 9000), (m - 4096, m)):
                exp = O.shuffle_indices_range(m, 0x5EED, variant, 24, a, b)
                out = cuda.empty((b - a, 2), dtype=cuda.int64, device="cuda")
                cnt = ctypes.c_uint64()
                _lib.check(_lib.lib.bsg_shuffle_range(m, ctypes.byref(cfg), a, b, None, ctypes.byref(sh),
                                                      out.data_ptr(), 16, ctypes.addressof(cnt), None), "c5 range")
                assert cnt.value == b - a
                got = out.cpu().numpy().view(np.uint64)
                assert np.array_equal(got[:, 0], exp & np.uint64(S - 1)), (variant, a)
                assert np.array_equal(got[:, 1], np.where((exp >> np.uint64(30)) & np.uint64(1), np.uint64(tags[1]),
                                                          np.uint64(tags[0]))), (variant, a)
    finally:
        del bufs
        cuda.cuda.empty_cache()


def test_partition_path_unaligned_input(bsg, cuda):
    """an element-aligned but not 16-byte-aligned input (the view x[1:]) on the partitioned path with
    the LCG (whose P1 is TMA-fed when the input is aligned) must not fault and must match the oracle."""
    for m, path in (((1 << 25), 0), ((1 << 20), 2), ((1 << 20) + 3, 2)):
        base = cuda.arange(m + 1, dtype=cuda.int64, device="cuda")
        x = base[1:]
        assert x.data_ptr() % 16 == 8
        old = bsg.set_path(path)
        try:
            out = bsg.shuffle_values(x, cfg_of(bsg, seed=77, variant=LCG))
        finally:
            bsg.set_path(old)
        exp = O.shuffle_indices(m, 77, LCG, 24) + np.uint64(1)
        assert np.array_equal(out.cpu().numpy().view(np.uint64), exp), (m, path)
    # the scatter-by-permutation entry point takes the same TMA-fed P1 for its values
    from paper_2106_06161_b200 import _lib
    n = 1 << 20
    vals = cuda.arange(n + 1, dtype=cuda.int64, device="cuda")[1:]
    dest = cuda.from_numpy(O.shuffle_indices(n, 5).astype(np.int64)).to("cuda").to(cuda.int32)
    out = cuda.empty(n, dtype=cuda.int64, device="cuda")
    old = bsg.set_path(2)
    try:
        _lib.check(_lib.lib.bsg_scatter_permutation(vals.data_ptr(), dest.data_ptr(), n, out.data_ptr(), 8, None),
                   "scatter")
    finally:
        bsg.set_path(old)
    exp = np.empty(n, dtype=np.uint64)
    exp[O.shuffle_indices(n, 5)] = np.arange(1, n + 1, dtype=np.uint64)
    assert np.array_equal(out.cpu().numpy().view(np.uint64), exp)


def test_workspace_bytes_and_release(bsg, cuda):
    vals = cuda.arange(1 << 20, dtype=cuda.int64, device="cuda")
    old = bsg.set_path(2)
    try:
        bsg.shuffle_values(vals, cfg_of(bsg, seed=1))
    finally:
        bsg.set_path(old)
    cuda.cuda.synchronize()
    held = bsg.workspace_bytes()
    assert held >= (1 << 20) * 14
    bsg.release_workspace()
    assert bsg.workspace_bytes() < held
