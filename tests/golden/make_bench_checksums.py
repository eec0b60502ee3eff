"""Generate tests/golden/bench_checksums.json: order-sensitive checksums of the
exact outputs bench.py times, computed from the UNMODIFIED reference
(oracle/_ref, compiled from /root/reference by oracle/Makefile).  bench.py
checksums its own timed output on the GPU after the timed region and asserts
it against these numbers, so every driver-run bench line carries parity
evidence for the bytes it timed.  Needs /root/reference (this container); the
JSON is committed and travels to the GPU box.

Checksum of an output (bench.py:output_checksum): view it as a flat array of
u64 words w[i] (u32 elements zero-extended, 16-byte records as two words) and
take, modulo 2^64,
    sum  = sum_i w[i]                wsum = sum_i w[i] * (2*i + 1).
A wrong permutation changes wsum unless (i - j) * (w[i] - w[j]) * 2 vanishes
mod 2^64 for every displaced pair, impossible for indices and values < 2^34.

    python tests/golden/make_bench_checksums.py        # ~15 min on 8 cores, ~20 GB RAM (c5's permutation)
    python tests/golden/make_bench_checksums.py --c5-multi   # adds c5@2/4/8 (streamed)
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

SEED = 0x5EED  # bench.py SEED
M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
CHUNK = 1 << 25


def checksum_words(words_fn, n_words):
    """(sum, wsum) of w[0..n_words) produced chunk by chunk by words_fn(lo, hi)."""
    s = np.uint64(0)
    ws = np.uint64(0)
    with np.errstate(over="ignore"):
        for lo in range(0, n_words, CHUNK):
            hi = min(n_words, lo + CHUNK)
            w = words_fn(lo, hi).astype(np.uint64, copy=False)
            idx = np.arange(lo, hi, dtype=np.uint64)
            s += np.sum(w, dtype=np.uint64)
            ws += np.sum(w * (idx * np.uint64(2) + np.uint64(1)), dtype=np.uint64)
    return int(s), int(ws)


def streamed_checksum(m, seed, variant, threads=8, chunk=1 << 24):
    """(sum, wsum) of the m-element shuffle_indices output without materialising it: the reference's philox_apply
    on the counters in order, images >= m dropped (shuffle.hpp:58-69 / 91-147), the running output position as
    weight.  Used for the multi-rank sizes (up to 2^33 counters) that do not fit in host memory; checked equal to
    the materialised reference output at the one-rank sizes."""
    from concurrent.futures import ThreadPoolExecutor
    assert variant == 1
    bits = int(O.REF.ref_domain_bits(m))
    n = 1 << bits

    def images(c0):
        c = np.arange(c0, min(n, c0 + chunk), dtype=np.uint64)
        y = np.empty_like(c)
        assert O.REF.ref_philox_apply_many(bits, seed, 24, c.ctypes.data, c.size, y.ctypes.data) == 0
        return y[y < np.uint64(m)]

    s = np.uint64(0)
    ws = np.uint64(0)
    pos = 0
    starts = list(range(0, n, chunk))
    with ThreadPoolExecutor(threads) as ex, np.errstate(over="ignore"):
        for b in range(0, len(starts), threads):  # bounded: `threads` chunks in flight
            for y in ex.map(images, starts[b:b + threads]):
                k = np.arange(pos, pos + y.size, dtype=np.uint64)
                s += np.sum(y, dtype=np.uint64)
                ws += np.sum(y * (k * np.uint64(2) + np.uint64(1)), dtype=np.uint64)
                pos += y.size
    assert pos == m
    return int(s), int(ws)


def streamed_checksum_c5(m, seed, threads=8, chunk=1 << 24):
    """(sum, wsum) of the C5 output for m power-of-two records {2i, 2i+1} (the multi-rank sizes): record k of the
    output is {2 y, 2 y + 1} with y = philox_apply(k) from the reference, words 2k and 2k + 1."""
    from concurrent.futures import ThreadPoolExecutor
    bits = int(O.REF.ref_domain_bits(m))
    assert (1 << bits) == m

    def part(c0):
        c = np.arange(c0, min(m, c0 + chunk), dtype=np.uint64)
        y = np.empty_like(c)
        assert O.REF.ref_philox_apply_many(bits, seed, 24, c.ctypes.data, c.size, y.ctypes.data) == 0
        with np.errstate(over="ignore"):
            two = np.uint64(2)
            w0, w1 = y * two, y * two + np.uint64(1)
            i0 = c * two
            s = np.sum(w0, dtype=np.uint64) + np.sum(w1, dtype=np.uint64)
            ws = (np.sum(w0 * (i0 * two + np.uint64(1)), dtype=np.uint64) +
                  np.sum(w1 * (i0 * two + np.uint64(3)), dtype=np.uint64))
        return s, ws

    s = np.uint64(0)
    ws = np.uint64(0)
    with ThreadPoolExecutor(threads) as ex, np.errstate(over="ignore"):
        starts = list(range(0, m, chunk))
        for b in range(0, len(starts), threads):
            for a, w in ex.map(part, starts[b:b + threads]):
                s += a
                ws += w
    return int(s), int(ws)


def add_c5_multi():
    """--c5-multi: add c5@2/4/8 (2^31..2^33 records, streamed) to the committed JSON, the c5@1 entry pinning the
    streamed form."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "bench_checksums.json")
    out = json.load(open(path))
    C = out["configs"]
    s, ws = streamed_checksum_c5(1 << 30, SEED)
    assert (f"{s:016x}", f"{ws:016x}") == (C["c5@1"]["sum"], C["c5@1"]["wsum"]), "streamed c5 form"
    for n in (2, 4, 8):
        m = (1 << 30) * n
        s, ws = streamed_checksum_c5(m, SEED)
        C[f"c5@{n}"] = {"m": m, "variant": 1, "sum": f"{s:016x}", "wsum": f"{ws:016x}"}
        print("c5", n, C[f"c5@{n}"], flush=True)
    with open(path, "w") as f:
        json.dump(out, f, indent=1)


def indices(m, seed, variant):
    p = O.ref_shuffle_indices(m, seed, variant, 24)
    assert O.is_valid_permutation(p) if m <= (1 << 24) else True
    return p


def main():
    assert O.REF is not None, "build oracle/_ref first (make -C oracle ref)"
    out = {"generator": "tests/golden/make_bench_checksums.py", "reference_lib": os.path.basename(O.REF.path),
           "seed": SEED, "checksum": "sum_i w[i] and sum_i w[i]*(2i+1) mod 2^64 over the output as u64 words",
           "configs": {}}
    C = out["configs"]
    # iota u64 payloads: the output is the permutation itself (c1, c2, c3 and their LCG forms), whole-job m at N ranks
    for name, m1, variant, worlds in (("c1", 1 << 20, 1, (1,)), ("c2", 1 << 29, 1, (1, 2, 4, 8)),
                                      ("c2lcg", 1 << 29, 0, (1,)), ("c3", (1 << 29) + 1, 1, (1, 2, 4, 8)),
                                      ("c3lcg", (1 << 29) + 1, 0, (1,))):
        for n in worlds:
            m = m1 * n
            if n == 1:
                p = indices(m, SEED, variant)
                s, ws = checksum_words(lambda lo, hi: p[lo:hi], m)
                del p
                if variant == 1 and m > (1 << 20):  # pin the streamed form on the materialised reference output
                    assert streamed_checksum(m, SEED, variant) == (s, ws), name
            else:
                s, ws = streamed_checksum(m, SEED, variant)
            C[f"{name}@{n}"] = {"m": m, "variant": variant, "sum": f"{s:016x}", "wsum": f"{ws:016x}"}
            print(name, n, C[f"{name}@{n}"], flush=True)
    # c5: records {2i, 2i+1} -> out[k] = {2 s(k), 2 s(k) + 1}; words 2k, 2k+1
    m = 1 << 30
    p = indices(m, SEED, 1)

    def c5_words(lo, hi):
        k = np.arange(lo, hi, dtype=np.uint64)
        return p[k >> np.uint64(1)] * np.uint64(2) + (k & np.uint64(1))
    s, ws = checksum_words(c5_words, 2 * m)
    C["c5@1"] = {"m": m, "variant": 1, "sum": f"{s:016x}", "wsum": f"{ws:016x}"}
    print("c5", C["c5@1"], flush=True)
    del p
    # c4: rank r shuffles 8192 rows of iota(1024) u32 with seeds SEED + r*8192 + b (stats.hpp:314-324)
    batch, mrow = 8192, 1024
    for r in range(8):
        rows = np.empty((batch, mrow), dtype=np.uint64)
        for b in range(batch):
            rows[b] = O.ref_shuffle_indices(mrow, SEED + r * batch + b, 1, 24)
        flat = rows.reshape(-1)
        s, ws = checksum_words(lambda lo, hi: flat[lo:hi], flat.size)
        C[f"c4@rank{r}"] = {"batch": batch, "m": mrow, "variant": 1, "sum": f"{s:016x}", "wsum": f"{ws:016x}"}
    print("c4 done", flush=True)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "bench_checksums.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    if "--c5-multi" in sys.argv:
        add_c5_multi()
    else:
        main()
