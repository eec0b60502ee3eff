"""Generate tests/golden/golden_ref.json from the UNMODIFIED reference.

Runs the reference library itself (oracle/_ref/libbijshuf_ref.so, compiled by
oracle/Makefile from /root/reference/proj/include) -- not our restatement --
so the fixtures pin both the C oracle (tests/test_oracle.py) and the GPU
kernels (tests/test_shuffle_gpu.py).  Needs /root/reference (this container);
the JSON it writes is committed and travels to the GPU box.

    python tests/golden/make_golden.py [--full]    # --full adds the 2^29 / 2^30 hashes (~1 min, 25 GB RAM)
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402

LCG, PHILOX = 0, 1
U64 = 0xFFFFFFFFFFFFFFFF


def fnv(a) -> str:
    return f"{O.fnv1a64(np.ascontiguousarray(a).view(np.uint64)):016x}"


def ref_keys(seed, rounds):
    k = (ctypes.c_uint32 * rounds)()
    assert O.REF.ref_derive_round_keys(seed & U64, rounds, k) == 0
    return list(k)


def ref_apply(bits, seed, rounds, x):
    y = ctypes.c_uint64()
    rc = O.REF.ref_philox_apply(bits, seed & U64, rounds, x, ctypes.byref(y))
    return rc, y.value


def ref_invert(bits, seed, rounds, y):
    x = ctypes.c_uint64()
    rc = O.REF.ref_philox_invert(bits, seed & U64, rounds, y, ctypes.byref(x))
    return rc, x.value


def ref_values(values: np.ndarray, seed, variant, rounds, workers=0):
    out = np.empty_like(values)
    eb = values.itemsize * (values.size // values.shape[0])
    rc = O.REF.ref_shuffle_values(values.ctypes.data, out.ctypes.data, values.shape[0], eb, seed & U64, variant,
                                  rounds, workers)
    assert rc == 0, rc
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", action="store_true")
    args = ap.parse_args()
    assert O.REF is not None, "build oracle/_ref first (make -C oracle)"
    g = {"generator": "tests/golden/make_golden.py", "reference_lib": os.path.basename(O.REF.path),
         "avx512": bool(O.REF.ref_avx512_active())}

    g["round_keys"] = [{"seed": s, "rounds": r, "keys": ref_keys(s, r)}
                       for s, r in [(42, 4), (0, 24), (1, 24), (0x5EED, 24), (U64, 7), (123, 1)]]
    lcg = []
    for bits in [1, 2, 3, 4, 10, 16, 29, 30, 32, 33, 47, 63]:
        for seed in [0, 1, 7, 0x5EED, U64 - 3]:
            a, c = ctypes.c_uint64(), ctypes.c_uint64()
            assert O.REF.ref_make_lcg(bits, seed, ctypes.byref(a), ctypes.byref(c)) == 0
            lcg.append({"bits": bits, "seed": seed, "a": a.value, "c": c.value})
    g["make_lcg"] = lcg

    rng = np.random.default_rng(2106_06161)
    apply_kat, invert_kat = [], []
    for bits in range(2, 64):
        for rounds in ([24, 3, 12] if bits % 5 else [24, 3, 12, 25, 64, 100]):
            seed = int(rng.integers(0, 2**63)) if bits % 3 else bits
            xs = sorted({0, (1 << bits) - 1} | {int(v) for v in rng.integers(0, 1 << min(bits, 62), size=6)} |
                        {int(rng.integers(0, 2**62)) & ((1 << bits) - 1)})
            for x in xs:
                rc, y = ref_apply(bits, seed, rounds, x)
                assert rc == 0
                apply_kat.append([bits, seed, rounds, x, y])
                rc, xi = ref_invert(bits, seed, rounds, y)
                assert rc == 0 and xi == x
                invert_kat.append([bits, seed, rounds, y, x])
    g["philox_apply"] = apply_kat
    g["philox_invert"] = invert_kat

    full = []
    for m in [3, 4, 5, 8, 9, 15, 16, 17, 31, 33, 100, 255, 256, 257, 1000, 1023, 1024, 1025]:
        for variant, seed, rounds in [(PHILOX, 0, 24), (PHILOX, 7, 24), (PHILOX, 0xDEADBEEF, 3), (PHILOX, 5, 12),
                                      (LCG, 0, 24), (LCG, 1, 24), (LCG, 99, 0)]:
            p = O.ref_shuffle_indices(m, seed, variant, rounds)
            full.append({"m": m, "seed": seed, "variant": variant, "rounds": rounds, "perm": [int(v) for v in p]})
    g["indices_full"] = full

    hashed = []
    cases = [((1 << 16) + 1, 0), (1 << 20, 0), ((1 << 20) + 1, 0), (1000001, 7), ((1 << 18) + 12345, 17),
             ((1 << 22) - 3, 0x5EED), (70000, 31), (2**24 + 1, 1), (3 * 2**21, 11)]
    for m, seed in cases:
        for variant, rounds in [(PHILOX, 24), (LCG, 24), (PHILOX, 12), (PHILOX, 31)]:
            p = O.ref_shuffle_indices(m, seed, variant, rounds)
            hashed.append({"m": m, "seed": seed, "variant": variant, "rounds": rounds, "fnv": fnv(p),
                           "head": [int(v) for v in p[:8]], "tail": [int(v) for v in p[-4:]]})
    g["indices_hash"] = hashed

    vals = []
    for m, eb, seed, variant in [(70000, 8, 31, PHILOX), (12345, 4, 8, PHILOX), (5000, 16, 3, LCG),
                                 ((1 << 17) + 999, 8, 5, PHILOX), (4096, 1, 9, PHILOX), (4097, 2, 10, LCG),
                                 (3001, 12, 12, PHILOX), (1 << 16, 16, 77, PHILOX)]:
        raw = (np.arange(m * eb, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)).astype(np.uint8)
        raw = raw.reshape(m, eb)
        out = ref_values(raw, seed, variant, 24)
        vals.append({"m": m, "elem_bytes": eb, "seed": seed, "variant": variant, "rounds": 24,
                     "input": "u8[i] = (i * 0x9E3779B97F4A7C15) mod 256 over m*elem_bytes bytes",
                     "fnv_bytes": f"{O.fnv1a64(np.frombuffer(np.ascontiguousarray(out).tobytes() + bytes((-out.size) % 8), dtype=np.uint64)):016x}"})
    g["values_hash"] = vals

    batched = []
    for m, variant in [(1024, PHILOX), (1000, PHILOX), (1024, LCG), (17, PHILOX)]:
        rows = []
        for b in range(4):
            p = O.ref_shuffle_indices(m, 1000 + b, variant, 24)
            rows.append({"b": b, "fnv": fnv(p), "head": [int(v) for v in p[:4]]})
        batched.append({"m": m, "seed": 1000, "variant": variant, "rounds": 24, "rows": rows})
    g["batched"] = batched

    if args.full:
        big = []
        for m, variant in [(1 << 29, PHILOX), ((1 << 29) + 1, PHILOX), ((1 << 29) + 1, LCG), (1 << 29, LCG),
                           ((1 << 30) + 1, PHILOX)]:
            _, h = O.ref_time_shuffle_u64(m, 0x5EED, variant, 24, 0)
            big.append({"m": m, "seed": 0x5EED, "variant": variant, "rounds": 24, "values": "iota u64",
                        "fnv": f"{h:016x}"})
            print("full", m, variant, f"{h:016x}", flush=True)
        g["values_full_hash"] = big
    else:
        old = os.path.join(os.path.dirname(__file__), "golden_ref.json")
        if os.path.exists(old):
            g["values_full_hash"] = json.load(open(old)).get("values_full_hash", [])

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_ref.json")
    with open(path, "w") as f:
        json.dump(g, f, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
