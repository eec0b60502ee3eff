"""ctypes loader for the parity checkers.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module.  It exposes
  * C   -- oracle/liboracle.so, the plain-C restatement of the reference
           algorithm (oracle/bijshuf_oracle.c);
  * REF -- oracle/_ref/libbijshuf_ref*.so, the unmodified reference headers
           compiled behind oracle/ref_driver.cpp (None when not built).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_double, c_int, c_size_t, c_uint32, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libbijshuf_ref.so")
REF_SCALAR_SO = os.path.join(HERE, "_ref", "libbijshuf_ref_scalar.so")

LCG, PHILOX = 0, 1


def _cpu_has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            return " avx512f" in f.read()
    except OSError:
        return False


def build_oracle() -> None:
    """Compile liboracle.so (gcc, seconds); the reference build needs /root/reference."""
    subprocess.run(["make", "-C", HERE, os.path.join(HERE, "liboracle.so")], check=True,
                   stdout=subprocess.DEVNULL)


def _load_c():
    if not os.path.exists(ORACLE_SO):
        build_oracle()
    lib = ctypes.CDLL(ORACLE_SO)
    sig = {
        "orc_mix64": (c_uint64, [c_uint64]),
        "orc_derive_round_keys": (c_int, [c_uint64, c_int, POINTER(c_uint32)]),
        "orc_make_lcg": (c_int, [c_int, c_uint64, POINTER(c_uint64), POINTER(c_uint64)]),
        "orc_lcg_apply": (c_int, [c_int, c_uint64, c_uint64, c_uint64, POINTER(c_uint64)]),
        "orc_philox_apply": (c_int, [c_int, POINTER(c_uint32), c_int, c_uint64, POINTER(c_uint64)]),
        "orc_philox_invert": (c_int, [c_int, POINTER(c_uint32), c_int, c_uint64, POINTER(c_uint64)]),
        "orc_domain_bits": (c_int, [c_uint64]),
        "orc_shuffle_indices": (c_int, [c_uint64, c_uint64, c_int, c_int, c_void_p]),
        "orc_shuffle_indices_range": (c_int, [c_uint64, c_uint64, c_int, c_int, c_uint64, c_uint64, c_void_p,
                                              POINTER(c_uint64)]),
        "orc_shuffle_values": (c_int, [c_void_p, c_void_p, c_uint64, c_size_t, c_uint64, c_int, c_int]),
        "orc_shuffle_values_batched": (c_int, [c_void_p, c_void_p, c_uint64, c_uint64, c_size_t, c_uint64, c_int,
                                               c_int]),
        "orc_gather": (None, [c_void_p, c_void_p, c_void_p, c_uint64, c_size_t]),
        "orc_fnv1a64_u64": (c_uint64, [c_void_p, c_uint64]),
        "orc_is_valid_permutation": (c_int, [c_void_p, c_uint64, c_void_p]),
    }
    for k, (r, a) in sig.items():
        f = getattr(lib, k)
        f.restype = r
        f.argtypes = a
    return lib


def _load_ref():
    path = REF_SO if (_cpu_has_avx512() and os.path.exists(REF_SO)) else REF_SCALAR_SO
    if not os.path.exists(path):
        return None
    lib = ctypes.CDLL(path)
    sig = {
        "ref_avx512_active": (c_int, []),
        "ref_hardware_threads": (c_int, []),
        "ref_mix64": (c_uint64, [c_uint64]),
        "ref_derive_round_keys": (c_int, [c_uint64, c_int, POINTER(c_uint32)]),
        "ref_domain_bits": (c_int, [c_uint64]),
        "ref_philox_apply": (c_int, [c_int, c_uint64, c_int, c_uint64, POINTER(c_uint64)]),
        "ref_philox_apply_many": (c_int, [c_int, c_uint64, c_int, c_void_p, c_uint64, c_void_p]),
        "ref_philox_invert": (c_int, [c_int, c_uint64, c_int, c_uint64, POINTER(c_uint64)]),
        "ref_make_lcg": (c_int, [c_int, c_uint64, POINTER(c_uint64), POINTER(c_uint64)]),
        "ref_shuffle_indices": (c_int, [c_uint64, c_uint64, c_int, c_int, c_int, c_void_p]),
        "ref_shuffle_values": (c_int, [c_void_p, c_void_p, c_uint64, c_uint32, c_uint64, c_int, c_int, c_int]),
        "ref_time_shuffle_u64": (c_int, [c_uint64, c_uint64, c_int, c_int, c_int, c_int, POINTER(c_double),
                                         POINTER(c_uint64)]),
        "ref_time_shuffle_u64_calls": (c_int, [c_uint64, c_uint64, c_int, c_int, c_int, c_int, c_void_p,
                                               POINTER(c_uint64)]),
        "ref_time_shuffle_pairs_calls": (c_int, [c_uint64, c_uint64, c_int, c_int, c_int, c_int, c_void_p]),
        "ref_time_batched_u32_calls": (c_int, [c_uint64, c_uint64, c_uint64, c_int, c_int, c_int, c_int, c_void_p]),
    }
    for k, (r, a) in sig.items():
        f = getattr(lib, k)
        f.restype = r
        f.argtypes = a
    lib.path = path
    return lib


C = _load_c()
REF = _load_ref()

U64 = 0xFFFFFFFFFFFFFFFF


# ---------------------------------------------------------- C restatement --
def keys(seed: int, rounds: int):
    k = (c_uint32 * max(rounds, 1))()
    rc = C.orc_derive_round_keys(seed & U64, rounds, k)
    if rc:
        raise ValueError("derive_round_keys")
    return k


def philox_apply(bits: int, seed: int, rounds: int, x: int) -> int:
    y = c_uint64()
    rc = C.orc_philox_apply(bits, keys(seed, rounds), rounds, x, ctypes.byref(y))
    if rc:
        raise ValueError(rc)
    return y.value


def philox_invert(bits: int, seed: int, rounds: int, y: int) -> int:
    x = c_uint64()
    rc = C.orc_philox_invert(bits, keys(seed, rounds), rounds, y, ctypes.byref(x))
    if rc:
        raise ValueError(rc)
    return x.value


def make_lcg(bits: int, seed: int):
    a, c = c_uint64(), c_uint64()
    rc = C.orc_make_lcg(bits, seed & U64, ctypes.byref(a), ctypes.byref(c))
    if rc:
        raise ValueError(rc)
    return a.value, c.value


def shuffle_indices(m: int, seed: int = 0, variant: int = PHILOX, rounds: int = 24) -> np.ndarray:
    out = np.empty(max(m, 1), dtype=np.uint64)
    rc = C.orc_shuffle_indices(m, seed & U64, variant, rounds, out.ctypes.data)
    if rc:
        raise ValueError(rc)
    return out[:m]


def shuffle_indices_range(m: int, seed: int, variant: int, rounds: int, c0: int, c1: int) -> np.ndarray:
    out = np.empty(max(c1 - c0, 1), dtype=np.uint64)
    cnt = c_uint64()
    rc = C.orc_shuffle_indices_range(m, seed & U64, variant, rounds, c0, c1, out.ctypes.data, ctypes.byref(cnt))
    if rc:
        raise ValueError(rc)
    return out[:cnt.value]


def shuffle_values(values: np.ndarray, seed: int = 0, variant: int = PHILOX, rounds: int = 24) -> np.ndarray:
    values = np.ascontiguousarray(values)
    out = np.empty_like(values)
    rc = C.orc_shuffle_values(values.ctypes.data, out.ctypes.data, values.shape[0], values.itemsize *
                              (values.size // max(values.shape[0], 1)), seed & U64, variant, rounds)
    if rc:
        raise ValueError(rc)
    return out


def shuffle_values_batched(values: np.ndarray, seed: int, variant: int = PHILOX, rounds: int = 24) -> np.ndarray:
    values = np.ascontiguousarray(values)
    out = np.empty_like(values)
    batch, m = values.shape[0], values.shape[1]
    rc = C.orc_shuffle_values_batched(values.ctypes.data, out.ctypes.data, batch, m, values.itemsize, seed & U64,
                                      variant, rounds)
    if rc:
        raise ValueError(rc)
    return out


def fnv1a64(a: np.ndarray) -> int:
    a = np.ascontiguousarray(a, dtype=np.uint64)
    return int(C.orc_fnv1a64_u64(a.ctypes.data, a.size))


def is_valid_permutation(p: np.ndarray) -> bool:
    p = np.ascontiguousarray(p, dtype=np.uint64)
    scratch = np.empty(max(p.size, 1), dtype=np.uint8)
    return bool(C.orc_is_valid_permutation(p.ctypes.data, p.size, scratch.ctypes.data))


# ------------------------------------------------------------- reference --
def ref_shuffle_indices(m: int, seed: int = 0, variant: int = PHILOX, rounds: int = 24, workers: int = 0):
    out = np.empty(max(m, 1), dtype=np.uint64)
    rc = REF.ref_shuffle_indices(m, seed & U64, variant, rounds, workers, out.ctypes.data)
    if rc:
        raise ValueError(rc)
    return out[:m]


def ref_time_shuffle_u64(m: int, seed: int, variant: int, rounds: int, trials: int, workers: int = 0):
    """Mean seconds of the reference shuffle_values_into on iota u64 (bench_bijective) and output FNV."""
    mean, fnv = c_double(), c_uint64()
    rc = REF.ref_time_shuffle_u64(m, seed & U64, variant, rounds, workers, trials, ctypes.byref(mean),
                                  ctypes.byref(fnv))
    if rc:
        raise ValueError(rc)
    return mean.value, fnv.value
