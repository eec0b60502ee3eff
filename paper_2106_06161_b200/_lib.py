"""ctypes binding of libbsg.so (the C ABI declared in include/bsg.h).

The product path has no CPU fallback: if the CUDA library is missing this
module raises at import time, and every data-path call returns a CUDA error
when no GPU is present.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import (POINTER, Structure, c_char_p, c_int32, c_uint32, c_uint64, c_ubyte, c_void_p)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BSG_LIB") or os.path.join(_HERE, "lib", "libbsg.so")  # BSG_LIB: experiment builds

# bsg_status
OK, EINVAL, ERANGE, EALIAS, ENOMEM, ECUDA, ENODEV, EUNSUPPORTED = range(8)


class bsg_config(Structure):
    _fields_ = [("seed", c_uint64), ("variant", c_int32), ("num_rounds", c_int32), ("workers", c_int32),
                ("reserved", c_int32)]


class bsg_shards(Structure):
    _fields_ = [("ptrs", c_void_p * 16), ("count", c_int32), ("reserved", c_int32), ("shard_elems", c_uint64)]


class bsg_philox_params(Structure):
    _fields_ = [("total_bits", c_int32), ("left_side_bits", c_int32), ("right_side_bits", c_int32),
                ("num_rounds", c_int32), ("left_side_mask", c_uint64), ("right_side_mask", c_uint64),
                ("round_keys", POINTER(c_uint32)), ("num_keys", c_uint64)]


ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, POINTER(c_uint64), POINTER(c_uint64), c_void_p)

# name -> (restype, argtypes); every symbol of include/bsg.h
SIGNATURES = {
    "bsg_config_default": (bsg_config, []),
    "bsg_mix64": (c_uint64, [c_uint64]),
    "bsg_derive_round_keys": (c_int32, [c_uint64, c_int32, POINTER(c_uint32)]),
    "bsg_domain_bits": (c_int32, [c_uint64]),
    "bsg_make_lcg": (c_int32, [c_int32, c_uint64, POINTER(c_uint64), POINTER(c_uint64)]),
    "bsg_lcg_apply": (c_int32, [c_int32, c_uint64, c_uint64, c_uint64, POINTER(c_uint64)]),
    "bsg_philox_apply": (c_int32, [c_int32, c_uint64, c_int32, c_uint64, POINTER(c_uint64)]),
    "bsg_philox_invert": (c_int32, [c_int32, c_uint64, c_int32, c_uint64, POINTER(c_uint64)]),
    "bsg_philox_apply_params": (c_int32, [POINTER(bsg_philox_params), c_uint64, POINTER(c_uint64)]),
    "bsg_philox_invert_params": (c_int32, [POINTER(bsg_philox_params), c_uint64, POINTER(c_uint64)]),
    "bsg_bijection_apply": (c_int32, [c_int32, c_int32, c_uint64, c_int32, c_int32, c_void_p, c_uint64, c_void_p,
                                      c_uint64, c_void_p]),
    "bsg_shuffle_indices": (c_int32, [c_uint64, POINTER(bsg_config), c_void_p, c_void_p]),
    "bsg_shuffle_values": (c_int32, [c_void_p, c_void_p, c_uint64, c_uint32, POINTER(bsg_config), c_void_p]),
    "bsg_shuffle_values_batched": (c_int32, [c_void_p, c_void_p, c_uint64, c_uint64, c_uint32, POINTER(bsg_config),
                                             c_void_p]),
    "bsg_gather": (c_int32, [c_void_p, c_uint64, c_void_p, c_void_p, c_uint64, c_uint32, c_void_p]),
    "bsg_shuffle_range": (c_int32, [c_uint64, POINTER(bsg_config), c_uint64, c_uint64, c_void_p, POINTER(bsg_shards),
                                    c_void_p, c_uint32, c_void_p, c_void_p]),
    "bsg_range_count": (c_int32, [c_uint64, POINTER(bsg_config), c_uint64, c_uint64, POINTER(c_uint64), c_void_p]),
    "bsg_dist_shuffle_values": (c_int32, [c_uint64, POINTER(bsg_config), c_int32, c_int32, c_void_p,
                                          POINTER(bsg_shards), c_void_p, c_uint32, ALLGATHER_FN, c_void_p,
                                          POINTER(c_uint64), POINTER(c_uint64), c_void_p]),
    "bsg_dist_counter_range": (c_int32, [c_uint64, c_int32, c_int32, POINTER(c_uint64), POINTER(c_uint64)]),
    "bsg_route_by_dest": (c_int32, [c_void_p, c_uint64, c_uint64, c_uint64, POINTER(bsg_config), c_int32, c_void_p,
                                    c_void_p, POINTER(c_uint64), c_uint32, c_void_p]),
    "bsg_scatter_permutation": (c_int32, [c_void_p, c_void_p, c_uint64, c_void_p, c_uint32, c_void_p]),
    "bsg_ipc_export": (c_int32, [c_void_p, POINTER(c_ubyte)]),
    "bsg_ipc_open": (c_int32, [POINTER(c_ubyte), POINTER(c_void_p)]),
    "bsg_ipc_close": (c_int32, [c_void_p]),
    "bsg_pipeline_create": (c_int32, [c_uint64, c_uint32, c_int32, POINTER(c_void_p)]),
    "bsg_pipeline_submit": (c_int32, [c_void_p, c_void_p, c_void_p, c_uint64, POINTER(bsg_config), POINTER(c_uint64)]),
    "bsg_pipeline_submit_batched": (c_int32, [c_void_p, c_void_p, c_void_p, c_uint64, c_uint64, POINTER(bsg_config),
                                              POINTER(c_uint64)]),
    "bsg_pipeline_wait": (c_int32, [c_void_p, c_uint64]),
    "bsg_pipeline_destroy": (c_int32, [c_void_p]),
    "bsg_sort_shuffle_u64": (c_int32, [c_void_p, c_void_p, c_uint64, c_uint64, c_void_p]),
    "bsg_status_string": (c_char_p, [c_int32]),
    "bsg_last_error": (c_char_p, []),
    "bsg_version": (c_int32, []),
    "bsg_kernel_launches": (c_uint64, []),
    "bsg_set_force_compact": (c_int32, [c_int32]),
    "bsg_set_path": (c_int32, [c_int32]),
    "bsg_set_rank_stage_cap": (c_uint32, [c_uint32]),
    "bsg_xpart_workspace_bytes": (c_int32, [c_uint64, c_uint32, c_int32, POINTER(c_uint64)]),
    "bsg_xpart_route": (c_int32, [c_void_p, c_uint64, c_uint32, POINTER(bsg_config), c_int32, c_int32,
                                  POINTER(c_void_p), c_void_p]),
    "bsg_xpart_place": (c_int32, [c_uint64, c_uint32, c_int32, c_int32, POINTER(c_void_p), c_void_p, c_void_p]),
    "bsg_set_bulk_stores": (c_int32, [c_int32]),
    "bsg_workspace_bytes": (c_int32, [POINTER(c_uint64)]),
    "bsg_release_workspace": (c_int32, []),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libbsg.so not found at {LIB_PATH}: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


class BsgError(RuntimeError):
    """Base class of errors raised by the shuffle library."""


class InvalidArgument(BsgError, ValueError):
    """std::invalid_argument of the reference."""


class OutOfRange(BsgError, IndexError):
    """std::out_of_range of the reference."""


class CudaError(BsgError):
    """CUDA runtime failure (includes 'no CUDA device')."""


def check(status: int, what: str = "") -> None:
    if status == OK:
        return
    detail = lib.bsg_last_error().decode()
    msg = f"{what}: {lib.bsg_status_string(status).decode()}" + (f" ({detail})" if detail else "")
    if status in (EINVAL, EALIAS, EUNSUPPORTED):
        raise InvalidArgument(msg)
    if status == ERANGE:
        raise OutOfRange(msg)
    if status == ENOMEM:
        raise MemoryError(msg)
    raise CudaError(msg)
