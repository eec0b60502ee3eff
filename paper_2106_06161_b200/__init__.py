"""B200-native bijective shuffle -- Python mirror of the reference `bijshuf` API.

Every function keeps the name, argument meaning and error behaviour of the
reference header it cites (/root/reference/proj/include/bijshuf/...), and
runs on the GPU through the C ABI of libbsg.so (include/bsg.h):

    reference (C++)                          here
    ---------------------------------------  --------------------------------------
    ShuffleConfig, BijectionVariant          ShuffleConfig, BijectionVariant
      (shuffle.hpp:20-30)
    shuffle_domain_bits (shuffle.hpp:49-52)  shuffle_domain_bits
    shuffle_indices[_into] (:280-293)        shuffle_indices[_into]
    shuffle_values[_into]<T> (:298-315)      shuffle_values[_into]
    gather[_into]<T> (:340-362)              gather[_into]
    compact_permutation (:34-42)             compact_permutation
    mix64, derive_round_keys (splitmix.hpp)  mix64, derive_round_keys
    make_lcg/lcg_apply, make_philox/         make_lcg/lcg_apply, make_philox/
      philox_apply/philox_invert               philox_apply/philox_invert
      (bijection.hpp)
    BijectiveShuffleSampler (stats.hpp:314)  shuffle_values_batched (seed + b)

Arrays are numpy arrays (host memory) or torch tensors (host or CUDA).  CUDA
tensors run asynchronously on torch's current stream; host arrays are staged
through device memory and the call returns with the result on the host.
std::invalid_argument maps to InvalidArgument (a ValueError),
std::out_of_range to OutOfRange (an IndexError).
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field
from typing import Any, List, Optional

import numpy as np

from . import _lib
from ._lib import BsgError, CudaError, InvalidArgument, OutOfRange, check, lib

__all__ = [
    "BijectionVariant", "ShuffleConfig", "shuffle_domain_bits", "shuffle_indices", "shuffle_indices_into",
    "shuffle_values", "shuffle_values_into", "shuffle_values_batched", "gather", "gather_into",
    "compact_permutation", "mix64", "derive_round_keys", "LcgParams", "make_lcg", "lcg_apply",
    "VariablePhiloxParams", "make_philox", "philox_apply", "philox_invert", "bijection_apply", "sort_shuffle_u64",
    "SplitMix64", "BijectionSpec", "make_bijection", "workspace_bytes", "release_workspace",
    "kernel_launches", "Pipeline", "BsgError", "CudaError", "InvalidArgument", "OutOfRange", "Permutation",
]

Permutation = np.ndarray  # permutation.hpp:15 -- one-line notation, entry k = source index of slot k


class BijectionVariant(enum.IntEnum):  # shuffle.hpp:20
    Lcg = 0
    VariablePhilox = 1


@dataclass
class ShuffleConfig:  # shuffle.hpp:25-30
    seed: int = 0
    variant: BijectionVariant = BijectionVariant.VariablePhilox
    num_rounds: int = 24
    workers: int = 0  # accepted for API parity; the GPU output never depends on it

    def _c(self) -> _lib.bsg_config:
        return _lib.bsg_config(self.seed & 0xFFFFFFFFFFFFFFFF, int(self.variant), int(self.num_rounds),
                               int(self.workers), 0)


# ----------------------------------------------------------------- buffers --
def _is_torch(x: Any) -> bool:
    return type(x).__module__.startswith("torch")


class _Buf:
    """Pointer view of a numpy array or torch tensor."""

    def __init__(self, x: Any):
        if _is_torch(x):
            if not x.is_contiguous():
                raise InvalidArgument("tensor must be contiguous")
            self.ptr = x.data_ptr()
            self.itemsize = x.element_size()
            self.nelem = x.numel()
            self.cuda = x.is_cuda
            self.obj = x
        else:
            if not isinstance(x, np.ndarray):
                raise InvalidArgument("expected a numpy array or torch tensor")
            if not x.flags["C_CONTIGUOUS"]:
                raise InvalidArgument("array must be C-contiguous")
            self.ptr = x.ctypes.data
            self.itemsize = x.itemsize
            self.nelem = x.size
            self.cuda = False
            self.obj = x

    def stream(self) -> Optional[int]:
        if self.cuda:
            import torch
            return torch.cuda.current_stream(self.obj.device).cuda_stream
        return None


def _stream_of(*bufs: _Buf) -> Optional[int]:
    for b in bufs:
        if b.cuda:
            return b.stream()
    return None


def _empty_like(x: Any, n: int, dtype=None):
    if _is_torch(x):
        import torch
        return torch.empty(n, dtype=dtype or x.dtype, device=x.device)
    return np.empty(n, dtype=dtype or x.dtype)


def _device_ctx(x: Any):
    """Make x's CUDA device current for the call (the library works on the current device)."""
    if _is_torch(x) and x.is_cuda:
        import torch
        return torch.cuda.device(x.device)
    import contextlib
    return contextlib.nullcontext()


# ------------------------------------------------------------- bijections --
def mix64(z: int) -> int:  # splitmix.hpp:11-15
    return int(lib.bsg_mix64(z & 0xFFFFFFFFFFFFFFFF))


def derive_round_keys(seed: int, num_rounds: int) -> List[int]:  # splitmix.hpp:22-31
    if num_rounds < 1:
        raise InvalidArgument("num_rounds must be >= 1")
    keys = (ctypes.c_uint32 * num_rounds)()
    check(lib.bsg_derive_round_keys(seed & 0xFFFFFFFFFFFFFFFF, num_rounds, keys), "derive_round_keys")
    return list(keys)


def shuffle_domain_bits(m: int) -> int:  # shuffle.hpp:49-52
    return int(lib.bsg_domain_bits(m))


@dataclass
class LcgParams:  # bijection.hpp:14-22
    modulus_bits: int = 0
    a: int = 1
    c: int = 0

    def domain_mask(self) -> int:
        return (1 << 64) - 1 if self.modulus_bits >= 64 else (1 << self.modulus_bits) - 1


def make_lcg(modulus_bits: int, seed: int) -> LcgParams:  # bijection.hpp:25-34
    a, c = ctypes.c_uint64(), ctypes.c_uint64()
    check(lib.bsg_make_lcg(modulus_bits, seed & 0xFFFFFFFFFFFFFFFF, ctypes.byref(a), ctypes.byref(c)), "make_lcg")
    return LcgParams(modulus_bits, a.value, c.value)


def lcg_apply(p: LcgParams, x: int) -> int:  # bijection.hpp:36-40
    y = ctypes.c_uint64()
    if x < 0 or x > p.domain_mask():
        raise OutOfRange("lcg_apply: x outside [0, 2^bits)")
    check(lib.bsg_lcg_apply(p.modulus_bits, p.a, p.c, x, ctypes.byref(y)), "lcg_apply")
    return y.value


@dataclass
class VariablePhiloxParams:  # bijection.hpp:45-53
    total_bits: int = 0
    left_side_bits: int = 0
    right_side_bits: int = 0
    num_rounds: int = 0
    left_side_mask: int = 0
    right_side_mask: int = 0
    round_keys: List[int] = field(default_factory=list)

    def _c(self):
        keys = (ctypes.c_uint32 * max(1, len(self.round_keys)))(*[k & 0xFFFFFFFF for k in self.round_keys])
        p = _lib.bsg_philox_params(self.total_bits, self.left_side_bits, self.right_side_bits, self.num_rounds,
                                   self.left_side_mask & 0xFFFFFFFFFFFFFFFF, self.right_side_mask & 0xFFFFFFFFFFFFFFFF,
                                   ctypes.cast(keys, ctypes.POINTER(ctypes.c_uint32)), len(self.round_keys))
        p._keep = keys
        return p


def make_philox(total_bits: int, seed: int, num_rounds: int = 24) -> VariablePhiloxParams:  # bijection.hpp:73-88
    if total_bits < 2 or total_bits > 63:
        raise InvalidArgument("total_bits must be in [2, 63]")
    if num_rounds < 3:
        raise InvalidArgument("num_rounds must be >= 3")
    L = total_bits // 2
    R = total_bits - L
    return VariablePhiloxParams(total_bits, L, R, num_rounds, (1 << L) - 1, (1 << R) - 1,
                                derive_round_keys(seed, num_rounds))


def philox_apply(p: VariablePhiloxParams, x: int) -> int:  # bijection.hpp:94-111 (honours every field of p)
    if x < 0 or (p.total_bits < 64 and (x >> p.total_bits) != 0):
        raise OutOfRange("philox_apply: x outside [0, 2^total_bits)")
    y = ctypes.c_uint64()
    check(lib.bsg_philox_apply_params(ctypes.byref(p._c()), x, ctypes.byref(y)), "philox_apply")
    return y.value


def philox_invert(p: VariablePhiloxParams, y: int) -> int:  # bijection.hpp:117-143 (honours every field of p)
    if y < 0 or (p.total_bits < 64 and (y >> p.total_bits) != 0):
        raise OutOfRange("philox_invert: y outside [0, 2^total_bits)")
    x = ctypes.c_uint64()
    check(lib.bsg_philox_invert_params(ctypes.byref(p._c()), y, ctypes.byref(x)), "philox_invert")
    return x.value


class SplitMix64:  # splitmix.hpp:35-63
    """Counter-based generator over the SplitMix64 stream: draw k of seed s is mix64(s + k * gamma)."""

    GAMMA = 0x9E3779B97F4A7C15

    def __init__(self, seed: int):
        self.state = seed & 0xFFFFFFFFFFFFFFFF

    def __call__(self) -> int:
        self.state = (self.state + self.GAMMA) & 0xFFFFFFFFFFFFFFFF
        return mix64(self.state)

    @staticmethod
    def min() -> int:
        return 0

    @staticmethod
    def max() -> int:
        return 0xFFFFFFFFFFFFFFFF

    def below(self, bound: int) -> int:
        """Unbiased draw from [0, bound) by rejection (splitmix.hpp:49-59)."""
        if bound == 0:
            raise InvalidArgument("bound must be >= 1")
        full = 0xFFFFFFFFFFFFFFFF
        limit = full - (full % bound)
        while True:
            v = self()
            if v < limit:
                return v % bound


@dataclass
class BijectionSpec:  # bijection.hpp:146-150
    variant: Any = None  # LcgParams or VariablePhiloxParams
    domain_bits: int = 0


def make_bijection(p: Any) -> BijectionSpec:  # bijection.hpp:152-158
    if isinstance(p, LcgParams):
        return BijectionSpec(p, p.modulus_bits)
    if isinstance(p, VariablePhiloxParams):
        return BijectionSpec(p, p.total_bits)
    raise InvalidArgument("make_bijection: LcgParams or VariablePhiloxParams expected")


def bijection_spec_apply(spec: BijectionSpec, x: int) -> int:  # bijection.hpp:160-169
    """bijection_apply(const BijectionSpec&, x) of the reference (the GPU batch form is bijection_apply)."""
    if isinstance(spec.variant, LcgParams):
        return lcg_apply(spec.variant, x)
    return philox_apply(spec.variant, x)


def bijection_apply(variant: Any, bits: int = 0, seed: int = 0, num_rounds: int = 24, x: Any = None, *,
                    start: int = 0, n: Optional[int] = None, inverse: bool = False, out: Any = None):
    """GPU batch evaluation y[i] = f(x[i]) (or f^-1).  x=None evaluates counters start..start+n-1.

    Called as bijection_apply(spec, x) with a BijectionSpec and an integer x it is the reference's scalar
    bijection_apply (bijection.hpp:160-169)."""
    if isinstance(variant, BijectionSpec):
        return bijection_spec_apply(variant, bits if x is None else x)
    if x is not None:
        xb = _Buf(x)
        if xb.itemsize != 8:
            raise InvalidArgument("x must hold 64-bit integers")
        n = xb.nelem
        like = x
    else:
        if n is None:
            raise InvalidArgument("n required when x is None")
        xb = None
        like = np.empty(0, dtype=np.uint64)
    if out is None:
        out = _empty_like(like, n, dtype=None if _is_torch(like) else np.uint64)
    ob = _Buf(out)
    with _device_ctx(out):
        check(lib.bsg_bijection_apply(int(variant), bits, seed & 0xFFFFFFFFFFFFFFFF, num_rounds, 1 if inverse else 0,
                                      xb.ptr if xb else None, start, ob.ptr, n, _stream_of(*(b for b in (xb, ob) if b))),
              "bijection_apply")
    return out


# ----------------------------------------------------------------- shuffle --
def compact_permutation(w: Any, m: int):  # shuffle.hpp:34-42 (host helper)
    if m > len(w):
        raise InvalidArgument("compact_permutation: m exceeds length")
    w = np.asarray(w, dtype=np.uint64)
    return w[w < np.uint64(m)]


def shuffle_indices_into(m: int, cfg: ShuffleConfig, out: Any) -> None:  # shuffle.hpp:289-293
    ob = _Buf(out)
    if ob.itemsize != 8 or ob.nelem < m:
        raise InvalidArgument("out must hold m 64-bit entries")
    with _device_ctx(out):
        check(lib.bsg_shuffle_indices(m, ctypes.byref(cfg._c()), ob.ptr, ob.stream()), "shuffle_indices")


def shuffle_indices(m: int, cfg: Optional[ShuffleConfig] = None, device: Any = None):  # shuffle.hpp:280-284
    """Permutation of {0..m-1} as uint64 (numpy; a CUDA tensor when device is given)."""
    cfg = cfg or ShuffleConfig()
    if device is not None:
        import torch
        out = torch.empty(m, dtype=torch.int64, device=device)
    else:
        out = np.empty(m, dtype=np.uint64)
    shuffle_indices_into(m, cfg, out)
    return out


def shuffle_values_into(values: Any, cfg: ShuffleConfig, out: Any) -> None:  # shuffle.hpp:308-315
    if out is values:
        raise InvalidArgument("shuffle_values_into: out aliases input")
    vb, ob = _Buf(values), _Buf(out)
    if ob.nelem * ob.itemsize < vb.nelem * vb.itemsize:
        raise InvalidArgument("out is smaller than values")
    with _device_ctx(values if vb.cuda else out):
        check(lib.bsg_shuffle_values(vb.ptr, ob.ptr, vb.nelem, vb.itemsize, ctypes.byref(cfg._c()),
                                     _stream_of(vb, ob)), "shuffle_values")


def shuffle_values(values: Any, cfg: Optional[ShuffleConfig] = None):  # shuffle.hpp:298-304
    """out[k] = values[sigma(k)], same container kind as `values`."""
    cfg = cfg or ShuffleConfig()
    if _is_torch(values):
        out = values.new_empty(values.shape)
    else:
        out = np.empty_like(values)
    shuffle_values_into(values, cfg, out)
    return out


def shuffle_values_batched(values: Any, cfg: Optional[ShuffleConfig] = None, out: Any = None):
    """Row b of a (batch, m) array shuffled with seed cfg.seed + b (stats.hpp:314-324)."""
    cfg = cfg or ShuffleConfig()
    if len(values.shape) != 2:
        raise InvalidArgument("values must be 2-D (batch, m)")
    batch, m = int(values.shape[0]), int(values.shape[1])
    if out is None:
        out = values.new_empty(values.shape) if _is_torch(values) else np.empty_like(values)
    if out is values:
        raise InvalidArgument("shuffle_values_batched: out aliases input")
    vb, ob = _Buf(values), _Buf(out)
    with _device_ctx(values if vb.cuda else out):
        check(lib.bsg_shuffle_values_batched(vb.ptr, ob.ptr, batch, m, vb.itemsize, ctypes.byref(cfg._c()),
                                             _stream_of(vb, ob)), "shuffle_values_batched")
    return out


def gather_into(src: Any, indices: Any, out: Any, workers: int = 0) -> None:  # shuffle.hpp:352-362
    if out is src or out is indices:
        raise InvalidArgument("gather_into: out aliases an input")
    sb, ib, ob = _Buf(src), _Buf(indices), _Buf(out)
    if ib.itemsize != 8:
        raise InvalidArgument("indices must be 64-bit")
    with _device_ctx(src if sb.cuda else out):
        check(lib.bsg_gather(sb.ptr, sb.nelem, ib.ptr, ob.ptr, ib.nelem, sb.itemsize, _stream_of(sb, ib, ob)),
              "gather")


def gather(src: Any, indices: Any, workers: int = 0):  # shuffle.hpp:340-348
    out = (src.new_empty(indices.shape[0]) if _is_torch(src) else np.empty(len(indices), dtype=src.dtype))
    gather_into(src, indices, out, workers)
    return out


def sort_shuffle_u64(values: Any, seed: int, out: Any = None):
    """The paper's SortShuffle comparator (CUB radix sort of random 64-bit keys); CUDA tensors only."""
    if out is None:
        out = values.new_empty(values.shape)
    vb, ob = _Buf(values), _Buf(out)
    with _device_ctx(values):
        check(lib.bsg_sort_shuffle_u64(vb.ptr, ob.ptr, vb.nelem, seed & 0xFFFFFFFFFFFFFFFF, vb.stream()),
              "sort_shuffle")
    return out


class Pipeline:
    """Streaming shuffles of HOST buffers (bsg_pipeline_*): H2D of shuffle i+1 overlaps the D2H of shuffle i.

    Host arrays should be pinned (torch `pin_memory()`); keep them alive and untouched until `wait(ticket)`.
    """

    def __init__(self, max_m: int, elem_bytes: int, depth: int = 2):
        self._h = ctypes.c_void_p()
        self._keep = {}
        check(lib.bsg_pipeline_create(max_m, elem_bytes, depth, ctypes.byref(self._h)), "pipeline_create")
        self.elem_bytes = elem_bytes

    def submit(self, values: Any, out: Any, cfg: Optional[ShuffleConfig] = None) -> int:
        cfg = cfg or ShuffleConfig()
        vb, ob = _Buf(values), _Buf(out)
        if vb.itemsize * vb.nelem != self.elem_bytes * vb.nelem or ob.nelem * ob.itemsize < vb.nelem * vb.itemsize:
            raise InvalidArgument("pipeline: element size / output size mismatch")
        t = ctypes.c_uint64()
        check(lib.bsg_pipeline_submit(self._h, vb.ptr, ob.ptr, vb.nelem, ctypes.byref(cfg._c()), ctypes.byref(t)),
              "pipeline_submit")
        self._keep[t.value] = (values, out)
        return t.value

    def submit_batched(self, values: Any, out: Any, cfg: Optional[ShuffleConfig] = None) -> int:
        """Rows of a 2-D host array, row b shuffled with seed + b (shuffle_values_batched), streamed."""
        cfg = cfg or ShuffleConfig()
        if len(values.shape) != 2 or tuple(out.shape) != tuple(values.shape):
            raise InvalidArgument("pipeline: batched values must be 2-D (batch, m) and out of the same shape")
        batch, m = int(values.shape[0]), int(values.shape[1])
        vb, ob = _Buf(values), _Buf(out)
        if vb.itemsize != self.elem_bytes or ob.itemsize != self.elem_bytes:
            raise InvalidArgument("pipeline: element size mismatch")
        t = ctypes.c_uint64()
        check(lib.bsg_pipeline_submit_batched(self._h, vb.ptr, ob.ptr, batch, m, ctypes.byref(cfg._c()),
                                              ctypes.byref(t)), "pipeline_submit_batched")
        self._keep[t.value] = (values, out)
        return t.value

    def wait(self, ticket: int) -> None:
        check(lib.bsg_pipeline_wait(self._h, ticket), "pipeline_wait")
        self._keep.pop(ticket, None)

    def close(self) -> None:
        if self._h:
            check(lib.bsg_pipeline_destroy(self._h), "pipeline_destroy")
            self._h = ctypes.c_void_p()
            self._keep.clear()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def workspace_bytes() -> int:
    """Device memory held by the library's cached workspaces on the current device (bsg_workspace_bytes)."""
    b = ctypes.c_uint64()
    check(lib.bsg_workspace_bytes(ctypes.byref(b)), "workspace_bytes")
    return b.value


def release_workspace() -> None:
    """Free the cached workspaces of the current device (bsg_release_workspace); graphs captured from earlier
    calls must not be replayed afterwards."""
    check(lib.bsg_release_workspace(), "release_workspace")


def kernel_launches() -> int:
    """Kernels launched by libbsg.so in this process."""
    return int(lib.bsg_kernel_launches())


def set_path(path: int) -> int:
    """0 = automatic, 1 = single fused pass only, 2 = partitioned passes whenever eligible (whole domains of
    2^14..2^32 counters; non-power-of-two domains for elements of at most 8 bytes).  Outputs are identical."""
    return int(lib.bsg_set_path(int(path)))


def set_rank_stage_cap(cap: int) -> int:
    """Testing knob (bsg_set_rank_stage_cap): survivors per counter window the persistent last pass of padded
    partitioned shuffles stages in shared memory (default and maximum 9216); windows holding more take the
    round-based pass.  Outputs are identical."""
    return int(lib.bsg_set_rank_stage_cap(int(cap)))


def set_bulk_stores(on: bool) -> bool:
    """Testing knob (bsg_set_bulk_stores): the partitioned path's last passes write their placed windows with bulk
    shared->global copies (default) or plain stores.  Outputs are identical."""
    return bool(lib.bsg_set_bulk_stores(1 if on else 0))


def set_force_compact(on: bool) -> bool:
    """Testing knob: route power-of-two sizes through the look-back kernel too."""
    return bool(lib.bsg_set_force_compact(1 if on else 0))
