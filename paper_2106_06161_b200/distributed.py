"""Multi-GPU bijective shuffle: one process per GPU, torch.distributed for the
plumbing (NCCL on GPUs; gloo works for the host logic).

The scheme of the north star:
  1. the padded counter domain [0, 2^bits) is split into `world` contiguous
     ranges (bsg_dist_counter_range);
  2. each rank runs the fused kernel on its range (bsg_shuffle_range): the
     survivors of a range are a contiguous run of the global output, written
     to the rank's local buffer in counter order;
  3. ranks all-gather their survivor counts (one u64 per rank -- an 8-element
     NCCL all-gather) and take the exclusive prefix as their global offset;
  4. optionally `rebalance` moves the pieces into equal contiguous output
     shards with one all-to-all of contiguous runs (only boundary slack moves).
Payload reads go to the local replica, or to peer HBM over NVLink through
CUDA-IPC-mapped shard pointers when the input is sharded (`ipc_shards`).
The output is bit-identical to the single-GPU shuffle of all m elements.
"""
from __future__ import annotations

import ctypes
from typing import Callable, List, Optional, Sequence, Tuple

from . import ShuffleConfig, _lib
from ._lib import check, lib


def counter_range(m: int, rank: int, world: int) -> Tuple[int, int]:
    """Counter range [begin, end) of the padded domain owned by `rank`."""
    b, e = ctypes.c_uint64(), ctypes.c_uint64()
    check(lib.bsg_dist_counter_range(m, rank, world, ctypes.byref(b), ctypes.byref(e)), "dist_counter_range")
    return b.value, e.value


def offsets_from_counts(counts: Sequence[int], rank: int) -> int:
    """Exclusive prefix of the gathered survivor counts: this rank's first global output position."""
    return int(sum(int(c) for c in counts[:rank]))


def equal_shards(m: int, world: int) -> List[Tuple[int, int]]:
    """Target layout for `rebalance`: contiguous, near-equal output shards."""
    base, rem = divmod(m, world)
    out, start = [], 0
    for r in range(world):
        n = base + (1 if r < rem else 0)
        out.append((start, start + n))
        start += n
    return out


def transfer_plan(counts: Sequence[int], m: int, world: int) -> List[List[int]]:
    """send[src][dst] = elements rank src sends to rank dst so that piece
    [off_src, off_src + count_src) lands in the equal shards."""
    shards = equal_shards(m, world)
    plan = [[0] * world for _ in range(world)]
    off = 0
    for src, c in enumerate(counts):
        lo, hi = off, off + int(c)
        for dst, (a, b) in enumerate(shards):
            ov = min(hi, b) - max(lo, a)
            if ov > 0:
                plan[src][dst] = ov
        off = hi
    return plan


def _gpu_range(m: int, cfg: ShuffleConfig, begin: int, end: int, values, out, shards=None) -> int:
    """Fused kernel on one counter range; returns the survivor count (device path, current stream)."""
    import torch
    count = ctypes.c_uint64()
    stream = torch.cuda.current_stream(out.device).cuda_stream
    elem = out.element_size()
    check(lib.bsg_shuffle_range(m, ctypes.byref(cfg._c()), begin, end,
                                values.data_ptr() if values is not None else None,
                                ctypes.byref(shards) if shards is not None else None, out.data_ptr(), elem,
                                ctypes.addressof(count), stream), "shuffle_range")
    return count.value


def shuffle_values(values, m: int, cfg: Optional[ShuffleConfig] = None, group=None, out=None, shards=None,
                   range_fn: Optional[Callable] = None, dtype=None):
    """Distributed shuffle of m elements.

    values: the full input replicated on this rank (or None with `shards`, the `.table` of `ipc_shards`, in which
    case `out` or `dtype` gives the element type).
    Returns (piece, global_offset, counts): piece[:counts[rank]] are global output positions
    [global_offset, global_offset + counts[rank]).
    `range_fn(m, cfg, begin, end, values, out) -> count` replaces the GPU kernel (tests inject the oracle).
    """
    import torch
    import torch.distributed as dist
    cfg = cfg or ShuffleConfig()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if m <= 2:
        raise _lib.InvalidArgument("distributed shuffle needs m >= 3")
    begin, end = counter_range(m, rank, world)
    if out is None:
        like = values if values is not None else None
        dtype = like.dtype if like is not None else (dtype or torch.int64)
        device = like.device if like is not None else torch.device("cuda", torch.cuda.current_device())
        out = torch.empty(end - begin, dtype=dtype, device=device)
    fn = range_fn or (lambda *a: _gpu_range(*a, shards=shards))
    cnt = fn(m, cfg, begin, end, values, out)
    dev = out.device
    mine = torch.tensor([cnt], dtype=torch.int64, device=dev)
    allc = torch.zeros(world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(allc, mine, group=group)  # the 8-byte-per-rank count exchange
    counts = [int(x) for x in allc.tolist()]
    if sum(counts) != m:
        raise _lib.CudaError(f"survivor counts {counts} do not sum to m={m}")
    return out, offsets_from_counts(counts, rank), counts


def rebalance(piece, counts: Sequence[int], m: int, group=None):
    """Move the per-rank pieces into equal contiguous output shards (one all-to-all of contiguous runs)."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    plan = transfer_plan(counts, m, world)
    send = plan[rank]
    recv = [plan[src][rank] for src in range(world)]
    out = torch.empty(sum(recv), dtype=piece.dtype, device=piece.device)
    dist.all_to_all_single(out, piece[:counts[rank]].contiguous(), output_split_sizes=recv,
                           input_split_sizes=send, group=group)
    return out


def _gpu_route(local, m, cfg, rank, world):
    import torch
    S = local.numel()
    vals = torch.empty_like(local)
    dl = torch.empty(S, dtype=torch.int32, device=local.device)
    counts = (ctypes.c_uint64 * world)()
    stream = torch.cuda.current_stream(local.device).cuda_stream
    check(lib.bsg_route_by_dest(local.data_ptr(), S, rank * S, m, ctypes.byref(cfg._c()), world, vals.data_ptr(),
                                dl.data_ptr(), counts, local.element_size(), stream), "route_by_dest")
    return vals, dl, [int(c) for c in counts]


def _gpu_scatter(vals, dest, n):
    import torch
    out = torch.empty(n, dtype=vals.dtype, device=vals.device)
    stream = torch.cuda.current_stream(vals.device).cuda_stream
    check(lib.bsg_scatter_permutation(vals.data_ptr(), dest.data_ptr(), n, out.data_ptr(), vals.element_size(),
                                      stream), "scatter_permutation")
    return out


def shuffle_values_sharded(local_shard, m: int, cfg: Optional[ShuffleConfig] = None, group=None,
                           route_fn: Optional[Callable] = None, scatter_fn: Optional[Callable] = None):
    """Power-of-two shuffle of an input sharded in `world` equal contiguous pieces; returns this rank's
    equal output shard out[rank*S:(rank+1)*S].  Bulk transfers only:
    route local elements by destination rank (f^-1, bsg_route_by_dest), one NCCL all-to-all of the
    groups (values and in-shard destinations), then place them (bsg_scatter_permutation)."""
    import torch
    import torch.distributed as dist
    cfg = cfg or ShuffleConfig()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if m & (m - 1) or m % world or local_shard.numel() != m // world:
        raise _lib.InvalidArgument("sharded shuffle: m must be a power of two split evenly over the ranks")
    S = m // world
    vals, dl, send = (route_fn or _gpu_route)(local_shard, m, cfg, rank, world)
    dev = local_shard.device
    sc = torch.tensor(send, dtype=torch.int64, device=dev)
    rc = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_to_all_single(rc, sc, group=group)  # group sizes
    recv = [int(x) for x in rc.tolist()]
    if sum(recv) != S:
        raise _lib.CudaError(f"sharded shuffle: received {sum(recv)} elements for a shard of {S}")
    rv = torch.empty(S, dtype=vals.dtype, device=dev)
    rd = torch.empty(S, dtype=dl.dtype, device=dev)
    dist.all_to_all_single(rv, vals, output_split_sizes=recv, input_split_sizes=send, group=group)
    dist.all_to_all_single(rd, dl, output_split_sizes=recv, input_split_sizes=send, group=group)
    return (scatter_fn or _gpu_scatter)(rv, rd, S)


IPC_HANDLE_BYTES = 80  # BSG_IPC_HANDLE_BYTES: CUDA IPC handle of the allocation + offset of the shard in it


class IpcShards:
    """The bsg_shards table of a sharded input (every rank's shard mapped into this process) and the peer
    mappings behind it; `close()` (or a with-block) unmaps them."""

    def __init__(self, table, opened):
        self.table = table
        self._opened = opened

    def close(self):
        while self._opened:
            check(lib.bsg_ipc_close(self._opened.pop()), "ipc_close")

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def ipc_shards(local_shard, group=None) -> IpcShards:
    """Exchange CUDA IPC handles of each rank's equally sized input shard and map every peer's shard
    (NVLink peer reads).  Handles carry the shard's offset inside its allocation, so tensors from PyTorch's
    caching allocator map correctly.  Returns an IpcShards whose `.table` is the bsg_shards table for
    `shuffle_values(..., shards=...)`; close it when done."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    h = (ctypes.c_ubyte * IPC_HANDLE_BYTES)()
    check(lib.bsg_ipc_export(local_shard.data_ptr(), h), "ipc_export")
    handles = [None] * world
    dist.all_gather_object(handles, (bytes(h), local_shard.numel()), group=group)
    sizes = {n for _, n in handles}
    if len(sizes) != 1:
        raise _lib.InvalidArgument("input shards must be equally sized")
    tab = _lib.bsg_shards()
    opened = []
    try:
        for g, (hb, _) in enumerate(handles):
            if g == rank:
                tab.ptrs[g] = local_shard.data_ptr()
                continue
            p = ctypes.c_void_p()
            check(lib.bsg_ipc_open((ctypes.c_ubyte * IPC_HANDLE_BYTES).from_buffer_copy(hb), ctypes.byref(p)),
                  "ipc_open")
            opened.append(p.value)
            tab.ptrs[g] = p.value
    except BaseException:
        IpcShards(tab, opened).close()
        raise
    tab.count = world
    tab.shard_elems = sizes.pop()
    return IpcShards(tab, opened)


class ExchangeShuffle:
    """Two-rank exchange-partitioned shuffle of a power-of-two domain sharded in halves (bsg_xpart_*, DESIGN.md
    section 7): rank r holds input elements and output positions [r*m/2, (r+1)*m/2).  Each rank streams its input
    half through the inverse cipher once and appends every element to its destination bucket in the owner rank's
    workspace -- rank 0 from the bucket's front, rank 1 from its back, so the buckets end up exactly full (peer
    stores through a CUDA-IPC mapping, NVLink between GPUs, no remote atomics); then each rank partitions and
    places its own buckets.  The concatenated halves equal the single-GPU shuffle.
    The workspaces are allocated and mapped once (m and the element type fixed); `close()` unmaps the peer's."""

    def __init__(self, m: int, dtype, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.group = group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.m = int(m)
        self.itemsize = torch.empty((), dtype=dtype).element_size()
        nbytes = ctypes.c_uint64()
        check(lib.bsg_xpart_workspace_bytes(self.m, self.itemsize, self.world, ctypes.byref(nbytes)),
              "xpart_workspace_bytes")
        device = device or torch.device("cuda", torch.cuda.current_device())
        self.ws = torch.empty(nbytes.value, dtype=torch.uint8, device=device)
        h = (ctypes.c_ubyte * IPC_HANDLE_BYTES)()
        check(lib.bsg_ipc_export(self.ws.data_ptr(), h), "ipc_export")
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(h), group=group)
        self._opened = []
        self.ptrs = (ctypes.c_void_p * self.world)()
        for g, hb in enumerate(handles):
            if g == self.rank:
                self.ptrs[g] = self.ws.data_ptr()
                continue
            p = ctypes.c_void_p()
            check(lib.bsg_ipc_open((ctypes.c_ubyte * IPC_HANDLE_BYTES).from_buffer_copy(hb), ctypes.byref(p)),
                  "ipc_open")
            self._opened.append(p.value)
            self.ptrs[g] = p.value

    def route(self, local_half, cfg: ShuffleConfig):
        """Pass 1 of this rank (asynchronous on the current stream)."""
        import torch
        stream = torch.cuda.current_stream(local_half.device).cuda_stream
        check(lib.bsg_xpart_route(local_half.data_ptr(), self.m, self.itemsize, ctypes.byref(cfg._c()), self.rank,
                                  self.world, self.ptrs, stream), "xpart_route")

    def place(self, out_half):
        """Passes 2 and 3 of this rank's buckets (after every rank's route finished)."""
        import torch
        stream = torch.cuda.current_stream(out_half.device).cuda_stream
        check(lib.bsg_xpart_place(self.m, self.itemsize, self.rank, self.world, self.ptrs, out_half.data_ptr(),
                                  stream), "xpart_place")

    def shuffle(self, local_half, cfg: Optional[ShuffleConfig] = None, out=None):
        """This rank's output half.  Host barriers order the passes across the pair: nobody appends into a
        workspace (or resets its cursors) before its owner finished the previous place, and nobody places
        before every rank's route completed."""
        import torch
        import torch.distributed as dist
        cfg = cfg or ShuffleConfig()
        if local_half.numel() * self.world != self.m or local_half.element_size() != self.itemsize:
            raise _lib.InvalidArgument("exchange shuffle: local half of m elements of the workspace's type")
        out = torch.empty_like(local_half) if out is None else out
        torch.cuda.current_stream(local_half.device).synchronize()
        dist.barrier(group=self.group)
        self.route(local_half, cfg)
        torch.cuda.current_stream(local_half.device).synchronize()
        dist.barrier(group=self.group)
        self.place(out)
        return out

    def close(self):
        while self._opened:
            check(lib.bsg_ipc_close(self._opened.pop()), "ipc_close")

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
