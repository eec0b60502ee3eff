"""Multi-rank paths with the real GPU kernels: two processes share cuda:0 and talk over gloo (the
driver's multi-GPU runs use one GPU per rank and NCCL; the host logic and kernels are the same)."""
from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import paper_2106_06161_b200 as bsg
    from paper_2106_06161_b200 import distributed as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        # counter-range partition with the replicated input (the north-star scheme)
        for m, variant in ((1000001, 1), (1 << 20, 1), ((1 << 20) + 5, 0)):
            cfg = bsg.ShuffleConfig(seed=m, variant=bsg.BijectionVariant(variant))
            vals = torch.arange(m, dtype=torch.int64, device="cuda") * 3
            piece, off, counts = D.shuffle_values(vals, m, cfg)
            res[("range", m)] = (off, piece[:counts[rank]].cpu().numpy().copy())
            shard = D.rebalance(piece, counts, m)
            res[("rebal", m)] = shard.cpu().numpy().copy()
        # sharded power-of-two input: route by destination + all-to-all + place
        m = 1 << 20
        S = m // world
        local = torch.arange(rank * S, (rank + 1) * S, dtype=torch.int64, device="cuda") * 7
        out = D.shuffle_values_sharded(local, m, bsg.ShuffleConfig(seed=5))
        res[("sharded", m)] = out.cpu().numpy().copy()
        # exchange partition (bsg_xpart_*): input halves, peer stores into the owner's buckets, local P2/P3
        for m, variant, dt, seed, rounds in (((1 << 20), 1, torch.int64, 11, 24), ((1 << 21), 0, torch.int32, 12, 24),
                                             ((1 << 17), 1, torch.int64, 13, 7), ((1 << 22), 1, torch.int32, 14, 24)):
            S = m // world
            local = torch.arange(rank * S, (rank + 1) * S, dtype=dt, device="cuda") * 3 + 1
            cfg = bsg.ShuffleConfig(seed=seed, variant=bsg.BijectionVariant(variant), num_rounds=rounds)
            with D.ExchangeShuffle(m, dt) as X:
                a = X.shuffle(local, cfg)
                b = X.shuffle(local, cfg)  # reuse of the mapped workspaces
                assert torch.equal(a, b)
            res[("xpart", m)] = a.to(torch.int64).cpu().numpy().copy()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_two_ranks_on_one_gpu(orc):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for m, variant in ((1000001, 1), (1 << 20, 1), ((1 << 20) + 5, 0)):
        exp = orc.shuffle_values(np.arange(m, dtype=np.uint64) * 3, m, variant, 24)
        full = np.empty(m, dtype=np.uint64)
        for r in range(world):
            off, piece = out[r][("range", m)]
            full[off:off + len(piece)] = piece.view(np.uint64)
        assert np.array_equal(full, exp), m
        assert np.array_equal(np.concatenate([out[r][("rebal", m)] for r in range(world)]).view(np.uint64), exp)
    m = 1 << 20
    exp = orc.shuffle_values(np.arange(m, dtype=np.uint64) * 7, 5, 1, 24)
    assert np.array_equal(np.concatenate([out[r][("sharded", m)] for r in range(world)]).view(np.uint64), exp)
    for m, variant, seed, rounds in (((1 << 20), 1, 11, 24), ((1 << 21), 0, 12, 24), ((1 << 17), 1, 13, 7),
                                     ((1 << 22), 1, 14, 24)):
        exp = orc.shuffle_indices(m, seed, variant, rounds) * np.uint64(3) + np.uint64(1)
        got = np.concatenate([out[r][("xpart", m)] for r in range(world)]).view(np.uint64)
        assert np.array_equal(got, exp), (m, variant, rounds)


def _ipc_worker(rank, world, port, q):
    """Sharded input with real CUDA IPC: each rank owns one shard placed at an offset inside a larger torch
    allocation (the case the round-1 handle exchange got wrong), maps every peer's shard with ipc_shards and
    shuffles its counter range through the shard table (payload reads through the peer mappings)."""
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import paper_2106_06161_b200 as bsg
    from paper_2106_06161_b200 import distributed as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        for m, variant, eb in (((1 << 21), 1, 8), ((1 << 21) + 11, 1, 8), ((1 << 20) + 3, 0, 16), ((1 << 21), 1, 16)):
            S = (m + world - 1) // world
            lo = rank * S
            if eb == 8:
                big = torch.empty(S + 4096, dtype=torch.int64, device="cuda")
                local = big[4096:]  # 32 KiB into the allocation
                local.copy_(torch.arange(lo, lo + S, dtype=torch.int64, device="cuda") * 3 + 1)
                dtype = torch.int64
            else:
                big = torch.empty((S + 256, 2), dtype=torch.int64, device="cuda")
                local = big[256:]
                idx = torch.arange(lo, lo + S, dtype=torch.int64, device="cuda")
                local[:, 0] = idx
                local[:, 1] = idx * 7 + 5
                local = local.view(torch.complex128).view(-1)
                dtype = torch.complex128
            torch.cuda.synchronize()
            dist.barrier()
            with D.ipc_shards(local) as ipc:
                piece, off, counts = D.shuffle_values(None, m, bsg.ShuffleConfig(seed=m, variant=bsg.BijectionVariant(
                    variant)), shards=ipc.table, dtype=dtype)
                torch.cuda.synchronize()
                dist.barrier()  # peers keep reading this rank's shard until every rank is done
            res[(m, variant, eb)] = (off, piece[:counts[rank]].view(torch.int64).cpu().numpy().copy())
            del big, local
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ipc_sharded_ranks_on_one_gpu(orc, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for m, variant, eb in (((1 << 21), 1, 8), ((1 << 21) + 11, 1, 8), ((1 << 20) + 3, 0, 16), ((1 << 21), 1, 16)):
        perm = orc.shuffle_indices(m, m, variant, 24)
        if eb == 8:
            exp = perm * np.uint64(3) + np.uint64(1)
        else:
            exp = np.stack([perm, perm * np.uint64(7) + np.uint64(5)], axis=1).reshape(-1)
        full = np.empty(m * (eb // 8), dtype=np.uint64)
        k = eb // 8
        for r in range(world):
            off, piece = out[r][(m, variant, eb)]
            full[off * k:off * k + len(piece)] = piece.view(np.uint64)
        assert np.array_equal(full, exp), (world, m, variant, eb)


def _xpart_max_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import paper_2106_06161_b200 as bsg
    from paper_2106_06161_b200 import distributed as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = 1 << 32  # the largest exchange domain: 32-bit global indices and bucket positions
        S = m // world
        local = torch.arange(rank * S, (rank + 1) * S, dtype=torch.int64, device="cuda").to(torch.int32)
        with D.ExchangeShuffle(m, torch.int32) as X:
            out = X.shuffle(local, bsg.ShuffleConfig(seed=77))
        del local
        pieces = {}
        for c0 in (0, S - 4096, S, m - 4096):  # head, both sides of the rank boundary, tail
            if rank * S <= c0 < (rank + 1) * S:
                pieces[c0] = out[c0 - rank * S:c0 - rank * S + 4096].to(torch.int64).cpu().numpy() & 0xFFFFFFFF
        q.put((rank, pieces))
        del out
        torch.cuda.empty_cache()
    except BaseException as e:  # report instead of leaving the parent waiting on the queue
        q.put((rank, {"error": repr(e)}))
        raise
    finally:
        dist.destroy_process_group()


def test_exchange_partition_full_32_bit_domain(orc):
    """bsg_xpart_* at m = 2^32 u32 (each rank 2^31 elements): global indices, bucket positions and the front/back
    fills at the top of the 32-bit range; slices of the output against the oracle's counter-range images."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_xpart_max_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        got.update(q.get(timeout=900)[1])
        assert "error" not in got, got.get("error")
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    m = 1 << 32
    for c0, piece in sorted(got.items()):
        exp = orc.shuffle_indices_range(m, 77, 1, 24, c0, c0 + 4096)
        assert np.array_equal(piece.astype(np.uint64), exp), c0
