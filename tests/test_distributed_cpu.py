"""Multi-process host logic of the distributed shuffle on CPU (gloo, world 2
and 3): counter partition, count all-gather, offsets and rebalancing yield
exactly the single-process shuffle.  The per-range compute is injected from
the oracle here (test infrastructure); on GPUs it is bsg_shuffle_range."""
from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import ROOT, ensure_lib


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, m, seed, variant, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch.distributed as dist

    import oracle as O
    import paper_2106_06161_b200 as bsg
    from paper_2106_06161_b200 import distributed as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def oracle_range(m_, cfg, b, e, values, out):
            img = O.shuffle_indices_range(m_, cfg.seed, int(cfg.variant), cfg.num_rounds, b, e)
            vals = values.numpy().view(np.uint64)[img.astype(np.int64)]
            out[:len(vals)] = torch.from_numpy(vals.view(np.int64))
            return len(vals)

        values = torch.arange(m, dtype=torch.int64) * 7 + 1
        cfg = bsg.ShuffleConfig(seed=seed, variant=bsg.BijectionVariant(variant))
        piece, off, counts = D.shuffle_values(values, m, cfg, range_fn=oracle_range)
        shard = D.rebalance(piece, counts, m)
        q.put((rank, off, counts, piece[:counts[rank]].numpy().copy(), shard.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,m,variant", [(2, 5000, 1), (3, (1 << 16) + 7, 1), (2, 4097, 0)])
def test_distributed_equals_single(world, m, variant, orc):
    ensure_lib()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, 99, variant, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    exp = orc.shuffle_values(np.arange(m, dtype=np.uint64) * 7 + 1, 99, variant, 24)
    full = np.empty(m, dtype=np.uint64)
    for rank, off, counts, piece, _ in res:
        assert off == sum(counts[:rank])
        full[off:off + len(piece)] = piece.view(np.uint64)
    assert np.array_equal(full, exp)
    shards = np.concatenate([r[4].view(np.uint64) for r in res])
    assert np.array_equal(shards, exp)
    sizes = [len(r[4]) for r in res]
    assert max(sizes) - min(sizes) <= 1


def _sharded_worker(rank, world, port, m, seed, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch.distributed as dist

    import oracle as O
    import paper_2106_06161_b200 as bsg
    from paper_2106_06161_b200 import distributed as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        bits = m.bit_length() - 1

        def route(local, m_, cfg, r, w):  # oracle stand-in for bsg_route_by_dest
            S = local.numel()
            dest = np.array([O.philox_invert(bits, cfg.seed, cfg.num_rounds, r * S + i) for i in range(S)],
                            dtype=np.int64)
            part = dest // (m_ // w)
            order = np.argsort(part, kind="stable")
            counts = [int((part == p).sum()) for p in range(w)]
            return (local[torch.from_numpy(order)], torch.from_numpy((dest % (m_ // w))[order]).to(torch.int32),
                    counts)

        def scatter(vals, dest, n):  # oracle stand-in for bsg_scatter_permutation
            out = torch.empty(n, dtype=vals.dtype)
            out[dest.long()] = vals
            return out

        S = m // world
        local = torch.arange(rank * S, (rank + 1) * S, dtype=torch.int64) * 3
        out = D.shuffle_values_sharded(local, m, bsg.ShuffleConfig(seed=seed), route_fn=route, scatter_fn=scatter)
        q.put((rank, out.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_by_destination_equals_single(world, orc):
    ensure_lib()
    m = 1 << 12
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, world, port, m, 77, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = np.concatenate([r[1] for r in res]).view(np.uint64)
    exp = orc.shuffle_values(np.arange(m, dtype=np.uint64) * 3, 77, 1, 24)
    assert np.array_equal(full, exp)
