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
