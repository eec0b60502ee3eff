"""A/B of the last passes' bulk shared->global stores (bsg_set_bulk_stores) on C2 and C3, alternating in one
process; prints ms per shuffle and checks the outputs are identical.  usage: python tools/exp_bulk.py [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2106_06161_b200 as bsg

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
for name, m in (("c2", 1 << 29), ("c3", (1 << 29) + 1)):
    x = torch.arange(m, dtype=torch.int64, device="cuda")
    out = torch.empty_like(x)
    cfg = bsg.ShuffleConfig(seed=0x5EED)
    res = {}
    ref = None
    for it in range(3):
        for bulk in (True, False):
            bsg.set_bulk_stores(bulk)
            bsg.shuffle_values_into(x, cfg, out)
            torch.cuda.synchronize()
            if ref is None:
                ref = out.clone()
            assert torch.equal(out, ref), (name, bulk)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                bsg.shuffle_values_into(x, cfg, out)
            b.record()
            torch.cuda.synchronize()
            res.setdefault(bulk, []).append(a.elapsed_time(b) / reps)
    bsg.set_bulk_stores(True)
    print(name, "bulk", " ".join(f"{t:.3f}" for t in res[True]), "| plain", " ".join(f"{t:.3f}" for t in res[False]))
    del x, out, ref
    torch.cuda.empty_cache()
