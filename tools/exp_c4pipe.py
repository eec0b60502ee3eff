import sys, time, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2106_06161_b200 as bsg
batch, m = 8192, 1024
vals = torch.arange(m, dtype=torch.int32).repeat(batch, 1).contiguous().pin_memory()
cfg = bsg.ShuffleConfig(seed=0x5EED)
for depth in (2, 3, 4):
    outs = [torch.empty_like(vals).pin_memory() for _ in range(depth)]
    with bsg.Pipeline(batch * m, 4, depth=depth) as pl:
        pl.wait(pl.submit_batched(vals, outs[0], cfg))
        for steps in (10, 40):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ts = [pl.submit_batched(vals, outs[i % depth], cfg) for i in range(steps)]
            pl.wait(ts[-1])
            el = time.perf_counter() - t0
            print(f"depth {depth} steps {steps}: {2 * batch * m * 4 * steps / el / 1e9:.1f} GB/s")
