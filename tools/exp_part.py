"""Single fused pass vs partitioned three-pass on power-of-two shuffles."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_06161_b200 as bsg

def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps

for variant in (1, 0):
    cfg = bsg.ShuffleConfig(seed=0x5EED, variant=bsg.BijectionVariant(variant))
    for bits, dt in ((29, torch.int64), (28, torch.int64), (26, torch.int64), (24, torch.int64), (22, torch.int64), (29, torch.int32), (30, torch.int64)):
        m = 1 << bits
        vals = torch.arange(m, dtype=dt, device="cuda")
        out = torch.empty_like(vals)
        res = {}
        for path in (1, 2):
            bsg.set_path(path)
            res[path] = t(lambda: bsg.shuffle_values_into(vals, cfg, out))
            if path == 1:
                ref = out.clone()
            else:
                ok = torch.equal(ref, out)
        eb = vals.element_size()
        print(f"variant {variant} 2^{bits} {str(dt):12s} single {res[1]:8.3f} ms ({2*m*eb/res[1]/1e6:7.1f} GB/s)  "
              f"partitioned {res[2]:8.3f} ms ({2*m*eb/res[2]/1e6:7.1f} GB/s)  equal={ok}", flush=True)
        del vals, out, ref
        torch.cuda.empty_cache()
bsg.set_path(0)
