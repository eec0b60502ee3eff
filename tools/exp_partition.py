"""Partitioned path (set_path(2)) vs the single pass: bit equality and time per case.  BSG_LIB selects a variant
build (tools/run_var.sh); the first argument limits the number of cases."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2106_06161_b200 as bsg


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


tag = " ".join(f"{k}={os.environ[k]}" for k in ("BSG_LIB",) if k in os.environ)
cases = [(29, torch.int64, 1), (29, torch.int64, 0), (28, torch.int32, 1), (24, torch.int64, 1), (20, torch.int64, 1),
         (16, torch.int64, 1), (14, torch.int32, 1), (26, torch.complex128, 1)]
if len(sys.argv) > 1:
    cases = cases[: int(sys.argv[1])]
for bits, dt, variant in cases:
    cfg = bsg.ShuffleConfig(seed=0x5EED, variant=bsg.BijectionVariant(variant))
    m = 1 << bits
    if dt == torch.complex128:
        vals = torch.randn(m, dtype=dt, device="cuda")
    else:
        vals = torch.arange(m, dtype=dt, device="cuda")
    out = torch.empty_like(vals)
    bsg.set_path(1)
    bsg.shuffle_values_into(vals, cfg, out)
    ref = out.clone()
    bsg.set_path(2)
    out.zero_()
    ms = t(lambda: bsg.shuffle_values_into(vals, cfg, out))
    ok = torch.equal(ref.view(torch.uint8), out.view(torch.uint8))
    eb = vals.element_size()
    print(f"[{tag}] variant {variant} 2^{bits} {str(dt):16s} partitioned {ms:8.3f} ms ({2*m*eb/ms/1e6:7.1f} GB/s) "
          f"equal={ok}", flush=True)
    del vals, out, ref
    torch.cuda.empty_cache()
bsg.set_path(0)
