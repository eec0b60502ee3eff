"""C3 diagnosis: where does the look-back kernel lose time vs the pow2 kernel?"""
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

cfg = bsg.ShuffleConfig(seed=0x5EED)
for m in (1 << 29, (1 << 29) + 1, 1 << 28, (1 << 28) + 1):
    vals = torch.arange(m, dtype=torch.int64, device="cuda")
    out = torch.empty_like(vals)
    print(f"m={m:>11d} values   {t(lambda: bsg.shuffle_values_into(vals, cfg, out)):8.3f} ms")
    print(f"m={m:>11d} indices  {t(lambda: bsg.shuffle_indices_into(m, cfg, out)):8.3f} ms")
    if (m & (m - 1)) == 0:
        bsg.set_force_compact(True)
        print(f"m={m:>11d} values forced look-back {t(lambda: bsg.shuffle_values_into(vals, cfg, out)):8.3f} ms")
        print(f"m={m:>11d} indices forced look-back {t(lambda: bsg.shuffle_indices_into(m, cfg, out)):8.3f} ms")
        bsg.set_force_compact(False)
    del vals, out
    torch.cuda.empty_cache()
