"""Per-kernel device times of one shuffle configuration (torch.profiler / CUPTI, warm, back to back), for A/B
comparisons of variant builds:  BSG_LIB=/path/libbsg_x.so python tools/ktime.py c2 [reps]
Also checks the output against a reference build's output when BSG_LIB_REF is given (bit equality)."""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2106_06161_b200 as bsg

CFG = {"c2": (1 << 29, torch.int64, 1), "c2lcg": (1 << 29, torch.int64, 0), "c3": ((1 << 29) + 1, torch.int64, 1),
       "c3lcg": ((1 << 29) + 1, torch.int64, 0), "c5": (1 << 30, torch.complex128, 1), "c1": (1 << 20, torch.int64, 1),
       "c4": (1024, torch.int32, 1)}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    m, dt, variant = CFG[name]
    cfg = bsg.ShuffleConfig(seed=0x5EED, variant=bsg.BijectionVariant(variant))
    if name == "c4":
        vals = torch.arange(m, dtype=dt, device="cuda").repeat(8192, 1)
        fn = lambda: bsg.shuffle_values_batched(vals, cfg, out=out)  # noqa: E731
        out = torch.empty_like(vals)
    else:
        vals = (torch.arange(2 * m, dtype=torch.int64, device="cuda").view(dt) if dt == torch.complex128
                else torch.arange(m, dtype=dt, device="cuda"))
        out = torch.empty_like(vals)
        fn = lambda: bsg.shuffle_values_into(vals, cfg, out)  # noqa: E731
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
    agg = defaultdict(float)
    cnt = defaultdict(int)
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            k = e.name.split("<")[0].replace("void ", "").replace("(anonymous namespace)::", "")
            agg[k] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
            cnt[k] += 1
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    tag = os.path.basename(os.environ.get("BSG_LIB", "libbsg.so"))
    print(f"[{tag}] {name}: {a.elapsed_time(b) / reps:.3f} ms/shuffle (events)")
    for k in sorted(agg, key=lambda k: -agg[k]):
        print(f"    {k:40s} {agg[k] / reps / 1000:8.3f} ms/shuffle  ({cnt[k] // reps} launches)")
    h = torch.zeros((), dtype=torch.int64, device="cuda")
    w = out.reshape(-1).view(torch.int64) if dt != torch.int32 else out.reshape(-1).to(torch.int64)
    for lo in range(0, w.numel(), 1 << 26):
        x = w[lo:lo + (1 << 26)]
        h += (x * (2 * torch.arange(lo, lo + x.numel(), device="cuda") + 1)).sum()
    print(f"    checksum wsum {int(h) & 0xFFFFFFFFFFFFFFFF:016x}")


if __name__ == "__main__":
    main()
