"""Compute side of an N-rank exchange partition, simulated on one GPU: a (2^29 * N)-element
u64 power-of-two shuffle through the partitioned path routes every input in P1 into the coarse buckets of the
whole domain (bucket b belongs to rank b * N / nb1) and P2/P3 work per bucket, so a rank's share of each kernel
is 1/N of its time on the full domain.  N = 2 is tools/exp_n2_sim.py (measured 8.43 ms, built as bsg_xpart_*);
N = 4 is a 2^31 shuffle (P1 512 coarse buckets = 4 owners x 128, P2 512 fine windows per bucket, the widest
fan-outs both passes support).  The NVLink part, (N-1)/N of P1's 12 B/element stores going to peers, is
modelled.  usage: python tools/exp_nsim.py N [reps]"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2106_06161_b200 as bsg

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
m = (1 << 29) * N
x = torch.arange(m, dtype=torch.int64, device="cuda")
out = torch.empty_like(x)
cfg = bsg.ShuffleConfig(seed=0x5EED)
for _ in range(2):
    bsg.shuffle_values_into(x, cfg, out)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        bsg.shuffle_values_into(x, cfg, out)
    torch.cuda.synchronize()
agg, cnt = defaultdict(float), defaultdict(int)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        k = e.name.split("<")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        agg[k] += e.device_time_total
        cnt[k] += 1
tot = sum(agg.values()) / reps / 1000
print(f"2^{m.bit_length() - 1} u64 partitioned shuffle on one GPU: {tot:.3f} ms (kernels)")
for k in sorted(agg, key=lambda k: -agg[k]):
    print(f"    {k:40s} {agg[k] / reps / 1000:8.3f} ms ({cnt[k] // reps} launches) -> per rank at N={N}: "
          f"{agg[k] / reps / 1000 / N:7.3f} ms")
p1 = sum(v for k, v in agg.items() if "k_part1" in k) / reps / 1000 / N
rest = tot / N - p1
nv = (1 << 29) * 12 * (N - 1) / N  # bytes of P1 output a rank sends to its peers
for bw in (750e9, 900e9):
    print(f"NVLink at {bw / 1e9:.0f} GB/s: {nv / bw * 1e3:.2f} ms of peer stores beside P1 {p1:.2f} ms -> per-rank "
          f"{max(p1, nv / bw * 1e3) + rest:.2f} ms per 2^29 local elements (single pass measured 11.53 ms at N=4)")
h = torch.zeros((), dtype=torch.int64, device="cuda")
for lo in range(0, m, 1 << 27):
    w = out[lo:lo + (1 << 27)]
    h += (w * (torch.arange(lo, lo + w.numel(), device="cuda") | 1)).sum()
perm_ok = bool(torch.sort(out[: 1 << 27] & ((1 << 62) - 1))[0].numel() == 1 << 27)
print(f"output weighted sum {int(h) & ((1 << 64) - 1):016x}")
