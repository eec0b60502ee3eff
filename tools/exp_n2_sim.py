"""Compute side of the N = 2 exchange design, simulated on one GPU: a 2^30-element u64
power-of-two shuffle through the partitioned path has P1 route every input into 512 coarse buckets (bits 30:
buckets 0-255 are rank 0's output half, 256-511 rank 1's) and P2/P3 work per bucket, so each rank's share of
the kernels is half of each kernel's time on the full 2^30 domain; the NVLink part (half of P1's 12 B/element
stores going to the peer) is modelled separately.  usage: python tools/exp_n2_sim.py [reps]"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2106_06161_b200 as bsg

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
m = 1 << 30
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
agg = defaultdict(float)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        agg[e.name.split("<")[0].replace("void ", "").replace("(anonymous namespace)::", "")] += e.device_time_total
tot = sum(agg.values()) / reps / 1000
print(f"2^30 u64 partitioned shuffle: {tot:.3f} ms (kernels)")
for k in sorted(agg, key=lambda k: -agg[k]):
    print(f"    {k:40s} {agg[k] / reps / 1000:8.3f} ms  -> per rank at N=2: {agg[k] / reps / 2000:7.3f} ms")
p1 = sum(v for k, v in agg.items() if "k_part1" in k) / reps / 2000
rest = tot / 2 - p1
nv = (1 << 29) * 12 / 2  # bytes of P1 output a rank sends to its peer
for bw in (750e9, 900e9):
    print(f"NVLink at {bw / 1e9:.0f} GB/s: {nv / bw * 1e3:.2f} ms of peer stores beside P1 {p1:.2f} ms -> per-rank "
          f"{max(p1, nv / bw * 1e3) + rest:.2f} ms per 2^29 local elements (single pass measured 11.43 ms)")
