"""Per-rank kernel times of the two-rank exchange partition (bsg_xpart_*) on ONE GPU: both ranks' workspaces are
local allocations in this process, so route(0), route(1), place(0), place(1) run back to back and each rank's
share is its own kernels (the peer stores of route land in local memory here; over NVLink they add the modelled
3.2 GB per rank).  Checks the concatenated halves against the reference checksum of C2 at N = 2 (c2@2).
usage: python tools/exp_xpart.py [reps]"""
import ctypes
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import paper_2106_06161_b200 as bsg
from paper_2106_06161_b200._lib import check, lib

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
m = 1 << 30
S = m // 2
cfg = bsg.ShuffleConfig(seed=0x5EED)
nb = ctypes.c_uint64()
check(lib.bsg_xpart_workspace_bytes(m, 8, 2, ctypes.byref(nb)), "ws")
ws = [torch.empty(nb.value, dtype=torch.uint8, device="cuda") for _ in range(2)]
ptrs = (ctypes.c_void_p * 2)(ws[0].data_ptr(), ws[1].data_ptr())
x = torch.arange(m, dtype=torch.int64, device="cuda")
out = torch.empty_like(x)
st = torch.cuda.current_stream().cuda_stream


def run():
    for r in range(2):
        check(lib.bsg_xpart_route(x[r * S:].data_ptr(), m, 8, ctypes.byref(cfg._c()), r, 2, ptrs, st), "route")
    for r in range(2):
        check(lib.bsg_xpart_place(m, 8, r, 2, ptrs, out[r * S:].data_ptr(), st), "place")


run()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        run()
    torch.cuda.synchronize()
agg = defaultdict(float)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        agg[e.name.split("<")[0].replace("void ", "").replace("(anonymous namespace)::", "")] += e.device_time_total
per_rank = sum(agg.values()) / reps / 2 / 1000
print(f"exchange partition, C2 at N=2 (2^30 u64, 2^29 per rank): {per_rank:.3f} ms of kernels per rank")
for k in sorted(agg, key=lambda k: -agg[k]):
    print(f"    {k:40s} {agg[k] / reps / 2000:8.3f} ms per rank")
# order-sensitive checksum of the global output (bench.py output_checksum) against the reference's c2@2
w = out.view(torch.int64)
s = torch.zeros((), dtype=torch.int64, device="cuda")
ws_ = torch.zeros((), dtype=torch.int64, device="cuda")
for lo in range(0, m, 1 << 26):
    c = w[lo:lo + (1 << 26)]
    k = torch.arange(lo, lo + c.numel(), dtype=torch.int64, device="cuda")
    s += c.sum()
    ws_ += (c * (2 * k + 1)).sum()
gold = json.load(open(os.path.join(ROOT, "tests", "golden", "bench_checksums.json")))["configs"]["c2@2"]
got = (f"{int(s) & (2**64 - 1):016x}", f"{int(ws_) & (2**64 - 1):016x}")
print("checksum", got, "reference c2@2", (gold["sum"], gold["wsum"]), "OK" if got == (gold["sum"], gold["wsum"]) else "MISMATCH")
nv = S * 12 / 2
for bw in (750e9, 900e9):
    p1 = agg.get("bsg::k_part1x", 0) / reps / 2000
    print(f"NVLink {bw / 1e9:.0f} GB/s: {nv / bw * 1e3:.2f} ms of peer stores beside route {p1:.2f} ms -> per rank "
          f"{per_rank - p1 + max(p1, nv / bw * 1e3):.2f} ms")
