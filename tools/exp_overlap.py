"""Experiment: do consecutive independent C2 shuffles gain from running concurrently (P1 of one call beside
P2/P3 of the previous) when each has its own workspace?  Two copies of libbsg.so (separate device contexts and
workspaces) are driven on two streams, alternating calls; compared with back-to-back calls on one stream.
usage: python tools/exp_overlap.py [steps]"""
import ctypes
import os
import shutil
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2106_06161_b200 as bsg
from paper_2106_06161_b200 import _lib

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
m = 1 << 29
libs = [bsg.lib]
for k in range(1, 2):
    dst = f"/tmp/libbsg_copy{k}.so"
    shutil.copy(_lib.LIB_PATH, dst)
    L = ctypes.CDLL(dst)
    for name, (res, args) in _lib.SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype, fn.argtypes = res, args
    libs.append(L)
cfg = bsg.ShuffleConfig(seed=0x5EED)._c()
x = torch.arange(m, dtype=torch.int64, device="cuda")
outs = [torch.empty_like(x) for _ in range(2)]
streams = [torch.cuda.Stream() for _ in range(2)]


def call(k, s):
    rc = libs[k].bsg_shuffle_values(x.data_ptr(), outs[k].data_ptr(), m, 8, ctypes.byref(cfg), s.cuda_stream)
    assert rc == 0, rc


for k in range(2):
    call(k, streams[k])
torch.cuda.synchronize()
ref = outs[0].clone()
assert torch.equal(outs[1], ref)
# serial: one stream, one library
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s0 = streams[0]
a.record(s0)
for i in range(steps):
    call(0, s0)
b.record(s0)
torch.cuda.synchronize()
serial = a.elapsed_time(b) / steps
# overlapped: call i on stream i%2 through library i%2
ev = [torch.cuda.Event() for _ in range(2)]
start = torch.cuda.Event(enable_timing=True)
start.record(streams[0])
streams[1].wait_event(start)
for i in range(steps):
    call(i % 2, streams[i % 2])
end = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for k in range(2):
    end[k].record(streams[k])
torch.cuda.synchronize()
over = max(start.elapsed_time(e) for e in end) / steps
assert torch.equal(outs[0], ref) and torch.equal(outs[1], ref)
print(f"C2 serial {serial:.3f} ms/shuffle   two streams, two workspaces {over:.3f} ms/shuffle")
