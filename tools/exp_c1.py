"""A/B of two libbsg builds on C1 (2^20 u64, L2 flushed before every timed shuffle), alternating in one process.
usage: python tools/exp_c1.py libA.so libB.so [reps]"""
import ctypes
import os
import shutil
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2106_06161_b200 import _lib
import paper_2106_06161_b200 as bsg

paths = sys.argv[1:3]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
libs = []
for k, pth in enumerate(paths):
    dst = f"/tmp/libbsg_ab{k}.so"
    shutil.copy(pth, dst)
    L = ctypes.CDLL(dst)
    for name, (res, args) in _lib.SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype, fn.argtypes = res, args
    libs.append(L)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for m in (1 << 20, (1 << 20) + 1, 1 << 22, (1 << 22) + 1, 1 << 24):
    x = torch.arange(m, dtype=torch.int64, device="cuda")
    outs = [torch.empty_like(x) for _ in libs]
    cfg = bsg.ShuffleConfig(seed=0x5EED)._c()
    s = torch.cuda.current_stream()
    times = [[] for _ in libs]
    for r in range(reps):
        for k, L in enumerate(libs):
            flush.fill_(r & 255)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            assert L.bsg_shuffle_values(x.data_ptr(), outs[k].data_ptr(), m, 8, ctypes.byref(cfg), s.cuda_stream) == 0
            b.record()
            torch.cuda.synchronize()
            times[k].append(a.elapsed_time(b) * 1000)
    assert torch.equal(outs[0], outs[1])
    med = [sorted(t)[len(t) // 2] for t in times]
    print(f"m={m}: " + "  ".join(f"{os.path.basename(os.path.dirname(p)) or p}: {v:.1f} us" for p, v in zip(paths, med)))
