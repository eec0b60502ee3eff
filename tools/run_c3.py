"""One C3 shuffle (2^29+1 u64) on the chosen path (for ncu launch lists): python tools/run_c3.py [path] [variant]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_06161_b200 as bsg
path = int(sys.argv[1]) if len(sys.argv) > 1 else 0
variant = int(sys.argv[2]) if len(sys.argv) > 2 else 1
m = (1 << 29) + 1
v = torch.arange(m, dtype=torch.int64, device="cuda")
o = torch.empty_like(v)
bsg.set_path(path)
for _ in range(2):
    bsg.shuffle_values_into(v, bsg.ShuffleConfig(seed=0x5EED, variant=bsg.BijectionVariant(variant)), o)
torch.cuda.synchronize()
