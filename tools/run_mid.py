"""One shuffle of 2^24+1 u64 (acceptance criterion 9 size), for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_06161_b200 as bsg
m = (1 << 24) + int(sys.argv[1] if len(sys.argv) > 1 else 1)
v = torch.arange(m, dtype=torch.int64, device="cuda")
o = torch.empty_like(v)
for _ in range(3):
    bsg.shuffle_values_into(v, bsg.ShuffleConfig(seed=1), o)
torch.cuda.synchronize()
