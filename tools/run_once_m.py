"""One shuffle of m u64 on the chosen path (for ncu): run_once_m.py m path variant"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_06161_b200 as bsg
m, path, variant = int(sys.argv[1], 0), int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 1
vals = torch.arange(m, dtype=torch.int64, device="cuda")
out = torch.empty_like(vals)
bsg.set_path(path)
cfg = bsg.ShuffleConfig(seed=0x5EED, variant=bsg.BijectionVariant(variant))
for _ in range(2):
    bsg.shuffle_values_into(vals, cfg, out)
torch.cuda.synchronize()
