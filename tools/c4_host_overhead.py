import sys, os, time
sys.path.insert(0, os.getcwd())
import torch, paper_2106_06161_b200 as bsg
vals = torch.arange(1024, dtype=torch.int32, device="cuda").repeat(8192, 1)
out = torch.empty_like(vals)
cfg = bsg.ShuffleConfig(seed=1)
for _ in range(10): bsg.shuffle_values_batched(vals, cfg, out=out)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200): bsg.shuffle_values_batched(vals, cfg, out=out)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {(t1-t0)/200*1e6:.1f} us/call, wall {(t2-t0)/200*1e6:.1f} us/call")
# GPU-only via graph
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    bsg.shuffle_values_batched(vals, cfg, out=out)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for _ in range(20): bsg.shuffle_values_batched(vals, cfg, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
print(f"graph: {e0.elapsed_time(e1)/20*1e3:.1f} us/call")
