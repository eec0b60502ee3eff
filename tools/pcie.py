"""Host<->device copy ceilings for the e2e numbers: pinned 4 GiB H2D, D2H, and both at once."""
import time, torch
n = 1 << 29
h_in = torch.arange(n, dtype=torch.int64).pin_memory()
h_out = torch.empty(n, dtype=torch.int64).pin_memory()
d_a = torch.empty(n, dtype=torch.int64, device="cuda")
d_b = torch.empty(n, dtype=torch.int64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=4):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
gb = n * 8 / 1e9
h2d = t(lambda: d_a.copy_(h_in, non_blocking=True))
d2h = t(lambda: h_out.copy_(d_b, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
bi = t(both)
print(f"H2D {gb/h2d:6.1f} GB/s ({h2d*1e3:.1f} ms)   D2H {gb/d2h:6.1f} GB/s ({d2h*1e3:.1f} ms)   "
      f"concurrent: {2*gb/bi:6.1f} GB/s total ({bi*1e3:.1f} ms for 4 GiB each way)")
