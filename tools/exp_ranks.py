"""Per-rank time of the counter-range scheme on one GPU: rank r of N with a replicated N x 2^29 u64 input
(the work one GPU does in bench.py --gpus N)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_06161_b200 as bsg
from paper_2106_06161_b200 import _lib

def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps

cfg = bsg.ShuffleConfig(seed=0x5EED)
cc = cfg._c()
stream = torch.cuda.current_stream().cuda_stream
for N in (1, 2, 4, 8):
    m_total = (1 << 29) * N
    vals = torch.arange(m_total, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    for r in sorted({0, N - 1}):
        b, e = ctypes.c_uint64(), ctypes.c_uint64()
        _lib.check(_lib.lib.bsg_dist_counter_range(m_total, r, N, ctypes.byref(b), ctypes.byref(e)))
        out = torch.empty(e.value - b.value, dtype=torch.int64, device="cuda")
        ms = t(lambda: _lib.check(_lib.lib.bsg_shuffle_range(m_total, ctypes.byref(cc), b.value, e.value,
                                                              vals.data_ptr(), None, out.data_ptr(), 8,
                                                              cnt.data_ptr(), stream)))
        print(f"N={N} rank {r}: {ms:.3f} ms  ({2 * (e.value - b.value) * 8 / ms / 1e6:.1f} GB/s per GPU)", flush=True)
        del out
    del vals
    torch.cuda.empty_cache()
