"""Small shuffles through every kernel family, for compute-sanitizer (memcheck/racecheck/synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np, torch
import oracle as O
import paper_2106_06161_b200 as bsg
from paper_2106_06161_b200 import distributed as D

NO_BULK = os.environ.get("BSG_SAN_NO_BULK") == "1"  # initcheck: plain stores in the last passes
if NO_BULK:
    bsg.set_bulk_stores(False)
ok = True
def check(name, got, exp):
    global ok
    if not np.array_equal(got, exp):
        ok = False
        print("MISMATCH", name)

for m, v in ((5000, 1), ((1 << 14) + 3, 0), (1 << 12, 1)):
    cfg = bsg.ShuffleConfig(seed=m, variant=bsg.BijectionVariant(v))
    vals = torch.arange(m, dtype=torch.int64, device="cuda")
    check(f"values {m}", bsg.shuffle_values(vals, cfg).cpu().numpy().view(np.uint64), O.shuffle_indices(m, m, v, 24))
    check(f"indices {m}", bsg.shuffle_indices(m, cfg, device="cuda").cpu().numpy().view(np.uint64),
          O.shuffle_indices(m, m, v, 24))
bsg.set_force_compact(True)
check("forced compact", bsg.shuffle_indices(1 << 13, bsg.ShuffleConfig(seed=3), device="cuda").cpu().numpy().view(np.uint64),
      O.shuffle_indices(1 << 13, 3))
bsg.set_force_compact(False)
bsg.set_path(2)
vals = torch.arange(1 << 16, dtype=torch.int64, device="cuda")
check("partitioned", bsg.shuffle_values(vals, bsg.ShuffleConfig(seed=9)).cpu().numpy().view(np.uint64),
      O.shuffle_indices(1 << 16, 9))
for m, v in (((1 << 16) + 5, 1), ((1 << 16) + 4099, 0), (1 << 16, 0)):  # padded / LCG (TMA-fed P1) partitions
    vals = torch.arange(m, dtype=torch.int64, device="cuda")
    check(f"partitioned {m} v{v}", bsg.shuffle_values(vals, bsg.ShuffleConfig(seed=7, variant=bsg.BijectionVariant(v))
                                                      ).cpu().numpy().view(np.uint64), O.shuffle_indices(m, 7, v, 24))
vals = torch.arange((1 << 16) + 77, dtype=torch.int32, device="cuda")  # padded u32: k_place_rank<uint32_t>
check("partitioned u32 padded", bsg.shuffle_values(vals, bsg.ShuffleConfig(seed=8)).cpu().numpy().astype(np.uint64),
      O.shuffle_indices((1 << 16) + 77, 8))
for cap in (8192, 0):  # windows above the staging cap: the list-driven k_place_rank beside k_place_rank_t
    old_cap = bsg.set_rank_stage_cap(cap)
    m = (1 << 16) + 5
    vals = torch.arange(m, dtype=torch.int64, device="cuda")
    check(f"partitioned padded cap {cap}", bsg.shuffle_values(vals, bsg.ShuffleConfig(seed=11)).cpu().numpy().view(np.uint64),
          O.shuffle_indices(m, 11))
    bsg.set_rank_stage_cap(old_cap)
for m in ((1 << 16), (1 << 16) + 9):  # host buffers: chunked H2D under P1, chunked D2H under P3 (StageIO)
    hv = np.arange(m, dtype=np.uint64)
    check(f"partitioned host staged {m}", bsg.shuffle_values(hv, bsg.ShuffleConfig(seed=13)), O.shuffle_indices(m, 13))
rec = torch.arange(2 * (1 << 16), dtype=torch.int64, device="cuda").view(-1, 2)  # 16-byte records: k_part2t<uint4>
got = bsg.shuffle_values(rec.view(torch.complex128), bsg.ShuffleConfig(seed=12)).view(torch.int64).view(-1, 2)
check("partitioned 16-byte", got[:, 0].cpu().numpy().astype(np.uint64) // 2, O.shuffle_indices(1 << 16, 12))
# two-rank exchange partition in one process (both workspaces local): k_part1x, k_xfill, P2 over regions, P3
import ctypes
from paper_2106_06161_b200._lib import check as _check, lib as _L
for m, dt, eb in (((1 << 17), torch.int64, 8), ((1 << 18), torch.int32, 4)):
    nb = ctypes.c_uint64()
    _check(_L.bsg_xpart_workspace_bytes(m, eb, 2, ctypes.byref(nb)), "ws")
    wsx = [torch.empty(nb.value, dtype=torch.uint8, device="cuda") for _ in range(2)]
    ptrs = (ctypes.c_void_p * 2)(wsx[0].data_ptr(), wsx[1].data_ptr())
    xin = torch.arange(m, dtype=dt, device="cuda")
    xout = torch.empty_like(xin)
    st = torch.cuda.current_stream().cuda_stream
    xc = bsg.ShuffleConfig(seed=21)._c()
    for r in range(2):
        _check(_L.bsg_xpart_route(xin[r * (m // 2):].data_ptr(), m, eb, ctypes.byref(xc), r, 2, ptrs, st), "route")
    for r in range(2):
        _check(_L.bsg_xpart_place(m, eb, r, 2, ptrs, xout[r * (m // 2):].data_ptr(), st), "place")
    check(f"xpart {m}", xout.cpu().numpy().astype(np.uint64), O.shuffle_indices(m, 21))
bsg.set_path(0)
rows = torch.arange(1024, dtype=torch.int32, device="cuda").repeat(16, 1)
out = bsg.shuffle_values_batched(rows, bsg.ShuffleConfig(seed=1000)).cpu().numpy()
for b in range(16):
    check(f"batched {b}", out[b].astype(np.uint64), O.shuffle_indices(1024, 1000 + b))
rows = torch.arange(1000, dtype=torch.int32, device="cuda").repeat(8, 1)
out = bsg.shuffle_values_batched(rows, bsg.ShuffleConfig(seed=5)).cpu().numpy()
for b in range(8):
    check(f"batched1000 {b}", out[b].astype(np.uint64), O.shuffle_indices(1000, 5 + b))
m, W = 1 << 16, 4
S = m // W
full = torch.arange(m, dtype=torch.int64, device="cuda")
cfg = bsg.ShuffleConfig(seed=11)
routed = [D._gpu_route(full[r * S:(r + 1) * S].contiguous(), m, cfg, r, W) for r in range(W)]
parts = []
for dst in range(W):
    vs = [routed[s][0][sum(routed[s][2][:dst]):sum(routed[s][2][:dst + 1])] for s in range(W)]
    ds = [routed[s][1][sum(routed[s][2][:dst]):sum(routed[s][2][:dst + 1])] for s in range(W)]
    parts.append(D._gpu_scatter(torch.cat(vs), torch.cat(ds), S))
check("sharded", torch.cat(parts).cpu().numpy().view(np.uint64), O.shuffle_indices(m, 11))
idx = torch.randint(0, 1 << 12, (5000,), device="cuda")
src = torch.arange(1 << 12, dtype=torch.int64, device="cuda")
check("gather", bsg.gather(src, idx).cpu().numpy(), src.cpu().numpy()[idx.cpu().numpy()])
torch.cuda.synchronize()
print("sanitize-run", "OK" if ok else "FAILED")
