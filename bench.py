#!/usr/bin/env python
"""Benchmark of the bijective shuffle hot path (BASELINE.json north star).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2|c3|c1|c4]
    torchrun --nproc-per-node N bench.py --gpus N ...     (one rank per GPU, NCCL)

A step = one full shuffle of the configured workload.  `value` is the
whole-job effective bandwidth 2*n*elem_bytes / time with inputs resident in
HBM (CUDA events on the launching stream, max over ranks); `e2e` is the same
metric through the public API with pinned HOST buffers (H2D + shuffle + D2H
every step).  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "effective shuffle GB/s (2·n·bytes/time) vs HBM peak, n=2^29 u64, 1/2/4/8 B200"
SEED = 0x5EED

CONFIGS = {
    # name: (m per GPU, elem bytes, variant, batch, description)
    "c2": (1 << 29, 8, 1, 0, "C2: n=2^29 uint64, power-of-two domain, VariablePhilox-24"),
    "c3": ((1 << 29) + 1, 8, 1, 0, "C3: n=2^29+1 uint64, worst-case padding (2^30 counters), VariablePhilox-24"),
    "c3lcg": ((1 << 29) + 1, 8, 0, 0, "C3: n=2^29+1 uint64, worst-case padding (2^30 counters), LCG"),
    "c2lcg": (1 << 29, 8, 0, 0, "C2: n=2^29 uint64, power-of-two domain, LCG"),
    "c1": (1 << 20, 8, 1, 0, "C1: n=2^20 uint64, VariablePhilox-24"),
    "c4": (1024, 4, 1, 8192, "C4: 8192 shuffles of n=1024 uint32 per GPU (65536 over 8), VariablePhilox-24"),
    "c5": (1 << 30, 16, 1, 0, "C5: 16-byte {u64 key, u64 value} records, 2^30 per GPU (n=2^33 over 8 GPUs), "
                              "VariablePhilox-24"),
}
DTYPES = {4: "u32", 8: "u64", 16: "u64x2 (key+value record)"}


def make_values(torch, n, eb, device=None, pin=False):
    """Synthetic payload: iota for 4/8-byte elements; {key=2i, value=2i+1} records for 16-byte ones."""
    if eb == 16:
        t = torch.arange(2 * n, dtype=torch.int64, device=device).view(torch.complex128)
    else:
        t = torch.arange(n, dtype={4: torch.int32, 8: torch.int64}[eb], device=device)
    return t.pin_memory() if pin else t


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--no-comparators", action="store_true", help="skip gather-bound / CUB sort-shuffle timing")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=0, help="e2e steps (default: --steps)")
    ap.add_argument("--cpu-leg", action="store_true", help=argparse.SUPPRESS)  # internal: the CPU baseline leg
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons = [], 0
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 -- clocks are evidence, not the measurement
            self.nv = None
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "samples": len(s),
                "reasons": [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1]}


# --------------------------------------------------------------- reference --
def reference_arm(args, rank, world):
    """The reference's own CPU implementation (oracle/_ref = bijshuf::shuffle_values_into compiled from the
    reference headers) on all host threads; rank 0 only."""
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ctypes

    import oracle as O
    m, eb, variant, batch, desc = CONFIGS[args.config]
    if O.REF is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference)"}))
        return
    if batch:
        m_sample, note = m, f"{batch} independent shuffles of {m} timed as one step"
    else:
        m_sample, note = m, "full per-GPU workload"
    calls = args.warmup + args.steps
    per = (ctypes.c_double * calls)()
    fnv = ctypes.c_uint64()
    if batch:
        # BijectiveShuffleSampler convention (seed + b, stats.hpp:314-324): one shuffle_values_into call per u32 row,
        # rows spread over all host threads.
        note = f"{batch} shuffle_values_into calls on iota({m}) u32 rows (seed + b) over all host threads"
        rc = O.REF.ref_time_batched_u32_calls(batch, m, SEED, variant, 24, 0, calls, per)
        assert rc == 0, rc
        times = list(per)[args.warmup:]
        bytes_step = 2 * batch * m * eb
    elif eb == 16:
        m_sample = min(m, 1 << 28)
        note = f"{m_sample} 16-byte records per step (of the {m} per GPU)"
        rc = O.REF.ref_time_shuffle_pairs_calls(m_sample, SEED, variant, 24, 0, calls, per)
        assert rc == 0, rc
        times = list(per)[args.warmup:]
        bytes_step = 2 * m_sample * 16
    else:
        rc = O.REF.ref_time_shuffle_u64_calls(m_sample, SEED, variant, 24, 0, calls, per, ctypes.byref(fnv))
        assert rc == 0, rc
        times = list(per)[args.warmup:]
        bytes_step = 2 * m_sample * 8
    mean = sum(times) / len(times)
    val = bytes_step / mean / 1e9
    cores = int(O.REF.ref_hardware_threads())
    line = {
        "impl": "reference", "metric": METRIC, "value": round(val, 3), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(mean * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": DTYPES[eb],
        "data": "synthetic (iota values)",
        "config": {"workload": desc + (f" (reference sample: {note})"), "n": m_sample, "elem_bytes": eb,
                   "seed": SEED, "rounds": 24, "variant": "VariablePhilox" if variant else "Lcg"},
        "cpu_baseline": {"value": round(val, 3), "unit": "GB/s", "cores": cores, "kind": "reference",
                         "sample": f"n={m_sample} {DTYPES[eb]} per step ({note}); {os.path.basename(O.REF.path)}, "
                                   f"avx512={bool(O.REF.ref_avx512_active())}, workers=0 (all host threads), "
                                   f"host CPU: {cpu_model()}"},
        "e2e": {"value": round(val, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline_leg(args, cfgname):
    """Reference CPU shuffle on this host, bounded sample (rank 0, N=1; run in its own process by main())."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ctypes

    import oracle as O
    if O.REF is None:
        return None
    m, eb, variant, batch, desc = CONFIGS[cfgname]
    cores = int(O.REF.ref_hardware_threads())
    lib = f"{os.path.basename(O.REF.path)}, avx512={bool(O.REF.ref_avx512_active())}, host CPU: {cpu_model()}"
    trials = 3 if m >= (1 << 26) else 5
    per = (ctypes.c_double * (trials + 1))()
    if batch:
        assert O.REF.ref_time_batched_u32_calls(batch, m, SEED, variant, 24, 0, trials + 1, per) == 0
        mean = sum(list(per)[1:]) / trials
        return {"value": round(2 * batch * m * eb / mean / 1e9, 3), "unit": "GB/s", "cores": cores,
                "kind": "reference",
                "sample": f"the full per-GPU workload: {batch} shuffle_values_into calls on iota({m}) u32 rows, seed+b "
                          f"(BijectiveShuffleSampler, stats.hpp:314-324), rows spread over {cores} threads; "
                          f"1 warm-up + mean of {trials}; {lib}"}
    if eb == 16:
        ms = min(m, 1 << 28)
        assert O.REF.ref_time_shuffle_pairs_calls(ms, SEED, variant, 24, 0, trials + 1, per) == 0
        mean = sum(list(per)[1:]) / trials
        return {"value": round(2 * ms * 16 / mean / 1e9, 3), "unit": "GB/s", "cores": cores, "kind": "reference",
                "sample": f"n={ms} 16-byte records (bench.hpp:112-114 Pair), 1 warm-up + mean of {trials}, {lib}"}
    mean, _ = O.ref_time_shuffle_u64(m, SEED, variant, 24, trials)
    return {"value": round(2 * m * 8 / mean / 1e9, 3), "unit": "GB/s", "cores": cores, "kind": "reference",
            "sample": f"n={m} u64 (the full per-GPU workload), 1 warm-up + mean of {trials} "
                      f"(bench.hpp:41-59), {lib}"}


# -------------------------------------------------------------------- ours --
def output_checksum(torch, t, first_word=0):
    """(sum, wsum) mod 2^64 of a CUDA tensor viewed as u64 words w[i] (u32 zero-extended, 16-byte records as two
    words), wsum = sum w[i] * (2 * (first_word + i) + 1) -- the checksum of tests/golden/make_bench_checksums.py.
    int64 products and sums wrap modulo 2^64 on the GPU, which is the arithmetic wanted."""
    if t.dtype == torch.int32:
        w = t.reshape(-1).to(torch.int64) & 0xFFFFFFFF
    else:
        w = t.reshape(-1).view(torch.int64)
    s = torch.zeros((), dtype=torch.int64, device=t.device)
    ws = torch.zeros((), dtype=torch.int64, device=t.device)
    chunk = 1 << 26
    for lo in range(0, w.numel(), chunk):
        x = w[lo:lo + chunk]
        k = torch.arange(first_word + lo, first_word + lo + x.numel(), dtype=torch.int64, device=t.device)
        s += x.sum()
        ws += (x * (2 * k + 1)).sum()
    return s, ws


def hex64(v) -> str:
    return f"{int(v) & 0xFFFFFFFFFFFFFFFF:016x}"


def ours_arm(args, rank, world, local, cpu=None):
    import torch
    import paper_2106_06161_b200 as bsg
    from paper_2106_06161_b200 import _lib

    # BSG_BENCH_DEVICE / BSG_BENCH_BACKEND: debugging knobs to exercise the multi-rank code path with several
    # ranks on one GPU (gloo); the driver's runs use one GPU per rank and NCCL.
    local = int(os.environ.get("BSG_BENCH_DEVICE", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("BSG_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    m_gpu, eb, variant, batch, desc = CONFIGS[args.config]
    cfg = bsg.ShuffleConfig(seed=SEED, variant=bsg.BijectionVariant(variant))
    stream = torch.cuda.current_stream(dev)
    tdt = {4: torch.int32, 8: torch.int64, 16: torch.complex128}[eb]

    xchg = False  # the two-rank exchange partition (set below for power-of-two domains at N = 2)
    if batch:
        m_total = m_gpu
        vals = torch.arange(m_gpu, dtype=tdt, device=dev).repeat(batch, 1)
        out = torch.empty_like(vals)
        step_bytes_rank = 2 * batch * m_gpu * eb

        def step():
            bsg.shuffle_values_batched(vals, bsg.ShuffleConfig(seed=SEED + rank * batch, variant=cfg.variant),
                                       out=out)
        dominant = "bsg::k_batched"
    else:
        m_total = m_gpu * world  # weak scaling: one global shuffle of N * n elements
        # 16-byte records (C5) at N > 1: the input is SHARDED (rank r holds records [r*n, (r+1)*n)) and payload
        # reads go to peer HBM through CUDA-IPC mappings (NVLink); smaller payloads are replicated.
        sharded = eb == 16 and world > 1
        pow2 = (m_total & (m_total - 1)) == 0
        # Two ranks, power-of-two u32/u64 domain: the exchange partition (bsg_xpart_*) --
        # rank r holds input half r, routes every element into its owner's buckets by peer stores and places its
        # own output half.  BSG_BENCH_XPART=0 selects the counter-range single pass instead.
        xchg = (world == 2 and pow2 and eb in (4, 8) and m_total <= (1 << 32)
                and os.environ.get("BSG_BENCH_XPART", "1") == "1")
        if xchg:
            from paper_2106_06161_b200 import distributed as D
            S = m_total // 2
            vals = torch.arange(rank * S, (rank + 1) * S, dtype=tdt, device=dev)  # input half r (iota slice)
            xpart = D.ExchangeShuffle(m_total, tdt, device=dev)
        elif sharded:
            from paper_2106_06161_b200 import distributed as D
            vals = torch.arange(2 * rank * m_gpu, 2 * (rank + 1) * m_gpu, dtype=torch.int64,
                                device=dev).view(torch.complex128)
            ipc = D.ipc_shards(vals)
        else:
            vals = make_values(torch, m_total, eb, device=dev)  # replicated input
        step_bytes_rank = 2 * m_gpu * eb
        if xchg:
            out = torch.empty(S, dtype=tdt, device=dev)

            def step():
                xpart.shuffle(vals, cfg, out)
        elif world == 1:
            out = torch.empty(m_total, dtype=tdt, device=dev)

            def step():
                bsg.shuffle_values_into(vals, cfg, out)
        else:
            import ctypes

            import torch.distributed as dist
            b, e = ctypes.c_uint64(), ctypes.c_uint64()
            _lib.check(_lib.lib.bsg_dist_counter_range(m_total, rank, world, ctypes.byref(b), ctypes.byref(e)))
            out = torch.empty(e.value - b.value, dtype=tdt, device=dev)
            cnt_dev = torch.zeros(1, dtype=torch.int64, device=dev)
            counts = torch.zeros(world, dtype=torch.int64, device=dev)
            ccfg = cfg._c()

            src = (None, ctypes.byref(ipc.table)) if sharded else (vals.data_ptr(), None)

            def step():
                _lib.check(_lib.lib.bsg_shuffle_range(m_total, ctypes.byref(ccfg), b.value, e.value, src[0], src[1],
                                                      out.data_ptr(), eb, cnt_dev.data_ptr(),
                                                      stream.cuda_stream), "shuffle_range")
                dist.all_gather_into_tensor(counts, cnt_dev)  # the 8-byte count exchange (NCCL)
        partitioned = world == 1 and m_total * eb >= (256 << 20) and eb <= 8  # whole domain, >= 256 MiB
        if xchg:
            dominant = "bsg::k_part1x+k_part2t+k_place"
        elif partitioned:
            dominant = "bsg::k_part1+k_part2t+k_place" if pow2 else "bsg::k_part1+k_part2t+k_place_rank"
        elif not pow2:
            dominant = "bsg::k_compact_smem"
        else:
            dominant = "bsg::k_pow2"  # counter-range shards and 16-byte records take the single fused pass

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        step()
    barrier()
    # Working sets that fit in L2 (C1) are flushed between timed steps by writing a 512 MiB buffer; each step
    # is then timed on its own (events around the step only) and the step times are summed.
    footprint = 2 * (batch * m_gpu if batch else m_total) * eb
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if footprint < (256 << 20) else None
    launches0 = bsg.kernel_launches()
    with ClockSampler(local) as clk:
        if flush is None:
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
            evs[0].record(stream)
            for i in range(args.steps):
                step()
                evs[i + 1].record(stream)
            barrier()
            per_step = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
        else:
            pairs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                     for _ in range(args.steps)]
            for a, b in pairs:
                flush.zero_()
                a.record(stream)
                step()
                b.record(stream)
            barrier()
            per_step = [a.elapsed_time(b) for a, b in pairs]
    launches = bsg.kernel_launches() - launches0
    total_ms = sum(per_step)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_step = total_ms / args.steps
    value = step_bytes_rank * world / (ms_step * 1e-3) / 1e9

    # Same steps replayed from a CUDA graph (one GPU): separates the device time from the per-call host cost,
    # which dominates the small configurations (C1, C4) when each step is a Python call.
    graph = None
    if world == 1:
        try:
            gs = torch.cuda.Stream(dev)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(gs):
                step()  # uncaptured call on the capture stream sizes every workspace
                torch.cuda.synchronize(dev)
                with torch.cuda.graph(g, stream=gs):
                    for _ in range(args.steps):
                        step()
            g.replay()
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(gs)
            with torch.cuda.stream(gs):
                g.replay()
            e1.record(gs)
            torch.cuda.synchronize(dev)
            gms = e0.elapsed_time(e1) / args.steps
            graph = {"ms_per_step": round(gms, 4), "value": round(step_bytes_rank / (gms * 1e-3) / 1e9, 3),
                     "what": f"the same {args.steps} steps captured into one CUDA graph and replayed"
                             + ("" if flush is None else " back to back (L2-warm: no flush between steps)")}
            del g
        except Exception as e:  # noqa: BLE001 -- evidence only
            graph = {"error": str(e)[:200]}

    # Parity of the timed output itself: its checksum against the reference's (tests/golden/bench_checksums.json,
    # generated from the unmodified reference by tests/golden/make_bench_checksums.py).  At N > 1 each rank
    # checksums its piece at its global word offset and the pieces are summed over ranks (mod 2^64).
    torch.cuda.synchronize(dev)
    if batch:
        cs, cws = output_checksum(torch, out)
        key = f"{args.config}@rank{rank}"
        piece_words = 0
    else:
        if world == 1:
            off_elems, n_elems = 0, m_total
        elif xchg:
            off_elems, n_elems = rank * S, S
        else:
            allc = [int(x) for x in counts.tolist()]
            off_elems, n_elems = sum(allc[:rank]), allc[rank]
        k = 2 if eb == 16 else 1
        cs, cws = output_checksum(torch, out[:n_elems], first_word=off_elems * k)
        if world > 1:
            import torch.distributed as dist
            both = torch.stack([cs, cws])
            dist.all_reduce(both)  # int64 sums wrap modulo 2^64
            cs, cws = both[0], both[1]
        key = f"{args.config}@{world}"
    gold = ((load_json(os.path.join(ROOT, "tests", "golden", "bench_checksums.json")) or {}).get("configs", {})
            .get(key))
    output_check = {"sum": hex64(cs), "wsum": hex64(cws), "golden": key if gold else None,
                    "what": "checksum of the timed output vs the unmodified reference's output of the same workload"}
    if gold:
        output_check["ok"] = gold["sum"] == output_check["sum"] and gold["wsum"] == output_check["wsum"]
        assert output_check["ok"], f"timed output differs from the reference: {output_check} vs {gold}"

    # ---- e2e: public API with pinned HOST buffers, H2D + shuffle + D2H every step.
    # Headline: the streaming C-ABI (bsg_pipeline_*), where step i+1's H2D overlaps step i's D2H;
    # also reported: the synchronous bsg_shuffle_values(host, host) call, one step at a time.
    e2e = None
    # as many e2e steps as timed device steps: a stream of K shuffles pays the pipeline's fill (the first H2D
    # alone) and drain (the last D2H alone) once, as a job of K shuffles does
    e2e_steps = args.e2e_steps or args.steps
    if batch:
        # the public API with pinned HOST rows: bsg.shuffle_values_batched(host in, out=host out) stages the rows
        # through device memory (H2D + kernel + D2H) and returns with the result on the host
        host_in = vals.cpu().pin_memory()
        host_out = torch.empty_like(host_in).pin_memory()
        bcfg = bsg.ShuffleConfig(seed=SEED + rank * batch, variant=cfg.variant)
        nb = batch * m_gpu * eb
        # headline: the streaming C-ABI (bsg_pipeline_submit_batched): step i+1's H2D overlaps step i's D2H;
        # each step is a full batch of shuffles whose result lands in its own pinned host buffer.  A batch moves
        # only 2 x 32 MiB, so the stream runs at least 40 steps (~40 ms) for the pipeline's fill and drain (one
        # H2D and one D2H alone) to be paid once per job rather than dominate it.
        e2e_steps = max(e2e_steps, 40)
        outs = [torch.empty_like(host_in).pin_memory() for _ in range(2)]
        with bsg.Pipeline(batch * m_gpu, eb, depth=2) as pl:
            pl.wait(pl.submit_batched(host_in, outs[0], bcfg))
            barrier()
            t0 = time.perf_counter()
            tickets = [pl.submit_batched(host_in, outs[i % 2], bcfg) for i in range(e2e_steps)]
            pl.wait(tickets[-1])
            el = time.perf_counter() - t0
        ref_rows = out.cpu()
        assert torch.equal(outs[0], ref_rows) and torch.equal(outs[(e2e_steps - 1) % 2], ref_rows), \
            "e2e output mismatch"
        # also reported: the synchronous public call, one batch at a time
        bsg.shuffle_values_batched(host_in, bcfg, out=host_out)
        ts = time.perf_counter()
        for _ in range(e2e_steps):
            bsg.shuffle_values_batched(host_in, bcfg, out=host_out)
        sync_s = (time.perf_counter() - ts) / e2e_steps
        assert torch.equal(host_out, ref_rows), "e2e output mismatch"
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([el, sync_s], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el, sync_s = float(t[0].item()), float(t[1].item())
        e2e = {"value": round(step_bytes_rank * world / (el / e2e_steps) / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": nb, "d2h_bytes_per_step": nb, "steps": e2e_steps,
               "ms_per_step": round(el / e2e_steps * 1e3, 3),
               "path": "bsg_pipeline_submit_batched/wait (C ABI): per step H2D of the pinned host rows, the batched "
                       "kernel, D2H to pinned host rows; 3 streams, 2 device slots, so step i+1's H2D overlaps "
                       "step i's D2H",
               "sync": {"value": round(step_bytes_rank * world / sync_s / 1e9, 3),
                        "ms_per_step": round(sync_s * 1e3, 3),
                        "path": "bsg_shuffle_values_batched(pinned host rows in, pinned host rows out), "
                                "synchronous per call"}}
        del host_in, host_out, outs
    else:
        if world == 1:
            # two host (in, out) pairs so step i+1 never touches step i's buffers; one pair for 16-byte records
            # (2 x 16 GiB pinned), where consecutive steps write the same output bytes
            pairs = [(make_values(torch, m_total, eb, pin=True), torch.empty(m_total, dtype=tdt).pin_memory())
                     for _ in range(1 if eb == 16 else 2)]
            h2d, d2h = m_total * eb, m_total * eb
            if h2d < (256 << 20):
                e2e_steps = max(e2e_steps, 40)  # small steps (C1): pay the pipeline's fill and drain once per job
            with bsg.Pipeline(m_total, eb, depth=2) as pipe:
                P = len(pairs)
                tk = [pipe.submit(pairs[i % P][0], pairs[i % P][1], cfg) for i in range(2)]  # warm-up
                for x in tk:
                    pipe.wait(x)
                t0 = time.perf_counter()
                tk = [pipe.submit(pairs[i % P][0], pairs[i % P][1], cfg) for i in range(e2e_steps)]
                for x in tk:
                    pipe.wait(x)
                el = time.perf_counter() - t0
            # result check of the last step against the device path
            ref = bsg.shuffle_values(vals, cfg).cpu()
            assert torch.equal(pairs[(e2e_steps - 1) % P][1].view(torch.int64), ref.view(torch.int64)), \
                "e2e output mismatch"
            del ref
            host_in, host_out = pairs[0]
            bsg.shuffle_values_into(host_in, cfg, host_out)
            t1 = time.perf_counter()
            nsync = max(2, min(e2e_steps, 6) // 2)
            for _ in range(nsync):
                bsg.shuffle_values_into(host_in, cfg, host_out)
            sync_ms = (time.perf_counter() - t1) / nsync * 1e3
            path = (f"bsg_pipeline_submit/wait (C ABI): per step H2D of n*{eb} B from pinned host memory, the "
                    f"shuffle kernels, D2H of n*{eb} B to pinned host memory; 3 streams, 2 device slots, so step "
                    "i+1's H2D overlaps step i's D2H")
            sync = {"value": round(step_bytes_rank / (sync_ms * 1e-3) / 1e9, 3), "ms_per_step": round(sync_ms, 3),
                    "path": "bsg_shuffle_values(host pinned in, host pinned out), synchronous per call (partitioned path: "
                            "its H2D chunked under P1, its D2H under P3)"}
            del pairs
        elif xchg:
            # each rank's host holds its input half: H2D, the exchange partition (route into the owners' buckets,
            # barrier, place its own), D2H of its output half
            host_in = vals.cpu().pin_memory()
            host_out = torch.empty(S, dtype=tdt).pin_memory()

            def e2e_step():
                vals.copy_(host_in, non_blocking=True)
                xpart.shuffle(vals, cfg, out)
                host_out.copy_(out, non_blocking=True)
                torch.cuda.current_stream(dev).synchronize()
            h2d, d2h = S * eb, S * eb
            e2e_step()
            barrier()
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                e2e_step()
            barrier()
            el = time.perf_counter() - t0
            path = ("per rank: H2D of its input half, exchange partition (P1 stores into the owner rank's buckets "
                    "through CUDA-IPC peer mappings, P2/P3 of its own buckets), D2H of its output half "
                    "(distributed.ExchangeShuffle)")
            sync = None
            del host_in, host_out
        elif sharded:
            # each rank's host holds its input shard: H2D into the IPC-exported device shard, barrier, the
            # counter-range shuffle reading peers over NVLink, D2H of this rank's output piece
            host_in = vals.cpu().pin_memory()
            host_out = torch.empty(out.numel(), dtype=tdt).pin_memory()

            def e2e_step():
                vals.copy_(host_in, non_blocking=True)
                torch.cuda.current_stream(dev).synchronize()
                dist.barrier()  # every shard is in place before anyone reads a peer
                step()
                host_out.copy_(out, non_blocking=True)
                torch.cuda.current_stream(dev).synchronize()
                dist.barrier()  # nobody overwrites its shard while a peer still reads it
            h2d, d2h = m_gpu * eb, out.numel() * eb
            e2e_step()
            barrier()
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                e2e_step()
            barrier()
            el = time.perf_counter() - t0
            path = ("per rank: H2D of its input shard, counter-range shuffle with payload reads from peer shards "
                    "over CUDA IPC / NVLink, 8-byte count all-gather, D2H of its output piece")
            sync = None
            del host_in, host_out
        else:
            # Distributed data: each rank's host holds one input shard; the global power-of-two shuffle is
            # routed by destination (bsg_route_by_dest), exchanged with one NCCL all-to-all and placed
            # (bsg_scatter_permutation); each rank reads back its output shard.
            from paper_2106_06161_b200 import distributed as D
            S = m_total // world
            host_in = make_values(torch, m_total, eb)[rank * S:(rank + 1) * S].clone().pin_memory()
            host_out = torch.empty(S, dtype=tdt).pin_memory()
            dev_in = torch.empty(S, dtype=tdt, device=dev)

            def e2e_step():
                dev_in.copy_(host_in, non_blocking=True)
                res = D.shuffle_values_sharded(dev_in, m_total, cfg)
                host_out.copy_(res, non_blocking=True)
                torch.cuda.current_stream(dev).synchronize()
            h2d, d2h = S * eb, S * eb
            e2e_step()
            barrier()
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                e2e_step()
            barrier()
            el = time.perf_counter() - t0
            path = ("per rank: H2D of its input shard, route by destination, NCCL all-to-all, place, "
                    "D2H of its output shard (distributed.shuffle_values_sharded)")
            sync = None
            del host_in, host_out, dev_in
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([el], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        e2e = {"value": round(step_bytes_rank * world / (el / e2e_steps) / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": e2e_steps,
               "ms_per_step": round(el / e2e_steps * 1e3, 3), "path": path}
        if sync:
            e2e["sync"] = sync

    def finish():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            if sharded_ipc is not None:
                sharded_ipc.close()
            if xchg:
                xpart.close()
            dist.destroy_process_group()

    sharded_ipc = ipc if (not batch and sharded) else None
    if rank != 0:
        finish()
        return

    peaks = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json")) or {}
    peak = peaks.get("hbm_gbs")
    peak_src = "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    if not peak:
        peak, peak_src = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"
    kernel_ms = sum(per_step) / len(per_step)
    alg_bytes = step_bytes_rank  # per launch on this rank (one kernel per step)
    achieved = alg_bytes / (kernel_ms * 1e-3) / 1e9
    prof = load_json(os.path.join(ROOT, "profiles", "traffic.json")) or {}
    single = dominant in ("bsg::k_pow2", "bsg::k_compact_smem") and args.config in ("c2", "c3")
    tkey = args.config + ("_single" if single else "")  # BSG_PATH=1 runs of the partitioned configurations
    traffic = prof.get(tkey, {}).get("dram_bytes_per_launch")

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": DTYPES[eb], "data": "synthetic (iota values, device-generated)",
        "config": {"workload": desc + ("" if world == 1 or batch else
                                       f"; global shuffle of {world}x n elements, "
                                       + ("exchange partition: input halves, P1 stores into the owner rank's "
                                          "buckets through CUDA-IPC peer mappings, P2/P3 per rank" if xchg else
                                          "counter-range partition, "
                                          + ("input sharded over the ranks, payload read from peer HBM via CUDA IPC"
                                             if eb == 16 else "replicated input"))),
                   "n_per_gpu": m_gpu, "n_total": m_total if not batch else batch * m_gpu * world,
                   "elem_bytes": eb, "seed": SEED, "rounds": 24,
                   "variant": "VariablePhilox" if variant else "Lcg",
                   "l2": (f"in+out {footprint / 2**20:.0f} MiB per step > 126 MB L2; no flush" if flush is None
                          else f"in+out {footprint / 2**20:.0f} MiB fits in L2: a 512 MiB buffer is written "
                               "between timed steps (each step timed alone)"),
                   "parallelism": ("exchange partition x2" if xchg else f"counter-range partition x{world}")
                   if world > 1 else "single GPU"},
        "roofline": {"bound": "hbm", "kernel": dominant, "achieved": round(achieved, 3), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                     "algorithmic_bytes_per_launch": alg_bytes, "kernel_ms": round(kernel_ms, 4),
                     "peak_source": peak_src},
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
        "output_check": output_check,
        "graph_replay": graph,
        "e2e": e2e,
    }
    if traffic:
        # how close the kernels run to their own physical DRAM traffic at the measured peak
        line["roofline"]["traffic_floor_ms"] = round(traffic / (peak * 1e9) * 1e3, 4)
        line["roofline"]["frac_of_traffic_floor"] = round(traffic / (peak * 1e9) * 1e3 / kernel_ms, 4)
    if dominant.startswith("bsg::k_part1") and variant == 1:
        # Composite floor of the partitioned path: P1 cannot beat the 24-round inverse
        # cipher nor its own traffic; P2 and P3 cannot beat their traffic at the HBM peak.  Cipher issue floor per
        # round per warp (tools/microbench/mb8.cu, mb9.cu): odd widths (C2) run the high product on the FP64 pipe
        # and are bound by the ALU pipe (LOP3 + 2 SHF = 6 cycles); even widths (C3) keep IMAD + IMAD.HI + IMAD on
        # the FMA-heavy pipe (8 cycles).
        sms, hz = 148, (clk.summary().get("sm_mhz") or 1965) * 1e6
        bits = (m_total - 1).bit_length()
        cyc = 6 if bits % 2 else 8
        cipher_ms = m_total * 24 * cyc / 32 / (sms * 4 * hz) * 1e3
        p1_bytes, p23_bytes = m_total * (eb + eb + 4), m_total * ((eb + 4) + (eb + 2) + (eb + 2) + eb)
        p1_ms = max(cipher_ms, p1_bytes / (peak * 1e9) * 1e3)
        comp = p1_ms + p23_bytes / (peak * 1e9) * 1e3
        line["roofline"]["composite_floor"] = {
            "cipher_ms": round(cipher_ms, 3), "p1_traffic_ms": round(p1_bytes / (peak * 1e9) * 1e3, 3),
            "p2_p3_traffic_ms": round(p23_bytes / (peak * 1e9) * 1e3, 3), "floor_ms": round(comp, 3),
            "frac": round(comp / kernel_ms, 4),
            "what": "max(P1 inverse-cipher issue floor, P1 traffic) + P2/P3 traffic at the HBM peak"}
    if not args.no_comparators and world == 1 and not batch:
        line["comparators"] = comparators(bsg, torch, dev, vals, out, m_total, eb, cfg, stream)
        gb = line["comparators"].get("gather_bound", {}).get("value")
        if gb:
            line["comparators"]["value_over_gather_bound"] = round(value / gb, 3)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    finish()


def comparators(bsg, torch, dev, vals, out, m, eb, cfg, stream):
    """The paper's two GPU reference points on the same data: the random-gather upper bound through a
    precomputed permutation and SortShuffle (CUB radix sort of 64-bit keys)."""
    res = {}

    def t(fn, reps=5):
        fn()
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize(dev)
        return a.elapsed_time(b) / reps

    perm = bsg.shuffle_indices(m, cfg, device=dev)
    ms = t(lambda: bsg.gather_into(vals, perm, out))
    res["gather_bound"] = {"value": round(2 * m * eb / (ms * 1e-3) / 1e9, 3), "unit": "GB/s", "ms": round(ms, 3),
                           "what": "out[i] = in[perm[i]] through a precomputed permutation (reads the 8-byte index "
                                   "too: 24 B/elem of traffic for 16 B/elem of work)"}
    del perm
    if eb == 8:
        try:
            ms = t(lambda: bsg.sort_shuffle_u64(vals, SEED, out=out), reps=3)
            res["sort_shuffle"] = {"value": round(2 * m * eb / (ms * 1e-3) / 1e9, 3), "unit": "GB/s",
                                   "ms": round(ms, 3), "what": "CUB DeviceRadixSort::SortPairs of (mix64 key, value)"}
        except Exception as e:  # noqa: BLE001
            res["sort_shuffle"] = {"error": str(e)[:200]}
    torch.cuda.empty_cache()
    return res


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` run without a launcher: re-exec this command under torch.distributed.run with one rank
    per GPU (the same launch the driver uses), so the line is never silently a one-GPU number."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.cpu_leg:
        print(json.dumps(cpu_baseline_leg(args, args.config)), flush=True)
        return
    rank, world, local = dist_env()
    if args.impl == "reference":
        reference_arm(args, rank, world if "WORLD_SIZE" in os.environ else args.gpus)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started {world} ranks")
    # The CPU baseline leg runs first, in its own process, before this process touches the GPU or pins host
    # memory (a leg run after 16 GiB of cached pinned buffers measured the CPU 1.7x slow in round 1).
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        r = subprocess.run([sys.executable, os.path.abspath(__file__), "--cpu-leg", "--config", args.config],
                           capture_output=True, text=True)
        try:
            cpu = json.loads(r.stdout.strip().splitlines()[-1])
        except (ValueError, IndexError):
            cpu = {"error": (r.stderr or r.stdout)[-300:]}
    ours_arm(args, rank, world, local, cpu)


if __name__ == "__main__":
    main()
