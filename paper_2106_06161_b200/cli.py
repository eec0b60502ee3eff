"""Command-line front end mirroring the reference `bijshuf-cli`
(proj/tools/bijshuf_cli.cpp): `shuffle`, `test`, `bench`, same flags, JSON
report and CSV/JSON record schema, same exit codes (0 success / statistical
pass, 1 statistical fail, 2 usage or input error).  Work runs on the GPU.

    python -m paper_2106_06161_b200.cli shuffle --indices 1000 --seed 7
    python -m paper_2106_06161_b200.cli test --kind chi2 --gen philox --samples 100000
    python -m paper_2106_06161_b200.cli bench --sizes 1048577,16777217 --format csv
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from typing import List

BENCH_CSV_HEADER = "algorithm,input_size,trials,runtime_s,throughput_mitems_s"  # bench.hpp:209-210
GPU_ALGOS = ["bijective", "gather", "sort_shuffle"]


def default_bench_sizes() -> List[int]:  # bench.hpp:173-177
    return [(1 << w) + 1 for w in range(8, 27)]


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # CLI11 parse errors exit 2
        self.print_usage(sys.stderr)
        sys.stderr.write(f"{self.prog}: error: {message}\n")
        raise SystemExit(2)


def _common(p):
    p.add_argument("--seed", type=lambda s: int(s, 0), default=0)
    p.add_argument("--rounds", type=int, default=24)
    p.add_argument("--workers", type=int, default=0)
    p.add_argument("--entropy", action="store_true")


def _seed(a) -> int:
    if a.entropy:
        return int.from_bytes(os.urandom(8), "little")
    return a.seed


def _fmt(v: float) -> str:  # bench.hpp:213-217 (%.17g)
    return "%.17g" % v


def run_shuffle(a) -> int:
    import numpy as np

    import paper_2106_06161_b200 as bsg
    cfg = bsg.ShuffleConfig(seed=_seed(a), num_rounds=a.rounds, workers=a.workers)
    if a.indices is not None:
        perm = bsg.shuffle_indices(a.indices, cfg)
        out = sys.stdout
        for s in range(0, len(perm), 1 << 20):
            out.write("\n".join(map(str, perm[s:s + (1 << 20)].tolist())))
            out.write("\n")
        return 0
    if a.input is None:
        sys.stderr.write("shuffle: pass --indices m or an input file\n")
        return 2
    try:
        lines = sys.stdin.read().splitlines() if a.input == "-" else open(a.input).read().splitlines()
    except OSError:
        sys.stderr.write(f"shuffle: cannot read {a.input}\n")
        return 2
    perm = bsg.shuffle_indices(len(lines), cfg)  # GPU permutation, host moves the strings
    sys.stdout.write("".join(lines[int(i)] + "\n" for i in perm))
    return 0


def _fisher_yates_perms(n: int, samples: int, seed: int):
    """FisherYatesSampler (stats.hpp:329-337): SplitMix64::below + backward swaps (the uniform reference)."""
    import numpy as np
    M = (1 << 64) - 1
    state = seed & M

    def nxt():
        nonlocal state
        state = (state + 0x9E3779B97F4A7C15) & M
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)

    out = np.empty((samples, n), dtype=np.int64)
    for s in range(samples):
        p = list(range(n))
        for i in range(n, 1, -1):
            limit = M - (M % i)
            v = nxt()
            while v >= limit:
                v = nxt()
            j = v % i
            p[i - 1], p[j] = p[j], p[i - 1]
        out[s] = p
    return out


def run_test(a) -> int:
    import torch

    import paper_2106_06161_b200 as bsg
    from paper_2106_06161_b200 import stats as S
    n = a.n
    if a.kind == "chi2":
        if a.n_given and a.n != 5:
            sys.stderr.write("test: --kind chi2 is defined over permutations of 5 elements\n")
            return 2
        n = 5
    kind = {"chi2": S.TestKind.ChiSquared, "mmd-hoeffding": S.TestKind.MmdHoeffding,
            "mmd-normal": S.TestKind.MmdNormal}[a.kind]
    variant = bsg.BijectionVariant.Lcg if a.gen == "lcg" else bsg.BijectionVariant.VariablePhilox
    cfg = bsg.ShuffleConfig(seed=_seed(a), variant=variant, num_rounds=a.rounds, workers=a.workers)
    try:
        perms = None
        if a.gen == "fisher-yates":
            perms = torch.from_numpy(_fisher_yates_perms(n, a.samples, cfg.seed)).cuda()
        if kind == S.TestKind.ChiSquared:
            if perms is None:
                r = S.chi_squared_test(a.samples, cfg, a.alpha)
            else:
                if a.samples < 12000:
                    raise bsg.InvalidArgument("chi_squared_test: need >= 12000 samples")
                counts = torch.bincount(S.permutation_rank(perms), minlength=120).double()
                e = a.samples / 120.0
                stat = float(((counts - e) ** 2 / e).sum())
                thr = S.chi2_quantile(1.0 - a.alpha, 119)
                r = S.TestReport(kind, stat, thr, a.alpha, a.samples, stat < thr)
        else:
            r = S.mmd_test(n, a.samples, cfg, a.alpha, kind, a.lam, perms=perms)
    except (ValueError, IndexError) as e:
        sys.stderr.write(f"error: {e}\n")
        return 2
    print(json.dumps({"test_kind": a.kind, "statistic": r.statistic, "threshold": r.threshold, "alpha": r.alpha,
                      "sample_size": r.sample_size, "pass": bool(r.passed)}, indent=2))
    return 0 if r.passed else 1


def bench_records(sizes, algos, trials, seed, rounds=24):
    """run_suite (bench.hpp:186-207) on the GPU: device-resident iota u64, one warm-up, mean of `trials`
    (time_trials, bench.hpp:41-59) with CUDA events."""
    import torch

    import paper_2106_06161_b200 as bsg
    recs = []
    for size in sizes:
        vals = torch.arange(size, dtype=torch.int64, device="cuda")
        out = torch.empty_like(vals)
        cfg = bsg.ShuffleConfig(seed=seed, num_rounds=rounds)
        for algo in algos:
            if algo == "bijective":
                fn = lambda: bsg.shuffle_values_into(vals, cfg, out)  # noqa: E731
            elif algo == "gather":
                g = torch.Generator(device="cuda").manual_seed(seed & 0x7FFFFFFF)
                idx = torch.randint(0, size, (size,), device="cuda", generator=g)
                fn = lambda: bsg.gather_into(vals, idx, out)  # noqa: E731
            elif algo == "sort_shuffle":
                fn = lambda: bsg.sort_shuffle_u64(vals, seed, out=out)  # noqa: E731
            else:
                raise bsg.InvalidArgument(f"run_suite: unknown algorithm {algo} (GPU algorithms: {GPU_ALGOS})")
            fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(trials):
                fn()
            b.record()
            torch.cuda.synchronize()
            rt = a.elapsed_time(b) / 1e3 / trials
            recs.append({"algorithm": algo, "input_size": size, "trials": trials, "runtime_s": rt,
                         "throughput_mitems_s": size / rt / 1e6})
        del vals, out
    return recs


def write_csv(f, recs):  # bench.hpp:219-228
    f.write(BENCH_CSV_HEADER + "\n")
    for r in recs:
        f.write(f"{r['algorithm']},{r['input_size']},{r['trials']},{_fmt(r['runtime_s'])},"
                f"{_fmt(r['throughput_mitems_s'])}\n")


def write_json(f, recs):  # bench.hpp:230-241
    f.write("[\n")
    for i, r in enumerate(recs):
        f.write(f'  {{"algorithm": "{r["algorithm"]}", "input_size": {r["input_size"]}, "trials": {r["trials"]}, '
                f'"runtime_s": {_fmt(r["runtime_s"])}, "throughput_mitems_s": {_fmt(r["throughput_mitems_s"])}}}'
                + ("," if i + 1 < len(recs) else "") + "\n")
    f.write("]\n")


def run_bench(a) -> int:
    sizes = [int(s) for s in a.sizes.split(",")] if a.sizes else default_bench_sizes()
    algos = a.algos.split(",") if a.algos else GPU_ALGOS
    try:
        recs = bench_records(sizes, algos, a.trials, _seed(a), a.rounds)
    except ValueError as e:
        sys.stderr.write(f"error: {e}\n")
        return 2
    f = open(a.output, "w") if a.output else sys.stdout
    (write_json if a.format == "json" else write_csv)(f, recs)
    if a.output:
        f.close()
    return 0


def main(argv=None) -> int:
    ap = _Parser(prog="bijshuf-gpu", description="Deterministic pseudo-random shuffling on B200 "
                                                   "(bijshuf-cli compatible)")
    sub = ap.add_subparsers(dest="cmd", required=True, parser_class=_Parser)
    sh = sub.add_parser("shuffle")
    sh.add_argument("--indices", type=int)
    sh.add_argument("input", nargs="?")
    _common(sh)
    te = sub.add_parser("test")
    te.add_argument("--kind", required=True, choices=["chi2", "mmd-hoeffding", "mmd-normal"])
    te.add_argument("--gen", default="philox", choices=["philox", "lcg", "fisher-yates"])
    te.add_argument("--n", type=int, default=None)
    te.add_argument("--samples", type=int, default=100000)
    te.add_argument("--alpha", type=float, default=0.05)
    te.add_argument("--lambda", dest="lam", type=float, default=5.0)
    _common(te)
    be = sub.add_parser("bench")
    be.add_argument("--sizes", default="")
    be.add_argument("--algos", default="")
    be.add_argument("--trials", type=int, default=5)
    be.add_argument("--format", default="csv", choices=["csv", "json"])
    be.add_argument("--output", default="")
    _common(be)
    a = ap.parse_args(argv)
    if a.cmd == "shuffle" and a.indices is not None and a.input is not None:
        sys.stderr.write("shuffle: --indices excludes an input file\n")
        return 2
    if getattr(a, "entropy", False) and a.seed != 0:
        sys.stderr.write("--entropy excludes --seed\n")
        return 2
    if a.cmd == "test":
        a.n_given = a.n is not None
        a.n = a.n if a.n is not None else 5
        return run_test(a)
    if a.cmd == "shuffle":
        return run_shuffle(a)
    return run_bench(a)


if __name__ == "__main__":
    raise SystemExit(main())
