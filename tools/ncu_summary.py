#!/usr/bin/env python
"""Summarise ncu captures (from tools/profile.sh) into committed evidence:

    profiles/<round>_launches_<cfg>.csv   kernel, grid, block, duration (ns) per launch
    profiles/<round>_ncu_<cfg>.json       key metrics of the full-set capture of the dominant kernel
    profiles/<round>_summary.md           one table for all configs
    profiles/traffic.json                 dram bytes per launch (bench.py reads it for roofline.traffic)

usage: python tools/ncu_summary.py --round r01 [--src gpurun_out]
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "lts__t_sectors_srcunit_tex_op_read.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "launch__grid_size", "launch__block_size", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
    "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
]


def short_name(k: str) -> str:
    """Kernel name without template arguments and parameter list: 'void bsg::<unnamed>::k_part1<2, 1, ...>(...)'
    -> 'bsg::k_part1'."""
    head = re.sub(r"(<unnamed>|\(anonymous namespace\)|^void unnamed>|unnamed>)::", "", k.split("(")[0])
    bsg = "bsg::" in head or "k_" in head  # raw-page names lose the namespace prefix
    depth, base = 0, ""
    for ch in head:  # drop template argument lists
        if ch == "<":
            depth += 1
        elif ch == ">":
            depth -= 1
        elif depth == 0:
            base += ch
    name = base.replace("void ", "").strip().split("::")[-1]
    return ("bsg::" + name if bsg and name.startswith("k_") else name)[:60]


def launches(path: str):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, gi, bi, vi, mi = (hdr.index(x) for x in ("Kernel Name", "Grid Size", "Block Size", "Metric Value",
                                                  "Metric Name"))
    out = []
    for r in rows[1:]:
        if r[mi] == "gpu__time_duration.sum":
            out.append({"kernel": short_name(r[ki]), "full_name": r[ki][:160], "grid": r[gi], "block": r[bi],
                        "ns": float(r[vi].replace(",", ""))})
    return out


def raw_metrics_all(rep: str):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    return [raw_metrics_row(rows[0], rows[1], r) for r in rows[2:]]


def raw_metrics(rep: str):
    return raw_metrics_all(rep)[0]


def raw_metrics_row(hdr, units, vals):
    d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    res = {}
    for k in KEYS:
        if k in d:
            v, u = d[k]
            try:
                v = float(v.replace(",", ""))
            except ValueError:
                pass
            res[k] = {"value": v, "unit": u}
    stalls = []
    for h, (v, u) in d.items():
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                stalls.append((float(v.replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(s for s, _ in stalls) or 1.0
    res["stall_pct"] = {n: round(100 * s / tot, 1) for s, n in sorted(stalls, reverse=True)[:8]}
    res["kernel"] = short_name(d.get("Kernel Name", ("", ""))[0])
    return res


def to_bytes(entry):
    v, u = entry["value"], entry["unit"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
    return v * scale


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--src", default=os.path.join(ROOT, "gpurun_out"))
    ap.add_argument("--configs", default="c2,c3,c4,c5")
    args = ap.parse_args()
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    traffic_path = os.path.join(prof, "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    md = [f"# ncu evidence, round {args.round}", "",
          "Captured by `tools/profile.sh` under gpurun on one B200 (`--clock-control none`); summarised by "
          "`tools/ncu_summary.py`. Launch lists are cold-cache and serialised: compare shares, not absolutes.", ""]
    for cfg in args.configs.split(","):
        lp = os.path.join(args.src, f"launches_{cfg}.csv")
        if os.path.exists(lp):
            L = launches(lp)
            with open(os.path.join(prof, f"{args.round}_launches_{cfg}.csv"), "w", newline="") as f:
                w = csv.DictWriter(f, fieldnames=["kernel", "grid", "block", "ns", "full_name"])
                w.writeheader()
                w.writerows(L)
            tot = sum(x["ns"] for x in L)
            agg = {}
            for x in L:
                agg.setdefault(x["kernel"], [0, 0.0])
                agg[x["kernel"]][0] += 1
                agg[x["kernel"]][1] += x["ns"]
            md += [f"## {cfg}: launch list (`bench.py --config {cfg} --steps 2 --warmup 1`)", "",
                   "| kernel | launches | total ms | share |", "|---|---:|---:|---:|"]
            for k, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
                md.append(f"| `{k}` | {n} | {ns / 1e6:.3f} | {100 * ns / tot:.1f}% |")
            md.append("")
        for suffix in ("", "single"):
            rp = os.path.join(args.src, f"prof_{cfg}{suffix}.ncu-rep")
            if not os.path.exists(rp):
                continue
            RS = raw_metrics_all(rp)
            extra = os.path.join(args.src, f"prof_{cfg}rt.ncu-rep")  # a separate capture of more kernels of it
            if not suffix and os.path.exists(extra):
                RS = RS + raw_metrics_all(extra)
            with open(os.path.join(prof, f"{args.round}_ncu_{cfg}{suffix}.json"), "w") as f:
                json.dump(RS, f, indent=1)
            rd = sum(to_bytes(R["dram__bytes_read.sum"]) for R in RS if "dram__bytes_read.sum" in R)
            wr = sum(to_bytes(R["dram__bytes_write.sum"]) for R in RS if "dram__bytes_write.sum" in R)
            names = "+".join(R["kernel"] for R in RS)
            key = cfg + (f"_{suffix}" if suffix else "")
            traffic[key] = {"kernel": names, "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                            "source": f"profiles/{args.round}_ncu_{cfg}{suffix}.json",
                            "note": "sum over the kernels of one shuffle" if len(RS) > 1 else "one launch"}
            for R in RS:
                md += [f"## {key}: `{R['kernel']}` full-set capture", "", "| metric | value |", "|---|---:|"]
                for k in KEYS:
                    if k in R:
                        md.append(f"| `{k}` | {R[k]['value']} {R[k]['unit']} |")
                md.append(f"| warp stall mix (pc sampling) | "
                          f"{', '.join(f'{k} {v}%' for k, v in R['stall_pct'].items())} |")
                md.append("")
    with open(traffic_path, "w") as f:
        json.dump(traffic, f, indent=1)
    with open(os.path.join(prof, f"{args.round}_summary.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
