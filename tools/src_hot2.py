"""Top CUDA source lines by warp-stall samples from
`ncu -i rep --page source --csv --kernel-name K --print-source cuda,sass` (mixed cuda/sass layout).
usage: src_hot2.py file.csv [N]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
agg, src, fname, hdr = defaultdict(float), {}, "?", None
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = r
        S = hdr.index("Warp Stall Sampling (All Samples)")
    elif hdr and r[0].isdigit() and len(r) > S:
        try:
            v = float(r[S]) if r[S] not in ("", "-") else 0.0
        except ValueError:
            continue
        agg[(fname, int(r[0]))] += v
        src[(fname, int(r[0]))] = r[1].strip()
tot = sum(agg.values()) or 1
print(f"samples {tot:.0f}")
for k in sorted(agg, key=lambda k: -agg[k])[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{100 * agg[k] / tot:5.1f}%  {k[0]}:{k[1]:<5d} {src[k][:100]}")
