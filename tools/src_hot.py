"""Top CUDA source lines by warp-stall samples and shared wavefronts from
`ncu -i rep --page source --csv --kernel-name K --print-source cuda,sass` (usage: src_hot.py file.csv [N])."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
S = h.index("Warp Stall Sampling (All Samples)")
W = h.index("L1 Wavefronts Shared")
WI = h.index("L1 Wavefronts Shared Ideal")
lines = [r for r in rows[hi + 1:] if r and r[0] not in ("",) and r[0].isdigit()]
def num(x):
    try:
        return float(x)
    except ValueError:  # "-", "" or a source line of another file section that spilled into the column
        return 0.0
tot = sum(num(r[S]) for r in lines)
print(f"samples {tot:.0f}, shared wavefronts {sum(num(r[W]) for r in lines):.3g} (ideal {sum(num(r[WI]) for r in lines):.3g})")
for r in sorted(lines, key=lambda r: -num(r[S]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{100 * num(r[S]) / tot:5.1f}%  wf {num(r[W]):10.3g}/{num(r[WI]):9.3g}  L{r[0]:>4s} {r[1].strip()[:90]}")
