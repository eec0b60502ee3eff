"""Top SASS instructions by stall samples from `ncu --page source --csv --print-source sass` output, plus the
shared-memory wavefront totals per instruction (usage: python tools/sass_hot.py file.csv [N])."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr_i]
col = {n: i for i, n in enumerate(h)}
data = [r for r in rows[hdr_i + 1:] if len(r) == len(h) and r[0].startswith("0x")]
tot = sum(float(r[col["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
wf = sum(float(r[col["L1 Wavefronts Shared"]] or 0) for r in data)
wfi = sum(float(r[col["L1 Wavefronts Shared Ideal"]] or 0) for r in data)
print(f"samples {tot:.0f}; shared wavefronts {wf:.3g} (ideal {wfi:.3g})")
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for r in sorted(data, key=lambda r: -float(r[col["Warp Stall Sampling (All Samples)"]] or 0))[:N]:
    s = float(r[col["Warp Stall Sampling (All Samples)"]] or 0)
    print(f"{100*s/tot:5.1f}%  wf {r[col['L1 Wavefronts Shared']]:>10s}/{r[col['L1 Wavefronts Shared Ideal']]:>10s}  "
          f"{r[col['Address']][-5:]} {r[col['Source']].strip()[:70]}")
