"""Summarise ncu SASS-level warp-stall samples per warp-role region (development aid).
usage: ncu -i rep --page source --csv --print-source sass > x.csv; python tools/sass_stalls.py x.csv"""
import csv, sys, re
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) >= len(hdr) - 1]
region, regions, cur = [], {}, "prologue"
tot = 0
top = []
for d in data:
    src = d["Source"]
    if "USETMAXREG.TRY_ALLOC" in src: cur = "softmax"
    elif "USETMAXREG.DEALLOC" in src: cur = "dequant" if cur in ("softmax", "prologue") else "mma+tail"
    s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    regions.setdefault(cur, [0, 0])
    regions[cur][0] += s
    regions[cur][1] += int(d["Instructions Executed"] or 0)
    tot += s
    top.append((s, cur, d["Address"][-5:], src.strip()[:70]))
print("samples per region:", {k: (v[0], round(100 * v[0] / max(tot, 1), 1), v[1]) for k, v in regions.items()})
top.sort(reverse=True)
for t in top[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(t)
