"""Top stalled SASS instructions (ncu source page csv, first launch) with context.
    python tools/sass_top.py x.csv [N] [CONTEXT]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 12
CTX = int(sys.argv[3]) if len(sys.argv) > 3 else 0
hdr = rows[1]
ni, ie = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
sc = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not" not in h]
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) <= ie:
        continue
    data.append((r[1].strip(), float(r[ni] or 0), float(r[ie] or 0), r))
tot = sum(d[1] for d in data)
order = sorted(range(len(data)), key=lambda i: -data[i][1])[:N]
for i in order:
    src, s, n, r = data[i]
    rs = sorted(((float(r[k] or 0), hdr[k][6:]) for k in sc), reverse=True)[:2]
    print(f"{i:6d} {100 * s / tot:5.1f}% n={n:9.0f} {src[:60]:60s} {rs}")
    for j in range(max(0, i - CTX), min(len(data), i + CTX + 1)):
        if j != i and CTX:
            print(f"        {j:6d} {data[j][1]:5.0f} {data[j][2]:9.0f} {data[j][0][:70]}")
