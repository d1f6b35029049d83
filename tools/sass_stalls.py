"""Attribute ncu warp-stall samples (source page, SASS view) to opcode classes
and to the functions of a kernel (call targets split the listing).

    ncu -i rep --page source --csv --print-source sass -k regex:NAME > x.csv
    python tools/sass_stalls.py x.csv
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ai, si, ni = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
by_op = collections.Counter()
by_reason = collections.Counter()
by_block = collections.Counter()
tot = 0
block = 0
inst_tot = 0
dp = 0
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break  # first profiled launch only
    if len(r) <= ie:
        continue
    src = r[si].strip()
    try:
        s = float(r[ni] or 0)
        n = float(r[ie] or 0)
    except ValueError:
        continue
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    base = op.split(".")[0]
    by_op[base] += s
    tot += s
    inst_tot += n
    if base in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX", "MUFU"):
        dp += n if base != "MUFU" else 0
    for i in stall_cols:
        try:
            by_reason[hdr[i]] += float(r[i] or 0)
        except ValueError:
            pass
print(f"samples {tot:.0f}, warp instructions {inst_tot:.3e}, DP share of instructions {dp / max(1, inst_tot):.3f}")
for k, v in by_op.most_common(25):
    print(f"  {k:10s} {100 * v / tot:5.1f}%")
print("reasons:")
for k, v in by_reason.most_common(12):
    print(f"  {k:22s} {100 * v / tot:5.1f}%")
