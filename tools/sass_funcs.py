"""Executed-instruction split of one kernel of an ncu report between its body
and the __noinline__ functions it calls (from the report's own SASS page).

    python tools/sass_funcs.py report.ncu-rep kernel_regex
"""
import collections
import csv
import io
import re
import subprocess
import sys


def main(rep, kre):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", f"regex:{kre}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia = hdr.index("Instructions Executed")
    isamp = hdr.index("Warp Stall Sampling (All Samples)")
    ins, seen = [], set()
    for r in rows[2:]:
        try:
            a = int(r[0], 16)
        except ValueError:
            continue
        if a in seen:
            continue
        seen.add(a)
        n = int(r[ia]) if r[ia].isdigit() else 0
        s = int(r[isamp]) if r[isamp].isdigit() else 0
        ins.append((a, r[1].strip(), n, s))
    ins.sort()
    addr = [a for a, *_ in ins]
    targets = sorted(set(int(t, 16) for _, x, _, _ in ins
                         for t in re.findall(r"CALL\.REL\.NOINC (0x[0-9a-f]+)", x)))
    ranges = []
    for t in targets:
        if t not in addr:
            continue
        i = addr.index(t)
        j = i
        while j < len(ins) and "RET" not in ins[j][1]:
            j += 1
        ranges.append((t, ins[min(j, len(ins) - 1)][0]))
    agg, samp, dp, cnt = collections.Counter(), collections.Counter(), collections.Counter(), collections.Counter()
    for a, x, n, s in ins:
        f = "body"
        for t, e in ranges:
            if t <= a <= e:
                f = hex(t - ins[0][0])
        agg[f] += n
        samp[f] += s
        cnt[f] += 1
        op = x.split()[0] if x.split() else "?"
        if op.startswith("@"):
            op = x.split()[1]
        if op.split(".")[0] in ("DFMA", "DMUL", "DADD"):
            dp[f] += n
    tot = sum(agg.values())
    print(f"total warp instructions {tot}")
    for f, n in agg.most_common():
        if n == 0:
            continue
        print(f"{f:10s} static {cnt[f]:6d} exec {n:12d} {n / tot:6.3f} DP {dp[f] / max(1, n):5.2f} "
              f"stall {samp[f]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
