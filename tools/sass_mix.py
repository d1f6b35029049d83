"""Instruction mix and stall hot spots of one kernel in an ncu report (SASS page).

    python tools/sass_mix.py report.ncu-rep kernel_regex
"""
import collections
import csv
import io
import subprocess
import sys


def main(path, kre):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", f"regex:{kre}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia = hdr.index("Instructions Executed")
    isamp = hdr.index("Warp Stall Sampling (All Samples)")
    mix = collections.Counter()
    samp = collections.Counter()
    tot = 0
    lines = []
    for r in rows[2:]:
        if len(r) <= ia or not r[ia].strip().isdigit():
            continue
        n = int(r[ia])
        s = int(r[isamp]) if r[isamp].strip().isdigit() else 0
        op = r[1].split()[0] if r[1].split() else "?"
        if op.startswith("@"):
            op = r[1].split()[1]
        base = op.split(".")[0]
        mix[base] += n
        samp[base] += s
        tot += n
        lines.append((s, n, r[0], r[1].strip()))
    print(f"total warp instructions {tot}")
    dp = sum(v for k, v in mix.items() if k in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX"))
    print(f"DP share {dp / tot:.3f}")
    for k, v in mix.most_common(25):
        print(f"{k:10s} {v:12d} {v / tot:6.3f}  stall-samples {samp[k]}")
    print("hottest (stall samples):")
    for s, n, a, t in sorted(lines, reverse=True)[:25]:
        print(f"{s:6d} {n:10d} {a} {t}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
