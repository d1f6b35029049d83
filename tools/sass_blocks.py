"""Hottest straight-line blocks (by executed warp instructions) of a kernel's body."""
import csv
import io
import subprocess
import sys


def main(rep, kre, lim=0x7fffffff, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", f"regex:{kre}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia = hdr.index("Instructions Executed")
    L, seen, base = [], set(), None
    for r in rows[2:]:
        try:
            a = int(r[0], 16)
        except ValueError:
            continue
        if base is None:
            base = a
        if a in seen:
            continue
        seen.add(a)
        L.append((a - base, int(r[ia]) if r[ia].isdigit() else 0, r[1].strip()))
    L.sort()
    blocks = []
    for off, n, t in L:
        if off >= lim:
            continue
        if blocks and blocks[-1][1] == n and off - blocks[-1][2] == 16:
            blocks[-1][2] = off
            blocks[-1][3] += 1
            blocks[-1][4].append(t)
        else:
            blocks.append([off, n, off, 1, [t]])
    blocks.sort(key=lambda b: -b[1] * b[3])
    for b in blocks[:top]:
        print(hex(b[0]), hex(b[2]), "count", b[1], "len", b[3], "total", b[1] * b[3], "|",
              " ; ".join(x[:38] for x in b[4][:5]))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3], 16) if len(sys.argv) > 3 else 0x7fffffff)
