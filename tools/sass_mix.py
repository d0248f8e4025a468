#!/usr/bin/env python
"""Dynamic SASS mix of one kernel launch from an ncu --page source --print-source sass CSV.

    ncu -i rep --page source --csv --print-source sass -k regex:NAME --launch-skip S --launch-count 1 > x.csv
    python tools/sass_mix.py x.csv
Prints warp-instructions executed and stall samples per opcode, plus the
hottest instruction ranges (by address order) to locate loops."""
import collections
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    H = rows[hdr]
    ie, ss = H.index("Instructions Executed"), H.index("Warp Stall Sampling (All Samples)")
    mix, stall = collections.Counter(), collections.Counter()
    seq = []
    for r in rows[hdr + 1:]:
        if len(r) != len(H):
            continue
        src = r[1].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0].rstrip(";")
        n, s = float(r[ie] or 0), float(r[ss] or 0)
        mix[op] += n
        stall[op] += s
        seq.append((op, n, s, src))
    tot, tots = sum(mix.values()), sum(stall.values()) or 1
    print(f"{tot:.4g} warp-instructions, {tots:.0f} stall samples")
    for op, n in mix.most_common(top):
        print(f"{op:10s} {n:12.4g} {100 * n / tot:5.1f}%  stall {100 * stall[op] / tots:5.1f}%")
    return seq


if __name__ == "__main__":
    main(sys.argv[1])
