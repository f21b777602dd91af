#!/usr/bin/env python
"""Summarise an ncu report's SASS source page: instruction mix and the hottest
instructions (by executed count and by stall samples).

  python tools/ncu_hotspots.py report.ncu-rep kernel_regex [top]
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass",
                          "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:]
            if len(r) == len(hdr) and r[0] != "Address"]
    ie, ss = "Instructions Executed", "Warp Stall Sampling (All Samples)"
    tot = sum(float(d[ie] or 0) for d in data) or 1
    stot = sum(float(d[ss] or 0) for d in data) or 1
    mix = collections.Counter()
    stall = collections.Counter()
    for d in data:
        op = d["Source"].split()[0] if d["Source"].split() else "?"
        if op.startswith("@"):
            op = d["Source"].split()[1]
        op = op.split(".")[0]
        mix[op] += float(d[ie] or 0)
        stall[op] += float(d[ss] or 0)
    print(f"total warp instructions {tot:.3e}, stall samples {stot:.0f}")
    print("opcode mix (share of executed / share of stall samples):")
    for op, v in mix.most_common(top):
        print(f"  {op:10s} {100 * v / tot:5.1f}%  {100 * stall[op] / stot:5.1f}%")
    print("hottest by stall samples:")
    for d in sorted(data, key=lambda d: -float(d[ss] or 0))[:top]:
        print(f"  {100 * float(d[ss]) / stot:5.1f}%  {d['Source'].strip()[:90]}")


if __name__ == "__main__":
    main()
