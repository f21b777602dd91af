#!/usr/bin/env python
"""Per-CUDA-source-line instruction and stall totals of one kernel in an ncu report.

  python tools/ncu_lines.py report.ncu-rep kernel_regex [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    fname = "?"
    hdr = None
    agg = {}
    tot_i = tot_s = 0.0
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8 or not r[0]:
            continue
        try:
            ins = float(r[7] or 0)
            st = float(r[4] or 0)
        except ValueError:
            continue
        key = f"{fname}:{r[0]}"
        a = agg.setdefault(key, [0.0, 0.0, r[1][:90]])
        a[0] += ins
        a[1] += st
        tot_i += ins
        tot_s += st
    print(f"warp instructions {tot_i:.3e}, stall samples {tot_s:.0f}")
    for k, (i, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * i / tot_i:6.2f}% ins {100 * s / max(tot_s, 1):6.2f}% stall  {k:24s} {src}")


if __name__ == "__main__":
    main()
