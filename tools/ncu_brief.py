#!/usr/bin/env python
"""Key ncu sections of every kernel in a report: python tools/ncu_brief.py X.ncu-rep"""
import csv
import io
import subprocess
import sys

SECTIONS = ('GPU Speed Of Light Throughput', 'Memory Workload Analysis', 'Compute Workload Analysis',
            'Occupancy', 'Warp State Statistics', 'Launch Statistics')
KEEP = ('Duration', 'Memory Throughput', 'DRAM Throughput', 'L1/TEX Cache Throughput',
        'L2 Cache Throughput', 'Compute (SM) Throughput', 'Issue Slots Busy', 'L1/TEX Hit Rate',
        'L2 Hit Rate', 'Mem Pipes Busy', 'Warp Cycles Per Issued Instruction', 'Achieved Occupancy',
        'Theoretical Occupancy', 'Registers Per Thread', 'Dynamic Shared Memory Per Block',
        'Grid Size', 'Block Size', 'Block Limit Shared Mem', 'Block Limit Registers')


def main():
    txt = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[0]
    cur = None
    for r in rows[1:]:
        k = r[h.index('Kernel Name')][:90]
        if k != cur:
            print("==", k)
            cur = k
        sec, name = r[h.index('Section Name')], r[h.index('Metric Name')]
        if sec in SECTIONS and name in KEEP:
            print(f"   {name:40s} {r[h.index('Metric Value')]} {r[h.index('Metric Unit')]}")
    raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hh = rr[0]
    stall = [c for c in hh if c.startswith("smsp__average_warps_issue_stalled_") and c.endswith("_per_issue_active.ratio")]
    for row in rr[2:]:
        vals = sorted(((float(row[hh.index(c)] or 0), c) for c in stall), reverse=True)[:6]
        print("   top stalls:", ", ".join(f"{c[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]}={v:.2f}" for v, c in vals))


if __name__ == "__main__":
    main()
