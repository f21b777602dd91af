#!/usr/bin/env python
"""Turn a gpurun_out/<tag> profiling session (tools/gpu_profile.sh) into the
committed text summaries under profiles/<tag>_*.txt.

  python tools/summarize_profiles.py r1a
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

FULL_KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long scoreboard"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short scoreboard"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall MIO throttle"),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "stall LG throttle"),
]


def to_us(v, unit):
    v = float(v.replace(",", ""))
    return {"nsecond": v / 1e3, "ns": v / 1e3, "usecond": v, "us": v, "msecond": v * 1e3,
            "ms": v * 1e3, "second": v * 1e6, "s": v * 1e6}.get(unit, v)


def to_bytes(v, unit):
    v = float(v.replace(",", ""))
    mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
           "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9, "TB": 1e12}
    return v * mul.get(unit, 1)


def launch_summary(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, mi, ui, vi = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit",
                                             "Metric Value"))
    idi = hdr.index("ID")
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        names[r[idi]] = r[ki]
        per[r[idi]][r[mi]] = (r[vi], r[ui])
    agg = collections.defaultdict(lambda: [0.0, 0, 0.0])
    for lid, m in per.items():
        name = names[lid].split("(")[0].replace("void ", "")[:70]
        t = to_us(*m["gpu__time_duration.sum"]) if "gpu__time_duration.sum" in m else 0.0
        b = sum(to_bytes(*m[k]) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum") if k in m)
        agg[name][0] += t
        agg[name][1] += 1
        agg[name][2] += b
    tot = sum(a[0] for a in agg.values())
    lines = [f"{'kernel':70s} {'launches':>8s} {'total us':>10s} {'share':>6s} {'DRAM GB':>8s}"]
    for name, (t, n, b) in sorted(agg.items(), key=lambda x: -x[1][0]):
        lines.append(f"{name:70s} {n:8d} {t:10.1f} {100 * t / tot:5.1f}% {b / 1e9:8.3f}")
    lines.append(f"{'TOTAL (serialised, cold-cache ncu replay)':70s} {sum(a[1] for a in agg.values()):8d} "
                 f"{tot:10.1f}")
    return "\n".join(lines)


def full_summary(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        out.append("kernel: " + r[hdr.index("Kernel Name")])
        for k, label in FULL_KEYS:
            if k in hdr:
                out.append(f"  {label:28s} {r[hdr.index(k)]} {units[hdr.index(k)]}")
        out.append("")
    return "\n".join(out)


def main():
    tag = sys.argv[1]
    src = os.path.join(REPO, "gpurun_out", tag)
    dst = os.path.join(REPO, "profiles")
    os.makedirs(dst, exist_ok=True)
    for d in ("fwd", "bp"):
        p = os.path.join(src, f"launches_{d}.csv")
        if os.path.exists(p):
            open(os.path.join(dst, f"{tag}_launches_{d}.txt"), "w").write(
                f"# ncu launch list, one steady-state config-2 {d} step (tools/profile_step.py)\n"
                + launch_summary(p) + "\n")
        r = os.path.join(src, f"full_{d}.ncu-rep")
        if os.path.exists(r):
            open(os.path.join(dst, f"{tag}_ncu_full_{d}.txt"), "w").write(
                f"# ncu --set full, config-2 {d} step\n" + full_summary(r) + "\n")
    p = os.path.join(src, "launches.csv")
    if os.path.exists(p):
        open(os.path.join(dst, f"{tag}_launches.txt"), "w").write(
            "# ncu launch list, one config-4 step (type-2 + type-1, 100M points; "
            "tools/profile_step.py --config 4)\n" + launch_summary(p) + "\n")
    r = os.path.join(src, "full.ncu-rep")
    if os.path.exists(r):
        open(os.path.join(dst, f"{tag}_ncu_full.txt"), "w").write(
            "# ncu --set full, config-4 gather / spread\n" + full_summary(r) + "\n")
    for f in ("bench.json", "bench_back.json", "bench_c4.json", "smoke.txt", "pytest_gpu.txt"):
        p = os.path.join(src, f)
        if os.path.exists(p):
            open(os.path.join(dst, f"{tag}_{f}"), "w").write(open(p).read())
    print("wrote profiles for", tag)


if __name__ == "__main__":
    main()
