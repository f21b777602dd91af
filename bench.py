#!/usr/bin/env python
"""Benchmark: NUFFT cone-beam forward projector, BASELINE.json config 2.

One step = one full forward projection (``nufft_forward_project``) of the
seeded 256^3 30-ellipsoid phantom onto 360 cone-beam views (256^2 detector),
with the reference's view batching and per-batch resample scalings.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config 2] [--direction forward|back]

Under torchrun (N > 1) the views are sharded across ranks (strong scaling:
360 views in total); every rank computes the radial lattice itself.
``--impl reference`` times the CPU oracle port (oracle/cbn_oracle.py, the
reference algorithm in numpy/scipy) on a bounded, extrapolated sample.
Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

PEAKS_FILE = os.path.join(REPO, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0
# dram__bytes_read.sum + dram__bytes_write.sum per config-2 step, summed over
# the stage's launches, from the committed ncu launch lists
# (profiles/r1j_launches_fwd.txt, profiles/r1j_launches_bp.txt); stages not
# captured there report null
TRAFFIC: dict = {"resample_gather": 2.373e9, "grangeat_spread": 2.441e9 + 1.858e9,
                 "spectrum_gather": 0.966e9, "bp_spread": 1.024e9,
                 "transpose_spread": 0.839e9 + 0.725e9}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--direction", choices=["forward", "back"], default="forward")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def hbm_peak():
    try:
        with open(PEAKS_FILE) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(mx)) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------- roofline helpers
def stage_bytes(stage: str, w, views: int):
    """Algorithmic bytes of one step's stage: (compulsory HBM bytes, on-chip tap
    bytes).  DESIGN.md section 4 derives each; nodes/targets generated from
    index tables stream no coordinates (c = 0 in SURVEY 8(d))."""
    spec, cfg = w.spec, w.cfg
    n = w.n
    K3 = (2 * n) ** 3
    M = spec.n_rho * spec.n_theta * spec.n_phi
    dr = spec.n_rho + 2 * cfg.rho_pad
    D = dr * spec.n_theta * spec.n_phi
    Kr = 8 * D
    tpv = cfg.n_mu * cfg.n_t                  # umbrella targets per view
    grid2 = 4 * w.geom.nu * w.geom.nv          # oversampled detector cells per view
    J, Jr, Jg = 6, 3, 5
    if stage == "spectrum_gather":             # read K^3 grid once, write M lattice values
        return 8.0 * K3 + 8.0 * M, 8.0 * J ** 3 * M
    if stage == "resample_gather":             # read the resample grid once, write f32 values
        return 8.0 * Kr + 4.0 * tpv * views + 32.0 * tpv, 8.0 * Jr ** 3 * tpv * views
    if stage == "grangeat_spread":             # read t-spectra, RED the 2D grids once
        return 8.0 * tpv * views + 8.0 * grid2 * views + 56.0 * tpv, 16.0 * Jg ** 2 * tpv * views
    if stage == "bp_spread":                   # read M lattice values, write K^3 grid once
        return 8.0 * M + 8.0 * K3, 16.0 * J ** 3 * M
    if stage == "transpose_spread":            # transpose + gather: values 3x, grid once
        return 3 * 4.0 * tpv * views + 8.0 * Kr, 4.0 * Jr ** 3 * tpv * views
    if stage == "spectrum_pad":
        return 4.0 * n ** 3 + 8.0 * K3, 0.0
    if stage == "resample_pad":
        return 8.0 * D + 8.0 * Kr, 0.0
    return None


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_1605_05231_b200 import _lib
    from paper_1605_05231_b200.pipeline import Projector
    from paper_1605_05231_b200.workloads import workload

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1605_05231_b200 import pipeline as _pl
    from paper_1605_05231_b200 import sharding
    w = workload(args.config)
    V = w.geom.n_views
    per_view = w.cfg.n_mu * w.cfg.n_t
    lo, hi = sharding.view_shard(V, world, rank,
                                 sharding.view_batches(V, per_view, _pl._TARGET_BATCH))
    vol_host = w.volume()
    lib = _lib.load()
    direction = 1 if args.direction == "forward" else 2
    proj = Projector(w.geom, w.cfg, w.n, w.voxel, direction)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    if direction == 1:
        x_dev = torch.from_numpy(vol_host).cuda()
        if world > 1:
            # radial nodes and views sharded; the lattice summed with one NCCL all-reduce
            def step():
                return proj.forward_sharded(x_dev, lo, hi)
        else:
            def step():
                return proj.forward(x_dev, lo, hi)
    else:
        frames_dev = Projector(w.geom, w.cfg, w.n, w.voxel, 1).forward(torch.from_numpy(vol_host).cuda())
        x_dev = frames_dev
        if world > 1:
            # views and radial nodes sharded; lattice and grid summed with NCCL
            x_loc = x_dev[lo:hi].contiguous()

            def step():
                return proj.backproject_sharded(x_loc, lo, hi)
        else:
            def step():
                return proj.backproject(x_dev)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    n0 = lib.cbn_launch_count()
    torch.cuda.synchronize()
    barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = lib.cbn_launch_count() - n0
    ms = t0.elapsed_time(t1)
    clk = clocks.stop()
    # per-stage kernel times: a separate pass of the same steps with stage
    # events on, during which the operators keep every view block on one
    # stream (no overlap), so each stage's event time is its own kernels'
    # time and the shares agree with the serialised ncu launch list
    lib.cbn_projector_set_timing(proj._h, 1)
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    import ctypes
    cnt = ctypes.c_int32(64)
    stage_ms = (ctypes.c_double * 64)()
    names = ctypes.create_string_buffer(4096)
    lib.cbn_projector_stage_times(proj._h, stage_ms, ctypes.byref(cnt), names, 4096, 1)
    lib.cbn_projector_set_timing(proj._h, 0)
    stages = {nm: stage_ms[i] / args.steps
              for i, nm in enumerate(names.value.decode().split(";")[:cnt.value])}
    ms_t = torch.tensor([ms], device="cuda")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    units = V if direction == 1 else V        # views per step across all ranks
    value = units * args.steps / (ms_max / 1e3)

    # ---- end to end through the public API path: pinned host in, host out
    e2e = None
    if not args.no_e2e:
        if direction == 1:
            host_in = torch.from_numpy(vol_host).pin_memory()
            host_out = torch.empty((hi - lo, w.geom.nu, w.geom.nv), dtype=torch.float32).pin_memory()
        else:
            host_in = x_dev.cpu().pin_memory()
            host_out = torch.empty((w.n,) * 3, dtype=torch.float32).pin_memory()

        def run(dev):
            if direction == 1:
                return proj.forward_sharded(dev, lo, hi) if world > 1 else proj.forward(dev, lo, hi)
            if world > 1:
                return proj.backproject_sharded(dev[lo:hi].contiguous(), lo, hi)
            return proj.backproject(dev)

        # Pipelined through the public API: a copy stream brings step k+1's input
        # in while step k computes and takes step k-1's result out, so every
        # step's H2D and D2H are inside the timed region but overlap the compute
        copy_s = torch.cuda.Stream()
        dev_in = [torch.empty(host_in.shape, dtype=host_in.dtype, device="cuda") for _ in range(2)]
        host_outs = [host_out, torch.empty_like(host_out).pin_memory()]
        in_ready = [torch.cuda.Event() for _ in range(2)]
        out_ready = [torch.cuda.Event() for _ in range(2)]

        def pipeline(nsteps, start_event=None):
            with torch.cuda.stream(copy_s):
                if start_event is not None:
                    copy_s.wait_event(start_event)
                dev_in[0].copy_(host_in, non_blocking=True)
                in_ready[0].record(copy_s)
            for k in range(nsteps):
                slot = k % 2
                if k + 1 < nsteps:               # next input, once step k-1 released its slot
                    with torch.cuda.stream(copy_s):
                        if k >= 1:
                            copy_s.wait_event(out_ready[1 - slot])
                        dev_in[1 - slot].copy_(host_in, non_blocking=True)
                        in_ready[1 - slot].record(copy_s)
                stream.wait_event(in_ready[slot])
                out = run(dev_in[slot])
                out_ready[slot].record(stream)
                with torch.cuda.stream(copy_s):
                    copy_s.wait_event(out_ready[slot])
                    host_outs[slot].copy_(out, non_blocking=True)
                out.record_stream(copy_s)

        pipeline(2)
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        wall0 = time.perf_counter()
        e0.record(stream)
        pipeline(args.steps, e0)
        e1.record(copy_s)
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
        barrier()
        et = torch.tensor([e0.elapsed_time(e1)], device="cuda")
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e_ms = float(et.item())
        e2e = {"value": units * args.steps / (e_ms / 1e3), "unit": "views/s",
               "h2d_bytes_per_step": int(host_in.numel() * 4),
               "d2h_bytes_per_step": int(host_out.numel() * 4),
               "wall_s": wall, "api": "Projector.forward/backproject with pinned host tensors, "
                                      "copies on a second stream overlapping the previous/next step"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    peak, peak_kind = hbm_peak()
    # per-kernel rooflines for the stages that are a single kernel of ours
    kernels = {}
    for st, t_ms in stages.items():
        sb = stage_bytes(st, w, hi - lo)
        if sb is None or t_ms <= 0:
            continue
        hbm_b, chip_b = sb
        ach = hbm_b / (t_ms / 1e3) / 1e9
        kernels[st] = {"ms_per_step": round(t_ms, 3), "hbm_bytes": hbm_b,
                       "achieved_gbs": round(ach, 1), "hbm_frac": round(ach / peak, 4),
                       "onchip_tap_bytes": chip_b,
                       "onchip_tbs": round(chip_b / (t_ms / 1e3) / 1e12, 2)}
    roofline = None
    if kernels:
        st = max(kernels, key=lambda k: kernels[k]["ms_per_step"])
        kk = kernels[st]
        roofline = {"kernel": st, "bound": "hbm", "achieved": kk["achieved_gbs"], "peak": peak,
                    "unit": "GB/s", "frac": kk["hbm_frac"], "traffic": TRAFFIC.get(st),
                    "peak_kind": peak_kind,
                    "note": "achieved = compulsory bytes / CUDA-event stage time (serialised stage pass); these "
                            "gathers/spreads are bound on chip (tap traffic, onchip_tbs)",
                    "onchip_tbs": kk["onchip_tbs"]}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_sample(w, direction, n_samples=1)
    out = {
        "metric": "cone-beam views/s (NUFFT forward projector)" if direction == 1
        else "cone-beam views/s (NUFFT backprojector)",
        "value": round(value, 3),
        "unit": "views/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": max(args.warmup, 3),
        "ms_per_step": round(ms_max / args.steps, 3),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "c64/f32 (fp64 index math)",
        "data": f"synthetic: seeded random-ellipsoid phantom (BASELINE {w.name})",
        "config": {"workload": f"{w.name} {args.direction}: {w.n}^3 volume, "
                               f"{w.spec.n_rho}x{w.spec.n_theta}x{w.spec.n_phi} radial lattice, "
                               f"{V} views of {w.geom.nu}^2, KB J=6 sigma=2, resample J=3",
                   "views": V, "views_per_rank": hi - lo,
                   "parallelism": f"views sharded x{world}" + (
                       "" if world == 1 else ", radial nodes sharded, NCCL all-reduce of the "
                       + ("lattice" if direction == 1 else "lattice + grid")),
                   "l2": "working set > L2 (resample grid 2.4 GB per view batch)"},
        "e2e": e2e,
        "gpu_launches": int(launches),
        "gpu_launches_per_step": int(launches) // max(args.steps, 1),
        "clocks": clk,
        "roofline": roofline,
        "kernels": kernels,
        "stages_ms_per_step": {k: round(v, 3) for k, v in stages.items()},
        "cpu_baseline": cpu,
    }
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------- config 4: NUFFT stress microbench
C4_POINTS = 100_000_000
C4_GRID = 256
C4_J = 8


def run_nufft4(args):
    """BASELINE config 4: type-2 gather + type-1 spread of 100M float32 points
    (i.i.d. uniform in [-pi, pi)^3) against a 256^3 CN(0,1) grid, KB J=8,
    sigma 2.  One step = one type-2 and one type-1 over every point; the
    metric counts points per second through that pair.  Under torchrun the
    points are split evenly across ranks; type-2 needs no exchange (x is
    replicated), type-1's 256^3 outputs are summed and scattered by z-slab
    with one NCCL reduce-scatter (linear, so reducing after the crop moves
    1/8 of the oversampled grid's bytes)."""
    import torch
    import torch.distributed as dist
    from paper_1605_05231_b200 import _lib, nufft
    from paper_1605_05231_b200.workloads import config4_inputs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    m_total = int(os.environ.get("CBN_C4_POINTS", C4_POINTS))
    x_host, pts = config4_inputs(n_points=m_total, grid=C4_GRID)
    lo = m_total * rank // world
    hi = m_total * (rank + 1) // world
    pts = np.ascontiguousarray(pts[lo:hi])
    m = hi - lo
    lib = _lib.load()
    torch.cuda.synchronize()
    tp = time.perf_counter()
    plan = nufft.plan_nufft((C4_GRID,) * 3, pts, 2.0, C4_J)
    torch.cuda.synchronize()
    plan_s = time.perf_counter() - tp
    stream = torch.cuda.current_stream()
    import ctypes
    sp = ctypes.c_void_p(stream.cuda_stream)
    x = torch.from_numpy(x_host).cuda()
    y = torch.empty(m, dtype=torch.complex64, device="cuda")
    xa = torch.empty((C4_GRID,) * 3, dtype=torch.complex64, device="cuda")
    slab = torch.empty((C4_GRID // world, C4_GRID, C4_GRID), dtype=torch.complex64, device="cuda") \
        if world > 1 else None

    def type2():
        _lib.check(lib.cbn_nufft_type2(plan.handle, ctypes.c_void_p(x.data_ptr()),
                                       ctypes.c_void_p(y.data_ptr()), sp))

    def type1():
        _lib.check(lib.cbn_nufft_type1(plan.handle, ctypes.c_void_p(y.data_ptr()),
                                       ctypes.c_void_p(xa.data_ptr()), sp))
        if world > 1:
            dist.reduce_scatter_tensor(slab, xa)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(args.warmup, 3)):
        type2()
        type1()
    torch.cuda.synchronize()
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    n0 = lib.cbn_launch_count()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps + 1)]
    torch.cuda.synchronize()
    barrier()
    ev[0].record(stream)
    for k in range(args.steps):
        type2()
        ev[2 * k + 1].record(stream)
        type1()
        ev[2 * k + 2].record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = lib.cbn_launch_count() - n0
    clk = clocks.stop()
    t2 = sum(ev[2 * k].elapsed_time(ev[2 * k + 1]) for k in range(args.steps)) / args.steps
    t1 = sum(ev[2 * k + 1].elapsed_time(ev[2 * k + 2]) for k in range(args.steps)) / args.steps
    ms = ev[0].elapsed_time(ev[-1])
    tt = torch.tensor([ms, t2, t1], device="cuda")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms_max, t2, t1 = (float(v) for v in tt.tolist())
    value = m_total * args.steps / (ms_max / 1e3) / 1e6

    e2e = None
    if not args.no_e2e:
        # public API with pinned host buffers: x and the node values in, results out
        hx = torch.from_numpy(x_host).pin_memory()
        hy = torch.from_numpy(np.zeros(m, np.complex64)).pin_memory()
        hxa = torch.empty((C4_GRID,) * 3, dtype=torch.complex64).pin_memory()

        def e2e_step():
            xd = nufft.nufft_forward(plan, hx.to("cuda", non_blocking=True))
            hy.copy_(xd, non_blocking=True)
            yd = hy.to("cuda", non_blocking=True)
            hxa.copy_(nufft.nufft_adjoint(plan, yd), non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        et = torch.tensor([e0.elapsed_time(e1)], device="cuda")
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e_ms = float(et.item())
        e2e = {"value": round(m_total * args.steps / (e_ms / 1e3) / 1e6, 3), "unit": "Msamples/s",
               "h2d_bytes_per_step": int(hx.numel() * 8 + hy.numel() * 8),
               "d2h_bytes_per_step": int(hy.numel() * 8 + hxa.numel() * 8),
               "api": "nufft_forward / nufft_adjoint on pinned host-staged tensors"}
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    peak, peak_kind = hbm_peak()
    K3 = (2 * C4_GRID) ** 3
    # compulsory bytes: gather reads the oversampled grid once + 12 B nodes +
    # 8 B output per point; spread reads 12 B nodes + 8 B values and writes
    # the grid once
    gb = {"type2_step": 8.0 * K3 + 20.0 * m, "type1_step": 8.0 * K3 + 20.0 * m}
    taps = C4_J ** 3
    kernels = {
        "type2": {"ms_per_step": round(t2, 3), "achieved_gbs": round(gb["type2_step"] / t2 / 1e6, 1),
                  "onchip_tap_bytes": 8.0 * taps * m,
                  "onchip_tbs": round(8.0 * taps * m / t2 / 1e9, 2),
                  "msamples_s": round(m / t2 / 1e3, 2)},
        "type1": {"ms_per_step": round(t1, 3), "achieved_gbs": round(gb["type1_step"] / t1 / 1e6, 1),
                  "onchip_tap_bytes": 16.0 * taps * m,          # shared-memory read + write per tap
                  "onchip_tbs": round(16.0 * taps * m / t1 / 1e9, 2),
                  "msamples_s": round(m / t1 / 1e3, 2)},
    }
    st = "type1" if t1 >= t2 else "type2"
    roofline = {"kernel": st + " (whole transform incl. FFT)", "bound": "hbm",
                "achieved": kernels[st]["achieved_gbs"], "peak": peak, "unit": "GB/s",
                "frac": round(kernels[st]["achieved_gbs"] / peak, 4), "traffic": None,
                "peak_kind": peak_kind, "onchip_tbs": kernels[st]["onchip_tbs"]}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_sample_nufft4()
    out = {
        "metric": "NUFFT nonuniform Msamples/s (fwd+adj)",
        "value": round(value, 3), "unit": "Msamples/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": round(ms_max / args.steps, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "c64/f32 (fp64 index math)",
        "data": "synthetic: 256^3 CN(0,1) grid (seed 4), float32 points U[-pi,pi)^3 (seed 5)",
        "config": {"workload": f"config4: {m_total} points, {C4_GRID}^3 grid, KB J={C4_J}, sigma 2, "
                               "one type-2 + one type-1 per step",
                   "points_per_rank": m, "parallelism": f"points sharded x{world}",
                   "plan_s": round(plan_s, 3),
                   "l2": "working set > L2 (1.07 GB oversampled grid, 1.2 GB nodes)"},
        "e2e": e2e, "gpu_launches": int(launches),
        "gpu_launches_per_step": int(launches) // max(args.steps, 1),
        "clocks": clk, "roofline": roofline, "kernels": kernels,
        "stages_ms_per_step": {"type2": round(t2, 3), "type1": round(t1, 3)},
        "cpu_baseline": cpu,
    }
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cpu_sample_nufft4(n_sample: int = 1 << 17):
    """Oracle port on a 2^17-point sample of config 4 (plan excluded, like the
    GPU value): per-point type-2 + type-1 cost, plus one 512^3 FFT per
    transform, extrapolated to 100M points."""
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import cbn_oracle as orc
    from paper_1605_05231_b200.workloads import config4_inputs
    cores = os.cpu_count() or 1
    orc.WORKERS = cores
    x, pts = config4_inputs(n_points=n_sample, grid=C4_GRID)
    x = x.astype(np.complex128)
    plan = orc.make_plan((C4_GRID,) * 3, pts.astype(np.float64), 2.0, C4_J)
    y = np.ones(n_sample, np.complex128)
    t = time.perf_counter()
    orc.type2(plan, x)
    t2 = time.perf_counter() - t
    t = time.perf_counter()
    orc.type1(plan, y)
    t1 = time.perf_counter() - t
    # separate the FFT (fixed per transform) from the per-point part
    g = np.zeros((2 * C4_GRID,) * 3, np.complex128)
    t = time.perf_counter()
    orc.sfft.fftn(g, overwrite_x=True, workers=orc.WORKERS)
    tf = time.perf_counter() - t
    per_point = max(t2 + t1 - 2 * tf, 1e-12) / n_sample
    total = per_point * C4_POINTS + 2 * tf
    return {"value": round(C4_POINTS / total / 1e6, 6), "unit": "Msamples/s", "cores": cores,
            "kind": "port",
            "sample": f"oracle port: type-2 {t2:.2f}s + type-1 {t1:.2f}s on {n_sample} points "
                      f"(512^3 FFT {tf:.2f}s each), per-point part extrapolated to {C4_POINTS}",
            "extrapolated": True}


# --------------------------------------------------------- CPU (oracle) leg
def cpu_sample(w, direction: int, n_samples: int = 1):
    """Time the oracle port on a bounded sample and extrapolate to the full
    workload: one 2^21-node spectrum sub-plan (of ceil(M / 2^21)) and the
    resample + reverse Grangeat of one view (of V)."""
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import cbn_oracle as orc
    cores = os.cpu_count() or 1
    orc.WORKERS = cores
    spec, cfg, geom = w.spec, w.cfg, w.geom
    M = spec.n_rho * spec.n_theta * spec.n_phi
    n_chunks = -(-M // orc.PLAN_CHUNK)
    vol = w.volume(np.float64)
    nodes_all = None
    t_chunk, t_view = [], []
    rng = np.random.default_rng(0)
    for s in range(n_samples):
        if direction != 1:
            break
        # spectrum sub-plan sample
        t = time.perf_counter()
        if nodes_all is None:
            nodes_all = orc.wrap(orc.radial_direction_nodes(spec, w.voxel))
        lo = (s % n_chunks) * orc.PLAN_CHUNK
        hi = min(lo + orc.PLAN_CHUNK, M)
        plan = orc.make_plan((w.n,) * 3, nodes_all[lo:hi], 2.0, 6)
        orc.type2(plan, vol.astype(np.complex128))
        t_chunk.append(time.perf_counter() - t)
        del plan
        # one view: umbrella targets, per-batch resample plan + apply, reverse Grangeat
        t = time.perf_counter()
        lattice = (rng.standard_normal((spec.n_rho, spec.n_theta, spec.n_phi))
                   + 1j * rng.standard_normal((spec.n_rho, spec.n_theta, spec.n_phi)))
        t_lat = time.perf_counter() - t
        t = time.perf_counter()
        per_view = cfg.n_mu * cfg.n_t
        batch = orc.view_batches(geom.n_views, per_view)[s % geom.n_views]
        targets, valid = orc.umbrella_targets(geom, spec, batch, cfg.n_mu, cfg.n_t, cfg.t_pitch_mm)
        rs = orc.make_resampler(spec, targets, cfg.rho_pad, cfg.resample_j)
        vals = np.real(orc.resample_forward(rs, lattice))
        gp = orc.make_grangeat(geom, cfg.n_mu, cfg.n_t, t_pitch_mm=cfg.t_pitch_mm,
                               t_taper=cfg.t_taper)
        for i in range(len(batch)):
            orc.grangeat_reverse(vals[i * per_view:(i + 1) * per_view].reshape(cfg.n_mu, cfg.n_t), gp)
        t_view.append((time.perf_counter() - t) / len(batch))
        del lattice, rs
    if direction != 1:
        return None
    tc, tv = float(np.mean(t_chunk)), float(np.mean(t_view))
    total = n_chunks * tc + geom.n_views * tv
    return {"value": round(geom.n_views / total, 6), "unit": "views/s", "cores": cores,
            "kind": "port",
            "sample": f"oracle port: {len(t_chunk)} of {n_chunks} spectrum sub-plans (2^21 nodes) "
                      f"+ {len(t_view)} view(s) of {geom.n_views} (resample plan+apply, reverse "
                      f"Grangeat); extrapolated linearly; sub-plan {tc:.2f}s, view {tv:.2f}s; "
                      "scipy.fft uses all cores, the numpy gather/bincount one",
            "extrapolated": True}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1605_05231_b200.workloads import workload
    w = workload(args.config)
    direction = 1 if args.direction == "forward" else 2
    t0 = time.perf_counter()
    # each step is one bounded CPU sample (~17 s at config 2); no warm-up is
    # needed on the CPU and at most 3 samples are taken so the arm stays
    # within a few minutes for any --steps
    vals = [cpu_sample(w, direction, 1) for _ in range(max(1, min(args.steps, 3)))]
    timed = [v for v in vals if v is not None]
    wall = time.perf_counter() - t0
    if not timed:
        print(json.dumps({"impl": "reference", "unavailable": "backprojector CPU sample not implemented"}))
        return
    value = float(np.mean([v["value"] for v in timed]))
    cpu = dict(timed[-1])
    cpu["value"] = round(value, 6)
    out = {"impl": "reference",
           "metric": "cone-beam views/s (NUFFT forward projector)",
           "value": round(value, 6), "unit": "views/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(1e3 * w.geom.n_views / value, 1),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
           "dtype": "f64/c128", "data": f"synthetic: seeded random-ellipsoid phantom (BASELINE {w.name})",
           "config": {"workload": f"{w.name} {args.direction} (CPU oracle port, extrapolated)"},
           "cpu_baseline": cpu,
           "e2e": {"value": round(value, 6), "unit": "views/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0},
           "wall_s": round(wall, 1)}
    print(json.dumps(out), flush=True)


def run_reference_nufft4(args):
    if int(os.environ.get("RANK", "0")) != 0:
        return
    t0 = time.perf_counter()
    vals = [cpu_sample_nufft4() for _ in range(max(1, min(args.steps, 3)))]   # <= 3 samples
    timed = vals
    value = float(np.mean([v["value"] for v in timed]))
    cpu = dict(timed[-1])
    cpu["value"] = round(value, 6)
    print(json.dumps({
        "impl": "reference", "metric": "NUFFT nonuniform Msamples/s (fwd+adj)",
        "value": round(value, 6), "unit": "Msamples/s",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * C4_POINTS / (value * 1e6), 1),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64/c128",
        "data": "synthetic: config 4 inputs",
        "config": {"workload": "config4 (CPU oracle port, extrapolated)"}, "cpu_baseline": cpu,
        "e2e": {"value": round(value, 6), "unit": "Msamples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": round(time.perf_counter() - t0, 1)}), flush=True)


def main():
    args = parse_args()
    if args.config == 4:
        if args.impl == "reference":
            run_reference_nufft4(args)
        else:
            run_nufft4(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
