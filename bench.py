#!/usr/bin/env python
"""Benchmark of the NUFFT cone-beam projector pair and the NUFFT (BASELINE.json).

Default run (``python bench.py``, N = 1): ONE JSON line whose headline is the
config-2 forward projector (``nufft_forward_project``: 256^3 30-ellipsoid
phantom -> 360 cone-beam views of 256^2, the reference's view batching and
per-batch resample scalings) in views/s, with two sub-objects carrying the
rest of BASELINE's metric ("views/s and Msamples/s, fwd+adj"):
  * "adjoint": the config-2 backprojector (``nufft_backproject``), views/s;
  * "nufft4":  config 4, type-2 + type-1 of 100M unstructured points, Msamples/s
               (with and without the per-step bin sort).
Each carries ``roofline``, ``e2e`` (through the drop-in API with host numpy
buffers) and ``cpu_baseline`` (the oracle port on this host's cores).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config 2|3|4] [--direction forward|back] [--only]

``--only`` measures just the selected config/direction.  Under torchrun
(N > 1) views and radial nodes are sharded across ranks (strong scaling);
timings are the max over ranks.  ``--impl reference`` times the CPU oracle
port (oracle/cbn_oracle.py) on bounded, extrapolated samples.
"""

from __future__ import annotations

import argparse
import ctypes
import gc
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
FALLBACK_HBM_GBS = 6650.0       # B200_PROFILING.md fallback when no measured peak exists
SMEM_TBS = 148 * 128 * 1.965e9 / 1e12   # nominal shared-memory bandwidth
# dram__bytes_read.sum + dram__bytes_write.sum per config-2 step of the
# dominant kernels, from the committed ncu captures (profiles/)
TRAFFIC = {"forward": {"resample_gather": 1.736e9, "spectrum_gather": 1.470e9,
                       "grangeat_spread": 3.284e9, "grangeat_rows": 1.865e9},
           "back": {"bp_spread": 1.512e9, "transpose_spread": 0.828e9,
                    "grangeat_forward": 0.718e9}}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--direction", choices=["forward", "back"], default="forward")
    ap.add_argument("--only", action="store_true", help="skip the sub-object measurements")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--comm", choices=["capi", "torch"], default="capi",
                    help="multi-GPU collectives: NCCL behind the C ABI (libcbnufft_b200_comm) "
                         "or torch.distributed around the projector phases")
    return ap.parse_args()


def hbm_peak():
    try:
        with open(PEAKS_FILE) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))

    def init(self):
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(self.local)
        if self.world > 1 and not dist.is_initialized():
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max(self, vals):
        import torch
        t = torch.tensor(list(vals), dtype=torch.float64, device="cuda")
        if self.world > 1:
            import torch.distributed as dist
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(v) for v in t.tolist()]


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
        return self

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


def timed(fn, steps, d: Dist, stream):
    """K steps between a barrier + synchronize on both sides, CUDA events on
    the launching stream; returns the max-over-ranks milliseconds."""
    import torch
    # a full cyclic-GC pass over torch's object graph takes tens of ms; when
    # one landed inside the 20 timed calls of the drop-in API (which creates
    # 360 frame objects per call) it moved the average by 3-4 ms.  Collect now
    # and freeze the survivors so that no such pass runs inside the timed loop.
    gc.collect()
    gc.freeze()
    torch.cuda.synchronize()
    d.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    d.barrier()
    return d.max([e0.elapsed_time(e1)])[0]


def _discard_stage_times(lib, handle):
    cnt = ctypes.c_int32(64)
    ms = (ctypes.c_double * 64)()
    names = ctypes.create_string_buffer(4096)
    lib.cbn_projector_stage_times(handle, ms, ctypes.byref(cnt), names, 4096, 1)
    cnt = ctypes.c_int32(64)
    hb = (ctypes.c_double * 64)()
    cb = (ctypes.c_double * 64)()
    lib.cbn_projector_stage_bytes(handle, hb, cb, ctypes.byref(cnt), names, 4096, 1)


def roofline_from_stages(lib, handle, steps, peak, peak_kind, traffic):
    """Per-stage rooflines from the projector's stage events and its own
    algorithmic-byte accounting (cbn_projector_stage_bytes)."""
    cnt = ctypes.c_int32(64)
    ms = (ctypes.c_double * 64)()
    names = ctypes.create_string_buffer(4096)
    lib.cbn_projector_stage_times(handle, ms, ctypes.byref(cnt), names, 4096, 1)
    stages = {nm: ms[i] / steps for i, nm in enumerate(names.value.decode().split(";")[:cnt.value])}
    cnt = ctypes.c_int32(64)
    hb = (ctypes.c_double * 64)()
    cb = (ctypes.c_double * 64)()
    names = ctypes.create_string_buffer(4096)
    lib.cbn_projector_stage_bytes(handle, hb, cb, ctypes.byref(cnt), names, 4096, 1)
    kernels = {}
    for i, nm in enumerate(names.value.decode().split(";")[:cnt.value]):
        t = stages.get(nm, 0.0)
        if t <= 0:
            continue
        hbm, chip = hb[i] / steps, cb[i] / steps
        ach = hbm / (t / 1e3) / 1e9
        kernels[nm] = {"ms_per_step": round(t, 3), "hbm_bytes": hbm, "achieved_gbs": round(ach, 1),
                       "hbm_frac": round(ach / peak, 4), "onchip_bytes": chip,
                       "onchip_tbs": round(chip / (t / 1e3) / 1e12, 2),
                       "onchip_frac": round(chip / (t / 1e3) / 1e12 / SMEM_TBS, 3)}
    roofline = None
    if kernels:
        st = max(kernels, key=lambda k: kernels[k]["ms_per_step"])
        kk = kernels[st]
        tr = traffic.get(st)
        roofline = {"kernel": st, "bound": "hbm", "achieved": kk["achieved_gbs"], "peak": peak,
                    "unit": "GB/s", "frac": kk["hbm_frac"],
                    "traffic": tr, "peak_kind": peak_kind,
                    "algorithmic_bytes_per_step": kk["hbm_bytes"],
                    "note": "achieved = the stage's algorithmic (compulsory) HBM bytes per step / its "
                            "CUDA-event time in a serialised pass; traffic = ncu DRAM bytes per step "
                            "(profiles/); onchip_* = shared-memory/L1 tap bytes (the binding "
                            "resource of the J >= 3 gathers/spreads)",
                    "onchip_tbs": kk["onchip_tbs"], "onchip_frac": kk["onchip_frac"]}
    return stages, kernels, roofline


# ------------------------------------------------------ projector (configs 0-3)
def measure_projector(args, d: Dist, config: int, direction: str):
    import torch
    from paper_1605_05231_b200 import _lib
    from paper_1605_05231_b200 import pipeline as pl
    from paper_1605_05231_b200 import sharding
    from paper_1605_05231_b200.grangeat import DetectorFrame
    from paper_1605_05231_b200.phantom import Volume3D
    from paper_1605_05231_b200.workloads import workload

    w = workload(config)
    V = w.geom.n_views
    per_view = w.cfg.n_mu * w.cfg.n_t
    lo, hi = sharding.view_shard(V, d.world, d.rank,
                                 sharding.view_batches(V, per_view, pl._TARGET_BATCH))
    fwd = direction == "forward"
    vol_host = w.volume()
    lib = _lib.load()
    stream = torch.cuda.current_stream()
    proj = pl.Projector(w.geom, w.cfg, w.n, w.voxel, 1 if fwd else 2)
    cm = None
    if d.world > 1 and args.comm == "capi":
        # the C-ABI communicator has never met a multi-GPU node (this pool has
        # one GPU per box): if any rank cannot create it, every rank takes the
        # torch.distributed data plane instead of losing the run
        import torch.distributed as dist
        try:
            from paper_1605_05231_b200.comm import NcclComm
            cm = NcclComm.from_group()
        except Exception as e:   # noqa: BLE001
            print(f"[bench] rank {d.rank}: libcbnufft_b200_comm unavailable ({e}); "
                  "falling back to torch.distributed", file=sys.stderr)
            cm = None
        ok = torch.tensor([1 if cm is not None else 0], device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            cm = None
    if fwd:
        x_dev = torch.from_numpy(vol_host).cuda()
        if cm is not None:
            def step():
                return cm.forward_project(proj, x_dev, lo, hi)
        elif d.world > 1:
            def step():
                return proj.forward_sharded(x_dev, lo, hi)
        else:
            def step():
                return proj.forward(x_dev, lo, hi)
    else:
        fp = pl.Projector(w.geom, w.cfg, w.n, w.voxel, 1)
        x_dev = fp.forward(torch.from_numpy(vol_host).cuda())
        del fp
        gc.collect()
        x_loc = x_dev[lo:hi].contiguous()
        if cm is not None:
            def step():
                return cm.backproject(proj, x_loc, lo, hi)
        elif d.world > 1:
            def step():
                return proj.backproject_sharded(x_loc, lo, hi)
        else:
            def step():
                return proj.backproject(x_dev)

    t_plan = time.perf_counter()
    step()                                   # builds the plan (not timed)
    torch.cuda.synchronize()
    plan_s = time.perf_counter() - t_plan
    for _ in range(max(args.warmup, 3)):
        step()
    clocks = ClockSampler(d.local).start()
    n0 = lib.cbn_launch_count()
    ms = timed(step, args.steps, d, stream)
    launches = lib.cbn_launch_count() - n0
    clk = clocks.stop()
    value = V * args.steps / (ms / 1e3)

    # serialised pass with stage events + algorithmic bytes (per-kernel rooflines)
    lib.cbn_projector_set_timing(proj._h, 1)
    # one untimed step in the serialised mode first: it runs every view block
    # on one stream, whose cuFFT plans and buffers the overlapped steps never
    # built (their one-time creation is not a stage time)
    step()
    torch.cuda.synchronize()
    _discard_stage_times(lib, proj._h)
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    peak, peak_kind = hbm_peak()
    stages, kernels, roofline = roofline_from_stages(lib, proj._h, args.steps, peak, peak_kind,
                                                     TRAFFIC[direction])
    lib.cbn_projector_set_timing(proj._h, 0)
    stats = proj.plan_stats()

    e2e = e2e_proj = None
    if not args.no_e2e:
        if d.world == 1:
            # the drop-in API itself: host float64 numpy in, float64 results out
            # (nufft_forward_project -> list[DetectorFrame]; nufft_backproject -> Volume3D)
            if fwd:
                vol_api = Volume3D(vol_host, w.voxel)

                def api():
                    return pl.nufft_forward_project(vol_api, w.geom, w.cfg)
                h2d, d2h = vol_host.size * 4, V * w.geom.nu * w.geom.nv * 4
            else:
                fr = x_dev.cpu().numpy().astype(np.float64)
                frames_api = [DetectorFrame(k, fr[k], w.geom.pixel_mm) for k in range(V)]

                def api():
                    return pl.nufft_backproject(frames_api, w.geom, w.cfg, w.n, w.voxel)
                h2d, d2h = V * w.geom.nu * w.geom.nv * 4, w.n ** 3 * 4
            api()
            api()
            calls = []

            def api_timed():
                t0 = time.perf_counter()
                api()
                calls.append(1e3 * (time.perf_counter() - t0))
            w0 = time.perf_counter()
            e_ms = timed(api_timed, args.steps, d, stream)
            wall = time.perf_counter() - w0
            calls.sort()
            e2e = {"value": round(V * args.steps / (e_ms / 1e3), 3), "unit": "views/s",
                   "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                   "ms_per_step": round(e_ms / args.steps, 3), "wall_s": round(wall, 3),
                   # host wall clock of the individual calls (the value above is
                   # the mean over all of them; the host side varies from box to box)
                   "call_ms": {"min": round(calls[0], 3), "median": round(calls[len(calls) // 2], 3),
                               "max": round(calls[-1], 3)},
                   "api": ("pipeline.nufft_forward_project(Volume3D float64) -> list[DetectorFrame] "
                           "float64" if fwd else
                           "pipeline.nufft_backproject(list[DetectorFrame] float64) -> Volume3D "
                           "float64") + "; host conversions on threads via pinned staging"}
        e2e_proj = e2e_projector(proj, fwd, vol_host, x_dev, w, lo, hi, args, d, stream, cm)
    cpu = None
    if d.world == 1 and not args.no_cpu_baseline:
        cpu = _cpu_later(args, (lambda: cpu_forward(w)) if fwd else (lambda: cpu_backward(w)))
    del proj
    gc.collect()
    torch.cuda.empty_cache()
    return {
        "metric": "cone-beam views/s (NUFFT " + ("forward projector)" if fwd else "backprojector)"),
        "value": round(value, 3), "unit": "views/s", "n_gpus": d.world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": round(ms / args.steps, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "c64/f32 (fp64 index math)",
        "data": f"synthetic: seeded random-ellipsoid phantom (BASELINE {w.name})",
        "config": {"workload": f"{w.name} {direction}: {w.n}^3 volume, "
                               f"{w.spec.n_rho}x{w.spec.n_theta}x{w.spec.n_phi} radial lattice, "
                               f"{V} views of {w.geom.nu}^2, KB J=6 sigma=2, resample J=3",
                   "views": V, "views_per_rank": hi - lo,
                   "parallelism": f"views sharded x{d.world}" + (
                       "" if d.world == 1 else ", radial nodes sharded, NCCL collectives ("
                       + ("C ABI, libcbnufft_b200_comm" if cm is not None else "torch.distributed")
                       + ")"),
                   "l2": "inputs in HBM; working set > L2 every step (resample grid "
                         f"{stats.get('fwd_resample_cells', stats.get('bp_resample_cells', 0)) * 4 / 1e9:.1f}"
                         " GB), no flush needed",
                   "plan_s": round(plan_s, 3)},
        "e2e": e2e, "e2e_projector": e2e_proj,
        "gpu_launches": int(launches), "gpu_launches_per_step": int(launches) // max(args.steps, 1),
        "clocks": clk, "roofline": roofline, "kernels": kernels,
        "stages_ms_per_step": {k: round(v, 3) for k, v in stages.items()},
        "plan_stats": stats, "cpu_baseline": cpu,
    }


def e2e_projector(proj, fwd, vol_host, x_dev, w, lo, hi, args, d: Dist, stream, cm=None):
    """Projector API with pinned host tensors, copies on a second stream
    overlapping the previous/next step (a serving loop)."""
    import torch
    if fwd:
        host_in = torch.from_numpy(vol_host).pin_memory()
        host_out = torch.empty((hi - lo, w.geom.nu, w.geom.nv), dtype=torch.float32).pin_memory()
    else:
        host_in = x_dev.cpu().pin_memory()
        host_out = torch.empty((w.n,) * 3, dtype=torch.float32).pin_memory()

    def run(dev):
        if cm is not None:
            return (cm.forward_project(proj, dev, lo, hi) if fwd
                    else cm.backproject(proj, dev[lo:hi].contiguous(), lo, hi))
        if fwd:
            return proj.forward_sharded(dev, lo, hi) if d.world > 1 else proj.forward(dev, lo, hi)
        if d.world > 1:
            return proj.backproject_sharded(dev[lo:hi].contiguous(), lo, hi)
        return proj.backproject(dev)

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
            if k + 1 < nsteps:
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
    d.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    pipeline(args.steps, e0)
    e1.record(copy_s)
    torch.cuda.synchronize()
    d.barrier()
    e_ms = d.max([e0.elapsed_time(e1)])[0]
    return {"value": round(w.geom.n_views * args.steps / (e_ms / 1e3), 3), "unit": "views/s",
            "h2d_bytes_per_step": int(host_in.numel() * 4),
            "d2h_bytes_per_step": int(host_out.numel() * 4),
            "api": "Projector.forward/backproject on pinned float32 tensors, H2D/D2H on a copy "
                   "stream overlapping the neighbouring steps"}


# ------------------------------------------- config 4: NUFFT stress microbench
C4_POINTS = 100_000_000
C4_GRID = 256
C4_J = 8


def measure_nufft4(args, d: Dist):
    """BASELINE config 4: type-2 gather + type-1 spread of 100M float32 points
    (i.i.d. uniform in [-pi, pi)^3) against a 256^3 CN(0,1) grid, KB J=8,
    sigma 2.  One step = one type-2 and one type-1 over every point.  The
    headline excludes the plan (bin sort + LS fit, once per node set, as the
    reference's plan_nufft is); ``value_with_sort`` re-sorts the points every
    step ("sort + gather", "sort + spread").  Under torchrun the
    points are split evenly across ranks; type-1's 256^3 outputs are summed
    and scattered by z-slab with one NCCL reduce-scatter."""
    import torch
    import torch.distributed as dist
    from paper_1605_05231_b200 import _lib, nufft
    from paper_1605_05231_b200.workloads import config4_inputs

    m_total = int(os.environ.get("CBN_C4_POINTS", C4_POINTS))
    x_host, pts = config4_inputs(n_points=m_total, grid=C4_GRID)
    lo = m_total * d.rank // d.world
    hi = m_total * (d.rank + 1) // d.world
    pts = np.ascontiguousarray(pts[lo:hi])
    m = hi - lo
    lib = _lib.load()
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()
    tp = time.perf_counter()
    plan = nufft.plan_nufft((C4_GRID,) * 3, pts, 2.0, C4_J)
    torch.cuda.synchronize()
    plan_s = time.perf_counter() - tp
    sp = ctypes.c_void_p(stream.cuda_stream)
    x = torch.from_numpy(x_host).cuda()
    y = torch.empty(m, dtype=torch.complex64, device="cuda")
    xa = torch.empty((C4_GRID,) * 3, dtype=torch.complex64, device="cuda")
    slab = torch.empty((C4_GRID // d.world, C4_GRID, C4_GRID), dtype=torch.complex64,
                       device="cuda") if d.world > 1 else None

    def type2():
        _lib.check(lib.cbn_nufft_type2(plan.handle, ctypes.c_void_p(x.data_ptr()),
                                       ctypes.c_void_p(y.data_ptr()), sp))

    def type1():
        _lib.check(lib.cbn_nufft_type1(plan.handle, ctypes.c_void_p(y.data_ptr()),
                                       ctypes.c_void_p(xa.data_ptr()), sp))
        if d.world > 1:
            dist.reduce_scatter_tensor(torch.view_as_real(slab), torch.view_as_real(xa))

    def resort():
        _lib.check(lib.cbn_nufft_resort(plan.handle, sp))

    for _ in range(max(args.warmup, 3)):
        type2()
        type1()
    torch.cuda.synchronize()
    d.barrier()
    clocks = ClockSampler(d.local).start()
    n0 = lib.cbn_launch_count()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps + 1)]
    torch.cuda.synchronize()
    d.barrier()
    ev[0].record(stream)
    for k in range(args.steps):
        type2()
        ev[2 * k + 1].record(stream)
        type1()
        ev[2 * k + 2].record(stream)
    torch.cuda.synchronize()
    d.barrier()
    launches = lib.cbn_launch_count() - n0
    clk = clocks.stop()
    t2 = sum(ev[2 * k].elapsed_time(ev[2 * k + 1]) for k in range(args.steps)) / args.steps
    t1 = sum(ev[2 * k + 1].elapsed_time(ev[2 * k + 2]) for k in range(args.steps)) / args.steps
    ms = ev[0].elapsed_time(ev[-1])
    ms, t2, t1 = d.max([ms, t2, t1])
    value = m_total * args.steps / (ms / 1e3) / 1e6

    # the same steps with the device bin sort redone every step
    def step_sorted():
        resort()
        type2()
        type1()
    step_sorted()
    ms_sorted = timed(step_sorted, args.steps, d, stream)
    ts = timed(resort, args.steps, d, stream) / args.steps
    value_sorted = m_total * args.steps / (ms_sorted / 1e3) / 1e6

    e2e = None
    if not args.no_e2e and d.world == 1:
        # the drop-in API with host numpy buffers: nufft_forward(plan, x) ->
        # complex128 node values; nufft_adjoint(plan, y) -> complex128 grid
        x128 = x_host.astype(np.complex128)
        y128 = np.zeros(m, np.complex128)

        def api():
            nufft.nufft_forward(plan, x128)
            nufft.nufft_adjoint(plan, y128)
        api()
        e_ms = timed(api, max(2, args.steps // 4), d, stream)
        nst = max(2, args.steps // 4)
        e2e = {"value": round(m_total * nst / (e_ms / 1e3) / 1e6, 3), "unit": "Msamples/s",
               "h2d_bytes_per_step": int(x128.size * 16 + y128.size * 16),
               "d2h_bytes_per_step": int(m * 16 + x128.size * 16),
               "steps": nst,
               "api": "nufft.nufft_forward / nufft_adjoint with host complex128 numpy in and out "
                      "(the reference's types)"}
    peak, peak_kind = hbm_peak()
    K3 = (2 * C4_GRID) ** 3
    # compulsory bytes: the oversampled grid once (8 B/cell), 12 B float32
    # coordinates + 8 B value per point; the FFT/pad/crop passes not counted
    gbytes = 8.0 * K3 + 20.0 * m
    taps = C4_J ** 3
    # serialised pass with the plan's stage events: kernel times + bytes
    lib.cbn_nufft_set_timing(plan.handle, 1)
    for _ in range(args.steps):
        resort()
        type2()
        type1()
    torch.cuda.synchronize()
    st_t = stage_times_nufft(lib, plan, args.steps)
    lib.cbn_nufft_set_timing(plan.handle, 0)
    kernels = {
        "type2": {"ms_per_step": round(t2, 3), "hbm_bytes": gbytes,
                  "achieved_gbs": round(gbytes / t2 / 1e6, 1),
                  "onchip_bytes": 8.0 * taps * m, "onchip_tbs": round(8.0 * taps * m / t2 / 1e9, 2),
                  "msamples_s": round(m / t2 / 1e3, 2)},
        "type1": {"ms_per_step": round(t1, 3), "hbm_bytes": gbytes,
                  "achieved_gbs": round(gbytes / t1 / 1e6, 1),
                  "onchip_bytes": 16.0 * taps * m,
                  "onchip_tbs": round(16.0 * taps * m / t1 / 1e9, 2),
                  "msamples_s": round(m / t1 / 1e3, 2)},
        "sort": {"ms_per_step": round(ts, 3)},
    }
    kernels.update(st_t)
    dom = "gather" if st_t.get("gather", {}).get("ms_per_step", 0) >= \
        st_t.get("spread", {}).get("ms_per_step", 0) else "spread"
    roofline = None
    if dom in st_t:
        kk = st_t[dom]
        roofline = {"kernel": dom, "bound": "hbm", "achieved": kk["achieved_gbs"], "peak": peak,
                    "unit": "GB/s", "frac": kk["hbm_frac"],
                    # ncu dram bytes of the 100 M-point launch (profiles/r2z_c4_*): the
                    # excess over the algorithmic bytes is the caller-order value /
                    # result access (4.72e9 / 3.98e9 with bin-ordered points,
                    # profiles/r2y_c4_presort_traffic.txt)
                    "traffic": ({"spread": 17.38e9, "gather": 9.93e9}[dom]
                                if m == 100_000_000 else None),
                    "peak_kind": peak_kind, "algorithmic_bytes_per_step": kk["hbm_bytes"],
                    "onchip_tbs": kk["onchip_tbs"], "onchip_frac": kk["onchip_frac"]}
    cpu = None
    if d.world == 1 and not args.no_cpu_baseline:
        cpu = _cpu_later(args, cpu_nufft4)
    del plan
    gc.collect()
    torch.cuda.empty_cache()
    return {
        "metric": "NUFFT nonuniform Msamples/s (fwd+adj)",
        "value": round(value, 3), "value_with_sort": round(value_sorted, 3),
        "unit": "Msamples/s", "n_gpus": d.world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": round(ms / args.steps, 3),
        "ms_per_step_with_sort": round(ms_sorted / args.steps, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "c64/f32 (fp64 index math)",
        "data": "synthetic: 256^3 CN(0,1) grid (seed 4), float32 points U[-pi,pi)^3 (seed 5)",
        "config": {"workload": f"config4: {m_total} points, {C4_GRID}^3 grid, KB J={C4_J}, sigma 2, "
                               "one type-2 + one type-1 per step",
                   "points_per_rank": m, "parallelism": f"points sharded x{d.world}",
                   "plan_s": round(plan_s, 3),
                   "l2": "working set > L2 (1.07 GB oversampled grid, 1.2 GB coordinates)"},
        "e2e": e2e, "gpu_launches": int(launches),
        "gpu_launches_per_step": int(launches) // max(args.steps, 1),
        "clocks": clk, "roofline": roofline, "kernels": kernels,
        "stages_ms_per_step": {"type2": round(t2, 3), "type1": round(t1, 3), "sort": round(ts, 3)},
        "cpu_baseline": cpu,
    }


def stage_times_nufft(lib, plan, steps):
    """Sort / gather / spread kernel times per step from the plan's own stage
    events (cbn_nufft_stage_times), with their algorithmic bytes."""
    peak, _ = hbm_peak()
    cnt = ctypes.c_int32(16)
    ms = (ctypes.c_double * 16)()
    hb = (ctypes.c_double * 16)()
    cb = (ctypes.c_double * 16)()
    names = ctypes.create_string_buffer(1024)
    if lib.cbn_nufft_stage_times(plan.handle, ms, hb, cb, ctypes.byref(cnt), names, 1024) != 0:
        return {}
    out = {}
    for i, nm in enumerate(names.value.decode().split(";")[:cnt.value]):
        t, hbm, chip = ms[i] / steps, hb[i] / steps, cb[i] / steps
        if t <= 0:
            continue
        ach = hbm / (t / 1e3) / 1e9
        out[nm] = {"ms_per_step": round(t, 3), "hbm_bytes": hbm, "achieved_gbs": round(ach, 1),
                   "hbm_frac": round(ach / peak, 4), "onchip_bytes": chip,
                   "onchip_tbs": round(chip / (t / 1e3) / 1e12, 2),
                   "onchip_frac": round(chip / (t / 1e3) / 1e12 / SMEM_TBS, 3)}
    return out


# --------------------------------------------------------- CPU (oracle) legs
def _oracle():
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import cbn_oracle as orc
    orc.WORKERS = os.cpu_count() or 1
    return orc


SPEC_PIECE = 1 << 19     # nodes of one spectrum sub-plan timed per sample (of 2^21)


def cpu_forward_pieces(w, k: int, orc, state):
    """Piece k of the config's forward projector on the oracle port:
    even k: plan + gather of SPEC_PIECE nodes of one spectrum sub-plan
    (per-node cost); odd k: one view's umbrella targets, resample plan + apply
    and reverse Grangeat (per-view cost).  Fixed per-call costs -- the sub-plan
    pad + 512^3 FFT and the Grangeat plan -- are timed once in `state`."""
    spec, cfg, geom = w.spec, w.cfg, w.geom
    M = spec.n_rho * spec.n_theta * spec.n_phi
    if "nodes" not in state:
        state["nodes"] = orc.wrap(orc.radial_direction_nodes(spec, w.voxel))
        state["vol"] = w.volume(np.float64).astype(np.complex128)
        t = time.perf_counter()
        g = np.zeros((2 * w.n,) * 3, np.complex128)
        orc.sfft.fftn(g, overwrite_x=True, workers=orc.WORKERS)
        state["t_fft"] = time.perf_counter() - t
        t = time.perf_counter()
        state["gp"] = orc.make_grangeat(geom, cfg.n_mu, cfg.n_t, t_pitch_mm=cfg.t_pitch_mm,
                                        t_taper=cfg.t_taper)
        state["t_gp"] = time.perf_counter() - t
        rng = np.random.default_rng(0)
        state["lattice"] = (rng.standard_normal((spec.n_rho, spec.n_theta, spec.n_phi))
                            + 1j * rng.standard_normal((spec.n_rho, spec.n_theta, spec.n_phi)))
        state["node"], state["view"] = [], []
    t = time.perf_counter()
    if k % 2 == 0:
        chunk = (k // 2) % max(1, -(-M // orc.PLAN_CHUNK))
        lo = chunk * orc.PLAN_CHUNK
        hi = min(lo + SPEC_PIECE, M)
        plan = orc.make_plan((w.n,) * 3, state["nodes"][lo:hi], 2.0, 6)
        orc.type2(plan, state["vol"])
        # per-node part: plan + gather (the sub-plan's pad + FFT is the fixed t_fft)
        dt = max(time.perf_counter() - t - state["t_fft"], 1e-9)
        state["node"].append(dt / (hi - lo))
    else:
        # one reference view batch (one view at configs 2/3): per-batch resample
        # plan + apply, then reverse Grangeat of each of its views
        per_view = cfg.n_mu * cfg.n_t
        batches = orc.view_batches(geom.n_views, per_view)
        batch = batches[(k // 2 * 37) % len(batches)]
        targets, valid = orc.umbrella_targets(geom, spec, batch, cfg.n_mu, cfg.n_t, cfg.t_pitch_mm)
        rs = orc.make_resampler(spec, targets, cfg.rho_pad, cfg.resample_j)
        vals = np.real(orc.resample_forward(rs, state["lattice"]))
        vals[~valid] = 0.0
        for i in range(len(batch)):
            orc.grangeat_reverse(vals[i * per_view:(i + 1) * per_view].reshape(cfg.n_mu, cfg.n_t),
                                 state["gp"])
        state["view"].append((time.perf_counter() - t) / len(batch))
    return time.perf_counter() - t


def cpu_forward_value(w, orc, state):
    M = w.spec.n_rho * w.spec.n_theta * w.spec.n_phi
    n_chunks = -(-M // orc.PLAN_CHUNK)
    per_node = float(np.mean(state["node"])) if state["node"] else 0.0
    per_view = float(np.mean(state["view"])) if state["view"] else 0.0
    total = n_chunks * state["t_fft"] + M * per_node + state["t_gp"] + w.geom.n_views * per_view
    return w.geom.n_views / total, total, per_node, per_view, n_chunks


def cpu_forward(w, pieces: int = 2):
    orc = _oracle()
    state = {}
    t0 = time.perf_counter()
    for k in range(pieces):
        cpu_forward_pieces(w, k, orc, state)
    value, total, per_node, per_view, n_chunks = cpu_forward_value(w, orc, state)
    return {"value": round(value, 6), "unit": "views/s", "cores": os.cpu_count() or 1,
            "kind": "port",
            "sample": f"oracle port (reference algorithm, numpy/scipy): {n_chunks} spectrum "
                      f"sub-plans x (pad + {2 * w.n}^3 FFT {state['t_fft']:.2f}s) + "
                      f"{M_str(w)} nodes x {per_node * 1e6:.2f}us (plan + gather, sampled on "
                      f"{SPEC_PIECE} nodes) + Grangeat plan {state['t_gp']:.2f}s once + "
                      f"{w.geom.n_views} views x {per_view:.2f}s (targets, resample plan + apply, "
                      f"reverse Grangeat; sampled on {len(state['view'])} view batch(es)); extrapolated "
                      f"= {total:.0f}s per step; scipy.fft on all cores, numpy gather one core",
            "extrapolated": True, "sample_wall_s": round(time.perf_counter() - t0, 1)}


def M_str(w):
    return str(w.spec.n_rho * w.spec.n_theta * w.spec.n_phi)


def cpu_backward(w):
    """Oracle port of the config's backprojector on bounded samples: one view
    batch (forward Grangeat of its views, targets, resample plan, transposed
    resample of values and mask) and the plan + spread of SPEC_PIECE nodes of
    one 3D adjoint sub-plan, plus the per-sub-plan (2N)^3 inverse FFT;
    extrapolated to every batch and sub-plan."""
    from paper_1605_05231_b200.geometry import RadialGridSpec
    orc = _oracle()
    cfg, geom = w.cfg, w.geom
    t0 = time.perf_counter()
    n = w.n
    bspec = RadialGridSpec(2 * int(np.ceil(1.5 * n / 2.0)), w.spec.n_theta, w.spec.n_phi,
                           n * w.voxel * np.sqrt(3.0) / 2.0)
    n_t = 2 * geom.nu
    pad = min(bspec.n_rho // 8, 32)
    t = time.perf_counter()
    gp = orc.make_grangeat(geom, cfg.n_mu, n_t, t_pitch_mm=None)
    t_gp = time.perf_counter() - t
    batches = orc.view_batches(geom.n_views, cfg.n_mu * n_t)
    batch = batches[0]
    rng = np.random.default_rng(1)
    frames = rng.standard_normal((len(batch), geom.nu, geom.nv))
    t = time.perf_counter()
    vals = np.concatenate([orc.grangeat_forward(frames[i], gp).ravel() for i in range(len(batch))])
    targets, valid = orc.umbrella_targets(geom, bspec, batch, cfg.n_mu, n_t, gp.dt)
    rs = orc.make_resampler(bspec, targets, pad, cfg.resample_j, cfg.oversample_factor)
    orc.resample_adjoint(rs, np.where(valid, vals, 0.0).astype(np.complex128))
    orc.resample_adjoint(rs, valid.astype(np.complex128))
    t_batch = time.perf_counter() - t
    del rs
    M = bspec.n_rho * bspec.n_theta * bspec.n_phi
    nodes = orc.wrap(orc.radial_direction_nodes(bspec, w.voxel))[:SPEC_PIECE]
    y = np.ones(nodes.shape[0], np.complex128)
    t = time.perf_counter()
    g = np.zeros((2 * n,) * 3, np.complex128)
    orc.sfft.ifftn(g, overwrite_x=True, workers=orc.WORKERS)
    t_fft = time.perf_counter() - t
    t = time.perf_counter()
    plan = orc.make_plan((n,) * 3, nodes, 2.0, 6)
    orc.type1(plan, y)
    per_node = max(time.perf_counter() - t - t_fft, 1e-9) / nodes.shape[0]
    n_chunks = -(-M // orc.PLAN_CHUNK)
    total = t_gp + len(batches) * t_batch + n_chunks * t_fft + M * per_node
    return {"value": round(geom.n_views / total, 6), "unit": "views/s", "cores": os.cpu_count() or 1,
            "kind": "port",
            "sample": f"oracle port: Grangeat plan {t_gp:.2f}s once + {len(batches)} view batches x "
                      f"{t_batch:.2f}s (batch 0 of {len(batch)} views: forward Grangeat, targets, "
                      f"resample plan, transposed resample of values and mask) + {n_chunks} "
                      f"adjoint sub-plans x {2 * n}^3 IFFT {t_fft:.2f}s + {M} nodes x "
                      f"{per_node * 1e6:.2f}us (plan + spread, sampled on {SPEC_PIECE} nodes); "
                      f"extrapolated = {total:.0f}s per step",
            "extrapolated": True, "sample_wall_s": round(time.perf_counter() - t0, 1)}


def cpu_nufft4(n_sample: int = 1 << 17):
    """Oracle port on a 2^17-point sample of config 4 (plan excluded, like the
    GPU headline): per-point type-2 + type-1 cost plus one 512^3 FFT per
    transform, extrapolated to 100M points."""
    from paper_1605_05231_b200.workloads import config4_inputs
    orc = _oracle()
    t0 = time.perf_counter()
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
    g = np.zeros((2 * C4_GRID,) * 3, np.complex128)
    t = time.perf_counter()
    orc.sfft.fftn(g, overwrite_x=True, workers=orc.WORKERS)
    tf = time.perf_counter() - t
    per_point = max(t2 + t1 - 2 * tf, 1e-12) / n_sample
    total = per_point * C4_POINTS + 2 * tf
    return {"value": round(C4_POINTS / total / 1e6, 6), "unit": "Msamples/s",
            "cores": os.cpu_count() or 1, "kind": "port",
            "sample": f"oracle port: type-2 {t2:.2f}s + type-1 {t1:.2f}s on {n_sample} points "
                      f"(512^3 FFT {tf:.2f}s each), per-point part extrapolated to {C4_POINTS}",
            "extrapolated": True, "sample_wall_s": round(time.perf_counter() - t0, 1)}


# ------------------------------------------------------------ reference arm
def run_reference(args):
    """The reference algorithm on the host cores (oracle port; the reference
    package cannot travel to the GPU box).  Each of the K steps times one
    bounded piece of the config's forward projector (alternately a spectrum
    sub-plan sample and one view), and the views/s value extrapolates the
    measured per-node / per-view costs to the whole workload.  ms_per_step is
    the real time of a step (one piece); the extrapolated time of one full
    projection is extrapolated_ms_per_projection."""
    d = Dist()
    if d.rank != 0:
        return
    from paper_1605_05231_b200.workloads import workload
    if args.config == 4:
        t0 = time.perf_counter()
        vals = [cpu_nufft4() for _ in range(max(1, min(args.steps, 3)))]
        value = float(np.mean([v["value"] for v in vals]))
        cpu = dict(vals[-1])
        cpu["value"] = round(value, 6)
        wall = time.perf_counter() - t0
        print(json.dumps({
            "impl": "reference", "metric": "NUFFT nonuniform Msamples/s (fwd+adj)",
            "value": round(value, 6), "unit": "Msamples/s", "n_gpus": d.world,
            "steps": len(vals), "warmup": 0, "ms_per_step": round(1e3 * wall / len(vals), 1),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64/c128", "data": "synthetic: config 4 inputs",
            "config": {"workload": "config4 (CPU oracle port, extrapolated)"}, "cpu_baseline": cpu,
            "e2e": {"value": round(value, 6), "unit": "Msamples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}, "wall_s": round(wall, 1)}), flush=True)
        return
    w = workload(args.config)
    orc = _oracle()
    state = {}
    t0 = time.perf_counter()
    cpu_forward_pieces(w, 0, orc, state)      # warm-up piece (not counted)
    state["node"].clear()
    steps = max(2, args.steps)
    piece_s = [cpu_forward_pieces(w, k, orc, state) for k in range(steps)]
    value, total, per_node, per_view, n_chunks = cpu_forward_value(w, orc, state)
    wall = time.perf_counter() - t0
    cpu = {"value": round(value, 6), "unit": "views/s", "cores": os.cpu_count() or 1,
           "kind": "port",
           "sample": f"oracle port: {steps} pieces (spectrum sub-plan samples of {SPEC_PIECE} "
                     f"nodes and single views, alternating); per node {per_node * 1e6:.2f}us, "
                     f"per view {per_view:.2f}s, {n_chunks} x sub-plan FFT {state['t_fft']:.2f}s, "
                     f"Grangeat plan {state['t_gp']:.2f}s; extrapolated {total:.0f}s per projection",
           "extrapolated": True}
    out = {"impl": "reference",
           "metric": "cone-beam views/s (NUFFT forward projector)",
           "value": round(value, 6), "unit": "views/s", "n_gpus": d.world, "steps": steps,
           "warmup": 1, "ms_per_step": round(1e3 * float(np.mean(piece_s)), 1),
           "extrapolated_ms_per_projection": round(1e3 * total, 1),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
           "dtype": "f64/c128", "data": f"synthetic: seeded random-ellipsoid phantom (BASELINE {w.name})",
           "config": {"workload": f"{w.name} forward (CPU oracle port, bounded pieces, extrapolated)"},
           "cpu_baseline": cpu,
           "e2e": {"value": round(value, 6), "unit": "views/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0},
           "wall_s": round(wall, 1)}
    print(json.dumps(out), flush=True)


class _Deferred:
    """A CPU baseline to be timed after every GPU measurement of the run: a
    minute of all-core numpy work ahead of a drop-in e2e measurement slowed
    its host conversions (adjoint e2e 16.2 ms inside the combined run against
    14.5 ms alone)."""

    def __init__(self, thunk):
        self.thunk = thunk


def _cpu_later(args, thunk):
    if getattr(args, "defer_cpu", False):
        return _Deferred(thunk)
    return thunk()


def _resolve_deferred(obj):
    if isinstance(obj, dict):
        for k, v in list(obj.items()):
            if isinstance(v, _Deferred):
                obj[k] = v.thunk()
            else:
                _resolve_deferred(v)


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    d = Dist()
    d.init()
    args.defer_cpu = True
    if args.config == 4:
        out = measure_nufft4(args, d)
    else:
        out = measure_projector(args, d, args.config, args.direction)
        if not args.only and args.config == 2 and args.direction == "forward":
            out["adjoint"] = measure_projector(args, d, 2, "back")
            out["nufft4"] = measure_nufft4(args, d)
    _resolve_deferred(out)      # CPU baselines last (dict order: forward, adjoint, nufft4)
    if d.rank == 0:
        print(json.dumps(out), flush=True)
    if d.world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
