"""Host-side timeline of the drop-in forward call (config 2): where the
wall-clock of nufft_forward_project goes.  Diagnostic only."""
import time
import numpy as np
import torch
from paper_1605_05231_b200 import _lib, _device, _hostio
from paper_1605_05231_b200 import pipeline as pl
from paper_1605_05231_b200.grangeat import DetectorFrame
from paper_1605_05231_b200.phantom import Volume3D
from paper_1605_05231_b200.workloads import workload

w = workload(2)
vol = Volume3D(w.volume().astype(np.float64), w.voxel)
geom, cfg = w.geom, w.cfg
for _ in range(3):
    pl.nufft_forward_project(vol, geom, cfg)
lib = _lib.load()
T = time.perf_counter
for rep in range(6):
    stage = rep % 2 == 1          # odd reps: chunks staged as they are uploaded
    marks = []
    t0 = T()
    data = np.asarray(vol.data)
    proj = pl.get_projector(geom, cfg, data.shape[0], vol.voxel_mm, pl._FORWARD)
    s = proj._s
    marks.append(("plan lookup", T()))

    def on_chunk(dev, a, b):
        _lib.check(lib.cbn_forward_stage_volume(proj._h, _device.ptr(dev), a, b, s), "x")
    v = _hostio.upload(proj.stage, "vol", data, torch.float32, on_chunk=on_chunk if stage else None)
    marks.append(("upload enqueued", T()))
    out = torch.empty((geom.n_views, geom.nu, geom.nv), dtype=torch.float32, device="cuda")
    if stage:
        _lib.check(lib.cbn_forward_project_staged_async(proj._h, _device.ptr(out), 0, geom.n_views, s), "x")
    else:
        _lib.check(lib.cbn_forward_project_async(proj._h, _device.ptr(v), _device.ptr(out), 0, geom.n_views, s), "x")
    marks.append(("project enqueued (staged)" if stage else "project enqueued", T()))
    blocks = proj.blocks()
    waits = []
    def wait(k):
        _lib.check(lib.cbn_projector_block_sync(proj._h, k), "x")
        waits.append(T())
    frames = _hostio.download_blocks(proj.stage, "frames", out, blocks, wait)
    marks.append(("blocks downloaded+converted", T()))
    _lib.check(lib.cbn_forward_finish(proj._h, s), "x")
    marks.append(("finish", T()))
    res = [DetectorFrame._checked(k, frames[k], geom.pixel_mm) for k in range(geom.n_views)]
    marks.append(("frames wrapped", T()))
    print("rep", rep, " ".join(f"{n}={1e3 * (t - t0):.2f}" for n, t in marks))
    print("   block waits (ms):", " ".join(f"{1e3 * (t - t0):.2f}" for t in waits), "n_blocks", len(blocks))
    del res, frames
# pieces alone
data = np.asarray(vol.data)
pin = proj.stage.get("vol", data.shape, torch.float32)
hp = pin.numpy()
for _ in range(3):
    t0 = T(); _hostio.copy(hp, data); t1 = T()
    print(f"convert 256^3 f64->f32 pinned: {1e3 * (t1 - t0):.2f} ms")
dev = torch.empty(data.shape, dtype=torch.float32, device="cuda")
for _ in range(3):
    torch.cuda.synchronize(); t0 = T(); dev.copy_(pin, non_blocking=True); torch.cuda.synchronize(); t1 = T()
    print(f"H2D 67 MB: {1e3 * (t1 - t0):.2f} ms = {67.1 / (t1 - t0) / 1e3:.1f} GB/s")
o = torch.empty((360, 256, 256), dtype=torch.float32, device="cuda")
pf = proj.stage.get("frames", o.shape, o.dtype)
for _ in range(3):
    torch.cuda.synchronize(); t0 = T(); pf.copy_(o, non_blocking=True); torch.cuda.synchronize(); t1 = T()
    print(f"D2H 94 MB: {1e3 * (t1 - t0):.2f} ms = {94.4 / (t1 - t0) / 1e3:.1f} GB/s")
res = np.empty(o.shape, np.float64)
for _ in range(3):
    t0 = T(); _hostio._native_convert(res, pf.numpy()); t1 = T()
    print(f"convert frames f32->f64: {1e3 * (t1 - t0):.2f} ms")
import os
print("cpus", os.cpu_count(), "threads", _hostio._THREADS)
