"""Host-side timeline of the drop-in backprojector call (config 2).  Diagnostic only."""
import time
import numpy as np
import torch
from paper_1605_05231_b200 import _lib, _device, _hostio
from paper_1605_05231_b200 import pipeline as pl
from paper_1605_05231_b200.grangeat import DetectorFrame
from paper_1605_05231_b200.phantom import Volume3D
from paper_1605_05231_b200.workloads import workload

w = workload(2)
geom, cfg = w.geom, w.cfg
V = geom.n_views
rng = np.random.default_rng(0)
fr = rng.standard_normal((V, geom.nu, geom.nv))
frames = [DetectorFrame(k, fr[k], geom.pixel_mm) for k in range(V)]
for _ in range(3):
    pl.nufft_backproject(frames, geom, cfg, w.n, w.voxel)
lib = _lib.load()
T = time.perf_counter
for rep in range(4):
    marks = []
    t0 = T()
    proj = pl.get_projector(geom, cfg, w.n, w.voxel, pl._BACK)
    shape = (V, geom.nu, geom.nv)
    pin = proj.stage.get("frames", shape, torch.float32)
    host = pin.numpy()
    dev = torch.empty(shape, dtype=torch.float32, device="cuda")
    s = proj._s
    bounds = list(range(0, V, pl._BP_STAGE_VIEWS)) + [V]
    marks.append(("setup", T()))
    conv = []
    for a, b in zip(bounds[:-1], bounds[1:]):
        c0 = T()
        _hostio.gather_frames(host[a:b], [frames[k].data for k in range(a, b)])
        conv.append(1e3 * (T() - c0))
        dev[a:b].copy_(pin[a:b], non_blocking=True)
        _lib.check(lib.cbn_backproject_stage_views(proj._h, _device.ptr(dev[a]), a, b, s), "x")
    marks.append(("frames converted+staged", T()))
    vol = proj.backproject(dev)
    marks.append(("backproject enqueued", T()))
    torch.cuda.synchronize()
    marks.append(("device done", T()))
    ok = bool(torch.isfinite(vol).all())
    marks.append(("finite check", T()))
    out = _hostio.download(proj.stage, "vol", vol)
    marks.append(("downloaded+converted", T()))
    res = Volume3D._checked(out, w.voxel)
    marks.append(("wrapped", T()))
    print("rep", rep, " ".join(f"{n}={1e3 * (t - t0):.2f}" for n, t in marks))
    print("   per-block conversions (ms):", " ".join(f"{c:.2f}" for c in conv))
    del res, out
