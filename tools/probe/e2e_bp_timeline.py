"""Host timeline of one drop-in nufft_backproject call at config 2 (staged upload)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1605_05231_b200 import pipeline as pl, _hostio, _device, _lib
from paper_1605_05231_b200.grangeat import DetectorFrame
from paper_1605_05231_b200.workloads import workload
w = workload(2)
V = w.geom.n_views
rng = np.random.default_rng(3)
fr = rng.standard_normal((V, w.geom.nu, w.geom.nv))
frames = [DetectorFrame(k, fr[k], w.geom.pixel_mm) for k in range(V)]
for _ in range(3):
    r = pl.nufft_backproject(frames, w.geom, w.cfg, w.n, w.voxel); del r
proj = pl.get_projector(w.geom, w.cfg, w.n, w.voxel, pl._BACK)
lib = _lib.load()
shape = (V, w.geom.nu, w.geom.nv)
pin = proj.stage.get("frames", shape, torch.float32); host = pin.numpy()
T = []; t0 = time.perf_counter()
def mark(s): T.append((s, round((time.perf_counter() - t0) * 1e3, 2)))
dev = torch.empty(shape, dtype=torch.float32, device="cuda")
s = proj._s
for a in range(0, V, 64):
    b = min(V, a + 64)
    futs = [_hostio.pool().submit(np.copyto, host[k], frames[k].data, casting="unsafe") for k in range(a, b)]
    for f in futs: f.result()
    mark(f"conv{a}")
    dev[a:b].copy_(pin[a:b], non_blocking=True)
    lib.cbn_backproject_stage_views(proj._h, _device.ptr(dev[a]), a, b, s)
    mark(f"stage{a}")
vol = proj.backproject(dev); mark("bp enqueued")
torch.cuda.synchronize(); mark("bp done")
ok = bool(torch.isfinite(vol).all()); mark("isfinite")
out = _hostio.download(proj.stage, "vol", vol); mark("download")
print(T)
for rep in range(3):
    t = time.perf_counter(); r = pl.nufft_backproject(frames, w.geom, w.cfg, w.n, w.voxel); del r
    print("api", round((time.perf_counter() - t) * 1e3, 2))
