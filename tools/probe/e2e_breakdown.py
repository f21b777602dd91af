"""Host-side cost breakdown of the drop-in nufft_forward_project at config 2."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1605_05231_b200 import pipeline as pl, _hostio
from paper_1605_05231_b200.phantom import Volume3D
from paper_1605_05231_b200.workloads import workload
w = workload(2)
vol = Volume3D(w.volume(), w.voxel)
pl.nufft_forward_project(vol, w.geom, w.cfg)
proj = pl.get_projector(w.geom, w.cfg, w.n, w.voxel, pl._FORWARD)
def T(f, n=5):
    f(); torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(n): r = f()
    torch.cuda.synchronize(); return (time.perf_counter() - t) / n * 1e3, r
print("threads", _hostio._THREADS, "cpus", os.cpu_count())
t_up, v = T(lambda: _hostio.upload(proj.stage, "vol", vol.data, torch.float32))
t_fw, out = T(lambda: proj.forward(v))
t_dn, fr = T(lambda: _hostio.download(proj.stage, "frames", out))
t_obj, _ = T(lambda: [pl.DetectorFrame._checked(k, fr[k], w.geom.pixel_mm) for k in range(360)])
t_all, _ = T(lambda: pl.nufft_forward_project(vol, w.geom, w.cfg))
pin = proj.stage.get("frames", out.shape, torch.float32)
t_d2h, _ = T(lambda: pin.copy_(out, non_blocking=True))
t_alloc, _ = T(lambda: np.empty(out.shape, np.float64))
def conv():
    o = np.empty(out.shape, np.float64); _hostio.copy(o, pin.numpy()); return o
t_conv, _ = T(conv)
def conv1():
    return pin.numpy().astype(np.float64)
t_conv1, _ = T(conv1)
h = pin.numpy(); o = np.empty(out.shape, np.float64)
t_conv_warm, _ = T(lambda: _hostio.copy(o, h))
print(dict(upload=t_up, forward=t_fw, download=t_dn, frames=t_obj, total=t_all, d2h=t_d2h, alloc=t_alloc,
           conv_threads_fresh=t_conv, conv_numpy_fresh=t_conv1, conv_threads_warm=t_conv_warm))
# timeline of one async call
import ctypes
lib = pl._lib.load()
v = _hostio.upload(proj.stage, "vol", vol.data, torch.float32); torch.cuda.synchronize()
outd = torch.empty((360, 256, 256), dtype=torch.float32, device="cuda")
t0 = time.perf_counter()
pl._lib.check(lib.cbn_forward_project_async(proj._h, pl._device.ptr(v), pl._device.ptr(outd), 0, 360, proj._s))
t1 = time.perf_counter()
bl = proj.blocks()
ts = []
for k in range(len(bl)):
    lib.cbn_projector_block_sync(proj._h, k); ts.append(round((time.perf_counter() - t0) * 1e3, 2))
print("enqueue ms", round((t1 - t0) * 1e3, 2), "blocks", bl[:3], "done at", ts)
t0 = time.perf_counter(); pl.nufft_forward_project(vol, w.geom, w.cfg); print("api ms", (time.perf_counter() - t0) * 1e3)
