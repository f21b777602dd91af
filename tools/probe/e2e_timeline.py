"""Timeline of one drop-in nufft_forward_project call at config 2 (host side)."""
import sys, time, os, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1605_05231_b200 import pipeline as pl, _hostio, _device
from paper_1605_05231_b200.phantom import Volume3D
from paper_1605_05231_b200.workloads import workload
w = workload(2)
vol = Volume3D(w.volume(), w.voxel)
for _ in range(3): pl.nufft_forward_project(vol, w.geom, w.cfg)
proj = pl.get_projector(w.geom, w.cfg, w.n, w.voxel, pl._FORWARD)
lib = pl._lib.load()
T = []
t0 = time.perf_counter()
def mark(s): T.append((s, round((time.perf_counter() - t0) * 1e3, 2)))
v = _hostio.upload(proj.stage, "vol", np.asarray(vol.data), torch.float32); mark("upload issued")
out = torch.empty((360, 256, 256), dtype=torch.float32, device="cuda")
pl._lib.check(lib.cbn_forward_project_async(proj._h, _device.ptr(v), _device.ptr(out), 0, 360, proj._s)); mark("enqueued")
bl = proj.blocks()
def wait(k):
    lib.cbn_projector_block_sync(proj._h, k); mark(f"blk{k}")
fr = _hostio.download_blocks(proj.stage, "frames", out, bl, wait); mark("download done")
pl._lib.check(lib.cbn_forward_finish(proj._h, proj._s)); mark("finish")
fl = [pl.DetectorFrame._checked(k, fr[k], w.geom.pixel_mm) for k in range(360)]; mark("frames")
print(T)
del fl, fr
for rep in range(3):
    t = time.perf_counter(); r = pl.nufft_forward_project(vol, w.geom, w.cfg); del r
    print("api", (time.perf_counter() - t) * 1e3)
