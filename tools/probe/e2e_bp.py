"""Host-side timeline of the drop-in nufft_backproject at config 2."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1605_05231_b200 import pipeline as pl, _hostio
from paper_1605_05231_b200.phantom import Volume3D
from paper_1605_05231_b200.workloads import workload
w = workload(2)
vol = Volume3D(w.volume(), w.voxel)
frames = pl.nufft_forward_project(vol, w.geom, w.cfg)
for _ in range(2):
    r = pl.nufft_backproject(frames, w.geom, w.cfg, w.n, w.voxel); del r
proj = pl.get_projector(w.geom, w.cfg, w.n, w.voxel, pl._BACK)
shape = (w.geom.n_views, w.geom.nu, w.geom.nv)
pin = proj.stage.get("frames", shape, torch.float32)
host = pin.numpy()
def T(f, n=5):
    f(); torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(n): r = f()
    torch.cuda.synchronize(); return round((time.perf_counter() - t) / n * 1e3, 2), r
t_conv, _ = T(lambda: [_hostio.pool().submit(np.copyto, host[k], frames[k].data, casting="unsafe").result() for k in range(360)])
def conv_par():
    futs = [_hostio.pool().submit(np.copyto, host[k], frames[k].data, casting="unsafe") for k in range(360)]
    for f in futs: f.result()
t_convp, _ = T(conv_par)
dev = torch.empty(shape, dtype=torch.float32, device="cuda")
t_h2d, _ = T(lambda: dev.copy_(pin, non_blocking=True))
t_bp, v = T(lambda: proj.backproject(dev))
t_fin, _ = T(lambda: bool(torch.isfinite(v).all()))
t_dn, out = T(lambda: _hostio.download(proj.stage, "vol", v))
t_vol, _ = T(lambda: pl.Volume3D._checked(out, w.voxel))
t_all, _ = T(lambda: pl.nufft_backproject(frames, w.geom, w.cfg, w.n, w.voxel))
print(dict(conv_serial=t_conv, conv_parallel=t_convp, h2d=t_h2d, backproject=t_bp, isfinite=t_fin,
           download=t_dn, volume_obj=t_vol, total=t_all, threads=_hostio._THREADS, cpus=os.cpu_count()))
