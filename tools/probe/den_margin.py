"""How close the backprojector's den entries come to the den_tol * max threshold
(pipeline.py:187-188), over several fresh plans."""
import sys, os, gc, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1605_05231_b200 import pipeline as pl, _lib
from paper_1605_05231_b200.workloads import workload
cfgi = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = workload(cfgi)
lib = _lib.load()
def buf(proj, name, dt):
    n = ctypes.c_int64()
    _lib.check(lib.cbn_projector_debug_buffer(proj._h, name.encode(), None, ctypes.byref(n), proj._s))
    out = np.empty(n.value, np.uint8)
    _lib.check(lib.cbn_projector_debug_buffer(proj._h, name.encode(), out.ctypes.data, ctypes.byref(n), proj._s))
    return out.view(dt).copy()
fr = torch.zeros((w.geom.n_views, w.geom.nu, w.geom.nv), dtype=torch.float32, device="cuda")
dens = []
for k in range(4):
    proj = pl.Projector(w.geom, w.cfg, w.n, w.voxel, pl._BACK)
    proj.backproject(fr)
    den = buf(proj, "den_cache", np.float32).astype(np.float64)
    dmax = buf(proj, "den_max", np.float64)[0]
    thr = w.cfg.den_tol * dmax
    r = np.abs(den / thr - 1.0)
    print(k, "M", den.size, "dmax", dmax, "kept", int((den > thr).sum()),
          "within 1e-3/1e-4/1e-5/1e-6:", [int((r < t).sum()) for t in (1e-3, 1e-4, 1e-5, 1e-6)],
          "closest", np.sort(r)[:4], flush=True)
    dens.append(den)
    del proj; gc.collect(); torch.cuda.empty_cache()
d = np.stack(dens)
spread = (d.max(0) - d.min(0)) / (w.cfg.den_tol * dmax)
print("plan-to-plan den spread at threshold scale: max", spread.max(), "median", np.median(spread))
