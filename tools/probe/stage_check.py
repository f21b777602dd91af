"""Staged (cbn_backproject_stage_views) vs one-call backprojection at config 2."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1605_05231_b200 import pipeline as pl, _lib, _device
from paper_1605_05231_b200.workloads import workload
w = workload(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
V = w.geom.n_views
rng = np.random.default_rng(3)
fr = torch.from_numpy(rng.standard_normal((V, w.geom.nu, w.geom.nv)).astype(np.float32)).cuda()
proj = pl.get_projector(w.geom, w.cfg, w.n, w.voxel, pl._BACK)
one = proj.backproject(fr).cpu().numpy()
lib = _lib.load()
def rel(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))
for chunk in (V, 32, 64, 96):
    for a in range(0, V, chunk):
        b = min(V, a + chunk)
        rc = lib.cbn_backproject_stage_views(proj._h, _device.ptr(fr[a]), a, b, proj._s)
        assert rc == 0, (rc, lib.cbn_last_error())
    st = proj.backproject(fr).cpu().numpy()
    again = proj.backproject(fr).cpu().numpy()
    print("chunk", chunk, "staged vs one", rel(st, one), "unstaged again", rel(again, one))
