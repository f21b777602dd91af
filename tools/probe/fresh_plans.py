"""Backprojection through fresh plans, repeatedly: intermittent plan-state
corruption shows up as a plan whose result is off by much more than the
~5e-6 summation-order noise.  argv: config, repeats."""
import sys, os, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1605_05231_b200 import pipeline as pl
from paper_1605_05231_b200.workloads import workload
cfg_i = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
w = workload(cfg_i)
V = w.geom.n_views
rng = np.random.default_rng(3)
fr = torch.from_numpy(rng.standard_normal((V, w.geom.nu, w.geom.nv)).astype(np.float32)).cuda()
def rel(a, b): return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))
outs = []
for k in range(reps):
    proj = pl.Projector(w.geom, w.cfg, w.n, w.voxel, pl._BACK)
    a = proj.backproject(fr).cpu().numpy()
    b = proj.backproject(fr).cpu().numpy()
    outs.append(a)
    print(k, "vs first", rel(a, outs[0]), "repeat", rel(b, a), flush=True)
    del proj; gc.collect(); torch.cuda.synchronize(); torch.cuda.empty_cache()
med = np.median(np.stack(outs), axis=0)
print("vs median:", [round(rel(o, med), 8) for o in outs])
