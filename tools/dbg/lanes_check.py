import os, sys, numpy as np, torch, time
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from conftest import rel_l2, GOLDEN
from _cases import small_setup
from paper_1605_05231_b200 import pipeline as pl
from paper_1605_05231_b200.phantom import Volume3D
from paper_1605_05231_b200.workloads import workload
g = dict(np.load(os.path.join(GOLDEN, "pipeline_n12_v48.npz")))
geom, voxel, spec, cfg = small_setup(12, 48)
fr = np.stack([f.data for f in pl.nufft_forward_project(Volume3D(g["vol"], voxel), geom, cfg)])
err = [rel_l2(fr[k], g["frames"][k]) for k in range(48)]
print("lanes=%s total %.3e worst view %.3e at %d" % (os.environ.get("CBN_NO_VIEW_LANES"), rel_l2(fr, g["frames"]), max(err), int(np.argmax(err))))
w = workload(2)
proj = pl.Projector(w.geom, w.cfg, w.n, w.voxel, 1)
vol = torch.from_numpy(w.volume()).cuda()
for _ in range(3): proj.forward(vol)
torch.cuda.synchronize(); t = time.time()
for _ in range(5): proj.forward(vol)
torch.cuda.synchronize(); print("cfg2 forward ms/step", (time.time() - t) / 5 * 1e3)
