"""Small cases for compute-sanitizer (memcheck / racecheck): every gather /
spread kernel family of the projector pair and the NUFFT at n16 sizes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import numpy as np
import torch
from _cases import small_setup
from paper_1605_05231_b200 import nufft, pipeline as pl
from paper_1605_05231_b200.config import make_projector_config
from paper_1605_05231_b200.geometry import ConeGeometry
from paper_1605_05231_b200.grangeat import DetectorFrame
from paper_1605_05231_b200.phantom import Volume3D, random_ellipsoid_phantom

# views-in-lanes geometry (2 n_phi / V = 4): window gather, column gather, poles
for n, views in ((16, 8), (12, 24)):
    geom, voxel, spec, cfg = small_setup(n, views)
    vol = random_ellipsoid_phantom(n, 4, 1)
    fr = pl.nufft_forward_project(Volume3D(vol, voxel), geom, cfg)
    bp = pl.nufft_backproject(fr, geom, cfg, n, voxel)
    print("projector", n, views, float(np.abs(bp.data).max()))
# non-lane geometry with invalid targets + heavy reverse-Grangeat cells
geom = ConeGeometry(1100.0, 1500.0, 512.0, 512.0, 128, 128, 4, 360.0)
cfg = make_projector_config(geom, 8, "a")
fr = pl.nufft_forward_project(Volume3D(random_ellipsoid_phantom(8, 3, 2), 45.0), geom, cfg)
pl.nufft_backproject(fr, geom, cfg, 8, 45.0)
print("cli geometry ok")
rng = np.random.default_rng(0)
for dims, j, m in (((12, 10, 8), 6, 3000), ((12, 12, 12), 8, 3000), ((20, 16), 5, 2000)):
    nodes = rng.uniform(-np.pi, np.pi, (m, len(dims)))
    plan = nufft.plan_nufft(dims, nodes.astype(np.float32), 2.0, j)
    x = rng.standard_normal(dims) + 1j * rng.standard_normal(dims)
    y = nufft.nufft_forward(plan, x)
    nufft.nufft_adjoint(plan, y)
    print("nufft", dims, j, m)
torch.cuda.synchronize()
print("done")
