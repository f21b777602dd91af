"""Stage-by-stage device vs oracle comparison on one golden geometry (debug aid).

  python tools/dbg/stage_check.py pipeline_n12_v48
"""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [REPO, os.path.join(REPO, "tests"), os.path.join(REPO, "oracle")]
import cbn_oracle as orc  # noqa: E402
from conftest import GOLDEN, rel_l2  # noqa: E402
from _cases import small_setup  # noqa: E402
from paper_1605_05231_b200 import pipeline as pl  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "pipeline_n12_v48"
g = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
n, views = int(g["n"]), int(g["views"])
geom, voxel, spec, cfg = small_setup(n, views)
proj = pl.Projector(geom, cfg, n, voxel, 1)
lat_ref = orc.radial_lattice(g["vol"].astype(np.float64), voxel, spec, 6, 2.0, "trilinear")
lat = proj.radial_lattice(g["vol"]).cpu().numpy().transpose(2, 1, 0)
print("lattice", rel_l2(lat, lat_ref), "golden", rel_l2(lat, g["lattice"]))
per_view = cfg.n_mu * cfg.n_t
vals = proj.resample_views(np.ascontiguousarray(lat_ref.transpose(2, 1, 0)), 0, views).cpu().numpy()
targets, valid = orc.umbrella_targets(geom, spec, range(views), cfg.n_mu, cfg.n_t, cfg.t_pitch_mm)
rs = orc.make_resampler(spec, targets, cfg.rho_pad, cfg.resample_j)
ref_vals = np.where(valid, np.real(orc.resample_forward(rs, lat_ref)), 0.0).reshape(views, cfg.n_mu, cfg.n_t)
ev = [rel_l2(vals[k], ref_vals[k]) for k in range(views)]
print("resample all", rel_l2(vals, ref_vals), "worst view", max(ev), int(np.argmax(ev)))
gp = orc.make_grangeat(geom, cfg.n_mu, cfg.n_t, t_pitch_mm=cfg.t_pitch_mm, t_taper=cfg.t_taper)
fr = proj.grangeat_reverse(ref_vals.astype(np.float32)).cpu().numpy()
ref_fr = np.stack([orc.grangeat_reverse(ref_vals[k], gp) for k in range(views)])
ef = [rel_l2(fr[k], ref_fr[k]) for k in range(views)]
print("grangeat all", rel_l2(fr, ref_fr), "worst view", max(ef), int(np.argmax(ef)))
print("frames golden vs oracle-chain", rel_l2(ref_fr, g["frames"]))
# block-size dependence of the reverse Grangeat
for nb in (1, 4, 8, 16, 32):
    out = np.concatenate([proj.grangeat_reverse(ref_vals[k:k + nb].astype(np.float32)).cpu().numpy()
                          for k in range(0, views, nb)])
    print("grangeat block", nb, rel_l2(out, ref_fr))
