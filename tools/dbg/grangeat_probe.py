"""Reverse-Grangeat impulse probe: device vs oracle for single umbrella samples."""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [REPO, os.path.join(REPO, "tests"), os.path.join(REPO, "oracle")]
import cbn_oracle as orc  # noqa: E402
from conftest import rel_l2  # noqa: E402
from _cases import small_setup  # noqa: E402
from paper_1605_05231_b200 import pipeline as pl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
geom, voxel, spec, cfg = small_setup(n, 8)
proj = pl.Projector(geom, cfg, n, voxel, 1)
gp = orc.make_grangeat(geom, cfg.n_mu, cfg.n_t, t_pitch_mm=cfg.t_pitch_mm, t_taper=cfg.t_taper)
rng = np.random.default_rng(0)
worst = []
for trial in range(40):
    v = np.zeros((cfg.n_mu, cfg.n_t))
    im, jt = rng.integers(cfg.n_mu), rng.integers(cfg.n_t)
    v[im, jt] = 1.0
    got = proj.grangeat_reverse(v[None].astype(np.float32)).cpu().numpy()[0]
    ref = orc.grangeat_reverse(v, gp)
    worst.append((rel_l2(got, ref), im, jt))
worst.sort(reverse=True)
print("n", n, "worst impulses (err, mu, t):", [(f"{e:.2e}", a, b) for e, a, b in worst[:6]])
v = rng.standard_normal((cfg.n_mu, cfg.n_t))
print("random input err", rel_l2(proj.grangeat_reverse(v[None].astype(np.float32)).cpu().numpy()[0],
                                orc.grangeat_reverse(v, gp)))
# every node as an impulse, 32 views per call
bad = []
M = cfg.n_mu * cfg.n_t
for k0 in range(0, M, 32):
    ks = list(range(k0, min(M, k0 + 32)))
    v = np.zeros((len(ks), cfg.n_mu, cfg.n_t))
    for i, k in enumerate(ks):
        v[i].flat[k] = 1.0
    got = proj.grangeat_reverse(v.astype(np.float32)).cpu().numpy()
    for i, k in enumerate(ks):
        e = rel_l2(got[i], orc.grangeat_reverse(v[i], gp))
        if e > 1e-5:
            bad.append((k // cfg.n_t, k % cfg.n_t, round(e, 3)))
print("bad nodes (mu, t, err):", len(bad), bad[:20])
