"""Isolate the reverse-Grangeat line-8 discrepancy at n=12."""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [REPO, os.path.join(REPO, "tests"), os.path.join(REPO, "oracle")]
import cbn_oracle as orc  # noqa: E402
from conftest import rel_l2  # noqa: E402
from _cases import small_setup  # noqa: E402
from paper_1605_05231_b200 import nufft, pipeline as pl  # noqa: E402

n = 12
geom, voxel, spec, cfg = small_setup(n, 8)
gp = orc.make_grangeat(geom, cfg.n_mu, cfg.n_t, t_pitch_mm=cfg.t_pitch_mm, t_taper=cfg.t_taper)
proj = pl.Projector(geom, cfg, n, voxel, 1)
v = np.zeros((cfg.n_mu, cfg.n_t))
v[8, 5] = 1.0
ref = orc.grangeat_reverse(v, gp)
dev = proj.grangeat_reverse(v[None].astype(np.float32)).cpu().numpy()[0]
print("device vs oracle", rel_l2(dev, ref), "scale", np.vdot(ref, dev) / np.vdot(ref, ref))
# oracle pre-processing, device generic type 1
ds = v / gp.w2[None, :]
s = orc.centred_fft(ds.astype(np.complex128), axis=1) * gp.dt
y = s * (-1j * np.sign(gp.omega) * gp.taper)[None, :] * (1.0 / (2.0 * gp.n_mu * gp.n_t * gp.dt))
yy = y.ravel() * np.conj(gp.cphase)
plan = nufft.plan_nufft((n, n), gp.plan.nodes, 2.0, 5)
h_dev = nufft.nufft_adjoint(plan, yy)
h_ref = orc.type1(gp.plan, yy)
print("generic type1 on line-8 data", rel_l2(h_dev, h_ref))
nz = np.nonzero(np.abs(yy) > 0)[0]
print("nonzero nodes", len(nz), "line", set((nz // cfg.n_t).tolist()))
line = gp.plan.nodes[8 * cfg.n_t:9 * cfg.n_t]
print("line-8 wrapped nodes at +-pi:", np.sum(np.isclose(np.abs(line), np.pi, atol=1e-12)))
cp_once = np.mod(line * 1.0, 2 * np.pi)
print("cphase (once-wrapped) vs plan nodes angle check:",
      np.max(np.abs(np.angle(gp.cphase[8 * cfg.n_t:9 * cfg.n_t]) -
                    np.angle(np.exp(1j * (line @ np.array([n / 2 - 0.5, n / 2 - 0.5])))))))
