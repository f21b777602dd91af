"""Grangeat polar nodes through the generic (non-binned) device NUFFT vs the oracle."""
import os, sys
import numpy as np
REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [REPO, os.path.join(REPO, "tests"), os.path.join(REPO, "oracle")]
import cbn_oracle as orc
from conftest import rel_l2
from _cases import small_setup
from paper_1605_05231_b200 import nufft
n = 12
geom, voxel, spec, cfg = small_setup(n, 8)
gp = orc.make_grangeat(geom, cfg.n_mu, cfg.n_t, t_pitch_mm=cfg.t_pitch_mm, t_taper=cfg.t_taper)
nodes = gp.plan.nodes
plan = nufft.plan_nufft((n, n), nodes, 2.0, 5)
first = plan.first_indices()
ref_first = np.stack([np.mod(f, k).astype(int) for f, k in zip(gp.plan.first, gp.plan.kdims)], -1)
print("first mismatches", int((first != ref_first).any(-1).sum()))
rng = np.random.default_rng(1)
y = rng.standard_normal(nodes.shape[0]) + 1j * rng.standard_normal(nodes.shape[0])
print("generic type1 err", rel_l2(nufft.nufft_adjoint(plan, y), orc.type1(gp.plan, y)))
line = slice(8 * cfg.n_t, 9 * cfg.n_t)
print("line 8 nodes (u, v grid coords):")
u = np.mod(nodes[line], 2 * np.pi) * 24 / (2 * np.pi)
print(np.round(u[::6], 6))
