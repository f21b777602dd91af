"""Diagnostic: device radial lattice vs the oracle for the CLI default config."""
import os, sys
import numpy as np
REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [REPO, os.path.join(REPO, "oracle")]
import cbn_oracle as orc
from paper_1605_05231_b200 import io as cbio
from paper_1605_05231_b200.config import make_projector_config
from paper_1605_05231_b200.pipeline import Projector
g = cbio.load_geometry(os.path.join(REPO, "tests/golden/io/geom.json"))
vol = cbio.read_volume(os.path.join(REPO, "tests/golden/io/vol.raw"))
cfg = make_projector_config(g, vol.n, "a")
spec = cfg.radial_spec
ref = orc.radial_lattice(vol.data, vol.voxel_mm, spec, cfg.spectrum_j, 2.0, cfg.basis)   # (n_rho, n_theta, n_phi)
proj = Projector(g, cfg, vol.n, vol.voxel_mm, 1)
import torch
lat = proj.radial_lattice(torch.from_numpy(vol.data.astype(np.float32)).cuda()).cpu().numpy()  # (phi, theta, rho)
got = lat.transpose(2, 1, 0)
err = np.abs(got - ref)
print("rel", np.linalg.norm(err) / np.linalg.norm(ref))
per_rho = np.linalg.norm(err, axis=(1, 2)) / (np.linalg.norm(ref, axis=(1, 2)) + 1e-30)
print("per rho index:", np.round(per_rho, 4))
