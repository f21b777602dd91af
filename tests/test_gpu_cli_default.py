"""The reference CLI's default geometry (cli.py:29: SO 1100 mm, SD 1500 mm,
512 mm detector of 128^2, 360 mm object; 12 of its views here) with the
CLI's projector defaults (make_projector_config, spectrum J=3), N=16.

Two paths only run here:
  * invalid umbrella targets: planes with |rho| > rho_max are pinned to the
    origin and zeroed (pipeline.py:96-101,137,178) -- 316,416 of the
    forward's and 107,520 of the backprojector's targets;
  * reverse Grangeat's heavy cells: with nu = 128 the half-plane cells near the
    origin carry more than kGrHeavy CSR entries and get a CTA of their own
    (k_gr_gather_cells, item < 0).
Fixture: tests/golden/cli_default.npz (make_golden_r2.py cli).
"""

import dataclasses
import os

import numpy as np
import pytest

from conftest import GOLDEN, rel_l2

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module")
def case():
    from paper_1605_05231_b200.config import make_projector_config
    from paper_1605_05231_b200.geometry import ConeGeometry
    z = dict(np.load(os.path.join(GOLDEN, "cli_default.npz")))
    g = z["geom"]
    geom = ConeGeometry(float(g[0]), float(g[1]), float(g[2]), float(g[3]), int(g[4]), int(g[5]),
                        int(g[6]), float(g[7]))
    n = int(z["n"])
    cfg = make_projector_config(geom, n, "a")
    cfg.normalization = 1.0
    cfg.bp_normalization = 1.0
    return z, geom, n, float(z["voxel"]), cfg


def test_cli_geometry_forward_with_invalid_targets(case):
    from paper_1605_05231_b200 import pipeline as pl
    from paper_1605_05231_b200.phantom import Volume3D
    z, geom, n, voxel, cfg = case
    frames = pl.nufft_forward_project(Volume3D(z["vol"], voxel), geom, cfg)
    got = np.stack([f.data for f in frames])
    err = rel_l2(got, z["frames"])
    assert err < TOL, err
    proj = pl.get_projector(geom, cfg, n, voxel, pl._FORWARD)
    st = proj.plan_stats()
    assert st["fwd_umbrella_invalid_per_view"] * geom.n_views == int(z["invalid_fwd"]), st
    assert int(z["invalid_fwd"]) > 0
    # the heavy-cell branch of the reverse-Grangeat cell gather ran
    assert st["fwd_gr_heavy_cells"] > 0, st


def test_cli_geometry_backproject_with_invalid_targets(case):
    from paper_1605_05231_b200 import pipeline as pl
    from paper_1605_05231_b200.grangeat import DetectorFrame
    z, geom, n, voxel, cfg = case
    frames = [DetectorFrame(k, z["frames"][k].astype(np.float64), geom.pixel_mm)
              for k in range(geom.n_views)]
    vol = pl.nufft_backproject(frames, geom, cfg, n, voxel)
    err = rel_l2(vol.data, z["bp"])
    assert err < TOL, err
    proj = pl.get_projector(geom, cfg, n, voxel, pl._BACK)
    st = proj.plan_stats()
    assert st["bp_umbrella_invalid_per_view"] * geom.n_views == int(z["invalid_bp"]), st


def test_cli_geometry_reverse_grangeat_heavy_cells(case):
    """reverse_grangeat_view at nu = 128 on random umbrella values (two views)."""
    from paper_1605_05231_b200.pipeline import Projector
    z, geom, n, voxel, cfg = case
    proj = Projector(geom, cfg, n, voxel, 1)
    out = proj.grangeat_reverse(z["gr_values"]).cpu().numpy()
    err = rel_l2(out, z["gr_reverse"])
    assert err < TOL, err
    st = proj.plan_stats()
    assert st["fwd_gr_heavy_cells"] > 0 and st["fwd_gr_cell_items"] > 0, st
    # the strip form (k_gr_gather_strips, the default) ran, heavy strips included,
    # and the per-cell gather it replaced (CBN_GR_STRIPS=0) gives the same frames
    assert st["fwd_gr_heavy_strips"] > 0 and st["fwd_gr_strip_items"] > 0, st
    assert 0 < st["fwd_gr_strip_entries"] < st["fwd_gr_cell_entries"], st
    import os
    os.environ["CBN_GR_STRIPS"] = "0"
    try:
        cells = proj.grangeat_reverse(z["gr_values"]).cpu().numpy()
    finally:
        del os.environ["CBN_GR_STRIPS"]
    assert rel_l2(cells, out) < 1e-6
