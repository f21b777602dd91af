"""Resample method B (truncated centred periodic sinc, resampling.py:126-196)
on the device against the reference's own outputs (tests/golden/pipeline_n12_b.npz,
made by tests/golden/make_golden.py methodb): the stage operators
(resample_apply / resample_transpose), the forward projector and the
backprojector, each to relative L2 <= 1e-4; plus the exact-adjoint dot test."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, rel_l2
from _cases import small_setup

pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.fixture(scope="module")
def gb():
    return dict(np.load(os.path.join(GOLDEN, "pipeline_n12_b.npz")))


def _setup(g):
    n, views = int(g["n"]), int(g["views"])
    geom, voxel, spec, cfg = small_setup(n, views)
    cfg.method = "b"
    return n, views, geom, voxel, spec, cfg


def test_resample_b_stage(gb):
    from paper_1605_05231_b200 import resampling as rs
    n, views, geom, voxel, spec, cfg = _setup(gb)
    plan = rs.plan_resample(spec, gb["rs_targets"], "b", rho_pad=cfg.rho_pad)
    assert rel_l2(rs.resample_apply(plan, gb["lattice"]), gb["rs_apply"]) < TOL
    assert rel_l2(rs.resample_transpose(plan, gb["rs_y"]), gb["rs_transpose"]) < TOL


def test_resample_b_adjoint_dot(gb):
    from paper_1605_05231_b200 import resampling as rs
    n, views, geom, voxel, spec, cfg = _setup(gb)
    plan = rs.plan_resample(spec, gb["rs_targets"], "b", rho_pad=cfg.rho_pad, side_lobes=3)
    rng = np.random.default_rng(3)
    shape = (spec.n_rho, spec.n_theta, spec.n_phi)
    x = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    x[spec.n_rho // 2] = x[spec.n_rho // 2].mean()     # origin-averaged (the operator's range)
    y = rng.standard_normal(plan.n_targets) + 1j * rng.standard_normal(plan.n_targets)
    lhs = np.vdot(y, rs.resample_apply(plan, x))
    rhs = np.vdot(rs.resample_transpose(plan, y), x)
    assert abs(lhs - rhs) / abs(lhs) < 1e-5


def test_forward_projector_method_b(gb):
    from paper_1605_05231_b200 import pipeline as pl
    from paper_1605_05231_b200.phantom import Volume3D
    n, views, geom, voxel, spec, cfg = _setup(gb)
    frames = pl.nufft_forward_project(Volume3D(gb["vol"], voxel), geom, cfg)
    got = np.stack([f.data for f in frames])
    assert rel_l2(got, gb["frames"]) < TOL
    # batch boundaries do not change method B (no per-batch plan state)
    assert rel_l2(got, gb["frames_b5"]) < TOL


def test_backprojector_method_b(gb):
    from paper_1605_05231_b200 import pipeline as pl
    from paper_1605_05231_b200.grangeat import DetectorFrame
    n, views, geom, voxel, spec, cfg = _setup(gb)
    fr = [DetectorFrame(k, gb["frames"][k], geom.pixel_mm) for k in range(views)]
    bp = pl.nufft_backproject(fr, geom, cfg, n, voxel).data
    assert rel_l2(bp, gb["bp"]) < TOL
    assert rel_l2(bp, gb["bp_b4"]) < TOL
