"""Normalisation calibration against the reference's own
values (tests/golden/calibration_n16.npz, tests/golden/make_golden.py calib):
calibrate_normalization (pipeline.py:215-242), calibrate_bp_normalization
(pipeline.py:245-257) and the device ray-driven baseline projector it runs
(ct_project_linear, baseline.py:52-98)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, rel_l2
from _cases import small_setup

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gc():
    return dict(np.load(os.path.join(GOLDEN, "calibration_n16.npz")))


def test_ct_project_linear_matches_reference(gc):
    from paper_1605_05231_b200.baseline import ct_project_linear
    from paper_1605_05231_b200.phantom import Volume3D
    n, views = int(gc["n"]), int(gc["views"])
    geom, voxel, spec, cfg = small_setup(n, views)
    for vol, ref in ((gc["ball"], gc["ball_frames"]), (gc["vol"], gc["vol_frames"])):
        counter = {}
        frames = ct_project_linear(Volume3D(vol, voxel), geom, counter)
        assert [f.view_index for f in frames] == list(range(views))
        assert rel_l2(np.stack([f.data for f in frames]), ref) < 1e-5
        assert counter["mults"] == 8 * n * geom.nu * geom.nv * views


def test_calibrate_normalization(gc):
    from paper_1605_05231_b200 import pipeline as pl
    n, views = int(gc["n"]), int(gc["views"])
    geom, voxel, spec, cfg = small_setup(n, views)
    got = pl.calibrate_normalization(geom, n, cfg, voxel)
    assert cfg.normalization == got
    assert abs(got - float(gc["norm"])) / abs(float(gc["norm"])) < 1e-4


def test_calibrate_bp_normalization(gc):
    from paper_1605_05231_b200 import pipeline as pl
    n, views = int(gc["n"]), int(gc["views"])
    geom, voxel, spec, cfg = small_setup(n, views)
    got = pl.calibrate_bp_normalization(geom, n, cfg, voxel)
    assert cfg.bp_normalization == got
    assert abs(got - float(gc["bp_norm"])) / abs(float(gc["bp_norm"])) < 1e-4
