"""Unequal per-axis tap counts on the device (nufft.py:137 takes j per axis):
the kernels loop the largest count and the shorter axes' extra taps carry
zero weight; against fixtures the reference produced
(tests/golden/make_golden_taps.py)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, rel_l2

pytestmark = pytest.mark.gpu


def cases():
    z = np.load(os.path.join(GOLDEN, "nufft_taps.npz"))
    out = {}
    for key in z.files:
        name, field = key.split("__")
        out.setdefault(name, {})[field] = z[key]
    return out


@pytest.mark.parametrize("name", sorted(cases()))
def test_device_unequal_taps(name):
    from paper_1605_05231_b200 import nufft
    c = cases()[name]
    dims, j = tuple(int(v) for v in c["dims"]), tuple(int(v) for v in c["j"])
    plan = nufft.plan_nufft(dims, c["nodes"], 2.0, j)
    assert np.array_equal(plan.first_indices().astype(np.int64), c["first"].astype(np.int64))
    assert rel_l2(nufft.nufft_forward(plan, c["x"]), c["fwd"]) < 1e-5
    assert rel_l2(nufft.nufft_adjoint(plan, c["y"]), c["adj"]) < 1e-5


def test_projector_unequal_resample_taps():
    """ProjectorConfig.resample_j = (3, 5, 4) (per-axis resample taps,
    resampling.py:79-103): both operators against the reference's own
    forward projection and backprojection (tests/golden/make_golden_resj.py)."""
    from _cases import small_setup
    from paper_1605_05231_b200 import pipeline as pl
    from paper_1605_05231_b200.grangeat import DetectorFrame
    from paper_1605_05231_b200.phantom import Volume3D
    z = dict(np.load(os.path.join(GOLDEN, "pipeline_resj.npz")))
    n, views = int(z["n"]), int(z["views"])
    geom, voxel, spec, cfg = small_setup(n, views)
    cfg.resample_j = (3, 5, 4)
    frames = pl.nufft_forward_project(Volume3D(z["vol"], voxel), geom, cfg)
    err = rel_l2(np.stack([f.data for f in frames]), z["frames"])
    assert err < 1e-4, err
    fr = [DetectorFrame(k, z["frames"][k], geom.pixel_mm) for k in range(views)]
    err = rel_l2(pl.nufft_backproject(fr, geom, cfg, n, voxel).data, z["bp"])
    assert err < 1e-4, err
