"""plan_grangeat with any tap shape / oversampling (grangeat.py:93-170): the
standalone device NUFFT over the polar nodes plus the elementwise kernels,
against fixtures the reference produced (tests/golden/make_golden_grangeat.py).
The projector's own (5, 5), sigma = 2 path is covered in test_gpu_api.py."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, rel_l2

pytestmark = pytest.mark.gpu
TOL = 1e-4


def cases():
    z = np.load(os.path.join(GOLDEN, "grangeat_general.npz"))
    out = {}
    for key in z.files:
        name, field = key.split("__")
        out.setdefault(name, {})[field] = z[key]
    return out


@pytest.mark.parametrize("name", sorted(cases()))
def test_general_grangeat_views(name):
    from paper_1605_05231_b200.geometry import ConeGeometry, umbrella_coordinates
    from paper_1605_05231_b200.grangeat import (DetectorFrame, UmbrellaView,
                                                forward_grangeat_view, plan_grangeat,
                                                reverse_grangeat_view)
    c = cases()[name]
    nu, n_mu, n_t, j0, j1, sig, hann = c["case"]
    nu, n_mu, n_t = int(nu), int(n_mu), int(n_t)
    geom = ConeGeometry(3.0, 6.0, 2.0, 2.0, nu, nu, 8, 2.0)
    gp = plan_grangeat(geom, n_mu, n_t, j=(int(j0), int(j1)), oversample_factor=float(sig),
                       t_taper="hann" if hann else "none")
    assert gp.nufft_plan is not None
    fwd = forward_grangeat_view(DetectorFrame(3, c["frame"], geom.pixel_mm), gp).values
    err = rel_l2(fwd, c["fwd"])
    assert err < TOL, err
    coords = umbrella_coordinates(geom, 3, n_mu, n_t, gp.dt)
    rev = reverse_grangeat_view(UmbrellaView(3, c["vals"], coords), gp).data
    err = rel_l2(rev, c["rev"])
    assert err < TOL, err
