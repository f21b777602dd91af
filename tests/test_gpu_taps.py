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
