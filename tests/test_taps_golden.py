"""Unequal per-axis tap counts (nufft.py:137): the oracle against fixtures the
reference produced (tests/golden/make_golden_taps.py)."""

import os

import numpy as np
import pytest

import cbn_oracle as orc
from conftest import GOLDEN, rel_l2


def cases():
    z = np.load(os.path.join(GOLDEN, "nufft_taps.npz"))
    out = {}
    for key in z.files:
        name, field = key.split("__")
        out.setdefault(name, {})[field] = z[key]
    return out


@pytest.mark.parametrize("name", sorted(cases()))
def test_oracle_unequal_taps(name):
    c = cases()[name]
    dims, j = tuple(int(v) for v in c["dims"]), tuple(int(v) for v in c["j"])
    ref = orc.make_plan(dims, c["nodes"], 2.0, j)
    first = np.stack([np.mod(f, k) for f, k in zip(ref.first, ref.kdims)], axis=1)
    assert np.array_equal(first, c["first"])
    assert rel_l2(orc.type2(ref, c["x"]), c["fwd"]) < 1e-12
    assert rel_l2(orc.type1(ref, c["y"]), c["adj"]) < 1e-12
