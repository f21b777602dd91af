"""Bit-exact first-tap indices on the node sets the projector itself plans
(north star: "an integer bin-sort of the nonuniform points, bit-exact to the
reference's indexing").

Reference: ``plan_nufft(...).interp.indices[:, 0]`` decoded per axis into
``first mod K`` (nufft.py:171-179), for every plan the reference builds at
config 0 / config 1 (tests/golden/bins_config0.npz, written by
make_golden_r2.py bins0):
  * the radial spectrum lattice, 1,048,576 nodes, J=6 (radon_fourier.py:89-108);
  * every umbrella view batch, J=3 -- 5 forward batches (4.42M targets) and 2
    backprojector batches (pipeline.py:130-137,174-182, resampling.py:79-103);
    J=3 is odd, so half-integer ties are not snapped by the reference;
  * the polar Grangeat nodes of both directions, J=5 (grangeat.py:93-128);
  * the backprojector's 3D adjoint node set, J=6 (pipeline.py:202-210).
The device values come from cbn_projector_first_indices, which evaluates the
same node sources and tap setup as the projector's gathers and spreads (for
umbrella batches on the views-in-lanes path: view 0's taps plus the whole-cell
phi shift).  The mismatch count is the assertion message.
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN, unpack_int
from _cases import config_setup

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref_bins():
    return np.load(os.path.join(GOLDEN, "bins_config0.npz"))


@pytest.fixture(scope="module")
def projector():
    from paper_1605_05231_b200.pipeline import Projector
    geom, voxel, spec, cfg = config_setup(0)
    return Projector(geom, cfg, 64, voxel, 3)


def mismatches(got, ref):
    got = np.asarray(got, dtype=np.int64)
    assert got.shape == ref.shape, (got.shape, ref.shape)
    bad = np.any(got != ref, axis=1)
    return int(bad.sum()), np.nonzero(bad)[0][:10]


@pytest.mark.parametrize("direction,key", [("forward", "radial"), ("back", "radial_bp"),
                                           ("forward", "polar_fwd"), ("back", "polar_bp")])
def test_bins_radial_and_polar(projector, ref_bins, direction, key):
    node_set = "radial" if key.startswith("radial") else "polar"
    ref = unpack_int(ref_bins, key)
    got = projector.first_indices(direction, node_set)
    n, where = mismatches(got, ref)
    assert n == 0, f"{key}: {n} of {ref.shape[0]} nodes differ, e.g. rows {where}"


@pytest.mark.parametrize("direction,tag,batches", [("forward", "fwd", 5), ("back", "bp", 2)])
def test_bins_umbrella_batches(projector, ref_bins, direction, tag, batches):
    total = 0
    for b in range(batches):
        ref = unpack_int(ref_bins, f"umb_{tag}_{b}")
        got = projector.first_indices(direction, "umbrella", b)
        n, where = mismatches(got, ref)
        total += ref.shape[0]
        assert n == 0, f"umbrella {tag} batch {b}: {n} of {ref.shape[0]} targets differ, rows {where}"
    assert total == (4_423_680 if tag == "fwd" else 90 * 128 * 128)


def test_bins_plan_stats(projector):
    st = projector.plan_stats()
    assert st["fwd_spectrum_nodes"] == 1_048_576
    assert st["fwd_umbrella_invalid_per_view"] == 0 and st["bp_umbrella_invalid_per_view"] == 0
