"""Pin the CPU oracle (oracle/cbn_oracle.py) against golden vectors that the
reference itself produced (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

import cbn_oracle as orc
from conftest import rel_l2
from _cases import small_setup

CASES = ["r3_j6", "r3_j3_odd", "r2_j5", "r1_j6", "r3_j8", "r3_big",
         "edge_j6", "edge_j3", "edge_j5_2d"]


@pytest.mark.parametrize("name", CASES)
def test_oracle_nufft_matches_reference(nufft_cases, name):
    c = nufft_cases[name]
    dims = tuple(int(v) for v in c["dims"])
    plan = orc.make_plan(dims, c["nodes"], 2.0, tuple(int(v) for v in c["j"]))
    assert np.array_equal(plan.nodes, c["wrapped"])
    first = np.stack([np.mod(f, k).astype(np.int64) for f, k in zip(plan.first, plan.kdims)], -1)
    assert np.array_equal(first, c["first"])                        # bit-exact bins
    assert rel_l2(plan.scaling_grid().ravel(), c["scaling"]) < 1e-12
    assert rel_l2(orc.type2(plan, c["x"]), c["fwd"]) < 1e-12
    assert rel_l2(orc.type1(plan, c["y"]), c["adj"]) < 1e-12


@pytest.mark.parametrize("dims", [(32,), (16, 16), (8, 8, 8)])
def test_oracle_matches_nudft(dims):
    """The reference's own brute-force NUDFT bound (pkg/tests/test_nufft.py:25-53)."""
    rng = np.random.default_rng(7)
    nodes = rng.uniform(-np.pi, np.pi, (200, len(dims)))
    x = rng.standard_normal(dims) + 1j * rng.standard_normal(dims)
    got = orc.type2(orc.make_plan(dims, nodes, 2.0, 6), x)
    assert rel_l2(got, orc.nudft(dims, nodes, x)) < 1e-5


def test_oracle_pipeline_stages(golden_n16):
    g = golden_n16
    geom, voxel, spec, cfg = small_setup()
    vol = g["vol"].astype(np.float64)
    lat = orc.radial_lattice(vol, voxel, spec, 6, 2.0, "trilinear")
    assert rel_l2(lat, g["lattice"]) < 1e-12
    assert rel_l2(orc.radial_spectrum(vol, voxel, spec, 6), g["spectrum"]) < 1e-12
    dt = cfg.t_pitch_mm
    targets, valid = orc.umbrella_targets(geom, spec, range(0, 3), cfg.n_mu, cfg.n_t, dt)
    assert np.array_equal(valid, g["rs_valid"])
    assert np.max(np.abs(targets - g["rs_targets"])) < 1e-12
    rs = orc.make_resampler(spec, targets, cfg.rho_pad, cfg.resample_j)
    assert rel_l2(orc.resample_forward(rs, g["lattice"]), g["rs_apply"]) < 1e-12
    assert rel_l2(orc.resample_adjoint(rs, g["rs_y"]), g["rs_transpose"]) < 1e-12
    gp = orc.make_grangeat(geom, cfg.n_mu, cfg.n_t, t_pitch_mm=dt, t_taper=cfg.t_taper)
    assert rel_l2(orc.grangeat_reverse(g["gr_values"], gp), g["gr_reverse"]) < 1e-12
    gpb = orc.make_grangeat(geom, cfg.n_mu, 2 * geom.nu)
    assert rel_l2(orc.grangeat_forward(g["frames"][1], gpb), g["gr_forward"]) < 1e-12


@pytest.mark.parametrize("which", ["n16", "n12"])
def test_oracle_end_to_end(which, golden_n16, golden_n12):
    g = golden_n16 if which == "n16" else golden_n12
    n, views = int(g["n"]), int(g["views"])
    geom, voxel, spec, cfg = small_setup(n, views, "trilinear" if which == "n16" else "dirac")
    frames = orc.forward_project(g["vol"], voxel, geom, cfg)
    assert rel_l2(frames, g["frames"]) < 1e-11
    bp = orc.backproject(g["frames"], geom, cfg, n, voxel)
    assert rel_l2(bp, g["bp"]) < 1e-11
    if which == "n16":
        fb5 = orc.forward_project(g["vol"], voxel, geom, cfg, target_batch=cfg.n_mu * cfg.n_t * 5)
        assert rel_l2(fb5, g["frames_b5"]) < 1e-11
        assert rel_l2(orc.backproject(g["frames"], geom, cfg, n, voxel, target_batch=4096),
                      g["bp_b4"]) < 1e-11


def test_oracle_method_b():
    """Resample method B (periodic sinc) stages and both projectors vs the reference."""
    import os
    from conftest import GOLDEN
    g = dict(np.load(os.path.join(GOLDEN, "pipeline_n12_b.npz")))
    n, views = int(g["n"]), int(g["views"])
    geom, voxel, spec, cfg = small_setup(n, views)
    cfg.method = "b"
    assert rel_l2(orc.resample_b_forward(spec, g["rs_targets"], g["lattice"], cfg.rho_pad),
                  g["rs_apply"]) < 1e-12
    assert rel_l2(orc.resample_b_adjoint(spec, g["rs_targets"], g["rs_y"], cfg.rho_pad),
                  g["rs_transpose"]) < 1e-12
    assert rel_l2(orc.forward_project(g["vol"], voxel, geom, cfg), g["frames"]) < 1e-11
    assert rel_l2(orc.backproject(g["frames"], geom, cfg, n, voxel), g["bp"]) < 1e-11


@pytest.mark.parametrize("name", ["pipeline_n16_v8", "pipeline_n12_v48", "pipeline_n12_v24"])
def test_oracle_rotation_aligned(name):
    import os
    from conftest import GOLDEN
    g = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    n, views = int(g["n"]), int(g["views"])
    geom, voxel, spec, cfg = small_setup(n, views)
    assert rel_l2(orc.forward_project(g["vol"], voxel, geom, cfg), g["frames"]) < 1e-11


def test_smooth_ball_phantom_matches_reference():
    """Host restatement of the calibration phantom (phantom.py:179-214)."""
    import os
    from conftest import GOLDEN
    from paper_1605_05231_b200.phantom import smooth_ball_line_integral, smooth_ball_volume
    g = dict(np.load(os.path.join(GOLDEN, "calibration_n16.npz")))
    n = int(g["n"])
    voxel = 2.0 / n
    assert np.array_equal(smooth_ball_volume(n, voxel, 0.28 * n * voxel).data, g["ball"])
    d = np.array([[1.0, 0.0, 0.0], [0.0, 0.6, 0.8]])
    p = np.array([[-3.0, 0.1, 0.0], [0.0, 0.0, 0.0]])
    got = smooth_ball_line_integral(p, d, radius=0.5)
    half = np.sqrt(np.maximum(0.25 - np.array([0.01, 0.0]), 0.0))
    assert np.allclose(got, 16.0 * half ** 5 / (15.0 * 0.5 ** 4), rtol=1e-14)
