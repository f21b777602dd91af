"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py            # all fixtures
    python tests/golden/make_golden.py small      # skip the config-0/1 runs

Outputs (committed, small): tests/golden/*.npz.  Nothing at test or bench
time reads /root/reference; everything it needs is in these files.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import cbnufft.nufft as rnufft                           # noqa: E402
import cbnufft.pipeline as rpipe                          # noqa: E402
from cbnufft.geometry import ConeGeometry, RadialGridSpec  # noqa: E402
from cbnufft.grangeat import (DetectorFrame, UmbrellaView, forward_grangeat_view,  # noqa: E402
                              plan_grangeat, reverse_grangeat_view)
from cbnufft.phantom import Volume3D                      # noqa: E402
from cbnufft.radon_fourier import image_to_radial_spectrum  # noqa: E402
from cbnufft.resampling import plan_resample, resample_apply, resample_transpose  # noqa: E402
from cbnufft.geometry import umbrella_coordinates        # noqa: E402

from paper_1605_05231_b200.phantom import random_ellipsoid_phantom  # noqa: E402


def crandn(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def first_mod_k(plan):
    """Decode interp.indices[:, 0] into per-axis (first mod K)."""
    flat = plan.interp.indices[:, 0].astype(np.int64)
    out = []
    for a in reversed(range(len(plan.k_dims))):
        out.append(flat % plan.k_dims[a])
        flat //= plan.k_dims[a]
    return np.stack(out[::-1], axis=-1)


def nufft_cases():
    cases = {}
    rng = np.random.default_rng(1234)

    def add(name, dims, nodes, j):
        x = crandn(rng, dims)
        y = crandn(rng, (nodes.shape[0],))
        plan = rnufft.plan_nufft(dims, nodes, 2.0, j)
        cases[name] = dict(dims=np.array(dims), j=np.array(np.broadcast_to(j, (len(dims),))),
                           nodes=nodes, x=x, y=y,
                           fwd=rnufft.nufft_forward(plan, x), adj=rnufft.nufft_adjoint(plan, y),
                           scaling=plan.scaling, first=first_mod_k(plan),
                           wrapped=plan.nodes)

    add("r3_j6", (8, 8, 8), rng.uniform(-np.pi, np.pi, (200, 3)), 6)
    add("r3_j3_odd", (7, 10, 9), rng.uniform(-np.pi, np.pi, (300, 3)), 3)
    add("r2_j5", (16, 12), rng.uniform(-np.pi, np.pi, (250, 2)), 5)
    add("r1_j6", (32,), rng.uniform(-np.pi, np.pi, (64, 1)), 6)
    add("r3_j8", (12, 12, 12), rng.uniform(-np.pi, np.pi, (400, 3)), 8)
    add("r3_big", (16, 16, 16), rng.uniform(-3 * np.pi, 3 * np.pi, (20000, 3)), 6)
    # edge cases: on-grid nodes, near-grid (snap), the +-pi seam, aliases
    k = 32
    on = 2 * np.pi * rng.integers(-40, 40, (64, 3)) / k
    near = on + rng.choice([-1, 1], on.shape) * 10.0 ** rng.uniform(-12, -10, on.shape)
    seam = np.array([[np.pi, -np.pi, 0.0], [-np.pi, np.pi, 3 * np.pi],
                     [np.nextafter(np.pi, 0), -np.nextafter(np.pi, 0), 1e-300],
                     [0.0, -0.0, 2 * np.pi]])
    half = 2 * np.pi * (rng.integers(-20, 20, (32, 3)) + 0.5) / k
    edge = np.concatenate([on, near, seam, half])
    add("edge_j6", (16, 16, 16), edge, 6)
    add("edge_j3", (16, 16, 16), edge, 3)
    add("edge_j5_2d", (16, 16), edge[:, :2], 5)
    return cases


def small_geometry(n=16, views=12):
    geom = ConeGeometry(3.0, 6.0, 2.0, 2.0, n, n, views, 2.0)
    voxel = 2.0 / n
    spec = RadialGridSpec(2 * n, n, 2 * n, 2 * n * voxel / 2.0)
    cfg = rpipe.make_projector_config(geom, n, "a", radial_spec=spec, spectrum_j=6,
                                      rho_pad=min(spec.n_rho // 8, 32))
    cfg.normalization = 1.0
    cfg.bp_normalization = 1.0
    return geom, voxel, spec, cfg


def frames_array(frames):
    return np.stack([f.data for f in frames])


def pipeline_small(n=16, views=12, seed=11, basis="trilinear", method="a"):
    geom, voxel, spec, cfg = small_geometry(n, views)
    cfg.basis = basis
    cfg.method = method
    vol32 = random_ellipsoid_phantom(n, 5, seed)
    vol = Volume3D(vol32, voxel)
    out = dict(vol=vol32, voxel=voxel, n=n, views=views,
               spec=np.array([spec.n_rho, spec.n_theta, spec.n_phi, spec.rho_max]))
    out["spectrum"] = image_to_radial_spectrum(vol, spec, j=6).data
    out["lattice"] = rpipe._radial_lattice(vol, cfg)
    frames = rpipe.nufft_forward_project(vol, geom, cfg)
    out["frames"] = frames_array(frames)
    # per-batch resample scalings exercised with several batches
    saved = rpipe._TARGET_BATCH
    try:
        rpipe._TARGET_BATCH = cfg.n_mu * cfg.n_t * 5
        out["frames_b5"] = frames_array(rpipe.nufft_forward_project(vol, geom, cfg))
        rpipe._TARGET_BATCH = 4096
        out["bp_b4"] = rpipe.nufft_backproject(frames, geom, cfg, n, voxel).data
    finally:
        rpipe._TARGET_BATCH = saved
    out["bp"] = rpipe.nufft_backproject(frames, geom, cfg, n, voxel).data
    # stage fixtures: resample of views 0..2, grangeat of view 1
    targets, valid = rpipe._umbrella_targets(geom, cfg, range(0, 3))
    rp = plan_resample(spec, targets, method, rho_pad=cfg.rho_pad, j=cfg.resample_j)
    out["rs_targets"] = targets
    out["rs_valid"] = valid
    out["rs_apply"] = resample_apply(rp, out["lattice"])
    rng = np.random.default_rng(5)
    yv = crandn(rng, (targets.shape[0],))
    out["rs_y"] = yv
    out["rs_transpose"] = resample_transpose(rp, yv)
    gp = plan_grangeat(geom, cfg.n_mu, cfg.n_t, t_pitch_mm=cfg.t_pitch_mm, t_taper=cfg.t_taper)
    vals = np.real(resample_apply(rp, out["lattice"]))[cfg.n_mu * cfg.n_t:2 * cfg.n_mu * cfg.n_t]
    vals = vals.reshape(cfg.n_mu, cfg.n_t)
    coords = umbrella_coordinates(geom, 1, cfg.n_mu, cfg.n_t, cfg.t_pitch_mm)
    out["gr_values"] = vals
    out["gr_reverse"] = reverse_grangeat_view(UmbrellaView(1, vals, coords), gp).data
    gpb = plan_grangeat(geom, cfg.n_mu, 2 * geom.nu)
    fr = DetectorFrame(1, out["frames"][1], geom.pixel_mm)
    out["gr_forward"] = forward_grangeat_view(fr, gpb).values
    return out


def calibration(n=16, views=12):
    """calibrate_normalization / calibrate_bp_normalization (pipeline.py:215-257)
    and the baseline ray-driven projector they rely on (baseline.py:52-98)."""
    from cbnufft.baseline import ct_project_linear
    from cbnufft.phantom import smooth_ball_volume
    geom, voxel, spec, cfg = small_geometry(n, views)
    out = dict(n=n, views=views)
    out["norm"] = rpipe.calibrate_normalization(geom, n, cfg, voxel)
    geom, voxel, spec, cfg = small_geometry(n, views)
    out["bp_norm"] = rpipe.calibrate_bp_normalization(geom, n, cfg, voxel)
    ball = smooth_ball_volume(n, voxel, 0.28 * n * voxel)
    out["ball"] = ball.data
    out["ball_frames"] = frames_array(ct_project_linear(ball, geom))
    vol32 = random_ellipsoid_phantom(n, 5, 41)
    out["vol"] = vol32
    out["vol_frames"] = frames_array(ct_project_linear(Volume3D(vol32, voxel), geom))
    return out


def io_and_cli(out_dir):
    """Files written by the reference's io.py, and its CLI project/backproject
    outputs on a small volume (cli.py:78-100)."""
    import cbnufft.io as rio
    from cbnufft.cli import main as rcli
    os.makedirs(out_dir, exist_ok=True)
    geom, voxel, spec, cfg = small_geometry(12, 8)
    vol = Volume3D(random_ellipsoid_phantom(12, 4, 51), voxel)
    rio.write_volume(os.path.join(out_dir, "vol.raw"), vol)
    rio.save_geometry(os.path.join(out_dir, "geom.json"), geom)
    for method in ("nufft-a", "nufft-b", "linear"):
        code = rcli(["project", "--method", method, "--volume", os.path.join(out_dir, "vol.raw"),
                     "--geometry", os.path.join(out_dir, "geom.json"),
                     "--out", os.path.join(out_dir, f"proj_{method}.raw")])
        assert code == 0
    for method in ("nufft-a", "nufft-b"):
        code = rcli(["backproject", "--method", method,
                     "--projections", os.path.join(out_dir, "proj_nufft-a.raw"), "--n", "12",
                     "--out", os.path.join(out_dir, f"bp_{method}.raw")])
        assert code == 0


def config0():
    geom = ConeGeometry(3.0, 6.0, 2.0, 2.0, 64, 64, 90, 2.0)
    n = 64
    voxel = 2.0 / n
    spec = RadialGridSpec(128, 64, 128, 128 * voxel / 2.0)
    cfg = rpipe.make_projector_config(geom, n, "a", radial_spec=spec, spectrum_j=6,
                                      rho_pad=min(spec.n_rho // 8, 32))
    cfg.normalization = 1.0
    cfg.bp_normalization = 1.0
    vol32 = random_ellipsoid_phantom(n, 10, 0)
    t0 = time.time()
    frames = rpipe.nufft_forward_project(Volume3D(vol32, voxel), geom, cfg)
    t1 = time.time()
    bp = rpipe.nufft_backproject(frames, geom, cfg, n, voxel)
    t2 = time.time()
    print(f"config0 forward {t1 - t0:.1f}s backproject {t2 - t1:.1f}s", flush=True)
    return dict(vol=vol32, frames=frames_array(frames).astype(np.float32),
                bp=bp.data.astype(np.float32), fwd_seconds=t1 - t0, bp_seconds=t2 - t1)


def main():
    which = sys.argv[1:] or ["small", "big"]
    if "small" in which:
        t = time.time()
        cases = nufft_cases()
        flat = {f"{k}__{f}": v for k, c in cases.items() for f, v in c.items()}
        np.savez_compressed(os.path.join(HERE, "nufft_cases.npz"), **flat)
        np.savez_compressed(os.path.join(HERE, "pipeline_n16.npz"), **pipeline_small())
        np.savez_compressed(os.path.join(HERE, "pipeline_n12_dirac.npz"),
                            **pipeline_small(12, 8, 3, "dirac"))
        print(f"small fixtures {time.time() - t:.1f}s", flush=True)
    if "small" in which or "rot" in which:
        # geometries where 2 n_phi / V is an integer (whole oversampled phi cells
        # per view): the device's views-in-lanes resample path
        np.savez_compressed(os.path.join(HERE, "pipeline_n16_v8.npz"),
                            **pipeline_small(16, 8, 21, "trilinear"))
        np.savez_compressed(os.path.join(HERE, "pipeline_n12_v48.npz"),
                            **pipeline_small(12, 48, 22, "trilinear"))
    if "small" in which or "rot2" in which:
        # 2 n_phi / V = 2 (as configs 2 and 3): the paired column gather of the
        # backprojector's transposed resample
        np.savez_compressed(os.path.join(HERE, "pipeline_n12_v24.npz"),
                            **pipeline_small(12, 24, 23, "trilinear"))
    if "small" in which or "methodb" in which:
        # resample method B (truncated periodic sinc, side_lobes 2): stage
        # fixtures (apply / transpose) and both projectors, one and several batches
        np.savez_compressed(os.path.join(HERE, "pipeline_n12_b.npz"),
                            **pipeline_small(12, 10, 31, "trilinear", "b"))
    if "small" in which or "calib" in which:
        np.savez_compressed(os.path.join(HERE, "calibration_n16.npz"), **calibration())
    if "small" in which or "io" in which:
        io_and_cli(os.path.join(HERE, "io"))
    if "big" in which:
        np.savez_compressed(os.path.join(HERE, "config0.npz"), **config0())


if __name__ == "__main__":
    main()
