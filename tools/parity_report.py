#!/usr/bin/env python
"""Observed device-vs-reference parity on every committed golden fixture.

  python tools/parity_report.py > profiles/<tag>_parity.txt     (needs a GPU)
"""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [REPO, os.path.join(REPO, "tests")]
from conftest import GOLDEN, load_cases, rel_l2  # noqa: E402
from _cases import config_setup, small_setup  # noqa: E402


def main():
    from paper_1605_05231_b200 import nufft, pipeline as pl
    from paper_1605_05231_b200.grangeat import DetectorFrame
    from paper_1605_05231_b200.phantom import Volume3D
    rows = []
    for name, c in load_cases().items():
        dims = tuple(int(v) for v in c["dims"])
        plan = nufft.plan_nufft(dims, c["nodes"], 2.0, tuple(int(v) for v in c["j"]))
        bins = int((plan.first_indices().astype(np.int64) != c["first"]).any(-1).sum())
        rows.append((f"nufft {name} J={int(c['j'][0])} m={c['nodes'].shape[0]}",
                     f"bin mismatches {bins}/{c['nodes'].shape[0]}",
                     rel_l2(plan.scaling, c["scaling"]),
                     rel_l2(nufft.nufft_forward(plan, c["x"]), c["fwd"]),
                     rel_l2(nufft.nufft_adjoint(plan, c["y"]), c["adj"])))
    print(f"{'NUFFT case':40s} {'bins':28s} {'scaling':>9s} {'type2':>9s} {'type1':>9s}")
    for r in rows:
        print(f"{r[0]:40s} {r[1]:28s} {r[2]:9.1e} {r[3]:9.1e} {r[4]:9.1e}")
    print()
    print(f"{'projector case':34s} {'forward rel L2':>15s} {'worst view':>11s} {'backproject':>12s}")
    cases = [("pipeline_n16", 16, 12, "trilinear"), ("pipeline_n12_dirac", 12, 8, "dirac"),
             ("pipeline_n16_v8", 16, 8, "trilinear"), ("pipeline_n12_v48", 12, 48, "trilinear"),
             ("pipeline_n12_v24", 12, 24, "trilinear")]
    for name, n, views, basis in cases:
        g = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
        geom, voxel, spec, cfg = small_setup(n, views, basis)
        fr = np.stack([f.data for f in pl.nufft_forward_project(Volume3D(g["vol"], voxel), geom, cfg)])
        worst = max(rel_l2(fr[k], g["frames"][k]) for k in range(views))
        frames = [DetectorFrame(k, g["frames"][k], geom.pixel_mm) for k in range(views)]
        bp = pl.nufft_backproject(frames, geom, cfg, n, voxel).data
        print(f"{name:34s} {rel_l2(fr, g['frames']):15.2e} {worst:11.2e} {rel_l2(bp, g['bp']):12.2e}")
    z = np.load(os.path.join(GOLDEN, "config0.npz"))
    geom, voxel, spec, cfg = config_setup(0)
    fr = np.stack([f.data for f in pl.nufft_forward_project(Volume3D(z["vol"], voxel), geom, cfg)])
    worst = max(rel_l2(fr[k], z["frames"][k]) for k in range(geom.n_views))
    frames = [DetectorFrame(k, z["frames"][k].astype(np.float64), geom.pixel_mm)
              for k in range(geom.n_views)]
    bp = pl.nufft_backproject(frames, geom, cfg, 64, voxel).data
    print(f"{'config0 fwd / config1 bp (64^3, 90v)':34s} {rel_l2(fr, z['frames']):15.2e} {worst:11.2e} "
          f"{rel_l2(bp, z['bp']):12.2e}")
    # round-2 fixtures: CLI default geometry, config 2, bins at config 0/1
    from conftest import unpack_int
    from paper_1605_05231_b200.config import make_projector_config
    from paper_1605_05231_b200.geometry import ConeGeometry
    from paper_1605_05231_b200.phantom import random_ellipsoid_phantom, random_ellipsoids
    from paper_1605_05231_b200.workloads import analytic_projections
    z = dict(np.load(os.path.join(GOLDEN, "cli_default.npz")))
    g = z["geom"]
    geom = ConeGeometry(float(g[0]), float(g[1]), float(g[2]), float(g[3]), int(g[4]),
                        int(g[5]), int(g[6]), float(g[7]))
    n, voxel = int(z["n"]), float(z["voxel"])
    cfg = make_projector_config(geom, n, "a")
    fr = np.stack([f.data for f in pl.nufft_forward_project(Volume3D(z["vol"], voxel), geom, cfg)])
    bp = pl.nufft_backproject([DetectorFrame(k, z["frames"][k].astype(np.float64), geom.pixel_mm)
                               for k in range(geom.n_views)], geom, cfg, n, voxel).data
    st = pl.get_projector(geom, cfg, n, voxel, pl._FORWARD).plan_stats()
    print(f"{'CLI default geometry (N=16, 12v)':34s} {rel_l2(fr, z['frames']):15.2e} "
          f"{max(rel_l2(fr[k], z['frames'][k]) for k in range(geom.n_views)):11.2e} "
          f"{rel_l2(bp, z['bp']):12.2e}   invalid targets {int(z['invalid_fwd'])}, "
          f"heavy cells {st['fwd_gr_heavy_cells']}")
    geom, voxel, spec, cfg = config_setup(2)
    vol = random_ellipsoid_phantom(256, 30, 2)
    z = np.load(os.path.join(GOLDEN, "config2_fwd.npz"))
    proj = pl.Projector(geom, cfg, 256, voxel, 1)
    lat = proj.radial_lattice(vol).cpu().numpy()
    r, t, p = (np.asarray(a, dtype=np.int64) for a in z["lat_idx"].T)
    e_lat = rel_l2(lat[p, t, r], z["lat_val"])
    del lat
    frs = pl.nufft_forward_project(Volume3D(vol, voxel), geom, cfg)
    errs = [rel_l2(frs[int(k)].data, z["frames"][i]) for i, k in enumerate(z["views"])]
    zb = np.load(os.path.join(GOLDEN, "config2_bp.npz"))
    af = analytic_projections(geom, random_ellipsoids(30, 2))
    vb = pl.nufft_backproject([DetectorFrame(k, af[k], geom.pixel_mm) for k in range(360)],
                              geom, cfg, 256, voxel).data
    blocks = vb.reshape(64, 4, 64, 4, 64, 4).mean(axis=(1, 3, 5))
    e_bp = max(rel_l2(vb[128], zb["x"]), rel_l2(vb[:, 128], zb["y"]), rel_l2(vb[:, :, 128], zb["z"]))
    print(f"{'config 2 (256^3, 360v)':34s} {'lattice':>7s} {e_lat:.2e}  views "
          + " ".join(f"{e:.2e}" for e in errs)
          + f"  bp slices {e_bp:.2e} blocks {rel_l2(blocks, zb['blocks']):.2e}")
    print()
    zb = np.load(os.path.join(GOLDEN, "bins_config0.npz"))
    geom, voxel, spec, cfg = config_setup(0)
    proj = pl.Projector(geom, cfg, 64, voxel, 3)
    total = bad = 0
    for key in [k[:-3] for k in zb.files if k.endswith("__z")]:
        direction = "back" if key.endswith("_bp") or key.startswith("umb_bp") else "forward"
        node_set = "radial" if key.startswith("radial") else ("polar" if key.startswith("polar")
                                                             else "umbrella")
        batch = int(key.rsplit("_", 1)[1]) if node_set == "umbrella" else 0
        ref = unpack_int(zb, key)
        got = proj.first_indices(direction, node_set, batch).astype(np.int64)
        nb = int(np.any(got != ref, axis=1).sum())
        total += ref.shape[0]
        bad += nb
        print(f"bins {key:14s} {ref.shape[0]:9d} nodes  mismatches {nb}")
    print(f"bins total {total} nodes, mismatches {bad}")
    print()
    # config 4 shapes: 256^3 grid, 1M float32 points, J=8, against the direct DFT
    import cbn_oracle as orc
    from paper_1605_05231_b200.workloads import config4_inputs
    x, pts = config4_inputs(n_points=1 << 20)
    plan = nufft.plan_nufft(x.shape, pts, 2.0, 8)
    y = nufft.nufft_forward(plan, x)
    sel = np.random.default_rng(7).choice(pts.shape[0], 2000, replace=False)
    ref = orc.separable_dft(x.astype(np.complex128), orc.wrap(pts[sel].astype(np.float64)))
    print()
    print(f"config 4 shapes (256^3, 1M fp32 points, J=8): type-2 vs direct DFT at 2000 points "
          f"{rel_l2(y[sel], ref):.2e}")


if __name__ == "__main__":
    main()
