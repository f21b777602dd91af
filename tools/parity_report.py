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
