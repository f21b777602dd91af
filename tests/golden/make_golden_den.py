"""The backprojector's den lattice at config 2, computed by the REFERENCE itself
(pipeline.py:171-187: the resample transpose of every batch's validity mask),
and its margin to the keep threshold den > den_tol * max(den).

    python tests/golden/make_golden_den.py      # ~30 min on 8 cores
    python tests/golden/make_golden_den.py --from-cache   # re-summarise /tmp/config2_den_ref.npy

Writes tests/golden/config2_den.npz with, for every (rho, theta) ring of the
lattice (the den of a rotation-aligned view set is phi-invariant up to
rounding), the ring's min and max over phi of den / (den_tol * max(den)) for
the rings within 1e-2 of the threshold, the threshold itself, den's max and
the phi = 0 plane of den (float32, (n_rho, n_theta)).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))



def main():
    sys.path.insert(0, REF)
    from dataclasses import replace

    from cbnufft import pipeline as rpipe
    from cbnufft.geometry import ConeGeometry, RadialGridSpec
    from cbnufft.resampling import plan_resample, resample_transpose

    # config 2: 256^3, 360 views of 256^2, lattice 512 x 180 x 360
    n, views = 256, 360
    geom = ConeGeometry(3.0, 6.0, 2.0, 2.0, n, n, views, 2.0)
    voxel = 2.0 / n
    spec0 = RadialGridSpec(512, 180, 360, 512 * voxel / 2.0)
    cfg = rpipe.make_projector_config(geom, n, "a", radial_spec=spec0, spectrum_j=6,
                                      rho_pad=min(spec0.n_rho // 8, 32))
    # the backprojector's own spec and t grid (pipeline.py:164-170)
    extent = n * voxel
    bp_spec = RadialGridSpec(2 * int(np.ceil(1.5 * n / 2.0)), spec0.n_theta, spec0.n_phi,
                             extent * np.sqrt(3.0) / 2.0)
    cfg = replace(cfg, n_t=2 * geom.nu, t_pitch_mm=None, radial_spec=bp_spec,
                  rho_pad=min(bp_spec.n_rho // 8, 32))
    spec = cfg.radial_spec
    cache = "/tmp/config2_den_ref.npy"
    if "--from-cache" in sys.argv and os.path.exists(cache):
        return summarise(np.load(cache), cfg.den_tol)
    den = np.zeros((spec.n_rho, spec.n_theta, spec.n_phi))
    t0 = time.time()
    batches = list(rpipe._view_batches(geom, cfg))
    for i, batch in enumerate(batches):
        targets, valid = rpipe._umbrella_targets(geom, cfg, batch)
        rplan = plan_resample(spec, targets, cfg.method, rho_pad=cfg.rho_pad, j=cfg.resample_j,
                              oversample_factor=cfg.oversample_factor, side_lobes=cfg.side_lobes)
        den += np.real(resample_transpose(rplan, valid.astype(np.complex128)))
        del rplan
        if i % 10 == 0:
            print(f"batch {i}/{len(batches)} {time.time() - t0:.0f}s", flush=True)
    np.save(cache, den)
    summarise(den, cfg.den_tol)


def summarise(den, den_tol):
    thr = den_tol * den.max()
    r = den / thr
    lo, hi = r.min(axis=2), r.max(axis=2)
    near = np.argwhere((np.abs(lo - 1.0) < 1e-2) | (np.abs(hi - 1.0) < 1e-2))
    np.savez_compressed(os.path.join(HERE, "config2_den.npz"), rings=near.astype(np.int32),
                        ring_min=lo[near[:, 0], near[:, 1]], ring_max=hi[near[:, 0], near[:, 1]],
                        thr=np.float64(thr), dmax=np.float64(den.max()),
                        kept=np.int64((den > thr).sum()),
                        phi_spread=np.float64(np.max((hi - lo) * thr / den.max())),
                        plane0=den[:, :, 0].astype(np.float32))
    print("rings near threshold", len(near), "kept", int((den > thr).sum()), "thr", thr,
          "max phi spread / max", np.max((hi - lo) * thr / den.max()))


if __name__ == "__main__":
    main()
