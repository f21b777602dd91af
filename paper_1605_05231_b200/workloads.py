"""BASELINE.json configs 0-4 as seeded synthetic workloads.

There is no public dataset for this path: every input is generated from a
seed with the shapes and value distributions BASELINE.json states.
Geometry reading: source radius 3.0 mm, source-to-detector 6.0 mm (``sd_mm``,
geometry.py:26), detector D x D with width 2.0 mm, object extent 2.0 mm.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .config import ProjectorConfig, make_projector_config
from .geometry import ConeGeometry, RadialGridSpec
from .phantom import random_ellipsoid_phantom

#                  N    views polar azim  n_rho ellipsoids seed
_TABLE = {0: (64, 90, 64, 128, 128, 10, 0),
          1: (64, 90, 64, 128, 128, 10, 0),
          2: (256, 360, 180, 360, 512, 30, 2),
          3: (512, 720, 360, 720, 1024, 50, 3)}


@dataclass
class Workload:
    index: int
    n: int
    voxel: float
    geom: ConeGeometry
    spec: RadialGridSpec
    cfg: ProjectorConfig
    n_ellipsoids: int
    seed: int

    def volume(self, dtype=np.float32) -> np.ndarray:
        return random_ellipsoid_phantom(self.n, self.n_ellipsoids, self.seed, dtype)

    @property
    def name(self) -> str:
        return f"config{self.index}"


def workload(index: int) -> Workload:
    n, views, polar, azim, n_rho, n_ell, seed = _TABLE[index]
    geom = ConeGeometry(3.0, 6.0, 2.0, 2.0, n, n, views, 2.0)
    voxel = 2.0 / n
    spec = RadialGridSpec(n_rho, polar, azim, n_rho * voxel / 2.0)
    cfg = make_projector_config(geom, n, "a", radial_spec=spec, spectrum_j=6,
                                rho_pad=min(n_rho // 8, 32))
    return Workload(index, n, voxel, geom, spec, cfg, n_ell, seed)


def config4_inputs(n_points: int = 100_000_000, grid: int = 256):
    """Config 4: x ~ CN(0,1) on 256^3 (seed 4); points U[-pi,pi)^3 (seed 5),
    generated in float64 and stored as float32 (the oracle consumes the same
    float32-rounded values cast to float64)."""
    rng = np.random.default_rng(4)
    x = ((rng.standard_normal((grid,) * 3, dtype=np.float32)
          + 1j * rng.standard_normal((grid,) * 3, dtype=np.float32)) / np.sqrt(2)).astype(np.complex64)
    rng = np.random.default_rng(5)
    pts = rng.uniform(-np.pi, np.pi, (n_points, 3)).astype(np.float32)
    return x, pts
