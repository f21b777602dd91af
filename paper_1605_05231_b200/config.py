"""Projector configuration (pipeline.py:31-80 of the reference).

``ProjectorConfig`` keeps the reference's field names, defaults and
validation; ``make_projector_config`` keeps its practical-rate defaults.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from .geometry import ConeGeometry, RadialGridSpec


@dataclass
class ProjectorConfig:
    """Settings of the NUFFT forward projector / backprojector (pipeline.py:31-56)."""

    method: str
    radial_spec: RadialGridSpec
    n_mu: int
    n_t: int
    t_pitch_mm: float | None = None
    t_taper: str = "hann"
    spectrum_j: int = 3
    resample_j: tuple = (3, 3, 3)
    side_lobes: int = 2
    oversample_factor: float = 2.0
    rho_pad: int | None = None
    basis: str = "trilinear"
    normalization: float = 1.0
    bp_normalization: float = 1.0
    den_tol: float = 1e-3

    def __post_init__(self):
        m = str(self.method).lower()
        if m not in ("a", "b"):
            raise ValueError("method must be 'a' or 'b'")
        self.method = m
        if self.basis not in ("trilinear", "dirac"):
            raise ValueError("basis must be 'trilinear' or 'dirac'")


def make_projector_config(geom: ConeGeometry, n: int, method: str = "a",
                          **overrides) -> ProjectorConfig:
    """Defaults of pipeline.py:59-80: n_rho = 4.5 N (even), n_theta = n_phi = 2N,
    rho_max = sqrt(3)/2 * extent, n_mu = 2 nu, n_t = 6 nu at third-pixel pitch."""
    n_rho = 2 * int(math.ceil(4.5 * n / 2.0))
    spec = RadialGridSpec(n_rho, 2 * n, 2 * n,
                          float(geom.object_extent_mm) * math.sqrt(3.0) / 2.0)
    cfg = ProjectorConfig(method, spec, n_mu=2 * geom.nu, n_t=6 * geom.nu,
                          t_pitch_mm=geom.virtual_pixel_mm[0] / 3.0,
                          rho_pad=min(n_rho // 8, 32))
    for key, value in overrides.items():
        setattr(cfg, key, value)
    return cfg
