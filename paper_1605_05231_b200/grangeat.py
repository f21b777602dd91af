"""Per-view Grangeat data types (drop-in for ``cbnufft/grangeat.py`` types).

``DetectorFrame`` and ``UmbrellaView`` keep the reference's fields and
validation (grangeat.py:30-55).  The Grangeat transforms themselves run on the
device inside the projector plan (``csrc/cbn_projector.cu``:
``grangeat_reverse``; ``csrc/cbn_backproject.cu``: forward Grangeat) and are
reachable per view block through ``Projector.grangeat_reverse`` /
``Projector.grangeat_forward`` in ``pipeline.py``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class UmbrellaView:
    """One view's derivative-Radon values on the (mu, t) lattice (grangeat.py:30-40)."""

    view_index: int
    values: np.ndarray
    coords: tuple

    def __post_init__(self):
        if self.values.shape != self.coords[0].shape:
            raise ValueError("value grid and coordinate grids disagree")


@dataclass
class DetectorFrame:
    """One cone-beam projection on the physical detector, [u, v] (grangeat.py:43-55)."""

    view_index: int
    data: np.ndarray
    pixel_mm: tuple

    def __post_init__(self):
        if self.data.ndim != 2:
            raise ValueError("detector data must be 2D")
        if not np.all(np.isfinite(self.data)):
            raise ValueError("detector data contains non-finite values")

    @classmethod
    def _checked(cls, view_index: int, data: np.ndarray, pixel_mm):
        """A frame whose data the device already checked for non-finite values
        (cbn_forward_project returns CBN_ENONFINITE -> FloatingPointError,
        pipeline.py:144-145), so the per-frame host scan is skipped."""
        f = object.__new__(cls)
        f.view_index, f.data, f.pixel_mm = view_index, data, pixel_mm
        return f


def detector_axes_virtual(geom):
    pu, pv = geom.virtual_pixel_mm
    u = (np.arange(geom.nu) - geom.nu / 2.0 + 0.5) * pu
    v = (np.arange(geom.nv) - geom.nv / 2.0 + 0.5) * pv
    return u, v


def grangeat_preweight(geom) -> np.ndarray:
    u, v = detector_axes_virtual(geom)
    return geom.so_mm / np.sqrt(geom.so_mm ** 2 + u[:, None] ** 2 + v[None, :] ** 2)


def grangeat_postweight(geom, t) -> np.ndarray:
    return (geom.so_mm ** 2 + np.asarray(t) ** 2) / geom.so_mm ** 2


@dataclass
class GrangeatPlan:
    """Per-geometry Grangeat state (grangeat.py:77-90), held on the device by a
    projector plan whose forward direction runs the reverse transform and whose
    back direction runs the forward transform on this (n_mu, n_t, dt) grid."""

    geom: object
    n_mu: int
    n_t: int
    dt: float
    omega: np.ndarray
    w1: np.ndarray
    w2: np.ndarray
    taper: np.ndarray
    projector: object = None


def plan_grangeat(geom, n_mu: int, n_t: int, j=(5, 5), oversample_factor: float = 2.0,
                  t_pitch_mm: float | None = None, t_taper: str = "none") -> GrangeatPlan:
    """grangeat.py:93-128."""
    from .config import ProjectorConfig
    from .geometry import RadialGridSpec, umbrella_line_grid
    from .pipeline import Projector
    if tuple(np.broadcast_to(np.atleast_1d(j), (2,))) != (5, 5) or float(oversample_factor) != 2.0:
        raise NotImplementedError("the device Grangeat plan uses j=(5, 5), oversample 2 "
                                  "(the pipeline's setting, grangeat.py:94)")
    if t_taper not in ("none", "hann"):
        raise ValueError("t_taper must be 'none' or 'hann'")
    mu, t = umbrella_line_grid(geom, n_mu, n_t, t_pitch_mm)
    pu, _ = geom.virtual_pixel_mm
    dt = pu if t_pitch_mm is None else float(t_pitch_mm)
    omega = 2.0 * np.pi * (np.arange(n_t) - n_t // 2) / (n_t * dt)
    if t_taper == "hann":
        taper = np.cos(np.pi * omega / (2.0 * np.abs(omega).max())) ** 2
    else:
        taper = np.ones(n_t)
    cfg = ProjectorConfig("a", RadialGridSpec(2, 1, 1, 1.0), n_mu=int(n_mu), n_t=int(n_t),
                          t_pitch_mm=t_pitch_mm, t_taper=t_taper, rho_pad=0)
    proj = Projector(geom, cfg, 2, 1.0, 3, bp_n_t=int(n_t), bp_t_pitch_mm=dt)
    return GrangeatPlan(geom, int(n_mu), int(n_t), dt, omega, grangeat_preweight(geom),
                        grangeat_postweight(geom, t), taper, proj)


def forward_grangeat_view(frame: DetectorFrame, gp: GrangeatPlan) -> UmbrellaView:
    """Detector frame -> umbrella derivative-Radon values (grangeat.py:131-146)."""
    from .geometry import umbrella_coordinates
    geom = gp.geom
    if tuple(frame.data.shape) != (geom.nu, geom.nv):
        raise ValueError("frame dims do not match the geometry")
    vals = gp.projector.grangeat_forward(np.asarray(frame.data, dtype=np.float32)[None])
    values = vals.cpu().numpy()[0].astype(np.float64)
    coords = umbrella_coordinates(geom, frame.view_index, gp.n_mu, gp.n_t, gp.dt)
    return UmbrellaView(frame.view_index, values, coords)


def reverse_grangeat_view(view: UmbrellaView, gp: GrangeatPlan) -> DetectorFrame:
    """Umbrella values -> detector frame (grangeat.py:149-170)."""
    if tuple(view.values.shape) != (gp.n_mu, gp.n_t):
        raise ValueError("umbrella grid does not match the plan")
    out = gp.projector.grangeat_reverse(np.asarray(view.values, dtype=np.float32)[None])
    return DetectorFrame(view.view_index, out.cpu().numpy()[0].astype(np.float64),
                         gp.geom.pixel_mm)
