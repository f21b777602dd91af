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
