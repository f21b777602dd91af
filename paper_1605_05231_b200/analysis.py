"""Angular-sampling sweep and sampling-rate helpers (drop-in for ``cbnufft/analysis.py``).

The sweep (analysis.py:103-126) is the 2D workload of the paper's sampling
study: for every angular count the image goes to its radial-line spectrum
through a device 2D type-2 NUFFT, and comes back through the device 2D
filtered backprojection (a type-1 NUFFT with the ramp), both in
``radon_fourier``.  The per-point error is the mean absolute pixel
difference over the inscribed disk; the plateau is the first angular count
whose error is within 2% of the densest one's.  The rate calculators
(analysis.py:51-83) are closed-form scalars.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .radon_fourier import fbp2d_nufft, image_to_radial_spectrum_2d


@dataclass
class SamplingRates:
    """Sinogram sample counts and spacings (analysis.py:20-36)."""

    n_rho: int
    n_theta: int
    delta_rho: float
    delta_theta: float
    n_phi: int | None = None

    def __post_init__(self):
        if min(self.n_rho, self.n_theta) <= 0:
            raise ValueError("sample counts must be positive")
        if min(self.delta_rho, self.delta_theta) <= 0:
            raise ValueError("sample spacings must be positive")
        if self.n_phi is not None and self.n_phi <= 0:
            raise ValueError("n_phi must be positive")


@dataclass
class SweepResult:
    """(n_theta, error) points in increasing n_theta and the plateau (analysis.py:39-48)."""

    points: list
    plateau: int

    def __post_init__(self):
        counts = [int(p[0]) for p in self.points]
        if any(later <= earlier for earlier, later in zip(counts[:-1], counts[1:])):
            raise ValueError("n_theta values must be strictly increasing")


def nyquist_rates(x_max: float, w_max: float) -> tuple[float, float]:
    """(spacing pi / w_max, unrounded count 2 x_max w_max / pi) (analysis.py:51-61)."""
    if not (x_max > 0 and w_max > 0):
        raise ValueError("x_max and w_max must be positive")
    return math.pi / w_max, 2.0 * x_max * w_max / math.pi


def sinogram_rates(x_max: float, w_max: float, hexagonal: bool = False) -> SamplingRates:
    """Radial/angular sinogram rates for one band budget (analysis.py:64-83)."""
    spacing, count = nyquist_rates(x_max, w_max)
    n_rho = int(round(count))
    if hexagonal:
        return SamplingRates(2 * n_rho, 2 * n_rho, spacing / 2.0, math.pi / (2 * n_rho))
    return SamplingRates(n_rho, int(math.ceil(math.pi * count)), spacing,
                         math.pi / (x_max * w_max + 1.0))


def inscribed_disk_mask(n: int) -> np.ndarray:
    """Pixel centres inside the disk of radius n/2 (analysis.py:86-90)."""
    r = np.arange(n) + 0.5 - n / 2.0
    return r[:, None] ** 2 + r[None, :] ** 2 <= (n / 2.0) ** 2


def masked_error_metrics(a, b, mask):
    """(mean |a-b|, RMSE, max |a-b|) over the mask (analysis.py:93-100)."""
    a = np.asarray(a)
    b = np.asarray(b)
    mask = np.asarray(mask, dtype=bool)
    if not (a.shape == b.shape == mask.shape):
        raise ValueError("a, b and mask must share one shape")
    if not mask.any():
        raise ValueError("mask selects no elements")
    diff = (a - b)[mask]
    ad = np.abs(diff)
    return float(ad.mean()), float(np.sqrt(np.mean(diff * diff))), float(ad.max())


def angular_sweep(image, n_theta_list, n_rho: int) -> SweepResult:
    """Reconstruction error versus angular count (analysis.py:103-126), device NUFFTs."""
    image = np.asarray(image, dtype=np.float64)
    if image.ndim != 2 or image.shape[0] != image.shape[1]:
        raise ValueError("image must be square")
    n = image.shape[0]
    mask = inscribed_disk_mask(n)
    points = []
    for n_theta in sorted(int(v) for v in n_theta_list):
        recon, _ = fbp2d_nufft(image_to_radial_spectrum_2d(image, n_rho, n_theta), n)
        points.append((n_theta, masked_error_metrics(recon, image, mask)[0]))
    floor = points[-1][1]
    plateau = next(nt for nt, err in points if err <= 1.02 * floor)
    return SweepResult(points, plateau)

