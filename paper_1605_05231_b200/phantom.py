"""Volume type and the seeded benchmark phantoms (input generation only).

``Volume3D`` mirrors the reference API type (``cbnufft/phantom.py:52-74``):
a cubic (N, N, N) grid indexed [ix, iy, iz] with a physical voxel pitch.
The reference stores float64; this package keeps the caller's float32 data
as well so the device upload is a straight copy.

``random_ellipsoid_phantom`` is the seeded workload of BASELINE.json configs
0-3: ellipsoids with centres U[-0.6, 0.6]^3,
semi-axes U[0.05, 0.4]^3, Haar-uniform rotations and additive densities
U[-0.5, 1.0], voxel-centre sampled on [-1, 1]^3.  It is not on the hot path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Volume3D:
    """Cubic voxel grid (phantom.py:52-74)."""

    data: np.ndarray
    voxel_mm: float

    def __post_init__(self):
        self.data = np.asarray(self.data, dtype=np.float64)
        if self.data.ndim != 3 or len(set(self.data.shape)) != 1:
            raise ValueError("volume must be cubic (N, N, N)")
        if not np.all(np.isfinite(self.data)):
            raise ValueError("volume contains non-finite values")
        if not self.voxel_mm > 0:
            raise ValueError("voxel_mm must be positive")

    @classmethod
    def _checked(cls, data: np.ndarray, voxel_mm: float):
        """A float64 cubic volume already checked for non-finite values on
        the device (nufft_backproject), so the host scan is skipped."""
        v = object.__new__(cls)
        v.data, v.voxel_mm = data, float(voxel_mm)
        return v

    @property
    def n(self) -> int:
        return self.data.shape[0]

    @property
    def extent_mm(self) -> float:
        return self.n * self.voxel_mm


def voxel_centers(n: int) -> np.ndarray:
    """Voxel-centre coordinates on [-1, 1]."""
    return -1.0 + (np.arange(n) + 0.5) * (2.0 / n)


def haar_rotation(rng: np.random.Generator) -> np.ndarray:
    """Uniform random rotation: QR of a Gaussian matrix, signs fixed, det = +1."""
    q, r = np.linalg.qr(rng.standard_normal((3, 3)))
    q = q * np.sign(np.diag(r))[None, :]
    if np.linalg.det(q) < 0:
        q[:, 0] = -q[:, 0]
    return q


def random_ellipsoids(n_ellipsoids: int, seed: int):
    """Draw the ellipsoid table: list of (centre, semi_axes, rotation, density)."""
    rng = np.random.default_rng(seed)
    table = []
    for _ in range(n_ellipsoids):
        centre = rng.uniform(-0.6, 0.6, 3)
        axes = rng.uniform(0.05, 0.4, 3)
        rot = haar_rotation(rng)
        density = rng.uniform(-0.5, 1.0)
        table.append((centre, axes, rot, float(density)))
    return table


def random_ellipsoid_phantom(n: int, n_ellipsoids: int, seed: int,
                             dtype=np.float32) -> np.ndarray:
    """Voxel-centre sampled additive ellipsoid phantom on [-1, 1]^3, [ix, iy, iz]."""
    c = voxel_centers(n)
    vol = np.zeros((n, n, n), dtype=np.float64)
    # process x-slabs to bound the temporaries at large n
    slab = max(1, (1 << 22) // (n * n))
    for centre, axes, rot, density in random_ellipsoids(n_ellipsoids, seed):
        # voxels farther than the largest semi-axis from the centre are outside
        # (q >= |p - c|^2 / a_max^2), so only a bounding box is evaluated
        r = float(np.max(axes))
        sl = [np.nonzero(np.abs(c - centre[k]) <= r * (1.0 + 1e-9))[0] for k in range(3)]
        if any(s.size == 0 for s in sl):
            continue
        (i0, i1), (j0, j1), (k0, k1) = ((s[0], s[-1] + 1) for s in sl)
        py = c[None, j0:j1, None] - centre[1]
        pz = c[None, None, k0:k1] - centre[2]
        for x0 in range(i0, i1, slab):
            xs = c[x0:min(x0 + slab, i1)]
            px = xs[:, None, None] - centre[0]
            # body coordinates: R^T (p - centre)
            q = 0.0
            for k in range(3):
                bk = (rot[0, k] * px + rot[1, k] * py + rot[2, k] * pz) / axes[k]
                q = q + bk * bk
            vol[x0:x0 + xs.size, j0:j1, k0:k1] += density * (q <= 1.0)
    return vol.astype(dtype)


def smooth_ball_volume(n: int, voxel_mm: float, radius_mm: float, density: float = 1.0,
                       center_mm=(0.0, 0.0, 0.0)) -> Volume3D:
    """C1 bump density (1 - r^2/R^2)^2 inside R, voxel-centre sampled -- the
    calibration phantom of the reference (phantom.py:207-214)."""
    c = (np.arange(n) - n / 2.0 + 0.5) * voxel_mm
    x, y, z = np.meshgrid(c - center_mm[0], c - center_mm[1], c - center_mm[2], indexing="ij")
    r2 = (x * x + y * y + z * z) / radius_mm ** 2
    return Volume3D(density * np.maximum(1.0 - r2, 0.0) ** 2, voxel_mm)


def smooth_ball_line_integral(point, direction, center=(0.0, 0.0, 0.0), radius: float = 1.0,
                              density: float = 1.0):
    """Closed-form line integral of the same bump, 16 density L^5 / (15 R^4) with L
    the half chord (phantom.py:179-191); rows of (M, 3) points / unit directions."""
    p = np.atleast_2d(np.asarray(point, dtype=np.float64)) - np.asarray(center)
    d = np.atleast_2d(np.asarray(direction, dtype=np.float64))
    b = np.sum(p * d, axis=-1)
    d2 = np.sum(p * p, axis=-1) - b * b
    half = np.sqrt(np.maximum(radius ** 2 - d2, 0.0))
    return 16.0 * density * half ** 5 / (15.0 * radius ** 4)
