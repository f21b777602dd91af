"""ORACLE -- TEST INFRASTRUCTURE ONLY.

A float64 numpy/scipy restatement of the reference ``cbnufft`` hot path
(``/root/reference/pkg/src/cbnufft``), written from the reference's published
algorithm for use as

* the checker in ``tests/`` and ``__graft_entry__.smoke()``, and
* the ``cpu_baseline`` / ``--impl reference`` leg of ``bench.py``
  (``kind: "port"`` -- the reference package itself cannot travel to the GPU
  box).

It is never imported by the product package ``paper_1605_05231_b200``.

Parity pinning: ``tests/test_oracle_golden.py`` checks every function here
against golden vectors produced by running the reference itself
(``tests/golden/make_golden.py``) to ~1e-10 relative; the reference's own
brute-force NUDFT oracle (``pkg/tests/test_nufft.py:13-18``) is restated in
``nudft`` below and checked too.

Differences from the reference that do not change results beyond float64
round-off: interpolation weights are recomputed per row chunk instead of being
stored as a dense (m, J^d) matrix (``nufft.py:188-213``), and sums run in a
different order.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
from scipy import fft as sfft
from scipy.special import i0

PLAN_CHUNK = 1 << 21      # nufft.py:24  nodes per sub-plan (chunked variants)
TARGET_BATCH = 1 << 20    # pipeline.py:28  umbrella targets per resample plan
LS_SAMPLES = 8192         # nufft.py:163-168  scaling-fit subsample
_ROWS = 1 << 15           # rows per gather/spread block (memory bound only)
WORKERS = os.cpu_count() or 1

TWO_PI = 2.0 * np.pi


# --------------------------------------------------------------------------
# Kaiser-Bessel gridding kernel and per-axis index math   (nufft.py:36-56,171-179)
# --------------------------------------------------------------------------

def beatty_beta(j: int, alpha: float) -> float:
    """nufft.py:53-56."""
    return float(np.pi * np.sqrt(max((j / alpha) ** 2 * (alpha - 0.5) ** 2 - 0.8, 0.0)))


def kb_kernel(x, j: int, beta: float):
    """KB value at offset x; exactly zero for |x| >= j/2 (nufft.py:36-41)."""
    x = np.asarray(x, dtype=np.float64)
    arg = 1.0 - (2.0 * x / j) ** 2
    return np.where(arg > 0.0, i0(beta * np.sqrt(np.maximum(arg, 0.0))), 0.0)


def wrap(w):
    """Alias to [-pi, pi) (nufft.py:104-108, radon_fourier.py:70-72)."""
    return np.mod(np.asarray(w, dtype=np.float64) + np.pi, TWO_PI) - np.pi


def axis_coords(w, k: int, j: int):
    """Grid coordinate u, first tap and fractional offsets for one axis.

    u = mod(w, 2 pi) * K / (2 pi), snapped to the nearest integer within 1e-9,
    first = ceil(u - J/2)   (nufft.py:173-176).
    """
    u = np.mod(w, TWO_PI) * k / TWO_PI
    ur = np.round(u)
    u = np.where(np.abs(u - ur) < 1e-9, ur, u)
    first = np.ceil(u - j / 2.0)
    return u, first


def axis_weights(u, first, j: int, beta: float):
    offs = first[:, None] + np.arange(j)[None, :]
    return kb_kernel(u[:, None] - offs, j, beta)


def ls_rows(m: int) -> np.ndarray:
    """Rows used by the scaling fit (nufft.py:163-168)."""
    if m > LS_SAMPLES:
        sel = np.random.default_rng(0).choice(m, LS_SAMPLES, replace=False)
        sel.sort()
        return sel
    return np.arange(m)


def ls_scaling(n: int, k: int, j: int, u, first, w) -> np.ndarray:
    """Least-squares per-axis deapodisation (nufft.py:111-134) on pre-selected rows."""
    nu = (np.arange(n) - n // 2) / k
    frac = u - first
    num = np.zeros(n)
    resp = np.zeros((u.shape[0], n), dtype=np.complex128)
    for p in range(j):
        num += w[:, p] @ np.cos(TWO_PI * np.outer(frac - p, nu))
        resp += w[:, p, None] * np.exp(-2j * np.pi * p * nu)[None, :]
    den = np.sum(resp.real ** 2 + resp.imag ** 2, axis=0)
    s = num / np.maximum(den, 1e-300)
    return np.maximum(s, 1e-8 * np.max(s))


@dataclass
class Plan:
    """Gridding plan: per-axis first taps / weights / scalings (nufft.py:88-101)."""

    dims: tuple
    kdims: tuple
    taps: tuple
    betas: tuple
    nodes: np.ndarray        # (m, d) wrapped
    first: list              # per axis (m,) float first-tap index
    weights: list            # per axis (m, J) float64
    scale: list              # per axis (n,) float64
    phase: np.ndarray        # (m,) exp(-i w . (N//2))

    @property
    def m(self) -> int:
        return self.nodes.shape[0]

    def scaling_grid(self) -> np.ndarray:
        s = self.scale[0]
        for v in self.scale[1:]:
            s = np.multiply.outer(s, v)
        return s


def make_plan(dims, nodes, sigma: float = 2.0, j=6) -> Plan:
    """nufft.py:137-218 (weights kept per axis; tensor product formed on use)."""
    dims = tuple(int(v) for v in np.atleast_1d(dims))
    if sigma < 1.0:
        raise ValueError("oversample_factor must be >= 1")
    nodes = np.asarray(nodes, dtype=np.float64)
    if nodes.ndim == 1:
        nodes = nodes[:, None]
    nodes = np.atleast_2d(nodes)
    if not np.all(np.isfinite(nodes)):
        raise ValueError("nodes must be finite")
    nodes = wrap(nodes)
    d = len(dims)
    if nodes.shape[1] != d:
        raise ValueError(f"nodes must have {d} coordinates per row")
    taps = tuple(int(t) for t in np.broadcast_to(np.atleast_1d(j), (d,)))
    if min(taps) < 1:
        raise ValueError("tap counts must be >= 1")
    mult = int(np.ceil(sigma - 1e-12))
    kdims = tuple(n * mult for n in dims)
    betas = tuple(beatty_beta(t, kk / n) for t, kk, n in zip(taps, kdims, dims))
    sel = ls_rows(nodes.shape[0])
    firsts, weights, scales = [], [], []
    for a in range(d):
        u, first = axis_coords(nodes[:, a], kdims[a], taps[a])
        w = axis_weights(u, first, taps[a], betas[a])
        scales.append(ls_scaling(dims[a], kdims[a], taps[a], u[sel], first[sel], w[sel]))
        firsts.append(first)
        weights.append(w)
    centre = np.array([n // 2 for n in dims], dtype=np.float64)
    phase = np.exp(-1j * (nodes @ centre))
    return Plan(dims, kdims, taps, betas, nodes, firsts, weights, scales, phase)


def _roll_index(n: int, k: int) -> np.ndarray:
    return np.mod(np.arange(n) - n // 2, k)


def _tap_block(plan: Plan, lo: int, hi: int):
    """Flat K-grid indices and tensor weights for rows [lo, hi)."""
    idx = np.zeros((hi - lo,) + (1,) * len(plan.dims), dtype=np.int64)
    wt = np.ones((hi - lo,) + (1,) * len(plan.dims))
    stride = 1
    for a in reversed(range(len(plan.dims))):
        cols = np.mod(plan.first[a][lo:hi, None] + np.arange(plan.taps[a])[None, :],
                      plan.kdims[a]).astype(np.int64)
        shape = [hi - lo] + [1] * len(plan.dims)
        shape[1 + a] = plan.taps[a]
        idx = idx + (cols * stride).reshape(shape)
        wt = wt * plan.weights[a][lo:hi].reshape(shape)
        stride *= plan.kdims[a]
    return idx.reshape(hi - lo, -1), wt.reshape(hi - lo, -1)


def type2(plan: Plan, x) -> np.ndarray:
    """Uniform grid -> node values (nufft.py:221-233)."""
    x = np.asarray(x)
    if x.shape != plan.dims:
        raise ValueError(f"input shape {x.shape} does not match plan dims {plan.dims}")
    grid = np.zeros(plan.kdims, dtype=np.complex128)
    grid[np.ix_(*[_roll_index(n, k) for n, k in zip(plan.dims, plan.kdims)])] = \
        (x * plan.scaling_grid()).astype(np.complex128)
    flat = sfft.fftn(grid, overwrite_x=True, workers=WORKERS).ravel()
    out = np.empty(plan.m, dtype=np.complex128)
    for lo in range(0, plan.m, _ROWS):
        hi = min(lo + _ROWS, plan.m)
        idx, wt = _tap_block(plan, lo, hi)
        out[lo:hi] = np.einsum("ij,ij->i", flat[idx], wt)
    return out * plan.phase


def type1(plan: Plan, y) -> np.ndarray:
    """Exact adjoint of type2 (nufft.py:236-247)."""
    y = np.asarray(y, dtype=np.complex128)
    if y.shape != (plan.m,):
        raise ValueError(f"expected {plan.m} node values, got {y.shape}")
    y = y * np.conj(plan.phase)
    ktot = int(np.prod(plan.kdims))
    acc_re = np.zeros(ktot)
    acc_im = np.zeros(ktot)
    for lo in range(0, plan.m, _ROWS):
        hi = min(lo + _ROWS, plan.m)
        idx, wt = _tap_block(plan, lo, hi)
        v = wt * y[lo:hi, None]
        acc_re += np.bincount(idx.ravel(), weights=v.real.ravel(), minlength=ktot)
        acc_im += np.bincount(idx.ravel(), weights=v.imag.ravel(), minlength=ktot)
    grid = (acc_re + 1j * acc_im).reshape(plan.kdims)
    grid = sfft.ifftn(grid, overwrite_x=True, workers=WORKERS) * ktot
    out = grid[np.ix_(*[_roll_index(n, k) for n, k in zip(plan.dims, plan.kdims)])]
    return out * plan.scaling_grid()


def type2_chunked(dims, nodes, x, sigma=2.0, j=6, chunk=None):
    """nufft.py:250-265: one sub-plan (own scaling fit) per PLAN_CHUNK nodes."""
    chunk = PLAN_CHUNK if chunk is None else chunk
    nodes = np.atleast_2d(np.asarray(nodes, dtype=np.float64))
    out = np.empty(nodes.shape[0], dtype=np.complex128)
    for lo in range(0, nodes.shape[0], chunk):
        hi = min(lo + chunk, nodes.shape[0])
        out[lo:hi] = type2(make_plan(dims, nodes[lo:hi], sigma, j), x)
    return out


def type1_chunked(dims, nodes, y, sigma=2.0, j=6, chunk=None):
    """nufft.py:268-282."""
    chunk = PLAN_CHUNK if chunk is None else chunk
    nodes = np.atleast_2d(np.asarray(nodes, dtype=np.float64))
    y = np.asarray(y, dtype=np.complex128)
    acc = np.zeros(tuple(int(v) for v in np.atleast_1d(dims)), dtype=np.complex128)
    for lo in range(0, nodes.shape[0], chunk):
        hi = min(lo + chunk, nodes.shape[0])
        acc += type1(make_plan(dims, nodes[lo:hi], sigma, j), y[lo:hi])
    return acc


def nudft(dims, nodes, x):
    """Brute force X(w) = sum_n x(n) exp(-i w.n)  (pkg/tests/test_nufft.py:13-18)."""
    dims = tuple(int(v) for v in np.atleast_1d(dims))
    pos = np.stack([g.ravel() for g in np.meshgrid(*[np.arange(v) for v in dims],
                                                   indexing="ij")], axis=-1)
    return np.exp(-1j * np.atleast_2d(nodes) @ pos.T) @ np.asarray(x).ravel()


def separable_dft(x, nodes):
    """Direct DTFT of a 3D array at nodes via per-axis phasors (memory O(m N))."""
    x = np.asarray(x)
    e = [np.exp(-1j * np.outer(nodes[:, a], np.arange(x.shape[a]))) for a in range(3)]
    out = np.empty(nodes.shape[0], dtype=np.complex128)
    for lo in range(0, nodes.shape[0], 256):
        hi = min(lo + 256, nodes.shape[0])
        out[lo:hi] = np.einsum("pi,pj,pk,ijk->p", e[0][lo:hi], e[1][lo:hi], e[2][lo:hi], x,
                               optimize=True)
    return out


# --------------------------------------------------------------------------
# Fourier-slice transforms   (radon_fourier.py)
# --------------------------------------------------------------------------

def radial_omega(n_rho: int, delta_rho: float) -> np.ndarray:
    """radon_fourier.py:46-49 (rad per length unit)."""
    k = np.arange(n_rho) - n_rho // 2
    return 2.0 * np.pi * k / (n_rho * delta_rho)


def spec_arrays(spec):
    n_r, n_t, n_p, rmax = int(spec.n_rho), int(spec.n_theta), int(spec.n_phi), float(spec.rho_max)
    d_rho = 2.0 * rmax / n_r
    theta = np.arange(n_t) * np.pi / n_t
    phi = np.arange(n_p) * 2.0 * np.pi / n_p
    return n_r, n_t, n_p, rmax, d_rho, theta, phi


def radial_direction_nodes(spec, voxel_mm: float) -> np.ndarray:
    """radon_fourier.py:59-67: (m, 3) unwrapped, rho fastest, then theta, then phi."""
    n_r, n_t, n_p, _, d_rho, theta, phi = spec_arrays(spec)
    om = radial_omega(n_r, d_rho) * voxel_mm
    th = np.repeat(np.tile(theta, n_p), n_r)
    ph = np.repeat(phi, n_t * n_r)
    st = np.sin(th)
    direc = np.stack([np.cos(ph) * st, np.sin(ph) * st, np.cos(th)], axis=-1)
    return np.tile(om, n_t * n_p)[:, None] * direc


def centre_phase(nodes, dims):
    """radon_fourier.py:52-56."""
    shift = np.array([n / 2.0 - 0.5 for n in dims])
    return np.exp(1j * (nodes @ shift))


def to_lattice(values, spec):
    """Node order (phi, theta, rho) -> reference lattice layout (rho, theta, phi)."""
    return values.reshape(int(spec.n_phi), int(spec.n_theta), int(spec.n_rho)).transpose(2, 1, 0)


def radial_spectrum(vol, voxel_mm, spec, j=6, sigma=2.0, chunk=None):
    """image_to_radial_spectrum (radon_fourier.py:89-108) -> lattice layout."""
    n = vol.shape[0]
    nodes = wrap(radial_direction_nodes(spec, voxel_mm))
    vals = type2_chunked((n, n, n), nodes, np.asarray(vol, dtype=np.complex128),
                         sigma, j, chunk)
    vals *= centre_phase(nodes, (n, n, n))
    return to_lattice(vals, spec)


def trilinear_transfer(spec, voxel_mm):
    """radon_fourier.py:75-86."""
    nodes = radial_direction_nodes(spec, voxel_mm)
    return to_lattice(np.prod(np.sinc(nodes / TWO_PI), axis=-1) ** 2, spec)


def centred_fft(x, axis=0):
    return np.fft.fftshift(np.fft.fft(np.fft.ifftshift(x, axes=axis), axis=axis), axes=axis)


def centred_ifft(x, axis=0):
    return np.fft.fftshift(np.fft.ifft(np.fft.ifftshift(x, axes=axis), axis=axis), axes=axis)


def radial_lattice(vol, voxel_mm, spec, spectrum_j=6, sigma=2.0, basis="trilinear",
                   chunk=None):
    """pipeline.py:113-119: complex derivative-Radon lattice (rho, theta, phi)."""
    s = radial_spectrum(vol, voxel_mm, spec, spectrum_j, sigma, chunk)
    if basis == "trilinear":
        s = s * trilinear_transfer(spec, voxel_mm)
    n_r, _, _, _, d_rho, _, _ = spec_arrays(spec)
    s = s * (1j * radial_omega(n_r, d_rho))[:, None, None]          # radon_fourier.py:111-114
    return centred_ifft(s, axis=0) / d_rho                          # radon_fourier.py:133-135


# --------------------------------------------------------------------------
# Geometry: umbrella planes   (geometry.py:143-217)
# --------------------------------------------------------------------------

def canonical(rho, theta, phi):
    """geometry.py:143-159."""
    rho = np.array(rho, dtype=np.float64)
    st = np.sin(theta)
    n = np.stack([np.cos(phi) * st, np.sin(phi) * st, np.cos(theta) * np.ones_like(phi * theta)],
                 axis=-1)
    flip = n[..., 2] < 0.0
    n = np.where(flip[..., None], -n, n)
    rho = np.where(flip, -rho, rho)
    th = np.arccos(np.clip(n[..., 2], -1.0, 1.0))
    ph = np.mod(np.arctan2(n[..., 1], n[..., 0]), TWO_PI)
    return rho, np.where(th >= np.pi, 0.0, th), ph


def umbrella_planes(geom, view: int, n_mu: int, n_t: int, dt: float):
    """geometry.py:190-217 with t pitch dt; returns (rho, theta, phi) (n_mu, n_t)."""
    mu = np.arange(n_mu) * np.pi / n_mu
    t = (np.arange(n_t) - n_t // 2) * dt
    a = 2.0 * np.pi * view / geom.n_views
    s = geom.so_mm * np.array([np.cos(a), np.sin(a), 0.0])
    uh = np.array([-np.sin(a), np.cos(a), 0.0])
    vh = np.array([0.0, 0.0, 1.0])
    e = np.cos(mu)[:, None, None] * uh + np.sin(mu)[:, None, None] * vh
    d = -np.sin(mu)[:, None, None] * uh + np.cos(mu)[:, None, None] * vh
    p0 = t[None, :, None] * e
    n = np.cross(p0 - s, np.broadcast_to(d, p0.shape))
    n /= np.linalg.norm(n, axis=-1, keepdims=True)
    rho = np.sum(n * s, axis=-1)
    th = np.arccos(np.clip(n[..., 2], -1.0, 1.0))
    ph = np.mod(np.arctan2(n[..., 1], n[..., 0]), TWO_PI)
    return canonical(rho, th, ph)


def polar_index(coords, spec):
    """resampling.py:38-59 (fractional lattice indices)."""
    n_r, n_t, n_p, rmax, d_rho, _, _ = spec_arrays(spec)
    rho, th, ph = canonical(coords[:, 0], coords[:, 1], coords[:, 2])
    if np.any(np.abs(rho) > rmax * (1.0 + 1e-12)):
        raise ValueError("rho outside the radial grid support")
    ir = rho / d_rho + n_r / 2.0
    it = th * n_t / np.pi
    ip = ph * n_p / TWO_PI
    top = ir >= n_r - 1e-9
    return np.stack([np.where(top, 0.0, ir),
                     np.where(top, np.mod(n_t - it, n_t), it),
                     np.where(top, np.mod(ip + n_p / 2.0, n_p), ip)], axis=-1)


def umbrella_targets(geom, spec, views, n_mu, n_t, dt):
    """pipeline.py:83-102: (targets, valid) for a list of views."""
    rows = []
    for k in views:
        r, th, ph = umbrella_planes(geom, k, n_mu, n_t, dt)
        rows.append(np.stack([r.ravel(), th.ravel(), ph.ravel()], axis=-1))
    coords = np.concatenate(rows, axis=0)
    valid = np.abs(coords[:, 0]) <= float(spec.rho_max) * (1.0 + 1e-12)
    coords[~valid] = 0.0
    return polar_index(coords, spec), valid


def view_batches(n_views: int, per_view: int, target_batch: int = None):
    """pipeline.py:105-110."""
    tb = TARGET_BATCH if target_batch is None else target_batch
    step = max(1, tb // per_view)
    return [range(lo, min(lo + step, n_views)) for lo in range(0, n_views, step)]


# --------------------------------------------------------------------------
# Radial -> umbrella resampling, method A   (resampling.py:79-123,136-196)
# --------------------------------------------------------------------------

@dataclass
class Resampler:
    spec: object
    targets: np.ndarray
    pad: int
    padded: tuple
    plan: Plan


def make_resampler(spec, targets, rho_pad=None, j=(3, 3, 3), sigma=2.0) -> Resampler:
    n_r, n_t, n_p = int(spec.n_rho), int(spec.n_theta), int(spec.n_phi)
    targets = np.atleast_2d(np.asarray(targets, dtype=np.float64))
    lim = np.array([n_r, n_t, n_p], dtype=np.float64)
    if targets.shape[-1] != 3:
        raise ValueError("targets must be (m, 3) fractional indices")
    if np.any(targets < -1e-9) or np.any(targets >= lim + 1e-9):
        raise ValueError("targets must be wrapped into the lattice index range")
    pad = n_r // 2 if rho_pad is None else int(rho_pad)
    padded = (n_r + 2 * pad, n_t, n_p)
    pos = targets.copy()
    pos[:, 0] += pad
    nodes = -2.0 * np.pi * pos / np.array(padded, dtype=np.float64)
    return Resampler(spec, targets, pad, padded, make_plan(padded, nodes, sigma, j))


def origin_average(x, spec):
    out = np.array(x, copy=True)
    row = int(spec.n_rho) // 2
    out[row] = np.mean(x[row])
    return out


def shift_phase(pos, dims):
    shift = np.array([2.0 * np.pi * (n // 2) / n for n in dims])
    return np.exp(-1j * (pos @ shift))


def resample_forward(rs: Resampler, lattice):
    """resample_apply, method A (resampling.py:136-148)."""
    x = origin_average(np.asarray(lattice, dtype=np.complex128), rs.spec)
    if rs.pad:
        x = np.pad(x, ((rs.pad, rs.pad), (0, 0), (0, 0)))
    spec_x = np.fft.fftshift(sfft.fftn(x, workers=WORKERS)) / x.size
    pos = rs.targets.copy()
    pos[:, 0] += rs.pad
    return type2(rs.plan, spec_x) * shift_phase(pos, rs.padded)


def resample_adjoint(rs: Resampler, values):
    """resample_transpose, method A (resampling.py:164-196)."""
    pos = rs.targets.copy()
    pos[:, 0] += rs.pad
    y = np.asarray(values, dtype=np.complex128) * np.conj(shift_phase(pos, rs.padded))
    g = sfft.ifftn(np.fft.ifftshift(type1(rs.plan, y).reshape(rs.padded)), workers=WORKERS)
    if rs.pad:
        g = g[rs.pad:rs.pad + int(rs.spec.n_rho)]
    return origin_average(g, rs.spec)


def dirichlet(t, n: int):
    """Periodic interpolating kernel (nufft.py:285-298): phasor x periodic sinc."""
    t = np.asarray(t, dtype=np.float64)
    phase = np.exp(1j * np.pi * t * (n - 1) / n)
    den = n * np.sin(np.pi * t / n)
    near = np.abs(den) < 1e-9
    ratio = np.where(near, np.cos(np.pi * t) / np.cos(np.pi * t / n),
                     np.sin(np.pi * t) / np.where(near, 1.0, den))
    return phase * ratio


def b_axis_taps(pos, dim: int, taps: int):
    """The `taps` nearest centred periodic-sinc taps of one axis (resampling.py:126-133)."""
    first = np.ceil(pos - taps / 2.0)
    offs = first[:, None] + np.arange(taps)[None, :]
    t = pos[:, None] - offs
    w = dirichlet(t, dim) * np.exp(-2j * np.pi * (dim // 2) * t / dim)
    return np.mod(offs.astype(np.int64), dim), w


def _b_index(spec, targets, rho_pad, side_lobes):
    n_r, n_t, n_p = int(spec.n_rho), int(spec.n_theta), int(spec.n_phi)
    pad = n_r // 2 if rho_pad is None else int(rho_pad)
    dims = (n_r + 2 * pad, n_t, n_p)
    pos = np.atleast_2d(np.asarray(targets, dtype=np.float64)).copy()
    pos[:, 0] += pad
    taps = side_lobes + 1
    c0, w0 = b_axis_taps(pos[:, 0], dims[0], taps)
    c1, w1 = b_axis_taps(pos[:, 1], dims[1], taps)
    c2, w2 = b_axis_taps(pos[:, 2], dims[2], taps)
    idx = (c0[:, :, None, None] * dims[1] + c1[:, None, :, None]) * dims[2] + c2[:, None, None, :]
    return pad, dims, idx, (w0, w1, w2)


def resample_b_forward(spec, targets, lattice, rho_pad=None, side_lobes=2):
    """resample_apply, method B (resampling.py:149-161)."""
    pad, dims, idx, (w0, w1, w2) = _b_index(spec, targets, rho_pad, side_lobes)
    x = origin_average(np.asarray(lattice, dtype=np.complex128), spec)
    if pad:
        x = np.pad(x, ((pad, pad), (0, 0), (0, 0)))
    return np.einsum("ma,mb,mc,mabc->m", w0, w1, w2, x.ravel()[idx])


def resample_b_adjoint(spec, targets, values, rho_pad=None, side_lobes=2):
    """resample_transpose, method B (resampling.py:176-196)."""
    pad, dims, idx, (w0, w1, w2) = _b_index(spec, targets, rho_pad, side_lobes)
    vals = np.einsum("m,ma,mb,mc->mabc", np.asarray(values, dtype=np.complex128),
                     np.conj(w0), np.conj(w1), np.conj(w2))
    flat = np.zeros(int(np.prod(dims)), dtype=np.complex128)
    np.add.at(flat, idx.ravel(), vals.ravel())
    g = flat.reshape(dims)
    if pad:
        g = g[pad:pad + int(spec.n_rho)]
    return origin_average(g, spec)


# --------------------------------------------------------------------------
# Per-view Grangeat   (grangeat.py:58-170)
# --------------------------------------------------------------------------

@dataclass
class Grangeat:
    geom: object
    n_mu: int
    n_t: int
    dt: float
    plan: Plan
    cphase: np.ndarray
    omega: np.ndarray
    w1: np.ndarray
    w2: np.ndarray
    taper: np.ndarray


def virtual_pixel(geom):
    m = geom.sd_mm / geom.so_mm
    return geom.det_width_mm / geom.nu / m, geom.det_height_mm / geom.nv / m


def make_grangeat(geom, n_mu, n_t, j=(5, 5), sigma=2.0, t_pitch_mm=None, t_taper="none"):
    """plan_grangeat (grangeat.py:93-128)."""
    pu, pv = virtual_pixel(geom)
    dt = pu if t_pitch_mm is None else float(t_pitch_mm)
    mu = np.arange(n_mu) * np.pi / n_mu
    omega = 2.0 * np.pi * (np.arange(n_t) - n_t // 2) / (n_t * dt)
    nodes_mm = np.stack([(omega[None, :] * np.cos(mu)[:, None]).ravel(),
                         (omega[None, :] * np.sin(mu)[:, None]).ravel()], axis=-1)
    nodes = wrap(nodes_mm * np.array([pu, pv]))
    plan = make_plan((geom.nu, geom.nv), nodes, sigma, j)
    if t_taper == "hann":
        taper = np.cos(np.pi * omega / (2.0 * np.abs(omega).max())) ** 2
    elif t_taper == "none":
        taper = np.ones(n_t)
    else:
        raise ValueError("t_taper must be 'none' or 'hann'")
    u = (np.arange(geom.nu) - geom.nu / 2.0 + 0.5) * pu
    v = (np.arange(geom.nv) - geom.nv / 2.0 + 0.5) * pv
    so = geom.so_mm
    w1 = so / np.sqrt(so ** 2 + u[:, None] ** 2 + v[None, :] ** 2)
    t = (np.arange(n_t) - n_t // 2) * dt
    w2 = (so ** 2 + t ** 2) / so ** 2
    return Grangeat(geom, n_mu, n_t, dt, plan, centre_phase(nodes, (geom.nu, geom.nv)),
                    omega, w1, w2, taper)


def grangeat_forward(frame, gp: Grangeat):
    """forward_grangeat_view values (grangeat.py:131-146)."""
    pu, pv = virtual_pixel(gp.geom)
    s = type2(gp.plan, (np.asarray(frame) * gp.w1).astype(np.complex128))
    s = (s * gp.cphase * (pu * pv)).reshape(gp.n_mu, gp.n_t) * (1j * gp.omega[None, :])
    return np.real(centred_ifft(s, axis=1) / gp.dt) * gp.w2[None, :]


def grangeat_reverse(values, gp: Grangeat):
    """reverse_grangeat_view data (grangeat.py:149-170)."""
    ds = np.asarray(values) / gp.w2[None, :]
    s = centred_fft(ds.astype(np.complex128), axis=1) * gp.dt
    c2 = 1.0 / (2.0 * gp.n_mu * gp.n_t * gp.dt)
    y = s * (-1j * np.sign(gp.omega) * gp.taper)[None, :] * c2
    g = np.real(type1(gp.plan, y.ravel() * np.conj(gp.cphase))) / gp.w1
    ring = np.zeros(g.shape, dtype=bool)
    ring[0, :] = ring[-1, :] = ring[:, 0] = ring[:, -1] = True
    return g - np.mean(g[ring])


# --------------------------------------------------------------------------
# End-to-end operators   (pipeline.py:122-212)
# --------------------------------------------------------------------------

def _cfg_dt(geom, cfg):
    return virtual_pixel(geom)[0] if cfg.t_pitch_mm is None else float(cfg.t_pitch_mm)


def forward_project(vol, voxel_mm, geom, cfg, target_batch=None, views=None):
    """nufft_forward_project, methods A and B (pipeline.py:122-147) -> (V, nu, nv).

    ``views`` restricts the output to a subset of the views (bounded CPU
    samples); each batch still uses the reference's batch boundaries.
    """
    if cfg.method not in ("a", "b"):
        raise ValueError("method must be 'a' or 'b'")
    spec = cfg.radial_spec
    lattice = radial_lattice(np.asarray(vol, dtype=np.float64), voxel_mm, spec,
                             cfg.spectrum_j, cfg.oversample_factor, cfg.basis)
    dt = _cfg_dt(geom, cfg)
    gp = make_grangeat(geom, cfg.n_mu, cfg.n_t, t_pitch_mm=cfg.t_pitch_mm, t_taper=cfg.t_taper)
    per_view = cfg.n_mu * cfg.n_t
    frames = {}
    for batch in view_batches(geom.n_views, per_view, target_batch):
        if views is not None and not any(k in views for k in batch):
            continue
        targets, valid = umbrella_targets(geom, spec, batch, cfg.n_mu, cfg.n_t, dt)
        if cfg.method == "b":
            vals = np.real(resample_b_forward(spec, targets, lattice, cfg.rho_pad, cfg.side_lobes))
        else:
            rs = make_resampler(spec, targets, cfg.rho_pad, cfg.resample_j, cfg.oversample_factor)
            vals = np.real(resample_forward(rs, lattice))
        vals[~valid] = 0.0
        for i, k in enumerate(batch):
            if views is not None and k not in views:
                continue
            v = vals[i * per_view:(i + 1) * per_view].reshape(cfg.n_mu, cfg.n_t)
            frames[k] = grangeat_reverse(v, gp) * cfg.normalization
    keys = sorted(frames)
    return np.stack([frames[k] for k in keys])


def backproject(frames, geom, cfg, out_size, voxel_mm, target_batch=None):
    """nufft_backproject, methods A and B (pipeline.py:150-212) -> (N, N, N) real."""
    if cfg.method not in ("a", "b"):
        raise ValueError("method must be 'a' or 'b'")
    frames = np.asarray(frames)
    extent = out_size * voxel_mm

    class _Spec:
        pass
    spec = _Spec()
    spec.n_rho = 2 * int(np.ceil(1.5 * out_size / 2.0))
    spec.n_theta = int(cfg.radial_spec.n_theta)
    spec.n_phi = int(cfg.radial_spec.n_phi)
    spec.rho_max = extent * np.sqrt(3.0) / 2.0
    n_t = 2 * geom.nu
    pad = min(spec.n_rho // 8, 32)
    gp = make_grangeat(geom, cfg.n_mu, n_t, t_pitch_mm=None)
    dt = gp.dt
    shape = (spec.n_rho, spec.n_theta, spec.n_phi)
    num = np.zeros(shape, dtype=np.complex128)
    den = np.zeros(shape)
    for batch in view_batches(geom.n_views, cfg.n_mu * n_t, target_batch):
        vals = np.concatenate([grangeat_forward(frames[k], gp).ravel() for k in batch])
        targets, valid = umbrella_targets(geom, spec, batch, cfg.n_mu, n_t, dt)
        vals = np.where(valid, vals, 0.0)
        if cfg.method == "b":
            num += resample_b_adjoint(spec, targets, vals.astype(np.complex128), pad, cfg.side_lobes)
            den += np.real(resample_b_adjoint(spec, targets, valid.astype(np.complex128), pad,
                                              cfg.side_lobes))
        else:
            rs = make_resampler(spec, targets, pad, cfg.resample_j, cfg.oversample_factor)
            num += resample_adjoint(rs, vals.astype(np.complex128))
            den += np.real(resample_adjoint(rs, valid.astype(np.complex128)))
    keep = den > cfg.den_tol * den.max()
    lat = np.where(keep, num / np.where(keep, den, 1.0), 0.0)
    n_r, n_th, n_ph, _, d_rho, theta, _ = spec_arrays(spec)
    s = centred_fft(lat.astype(np.complex128), axis=0) * d_rho
    om = radial_omega(n_r, d_rho)
    c3 = 1.0 / (4.0 * n_th * n_ph * n_r * d_rho)
    corner = np.pi * np.sqrt(3.0) / voxel_mm
    apod = np.cos(np.pi * np.minimum(np.abs(om) / corner, 1.0) / 2.0) ** 2
    s = s * (-1j * om * apod * c3)[:, None, None] * np.sin(theta)[None, :, None]
    if cfg.basis == "trilinear":
        s = s * trilinear_transfer(spec, voxel_mm)
    nodes = wrap(radial_direction_nodes(spec, voxel_mm))
    y = s.transpose(2, 1, 0).ravel() * np.conj(centre_phase(nodes, (out_size,) * 3))
    grid = type1_chunked((out_size,) * 3, nodes, y, cfg.oversample_factor, cfg.spectrum_j)
    return np.real(grid) * cfg.bp_normalization
