"""Radial -> umbrella resampling (drop-in for ``cbnufft/resampling.py``).

``plan_resample`` builds a device plan (``cbn_resample_*``).  Method A: a NUFFT
plan on the rho-padded lattice at nodes -2 pi pos / padded with the
reference's own least-squares scaling; ``resample_apply`` /
``resample_transpose`` run the origin average, padding, FFTs and the J=3
gather / spread on the device.  Method B: truncated centred periodic-sinc taps
(side_lobes + 1 per axis) applied to the padded lattice directly
(resampling.py:126-161,176-189).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _device, _lib
from .geometry import canonical_polar, spec_tuple


def polar_index_map(coords, spec) -> np.ndarray:
    """(rho, theta, phi) rows -> fractional lattice indices (resampling.py:38-59)."""
    coords = np.atleast_2d(np.asarray(coords, dtype=np.float64))
    if coords.shape[-1] != 3:
        raise ValueError("coords must have rows (rho, theta, phi)")
    n_r, n_t, n_p, rmax = spec_tuple(spec)
    rho, theta, phi = canonical_polar(coords[:, 0], coords[:, 1], coords[:, 2])
    if np.any(np.abs(rho) > rmax * (1.0 + 1e-12)):
        raise ValueError("rho outside the radial grid support")
    i_rho = rho / spec.delta_rho + n_r / 2.0
    i_theta = theta * n_t / np.pi
    i_phi = phi * n_p / (2.0 * np.pi)
    top = i_rho >= n_r - 1e-9
    return np.stack([np.where(top, 0.0, i_rho),
                     np.where(top, np.mod(n_t - i_theta, n_t), i_theta),
                     np.where(top, np.mod(i_phi + n_p / 2.0, n_p), i_phi)], axis=-1)


@dataclass
class ResamplePlan:
    """Prepared resampling operator (resampling.py:62-76)."""

    method: str
    spec: object
    targets: np.ndarray
    rho_pad: int
    side_lobes: int = 2
    padded_dims: tuple = field(default=())
    _handle: int = 0

    @property
    def n_targets(self) -> int:
        return self.targets.shape[0]

    def __del__(self):
        h, self._handle = self._handle, 0
        if h and _lib._lib is not None:
            _lib._lib.cbn_resample_destroy(ctypes.c_void_p(h))


def plan_resample(spec, targets, method: str = "a", rho_pad: int | None = None, j=(3, 3, 3),
                  oversample_factor: float = 2.0, side_lobes: int = 2) -> ResamplePlan:
    """resampling.py:79-103."""
    method = method.lower()
    if method not in ("a", "b"):
        raise ValueError("method must be 'a' or 'b'")
    targets = np.atleast_2d(np.asarray(targets, dtype=np.float64))
    if targets.shape[-1] != 3:
        raise ValueError("targets must be (m, 3) fractional indices")
    n_r, n_t, n_p, _ = spec_tuple(spec)
    lim = np.array([n_r, n_t, n_p], dtype=np.float64)
    if np.any(targets < -1e-9) or np.any(targets >= lim + 1e-9):
        raise ValueError("targets must be wrapped into the lattice index range")
    if rho_pad is None:
        rho_pad = n_r // 2
    padded = (n_r + 2 * rho_pad, n_t, n_p)
    plan = ResamplePlan(method, spec, targets, int(rho_pad), side_lobes, padded_dims=padded)
    if method == "b":
        if not 0 <= int(side_lobes) <= 7:
            raise ValueError("side_lobes must be 0..7")
        _device.require_cuda()
        tg, tp = _lib.f64_array(targets)
        h = ctypes.c_void_p()
        _lib.check(_lib.load().cbn_resample_create_b(
            ctypes.byref(h), n_r, n_t, n_p, int(rho_pad), int(side_lobes), tp, targets.shape[0],
            ctypes.c_void_p(_device.stream_ptr())), "plan_resample")
        plan._handle = h.value
        return plan
    taps = np.ascontiguousarray(np.broadcast_to(np.atleast_1d(j), (3,)), dtype=np.int32)
    _device.require_cuda()
    rows, rp = _lib.i64_array(_device.ls_rows(targets.shape[0]))
    tg, tp = _lib.f64_array(targets)
    h = ctypes.c_void_p()
    _lib.check(_lib.load().cbn_resample_create(
        ctypes.byref(h), n_r, n_t, n_p, int(rho_pad), taps.ctypes.data_as(_lib.P_i32),
        float(oversample_factor), tp, targets.shape[0], rp, rows.size,
        ctypes.c_void_p(_device.stream_ptr())), "plan_resample")
    plan._handle = h.value
    return plan


def resample_apply(plan: ResamplePlan, data):
    """Complex target values of the full radial lattice (resampling.py:136-161)."""
    t = _device.require_cuda()
    host = not isinstance(data, t.Tensor)
    if tuple(data.shape) != spec_tuple(plan.spec)[:3]:
        raise ValueError("data shape does not match the plan's radial grid")
    x = _device.to_device(data, t.complex64)
    out = t.empty(plan.n_targets, dtype=t.complex64, device="cuda")
    _lib.check(_lib.load().cbn_resample_apply(ctypes.c_void_p(plan._handle), _device.ptr(x),
                                              _device.ptr(out),
                                              ctypes.c_void_p(_device.stream_ptr())),
               "resample_apply")
    return out.cpu().numpy().astype(np.complex128) if host else out


def resample_transpose(plan: ResamplePlan, values):
    """Exact adjoint of resample_apply (resampling.py:164-196)."""
    t = _device.require_cuda()
    host = not isinstance(values, t.Tensor)
    if tuple(values.shape) != (plan.n_targets,):
        raise ValueError(f"expected {plan.n_targets} target values")
    y = _device.to_device(values, t.complex64)
    out = t.empty(spec_tuple(plan.spec)[:3], dtype=t.complex64, device="cuda")
    _lib.check(_lib.load().cbn_resample_transpose(ctypes.c_void_p(plan._handle), _device.ptr(y),
                                                  _device.ptr(out),
                                                  ctypes.c_void_p(_device.stream_ptr())),
               "resample_transpose")
    return out.cpu().numpy().astype(np.complex128) if host else out


def resample_method_a(data, targets, spec, **kwargs) -> np.ndarray:
    return np.real(resample_apply(plan_resample(spec, targets, "a", **kwargs), data))


def resample_method_b(data, targets, spec, **kwargs) -> np.ndarray:
    return np.real(resample_apply(plan_resample(spec, targets, "b", **kwargs), data))
