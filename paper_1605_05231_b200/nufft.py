"""Gridding NUFFT on the B200 (drop-in for ``cbnufft/nufft.py``).

Same public names, signatures, argument meaning and ``ValueError``
behaviour as the reference (nufft.py:28-282).  ``plan_nufft`` uploads the
nodes and fits the least-squares deapodisation on the device;
``nufft_forward`` / ``nufft_adjoint`` run deapodise+pad -> cuFFT -> KB gather
(type 2) and KB spread -> cuFFT -> crop+deapodise (type 1) through the C ABI.

Host arrays in, host arrays out (complex128, like the reference); torch CUDA
tensors in, torch CUDA tensors (complex64) out, with no host round trip.

Small host utilities that are not on the hot path (``kaiser_bessel``,
``kaiser_bessel_ft``, ``dirichlet``, ``sinc_resample``, ``wrap_nodes``) are
kept for API completeness.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _device, _hostio, _lib

_CHUNK = 1 << 19        # kept for API parity (the device path has no row chunks)
_PLAN_CHUNK = 1 << 21   # nodes per sub-plan in the *_chunked variants (nufft.py:24)
_WORKERS = 1


def set_threads(k: int) -> None:
    """Reference FFT worker knob (nufft.py:28-33); validated, no effect on the GPU."""
    global _WORKERS
    if int(k) < 1:
        raise ValueError("thread count must be >= 1")
    _WORKERS = int(k)


def kaiser_bessel(u, j: int, beta: float):
    from scipy.special import i0
    u = np.asarray(u, dtype=np.float64)
    t = 1.0 - (2.0 * u / j) ** 2
    return np.where(t > 0.0, i0(beta * np.sqrt(np.maximum(t, 0.0))), 0.0)


def kaiser_bessel_ft(nu, j: int, beta: float):
    nu = np.asarray(nu, dtype=np.float64)
    z = np.lib.scimath.sqrt(beta ** 2 - (np.pi * j * nu) ** 2)
    safe = np.where(z == 0, 1.0, z)
    return j * np.real(np.where(np.abs(z) < 1e-12, 1.0, np.sinh(z) / safe))


def _beatty_beta(j: int, alpha: float) -> float:
    return float(_lib.load().cbn_beatty_beta(int(j), float(alpha)))


def wrap_nodes(nodes: np.ndarray) -> np.ndarray:
    nodes = np.atleast_2d(np.asarray(nodes, dtype=np.float64))
    if not np.all(np.isfinite(nodes)):
        raise ValueError("nodes must be finite")
    return np.mod(nodes + np.pi, 2.0 * np.pi) - np.pi


def dirichlet(t, n: int):
    t = np.asarray(t, dtype=np.float64)
    den = n * np.sin(np.pi * t / n)
    near = np.abs(den) < 1e-9
    ratio = np.where(near, np.cos(np.pi * t) / np.cos(np.pi * t / n),
                     np.sin(np.pi * t) / np.where(near, 1.0, den))
    return np.exp(1j * np.pi * t * (n - 1) / n) * ratio


def sinc_resample(y: np.ndarray, positions) -> np.ndarray:
    y = np.asarray(y)
    pos = np.asarray(positions, dtype=np.float64)
    if y.ndim == 1 and pos.ndim == 1:
        pos = pos[:, None]
    pos = np.atleast_2d(pos)
    if pos.shape[1] != y.ndim:
        raise ValueError("positions must have one coordinate per signal axis")
    out = y.astype(np.complex128)
    # contract one axis at a time from the last
    mats = [dirichlet(pos[:, a:a + 1] - np.arange(k)[None, :], k) for a, k in enumerate(y.shape)]
    res = np.empty(pos.shape[0], dtype=np.complex128)
    for i in range(pos.shape[0]):
        v = out
        for a in reversed(range(y.ndim)):
            v = v @ mats[a][i]
        res[i] = v
    return res


@dataclass
class NufftPlan:
    """Device plan (nufft.py:88-101).  ``scaling``, ``nodes`` and ``phase`` are
    materialised on request; the dense interpolator of the reference is not
    formed (weights are recomputed in the kernels)."""

    dims: tuple
    k_dims: tuple
    j: tuple
    beta: tuple
    n_nodes: int
    _handle: int = 0

    def __del__(self):
        h, self._handle = self._handle, 0
        lib = getattr(_lib, "_lib", None) if _lib is not None else None
        if h and lib is not None:
            lib.cbn_nufft_destroy(ctypes.c_void_p(h))

    @property
    def handle(self):
        return ctypes.c_void_p(self._handle)

    def axis_scaling(self) -> list[np.ndarray]:
        out = np.empty(int(sum(self.dims)))
        _lib.check(_lib.load().cbn_nufft_scaling(self.handle, out.ctypes.data_as(_lib.P_f64)))
        parts, o = [], 0
        for n in self.dims:
            parts.append(out[o:o + n].copy())
            o += n
        return parts

    @property
    def scaling(self) -> np.ndarray:
        parts = self.axis_scaling()
        s = parts[0]
        for p in parts[1:]:
            s = np.multiply.outer(s, p)
        return s.ravel()

    @property
    def nodes(self) -> np.ndarray:
        out = np.empty((self.n_nodes, len(self.dims)))
        _lib.check(_lib.load().cbn_nufft_wrapped_nodes(self.handle, out.ctypes.data_as(_lib.P_f64)))
        return out

    @property
    def phase(self) -> np.ndarray:
        centers = np.array([n // 2 for n in self.dims], dtype=np.float64)
        return np.exp(-1j * (self.nodes @ centers))

    def first_indices(self) -> np.ndarray:
        """(m, d) int32 first tap index mod K per axis (the bin index)."""
        out = np.empty((self.n_nodes, len(self.dims)), dtype=np.int32)
        _lib.check(_lib.load().cbn_nufft_first_indices(
            self.handle, out.ctypes.data_as(_lib.P_i32), ctypes.c_void_p(_device.stream_ptr())))
        return out


def plan_nufft(dims, nodes, oversample_factor: float = 2.0, j=6) -> NufftPlan:
    """Device plan for uniform dims and frequency nodes (nufft.py:137-218).

    float32 nodes stay float32 on the device (wrapped in float64 inside the
    kernels), which gives the same plan as their float64 copy at half the
    storage -- the path the 100M-node stress configuration uses."""
    dims = tuple(int(d) for d in np.atleast_1d(dims))
    if oversample_factor < 1.0:
        raise ValueError("oversample_factor must be >= 1")
    f32 = isinstance(nodes, np.ndarray) and nodes.dtype == np.float32
    nodes = np.asarray(nodes, dtype=np.float32 if f32 else np.float64)
    if nodes.ndim == 1:
        nodes = nodes[:, None]
    nodes = np.atleast_2d(nodes)
    if not np.all(np.isfinite(nodes)):
        raise ValueError("nodes must be finite")
    d = len(dims)
    if nodes.shape[1] != d:
        raise ValueError(f"nodes must have {d} coordinates per row")
    taps = np.broadcast_to(np.atleast_1d(j), (d,)).astype(int)
    if np.any(taps < 1):
        raise ValueError("tap counts must be >= 1")
    mult = int(np.ceil(oversample_factor - 1e-12))
    k_dims = tuple(n * mult for n in dims)
    betas = tuple(_beatty_beta(int(t), k / n) for t, k, n in zip(taps, k_dims, dims))
    m = nodes.shape[0]
    lib = _lib.load()
    _device.require_cuda()
    rows, rows_p = _lib.i64_array(_device.ls_rows(m))
    dims_a, dims_p = _lib.i64_array(dims)
    taps_a = np.ascontiguousarray(taps, dtype=np.int32)
    h = ctypes.c_void_p()
    if f32:
        nodes_a = np.ascontiguousarray(nodes)
        _lib.check(lib.cbn_nufft_create_f32(
            ctypes.byref(h), d, dims_p, taps_a.ctypes.data_as(_lib.P_i32), float(oversample_factor),
            ctypes.c_void_p(nodes_a.ctypes.data), m, rows_p, rows.size,
            ctypes.c_void_p(_device.stream_ptr())), "plan_nufft")
    else:
        nodes_a, nodes_p = _lib.f64_array(nodes)
        _lib.check(lib.cbn_nufft_create(
            ctypes.byref(h), d, dims_p, taps_a.ctypes.data_as(_lib.P_i32), float(oversample_factor),
            nodes_p, m, rows_p, rows.size, ctypes.c_void_p(_device.stream_ptr())), "plan_nufft")
    return NufftPlan(dims, k_dims, tuple(int(t) for t in taps), betas, m, h.value)


# pinned staging of the host-array calls (complex128 numpy in and out, like
# the reference): native threaded conversions, chunked DMA (_hostio)
_STAGE = _hostio.Staging(single_shape=True)


def _input(x, dtype):
    """The device copy of an operator input: torch tensors as they are, numpy
    through the pinned staging."""
    t = _device.require_cuda()
    if isinstance(x, t.Tensor):
        return _device.to_device(x, dtype)
    arr = np.ascontiguousarray(np.asarray(x))
    if arr.ndim == 0 or arr.size == 0:
        return _device.to_device(arr, dtype)
    return _hostio.upload(_STAGE, "in", arr, dtype)


def _as_result(out, host: bool):
    if not host:
        return out
    if out.numel() == 0 or out.dim() == 0:
        return out.cpu().numpy().astype(np.complex128)
    return _hostio.download(_STAGE, "out", out, np.complex128)


def nufft_forward(plan: NufftPlan, x):
    """Uniform grid -> values at the nodes (nufft.py:221-233)."""
    t = _device.require_cuda()
    host = not isinstance(x, t.Tensor)
    shape = tuple(x.shape)
    if shape != plan.dims:
        raise ValueError(f"input shape {shape} does not match plan dims {plan.dims}")
    xd = _input(x, t.complex64)
    y = t.empty(plan.n_nodes, dtype=t.complex64, device="cuda")
    _lib.check(_lib.load().cbn_nufft_type2(plan.handle, _device.ptr(xd), _device.ptr(y),
                                           ctypes.c_void_p(_device.stream_ptr())), "nufft_forward")
    return _as_result(y, host)


def nufft_adjoint(plan: NufftPlan, y):
    """Exact conjugate transpose of nufft_forward (nufft.py:236-247)."""
    t = _device.require_cuda()
    host = not isinstance(y, t.Tensor)
    if tuple(y.shape) != (plan.n_nodes,):
        raise ValueError(f"expected {plan.n_nodes} node values, got {tuple(y.shape)}")
    yd = _input(y, t.complex64)
    x = t.empty(plan.dims, dtype=t.complex64, device="cuda")
    _lib.check(_lib.load().cbn_nufft_type1(plan.handle, _device.ptr(yd), _device.ptr(x),
                                           ctypes.c_void_p(_device.stream_ptr())), "nufft_adjoint")
    return _as_result(x, host)


def nufft_forward_chunked(dims, nodes, x, oversample_factor: float = 2.0, j=6):
    """Sub-plans of _PLAN_CHUNK nodes, each with its own scaling fit (nufft.py:250-265)."""
    t = _device.require_cuda()
    nodes = np.atleast_2d(np.asarray(nodes, dtype=np.float64))
    host = not isinstance(x, t.Tensor)
    xd = _device.to_device(x, t.complex64)
    out = t.empty(nodes.shape[0], dtype=t.complex64, device="cuda")
    for lo in range(0, nodes.shape[0], _PLAN_CHUNK):
        hi = min(lo + _PLAN_CHUNK, nodes.shape[0])
        plan = plan_nufft(dims, nodes[lo:hi], oversample_factor, j)
        out[lo:hi] = nufft_forward(plan, xd)
    return _as_result(out, host)


def nufft_adjoint_chunked(dims, nodes, y, oversample_factor: float = 2.0, j=6):
    """Sum of the sub-plan adjoints (nufft.py:268-282)."""
    t = _device.require_cuda()
    nodes = np.atleast_2d(np.asarray(nodes, dtype=np.float64))
    m = nodes.shape[0]
    if tuple(y.shape) != (m,):
        raise ValueError(f"expected {m} node values, got {tuple(y.shape)}")
    host = not isinstance(y, t.Tensor)
    yd = _device.to_device(y, t.complex64)
    dims = tuple(int(d) for d in np.atleast_1d(dims))
    acc = t.zeros(dims, dtype=t.complex64, device="cuda")
    for lo in range(0, m, _PLAN_CHUNK):
        hi = min(lo + _PLAN_CHUNK, m)
        acc += nufft_adjoint(plan_nufft(dims, nodes[lo:hi], oversample_factor, j), yd[lo:hi])
    return _as_result(acc, host)
