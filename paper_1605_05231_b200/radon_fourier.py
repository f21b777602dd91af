"""Fourier-slice transforms (drop-in for ``cbnufft/radon_fourier.py``).

Every data pass runs on the device: ``image_to_radial_spectrum`` (3D type-2
NUFFT onto the radial lines through the projector plan), ``radial_fft`` /
``radial_ifft`` (centred cuFFT along rho), the per-rho weights of
``spectral_rho_derivative`` / ``ramp_filter_radial`` and the sinc^2 transfer
(``csrc/cbn_lines.cu``), and the 2D helpers (device NUFFT plans plus the
node-phase kernel).  Only O(n_rho) weight vectors are formed on the host.
Layouts follow the reference: lattices are (n_rho, n_theta, n_phi).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _device, _lib
from .config import ProjectorConfig
from .geometry import ConeGeometry, RadialGridSpec, radial_nodes, spec_tuple


@dataclass
class RadialSpectrum3D:
    """Fourier samples along radial lines, (n_rho, n_theta, n_phi) (radon_fourier.py:20-30)."""

    spec: RadialGridSpec
    data: np.ndarray

    def __post_init__(self):
        want = spec_tuple(self.spec)[:3]
        if tuple(self.data.shape) != want:
            raise ValueError(f"data shape {self.data.shape} != {want}")


@dataclass
class RadialRadon3D:
    """Derivative-of-Radon values on the radial lattice (radon_fourier.py:33-43)."""

    spec: RadialGridSpec
    data: np.ndarray

    def __post_init__(self):
        want = spec_tuple(self.spec)[:3]
        if tuple(self.data.shape) != want:
            raise ValueError(f"data shape {self.data.shape} != {want}")


def radial_omega(spec) -> np.ndarray:
    n_rho = int(spec.n_rho)
    k = np.arange(n_rho) - n_rho // 2
    return 2.0 * np.pi * k / (n_rho * spec.delta_rho)


def _radial_direction_nodes(spec, voxel_mm: float) -> np.ndarray:
    """Unwrapped radial node set, rho fastest (radon_fourier.py:59-67)."""
    omega = radial_omega(spec) * voxel_mm
    polar = radial_nodes(spec)
    st = np.sin(polar[:, 1])
    direction = np.stack([np.cos(polar[:, 2]) * st, np.sin(polar[:, 2]) * st,
                          np.cos(polar[:, 1])], axis=-1)
    return np.tile(omega, int(spec.n_theta) * int(spec.n_phi))[:, None] * direction


def _wrap_nodes(nodes: np.ndarray) -> np.ndarray:
    return np.mod(nodes + np.pi, 2.0 * np.pi) - np.pi


def _center_phase(nodes: np.ndarray, dims) -> np.ndarray:
    shift = np.array([n / 2.0 - 0.5 for n in dims])
    return np.exp(1j * (nodes @ shift))


def _to_lattice(node_order: np.ndarray, spec) -> np.ndarray:
    n_r, n_t, n_p, _ = spec_tuple(spec)
    return node_order.reshape(n_p, n_t, n_r).transpose(2, 1, 0)


def trilinear_transfer(spec, voxel_mm: float) -> np.ndarray:
    """sinc^2 transfer of the trilinear voxel basis (radon_fourier.py:75-86), device kernel."""
    t = _device.require_cuda()
    n_r, n_t, n_p, _ = spec_tuple(spec)
    out = t.empty((n_p, n_t, n_r), dtype=t.float64, device="cuda")
    _lib.check(_lib.load().cbn_trilinear_transfer(n_r, n_t, n_p, float(spec.delta_rho),
                                                  float(voxel_mm), _device.ptr(out),
                                                  ctypes.c_void_p(_device.stream_ptr())),
               "trilinear_transfer")
    return _to_lattice(out.cpu().numpy().reshape(-1), spec)


def _rho_weighted(data, w: np.ndarray) -> np.ndarray:
    """data (n_rho, ...) complex times w[rho] (complex), on the device."""
    t = _device.require_cuda()
    arr = np.asarray(data)
    x = _device.to_device(arr, t.complex64).contiguous()
    n = arr.shape[0]
    inner = int(np.prod(arr.shape[1:])) if arr.ndim > 1 else 1
    wc = np.ascontiguousarray(np.stack([np.real(w), np.imag(w)], axis=-1), dtype=np.float64)
    _lib.check(_lib.load().cbn_line_weight(_device.ptr(x), 1, n, inner,
                                           wc.ctypes.data_as(_lib.P_f64),
                                           ctypes.c_void_p(_device.stream_ptr())), "line weight")
    return x.cpu().numpy().astype(np.complex128)


def _spectrum_projector(n: int, voxel_mm: float, spec, j, oversample_factor):
    from .pipeline import Projector
    geom = ConeGeometry(1.0e6, 2.0e6, 1.0, 1.0, 1, 1, 1, 1.0)
    cfg = ProjectorConfig("a", spec, n_mu=1, n_t=2, spectrum_j=int(j),
                          oversample_factor=float(oversample_factor), rho_pad=0)
    return Projector(geom, cfg, n, voxel_mm, 1)


def image_to_radial_spectrum(vol, spec, j=6, oversample_factor: float = 2.0) -> RadialSpectrum3D:
    """3D NUFFT of the volume at the radial node set (radon_fourier.py:89-108)."""
    t = _device.require_cuda()
    proj = _spectrum_projector(vol.data.shape[0], vol.voxel_mm, spec, j, oversample_factor)
    v = _device.to_device(vol.data, t.float32)
    n_r, n_t, n_p, _ = spec_tuple(spec)
    out = t.empty((n_p, n_t, n_r), dtype=t.complex64, device="cuda")
    _lib.check(_lib.load().cbn_projector_radial_spectrum(proj._h, _device.ptr(v), _device.ptr(out),
                                                         proj._s), "image_to_radial_spectrum")
    data = out.permute(2, 1, 0).cpu().numpy().astype(np.complex128)
    return RadialSpectrum3D(spec, data)


def spectral_rho_derivative(s: RadialSpectrum3D) -> RadialSpectrum3D:
    """x i*omega_rho along rho (radon_fourier.py:111-114), device kernel."""
    return RadialSpectrum3D(s.spec, _rho_weighted(s.data, 1j * radial_omega(s.spec)))


def _radial_transform(data, spec, inverse: bool, scale: float) -> np.ndarray:
    t = _device.require_cuda()
    n_r, n_t, n_p, _ = spec_tuple(spec)
    x = _device.to_device(np.asarray(data).transpose(2, 1, 0), t.complex64).contiguous()
    _lib.check(_lib.load().cbn_radial_fft(_device.ptr(x), n_r, n_t * n_p, 1 if inverse else 0,
                                          float(scale), ctypes.c_void_p(_device.stream_ptr())),
               "radial_fft")
    return x.permute(2, 1, 0).cpu().numpy().astype(np.complex128)


def radial_fft(r: RadialRadon3D) -> RadialSpectrum3D:
    """Centred FFT along rho times d_rho (radon_fourier.py:127-130)."""
    return RadialSpectrum3D(r.spec, _radial_transform(r.data, r.spec, False, r.spec.delta_rho))


def radial_ifft(s: RadialSpectrum3D) -> RadialRadon3D:
    """Centred IFFT along rho over d_rho (radon_fourier.py:133-135)."""
    return RadialRadon3D(s.spec, _radial_transform(s.data, s.spec, True, 1.0 / s.spec.delta_rho))


def ramp_weights(n_rho: int, delta_rho: float, n_theta: int, dimension: int,
                 n_phi: int = 1) -> np.ndarray:
    """radon_fourier.py:138-158."""
    if dimension not in (2, 3):
        raise ValueError("dimension must be 2 or 3")
    omega = 2.0 * np.pi * (np.arange(n_rho) - n_rho // 2) / (n_rho * delta_rho)
    dw = 2.0 * np.pi / (n_rho * delta_rho)
    if dimension == 2:
        c = 1.0 / (2.0 * n_theta * n_rho * delta_rho)
        w = c * np.abs(omega)
        w[n_rho // 2] = 0.25 * c * dw
    else:
        c = 1.0 / (4.0 * n_theta * n_phi * n_rho * delta_rho)
        w = c * omega ** 2
        w[n_rho // 2] = 0.25 * c * dw ** 2
    return w


def ramp_filter_radial(s: RadialSpectrum3D, dimension: int) -> RadialSpectrum3D:
    """Ramp weights along rho (radon_fourier.py:160-164), device kernel."""
    w = ramp_weights(int(s.spec.n_rho), s.spec.delta_rho, int(s.spec.n_theta), dimension,
                     int(s.spec.n_phi))
    return RadialSpectrum3D(s.spec, _rho_weighted(s.data, w.astype(np.complex128)))


def _polar_nodes_2d(n: int, n_rho: int, n_theta: int):
    delta_rho = 2.0 * n / n_rho
    omega = 2.0 * np.pi * (np.arange(n_rho) - n_rho // 2) / (n_rho * delta_rho)
    theta = np.arange(n_theta) * np.pi / n_theta
    ww, tt = np.meshgrid(omega, theta, indexing="ij")
    return np.stack([(ww * np.cos(tt)).ravel(), (ww * np.sin(tt)).ravel()], axis=-1), delta_rho


def _phase_on_device(values, nodes: np.ndarray, n, conj: bool, w=None, w_inner: int = 1):
    """values (device complex64) *= exp(+-i nodes . shift) [* w[i // w_inner]] in place;
    shift = dims / 2 - 1/2 (_center_phase), n an edge or the dims."""
    dims = (n, n) if np.isscalar(n) else tuple(n)
    shift = np.array([d / 2.0 - 0.5 for d in dims], dtype=np.float64)
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    wp = None
    if w is not None:
        w = np.ascontiguousarray(w, dtype=np.float64)
        wp = w.ctypes.data_as(_lib.P_f64)
    _lib.check(_lib.load().cbn_node_phase(_device.ptr(values), nodes.ctypes.data_as(_lib.P_f64),
                                          nodes.shape[0], nodes.shape[1],
                                          shift.ctypes.data_as(_lib.P_f64), 1 if conj else 0, wp,
                                          int(w_inner), ctypes.c_void_p(_device.stream_ptr())),
               "center phase")
    return values


def image_to_radial_spectrum_2d(image, n_rho: int, n_theta: int, j=6,
                                oversample_factor: float = 2.0) -> np.ndarray:
    """2D NUFFT onto radial lines (radon_fourier.py:168-188), device NUFFT + phase."""
    from .nufft import nufft_forward, plan_nufft
    t = _device.require_cuda()
    image = np.asarray(image)
    if image.ndim != 2 or image.shape[0] != image.shape[1]:
        raise ValueError("image must be square")
    n = image.shape[0]
    nodes, _ = _polar_nodes_2d(n, n_rho, n_theta)
    values = nufft_forward(plan_nufft((n, n), nodes, oversample_factor, j),
                           _device.to_device(image, t.complex64))
    _phase_on_device(values, nodes, n, conj=False)
    return values.cpu().numpy().astype(np.complex128).reshape(n_rho, n_theta)


def fbp2d_nufft(spectrum, out_size: int, j=6, oversample_factor: float = 2.0):
    """2D NUFFT filtered backprojection (radon_fourier.py:191-213), device NUFFT + ramp."""
    from .nufft import nufft_adjoint, plan_nufft
    t = _device.require_cuda()
    spectrum = np.asarray(spectrum)
    if spectrum.ndim != 2:
        raise ValueError("spectrum must be (n_rho, n_theta)")
    n_rho, n_theta = spectrum.shape
    n = int(out_size)
    nodes, delta_rho = _polar_nodes_2d(n, n_rho, n_theta)
    w = ramp_weights(n_rho, delta_rho, n_theta, 2)
    y = _device.to_device(spectrum.reshape(-1), t.complex64)
    _phase_on_device(y, nodes, n, conj=True, w=w, w_inner=n_theta)
    grid = nufft_adjoint(plan_nufft((n, n), nodes, oversample_factor, j), y)
    g = grid.cpu().numpy()
    re = g.real.astype(np.float64)
    real_norm = float(np.linalg.norm(re))
    return re, float(np.linalg.norm(g.imag.astype(np.float64))) / max(real_norm, 1e-300)
