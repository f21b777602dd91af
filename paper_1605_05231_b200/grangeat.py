"""Per-view Grangeat data types (drop-in for ``cbnufft/grangeat.py`` types).

``DetectorFrame`` and ``UmbrellaView`` keep the reference's fields and
validation (grangeat.py:30-55).  The Grangeat transforms themselves run on the
device inside the projector plan (``csrc/cbn_projector.cu``:
``grangeat_reverse``; ``csrc/cbn_backproject.cu``: forward Grangeat) and are
reachable per view block through ``Projector.grangeat_reverse`` /
``Projector.grangeat_forward`` in ``pipeline.py``.  ``plan_grangeat`` with
any other tap shape or oversampling than the projector's (5, 5), 2 runs the
same transforms through the standalone device NUFFT plus elementwise kernels
(``cbn_lines_*``, ``cbn_line_weight``, ``cbn_node_phase``, ``cbn_radial_fft``).
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
    # general shapes (j != (5, 5) or oversample != 2): the standalone device
    # NUFFT plan over the polar nodes and their centre phases' node set
    nufft_plan: object = None
    nodes: np.ndarray = None


def plan_grangeat(geom, n_mu: int, n_t: int, j=(5, 5), oversample_factor: float = 2.0,
                  t_pitch_mm: float | None = None, t_taper: str = "none") -> GrangeatPlan:
    """grangeat.py:93-128."""
    from .config import ProjectorConfig
    from .geometry import RadialGridSpec, umbrella_line_grid
    from .pipeline import Projector
    if t_taper not in ("none", "hann"):
        raise ValueError("t_taper must be 'none' or 'hann'")
    mu, t = umbrella_line_grid(geom, n_mu, n_t, t_pitch_mm)
    pu, pv = geom.virtual_pixel_mm
    dt = pu if t_pitch_mm is None else float(t_pitch_mm)
    omega = 2.0 * np.pi * (np.arange(n_t) - n_t // 2) / (n_t * dt)
    if t_taper == "hann":
        taper = np.cos(np.pi * omega / (2.0 * np.abs(omega).max())) ** 2
    else:
        taper = np.ones(n_t)
    w1, w2 = grangeat_preweight(geom), grangeat_postweight(geom, t)
    if tuple(np.broadcast_to(np.atleast_1d(j), (2,))) != (5, 5) or float(oversample_factor) != 2.0:
        # any other tap shape / oversampling: the standalone device NUFFT on
        # the polar nodes (grangeat.py:110-118), elementwise steps as kernels
        from .nufft import plan_nufft
        ww, mm = np.meshgrid(omega, mu, indexing="ij")
        nodes_mm = np.stack([(ww * np.cos(mm)).T.ravel(), (ww * np.sin(mm)).T.ravel()], axis=-1)
        nodes = np.mod(nodes_mm * np.array([pu, pv]) + np.pi, 2.0 * np.pi) - np.pi
        plan = plan_nufft((geom.nu, geom.nv), nodes, oversample_factor, j)
        return GrangeatPlan(geom, int(n_mu), int(n_t), dt, omega, w1, w2, taper,
                            nufft_plan=plan, nodes=nodes)
    cfg = ProjectorConfig("a", RadialGridSpec(2, 1, 1, 1.0), n_mu=int(n_mu), n_t=int(n_t),
                          t_pitch_mm=t_pitch_mm, t_taper=t_taper, rho_pad=0)
    proj = Projector(geom, cfg, 2, 1.0, 3, bp_n_t=int(n_t), bp_t_pitch_mm=dt)
    return GrangeatPlan(geom, int(n_mu), int(n_t), dt, omega, w1, w2, taper, proj)


def _forward_general(frame_data, gp: GrangeatPlan) -> np.ndarray:
    """forward_grangeat_view (grangeat.py:131-146) through the standalone NUFFT."""
    import ctypes
    from . import _device, _lib
    from .nufft import nufft_forward
    from .radon_fourier import _phase_on_device
    t = _device.require_cuda()
    lib, s = _lib.load(), ctypes.c_void_p(_device.stream_ptr())
    geom = gp.geom
    pu, pv = geom.virtual_pixel_mm
    f = _device.to_device(np.asarray(frame_data), t.float32)
    h = t.empty((geom.nu, geom.nv), dtype=t.complex64, device="cuda")
    w1 = np.ascontiguousarray(gp.w1, dtype=np.float64).ravel()
    _lib.check(lib.cbn_lines_real_in(_device.ptr(f), 1, w1.size, w1.ctypes.data_as(_lib.P_f64),
                                     _device.ptr(h), s), "forward_grangeat_view")
    sh = nufft_forward(gp.nufft_plan, h)                     # device, node order (mu, t)
    _phase_on_device(sh, gp.nodes, (geom.nu, geom.nv), conj=False,
                     w=np.array([pu * pv]), w_inner=sh.numel())
    iw = np.ascontiguousarray(np.stack([np.zeros(gp.n_t), gp.omega], axis=-1))
    _lib.check(lib.cbn_line_weight(_device.ptr(sh), gp.n_mu, gp.n_t, 1,
                                   iw.ctypes.data_as(_lib.P_f64), s), "forward_grangeat_view")
    _lib.check(lib.cbn_radial_fft(_device.ptr(sh), gp.n_t, gp.n_mu, 1, 1.0 / gp.dt, s),
               "forward_grangeat_view")
    out = t.empty((gp.n_mu, gp.n_t), dtype=t.float32, device="cuda")
    w2 = np.ascontiguousarray(gp.w2, dtype=np.float64)
    _lib.check(lib.cbn_lines_real_out(_device.ptr(sh), gp.n_mu, gp.n_t,
                                      w2.ctypes.data_as(_lib.P_f64), _device.ptr(out), s),
               "forward_grangeat_view")
    return out.cpu().numpy().astype(np.float64)


def _reverse_general(values, gp: GrangeatPlan) -> np.ndarray:
    """reverse_grangeat_view (grangeat.py:149-170) through the standalone NUFFT."""
    import ctypes
    from . import _device, _lib
    from .nufft import nufft_adjoint
    from .radon_fourier import _phase_on_device
    t = _device.require_cuda()
    lib, s = _lib.load(), ctypes.c_void_p(_device.stream_ptr())
    geom = gp.geom
    v = _device.to_device(np.asarray(values), t.float32)
    y = t.empty((gp.n_mu, gp.n_t), dtype=t.complex64, device="cuda")
    inv_w2 = np.ascontiguousarray(1.0 / gp.w2, dtype=np.float64)
    _lib.check(lib.cbn_lines_real_in(_device.ptr(v), gp.n_mu, gp.n_t,
                                     inv_w2.ctypes.data_as(_lib.P_f64), _device.ptr(y), s),
               "reverse_grangeat_view")
    _lib.check(lib.cbn_radial_fft(_device.ptr(y), gp.n_t, gp.n_mu, 0, gp.dt, s),
               "reverse_grangeat_view")
    c2 = 1.0 / (2.0 * gp.n_mu * gp.n_t * gp.dt)
    fw = -1j * np.sign(gp.omega) * gp.taper * c2
    fwc = np.ascontiguousarray(np.stack([fw.real, fw.imag], axis=-1))
    _lib.check(lib.cbn_line_weight(_device.ptr(y), gp.n_mu, gp.n_t, 1,
                                   fwc.ctypes.data_as(_lib.P_f64), s), "reverse_grangeat_view")
    yf = y.reshape(-1)
    _phase_on_device(yf, gp.nodes, (geom.nu, geom.nv), conj=True)
    h = nufft_adjoint(gp.nufft_plan, yf)
    g = t.empty((geom.nu, geom.nv), dtype=t.float32, device="cuda")
    inv_w1 = np.ascontiguousarray(1.0 / gp.w1, dtype=np.float64).ravel()
    _lib.check(lib.cbn_lines_real_out(_device.ptr(h), 1, inv_w1.size,
                                      inv_w1.ctypes.data_as(_lib.P_f64), _device.ptr(g), s),
               "reverse_grangeat_view")
    _lib.check(lib.cbn_frame_ring_center(_device.ptr(g), geom.nu, geom.nv, s),
               "reverse_grangeat_view")
    return g.cpu().numpy().astype(np.float64)


def forward_grangeat_view(frame: DetectorFrame, gp: GrangeatPlan) -> UmbrellaView:
    """Detector frame -> umbrella derivative-Radon values (grangeat.py:131-146)."""
    from .geometry import umbrella_coordinates
    geom = gp.geom
    if tuple(frame.data.shape) != (geom.nu, geom.nv):
        raise ValueError("frame dims do not match the geometry")
    if gp.nufft_plan is not None:
        values = _forward_general(frame.data, gp)
    else:
        vals = gp.projector.grangeat_forward(np.asarray(frame.data, dtype=np.float32)[None])
        values = vals.cpu().numpy()[0].astype(np.float64)
    coords = umbrella_coordinates(geom, frame.view_index, gp.n_mu, gp.n_t, gp.dt)
    return UmbrellaView(frame.view_index, values, coords)


def reverse_grangeat_view(view: UmbrellaView, gp: GrangeatPlan) -> DetectorFrame:
    """Umbrella values -> detector frame (grangeat.py:149-170)."""
    if tuple(view.values.shape) != (gp.n_mu, gp.n_t):
        raise ValueError("umbrella grid does not match the plan")
    if gp.nufft_plan is not None:
        return DetectorFrame(view.view_index, _reverse_general(view.values, gp), gp.geom.pixel_mm)
    out = gp.projector.grangeat_reverse(np.asarray(view.values, dtype=np.float32)[None])
    return DetectorFrame(view.view_index, out.cpu().numpy()[0].astype(np.float64),
                         gp.geom.pixel_mm)
