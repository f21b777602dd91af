"""Comparison-baseline cone-beam projector on the device (drop-in for
``cbnufft.baseline.ct_project_linear``, baseline.py:52-98).

Ray-driven projection with trilinear volume sampling: every ray takes N
midpoint samples over its chord through the volume cube, each scaled by the
step length (``cbn_ct_project_linear``).  The backprojector calibration
(``pipeline.calibrate_bp_normalization``) runs it.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _device, _lib
from .grangeat import DetectorFrame
from .phantom import Volume3D


def detector_axes_physical(geom):
    """Physical detector pixel-centre coordinates (u, v) in mm (baseline.py:20-25)."""
    pu, pv = geom.pixel_mm
    u = (np.arange(geom.nu) - geom.nu / 2.0 + 0.5) * pu
    v = (np.arange(geom.nv) - geom.nv / 2.0 + 0.5) * pv
    return u, v


def ct_project_linear(vol: Volume3D, geom, counter: dict | None = None) -> list[DetectorFrame]:
    """list[DetectorFrame] of every view (view order); `counter['mults']` counts
    8 N multiplies per ray as the reference does."""
    t = _device.require_cuda()
    from .pipeline import _geometry_struct
    n = vol.n
    vd = t.from_numpy(np.ascontiguousarray(vol.data, dtype=np.float32)).cuda()
    out = t.empty((geom.n_views, geom.nu, geom.nv), dtype=t.float32, device="cuda")
    g = _geometry_struct(geom)
    _lib.check(_lib.load().cbn_ct_project_linear(
        ctypes.byref(g), ctypes.c_void_p(vd.data_ptr()), int(n), float(vol.voxel_mm),
        ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(_device.stream_ptr())),
        "ct_project_linear")
    if counter is not None:
        counter["mults"] = counter.get("mults", 0) + 8 * n * geom.nu * geom.nv * geom.n_views
    host = out.cpu().numpy().astype(np.float64)
    return [DetectorFrame(k, host[k], geom.pixel_mm) for k in range(geom.n_views)]
