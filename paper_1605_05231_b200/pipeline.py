"""End-to-end NUFFT cone-beam operators on the B200 (drop-in for
``cbnufft/pipeline.py:1-212``).

``nufft_forward_project(vol, geom, cfg)`` and
``nufft_backproject(frames, geom, cfg, out_size, voxel_mm)`` keep the
reference's signatures, return types (``list[DetectorFrame]``,
``Volume3D``), view batching (``_TARGET_BATCH``, read at call time like the
reference module global) and exceptions (``ValueError`` for a frame-count
mismatch, ``FloatingPointError`` for non-finite projections).  The whole chain
runs in one C-ABI call per operator (``cbn_forward_project`` /
``cbn_backproject``); there is no host compute path.

``Projector`` exposes the same device plan with torch CUDA tensors in and out
(no host round trip) plus the stage entry points used by the parity tests.
"""

from __future__ import annotations

import ctypes
import os
from collections import OrderedDict

import numpy as np

from . import _device, _hostio, _lib
from .config import ProjectorConfig, make_projector_config  # noqa: F401  (API re-export)
from .geometry import ConeGeometry, RadialGridSpec  # noqa: F401
from .grangeat import DetectorFrame, UmbrellaView  # noqa: F401
from .phantom import Volume3D

_TARGET_BATCH = 1 << 20   # umbrella targets per resampling plan (pipeline.py:28)

_FORWARD, _BACK = 1, 2
# the drop-in forward call pads and 2D-transforms each uploaded chunk of the
# volume at once (cbn_forward_stage_volume); CBN_STAGE_VOLUME=0: plain call
_STAGE_VOLUME = os.environ.get("CBN_STAGE_VOLUME", "1") != "0"
_CACHE: "OrderedDict[tuple, Projector]" = OrderedDict()
_CACHE_SIZE = 2


def _geometry_struct(geom) -> _lib.Geometry:
    return _lib.Geometry(float(geom.so_mm), float(geom.sd_mm), float(geom.det_width_mm),
                         float(geom.det_height_mm), int(geom.nu), int(geom.nv),
                         int(geom.n_views), float(geom.object_extent_mm))


def _config_struct(cfg, target_batch: int, plan_chunk: int) -> _lib.ProjectorConfig:
    method = str(cfg.method).lower()
    if method not in ("a", "b"):
        raise ValueError("method must be 'a' or 'b'")
    if method == "b" and not 0 <= int(cfg.side_lobes) <= 7:
        raise ValueError("side_lobes must be 0..7")
    if cfg.t_taper not in ("none", "hann"):
        raise ValueError("t_taper must be 'none' or 'hann'")
    if cfg.basis not in ("trilinear", "dirac"):
        raise ValueError("basis must be 'trilinear' or 'dirac'")
    rj = np.broadcast_to(np.atleast_1d(cfg.resample_j), (3,)).astype(int)
    spec = cfg.radial_spec
    c = _lib.ProjectorConfig()
    c.method = 0 if method == "a" else 1
    c.spec = _lib.RadialSpec(int(spec.n_rho), int(spec.n_theta), int(spec.n_phi),
                             float(spec.rho_max))
    c.n_mu = int(cfg.n_mu)
    c.n_t = int(cfg.n_t)
    c.t_pitch_mm = -1.0 if cfg.t_pitch_mm is None else float(cfg.t_pitch_mm)
    if cfg.t_pitch_mm is not None and not float(cfg.t_pitch_mm) > 0:
        raise ValueError("t_pitch_mm must be positive")
    c.t_taper = 1 if cfg.t_taper == "hann" else 0
    c.spectrum_j = int(cfg.spectrum_j)
    for k in range(3):
        c.resample_j[k] = int(rj[k])
    c.side_lobes = int(cfg.side_lobes)
    c.oversample_factor = float(cfg.oversample_factor)
    c.rho_pad = -1 if cfg.rho_pad is None else int(cfg.rho_pad)
    c.basis = 0 if cfg.basis == "trilinear" else 1
    c.normalization = float(cfg.normalization)
    c.bp_normalization = float(cfg.bp_normalization)
    c.den_tol = float(cfg.den_tol)
    c.target_batch = int(target_batch)
    c.plan_chunk = int(plan_chunk)
    return c


def _key(geom, cfg, n, voxel, direction, target_batch, plan_chunk):
    spec = cfg.radial_spec
    return (tuple(float(getattr(geom, f)) for f in ("so_mm", "sd_mm", "det_width_mm",
                                                       "det_height_mm", "object_extent_mm")),
            int(geom.nu), int(geom.nv), int(geom.n_views),
            (int(spec.n_rho), int(spec.n_theta), int(spec.n_phi), float(spec.rho_max)),
            str(cfg.method), int(cfg.n_mu), int(cfg.n_t), cfg.t_pitch_mm, cfg.t_taper,
            int(cfg.spectrum_j), tuple(np.broadcast_to(np.atleast_1d(cfg.resample_j), (3,)).tolist()),
            float(cfg.oversample_factor), cfg.rho_pad, cfg.basis, float(cfg.normalization),
            float(cfg.bp_normalization), float(cfg.den_tol), int(cfg.side_lobes), int(n),
            float(voxel), direction,
            int(target_batch), int(plan_chunk))


class Projector:
    """Device plan of the forward projector and/or backprojector."""

    def __init__(self, geom, cfg, n: int, voxel_mm: float, direction: int = 3,
                 target_batch: int | None = None, plan_chunk: int | None = None,
                 bp_n_t: int | None = None, bp_t_pitch_mm: float | None = None):
        from . import nufft as _nufft
        lib = _lib.load()
        _device.require_cuda()
        self.geom, self.cfg, self.n, self.voxel = geom, cfg, int(n), float(voxel_mm)
        self.direction = direction
        tb = _TARGET_BATCH if target_batch is None else int(target_batch)
        pc = _nufft._PLAN_CHUNK if plan_chunk is None else int(plan_chunk)
        self._g = _geometry_struct(geom)
        self._c = _config_struct(cfg, tb, pc)
        self.bp_n_t = 2 * int(geom.nu) if bp_n_t is None else int(bp_n_t)
        self._c.bp_n_t = self.bp_n_t
        self._c.bp_t_pitch_mm = -1.0 if bp_t_pitch_mm is None else float(bp_t_pitch_mm)
        h = ctypes.c_void_p()
        _lib.check(lib.cbn_projector_create(ctypes.byref(h), ctypes.byref(self._g),
                                            ctypes.byref(self._c), self.n, self.voxel,
                                            direction), "projector")
        self._h = h
        self.stage = _hostio.Staging()
        cnt = ctypes.c_int32(64)
        sizes = (ctypes.c_int64 * 64)()
        _lib.check(lib.cbn_projector_ls_sizes(h, sizes, ctypes.byref(cnt)))
        for m in list(sizes)[:cnt.value]:
            rows, rp = _lib.i64_array(_device.ls_rows(int(m)))
            _lib.check(lib.cbn_projector_set_ls_rows(h, int(m), rp, rows.size))

    def __del__(self):
        h = getattr(self, "_h", None)
        lib = getattr(_lib, "_lib", None) if _lib is not None else None
        if h and h.value and lib is not None:
            lib.cbn_projector_destroy(h)
            self._h = ctypes.c_void_p()

    @property
    def _s(self):
        return ctypes.c_void_p(_device.stream_ptr())

    # ---- whole operators (device tensors)
    def forward(self, vol, view_lo: int = 0, view_hi: int | None = None):
        t = _device.require_cuda()
        view_hi = self.geom.n_views if view_hi is None else view_hi
        v = _device.to_device(vol, t.float32)
        if tuple(v.shape) != (self.n,) * 3:
            raise ValueError(f"volume must be ({self.n},)*3")
        out = t.empty((view_hi - view_lo, self.geom.nu, self.geom.nv), dtype=t.float32,
                      device="cuda")
        _lib.check(_lib.load().cbn_forward_project(self._h, _device.ptr(v), _device.ptr(out),
                                                   int(view_lo), int(view_hi), self._s),
                   "nufft_forward_project")
        return out

    def backproject(self, frames):
        t = _device.require_cuda()
        f = _device.to_device(frames, t.float32)
        if tuple(f.shape) != (self.geom.n_views, self.geom.nu, self.geom.nv):
            raise ValueError("frames must be (n_views, nu, nv)")
        out = t.empty((self.n,) * 3, dtype=t.float32, device="cuda")
        _lib.check(_lib.load().cbn_backproject(self._h, _device.ptr(f), _device.ptr(out), self._s),
                   "nufft_backproject")
        return out

    def blocks(self):
        """View blocks [(lo, hi), ...] of the last cbn_forward_project_async,
        in completion-event order (cbn_projector_blocks)."""
        lib = _lib.load()
        cnt = ctypes.c_int32(0)
        _lib.check(lib.cbn_projector_blocks(self._h, None, None, ctypes.byref(cnt)))
        lo = (ctypes.c_int32 * max(1, cnt.value))()
        hi = (ctypes.c_int32 * max(1, cnt.value))()
        _lib.check(lib.cbn_projector_blocks(self._h, lo, hi, ctypes.byref(cnt)))
        return [(int(lo[k]), int(hi[k])) for k in range(cnt.value)]

    # ---- forward phases (node / view sharding)
    def forward_lattice(self, vol, part: int = 0, nparts: int = 1, out=None):
        """Phase 1: spectrum-gather values of radial-node part `part` of `nparts`
        (zeros elsewhere), before the radial IFFT."""
        t = _device.require_cuda()
        v = _device.to_device(vol, t.float32)
        if tuple(v.shape) != (self.n,) * 3:
            raise ValueError(f"volume must be ({self.n},)*3")
        m = ctypes.c_int64()
        _lib.check(_lib.load().cbn_forward_lattice_size(self._h, ctypes.byref(m), self._s))
        out = t.empty(int(m.value), dtype=t.complex64, device="cuda") if out is None else out
        _lib.check(_lib.load().cbn_forward_lattice(self._h, _device.ptr(v), int(part), int(nparts),
                                                   _device.ptr(out), self._s),
                   "nufft_forward_project")
        return out

    def set_node_shard(self, part: int, nparts: int):
        """Restrict this forward-only plan's spectrum plan to the radial lines of
        share `part` of `nparts`; returns its lattice block (node_lo, node_hi)
        (cbn_projector_set_node_shard).  NotImplementedError when the lines do
        not split evenly."""
        lo, hi = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(_lib.load().cbn_projector_set_node_shard(self._h, int(part), int(nparts),
                                                            ctypes.byref(lo), ctypes.byref(hi),
                                                            self._s), "set_node_shard")
        return int(lo.value), int(hi.value)

    def forward_views(self, lattice, view_lo: int = 0, view_hi: int | None = None):
        """Phase 2: from the summed lattice (consumed), views [view_lo, view_hi)."""
        t = _device.require_cuda()
        view_hi = self.geom.n_views if view_hi is None else view_hi
        out = t.empty((view_hi - view_lo, self.geom.nu, self.geom.nv), dtype=t.float32,
                      device="cuda")
        _lib.check(_lib.load().cbn_forward_views(self._h, _device.ptr(lattice), _device.ptr(out),
                                                 int(view_lo), int(view_hi), self._s),
                   "nufft_forward_project")
        return out

    def forward_sharded(self, vol, view_lo: int, view_hi: int, group=None,
                        broadcast: bool = True):
        """nufft_forward_project over a process group: the volume (a torch tensor
        on the group's device) broadcast from the group's first rank unless
        `broadcast` is False, 1/world of the radial nodes (lattice summed with
        one NCCL all-reduce), then this rank's views."""
        import torch.distributed as dist
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        if world > 1 and broadcast:
            dist.broadcast(vol, dist.get_global_rank(group, 0) if group is not None else 0,
                           group=group)
        lat = self.forward_lattice(vol, rank, world)
        if world > 1:
            dist.all_reduce(lat, group=group)
        return self.forward_views(lat, view_lo, view_hi)

    # ---- backprojector phases (view / node sharding)
    def backproject_sizes(self):
        """(lattice_elems, grid_elems): complex64 sizes of the phase buffers."""
        a, b = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(_lib.load().cbn_backproject_sizes(self._h, ctypes.byref(a), ctypes.byref(b),
                                                     self._s), "nufft_backproject")
        return int(a.value), int(b.value)

    def backproject_views(self, frames, view_lo: int, view_hi: int, out=None):
        """Phase 1: transposed resample of views [view_lo, view_hi) (frames holds
        exactly those views) into a padded-lattice accumulator."""
        t = _device.require_cuda()
        f = _device.to_device(frames, t.float32)
        if tuple(f.shape) != (view_hi - view_lo, self.geom.nu, self.geom.nv):
            raise ValueError("frames must be (view_hi - view_lo, nu, nv)")
        n_lat, _ = self.backproject_sizes()
        out = t.empty(n_lat, dtype=t.complex64, device="cuda") if out is None else out
        _lib.check(_lib.load().cbn_backproject_views(self._h, _device.ptr(f), int(view_lo),
                                                     int(view_hi), _device.ptr(out), self._s),
                   "nufft_backproject")
        return out

    def backproject_finish(self, lattice, part: int = 0, nparts: int = 1, out=None):
        """Phase 2: from the summed accumulator (consumed), spread node part
        `part` of `nparts` into a (2N)^3 grid."""
        t = _device.require_cuda()
        _, n_grid = self.backproject_sizes()
        out = t.empty(n_grid, dtype=t.complex64, device="cuda") if out is None else out
        _lib.check(_lib.load().cbn_backproject_finish(self._h, _device.ptr(lattice), int(part),
                                                      int(nparts), _device.ptr(out), self._s),
                   "nufft_backproject")
        return out

    def backproject_crop(self, grid):
        """Phase 3: inverse FFT, crop and deapodisation of the summed grid (consumed)."""
        t = _device.require_cuda()
        out = t.empty((self.n,) * 3, dtype=t.float32, device="cuda")
        _lib.check(_lib.load().cbn_backproject_crop(self._h, _device.ptr(grid), _device.ptr(out),
                                                    self._s), "nufft_backproject")
        return out

    def backproject_crop_slab(self, slab, x_lo: int, x_hi: int, nparts: int):
        """Phase 3a (slab-distributed): planes [x_lo, x_hi) of the summed grid
        (consumed) -> y/z-cropped planes in the all-to-all send layout
        [y block d][x][y - y0_d][z] (y0_d = d * N // nparts)."""
        t = _device.require_cuda()
        send = t.empty((x_hi - x_lo) * self.n * self.n, dtype=t.complex64, device="cuda")
        _lib.check(_lib.load().cbn_backproject_crop_slab(self._h, _device.ptr(slab), int(x_lo),
                                                         int(x_hi), int(nparts),
                                                         _device.ptr(send), self._s),
                   "nufft_backproject")
        return send

    def backproject_crop_cols(self, cols, y_lo: int, y_hi: int):
        """Phase 3b: the received columns [2N][y_hi - y_lo][N] (consumed) -> the
        volume's y range, float32 (N, y_hi - y_lo, N)."""
        t = _device.require_cuda()
        out = t.empty((self.n, y_hi - y_lo, self.n), dtype=t.float32, device="cuda")
        _lib.check(_lib.load().cbn_backproject_crop_cols(self._h, _device.ptr(cols), int(y_lo),
                                                         int(y_hi), _device.ptr(out), self._s),
                   "nufft_backproject")
        return out

    def backproject_sharded(self, frames_local, view_lo: int, view_hi: int, group=None):
        """nufft_backproject over a process group: this rank's
        views (accumulators summed with an all-reduce), 1/world of the radial
        nodes spread into a local (2N)^3 grid, the grids reduce-scattered by
        slabs of x planes, slab IFFT + y/z crop, an all-to-all transpose to
        y ranges, x IFFT + crop, and an all-gather of the volume."""
        import torch.distributed as dist
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        lat = self.backproject_views(frames_local, view_lo, view_hi)
        if world > 1:
            dist.all_reduce(lat, group=group)
        grid = self.backproject_finish(lat, rank, world)
        if world == 1:
            return self.backproject_crop(grid)
        return sharded_crop(self, grid, rank, world, group)

    # ---- stages
    def radial_lattice(self, vol):
        """Complex lattice in node order (n_phi, n_theta, n_rho)."""
        t = _device.require_cuda()
        v = _device.to_device(vol, t.float32)
        spec = self.cfg.radial_spec
        out = t.empty((spec.n_phi, spec.n_theta, spec.n_rho), dtype=t.complex64, device="cuda")
        _lib.check(_lib.load().cbn_projector_radial_lattice(self._h, _device.ptr(v),
                                                            _device.ptr(out), self._s))
        return out

    def resample_views(self, lattice, view_lo: int, view_hi: int):
        t = _device.require_cuda()
        lat = _device.to_device(lattice, t.complex64)
        out = t.empty((view_hi - view_lo, self.cfg.n_mu, self.cfg.n_t), dtype=t.float32,
                      device="cuda")
        _lib.check(_lib.load().cbn_projector_resample_views(self._h, _device.ptr(lat),
                                                            _device.ptr(out), view_lo, view_hi,
                                                            self._s))
        return out

    def grangeat_reverse(self, values):
        t = _device.require_cuda()
        v = _device.to_device(values, t.float32)
        nb = v.shape[0]
        out = t.empty((nb, self.geom.nu, self.geom.nv), dtype=t.float32, device="cuda")
        _lib.check(_lib.load().cbn_projector_grangeat_reverse(self._h, _device.ptr(v),
                                                              _device.ptr(out), nb, self._s))
        return out

    def backproject_stage_transpose(self, frames, view_lo: int, view_hi: int):
        """(num, den) of the backprojector for views [view_lo, view_hi): the summed
        resample_transpose of the forward-Grangeat values and of the validity
        mask (pipeline.py:174-184), after the lattice IFFT, rho crop and origin
        average -- complex64 / float32 in node order (n_phi, n_theta, n_rho)."""
        t = _device.require_cuda()
        f = _device.to_device(frames, t.float32)
        if tuple(f.shape) != (view_hi - view_lo, self.geom.nu, self.geom.nv):
            raise ValueError("frames must be (view_hi - view_lo, nu, nv)")
        n_rho = 2 * int(np.ceil(1.5 * self.n / 2.0))
        shape = (self.cfg.radial_spec.n_phi, self.cfg.radial_spec.n_theta, n_rho)
        num = t.empty(shape, dtype=t.complex64, device="cuda")
        den = t.empty(shape, dtype=t.float32, device="cuda")
        _lib.check(_lib.load().cbn_backproject_stage_transpose(
            self._h, _device.ptr(f), int(view_lo), int(view_hi), _device.ptr(num),
            _device.ptr(den), self._s), "nufft_backproject")
        return num, den

    # ---- plan diagnostics
    _SETS = {("forward", "radial"): 0, ("forward", "umbrella"): 1, ("forward", "polar"): 2,
             ("back", "radial"): 3, ("back", "umbrella"): 4, ("back", "polar"): 5}

    def first_indices(self, direction: str, node_set: str, batch: int = 0) -> np.ndarray:
        """(m, d) int32 first-tap index mod K per axis of one of the projector's
        node sets (reference axis order), as its kernels use it -- comparable to
        plan_nufft(...).interp.indices[:, 0] of the reference (nufft.py:171-179)."""
        s = self._SETS[(direction, node_set)]
        lib = _lib.load()
        m = ctypes.c_int64(0)
        _lib.check(lib.cbn_projector_first_indices(self._h, s, int(batch), None, ctypes.byref(m),
                                                   self._s))
        d = 2 if node_set == "polar" else 3
        out = np.empty((m.value, d), dtype=np.int32)
        _lib.check(lib.cbn_projector_first_indices(self._h, s, int(batch),
                                                   out.ctypes.data_as(_lib.P_i32),
                                                   ctypes.byref(m), self._s))
        return out

    def plan_stats(self) -> dict:
        """Plan statistics (cbn_projector_plan_stats); -1 = not built yet."""
        lib = _lib.load()
        cnt = ctypes.c_int32(64)
        vals = (ctypes.c_int64 * 64)()
        names = ctypes.create_string_buffer(4096)
        _lib.check(lib.cbn_projector_plan_stats(self._h, vals, ctypes.byref(cnt), names, 4096,
                                                self._s))
        keys = names.value.decode().split(";")[:cnt.value]
        return {k: int(vals[i]) for i, k in enumerate(keys)}

    def grangeat_forward(self, frames):
        t = _device.require_cuda()
        f = _device.to_device(frames, t.float32)
        nb = f.shape[0]
        out = t.empty((nb, self.cfg.n_mu, self.bp_n_t), dtype=t.float32, device="cuda")
        _lib.check(_lib.load().cbn_projector_grangeat_forward(self._h, _device.ptr(f),
                                                              _device.ptr(out), nb, self._s))
        return out


def slab_ranges(extent: int, world: int) -> list[int]:
    """Balanced split points of `extent` planes over `world` ranks."""
    return [extent * r // world for r in range(world + 1)]


def sharded_crop(proj, grid, rank: int, world: int, group=None):
    """Slab-distributed phase 3 of the backprojector (adjoint
    steps 4-6) for a rank's un-summed (K, K, K) grid, K = 2N:
    reduce-scatter by x slab (all-reduce + slice when world does not divide K),
    2D IFFT + y/z crop of the slab, all-to-all to y ranges, x IFFT + crop, and
    an all-gather of the y ranges into the full N^3 volume on every rank."""
    import torch
    import torch.distributed as dist
    n = proj.n
    k = round(grid.numel() ** (1.0 / 3.0))
    if k ** 3 != grid.numel() or k < n:
        raise ValueError("grid is not a (2N)^3 cube")
    plane = k * k
    xs, ys = slab_ranges(k, world), slab_ranges(n, world)
    if k % world == 0:
        slab = torch.empty(plane * (k // world), dtype=grid.dtype, device=grid.device)
        # reduce_scatter_tensor has no complex path: reduce the (re, im) view
        real = torch.view_as_real if grid.is_complex() else (lambda t: t)
        dist.reduce_scatter_tensor(real(slab), real(grid), group=group)
    else:
        dist.all_reduce(grid, group=group)
        slab = grid[xs[rank] * plane: xs[rank + 1] * plane]
    send = proj.backproject_crop_slab(slab, xs[rank], xs[rank + 1], world)
    xc, yc = xs[rank + 1] - xs[rank], ys[rank + 1] - ys[rank]
    in_splits = [xc * (ys[d + 1] - ys[d]) * n for d in range(world)]
    out_splits = [(xs[q + 1] - xs[q]) * yc * n for q in range(world)]
    cols = torch.empty(sum(out_splits), dtype=send.dtype, device=send.device)
    dist.all_to_all_single(cols, send, out_splits, in_splits, group=group)
    part = proj.backproject_crop_cols(cols, ys[rank], ys[rank + 1])
    cap = max(ys[d + 1] - ys[d] for d in range(world))
    buf = torch.zeros((n, cap, n), dtype=part.dtype, device=part.device)
    buf[:, :yc] = part
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([parts[d][:, : ys[d + 1] - ys[d]] for d in range(world)], dim=1)


def get_projector(geom, cfg, n, voxel_mm, direction):
    from . import nufft as _nufft
    key = _key(geom, cfg, n, voxel_mm, direction, _TARGET_BATCH, _nufft._PLAN_CHUNK)
    p = _CACHE.get(key)
    if p is None:
        p = Projector(geom, cfg, n, voxel_mm, direction)
        _CACHE[key] = p
        while len(_CACHE) > _CACHE_SIZE:
            _CACHE.popitem(last=False)
    else:
        _CACHE.move_to_end(key)
    return p


def clear_plan_cache() -> None:
    _CACHE.clear()


def nufft_forward_project(vol: Volume3D, geom, cfg) -> list[DetectorFrame]:
    """NUFFT cone-beam forward projection of all views (pipeline.py:122-147).

    Host float64 volume in, ``list[DetectorFrame]`` (float64) out, like the
    reference.  The conversions run on host threads through the plan's pinned
    staging buffers (_hostio); non-finite projections raise FloatingPointError
    from the device check."""
    import torch
    data = np.asarray(vol.data)
    proj = get_projector(geom, cfg, data.shape[0], vol.voxel_mm, _FORWARD)
    if data.shape != (proj.n,) * 3:
        raise ValueError(f"volume must be ({proj.n},)*3")
    lib = _lib.load()
    s = proj._s
    staged = [_STAGE_VOLUME]

    def stage_rows(dev, a, b):
        # rows [a, b) are on their way: pad and 2D-transform them while the host
        # converts the next chunk (plans that cannot stage take the plain call)
        if staged[0]:
            rc = lib.cbn_forward_stage_volume(proj._h, _device.ptr(dev), a, b, s)
            if rc == _lib.CBN_EUNSUPPORTED:
                staged[0] = False
            else:
                _lib.check(rc, "nufft_forward_project")

    v = _hostio.upload(proj.stage, "vol", data, torch.float32, on_chunk=stage_rows)
    out = torch.empty((geom.n_views, geom.nu, geom.nv), dtype=torch.float32, device="cuda")
    # every kernel is enqueued at once; the frames of each reverse-Grangeat
    # block are copied out and converted while later blocks still compute
    if staged[0]:
        _lib.check(lib.cbn_forward_project_staged_async(proj._h, _device.ptr(out), 0, geom.n_views,
                                                        s), "nufft_forward_project")
    else:
        _lib.check(lib.cbn_forward_project_async(proj._h, _device.ptr(v), _device.ptr(out), 0,
                                                 geom.n_views, s), "nufft_forward_project")
    blocks = proj.blocks()
    # the result array and its per-view wrappers are made while the device is
    # still working towards the first view block
    frames = proj.stage.result("frames", tuple(out.shape), np.float64)
    result = [DetectorFrame._checked(k, frames[k], geom.pixel_mm) for k in range(geom.n_views)]
    _hostio.download_blocks(
        proj.stage, "frames", out, blocks,
        lambda k: _lib.check(lib.cbn_projector_block_sync(proj._h, k), "nufft_forward_project"),
        out=frames)
    _lib.check(lib.cbn_forward_finish(proj._h, s), "nufft_forward_project")
    return result


_BP_STAGE_VIEWS = 64   # views per upload block of the drop-in backprojector


def nufft_backproject(frames, geom, cfg, out_size: int, voxel_mm: float) -> Volume3D:
    """Direct NUFFT backprojection (pipeline.py:150-212): list of frames in,
    float64 ``Volume3D`` out (ValueError on non-finite values, as the
    reference's Volume3D raises)."""
    import torch
    if len(frames) != geom.n_views:
        raise ValueError("frame count does not match the geometry")
    proj = get_projector(geom, cfg, out_size, voxel_mm, _BACK)
    shape = (geom.n_views, geom.nu, geom.nv)
    pin = proj.stage.get("frames", shape, torch.float32)
    host = pin.numpy()
    for k, f in enumerate(frames):
        if np.shape(f.data) != shape[1:]:
            raise ValueError("frames must be (n_views, nu, nv)")
    dev = torch.empty(shape, dtype=torch.float32, device="cuda")
    V = geom.n_views
    lib = _lib.load()
    s = proj._s
    # blocks of 64 views: converted on the pool, copied on the device stream and
    # (where the plan allows) forward-Grangeat'ed at once, so the device works
    # on block k while the host converts block k + 1
    bounds = list(range(0, V, _BP_STAGE_VIEWS)) + [V]
    staged = True
    table = _hostio.frame_pointers([f.data for f in frames], shape[1:])
    for a, b in zip(bounds[:-1], bounds[1:]):
        if table is not None:
            _hostio.gather_block(host[a:b], table, a, b)
        else:
            _hostio.gather_frames(host[a:b], [frames[k].data for k in range(a, b)])
        dev[a:b].copy_(pin[a:b], non_blocking=True)
        if staged:
            rc = lib.cbn_backproject_stage_views(proj._h, _device.ptr(dev[a]), a, b, s)
            if rc == _lib.CBN_EUNSUPPORTED:
                staged = False
            else:
                _lib.check(rc, "nufft_backproject")
    vol = proj.backproject(dev)
    finite = torch.isfinite(vol).all()      # read after the download is under way
    out = _hostio.download(proj.stage, "vol", vol)
    if not bool(finite):
        raise ValueError("volume contains non-finite values")
    return Volume3D._checked(out, voxel_mm)


def calibrate_normalization(geom, n: int, cfg, voxel_mm: float) -> float:
    """Forward-projector scale fitted on the analytic smooth ball (pipeline.py:215-242):
    least-squares ratio between the closed-form view-0 projection and the
    projector's view-0 output; stored in cfg.normalization and returned."""
    from .phantom import smooth_ball_line_integral, smooth_ball_volume
    radius = 0.28 * n * voxel_mm
    vol = smooth_ball_volume(n, voxel_mm, radius)
    cfg.normalization = 1.0
    proj = get_projector(geom, cfg, n, voxel_mm, _FORWARD)
    got = proj.forward(vol.data, 0, 1).cpu().numpy().astype(np.float64)[0].ravel()
    s = geom.source_position(0)
    pu, pv = geom.pixel_mm
    u = (np.arange(geom.nu) - geom.nu / 2.0 + 0.5) * pu
    v = (np.arange(geom.nv) - geom.nv / 2.0 + 0.5) * pv
    uu, vv = np.meshgrid(u, v, indexing="ij")
    a = geom.view_angle(0)
    s_hat = np.array([np.cos(a), np.sin(a), 0.0])
    u_hat = np.array([-np.sin(a), np.cos(a), 0.0])
    v_hat = np.array([0.0, 0.0, 1.0])
    pts = (s - geom.sd_mm * s_hat)[None, :] \
        + uu.ravel()[:, None] * u_hat + vv.ravel()[:, None] * v_hat
    d = pts - s
    d /= np.linalg.norm(d, axis=-1, keepdims=True)
    ref = smooth_ball_line_integral(np.broadcast_to(s, d.shape), d, radius=radius)
    cfg.normalization = float(np.dot(ref, got) / np.dot(got, got))
    return cfg.normalization


def calibrate_bp_normalization(geom, n: int, cfg, voxel_mm: float) -> float:
    """Backprojector scale fitted on the smooth ball through the baseline
    ray-driven projector (pipeline.py:245-257); stored in cfg.bp_normalization."""
    from .baseline import ct_project_linear
    from .phantom import smooth_ball_volume
    radius = 0.28 * n * voxel_mm
    vol = smooth_ball_volume(n, voxel_mm, radius)
    frames = ct_project_linear(vol, geom)
    cfg.bp_normalization = 1.0
    rec = nufft_backproject(frames, geom, cfg, n, voxel_mm)
    mask = vol.data > 0.05
    cfg.bp_normalization = float(np.dot(vol.data[mask], rec.data[mask])
                                 / np.dot(rec.data[mask], rec.data[mask]))
    return cfg.bp_normalization
