"""Multi-GPU operators over NCCL through the C ABI (include/cbnufft_b200_comm.h).

``libcbnufft_b200_comm.so`` holds the collectives between the projector
phases; this module only binds it.  One process per GPU: rank
0 draws the NCCL unique id, any out-of-band channel hands it to the other
ranks (``NcclComm.from_group`` uses torch.distributed for that one exchange),
and every rank then calls the sharded operators with its own view range.  The
library is separate from libcbnufft_b200.so so that single-GPU hosts never
load NCCL.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import _device, _lib

_HERE = os.path.dirname(os.path.abspath(__file__))
COMM_LIB_PATH = os.path.join(_HERE, "libcbnufft_b200_comm.so")
ID_BYTES = 128

c_i32, c_vp = ctypes.c_int32, ctypes.c_void_p
P_i32 = ctypes.POINTER(c_i32)

_SIGS = {
    "cbn_comm_last_error": (ctypes.c_char_p, []),
    "cbn_comm_unique_id": (ctypes.c_int, [c_vp]),
    "cbn_comm_init": (ctypes.c_int, [ctypes.POINTER(c_vp), c_vp, c_i32, c_i32]),
    "cbn_comm_destroy": (ctypes.c_int, [c_vp]),
    "cbn_comm_rank": (ctypes.c_int, [c_vp, P_i32, P_i32]),
    "cbn_forward_project_sharded": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_vp]),
    "cbn_backproject_sharded": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp]),
}
EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_clib = None


def load(path: str = COMM_LIB_PATH):
    """Load and type the communicator library (no device work)."""
    global _clib
    with _lock:
        if _clib is not None:
            return _clib
        _lib.load()   # the projector library it links against, from this package
        if not os.path.exists(path):
            raise _lib.ExtensionMissing(f"{path} is not built; run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        missing = []
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name, None)
            if fn is None:
                missing.append(name)
                continue
            fn.restype = res
            fn.argtypes = args
        lib.cbn_missing_symbols = tuple(missing)
        _clib = lib
        return lib


def _check(status: int, what: str) -> None:
    if status == _lib.CBN_OK:
        return
    msg = load().cbn_comm_last_error().decode(errors="replace")
    if status == _lib.CBN_ENCCL:
        raise RuntimeError(f"{what}: NCCL failure: {msg}")
    if status == _lib.CBN_EINVAL:
        raise ValueError(f"{what}: {msg}")
    if status == _lib.CBN_ENONFINITE:
        raise FloatingPointError(f"{what}: {msg}")
    if status == _lib.CBN_ENOMEM:
        raise MemoryError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: CUDA failure ({status}) {msg}")


def unique_id() -> bytes:
    buf = ctypes.create_string_buffer(ID_BYTES)
    _check(load().cbn_comm_unique_id(buf), "cbn_comm_unique_id")
    return buf.raw


class NcclComm:
    """An NCCL communicator created through the C ABI (one GPU per rank)."""

    def __init__(self, uid: bytes, nranks: int, rank: int):
        _device.require_cuda()
        if len(uid) != ID_BYTES:
            raise ValueError("NCCL unique id must be 128 bytes")
        h = c_vp()
        _check(load().cbn_comm_init(ctypes.byref(h), ctypes.create_string_buffer(uid, ID_BYTES),
                                    int(nranks), int(rank)), "cbn_comm_init")
        self._h = h
        self.rank, self.nranks = int(rank), int(nranks)

    @classmethod
    def local(cls) -> "NcclComm":
        """A single-rank communicator (one process, one GPU)."""
        return cls(unique_id(), 1, 0)

    @classmethod
    def from_group(cls, group=None) -> "NcclComm":
        """One communicator per rank of a torch.distributed group: rank 0's id
        is broadcast over the group (the only use of torch.distributed)."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0,
                                   group=group)
        return cls(obj[0], world, rank)

    def close(self) -> None:
        if getattr(self, "_h", None):
            load().cbn_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def forward_project(self, proj, vol, view_lo: int, view_hi: int):
        """Sharded nufft_forward_project: vol (CUDA float32 N^3; rank 0's is
        broadcast into the others') -> this rank's frames [view_lo, view_hi)."""
        t = _device.require_cuda()
        if not (isinstance(vol, t.Tensor) and vol.is_cuda and vol.dtype == t.float32
                and vol.is_contiguous() and tuple(vol.shape) == (proj.n,) * 3):
            raise ValueError(f"vol must be a contiguous CUDA float32 ({proj.n},)*3 tensor")
        g = proj.geom
        out = t.empty((view_hi - view_lo, g.nu, g.nv), dtype=t.float32, device="cuda")
        _check(load().cbn_forward_project_sharded(proj._h, self._h, _device.ptr(vol),
                                                  _device.ptr(out) if out.numel() else None,
                                                  int(view_lo), int(view_hi), proj._s),
               "nufft_forward_project")
        return out

    def backproject(self, proj, frames_local, view_lo: int, view_hi: int):
        """Sharded nufft_backproject: this rank's frames [view_lo, view_hi)
        (CUDA float32) -> the N^3 volume on every rank."""
        t = _device.require_cuda()
        f = _device.to_device(frames_local, t.float32)
        g = proj.geom
        if tuple(f.shape) != (view_hi - view_lo, g.nu, g.nv):
            raise ValueError("frames must be (view_hi - view_lo, nu, nv)")
        vol = t.empty((proj.n,) * 3, dtype=t.float32, device="cuda")
        _check(load().cbn_backproject_sharded(proj._h, self._h,
                                              _device.ptr(f) if f.numel() else None,
                                              int(view_lo), int(view_hi), _device.ptr(vol), proj._s),
               "nufft_backproject")
        return vol
