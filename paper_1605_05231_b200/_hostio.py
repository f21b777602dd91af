"""Host side of the drop-in operators: pinned staging and threaded dtype
conversion (plumbing, no numerics).

The reference API is numpy in / numpy out with float64 results
(``DetectorFrame``/``Volume3D`` store float64).  The device
path computes in float32, so every call converts on the host: float64 volume
-> float32 upload, float32 frames -> float64 results (and the reverse for the
backprojector).  float64 <-> float32 conversions of contiguous arrays run in
the library's OpenMP threads (cbn_host_*, csrc/cbn_hostio.cu) outside the
interpreter lock; anything else is split over a Python thread pool (numpy
releases the GIL inside ``copyto``).  They go through pinned staging buffers
that each projector plan keeps, so the copies run at DMA speed and overlap the
conversion of the previous chunk.
"""

from __future__ import annotations

import os
import sys
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_POOL: ThreadPoolExecutor | None = None
_UPLOAD_CHUNKS = int(os.environ.get("CBN_UPLOAD_CHUNKS", "4"))
_THREADS = max(1, min(16, os.cpu_count() or 1))


def pool() -> ThreadPoolExecutor:
    global _POOL
    if _POOL is None:
        _POOL = ThreadPoolExecutor(max_workers=_THREADS, thread_name_prefix="cbn-host")
    return _POOL


def _native_convert(dst: np.ndarray, src: np.ndarray) -> bool:
    """float64 <-> float32 conversion of contiguous arrays in the library's
    OpenMP threads (cbn_host_*), outside the interpreter lock."""
    if dst.shape != src.shape or not (dst.flags.c_contiguous and src.flags.c_contiguous):
        return False
    if dst.dtype == np.complex64 and src.dtype == np.complex128:
        dst, src = dst.view(np.float32), src.view(np.float64)
    elif dst.dtype == np.complex128 and src.dtype == np.complex64:
        dst, src = dst.view(np.float64), src.view(np.float32)
    from . import _lib
    lib = _lib.load()
    if dst.dtype == np.float32 and src.dtype == np.float64:
        fn = lib.cbn_host_f64_to_f32
    elif dst.dtype == np.float64 and src.dtype == np.float32:
        fn = lib.cbn_host_f32_to_f64
    else:
        return False
    _lib.check(fn(src.ctypes.data, dst.ctypes.data, src.size, 0), "host conversion")
    return True


def gather_frames(dst: np.ndarray, arrays) -> None:
    """dst[k] = arrays[k] (float64 -> float32) for a list of equally shaped
    frames, in one native threaded call when they are contiguous float64."""
    import ctypes
    from . import _lib
    arrs = [np.asarray(a) for a in arrays]
    if (dst.dtype == np.float32 and dst.flags.c_contiguous and len(arrs) == dst.shape[0]
            and all(a.dtype == np.float64 and a.flags.c_contiguous and a.shape == dst.shape[1:]
                    for a in arrs)):
        ptrs = (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
        _lib.check(_lib.load().cbn_host_gather_f64_to_f32(ptrs, len(arrs), int(dst[0].size),
                                                          dst.ctypes.data, 0), "host conversion")
        return
    futs = [pool().submit(np.copyto, dst[k], a, casting="unsafe") for k, a in enumerate(arrs)]
    for f in futs:
        f.result()


def frame_pointers(arrays, shape):
    """ctypes pointer table of a list of equally shaped contiguous float64
    frames (one pass over the list), or None when any frame needs the general
    route; `gather_block` then converts ranges of it natively."""
    import ctypes
    arrs = [np.asarray(a) for a in arrays]
    shape = tuple(shape)
    for a in arrs:
        if a.dtype != np.float64 or not a.flags.c_contiguous or a.shape != shape:
            return None
    table = (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    table._keep = arrs      # the arrays stay alive with the table
    return table


def gather_block(dst: np.ndarray, table, lo: int, hi: int) -> None:
    """dst[k - lo] = float32(frame k) for lo <= k < hi, frames given by a
    `frame_pointers` table; dst is a contiguous float32 block."""
    import ctypes
    from . import _lib
    elems = int(dst[0].size) if hi > lo else 0
    ptr = ctypes.c_void_p(ctypes.addressof(table) + lo * ctypes.sizeof(ctypes.c_void_p))
    _lib.check(_lib.load().cbn_host_gather_f64_to_f32(ptr, hi - lo, elems, dst.ctypes.data, 0),
               "host conversion")


def copy(dst: np.ndarray, src: np.ndarray, min_chunk: int = 1 << 18) -> None:
    """dst[...] = src (with dtype conversion), split along axis 0 over threads."""
    if _native_convert(dst, src):
        return
    n = dst.shape[0]
    per = max(1, min_chunk // max(1, dst[0].size if dst.ndim > 1 else 1))
    parts = max(1, min(_THREADS, -(-n // per)))
    if parts == 1:
        np.copyto(dst, src, casting="unsafe")
        return
    bounds = [n * i // parts for i in range(parts + 1)]
    futs = [pool().submit(np.copyto, dst[a:b], src[a:b], casting="unsafe")
            for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
    for f in futs:
        f.result()


class Staging:
    """Pinned host buffers of one projector plan, keyed by (tag, shape, dtype),
    and its result arrays: a result whose previous instance nobody holds any
    more (the caller dropped every frame / volume that viewed it) is reused,
    which saves the first-touch page faults of a fresh 100+ MB array; while
    the caller holds it, a new one is allocated."""

    def __init__(self, single_shape: bool = False):
        self._bufs = {}
        self._results = {}
        self.single_shape = single_shape

    def result(self, tag: str, shape, dtype):
        key = (tag, tuple(shape), np.dtype(dtype).str)
        if self.single_shape:
            for k in [k for k in self._results if k[0] == tag and k != key]:
                del self._results[k]
        arr = self._results.get(key)
        # references: this dict, `arr`, getrefcount's argument
        if arr is not None and sys.getrefcount(arr) <= 3:
            return arr
        arr = np.empty(tuple(shape), dtype=dtype)
        self._results[key] = arr
        return arr

    def copy_stream(self):
        import torch
        if getattr(self, "_cs", None) is None:
            self._cs = torch.cuda.Stream()
        return self._cs

    def get(self, tag: str, shape, dtype):
        import torch
        key = (tag, tuple(shape), dtype)
        if self.single_shape:
            # one pinned buffer per tag: a new shape releases the old one
            for k in [k for k in self._bufs if k[0] == tag and k != key]:
                del self._bufs[k]
        b = self._bufs.get(key)
        if b is None:
            b = torch.empty(tuple(shape), dtype=dtype, pin_memory=True)
            self._bufs[key] = b
        return b


def upload(stage: Staging, tag: str, host: np.ndarray, dtype, chunks: int | None = None,
           on_chunk=None):
    """numpy (any real dtype) -> new CUDA tensor of `dtype`, through a pinned
    buffer filled by the thread pool; chunk k's DMA overlaps the conversion of
    chunk k + 1 (all copies on the current stream).  `on_chunk(dev, a, b)` runs
    after rows [a, b) have been enqueued (device work on them can follow on the
    same stream while the host converts the next chunk)."""
    import torch
    pin = stage.get(tag, host.shape, dtype)
    dev = torch.empty(tuple(host.shape), dtype=dtype, device="cuda")
    n = host.shape[0]
    if chunks is None:
        chunks = _UPLOAD_CHUNKS
    chunks = max(1, min(chunks, n))
    if chunks == 4 and n >= 16:
        # the DMA outruns the conversion, so only the last chunk's copy is
        # exposed: shrinking chunks (40 / 30 / 20 / 10 %) leave a short one
        bounds = [0, n * 4 // 10, n * 7 // 10, n * 9 // 10, n]
    else:
        bounds = [n * i // chunks for i in range(chunks + 1)]
    hp = pin.numpy()
    for a, b in zip(bounds[:-1], bounds[1:]):
        copy(hp[a:b], host[a:b])
        dev[a:b].copy_(pin[a:b], non_blocking=True)
        if on_chunk is not None:
            on_chunk(dev, a, b)
    return dev


def download_blocks(stage: Staging, tag: str, dev, blocks, wait, out_dtype=np.float64, out=None):
    """CUDA tensor -> numpy array while it is still being produced: for each
    block (lo, hi) of axis 0, in order, `wait(k)` returns once block k is
    complete on the device; its rows are then copied to a pinned buffer on a
    copy stream, and a converter thread turns each landed block into the
    result dtype on the pool while later blocks still compute.  `out`: the
    result array, when the caller took it from `stage.result` beforehand (to
    build its views while the device is still busy)."""
    import queue
    import torch
    pin = stage.get(tag, dev.shape, dev.dtype)
    host = pin.numpy()
    if out is None:
        out = stage.result(tag, tuple(dev.shape), out_dtype)
    cs = stage.copy_stream()
    q: "queue.Queue" = queue.Queue()
    futs = []

    def converter():
        while True:
            item = q.get()
            if item is None:
                return
            ev, a, b = item
            ev.synchronize()
            if _native_convert(out[a:b], host[a:b]):
                continue
            parts = max(1, min(_THREADS, b - a))
            cuts = [a + (b - a) * i // parts for i in range(parts + 1)]
            for x, y in zip(cuts[:-1], cuts[1:]):
                if y > x:
                    futs.append(pool().submit(np.copyto, out[x:y], host[x:y], casting="unsafe"))

    th = threading.Thread(target=converter, daemon=True)
    th.start()
    try:
        for k, (a, b) in enumerate(blocks):
            wait(k)
            with torch.cuda.stream(cs):
                pin[a:b].copy_(dev[a:b], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cs)
            q.put((ev, a, b))
    finally:
        q.put(None)
        th.join()
    for f in futs:
        f.result()
    return out


def download(stage: Staging, tag: str, dev, out_dtype=np.float64, chunks: int = 4) -> np.ndarray:
    """CUDA tensor -> new numpy array of `out_dtype`: chunked async copies into
    a pinned buffer, each chunk converted while the next one is in flight."""
    import torch
    pin = stage.get(tag, dev.shape, dev.dtype)
    out = stage.result(tag, tuple(dev.shape), out_dtype)
    n = dev.shape[0]
    chunks = max(1, min(chunks, n))
    if chunks == 4 and n >= 16:
        # only the last chunk's conversion is exposed: shrinking chunks
        bounds = [0, n * 4 // 10, n * 7 // 10, n * 9 // 10, n]
    else:
        bounds = [n * i // chunks for i in range(chunks + 1)]
    s = torch.cuda.current_stream()
    events = []
    for a, b in zip(bounds[:-1], bounds[1:]):
        pin[a:b].copy_(dev[a:b], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(s)
        events.append(ev)
    host = pin.numpy()
    for (a, b), ev in zip(zip(bounds[:-1], bounds[1:]), events):
        ev.synchronize()
        copy(out[a:b], host[a:b])
    return out
