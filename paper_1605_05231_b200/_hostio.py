"""Host side of the drop-in operators: pinned staging and threaded dtype
conversion (plumbing, no numerics).

The reference API is numpy in / numpy out with float64 results
(``DetectorFrame``/``Volume3D`` store float64).  The device
path computes in float32, so every call converts on the host: float64 volume
-> float32 upload, float32 frames -> float64 results (and the reverse for the
backprojector).  Those conversions are split over a thread pool (numpy
releases the GIL inside ``copyto``) and go through pinned staging buffers that
each projector plan keeps, so the copies run at DMA speed and overlap the
conversion of the previous chunk.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_POOL: ThreadPoolExecutor | None = None
_THREADS = max(1, min(16, os.cpu_count() or 1))


def pool() -> ThreadPoolExecutor:
    global _POOL
    if _POOL is None:
        _POOL = ThreadPoolExecutor(max_workers=_THREADS, thread_name_prefix="cbn-host")
    return _POOL


def copy(dst: np.ndarray, src: np.ndarray, min_chunk: int = 1 << 18) -> None:
    """dst[...] = src (with dtype conversion), split along axis 0 over threads."""
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
    """Pinned host buffers of one projector plan, keyed by (tag, shape, dtype)."""

    def __init__(self):
        self._bufs = {}

    def get(self, tag: str, shape, dtype):
        import torch
        key = (tag, tuple(shape), dtype)
        b = self._bufs.get(key)
        if b is None:
            b = torch.empty(tuple(shape), dtype=dtype, pin_memory=True)
            self._bufs[key] = b
        return b


def upload(stage: Staging, tag: str, host: np.ndarray, dtype):
    """numpy (any real dtype) -> new CUDA tensor of `dtype`, through a pinned
    buffer filled by the thread pool."""
    import torch
    pin = stage.get(tag, host.shape, dtype)
    copy(pin.numpy(), host)
    return pin.to("cuda", non_blocking=True)


def download(stage: Staging, tag: str, dev, out_dtype=np.float64, chunks: int = 4) -> np.ndarray:
    """CUDA tensor -> new numpy array of `out_dtype`: chunked async copies into
    a pinned buffer, each chunk converted while the next one is in flight."""
    import torch
    pin = stage.get(tag, dev.shape, dev.dtype)
    out = np.empty(tuple(dev.shape), dtype=out_dtype)
    n = dev.shape[0]
    chunks = max(1, min(chunks, n))
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
