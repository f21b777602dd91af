"""Device plumbing: torch tensors as containers, the current CUDA stream, and
the scaling-fit row subsample (the numpy generator is part of the reference's
numerics, nufft.py:163-168, so the host draws it and hands it to the device).
"""

from __future__ import annotations

import functools

import numpy as np

LS_SAMPLES = 8192


def torch():
    import torch as _t
    return _t


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("paper_1605_05231_b200 needs a CUDA device (B200); "
                           "there is no CPU fallback")
    return t


def stream_ptr() -> int:
    t = require_cuda()
    return int(t.cuda.current_stream().cuda_stream)


def ptr(tensor) -> int:
    return int(tensor.data_ptr())


@functools.lru_cache(maxsize=64)
def ls_rows(m: int) -> np.ndarray:
    """Rows of the least-squares scaling fit for an m-node plan."""
    if m > LS_SAMPLES:
        sel = np.random.default_rng(0).choice(m, LS_SAMPLES, replace=False)
        sel.sort()
        return sel.astype(np.int64)
    return np.arange(m, dtype=np.int64)


def to_device(a, dtype):
    """numpy (any real/complex dtype) or torch tensor -> contiguous CUDA tensor."""
    t = require_cuda()
    if isinstance(a, t.Tensor):
        return a.to(device="cuda", dtype=dtype).contiguous()
    arr = np.asarray(a)
    if dtype == t.complex64:
        arr = arr.astype(np.complex64, copy=False)
    elif dtype == t.float32:
        arr = arr.astype(np.float32, copy=False)
    host = t.from_numpy(np.ascontiguousarray(arr))
    return host.to("cuda", non_blocking=False)
