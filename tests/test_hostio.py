"""Host conversions of the drop-in operators (csrc/cbn_hostio.cu, no GPU
needed): float64 frames gathered into float32 staging, float32 results widened
to float64 -- exact IEEE conversions, bit-identical to numpy's casts."""

import numpy as np

from paper_1605_05231_b200 import _hostio


def test_gather_frames_matches_numpy_cast():
    rng = np.random.default_rng(0)
    frames = [rng.standard_normal((37, 41)) * 10.0 ** rng.integers(-30, 30) for _ in range(9)]
    dst = np.empty((9, 37, 41), np.float32)
    _hostio.gather_frames(dst, frames)
    assert np.array_equal(dst, np.stack(frames).astype(np.float32))
    # non-contiguous sources take the numpy path
    dst2 = np.empty((9, 37, 21), np.float32)
    _hostio.gather_frames(dst2, [f[:, ::2] for f in frames])
    assert np.array_equal(dst2, np.stack([f[:, ::2] for f in frames]).astype(np.float32))


def test_copy_widen_and_narrow():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((130, 1000)).astype(np.float32)
    y = np.empty(x.shape, np.float64)
    _hostio.copy(y, x)
    assert np.array_equal(y, x.astype(np.float64))
    z = np.empty(x.shape, np.float32)
    _hostio.copy(z, y * 3.0)
    assert np.array_equal(z, (y * 3.0).astype(np.float32))
    special = np.array([np.inf, -np.inf, np.nan, 1e-300, -0.0, 3.4e39], np.float64)
    out = np.empty(6, np.float32)
    _hostio.copy(out, special)
    assert np.array_equal(out, special.astype(np.float32), equal_nan=True)


def test_frame_pointer_table_blocks():
    """The backprojector's pointer table: ranges of it convert like numpy's
    cast; a frame of another dtype, shape or layout sends the caller to the
    general route."""
    rng = np.random.default_rng(2)
    frames = [rng.standard_normal((19, 23)) for _ in range(11)]
    table = _hostio.frame_pointers(frames, (19, 23))
    assert table is not None
    dst = np.zeros((11, 19, 23), np.float32)
    _hostio.gather_block(dst[0:4], table, 0, 4)
    _hostio.gather_block(dst[4:11], table, 4, 11)
    assert np.array_equal(dst, np.stack(frames).astype(np.float32))
    assert _hostio.frame_pointers(frames[:3] + [frames[3].astype(np.float32)], (19, 23)) is None
    assert _hostio.frame_pointers([f[:, ::2] for f in frames], (19, 12)) is None
    assert _hostio.frame_pointers(frames, (19, 24)) is None


def test_widen_unaligned_and_odd_lengths():
    """The streaming-store widening handles any destination alignment and tail."""
    rng = np.random.default_rng(3)
    base_src = rng.standard_normal(100_003).astype(np.float32)
    base_dst = np.empty(100_010, np.float64)
    for off in range(5):
        for n in (0, 1, 7, 8, 9, 16_385, 99_990):
            src = base_src[off:off + n]
            dst = base_dst[off:off + n]
            dst[...] = -1.0
            _hostio.copy(dst, src)
            assert np.array_equal(dst, src.astype(np.float64))
