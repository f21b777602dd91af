"""Host-side helpers of the sweep (analysis.py:20-100): the reference test
suite's own checks (pkg/tests/test_analysis.py:14-71) against this package."""

import numpy as np
import pytest

from paper_1605_05231_b200.analysis import (SamplingRates, SweepResult, inscribed_disk_mask,
                                            masked_error_metrics, nyquist_rates, sinogram_rates)


def test_nyquist_rates():
    dx, nx = nyquist_rates(1.0, 32.0 * np.pi)
    assert dx == pytest.approx(1.0 / 32.0)
    assert nx == pytest.approx(64.0)
    for bad in ((-1.0, 1.0), (1.0, 0.0)):
        with pytest.raises(ValueError):
            nyquist_rates(*bad)


def test_sinogram_rates_n128_budget():
    w_max = 64.0 * np.pi
    r = sinogram_rates(1.0, w_max)
    assert (r.n_rho, r.n_theta) == (128, 403)
    assert r.delta_theta == pytest.approx(np.pi / (w_max + 1.0))
    h = sinogram_rates(1.0, w_max, hexagonal=True)
    assert (h.n_rho, h.n_theta) == (256, 256)
    assert h.delta_rho == pytest.approx(nyquist_rates(1.0, w_max)[0] / 2.0)


def test_validation():
    for args, kw in (((0, 4, 1.0, 1.0), {}), ((4, 4, -1.0, 1.0), {}), ((4, 4, 1.0, 1.0), {"n_phi": 0})):
        with pytest.raises(ValueError):
            SamplingRates(*args, **kw)
    with pytest.raises(ValueError):
        SweepResult([(32, 1.0), (16, 2.0)], 16)
    SweepResult([(16, 2.0), (32, 1.0)], 32)


def test_mask_and_metrics():
    m = inscribed_disk_mask(16)
    assert m[8, 8] and not m[0, 0] and m.sum() == np.sum(
        ((np.arange(16) - 7.5)[:, None] ** 2 + (np.arange(16) - 7.5)[None, :] ** 2) <= 64.0)
    a = np.array([[1.0, 2.0], [3.0, 4.0]])
    b = np.ones((2, 2))
    mask = np.array([[True, True], [False, True]])
    mean_abs, rmse, max_abs = masked_error_metrics(a, b, mask)
    assert mean_abs == pytest.approx(4.0 / 3.0)
    assert rmse == pytest.approx(np.sqrt(10.0 / 3.0))
    assert max_abs == 3.0
    with pytest.raises(ValueError):
        masked_error_metrics(a, b, np.zeros((2, 2), dtype=bool))
    with pytest.raises(ValueError):
        masked_error_metrics(a, b[:1], np.ones((2, 2), dtype=bool))
