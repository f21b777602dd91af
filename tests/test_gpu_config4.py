"""Config 4 (BASELINE.json configs[4]): unstructured-point NUFFT stress case,
KB width 8, sigma 2, float32 nodes i.i.d. uniform in [-pi, pi)^3.

The float32-node plan (cbn_nufft_create_f32) must be the float64 plan of the
same values, bit for bit; its type-2 / type-1 outputs match the oracle and the
direct DFT (separable, oracle/cbn_oracle.py:254) to <= 1e-5 relative L2, the
tolerance BASELINE.json states for this configuration."""

import numpy as np
import pytest

import cbn_oracle as orc
from conftest import rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nf():
    from paper_1605_05231_b200 import nufft
    return nufft


def _points(m, seed):
    rng = np.random.default_rng(seed)
    pts = rng.uniform(-np.pi, np.pi, (m, 3)).astype(np.float32)
    # bin-boundary and wrap edge values in float32
    edge = np.float32([np.pi, -np.pi, 0.0, np.nextafter(np.float32(np.pi), np.float32(0)),
                       2 * np.pi / 48, -2 * np.pi / 48 * 7, 1e-30])
    block = np.stack([np.roll(edge, k) for k in range(3)], axis=1)
    pts[: block.shape[0]] = block
    return pts


def _first_mod_k(ref):
    return np.stack([np.mod(f, k) for f, k in zip(ref.first, ref.kdims)], axis=1).astype(np.int64)


def _grid(dims, seed):
    rng = np.random.default_rng(seed)
    return ((rng.standard_normal(dims) + 1j * rng.standard_normal(dims)) / np.sqrt(2)).astype(np.complex64)


def test_f32_plan_is_f64_plan(nf):
    dims = (24, 20, 16)
    pts = _points(40000, 1)
    p32 = nf.plan_nufft(dims, pts, 2.0, 8)
    p64 = nf.plan_nufft(dims, pts.astype(np.float64), 2.0, 8)
    assert np.array_equal(p32.nodes, p64.nodes)
    assert np.array_equal(p32.first_indices(), p64.first_indices())
    assert np.array_equal(p32.scaling, p64.scaling)
    x = _grid(dims, 2)
    y = _grid((40000,), 3)
    assert np.array_equal(nf.nufft_forward(p32, x), nf.nufft_forward(p64, x))
    # the spread's global flush is atomic, so summation order (not the plan) varies
    assert rel_l2(nf.nufft_adjoint(p32, y), nf.nufft_adjoint(p64, y)) < 1e-6


def test_j8_matches_oracle(nf):
    dims = (24, 20, 16)
    pts = _points(20000, 4)
    nodes = pts.astype(np.float64)
    ref = orc.make_plan(dims, nodes, 2.0, 8)
    plan = nf.plan_nufft(dims, pts, 2.0, 8)
    assert np.array_equal(plan.first_indices().astype(np.int64), _first_mod_k(ref))
    assert rel_l2(plan.scaling, ref.scaling_grid().ravel()) < 1e-10
    x = _grid(dims, 5).astype(np.complex128)
    y = _grid((20000,), 6).astype(np.complex128)
    assert rel_l2(nf.nufft_forward(plan, x), orc.type2(ref, x)) < 1e-5
    assert rel_l2(nf.nufft_adjoint(plan, y), orc.type1(ref, y)) < 1e-5


def test_config4_grid_direct_dft(nf):
    """256^3 CN(0,1) grid as in config 4, 1M float32 points; type-2 at 2000
    points against the separable direct DFT, type-1 at 48 grid entries against
    the direct adjoint sum, and the dot test over all points."""
    from paper_1605_05231_b200.workloads import config4_inputs
    x, pts = config4_inputs(n_points=1 << 20)
    dims = x.shape
    plan = nf.plan_nufft(dims, pts, 2.0, 8)
    y_all = nf.nufft_forward(plan, x)
    sel = np.random.default_rng(7).choice(pts.shape[0], 2000, replace=False)
    w = orc.wrap(pts[sel].astype(np.float64))
    ref = orc.separable_dft(x.astype(np.complex128), w)
    assert rel_l2(y_all[sel], ref) < 1e-5
    # adjoint: x_adj[n] = sum_p y_p exp(+i w_p . n)
    rng = np.random.default_rng(8)
    y = ((rng.standard_normal(pts.shape[0]) + 1j * rng.standard_normal(pts.shape[0])) / np.sqrt(2))
    xa = nf.nufft_adjoint(plan, y)
    wall = orc.wrap(pts.astype(np.float64))
    idx = rng.integers(0, 256, (48, 3))
    direct = np.array([np.sum(y * np.exp(1j * (wall @ n.astype(np.float64)))) for n in idx])
    got = xa[idx[:, 0], idx[:, 1], idx[:, 2]]
    assert rel_l2(got, direct) < 1e-5
    lhs = np.vdot(y, y_all)
    rhs = np.vdot(xa, x.astype(np.complex128))
    assert abs(lhs - rhs) / abs(lhs) < 1e-5


def test_2d_binned_paths(nf):
    """2D plans take the binned gather/spread too (tile 16)."""
    dims = (40, 36)
    rng = np.random.default_rng(11)
    nodes = rng.uniform(-np.pi, np.pi, (30000, 2))
    ref = orc.make_plan(dims, nodes, 2.0, 5)
    plan = nf.plan_nufft(dims, nodes, 2.0, 5)
    assert np.array_equal(plan.first_indices().astype(np.int64), _first_mod_k(ref))
    x = rng.standard_normal(dims) + 1j * rng.standard_normal(dims)
    y = rng.standard_normal(30000) + 1j * rng.standard_normal(30000)
    assert rel_l2(nf.nufft_forward(plan, x), orc.type2(ref, x)) < 1e-5
    assert rel_l2(nf.nufft_adjoint(plan, y), orc.type1(ref, y)) < 1e-5


def test_config4_full_size_10k_direct_dft(nf):
    """BASELINE config 4 at full size: all 100M float32 points (seed 5) on the
    256^3 CN(0,1) grid (seed 4), KB J=8, sigma 2.  Type 2 at 10,000 points
    drawn from the whole set against the separable direct DFT (<= 1e-5, the
    tolerance BASELINE.json states); type 1 through the dot test over all
    100M points.  Inputs and outputs stay on the device."""
    import torch
    from paper_1605_05231_b200.workloads import config4_inputs
    x, pts = config4_inputs()
    assert pts.shape == (100_000_000, 3)
    plan = nf.plan_nufft(x.shape, pts, 2.0, 8)
    xd = torch.from_numpy(x).cuda()
    y = nf.nufft_forward(plan, xd)
    sel = np.sort(np.random.default_rng(9).choice(pts.shape[0], 10_000, replace=False))
    got = y[torch.from_numpy(sel).cuda()].cpu().numpy()
    ref = orc.separable_dft(x.astype(np.complex128), orc.wrap(pts[sel].astype(np.float64)))
    err = rel_l2(got, ref)
    assert err < 1e-5, err
    g = torch.Generator(device="cuda").manual_seed(10)
    yr = torch.complex(torch.randn(pts.shape[0], generator=g, device="cuda"),
                       torch.randn(pts.shape[0], generator=g, device="cuda")) / np.sqrt(2)
    xa = nf.nufft_adjoint(plan, yr)
    lhs = torch.vdot(yr.to(torch.complex128), y.to(torch.complex128)).item()
    rhs = torch.vdot(xa.to(torch.complex128).ravel(), xd.to(torch.complex128).ravel()).item()
    assert abs(lhs - rhs) / abs(lhs) < 1e-5
