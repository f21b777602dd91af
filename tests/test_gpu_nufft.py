"""Device NUFFT (C ABI) against the reference's golden vectors: bit-exact
first-tap (bin) indices, scalings, type-2 / type-1 outputs, dot tests."""

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu

CASES = ["r3_j6", "r3_j3_odd", "r2_j5", "r1_j6", "r3_j8", "r3_big",
         "edge_j6", "edge_j3", "edge_j5_2d"]


@pytest.fixture(scope="module")
def nf():
    from paper_1605_05231_b200 import nufft
    return nufft


@pytest.mark.parametrize("name", CASES)
def test_first_indices_bit_exact(nf, nufft_cases, name):
    c = nufft_cases[name]
    dims = tuple(int(v) for v in c["dims"])
    plan = nf.plan_nufft(dims, c["nodes"], 2.0, tuple(int(v) for v in c["j"]))
    assert np.array_equal(plan.nodes, c["wrapped"])
    assert np.array_equal(plan.first_indices().astype(np.int64), c["first"])


@pytest.mark.parametrize("name", CASES)
def test_scaling_matches_reference(nf, nufft_cases, name):
    c = nufft_cases[name]
    dims = tuple(int(v) for v in c["dims"])
    plan = nf.plan_nufft(dims, c["nodes"], 2.0, tuple(int(v) for v in c["j"]))
    assert rel_l2(plan.scaling, c["scaling"]) < 1e-10


@pytest.mark.parametrize("name", CASES)
def test_type2_type1_match_reference(nf, nufft_cases, name):
    c = nufft_cases[name]
    dims = tuple(int(v) for v in c["dims"])
    plan = nf.plan_nufft(dims, c["nodes"], 2.0, tuple(int(v) for v in c["j"]))
    assert rel_l2(nf.nufft_forward(plan, c["x"]), c["fwd"]) < 1e-5
    assert rel_l2(nf.nufft_adjoint(plan, c["y"]), c["adj"]) < 1e-5


@pytest.mark.parametrize("dims", [(32,), (16, 16), (8, 8, 8), (20, 18, 16)])
def test_dot_test_fp32(nf, dims):
    rng = np.random.default_rng(9)
    nodes = rng.uniform(-np.pi, np.pi, (3000, len(dims)))
    plan = nf.plan_nufft(dims, nodes, 2.0, 6)
    x = rng.standard_normal(dims) + 1j * rng.standard_normal(dims)
    y = rng.standard_normal(3000) + 1j * rng.standard_normal(3000)
    lhs = np.vdot(y, nf.nufft_forward(plan, x))
    rhs = np.vdot(nf.nufft_adjoint(plan, y), x)
    assert abs(lhs - rhs) / abs(lhs) < 1e-5


def test_dot_test_config2_radial(nf):
    """Adjoint identity <A x, y> = <x, A^H y> at full config-2 sizes: the 33 M
    radial nodes of the 512 x 180 x 360 lattice on a 256^3 grid, J = 6
    (SURVEY 8(c) size-independent property; BASELINE config 1's dot check)."""
    from paper_1605_05231_b200 import radon_fourier as rf
    from paper_1605_05231_b200.geometry import RadialGridSpec
    n = 256
    spec = RadialGridSpec(512, 180, 360, 2.0)
    nodes = rf._radial_direction_nodes(spec, 2.0 / n)
    rng = np.random.default_rng(11)
    plan = nf.plan_nufft((n, n, n), nodes, 2.0, 6)
    x = (rng.standard_normal((n, n, n)) + 1j * rng.standard_normal((n, n, n))).astype(np.complex64)
    y = (rng.standard_normal(len(nodes)) + 1j * rng.standard_normal(len(nodes))).astype(np.complex64)
    lhs = np.vdot(y.astype(np.complex128), nf.nufft_forward(plan, x))
    rhs = np.vdot(nf.nufft_adjoint(plan, y), x.astype(np.complex128))
    assert abs(lhs - rhs) / abs(lhs) < 1e-5


def test_wrap_is_bitwise_numpy(nf):
    """Device remainder (fma-based fmod) == numpy's mod(x + pi, 2 pi) - pi, bit for bit."""
    rng = np.random.default_rng(3)
    k = rng.integers(-40, 40, 60000)
    vals = np.concatenate([
        rng.uniform(-20 * np.pi, 20 * np.pi, 100000),
        2 * np.pi * k / 64.0,                                   # grid-aligned
        np.nextafter(2 * np.pi * k / 64.0, np.inf),
        np.pi * rng.integers(-9, 9, 20000),                     # odd multiples of pi
        np.nextafter(np.pi * rng.integers(-9, 9, 20000), -np.inf),
        [0.0, -0.0, 1e-300, -1e-300, np.pi, -np.pi, 2 * np.pi, -2 * np.pi]])
    nodes = vals[: (vals.size // 3) * 3].reshape(-1, 3)
    plan = nf.plan_nufft((8, 8, 8), nodes, 2.0, 6)
    ref = np.mod(nodes + np.pi, 2.0 * np.pi) - np.pi
    got = plan.nodes
    assert np.array_equal(got.view(np.int64), ref.view(np.int64))


def test_validation_errors(nf):
    with pytest.raises(ValueError):
        nf.plan_nufft((8,), np.zeros((4, 2)), 2.0, 6)
    with pytest.raises(ValueError):
        nf.plan_nufft((8,), np.zeros((4, 1)), 0.5, 6)
    with pytest.raises(ValueError):
        nf.plan_nufft((8,), np.zeros((4, 1)), 2.0, 0)
    with pytest.raises(ValueError):
        nf.plan_nufft((8,), np.full((4, 1), np.nan), 2.0, 6)
    plan = nf.plan_nufft((8,), np.zeros((4, 1)), 2.0, 6)
    with pytest.raises(ValueError):
        nf.nufft_forward(plan, np.zeros(7))
    with pytest.raises(ValueError):
        nf.nufft_adjoint(plan, np.zeros(5))


def test_chunked_forward_matches_nudft(monkeypatch):
    """nufft_forward_chunked with 64-node sub-plans, each fitting its own
    scaling (the reference's test_nufft.py:80-92, _PLAN_CHUNK patched)."""
    import cbn_oracle as orc
    from paper_1605_05231_b200 import nufft
    monkeypatch.setattr(nufft, "_PLAN_CHUNK", 64)
    rng = np.random.default_rng(11)
    dims = (8, 8, 8)
    nodes = rng.uniform(-np.pi, np.pi, (200, 3))
    x = rng.standard_normal(dims) + 1j * rng.standard_normal(dims)
    ref = orc.nudft(dims, nodes, x)
    got = nufft.nufft_forward_chunked(dims, nodes, x, 2.0, 6)
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < 2e-5
    # the sub-plans are separate plans: chunk k equals a plan of its own nodes
    k = nufft.nufft_forward(nufft.plan_nufft(dims, nodes[64:128], 2.0, 6), x)
    assert np.array_equal(got[64:128], k)


def test_chunked_adjoint_is_adjoint_of_chunked_forward(monkeypatch):
    """(reference test_nufft.py:95-105) at fp32: dot test <= 1e-6."""
    from paper_1605_05231_b200 import nufft
    monkeypatch.setattr(nufft, "_PLAN_CHUNK", 64)
    rng = np.random.default_rng(12)
    dims = (8, 8, 8)
    nodes = rng.uniform(-np.pi, np.pi, (200, 3))
    x = rng.standard_normal(dims) + 1j * rng.standard_normal(dims)
    y = rng.standard_normal(200) + 1j * rng.standard_normal(200)
    lhs = np.vdot(y, nufft.nufft_forward_chunked(dims, nodes, x, 2.0, 3))
    rhs = np.vdot(nufft.nufft_adjoint_chunked(dims, nodes, y, 2.0, 3), x)
    assert abs(lhs - rhs) / abs(lhs) < 1e-6


def test_chunked_matches_oracle_per_chunk_scaling(monkeypatch):
    """Chunked forward/adjoint against the oracle's chunked restatement
    (oracle type2_chunked / type1_chunked, per-chunk LS scaling) at 1e-5."""
    import cbn_oracle as orc
    from paper_1605_05231_b200 import nufft
    monkeypatch.setattr(nufft, "_PLAN_CHUNK", 3000)
    rng = np.random.default_rng(13)
    dims = (16, 12, 10)
    nodes = rng.uniform(-np.pi, np.pi, (10000, 3))
    x = rng.standard_normal(dims) + 1j * rng.standard_normal(dims)
    y = rng.standard_normal(10000) + 1j * rng.standard_normal(10000)
    got = nufft.nufft_forward_chunked(dims, nodes, x, 2.0, 6)
    ref = orc.type2_chunked(dims, nodes, x, 2.0, 6, chunk=3000)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-5
    got = nufft.nufft_adjoint_chunked(dims, nodes, y, 2.0, 6)
    ref = orc.type1_chunked(dims, nodes, y, 2.0, 6, chunk=3000)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-5
