"""Module-level drop-in API on the device (radon_fourier, resampling, grangeat):
parity with the reference's golden stage outputs, plus the reference tests'
own analytic and adjoint properties re-expressed at fp32 tolerances."""

import numpy as np
import pytest

from conftest import rel_l2
from _cases import small_setup

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module")
def rf():
    from paper_1605_05231_b200 import radon_fourier
    return radon_fourier


@pytest.fixture(scope="module")
def rs():
    from paper_1605_05231_b200 import resampling
    return resampling


@pytest.fixture(scope="module")
def gr():
    from paper_1605_05231_b200 import grangeat
    return grangeat


def test_radial_spectrum_golden(rf, golden_n16):
    from paper_1605_05231_b200.phantom import Volume3D
    g = golden_n16
    geom, voxel, spec, cfg = small_setup()
    got = rf.image_to_radial_spectrum(Volume3D(g["vol"], voxel), spec, j=6).data
    err = rel_l2(got, g["spectrum"])
    assert err < TOL, err


def test_radial_spectrum_direct_sum(rf):
    """Every radial node equals the voxel-centre DFT sum (pkg/tests/test_radon_fourier.py:25-38)."""
    from paper_1605_05231_b200.geometry import RadialGridSpec
    from paper_1605_05231_b200.phantom import Volume3D
    n = 8
    rng = np.random.default_rng(30)
    vol = Volume3D(rng.standard_normal((n, n, n)), 1.5)
    spec = RadialGridSpec(10, 5, 4, n * 1.5 * np.sqrt(3) / 2.0)
    got = rf.image_to_radial_spectrum(vol, spec, j=8).data
    nodes = rf._radial_direction_nodes(spec, vol.voxel_mm)
    c = np.arange(n) - n / 2.0 + 0.5
    pts = np.stack([a.ravel() for a in np.meshgrid(c, c, c, indexing="ij")], axis=-1)
    ref = (np.exp(-1j * nodes @ pts.T) @ vol.data.ravel()).reshape(
        spec.n_phi, spec.n_theta, spec.n_rho).transpose(2, 1, 0)
    assert np.max(np.abs(got - ref)) < 2e-6 * np.max(np.abs(ref))
    # zero-frequency node = voxel sum (test_radon_fourier.py:41-47)
    assert np.allclose(got[spec.n_rho // 2], vol.data.sum(), rtol=1e-5)


def test_radial_spectrum_config2_separable(rf):
    """Full config-2 sizes (256^3 volume, 512 x 180 x 360 = 33 M radial nodes,
    J = 6, 16 sub-plans): the device spectrum against the exact voxel-centre
    DFT of a separable volume -- the sum factorises per axis, so it is cheap at
    any size -- on 20 000 seeded nodes (size-independent property)."""
    from paper_1605_05231_b200.geometry import RadialGridSpec
    from paper_1605_05231_b200.phantom import Volume3D
    n = 256
    voxel = 2.0 / n
    rng = np.random.default_rng(40)
    a, b, c = rng.standard_normal((3, n))
    vol = a[:, None, None] * b[None, :, None] * c[None, None, :]
    spec = RadialGridSpec(512, 180, 360, 512 * voxel / 2.0)
    got = rf.image_to_radial_spectrum(Volume3D(vol, voxel), spec, j=6).data
    nodes = rf._radial_direction_nodes(spec, voxel)
    idx = rng.choice(len(nodes), 20000, replace=False)
    w = nodes[idx]
    cc = np.arange(n) - n / 2.0 + 0.5
    ref = ((np.exp(-1j * np.outer(w[:, 0], cc)) @ a) * (np.exp(-1j * np.outer(w[:, 1], cc)) @ b)
           * (np.exp(-1j * np.outer(w[:, 2], cc)) @ c))
    ir, it, ip = idx % 512, (idx // 512) % 180, idx // (512 * 180)
    assert rel_l2(got[ir, it, ip], ref) < TOL
    # zero-frequency nodes = the voxel sum
    assert np.allclose(got[256], vol.sum(), rtol=1e-4)


def test_radial_fft_roundtrip_and_lattice(rf, golden_n16):
    from paper_1605_05231_b200.geometry import RadialGridSpec
    spec = RadialGridSpec(16, 4, 4, 2.0)
    rng = np.random.default_rng(32)
    r = rf.RadialRadon3D(spec, rng.standard_normal((16, 4, 4)).astype(complex))
    back = rf.radial_ifft(rf.radial_fft(r))
    assert np.max(np.abs(back.data - r.data)) < 1e-6
    # the golden lattice chain from the golden spectrum
    g = golden_n16
    geom, voxel, spec16, cfg = small_setup()
    s = rf.RadialSpectrum3D(spec16, g["spectrum"] * rf.trilinear_transfer(spec16, voxel))
    lat = rf.radial_ifft(rf.spectral_rho_derivative(s)).data
    assert rel_l2(lat, g["lattice"]) < TOL


def test_resample_apply_transpose_golden(rs, golden_n16):
    g = golden_n16
    geom, voxel, spec, cfg = small_setup()
    plan = rs.plan_resample(spec, g["rs_targets"], "a", rho_pad=cfg.rho_pad, j=cfg.resample_j)
    got = rs.resample_apply(plan, g["lattice"])
    err = rel_l2(got, g["rs_apply"])
    assert err < TOL, err
    got_t = rs.resample_transpose(plan, g["rs_y"])
    err_t = rel_l2(got_t, g["rs_transpose"])
    assert err_t < TOL, err_t


def test_resample_exact_at_nodes_and_adjoint(rs):
    """Method A reproduces lattice values at integer targets and is the exact
    adjoint of its transpose (pkg/tests/test_resampling.py:75-87,142-151)."""
    from paper_1605_05231_b200.geometry import RadialGridSpec
    spec = RadialGridSpec(16, 12, 10, 1.0)
    dims = (16, 12, 10)
    rng = np.random.default_rng(24)
    # lower-band data with a constant origin row (the reference tests' construction)
    spec_d = np.zeros(dims, dtype=np.complex128)
    sl = tuple(slice(0, max(1, d // 2 - 1)) for d in dims)
    spec_d[sl] = rng.standard_normal(spec_d[sl].shape) + 1j * rng.standard_normal(spec_d[sl].shape)
    data = np.fft.ifftn(spec_d)
    data = data - (data[8] - data[8].mean())[None]
    data = np.real(data)
    tg = np.stack(np.meshgrid(*[np.arange(d) for d in dims], indexing="ij"), -1).reshape(-1, 3)[::7]
    plan = rs.plan_resample(spec, tg.astype(float), "a")
    got = np.real(rs.resample_apply(plan, data))
    ref = data[tg[:, 0], tg[:, 1], tg[:, 2]]
    assert np.max(np.abs(got - ref)) < 1e-5 * max(1.0, np.max(np.abs(ref)))
    targets = rng.uniform(0, 1, (300, 3)) * np.array(dims, dtype=float)
    targets[:, 0] = rng.uniform(2.5, 16 - 2.5, 300)
    plan = rs.plan_resample(spec, targets, "a")
    x = rng.standard_normal(dims) + 1j * rng.standard_normal(dims)
    y = rng.standard_normal(300) + 1j * rng.standard_normal(300)
    lhs = np.vdot(y, rs.resample_apply(plan, x))
    rhs = np.vdot(rs.resample_transpose(plan, y), x)
    assert abs(lhs - rhs) / abs(lhs) < 1e-5


def test_resample_validation(rs):
    from paper_1605_05231_b200.geometry import RadialGridSpec
    spec = RadialGridSpec(16, 12, 10, 1.0)
    with pytest.raises(ValueError):
        rs.plan_resample(spec, np.zeros((4, 2)), "a")
    with pytest.raises(ValueError):
        rs.plan_resample(spec, np.zeros((4, 3)), "c")
    with pytest.raises(ValueError):
        rs.plan_resample(spec, np.full((4, 3), -5.0), "a")
    with pytest.raises(ValueError):
        rs.plan_resample(spec, np.zeros((4, 3)), "b", side_lobes=8)
    plan = rs.plan_resample(spec, np.zeros((4, 3)), "a")
    with pytest.raises(ValueError):
        rs.resample_apply(plan, np.zeros((3, 3, 3)))
    with pytest.raises(ValueError):
        rs.resample_transpose(plan, np.zeros(5))


def test_grangeat_views_golden(gr, golden_n16):
    g = golden_n16
    geom, voxel, spec, cfg = small_setup()
    gp = gr.plan_grangeat(geom, cfg.n_mu, cfg.n_t, t_pitch_mm=cfg.t_pitch_mm, t_taper=cfg.t_taper)
    coords = tuple(np.zeros((cfg.n_mu, cfg.n_t)) for _ in range(3))
    frame = gr.reverse_grangeat_view(gr.UmbrellaView(1, g["gr_values"], coords), gp)
    assert rel_l2(frame.data, g["gr_reverse"]) < TOL
    gpb = gr.plan_grangeat(geom, cfg.n_mu, 2 * geom.nu)
    view = gr.forward_grangeat_view(gr.DetectorFrame(1, g["frames"][1], geom.pixel_mm), gpb)
    assert rel_l2(view.values, g["gr_forward"]) < TOL
    assert view.coords[0].shape == (cfg.n_mu, 2 * geom.nu)


def test_fbp2d_roundtrip(rf):
    """Radial spectrum -> NUFFT FBP recovers a smooth image, device NUFFTs
    (pkg/tests/test_radon_fourier.py:130-143)."""
    n = 32
    c = (np.arange(n) - n / 2.0 + 0.5) / (n / 2.0)
    xx, yy = np.meshgrid(c, c, indexing="ij")
    img = np.maximum(1.0 - (xx ** 2 + yy ** 2) / 0.49, 0.0) ** 2
    spec = rf.image_to_radial_spectrum_2d(img, 2 * n, 100)
    rec, imag_ratio = rf.fbp2d_nufft(spec, n)
    assert imag_ratio < 1e-3
    mask = xx ** 2 + yy ** 2 <= 1.0
    assert np.mean(np.abs(rec - img)[mask]) / np.mean(np.abs(img[mask])) < 0.05
