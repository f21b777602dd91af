"""Projector stages and operators on the device against the reference's
golden vectors (tests/golden/*.npz).  Contract: relative L2 <= 1e-4 (fp32);
the observed error is reported in each assertion message."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, rel_l2
from _cases import config_setup, small_setup

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module")
def pl():
    from paper_1605_05231_b200 import pipeline
    return pipeline


def to_nodes(lat):
    """reference lattice (rho, theta, phi) -> device node order (phi, theta, rho)"""
    return np.ascontiguousarray(np.asarray(lat).transpose(2, 1, 0))


def test_radial_lattice(pl, golden_n16):
    g = golden_n16
    geom, voxel, spec, cfg = small_setup()
    proj = pl.Projector(geom, cfg, 16, voxel, 1)
    lat = proj.radial_lattice(g["vol"]).cpu().numpy()
    err = rel_l2(lat, to_nodes(g["lattice"]))
    assert err < TOL, err


def test_resample_views(pl, golden_n16):
    g = golden_n16
    geom, voxel, spec, cfg = small_setup()
    per_view = cfg.n_mu * cfg.n_t
    proj = pl.Projector(geom, cfg, 16, voxel, 1, target_batch=3 * per_view)
    vals = proj.resample_views(to_nodes(g["lattice"]), 0, 3).cpu().numpy().ravel()
    ref = np.where(g["rs_valid"], np.real(g["rs_apply"]), 0.0)
    err = rel_l2(vals, ref)
    assert err < TOL, err


def test_grangeat_reverse(pl, golden_n16):
    g = golden_n16
    geom, voxel, spec, cfg = small_setup()
    proj = pl.Projector(geom, cfg, 16, voxel, 1)
    out = proj.grangeat_reverse(g["gr_values"][None].astype(np.float32)).cpu().numpy()[0]
    err = rel_l2(out, g["gr_reverse"])
    assert err < TOL, err


def test_grangeat_forward(pl, golden_n16):
    g = golden_n16
    geom, voxel, spec, cfg = small_setup()
    proj = pl.Projector(geom, cfg, 16, voxel, 2)
    out = proj.grangeat_forward(g["frames"][1:2].astype(np.float32)).cpu().numpy()[0]
    err = rel_l2(out, g["gr_forward"])
    assert err < TOL, err


@pytest.mark.parametrize("which", ["n16", "n12"])
def test_forward_project(pl, which, golden_n16, golden_n12):
    from paper_1605_05231_b200.phantom import Volume3D
    g = golden_n16 if which == "n16" else golden_n12
    n, views = int(g["n"]), int(g["views"])
    geom, voxel, spec, cfg = small_setup(n, views, "trilinear" if which == "n16" else "dirac")
    frames = pl.nufft_forward_project(Volume3D(g["vol"], voxel), geom, cfg)
    err = rel_l2(np.stack([f.data for f in frames]), g["frames"])
    assert err < TOL, err


def test_forward_project_batches(pl, golden_n16, monkeypatch):
    """Per-batch resample scalings (pipeline.py:105-110): 5-view batches."""
    from paper_1605_05231_b200.phantom import Volume3D
    g = golden_n16
    geom, voxel, spec, cfg = small_setup()
    monkeypatch.setattr(pl, "_TARGET_BATCH", cfg.n_mu * cfg.n_t * 5)
    frames = pl.nufft_forward_project(Volume3D(g["vol"], voxel), geom, cfg)
    err = rel_l2(np.stack([f.data for f in frames]), g["frames_b5"])
    assert err < TOL, err


@pytest.mark.parametrize("which", ["n16", "n12"])
def test_backproject(pl, which, golden_n16, golden_n12):
    from paper_1605_05231_b200.grangeat import DetectorFrame
    g = golden_n16 if which == "n16" else golden_n12
    n, views = int(g["n"]), int(g["views"])
    geom, voxel, spec, cfg = small_setup(n, views, "trilinear" if which == "n16" else "dirac")
    frames = [DetectorFrame(k, g["frames"][k], geom.pixel_mm) for k in range(views)]
    vol = pl.nufft_backproject(frames, geom, cfg, n, voxel)
    err = rel_l2(vol.data, g["bp"])
    assert err < TOL, err


def test_backproject_batches(pl, golden_n16, monkeypatch):
    from paper_1605_05231_b200.grangeat import DetectorFrame
    g = golden_n16
    geom, voxel, spec, cfg = small_setup()
    monkeypatch.setattr(pl, "_TARGET_BATCH", 4096)
    frames = [DetectorFrame(k, g["frames"][k], geom.pixel_mm) for k in range(12)]
    vol = pl.nufft_backproject(frames, geom, cfg, 16, voxel)
    err = rel_l2(vol.data, g["bp_b4"])
    assert err < TOL, err


def test_config0_forward_and_config1_backproject(pl):
    from paper_1605_05231_b200.grangeat import DetectorFrame
    from paper_1605_05231_b200.phantom import Volume3D
    z = np.load(os.path.join(GOLDEN, "config0.npz"))
    geom, voxel, spec, cfg = config_setup(0)
    frames = pl.nufft_forward_project(Volume3D(z["vol"], voxel), geom, cfg)
    got = np.stack([f.data for f in frames])
    err = rel_l2(got, z["frames"])
    worst = max(rel_l2(got[k], z["frames"][k]) for k in range(geom.n_views))
    assert err < TOL and worst < 2 * TOL, (err, worst)
    ref_frames = [DetectorFrame(k, z["frames"][k].astype(np.float64), geom.pixel_mm)
                  for k in range(geom.n_views)]
    vol = pl.nufft_backproject(ref_frames, geom, cfg, 64, voxel)
    err = rel_l2(vol.data, z["bp"])
    assert err < TOL, err


@pytest.mark.parametrize("name", ["pipeline_n16_v8", "pipeline_n12_v48", "pipeline_n12_v24"])
def test_rotation_aligned_geometries(pl, name):
    """2 n_phi / V integer: the views-in-lanes resample gather (k_resample_views) and the
    backprojector's column gather (k_rs_gather_cols; k_rs_gather_cols2 when 2 n_phi / V = 2,
    as at configs 2 and 3), with one and with several view batches."""
    from paper_1605_05231_b200.grangeat import DetectorFrame
    from paper_1605_05231_b200.phantom import Volume3D
    g = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    n, views = int(g["n"]), int(g["views"])
    geom, voxel, spec, cfg = small_setup(n, views)
    frames = pl.nufft_forward_project(Volume3D(g["vol"], voxel), geom, cfg)
    err = rel_l2(np.stack([f.data for f in frames]), g["frames"])
    assert err < TOL, err
    fr = [DetectorFrame(k, g["frames"][k], geom.pixel_mm) for k in range(views)]
    err = rel_l2(pl.nufft_backproject(fr, geom, cfg, n, voxel).data, g["bp"])
    assert err < TOL, err
    saved = pl._TARGET_BATCH
    try:
        pl._TARGET_BATCH = 4096
        err = rel_l2(pl.nufft_backproject(fr, geom, cfg, n, voxel).data, g["bp_b4"])
    finally:
        pl._TARGET_BATCH = saved
    assert err < TOL, err


def test_frame_count_mismatch(pl):
    geom, voxel, spec, cfg = small_setup()
    with pytest.raises(ValueError):
        pl.nufft_backproject([], geom, cfg, 16, voxel)


def test_repeated_calls_use_cached_plan_data(pl, golden_n16):
    """Second call reuses the cached batch scalings and den lattice."""
    from paper_1605_05231_b200.grangeat import DetectorFrame
    from paper_1605_05231_b200.phantom import Volume3D
    g = golden_n16
    geom, voxel, spec, cfg = small_setup()
    vol = Volume3D(g["vol"], voxel)
    f1 = np.stack([f.data for f in pl.nufft_forward_project(vol, geom, cfg)])
    f2 = np.stack([f.data for f in pl.nufft_forward_project(vol, geom, cfg)])
    assert rel_l2(f2, f1) < 1e-6
    frames = [DetectorFrame(k, g["frames"][k], geom.pixel_mm) for k in range(12)]
    b1 = pl.nufft_backproject(frames, geom, cfg, 16, voxel).data
    b2 = pl.nufft_backproject(frames, geom, cfg, 16, voxel).data
    assert rel_l2(b2, b1) < 1e-6 and rel_l2(b2, g["bp"]) < TOL


def test_results_held_by_the_caller_are_not_reused(pl, golden_n16):
    """The plan recycles its float64 result array only when the caller has
    dropped every frame of the previous call."""
    from paper_1605_05231_b200.phantom import Volume3D
    g = golden_n16
    geom, voxel, spec, cfg = small_setup()
    held = pl.nufft_forward_project(Volume3D(g["vol"], voxel), geom, cfg)
    snap = np.stack([f.data for f in held]).copy()
    other = pl.nufft_forward_project(Volume3D(2.0 * g["vol"], voxel), geom, cfg)
    assert not np.shares_memory(other[0].data, held[0].data)
    assert np.array_equal(np.stack([f.data for f in held]), snap)
    assert rel_l2(np.stack([f.data for f in other]), 2.0 * snap) < 1e-6
    del held, other
    a = pl.nufft_forward_project(Volume3D(g["vol"], voxel), geom, cfg)
    addr = a[0].data.__array_interface__["data"][0]
    assert np.array_equal(np.stack([f.data for f in a]), snap)
    del a
    b = pl.nufft_forward_project(Volume3D(g["vol"], voxel), geom, cfg)   # released -> recycled
    assert b[0].data.__array_interface__["data"][0] == addr
    assert np.array_equal(np.stack([f.data for f in b]), snap)


def test_staged_volume_upload_matches_plain_call(pl, golden_n16, golden_n12, monkeypatch):
    """The drop-in forward pads and 2D-transforms each uploaded chunk of the
    volume at once (cbn_forward_stage_volume + cbn_forward_project_staged_async);
    the frames equal those of the plain call, for even and odd chunk splits, and
    the staged entry point refuses a volume that was not staged in full."""
    import torch
    from paper_1605_05231_b200 import _device, _hostio, _lib
    from paper_1605_05231_b200.phantom import Volume3D
    for g, basis in ((golden_n16, "trilinear"), (golden_n12, "dirac")):
        n, views = int(g["n"]), int(g["views"])
        geom, voxel, spec, cfg = small_setup(n, views, basis)
        vol = Volume3D(g["vol"], voxel)
        monkeypatch.setattr(pl, "_STAGE_VOLUME", False)
        plain = np.stack([f.data for f in pl.nufft_forward_project(vol, geom, cfg)])
        monkeypatch.setattr(pl, "_STAGE_VOLUME", True)
        for chunks in (4, 3, 1):
            monkeypatch.setattr(_hostio, "_UPLOAD_CHUNKS", chunks)
            staged = np.stack([f.data for f in pl.nufft_forward_project(vol, geom, cfg)])
            assert rel_l2(staged, plain) < 1e-6, (n, chunks)
            assert rel_l2(staged, g["frames"]) < TOL
    # misuse: rows staged out of order / not in full
    geom, voxel, spec, cfg = small_setup()
    proj = pl.get_projector(geom, cfg, 16, voxel, pl._FORWARD)
    lib = _lib.load()
    v = torch.zeros((16, 16, 16), dtype=torch.float32, device="cuda")
    out = torch.empty((geom.n_views, geom.nu, geom.nv), dtype=torch.float32, device="cuda")
    assert lib.cbn_forward_stage_volume(proj._h, _device.ptr(v), 4, 8, proj._s) == _lib.CBN_EINVAL
    assert lib.cbn_forward_stage_volume(proj._h, _device.ptr(v), 0, 8, proj._s) == _lib.CBN_OK
    assert lib.cbn_forward_project_staged_async(proj._h, _device.ptr(out), 0, geom.n_views,
                                                proj._s) == _lib.CBN_EINVAL
    torch.cuda.synchronize()


def test_view_range_matches_full(pl, golden_n16):
    """Sharded view ranges (multi-GPU path) reproduce the full projection."""
    g = golden_n16
    geom, voxel, spec, cfg = small_setup()
    proj = pl.Projector(geom, cfg, 16, voxel, 1, target_batch=cfg.n_mu * cfg.n_t * 5)
    full = proj.forward(g["vol"]).cpu().numpy()
    parts = [proj.forward(g["vol"], lo, hi).cpu().numpy() for lo, hi in ((0, 3), (3, 7), (7, 12))]
    assert rel_l2(np.concatenate(parts), full) < 1e-6


@pytest.mark.parametrize("name", ["pipeline_n16", "pipeline_n12_v24"])
def test_backprojector_phases_shard_exactly(pl, name):
    """The three backprojector phases split over 'ranks' (view ranges and node
    parts, sums done here) reproduce the one-call backprojection -- the
    decomposition the NCCL all-reduces of backproject_sharded rely on."""
    g = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    n, views = int(g["n"]), int(g["views"])
    geom, voxel, spec, cfg = small_setup(n, views)
    proj = pl.Projector(geom, cfg, n, voxel, 2)
    import torch
    frames = torch.from_numpy(g["frames"].astype(np.float32)).cuda()
    one = proj.backproject(frames).cpu().numpy()
    for world in (2, 3):
        cuts = [views * r // world for r in range(world + 1)]
        lat = sum(proj.backproject_views(frames[cuts[r]:cuts[r + 1]], cuts[r], cuts[r + 1])
                  for r in range(world))
        grid = sum(proj.backproject_finish(lat.clone(), r, world) for r in range(world))
        got = proj.backproject_crop(grid).cpu().numpy()
        assert rel_l2(got, one) < 1e-5, world
    assert rel_l2(one, g["bp"]) < TOL


@pytest.mark.parametrize("name", ["pipeline_n16", "pipeline_n12_v24"])
def test_backprojector_slab_crop_exact(pl, name):
    """Slab-distributed phase 3 (what backproject_sharded runs under NCCL): the
    summed grid cut into x slabs (reduce-scatter, even and uneven splits), each
    slab's 2D IFFT + y/z crop written in the all-to-all send layout, the chunks
    routed to y ranges here, then x IFFT + crop per range -- equals the
    one-device crop of the whole grid."""
    import torch
    g = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    n, views = int(g["n"]), int(g["views"])
    geom, voxel, spec, cfg = small_setup(n, views)
    proj = pl.Projector(geom, cfg, n, voxel, 2)
    frames = torch.from_numpy(g["frames"].astype(np.float32)).cuda()
    grid = proj.backproject_finish(proj.backproject_views(frames, 0, views))
    one = proj.backproject_crop(grid.clone()).cpu().numpy()
    assert rel_l2(one, proj.backproject(frames).cpu().numpy()) < 1e-6
    k = round(grid.numel() ** (1 / 3))
    plane = k * k
    for world in (1, 2, 3, 4):
        xs, ys = pl.slab_ranges(k, world), pl.slab_ranges(n, world)
        sends = [proj.backproject_crop_slab(grid[xs[r] * plane: xs[r + 1] * plane].clone(),
                                            xs[r], xs[r + 1], world) for r in range(world)]
        parts = []
        for d in range(world):
            yc = ys[d + 1] - ys[d]
            chunks = []
            for r in range(world):
                xc = xs[r + 1] - xs[r]
                off = xc * ys[d] * n
                chunks.append(sends[r][off: off + xc * yc * n])
            parts.append(proj.backproject_crop_cols(torch.cat(chunks), ys[d], ys[d + 1]))
        got = torch.cat(parts, dim=1).cpu().numpy()
        assert rel_l2(got, one) < 1e-6, world
    with pytest.raises(ValueError):
        proj.backproject_crop_slab(grid[:plane].clone(), 0, k + 1, 1)


@pytest.mark.parametrize("name", ["pipeline_n16", "pipeline_n12_v24"])
def test_forward_phases_shard_exactly(pl, name):
    """Forward phases split over 'ranks' (radial-node parts summed, then view
    ranges) reproduce the one-call forward projection -- what the NCCL
    all-reduce of forward_sharded relies on."""
    import torch
    g = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    n, views = int(g["n"]), int(g["views"])
    geom, voxel, spec, cfg = small_setup(n, views)
    proj = pl.Projector(geom, cfg, n, voxel, 1)
    vol = torch.from_numpy(g["vol"]).cuda()
    one = proj.forward(vol).cpu().numpy()
    assert rel_l2(one, g["frames"]) < TOL
    for world in (1, 2, 3):
        lat = sum(proj.forward_lattice(vol, r, world) for r in range(world))
        cuts = [views * r // world for r in range(world + 1)]
        got = np.concatenate([proj.forward_views(lat.clone(), cuts[r], cuts[r + 1]).cpu().numpy()
                              for r in range(world)])
        assert rel_l2(got, one) < 1e-6, world


def test_radial_lattice_conjugate_pairs_at_wrap_ties(pl):
    """The spectrum gather computes one node per +-rho pair and writes the mirror
    as the conjugate; where the reference's wrapping or its exact support test
    is not symmetric (components at odd multiples of pi, u - J/2 an integer on
    one side only -- the CLI's default config has both: J = 3, n_rho = 54,
    rho_max = sqrt(3)), the plan keeps the pair apart.  Lattice vs the oracle."""
    import torch
    import cbn_oracle as orc
    from paper_1605_05231_b200 import io as cbio
    from paper_1605_05231_b200.config import make_projector_config
    io_dir = os.path.join(GOLDEN, "io")
    geom = cbio.load_geometry(os.path.join(io_dir, "geom.json"))
    vol = cbio.read_volume(os.path.join(io_dir, "vol.raw"))
    cfg = make_projector_config(geom, vol.n, "a")
    spec = cfg.radial_spec
    ref = orc.radial_lattice(vol.data, vol.voxel_mm, spec, cfg.spectrum_j, 2.0, cfg.basis)
    proj = pl.Projector(geom, cfg, vol.n, vol.voxel_mm, 1)
    got = proj.radial_lattice(torch.from_numpy(vol.data.astype(np.float32)).cuda())
    got = got.cpu().numpy().transpose(2, 1, 0)
    assert rel_l2(got, ref) < 1e-5


def test_backproject_staged_upload(pl, monkeypatch):
    """The drop-in backprojector stages the forward Grangeat step block by block
    while later frames upload (cbn_backproject_stage_views): 32-view blocks on
    the 48-view rotation-aligned geometry (one scaling group) give the one-call
    result and the reference's; a plan with several scaling groups refuses the
    staging (CBN_EUNSUPPORTED) and the call falls back."""
    import torch
    from paper_1605_05231_b200 import _device, _lib
    from paper_1605_05231_b200.grangeat import DetectorFrame
    g = dict(np.load(os.path.join(GOLDEN, "pipeline_n12_v48.npz")))
    n, views = int(g["n"]), int(g["views"])
    geom, voxel, spec, cfg = small_setup(n, views)
    fr = [DetectorFrame(k, g["frames"][k], geom.pixel_mm) for k in range(views)]
    monkeypatch.setattr(pl, "_BP_STAGE_VIEWS", 32)
    staged = pl.nufft_backproject(fr, geom, cfg, n, voxel).data
    proj = pl.get_projector(geom, cfg, n, voxel, pl._BACK)
    one = proj.backproject(torch.from_numpy(g["frames"].astype(np.float32)).cuda()).cpu().numpy()
    assert rel_l2(staged, one) < 1e-6
    assert rel_l2(staged, g["bp"]) < TOL
    # out-of-order staging is an argument error and leaves nothing staged
    dev = torch.from_numpy(g["frames"].astype(np.float32)).cuda()
    rc = _lib.load().cbn_backproject_stage_views(proj._h, _device.ptr(dev[32]), 32, 48, proj._s)
    assert rc == _lib.CBN_EINVAL
    assert rel_l2(proj.backproject(dev).cpu().numpy(), one) < 1e-6
    # 4096-target batches: several batches, still one scaling group here
    monkeypatch.setattr(pl, "_TARGET_BATCH", 4096)
    err = rel_l2(pl.nufft_backproject(fr, geom, cfg, n, voxel).data, g["bp_b4"])
    assert err < TOL, err
    # method B has no views-in-lanes column gather: refused, the call falls back
    gb = dict(np.load(os.path.join(GOLDEN, "pipeline_n12_b.npz")))
    nb_, vb = int(gb["n"]), int(gb["views"])
    geom_b, voxel_b, _, cfg_b = small_setup(nb_, vb)
    cfg_b.method = "b"
    proj_b = pl.get_projector(geom_b, cfg_b, nb_, voxel_b, pl._BACK)
    devb = torch.from_numpy(gb["frames"].astype(np.float32)).cuda()
    rc = _lib.load().cbn_backproject_stage_views(proj_b._h, _device.ptr(devb), 0, vb, proj_b._s)
    assert rc == _lib.CBN_EUNSUPPORTED
    frb = [DetectorFrame(k, gb["frames"][k], geom_b.pixel_mm) for k in range(vb)]
    err = rel_l2(pl.nufft_backproject(frb, geom_b, cfg_b, nb_, voxel_b).data, gb["bp"])
    assert err < TOL, err


def test_spectrum_records_match_node_generation(pl, golden_n16, monkeypatch):
    """The record-driven spectrum gather (k_spec_gather: per-plan KB arguments,
    tile offsets, epilogue factors) and the per-step node generation path
    (CBN_SPEC_RECORDS=0, k_gather_binned) give the same lattice, and both the
    reference's."""
    g = golden_n16
    geom, voxel, spec, cfg = small_setup()
    proj = pl.Projector(geom, cfg, 16, voxel, 1)
    rec = proj.radial_lattice(g["vol"]).cpu().numpy()
    monkeypatch.setenv("CBN_SPEC_RECORDS", "0")
    gen = proj.radial_lattice(g["vol"]).cpu().numpy()
    assert rel_l2(rec, gen) < 1e-6
    assert rel_l2(rec, to_nodes(g["lattice"])) < TOL


def test_backprojector_records_match_node_generation(pl, golden_n16, monkeypatch):
    """The record-driven 3D spread (BpRecSrc: per-plan KB arguments, tile
    offsets, lattice indices and factors of each primary node and its mirror)
    and the per-step node generation path (CBN_BP_RECORDS=0) agree, and both
    match the reference's backprojection."""
    import torch
    g = golden_n16
    geom, voxel, spec, cfg = small_setup()
    frames = torch.from_numpy(g["frames"].astype(np.float32)).cuda()
    proj = pl.Projector(geom, cfg, 16, voxel, 2)
    rec = proj.backproject(frames).cpu().numpy()
    monkeypatch.setenv("CBN_BP_RECORDS", "0")
    gen = proj.backproject(frames).cpu().numpy()
    assert rel_l2(rec, gen) < 1e-5
    assert rel_l2(rec, g["bp"]) < TOL


def test_transposed_resample_strips_match_columns(pl, monkeypatch):
    """The strip form of the backprojector's transposed-resample gather
    (k_rs_gather_strips: per rho plane, 4 theta columns merged by target) and
    the per-column gather (CBN_RS_STRIPS=0) give the same backprojection, on a
    geometry with the 2-cell view shift of configs 2/3 (k_rs_gather_cols2)."""
    import torch
    g = dict(np.load(os.path.join(GOLDEN, "pipeline_n12_v24.npz")))
    n, views = int(g["n"]), int(g["views"])
    geom, voxel, spec, cfg = small_setup(n, views)
    frames = torch.from_numpy(g["frames"].astype(np.float32)).cuda()
    strips = pl.Projector(geom, cfg, n, voxel, 2).backproject(frames).cpu().numpy()
    monkeypatch.setenv("CBN_RS_STRIPS", "0")
    cols = pl.Projector(geom, cfg, n, voxel, 2).backproject(frames).cpu().numpy()
    assert rel_l2(strips, cols) < 1e-5
    assert rel_l2(strips, g["bp"]) < TOL
