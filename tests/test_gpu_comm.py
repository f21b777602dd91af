"""The NCCL operators behind the C ABI (include/cbnufft_b200_comm.h) on one
GPU: a single-rank communicator runs the whole sharded orchestration
(broadcast, node-share lattice + all-reduce, view range; views, accumulator
all-reduce, node-share spread, crop) and must reproduce the one-device
operators.  The multi-rank collectives (reduce-scatter by slab, grouped
send/recv, all-gather) mirror pipeline.sharded_crop, whose decomposition is
checked in tests/test_gpu_projector.py and tests/test_dist_gloo.py."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, rel_l2
from _cases import small_setup

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module")
def comm():
    from paper_1605_05231_b200.comm import NcclComm
    c = NcclComm.local()
    yield c
    c.close()


def test_single_rank_sharded_operators(comm):
    import torch
    from paper_1605_05231_b200 import pipeline as pl
    g = dict(np.load(os.path.join(GOLDEN, "pipeline_n12_v24.npz")))
    n, views = int(g["n"]), int(g["views"])
    geom, voxel, spec, cfg = small_setup(n, views)
    proj = pl.Projector(geom, cfg, n, voxel, 3)
    vol = torch.from_numpy(g["vol"].astype(np.float32)).cuda().contiguous()
    full = proj.forward(vol).cpu().numpy()
    got = comm.forward_project(proj, vol, 0, views).cpu().numpy()
    assert rel_l2(got, full) < 1e-6
    assert rel_l2(got, g["frames"]) < TOL
    part = comm.forward_project(proj, vol, 5, 17).cpu().numpy()
    assert rel_l2(part, full[5:17]) < 1e-6
    frames = torch.from_numpy(g["frames"].astype(np.float32)).cuda()
    one = proj.backproject(frames).cpu().numpy()
    bp = comm.backproject(proj, frames, 0, views).cpu().numpy()
    assert rel_l2(bp, one) < 1e-5
    assert rel_l2(bp, g["bp"]) < TOL
    with pytest.raises(ValueError):
        comm.forward_project(proj, vol, 0, views + 1)


def test_node_sharded_lattice_blocks_assemble_the_lattice():
    """Node-sharded forward plans (cbn_projector_set_node_shard): each share
    writes only its contiguous lattice block; the blocks in rank order (what
    the in-place NCCL all-gather of cbn_forward_project_sharded assembles) are
    the unsharded lattice, and a sharded plan refuses the other entry points."""
    import torch
    from paper_1605_05231_b200 import pipeline as pl
    g = dict(np.load(os.path.join(GOLDEN, "pipeline_n12_v24.npz")))
    n, views = int(g["n"]), int(g["views"])
    geom, voxel, spec, cfg = small_setup(n, views)
    vol = torch.from_numpy(g["vol"].astype(np.float32)).cuda().contiguous()
    full = pl.Projector(geom, cfg, n, voxel, 1).forward_lattice(vol).cpu().numpy()
    lines = spec.n_theta * spec.n_phi
    for nparts in (2, 3, 4):
        if lines % nparts:
            continue
        blocks = []
        for part in range(nparts):
            proj = pl.Projector(geom, cfg, n, voxel, 1)
            lo, hi = proj.set_node_shard(part, nparts)
            assert hi - lo == full.size // nparts and lo == part * (hi - lo)
            lat = proj.forward_lattice(vol, part, nparts).cpu().numpy()
            blocks.append(lat[lo:hi])
            with pytest.raises(ValueError):
                proj.forward(vol)
        got = np.concatenate(blocks)
        assert np.max(np.abs(got - full)) <= 1e-6 * np.max(np.abs(full))
    proj = pl.Projector(geom, cfg, n, voxel, 1)
    with pytest.raises(NotImplementedError):
        proj.set_node_shard(0, lines + 1)
