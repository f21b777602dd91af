"""World-size-2 gloo tests of the view-sharded forward path (CPU only).

Each rank projects its batch-aligned view range -- here with the CPU oracle
standing in for the device operator -- the blocks are all-gathered, and the
result must equal the single-process projection; the timing reduction is the
max over ranks.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from _cases import small_setup


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_path):
    import sys
    import torch
    import torch.distributed as dist
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [here, os.path.dirname(here), os.path.join(os.path.dirname(here), "oracle")]
    import cbn_oracle as orc
    from paper_1605_05231_b200 import sharding
    from paper_1605_05231_b200.phantom import random_ellipsoid_phantom
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    geom, voxel, spec, cfg = small_setup(12, 8, "dirac")
    vol = random_ellipsoid_phantom(12, 4, 7)
    per_view = cfg.n_mu * cfg.n_t
    target = per_view * 3                     # 3-view batches: (0,3) (3,6) (6,8)
    batches = sharding.view_batches(geom.n_views, per_view, target)
    lo, hi = sharding.view_shard(geom.n_views, world, rank, batches)
    local = orc.forward_project(vol, voxel, geom, cfg, target_batch=target,
                                views=set(range(lo, hi)))
    full = sharding.gather_views(torch.from_numpy(local), geom.n_views)
    t = sharding.max_over_ranks(1.0 + rank)
    if rank == 0:
        np.savez(result_path, full=full.numpy(), t=t, lo=lo, hi=hi)
    dist.barrier()
    dist.destroy_process_group()


def test_view_shard_ranges():
    from paper_1605_05231_b200 import sharding
    b = sharding.view_batches(360, 786432, 1 << 20)
    assert len(b) == 360
    ranges = [sharding.view_shard(360, 8, r, b) for r in range(8)]
    assert ranges[0][0] == 0 and ranges[-1][1] == 360
    assert all(ranges[i][1] == ranges[i + 1][0] for i in range(7))
    b0 = sharding.view_batches(90, 49152, 1 << 20)        # config 0: 21-view batches
    r0 = [sharding.view_shard(90, 2, r, b0) for r in range(2)]
    assert r0 == [(0, 42), (42, 90)]
    with pytest.raises(ValueError):
        sharding.view_shard(10, 2, 2)


def test_gloo_sharded_forward_matches_single(tmp_path):
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "oracle"))
    import cbn_oracle as orc
    from paper_1605_05231_b200.phantom import random_ellipsoid_phantom
    out = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    res = np.load(out)
    geom, voxel, spec, cfg = small_setup(12, 8, "dirac")
    vol = random_ellipsoid_phantom(12, 4, 7)
    ref = orc.forward_project(vol, voxel, geom, cfg, target_batch=cfg.n_mu * cfg.n_t * 3)
    assert np.allclose(res["full"], ref, rtol=0, atol=1e-12 * np.abs(ref).max())
    assert float(res["t"]) == 2.0


class _FakeProjector:
    """CPU stand-in for the device phases: fixed random linear maps with the same
    sharding contract (node parts summed over ranks, view ranges local) and the
    same separable crop structure (grid (K, K, K) -> volume (n, n, n))."""

    def __init__(self, views=6, n_vox=5, m=9, n=3, k=6, cplx=False):
        import torch
        g = torch.Generator().manual_seed(0)
        self.views, self.n, self.k = views, n, k
        self.A = torch.randn(m, n_vox, generator=g, dtype=torch.float64)       # vol -> lattice
        self.B = torch.randn(views, m, generator=g, dtype=torch.float64)       # lattice -> views
        self.C = torch.randn(m, views, generator=g, dtype=torch.float64)       # views -> lattice
        self.D = torch.randn(k ** 3, m, generator=g, dtype=torch.float64)      # lattice -> grid
        self.F = [torch.randn(n, k, generator=g, dtype=torch.float64) for _ in range(3)]
        if cplx:   # complex grid and crop maps, as the device path's complex64 buffers
            self.D = self.D + 1j * torch.randn(k ** 3, m, generator=g, dtype=torch.float64)
            self.F = [f + 1j * torch.randn(n, k, generator=g, dtype=torch.float64) for f in self.F]
            self.C = self.C.to(torch.complex128)

    @staticmethod
    def _rows(n, part, nparts):
        import torch
        mask = torch.zeros(n, 1, dtype=torch.float64)
        mask[part::nparts] = 1.0
        return mask

    def forward_lattice(self, vol, part, nparts):
        return (self.A @ vol) * self._rows(self.A.shape[0], part, nparts)[:, 0]

    def forward_views(self, lat, lo, hi):
        return (self.B @ lat)[lo:hi]

    def backproject_views(self, frames_local, lo, hi):
        return self.C[:, lo:hi] @ frames_local

    def backproject_finish(self, lat, part, nparts):
        return (self.D * self._rows(self.D.shape[1], part, nparts)[:, 0]) @ lat

    def backproject_crop(self, grid):
        import torch
        fx, fy, fz = self.F
        return torch.einsum("xa,yb,zc,abc->xyz", fx, fy, fz, grid.view(self.k, self.k, self.k))

    def backproject_crop_slab(self, slab, x_lo, x_hi, nparts):
        import torch
        _, fy, fz = self.F
        t = torch.einsum("yb,zc,abc->ayz", fy, fz, slab.reshape(x_hi - x_lo, self.k, self.k))
        ys = [self.n * d // nparts for d in range(nparts + 1)]
        return torch.cat([t[:, ys[d]:ys[d + 1]].reshape(-1) for d in range(nparts)])

    def backproject_crop_cols(self, cols, y_lo, y_hi):
        import torch
        return torch.einsum("xa,ayz->xyz", self.F[0], cols.view(self.k, y_hi - y_lo, self.n))


def _sharded_worker(rank, world, port, result_path, k=6, cplx=False):
    import sys
    import torch
    import torch.distributed as dist
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [here, os.path.dirname(here)]
    from paper_1605_05231_b200 import sharding
    from paper_1605_05231_b200.pipeline import Projector
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    fake = _FakeProjector(k=k, cplx=cplx)
    vol = torch.arange(5, dtype=torch.float64) + 1.0 if rank == 0 else torch.zeros(5, dtype=torch.float64)
    frames = torch.linspace(-1.0, 2.0, fake.views, dtype=torch.float64)
    lo, hi = sharding.view_shard(fake.views, world, rank)
    fwd_local = Projector.forward_sharded(fake, vol, lo, hi)
    fwd = sharding.gather_views(fwd_local, fake.views)
    bp = Projector.backproject_sharded(fake, frames[lo:hi].to(fake.C.dtype), lo, hi)
    if rank == 0:
        np.savez(result_path, fwd=fwd.numpy(), bp=bp.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,k,cplx", [(2, 6, False), (3, 6, False), (2, 5, False),
                                          (2, 6, True)])
def test_gloo_sharded_phase_orchestration(tmp_path, world, k, cplx):
    """Projector.forward_sharded / backproject_sharded over a gloo world: the
    volume broadcast, node-part sums (all-reduce), view ranges and the
    slab-distributed crop (reduce-scatter by x slab -- all-reduce + slice when
    the world does not divide the grid -- all-to-all to y ranges, all-gather)
    give the single-process maps."""
    out = str(tmp_path / "res.npz")
    mp.spawn(_sharded_worker, args=(world, _free_port(), out, k, cplx), nprocs=world, join=True)
    res = np.load(out)
    f = _FakeProjector(k=k, cplx=cplx)
    import torch
    vol = torch.arange(5, dtype=torch.float64) + 1.0
    frames = torch.linspace(-1.0, 2.0, f.views, dtype=torch.float64)
    assert np.allclose(res["fwd"], (f.B @ (f.A @ vol)).numpy(), rtol=1e-12)
    ref = f.backproject_crop(f.D @ (f.C @ frames.to(f.C.dtype))).numpy()
    assert res["bp"].shape == ref.shape
    assert np.allclose(res["bp"], ref, rtol=1e-12, atol=1e-12)
