"""Workload constructors shared by tests (mirror tests/golden/make_golden.py)."""

from paper_1605_05231_b200.config import make_projector_config
from paper_1605_05231_b200.geometry import ConeGeometry, RadialGridSpec


def small_setup(n=16, views=12, basis="trilinear"):
    geom = ConeGeometry(3.0, 6.0, 2.0, 2.0, n, n, views, 2.0)
    voxel = 2.0 / n
    spec = RadialGridSpec(2 * n, n, 2 * n, 2 * n * voxel / 2.0)
    cfg = make_projector_config(geom, n, "a", radial_spec=spec, spectrum_j=6,
                                rho_pad=min(spec.n_rho // 8, 32), basis=basis)
    return geom, voxel, spec, cfg


def config_setup(idx):
    """BASELINE.json configs 0-3; see workloads.py."""
    from paper_1605_05231_b200.workloads import workload
    w = workload(idx)
    return w.geom, w.voxel, w.spec, w.cfg
