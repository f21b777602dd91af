"""Command-line entry for the projector path (drop-in for the ``project`` and
``backproject`` subcommands of ``cbnufft/cli.py:78-100,202-221``).

    python -m paper_1605_05231_b200.cli project --method nufft-a|nufft-b|linear \
        --volume VOL [--geometry GEOM.json] --out PROJ
    python -m paper_1605_05231_b200.cli backproject [--method nufft-a|nufft-b] \
        --projections PROJ --n N [--voxel-mm V] --out VOL [--slice-pgm PGM]

Same flags, file formats (``io.py``), calibration calls and exit codes as the
reference: 0 success, 2 validation error, 3 non-finite result.  The other
reference subcommands (phantom, fdk, sweep, complexity, compare) are reports
and baselines outside the projector path and are not
provided here.
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np

from . import io as cbio
from .geometry import ConeGeometry
from .nufft import set_threads

DEFAULT_GEOMETRY = dict(so_mm=1100.0, sd_mm=1500.0, det_width_mm=512.0, det_height_mm=512.0,
                        nu=128, nv=128, n_views=256, object_extent_mm=360.0)


def _check_finite(arrays) -> None:
    for a in arrays:
        if not np.all(np.isfinite(a)):
            raise FloatingPointError("non-finite values in the result")


def _geometry(args) -> ConeGeometry:
    if args.geometry:
        return cbio.load_geometry(args.geometry)
    return ConeGeometry(**DEFAULT_GEOMETRY)


def _cmd_project(args) -> None:
    from .baseline import ct_project_linear
    from .pipeline import calibrate_normalization, make_projector_config, nufft_forward_project
    vol = cbio.read_volume(args.volume)
    geom = _geometry(args)
    if args.method == "linear":
        frames = ct_project_linear(vol, geom)
    else:
        cfg = make_projector_config(geom, vol.n, args.method[-1])
        calibrate_normalization(geom, vol.n, cfg, vol.voxel_mm)
        frames = nufft_forward_project(vol, geom, cfg)
    _check_finite([f.data for f in frames])
    cbio.write_projections(args.out, frames, geom)


def _cmd_backproject(args) -> None:
    from .pipeline import calibrate_bp_normalization, make_projector_config, nufft_backproject
    frames, geom = cbio.read_projections(args.projections)
    n = args.n
    voxel = args.voxel_mm or geom.object_extent_mm / n
    cfg = make_projector_config(geom, n, args.method[-1])
    calibrate_bp_normalization(geom, n, cfg, voxel)
    vol = nufft_backproject(frames, geom, cfg, n, voxel)
    _check_finite([vol.data])
    cbio.write_volume(args.out, vol)
    if args.slice_pgm:
        cbio.write_pgm16(args.slice_pgm, vol.data[:, :, vol.n // 2])


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="cbnufft", description=__doc__)
    p.add_argument("--threads", type=int, default=int(os.environ.get("CBNUFFT_THREADS", "1")))
    p.add_argument("--seed", type=int, default=0)
    sub = p.add_subparsers(dest="command", required=True)
    sp = sub.add_parser("project", help="cone-beam forward projection")
    sp.add_argument("--method", required=True, choices=["nufft-a", "nufft-b", "linear"])
    sp.add_argument("--volume", required=True)
    sp.add_argument("--geometry")
    sp.add_argument("--out", required=True)
    sp.set_defaults(func=_cmd_project)
    sp = sub.add_parser("backproject", help="direct NUFFT backprojection")
    sp.add_argument("--method", default="nufft-a", choices=["nufft-a", "nufft-b"])
    sp.add_argument("--projections", required=True)
    sp.add_argument("--n", type=int, required=True)
    sp.add_argument("--voxel-mm", type=float)
    sp.add_argument("--out", required=True)
    sp.add_argument("--slice-pgm")
    sp.set_defaults(func=_cmd_backproject)
    return p


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        set_threads(args.threads)
        args.func(args)
    except (ValueError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except FloatingPointError as e:
        print(f"numerical failure: {e}", file=sys.stderr)
        return 3
    return 0


if __name__ == "__main__":
    sys.exit(main())
