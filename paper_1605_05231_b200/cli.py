"""``cbnufft project`` / ``cbnufft backproject`` on the device (the projector
path of ``cbnufft/cli.py:78-100,213-290``).

    python -m paper_1605_05231_b200.cli project --method nufft-a|nufft-b|linear \
        --volume VOL [--geometry GEOM.json] --out PROJ
    python -m paper_1605_05231_b200.cli backproject [--method nufft-a|nufft-b] \
        --projections PROJ --n N [--voxel-mm V] --out VOL [--slice-pgm PGM]

The flags, file formats, normalisation calibration and exit codes are the
reference's: 0 success, 2 invalid input (ValueError / OSError), 3 non-finite
result (FloatingPointError).  Payloads move file -> pinned buffer -> device
-> pinned buffer -> file (io.read_volume_device & co.); the projections and
the volume never exist as float64 host arrays.  The report subcommands of the
reference (phantom, fdk, sweep, complexity, compare) are outside the
projector path and not provided.
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np

from . import io as cbio
from .baseline import ct_project_linear
from .geometry import ConeGeometry
from .nufft import set_threads

# the reference CLI's acquisition when --geometry is not given (cli.py:29)
DEFAULT_GEOMETRY = ConeGeometry(so_mm=1100.0, sd_mm=1500.0, det_width_mm=512.0,
                                det_height_mm=512.0, nu=128, nv=128, n_views=256,
                                object_extent_mm=360.0)

EXIT_OK, EXIT_INPUT, EXIT_NUMERIC = 0, 2, 3


def _require_finite(arrays) -> None:
    if not all(np.isfinite(a).all() for a in arrays):
        raise FloatingPointError("non-finite values in the result")


def run_project(args) -> None:
    from . import pipeline as pl
    geom = cbio.load_geometry(args.geometry) if args.geometry else DEFAULT_GEOMETRY
    if args.method == "linear":
        # the ray-driven baseline projector (baseline.py:52-98), host frames
        frames = ct_project_linear(cbio.read_volume(args.volume), geom)
        _require_finite(f.data for f in frames)
        cbio.write_projections(args.out, frames, geom)
        return
    vol, voxel = cbio.read_volume_device(args.volume)
    n = int(vol.shape[0])
    cfg = pl.make_projector_config(geom, n, args.method.split("-")[1])
    pl.calibrate_normalization(geom, n, cfg, voxel)
    proj = pl.get_projector(geom, cfg, n, voxel, pl._FORWARD)
    cbio.write_projections_device(args.out, proj.forward(vol), geom)


def run_backproject(args) -> None:
    from . import pipeline as pl
    frames, geom = cbio.read_projections_device(args.projections)
    n = args.n
    voxel = args.voxel_mm or geom.object_extent_mm / n
    cfg = pl.make_projector_config(geom, n, args.method.split("-")[1])
    pl.calibrate_bp_normalization(geom, n, cfg, voxel)
    vol = pl.get_projector(geom, cfg, n, voxel, pl._BACK).backproject(frames)
    cbio.write_volume_device(args.out, vol, voxel)
    if args.slice_pgm:
        cbio.write_pgm16(args.slice_pgm, vol[:, :, n // 2].double().cpu().numpy())


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="cbnufft", description=__doc__)
    parser.add_argument("--threads", type=int,
                        default=int(os.environ.get("CBNUFFT_THREADS", "1")))
    parser.add_argument("--seed", type=int, default=0)
    commands = parser.add_subparsers(dest="command", required=True)
    c = commands.add_parser("project", help="cone-beam forward projection")
    c.add_argument("--method", required=True, choices=["nufft-a", "nufft-b", "linear"])
    c.add_argument("--volume", required=True)
    c.add_argument("--geometry")
    c.add_argument("--out", required=True)
    c.set_defaults(run=run_project)
    c = commands.add_parser("backproject", help="direct NUFFT backprojection")
    c.add_argument("--method", default="nufft-a", choices=["nufft-a", "nufft-b"])
    c.add_argument("--projections", required=True)
    c.add_argument("--n", type=int, required=True)
    c.add_argument("--voxel-mm", type=float)
    c.add_argument("--out", required=True)
    c.add_argument("--slice-pgm")
    c.set_defaults(run=run_backproject)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        set_threads(args.threads)
        args.run(args)
    except FloatingPointError as err:
        print(f"numerical failure: {err}", file=sys.stderr)
        return EXIT_NUMERIC
    except (ValueError, OSError) as err:
        print(f"error: {err}", file=sys.stderr)
        return EXIT_INPUT
    return EXIT_OK


if __name__ == "__main__":
    sys.exit(main())
