"""CLI project / backproject (cli.py:78-100) end to end on the device against the
reference CLI's own output files (tests/golden/io): same flags, same formats,
same calibration calls; relative L2 <= 1e-4."""

import os

import pytest

from conftest import GOLDEN, rel_l2

pytestmark = pytest.mark.gpu
IO = os.path.join(GOLDEN, "io")


@pytest.mark.parametrize("method", ["nufft-a", "nufft-b", "linear"])
def test_cli_project(tmp_path, method):
    import numpy as np
    from paper_1605_05231_b200 import io as cbio
    from paper_1605_05231_b200.cli import main
    out = str(tmp_path / "p.raw")
    assert main(["project", "--method", method, "--volume", os.path.join(IO, "vol.raw"),
                 "--geometry", os.path.join(IO, "geom.json"), "--out", out]) == 0
    got, _ = cbio.read_projections(out)
    ref, _ = cbio.read_projections(os.path.join(IO, f"proj_{method}.raw"))
    assert rel_l2(np.stack([f.data for f in got]), np.stack([f.data for f in ref])) < 1e-4


@pytest.mark.parametrize("method", ["nufft-a", "nufft-b"])
def test_cli_backproject(tmp_path, method):
    from paper_1605_05231_b200 import io as cbio
    from paper_1605_05231_b200.cli import main
    out = str(tmp_path / "v.raw")
    assert main(["backproject", "--method", method,
                 "--projections", os.path.join(IO, "proj_nufft-a.raw"), "--n", "12",
                 "--out", out, "--slice-pgm", str(tmp_path / "s.pgm")]) == 0
    got = cbio.read_volume(out).data
    ref = cbio.read_volume(os.path.join(IO, f"bp_{method}.raw")).data
    assert rel_l2(got, ref) < 1e-4
    assert os.path.getsize(tmp_path / "s.pgm") > 12 * 12 * 2
