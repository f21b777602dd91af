"""On-disk formats (io.py) against files the reference itself wrote
(tests/golden/io, tests/golden/make_golden.py io): read them, rewrite them,
compare byte for byte.  CPU only."""

import filecmp
import json
import os
import shutil

import numpy as np
import pytest

from conftest import GOLDEN

IO = os.path.join(GOLDEN, "io")


def test_volume_roundtrip_bytes(tmp_path):
    from paper_1605_05231_b200 import io as cbio
    vol = cbio.read_volume(os.path.join(IO, "vol.raw"))
    assert vol.n == 12 and vol.data.dtype == np.float64
    out = str(tmp_path / "v.raw")
    cbio.write_volume(out, vol)
    assert filecmp.cmp(out, os.path.join(IO, "vol.raw"), shallow=False)
    assert json.load(open(out + ".json")) == json.load(open(os.path.join(IO, "vol.raw.json")))


@pytest.mark.parametrize("name", ["proj_nufft-a", "proj_nufft-b", "proj_linear"])
def test_projections_roundtrip_bytes(tmp_path, name):
    from paper_1605_05231_b200 import io as cbio
    frames, geom = cbio.read_projections(os.path.join(IO, name + ".raw"))
    assert len(frames) == geom.n_views == 8
    assert frames[0].data.shape == (geom.nu, geom.nv)
    out = str(tmp_path / "p.raw")
    cbio.write_projections(out, frames, geom)
    assert filecmp.cmp(out, os.path.join(IO, name + ".raw"), shallow=False)
    assert json.load(open(out + ".json")) == json.load(open(os.path.join(IO, name + ".raw.json")))


def test_geometry_file(tmp_path):
    from paper_1605_05231_b200 import io as cbio
    geom = cbio.load_geometry(os.path.join(IO, "geom.json"))
    out = str(tmp_path / "g.json")
    cbio.save_geometry(out, geom)
    assert filecmp.cmp(out, os.path.join(IO, "geom.json"), shallow=False)


def test_io_errors(tmp_path):
    from paper_1605_05231_b200 import io as cbio
    with pytest.raises(ValueError):
        cbio.read_volume(str(tmp_path / "missing.raw"))
    bad = tmp_path / "v.raw"
    shutil.copy(os.path.join(IO, "vol.raw"), bad)
    meta = json.load(open(os.path.join(IO, "vol.raw.json")))
    meta["dims"] = [13, 13, 13]
    json.dump(meta, open(str(bad) + ".json", "w"))
    with pytest.raises(ValueError):
        cbio.read_volume(str(bad))
    with pytest.raises(ValueError):
        cbio.load_geometry(str(tmp_path / "nope.json"))


def test_cli_validation_exit_code(tmp_path):
    from paper_1605_05231_b200.cli import main
    assert main(["project", "--method", "nufft-a", "--volume", str(tmp_path / "x.raw"),
                 "--out", str(tmp_path / "o.raw")]) == 2


def test_cli_numerical_failure_exit_code(tmp_path, monkeypatch):
    """Exit code 3 on a non-finite result (the reference's test_cli.py:118-131
    contract, with its monkeypatch of cli.ct_project_linear)."""
    from paper_1605_05231_b200 import cli

    def bad_project(vol, geom):
        class F:   # a frame the projector failed on (bypasses the frame validator)
            data = np.full((geom.nu, geom.nv), np.nan)
        return [F() for _ in range(geom.n_views)]
    monkeypatch.setattr(cli, "ct_project_linear", bad_project)
    code = cli.main(["project", "--method", "linear", "--volume", os.path.join(IO, "vol.raw"),
                     "--geometry", os.path.join(IO, "geom.json"),
                     "--out", str(tmp_path / "o.raw")])
    assert code == 3
