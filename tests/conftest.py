"""Shared test setup: the `gpu` marker, fixture paths, tolerance helpers."""

import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
for p in (REPO, os.path.join(REPO, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def rel_l2(got, ref):
    got = np.asarray(got)
    ref = np.asarray(ref)
    return float(np.linalg.norm((got - ref).ravel()) / max(np.linalg.norm(ref.ravel()), 1e-300))


def load_cases():
    z = np.load(os.path.join(GOLDEN, "nufft_cases.npz"))
    cases = {}
    for key in z.files:
        name, field = key.split("__")
        cases.setdefault(name, {})[field] = z[key]
    return cases


@pytest.fixture(scope="session")
def nufft_cases():
    return load_cases()


@pytest.fixture(scope="session")
def golden_n16():
    return dict(np.load(os.path.join(GOLDEN, "pipeline_n16.npz")))


@pytest.fixture(scope="session")
def golden_n12():
    return dict(np.load(os.path.join(GOLDEN, "pipeline_n12_dirac.npz")))


def unpack_int(z, key):
    """Decode an (m, d) integer fixture written by make_golden_r2.pack_int
    (row deltas, axis-major, zlib) -> int64 (m, d)."""
    import zlib
    shape = tuple(int(s) for s in z[key + "__shape"])
    d = np.frombuffer(zlib.decompress(z[key + "__z"].tobytes()), np.int16)
    d = d.reshape(shape[1], shape[0]).T.astype(np.int64)
    return np.cumsum(d, axis=0)
