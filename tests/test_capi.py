"""CPU checks of the C-ABI library: it loads, exports every symbol
include/cbnufft_b200.h declares, and its host-only entry points behave."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO
from _cases import small_setup


def header_symbols():
    text = open(os.path.join(REPO, "include", "cbnufft_b200.h")).read()
    return sorted(set(re.findall(r"\b(cbn_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_header_symbols():
    from paper_1605_05231_b200 import _lib
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert not lib.cbn_missing_symbols
    assert set(syms) == set(_lib.EXPORTED), set(syms) ^ set(_lib.EXPORTED)
    assert lib.cbn_version() >= 1


def test_beatty_beta_matches_reference_formula():
    from paper_1605_05231_b200 import _lib
    lib = _lib.load()
    for j in range(1, 10):
        for alpha in (1.0, 1.5, 2.0, 2.5):
            ref = np.pi * np.sqrt(max((j / alpha) ** 2 * (alpha - 0.5) ** 2 - 0.8, 0.0))
            assert lib.cbn_beatty_beta(j, alpha) == ref


def test_projector_create_validates_on_host():
    from paper_1605_05231_b200 import _lib
    from paper_1605_05231_b200.pipeline import _config_struct, _geometry_struct
    geom, voxel, spec, cfg = small_setup()
    lib = _lib.load()
    g = _geometry_struct(geom)
    c = _config_struct(cfg, 1 << 20, 1 << 21)
    h = ctypes.c_void_p()
    assert lib.cbn_projector_create(ctypes.byref(h), ctypes.byref(g), ctypes.byref(c), 16,
                                    voxel, 3) == 0
    cnt = ctypes.c_int32(16)
    sizes = (ctypes.c_int64 * 16)()
    assert lib.cbn_projector_ls_sizes(h, sizes, ctypes.byref(cnt)) == 0
    per_view = cfg.n_mu * cfg.n_t
    got = set(list(sizes)[:cnt.value])
    assert {spec.n_rho * spec.n_theta * spec.n_phi, 12 * per_view, per_view} <= got
    lib.cbn_projector_destroy(h)
    c.spec.n_rho = 7
    assert lib.cbn_projector_create(ctypes.byref(h), ctypes.byref(g), ctypes.byref(c), 16,
                                    voxel, 3) == 1
    assert b"n_rho" in lib.cbn_last_error()


def test_method_b_config_and_bad_taper():
    from paper_1605_05231_b200.pipeline import _config_struct
    geom, voxel, spec, cfg = small_setup()
    cfg.method = "b"
    assert _config_struct(cfg, 1, 1).method == 1
    cfg.side_lobes = 9
    with pytest.raises(ValueError):
        _config_struct(cfg, 1, 1)
    cfg.side_lobes = 2
    cfg.method = "c"
    with pytest.raises(ValueError):
        _config_struct(cfg, 1, 1)
    cfg.method = "a"
    cfg.t_taper = "tukey"
    with pytest.raises(ValueError):
        _config_struct(cfg, 1, 1)


def test_operators_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1605_05231_b200 import nufft
    with pytest.raises(RuntimeError):
        nufft.plan_nufft((8,), np.zeros((4, 1)), 2.0, 6)


def test_comm_library_exports_header_symbols():
    """libcbnufft_b200_comm.so (NCCL collectives behind the C ABI) loads without
    a GPU and exports every symbol include/cbnufft_b200_comm.h declares; the
    NCCL unique id is host-only."""
    from paper_1605_05231_b200 import comm
    text = open(os.path.join(REPO, "include", "cbnufft_b200_comm.h")).read()
    syms = sorted(set(re.findall(r"\b(cbn_[a-z0-9_]+)\s*\(", text)))
    lib = comm.load()
    assert not [s for s in syms if not hasattr(lib, s)]
    assert set(syms) == set(comm.EXPORTED), set(syms) ^ set(comm.EXPORTED)
    assert not lib.cbn_missing_symbols
    uid = comm.unique_id()
    assert len(uid) == comm.ID_BYTES and uid != comm.unique_id()
    h = ctypes.c_void_p()
    assert lib.cbn_comm_init(ctypes.byref(h), None, 1, 0) == 1   # CBN_EINVAL
    assert lib.cbn_comm_init(ctypes.byref(h), ctypes.create_string_buffer(uid, 128), 2, 2) == 1
