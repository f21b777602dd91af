"""ctypes binding of libcbnufft_b200.so (include/cbnufft_b200.h).

There is no CPU fallback: if the shared library is missing or no CUDA device
is present, every operator raises.  Status codes map onto the reference's
exceptions (ValueError for invalid arguments, FloatingPointError for
non-finite projections, pipeline.py:144-145).
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# CBN_LIB=check loads the bounds-checked build (csrc/Makefile target `check`);
# CBN_LIB=<name>.so another build of the library in this directory (A/B variants)
_ALT = os.environ.get("CBN_LIB", "")
LIB_PATH = os.path.join(_HERE, "libcbnufft_b200_check.so" if _ALT == "check"
                        else _ALT if _ALT.endswith(".so") else "libcbnufft_b200.so")

CBN_OK, CBN_EINVAL, CBN_ECUDA, CBN_ENOMEM, CBN_ENONFINITE, CBN_ENCCL, CBN_EUNSUPPORTED = range(7)

_lock = threading.Lock()
_lib = None

c_i32, c_i64, c_f64, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
P_i64 = ctypes.POINTER(c_i64)
P_i32 = ctypes.POINTER(c_i32)
P_f64 = ctypes.POINTER(c_f64)


class Geometry(ctypes.Structure):
    _fields_ = [("so_mm", c_f64), ("sd_mm", c_f64), ("det_width_mm", c_f64),
                ("det_height_mm", c_f64), ("nu", c_i32), ("nv", c_i32), ("n_views", c_i32),
                ("object_extent_mm", c_f64)]


class RadialSpec(ctypes.Structure):
    _fields_ = [("n_rho", c_i32), ("n_theta", c_i32), ("n_phi", c_i32), ("rho_max", c_f64)]


class ProjectorConfig(ctypes.Structure):
    _fields_ = [("method", c_i32), ("spec", RadialSpec), ("n_mu", c_i32), ("n_t", c_i32),
                ("t_pitch_mm", c_f64), ("t_taper", c_i32), ("spectrum_j", c_i32),
                ("resample_j", c_i32 * 3), ("side_lobes", c_i32), ("oversample_factor", c_f64),
                ("rho_pad", c_i32), ("basis", c_i32), ("normalization", c_f64),
                ("bp_normalization", c_f64), ("den_tol", c_f64), ("target_batch", c_i64),
                ("plan_chunk", c_i64), ("bp_n_t", c_i32), ("bp_t_pitch_mm", c_f64)]


_SIGS = {
    "cbn_last_error": (ctypes.c_char_p, []),
    "cbn_version": (ctypes.c_int, []),
    "cbn_beatty_beta": (c_f64, [ctypes.c_int, c_f64]),
    "cbn_nufft_create": (ctypes.c_int, [ctypes.POINTER(c_vp), ctypes.c_int, P_i64, P_i32, c_f64,
                                        P_f64, c_i64, P_i64, c_i64, c_vp]),
    "cbn_nufft_create_f32": (ctypes.c_int, [ctypes.POINTER(c_vp), ctypes.c_int, P_i64, P_i32, c_f64,
                                            c_vp, c_i64, P_i64, c_i64, c_vp]),
    "cbn_nufft_destroy": (ctypes.c_int, [c_vp]),
    "cbn_nufft_scaling": (ctypes.c_int, [c_vp, P_f64]),
    "cbn_nufft_wrapped_nodes": (ctypes.c_int, [c_vp, P_f64]),
    "cbn_nufft_first_indices": (ctypes.c_int, [c_vp, P_i32, c_vp]),
    "cbn_nufft_type2": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "cbn_nufft_type1": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "cbn_nufft_set_phase": (ctypes.c_int, [c_vp, c_i32]),
    "cbn_nufft_resort": (ctypes.c_int, [c_vp, c_vp]),
    "cbn_nufft_set_timing": (ctypes.c_int, [c_vp, c_i32]),
    "cbn_nufft_stage_times": (ctypes.c_int, [c_vp, P_f64, P_f64, P_f64, P_i32, ctypes.c_char_p,
                                             c_i32]),
    "cbn_resample_create": (ctypes.c_int, [ctypes.POINTER(c_vp), c_i32, c_i32, c_i32, c_i32, P_i32,
                                           c_f64, P_f64, c_i64, P_i64, c_i64, c_vp]),
    "cbn_resample_create_b": (ctypes.c_int, [ctypes.POINTER(c_vp), c_i32, c_i32, c_i32, c_i32,
                                             c_i32, P_f64, c_i64, c_vp]),
    "cbn_resample_destroy": (ctypes.c_int, [c_vp]),
    "cbn_resample_apply": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "cbn_resample_transpose": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "cbn_radial_fft": (ctypes.c_int, [c_vp, c_i64, c_i64, c_i32, c_f64, c_vp]),
    "cbn_lines_real_in": (ctypes.c_int, [c_vp, c_i64, c_i64, P_f64, c_vp, c_vp]),
    "cbn_lines_real_out": (ctypes.c_int, [c_vp, c_i64, c_i64, P_f64, c_vp, c_vp]),
    "cbn_frame_ring_center": (ctypes.c_int, [c_vp, c_i32, c_i32, c_vp]),
    "cbn_projector_set_node_shard": (ctypes.c_int, [c_vp, c_i32, c_i32, P_i64, P_i64, c_vp]),
    "cbn_host_gather_f64_to_f32": (ctypes.c_int, [c_vp, c_i64, c_i64, c_vp, c_i32]),
    "cbn_host_f64_to_f32": (ctypes.c_int, [c_vp, c_vp, c_i64, c_i32]),
    "cbn_host_f32_to_f64": (ctypes.c_int, [c_vp, c_vp, c_i64, c_i32]),
    "cbn_projector_info": (ctypes.c_int, [c_vp, P_i32, P_i32, P_i32, P_i32]),
    "cbn_projector_debug_buffer": (ctypes.c_int, [c_vp, ctypes.c_char_p, c_vp, P_i64, c_vp]),
    "cbn_backproject_stage_views": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i32, c_vp]),
    "cbn_line_weight": (ctypes.c_int, [c_vp, c_i64, c_i64, c_i64, P_f64, c_vp]),
    "cbn_node_phase": (ctypes.c_int, [c_vp, P_f64, c_i64, c_i32, P_f64, c_i32, P_f64, c_i64, c_vp]),
    "cbn_trilinear_transfer": (ctypes.c_int, [c_i32, c_i32, c_i32, c_f64, c_f64, c_vp, c_vp]),
    "cbn_projector_radial_spectrum": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "cbn_projector_grangeat_records": (ctypes.c_int, [c_vp, c_vp, P_i32, P_i64, c_vp]),
    "cbn_projector_create": (ctypes.c_int, [ctypes.POINTER(c_vp), ctypes.POINTER(Geometry),
                                            ctypes.POINTER(ProjectorConfig), c_i32, c_f64, c_i32]),
    "cbn_projector_destroy": (ctypes.c_int, [c_vp]),
    "cbn_projector_ls_sizes": (ctypes.c_int, [c_vp, P_i64, P_i32]),
    "cbn_projector_set_ls_rows": (ctypes.c_int, [c_vp, c_i64, P_i64, c_i64]),
    "cbn_projector_scratch_bytes": (ctypes.c_int, [c_vp, P_i64]),
    "cbn_forward_project": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i32, c_i32, c_vp]),
    "cbn_forward_project_async": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i32, c_i32, c_vp]),
    "cbn_forward_stage_volume": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i32, c_vp]),
    "cbn_forward_project_staged_async": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i32, c_vp]),
    "cbn_projector_blocks": (ctypes.c_int, [c_vp, P_i32, P_i32, P_i32]),
    "cbn_projector_block_sync": (ctypes.c_int, [c_vp, c_i32]),
    "cbn_forward_finish": (ctypes.c_int, [c_vp, c_vp]),
    "cbn_forward_lattice_size": (ctypes.c_int, [c_vp, P_i64, c_vp]),
    "cbn_forward_lattice": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i32, c_vp, c_vp]),
    "cbn_forward_views": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i32, c_i32, c_vp]),
    "cbn_backproject": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "cbn_backproject_sizes": (ctypes.c_int, [c_vp, P_i64, P_i64, c_vp]),
    "cbn_backproject_views": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i32, c_vp, c_vp]),
    "cbn_backproject_finish": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i32, c_vp, c_vp]),
    "cbn_backproject_crop": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "cbn_backproject_crop_slab": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i32, c_i32, c_vp, c_vp]),
    "cbn_backproject_crop_cols": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i32, c_vp, c_vp]),
    "cbn_projector_radial_lattice": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "cbn_projector_resample_views": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i32, c_i32, c_vp]),
    "cbn_projector_grangeat_reverse": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i32, c_vp]),
    "cbn_projector_grangeat_forward": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i32, c_vp]),
    "cbn_projector_set_timing": (ctypes.c_int, [c_vp, c_i32]),
    "cbn_projector_stage_times": (ctypes.c_int, [c_vp, P_f64, P_i32, ctypes.c_char_p, c_i32,
                                                 c_i32]),
    "cbn_backproject_stage_transpose": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i32, c_vp, c_vp,
                                                       c_vp]),
    "cbn_projector_first_indices": (ctypes.c_int, [c_vp, c_i32, c_i32, P_i32, P_i64, c_vp]),
    "cbn_projector_plan_stats": (ctypes.c_int, [c_vp, P_i64, P_i32, ctypes.c_char_p, c_i32, c_vp]),
    "cbn_projector_stage_bytes": (ctypes.c_int, [c_vp, P_f64, P_f64, P_i32, ctypes.c_char_p, c_i32,
                                                 c_i32]),
    "cbn_ct_project_linear": (ctypes.c_int, [ctypes.POINTER(Geometry), c_vp, c_i32, c_f64, c_vp,
                                             c_vp]),
    "cbn_launch_count": (ctypes.c_longlong, []),
}

EXPORTED = tuple(_SIGS)


class ExtensionMissing(RuntimeError):
    pass


def load(path: str = LIB_PATH):
    """Load and type the shared library (no device work)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ExtensionMissing(
                f"{path} is not built; run __graft_entry__.build() -- there is no CPU fallback")
        lib = ctypes.CDLL(path)
        missing = []
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name, None)
            if fn is None:
                missing.append(name)
                continue
            fn.restype = res
            fn.argtypes = args
        lib.cbn_missing_symbols = tuple(missing)
        _lib = lib
        return lib


def check(status: int, what: str = "") -> None:
    if status == CBN_OK:
        return
    msg = load().cbn_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status == CBN_EINVAL:
        raise ValueError(text)
    if status == CBN_ENONFINITE:
        raise FloatingPointError(text)
    if status == CBN_ENOMEM:
        raise MemoryError(text)
    if status == CBN_EUNSUPPORTED:
        raise NotImplementedError(text)
    raise RuntimeError(f"CUDA failure ({status}) {text}")


def i64_array(a) -> tuple[np.ndarray, object]:
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(P_i64)


def f64_array(a) -> tuple[np.ndarray, object]:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(P_f64)
