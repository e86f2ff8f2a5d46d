"""ctypes binding of libfastmusic_b200.so (include/fastmusic_b200.h).

The product path: every numeric entry point here calls a CUDA kernel through the C ABI.
There is no CPU fallback — if the shared library is missing, importing the binding raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfastmusic_b200.so")

FM_OK, FM_EINVAL, FM_ERANK, FM_ENOCONV, FM_ESINGULAR, FM_ECUDA, FM_ENOTSUP, FM_EIO = range(8)
FRAME_OK, FRAME_RANK, FRAME_NOCONV, FRAME_RANGE, FRAME_NONFINITE = 0, 1, 2, 4, 8
METHOD = {"exact": 0, "fast1": 1, "fast2": 2, "lanczos": 3, "fast1_norm2": 16}

# Every symbol declared in include/fastmusic_b200.h (checked by tests/test_capi_symbols.py).
EXPORTED = [
    "fm_abi_version", "fm_status_string", "fm_last_error", "fm_device_info", "fm_pack_peak_records",
    "fm_rng_derive", "fm_rng_normals", "fm_sample_without_replacement", "fm_gaussian_matrix_real",
    "fm_draw_omega_batch", "fm_draw_indices_batch", "fm_draw_uniforms_batch", "fm_generate_frames",
    "fm_plan_create", "fm_plan_destroy", "fm_plan_workspace_bytes", "fm_run_batch", "fm_rerun_frames",
    "fm_plan_launches_per_batch", "fm_plan_set_profiling", "fm_plan_stage_times", "fm_plan_set_concurrency", "fm_plan_set_graphs", "fm_estimate_batch_host",
    "fm_z_spatial_covariance", "fm_z_hermitian_eig", "fm_z_exact_signal_subspace", "fm_z_fast_music_1", "fm_z_fast_music_2",
    "fm_z_music_spectrum", "fm_z_extract_peaks",
    "fm_z_temporal_covariance", "fm_temporal_covariance_batch", "fm_z_block_lanczos_subspace",
    "fm_block_lanczos_batch",
    "fm_fmcx_write", "fm_fmcx_read_header", "fm_fmcx_read", "fm_z_fmcx_write", "fm_z_fmcx_read",
    "fm_fmcx_read_frames", "fm_fmcx_write_frames", "fm_z_write_matrix_csv", "fm_write_spectrum_csv",
]


class PlanDesc(C.Structure):
    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("k", C.c_int64), ("method", C.c_int32), ("p", C.c_int64),
                ("t", C.c_int32), ("grid_size", C.c_int64), ("theta0", C.c_double), ("theta1", C.c_double),
                ("d", C.c_double), ("lam", C.c_double), ("min_sep_cells", C.c_int64), ("max_frames", C.c_int64),
                ("flags", C.c_int32)]


PLAN_EXACT_JACOBI = 1
PLAN_TEMPORAL = 2


class BatchIO(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("x", "omega", "indices", "spectrum", "peak_cells", "peak_heights",
                                          "baseline", "peak_count", "status", "basis", "eigenvalues",
                                          "covariance")]


class HostOut(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("spectrum", "peak_cells", "peak_heights", "baseline", "peak_count",
                                          "status", "attempts")]


class SceneDesc(C.Structure):
    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("k", C.c_int64), ("theta_lo", C.c_double),
                ("theta_hi", C.c_double), ("min_sep", C.c_double), ("snr_lo_db", C.c_double),
                ("snr_hi_db", C.c_double), ("fixed_angles", C.c_void_p), ("d", C.c_double),
                ("lam", C.c_double)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1911_07434_b200.build` "
                          "(the CUDA extension is required; there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    i32, i64, u64, dbl, vp = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_void_p
    sig = {
        "fm_abi_version": (i32, []),
        "fm_status_string": (C.c_char_p, [i32]),
        "fm_last_error": (C.c_char_p, []),
        "fm_device_info": (i32, [i32, C.c_char_p, i32, vp]),
        "fm_rng_derive": (u64, [u64, u64]),
        "fm_rng_normals": (i32, [u64, i64, vp]),
        "fm_sample_without_replacement": (i32, [u64, i64, i64, vp]),
        "fm_gaussian_matrix_real": (i32, [i64, i64, u64, vp]),
        "fm_draw_omega_batch": (i32, [i64, vp, i64, i64, vp]),
        "fm_draw_indices_batch": (i32, [i64, vp, i64, i64, vp]),
        "fm_draw_uniforms_batch": (i32, [i64, vp, i64, vp]),
        "fm_generate_frames": (i32, [vp, u64, i64, i64, vp, vp, vp, i32]),
        "fm_plan_create": (i32, [vp, i32, vp]),
        "fm_plan_destroy": (i32, [vp]),
        "fm_plan_workspace_bytes": (i32, [vp, vp]),
        "fm_run_batch": (i32, [vp, i64, vp, vp]),
        "fm_rerun_frames": (i32, [vp, i64, vp, vp, vp]),
        "fm_plan_launches_per_batch": (i32, [vp]),
        "fm_plan_set_profiling": (i32, [vp, i32]),
        "fm_plan_stage_times": (i32, [vp, vp, vp]),
        "fm_plan_set_concurrency": (i32, [vp, i32]),
        "fm_plan_set_graphs": (i32, [vp, i32]),
        "fm_estimate_batch_host": (i32, [vp, i64, vp, vp, vp, vp]),
        "fm_pack_peak_records": (i32, [vp, vp, vp, i64, i64, vp, vp]),
        "fm_z_spatial_covariance": (i32, [i64, i64, vp, vp]),
        "fm_z_hermitian_eig": (i32, [i64, vp, vp, vp]),
        "fm_z_exact_signal_subspace": (i32, [i64, vp, i64, vp, vp, vp]),
        "fm_z_fast_music_1": (i32, [i64, vp, i64, i64, u64, vp, vp, vp]),
        "fm_z_fast_music_2": (i32, [i64, vp, i64, i64, i32, u64, vp, vp, vp, vp]),
        "fm_z_music_spectrum": (i32, [i64, i64, vp, i64, dbl, dbl, dbl, dbl, vp]),
        "fm_z_extract_peaks": (i32, [vp, i64, i64, i64, vp, vp, vp, vp, vp]),
        "fm_z_temporal_covariance": (i32, [i64, i64, vp, vp]),
        "fm_z_block_lanczos_subspace": (i32, [i64, vp, i64, i64, i32, vp, vp, vp, vp]),
        "fm_block_lanczos_batch": (i32, [vp, i64, i64, i64, i64, i32, vp, vp, vp, vp, vp]),
        "fm_temporal_covariance_batch": (i32, [vp, i64, i64, i64, vp, vp, vp, vp]),
        "fm_fmcx_write": (i32, [C.c_char_p, i64, i64, vp]),
        "fm_fmcx_read_header": (i32, [C.c_char_p, vp, vp]),
        "fm_fmcx_read": (i32, [C.c_char_p, i64, i64, vp]),
        "fm_z_fmcx_write": (i32, [C.c_char_p, i64, i64, vp]),
        "fm_z_fmcx_read": (i32, [C.c_char_p, i64, i64, vp]),
        "fm_fmcx_read_frames": (i32, [vp, i64, i64, i64, vp, i32]),
        "fm_fmcx_write_frames": (i32, [vp, i64, i64, i64, vp, i32]),
        "fm_z_write_matrix_csv": (i32, [C.c_char_p, i64, i64, vp]),
        "fm_write_spectrum_csv": (i32, [C.c_char_p, i64, dbl, dbl, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


LIB = _load()


def last_error() -> str:
    return LIB.fm_last_error().decode()


def ptr(a) -> int | None:
    """Address of a numpy array or torch tensor (None passes NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return int(a.data_ptr())
