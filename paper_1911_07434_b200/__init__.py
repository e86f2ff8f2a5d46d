"""fastmusic_b200 — B200-native (sm_100a) Fast-MUSIC hot path (arXiv 1911.07434).

The compute lives in ``libfastmusic_b200.so`` (hand-written CUDA kernels behind the
C ABI in ``include/fastmusic_b200.h``); this package is the Python mirror of the
reference estimator API over that ABI. Importing fails loudly if the library is absent.
"""
from .api import (AngleGrid, BatchPlan, CudaError, EigResult, Fast1Params, Fast2Params, NonConvergenceError, PeakSet,  # noqa: F401
                  PseudoSpectrum, RankDeficiencyError, SingularMatrixError, SubspaceEstimate, SvdResult, baseline_grid,
                  ensure_finite, hermitian_eig, is_finite, method_from_name, method_name,
                  block_lanczos_batch, block_lanczos_subspace, derive,
                  draw_indices_batch, draw_omega_batch, draw_uniforms_batch, exact_signal_subspace, extract_peaks, fast_music_1,
                  fast_music_2, gaussian_matrix_real, generate_frames, hermitian, music_spectrum, normals,
                  read_frames, read_matrix_binary, sample_without_replacement, spatial_covariance, steering_vector, temporal_covariance,
                  temporal_covariance_batch,
                  write_frames, write_matrix_binary, write_matrix_csv, write_spectrum_csv)
from ._capi import LIB_PATH  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]
