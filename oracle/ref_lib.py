"""ORACLE — test infrastructure only. ctypes binding of oracle/_ref/libref_fastmusic.so: the REFERENCE's own
scene / linalg / estimators / spectrum sources compiled in place against the Eigen-API shim (oracle/Makefile,
oracle/eigen_shim, oracle/ref_wrap.cpp). Exists only where /root/reference was present at build time (this dev
container); tests/golden/make_ref_golden.py turns its outputs into committed fixtures for everywhere else.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libref_fastmusic.so")
_LIB = None
STATUS = {0: "ok", 1: "invalid_argument", 2: "rank_deficiency", 3: "non_convergence"}


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _LIB
    if _LIB is None:
        L = C.CDLL(LIB_PATH)
        vp, i64, u64, dbl, i32 = C.c_void_p, C.c_int64, C.c_uint64, C.c_double, C.c_int32
        sig = {
            "ref_steering_vector": [dbl, i64, dbl, dbl, vp],
            "ref_spatial_covariance": [vp, i64, i64, vp],
            "ref_temporal_covariance": [vp, i64, i64, vp],
            "ref_exact_signal_subspace": [vp, i64, i64, vp, vp],
            "ref_fast_music_1": [vp, i64, i64, i64, u64, vp, vp],
            "ref_fast_music_2": [vp, i64, i64, i64, C.c_int, u64, vp, vp, vp],
            "ref_music_spectrum": [vp, i64, i64, i64, dbl, dbl, vp],
            "ref_extract_peaks": [vp, i64, i64, i64, vp, vp, vp, vp, vp],
            "ref_synthesize_beat_signal": [i64, i64, i64, vp, dbl, u64, vp],
            "ref_run_frame": [vp, i64, i64, C.c_int, C.c_int, i64, i64, C.c_int, u64, i64, i64, vp, vp, vp],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        _LIB = L
    return _LIB


def _p(a):
    return a.ctypes.data


def _cm(a):
    """column-major complex128 copy (Eigen layout)."""
    return np.asfortranarray(np.asarray(a, np.complex128))


def steering_vector(theta, m, d=0.5, lam=1.0):
    out = np.empty(m, np.complex128)
    assert lib().ref_steering_vector(theta, m, d, lam, _p(out)) == 0
    return out


def spatial_covariance(y):
    y = _cm(y)
    s = np.empty((y.shape[0], y.shape[0]), np.complex128, order="F")
    st = lib().ref_spatial_covariance(_p(y), y.shape[0], y.shape[1], _p(s))
    if st:
        raise ValueError(STATUS[st])
    return s


def temporal_covariance(y):
    y = _cm(y)
    t = np.empty((y.shape[1], y.shape[1]), np.complex128, order="F")
    st = lib().ref_temporal_covariance(_p(y), y.shape[0], y.shape[1], _p(t))
    if st:
        raise ValueError(STATUS[st])
    return t


def _estimate(fn, s, k, *args):
    s = _cm(s)
    m = s.shape[0]
    basis = np.empty((m, k), np.complex128, order="F")
    eig = np.empty(k, np.float64)
    st = fn(_p(s), m, k, *args, _p(basis), _p(eig))
    return st, basis, eig


def exact_signal_subspace(s, k):
    st, b, e = _estimate(lib().ref_exact_signal_subspace, s, k)
    if st:
        raise RuntimeError(STATUS[st])
    return b, e


def fast_music_1(s, k, p, seed):
    st, b, e = _estimate(lib().ref_fast_music_1, s, k, p, C.c_uint64(seed))
    if st:
        raise RuntimeError(STATUS[st])
    return b, e


def fast_music_2(s, k, p, t, seed):
    """(status, basis, eigenvalues, deficient column)."""
    s = _cm(s)
    m = s.shape[0]
    basis = np.empty((m, k), np.complex128, order="F")
    eig = np.empty(k, np.float64)
    col = C.c_int64(-1)
    st = lib().ref_fast_music_2(_p(s), m, k, p, t, C.c_uint64(seed), _p(basis), _p(eig), C.byref(col))
    return st, basis, eig, col.value


def music_spectrum(basis, L, d=0.5, lam=1.0):
    """On the reference grid AngleGrid(L) = [0, pi]."""
    b = _cm(basis)
    out = np.empty(L, np.float64)
    st = lib().ref_music_spectrum(_p(b), b.shape[0], b.shape[1], L, d, lam, _p(out))
    if st:
        raise ValueError(STATUS[st])
    return out


def extract_peaks(values, k, min_sep):
    v = np.ascontiguousarray(values, np.float64)
    cells = np.empty(max(k, 1), np.int64)
    heights = np.empty(max(k, 1), np.float64)
    cnt = C.c_int64(0)
    base = C.c_double(0.0)
    sf = C.c_int32(0)
    st = lib().ref_extract_peaks(_p(v), v.size, k, min_sep, _p(cells), _p(heights), C.byref(cnt), C.byref(base),
                                 C.byref(sf))
    if st:
        raise ValueError(STATUS[st])
    n = cnt.value
    return [int(c) for c in cells[:n]], [float(h) for h in heights[:n]], base.value, bool(sf.value)


def synthesize_beat_signal(m, n, angles, noise_var, seed):
    a = np.ascontiguousarray(angles, np.float64)
    y = np.empty((m, n), np.complex128, order="F")
    st = lib().ref_synthesize_beat_signal(m, n, a.size, _p(a), noise_var, C.c_uint64(seed), _p(y))
    if st:
        raise ValueError(STATUS[st])
    return y


METHODS = {"exact": 0, "fast1": 1, "fast2": 2, "lanczos": 3}


def run_frame(x, k, method, p, t, seed, L, min_sep=3, temporal=False, spectrum=False):
    """The reference path for one frame (ref_run_frame): returns (status, cells, spectrum or None)."""
    y = _cm(x)
    cells = np.empty(max(k, 1), np.int64)
    count = C.c_int64(0)
    spec = np.empty(L, np.float64) if spectrum else None
    st = lib().ref_run_frame(_p(y), y.shape[0], y.shape[1], 1 if temporal else 0, METHODS[method], k, p, t,
                             C.c_uint64(seed), L, min_sep, _p(cells), C.byref(count),
                             _p(spec) if spec is not None else None)
    return st, [int(c) for c in cells[:count.value]], spec
