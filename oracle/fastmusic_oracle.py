"""ORACLE — test infrastructure only (never imported by the product package).

fp64 CPU restatement of the reference Fast-MUSIC hot path (arXiv 1911.07434,
reference C++ at R/ = /root/reference/proj).  Only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference`` leg
of ``bench.py`` may import this module, and only as the checker / CPU baseline.

Each function cites the reference lines it restates.  Dense kernels come from
numpy/scipy LAPACK (Eigen 3, the reference's dependency, is absent from this
image — SURVEY.md §0 F3, §8c).  The algorithm (pivoted-QR rank rule, pinv
cutoff, Nystrom recovery, redraw policy, spectrum floor, peak rules) follows
the reference line by line; only decomposition *internals* differ, and the
outputs are invariant to those (bases up to unitary rotation, see
R/tests/test_spectrum.cpp:67-84).

Parity pinning: the random streams are pinned bit-for-bit to the
reference's own ``rng.hpp`` compiled here (tests/golden/rng_ref.json); the
linear algebra is pinned by re-running the reference's property tests
(R/tests/test_*.cpp tolerances) against this restatement; the reference ships
no golden vectors for the estimators, so those rows are "partially pinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
KPI = 3.14159265358979323846
EPS64 = np.finfo(np.float64).eps


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "_build", "liboracle_rng.so")
        if not os.path.exists(path):
            subprocess.run(["make", "-s", "-C", _HERE, "_build/liboracle_rng.so"], check=True)
        lib = ctypes.CDLL(path)
        u64, i64, dbl = ctypes.c_uint64, ctypes.c_int64, ctypes.c_double
        p = ctypes.c_void_p
        lib.or_derive.restype = u64
        lib.or_derive.argtypes = [u64, u64]
        lib.or_u64_stream.argtypes = [u64, i64, p]
        lib.or_uniform_stream.argtypes = [u64, i64, p]
        lib.or_normal_stream.argtypes = [u64, i64, p]
        lib.or_below_stream.argtypes = [u64, u64, i64, p]
        lib.or_sample_without_replacement.argtypes = [u64, i64, i64, p]
        lib.or_sample_without_replacement.restype = ctypes.c_int
        lib.or_gaussian_matrix_real.argtypes = [i64, i64, u64, p]
        lib.or_steering_vector.argtypes = [dbl, i64, dbl, dbl, p]
        lib.or_generate_frame.argtypes = [u64, i64, i64, i64, dbl, dbl, dbl, dbl, dbl, p, dbl, dbl,
                                          p, p, p]
        lib.or_generate_frame.restype = ctypes.c_int
        _LIB = lib
    return _LIB


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# --------------------------------------------------------------------------- errors
# R/include/fastmusic/types.hpp:18-43
class NonConvergenceError(RuntimeError):
    def __init__(self, what, residual):
        super().__init__(what)
        self.residual = residual


class RankDeficiencyError(RuntimeError):
    def __init__(self, what, column):
        super().__init__(what)
        self.column = column


# --------------------------------------------------------------------------- RNG
def derive(seed: int, tag: int) -> int:
    """R/src/linalg.cpp:70-75 (splitmix64 finalizer over seed ^ f(tag))."""
    return int(_lib().or_derive(seed & (2**64 - 1), tag & (2**64 - 1)))


def u64_stream(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.uint64)
    _lib().or_u64_stream(seed, n, _ptr(out))
    return out


def uniform_stream(seed: int, n: int) -> np.ndarray:
    """R/include/fastmusic/rng.hpp:23-25."""
    out = np.empty(n, np.float64)
    _lib().or_uniform_stream(seed, n, _ptr(out))
    return out


def normal_stream(seed: int, n: int) -> np.ndarray:
    """R/include/fastmusic/rng.hpp:28-39 (Box-Muller, cos first, cached sin)."""
    out = np.empty(n, np.float64)
    _lib().or_normal_stream(seed, n, _ptr(out))
    return out


def below_stream(seed: int, bound: int, n: int) -> np.ndarray:
    """R/include/fastmusic/rng.hpp:42-49."""
    out = np.empty(n, np.uint64)
    _lib().or_below_stream(seed, bound, n, _ptr(out))
    return out


def sample_without_replacement(seed: int, m: int, p: int) -> np.ndarray:
    """R/src/linalg.cpp:54-68 — partial Fisher-Yates, truncated, sorted."""
    out = np.empty(max(p, 0), np.int64)
    if _lib().or_sample_without_replacement(seed, m, p, _ptr(out)) != 0:
        raise ValueError("sample_without_replacement: need 1 <= p <= m")
    return out


def gaussian_matrix_real(m: int, p: int, seed: int) -> np.ndarray:
    """R/src/linalg.cpp:180-192 — M x p, row-major fill from Rng(seed).normal()."""
    if m < 1 or p < 1:
        raise ValueError("gaussian_matrix: need M, p >= 1")
    out = np.empty((m, p), np.float64)
    _lib().or_gaussian_matrix_real(m, p, seed, _ptr(out))
    return out


# --------------------------------------------------------------------------- scene
def steering_vector(theta: float, m: int, d: float = 0.5, lam: float = 1.0) -> np.ndarray:
    """R/src/scene.cpp:72-82 — a_i = polar(1, 2 pi d sin(theta) i / lambda)."""
    if m < 1 or d <= 0 or lam <= 0:
        raise ValueError("steering_vector: need M >= 1, d > 0, lambda > 0")
    buf = np.empty(2 * m, np.float64)
    _lib().or_steering_vector(float(theta), m, d, lam, _ptr(buf))
    return buf[0::2] + 1j * buf[1::2]


@dataclass
class SceneSpec:
    """Synthetic frame model for the BASELINE configs."""
    m: int
    n: int
    k: int
    theta_lo_deg: float = -60.0
    theta_hi_deg: float = 60.0
    min_sep_deg: float = 3.0
    snr_lo_db: float = 10.0
    snr_hi_db: float = 30.0
    fixed_angles_deg: tuple | None = None
    d: float = 0.5
    lam: float = 1.0


def frame_seed(base_seed: int, f: int) -> int:
    return derive(base_seed, f)


def generate_frame(fseed: int, spec: SceneSpec):
    """One frame: X (M x N complex64), true angles (rad, sorted), snr_db."""
    lib = _lib()
    x = np.empty((spec.m, spec.n), np.complex64)
    ang = np.empty(spec.k, np.float64)
    snr = np.empty(1, np.float64)
    fixed = None
    if spec.fixed_angles_deg is not None:
        fixed = np.array([a * KPI / 180.0 for a in spec.fixed_angles_deg], np.float64)
    rc = lib.or_generate_frame(fseed, spec.m, spec.n, spec.k, spec.theta_lo_deg * KPI / 180.0,
                               spec.theta_hi_deg * KPI / 180.0, spec.min_sep_deg * KPI / 180.0,
                               spec.snr_lo_db, spec.snr_hi_db,
                               _ptr(fixed) if fixed is not None else None, spec.d, spec.lam,
                               _ptr(x), _ptr(ang), _ptr(snr))
    if rc != 0:
        raise RuntimeError("generate_frame: cannot place targets at this separation")
    return x, ang, float(snr[0])


def generate_batch(base_seed: int, frames, spec: SceneSpec):
    xs, angs, snrs = [], [], []
    for f in frames:
        x, a, s = generate_frame(frame_seed(base_seed, f), spec)
        xs.append(x)
        angs.append(a)
        snrs.append(s)
    return np.stack(xs), np.stack(angs), np.array(snrs)


def spatial_covariance(y: np.ndarray) -> np.ndarray:
    """R/src/scene.cpp:138-159 + HermitianMatrix ctor R/src/linalg.cpp:46-52.

    S = Y Y^H / N, then 0.5 (S + S^H) (exactly Hermitian, real diagonal)."""
    y = np.asarray(y, np.complex128)
    if y.shape[0] < 1 or y.shape[1] < 1:
        raise ValueError("covariance: empty signal matrix")
    if not np.all(np.isfinite(y)):
        raise ValueError("covariance: non-finite entries")
    s = (y @ y.conj().T) / y.shape[1]
    return hermitian(s)


def temporal_covariance(y: np.ndarray) -> np.ndarray:
    """R/src/scene.cpp:140-153,161-163: T = Y^H Y / M (N x N), then 0.5 (T + T^H)."""
    y = np.asarray(y, np.complex128)
    if y.shape[0] < 1 or y.shape[1] < 1:
        raise ValueError("covariance: empty signal matrix")
    if not np.all(np.isfinite(y)):
        raise ValueError("covariance: non-finite entries")
    return hermitian((y.conj().T @ y) / y.shape[0])


def hermitian(a: np.ndarray) -> np.ndarray:
    """HermitianMatrix ctor, R/src/linalg.cpp:46-52."""
    a = np.asarray(a, np.complex128)
    if a.ndim != 2 or a.shape[0] != a.shape[1] or a.shape[0] < 1:
        raise ValueError("HermitianMatrix: input must be square and non-empty")
    if not np.all(np.isfinite(a)):
        raise ValueError("HermitianMatrix: non-finite entries")
    return 0.5 * (a + a.conj().T)


# --------------------------------------------------------------------------- linalg
def hermitian_eig(s: np.ndarray):
    """R/src/linalg.cpp:77-89 — full eig, eigenvalues descending."""
    w, v = np.linalg.eigh(s)
    return w[::-1].copy(), v[:, ::-1].copy()


def thin_svd(a: np.ndarray):
    """R/src/linalg.cpp:93-125 — thin SVD, sigma descending (u, sigma, v)."""
    if not np.all(np.isfinite(a)):
        raise ValueError("thin_svd: non-finite entries")
    u, s, vh = np.linalg.svd(a, full_matrices=False)
    return u, s, vh.conj().T


def _colpiv_rank(a: np.ndarray, r: np.ndarray) -> int:
    """Eigen ColPivHouseholderQR::rank() on the pivoted R of a: pivots counted while the remaining column
    norm stays above (maxColNorm*eps)^2/rows*(rows-k) (bug-941 rule), then |R_ii| > eps*diagsize*maxpivot."""
    rows, cols = a.shape
    diag = np.abs(np.diag(r))
    size = min(rows, cols)
    max_col_norm = np.max(np.linalg.norm(a, axis=0))
    thr_helper = (max_col_norm * EPS64) ** 2 / rows
    nonzero = size
    for k in range(size):
        if np.linalg.norm(r[k:, k]) ** 2 < thr_helper * (rows - k):
            nonzero = k
            break
    maxpivot = np.max(diag) if size else 0.0
    prem = maxpivot * EPS64 * size
    return int(np.sum(diag[:nonzero] > prem))


def qr_orthonormal(a: np.ndarray) -> np.ndarray:
    """R/src/linalg.cpp:127-141 — column-pivoted Householder QR.

    Rank follows Eigen's ColPivHouseholderQR::rank(): pivots counted while the
    remaining column norm stays above (maxColNorm*eps)^2/rows*(rows-k), then
    |R_ii| > eps*diagsize*maxpivot.  Deficient column = colsPermutation()(rank)."""
    if not np.all(np.isfinite(a)):
        raise ValueError("qr_orthonormal: non-finite entries")
    rows, cols = a.shape
    if cols < 1 or rows < cols:
        raise ValueError("qr_orthonormal: need rows >= cols >= 1")
    q, r, piv = scipy.linalg.qr(a, mode="economic", pivoting=True)
    rank = _colpiv_rank(a, r)
    if rank < cols:
        col = int(piv[rank])
        raise RankDeficiencyError(
            f"qr_orthonormal: rank {rank} < {cols} columns; column {col} is dependent", col)
    return q


def orthonormal_range(z: np.ndarray) -> np.ndarray:
    """R/src/estimators.cpp:143-149: Q of ColPivHouseholderQR(z) restricted to its numerical rank."""
    q, r, piv = scipy.linalg.qr(z, mode="economic", pivoting=True)
    return q[:, :_colpiv_rank(z, r)]


def pseudo_inverse(a: np.ndarray, rel_tol: float = 0.0) -> np.ndarray:
    """R/src/linalg.cpp:143-163 — SVD pinv, cutoff max(r,c)*eps*sigma1."""
    if not np.all(np.isfinite(a)):
        raise ValueError("pseudo_inverse: non-finite entries")
    if rel_tol < 0 or rel_tol >= 1:
        raise ValueError("pseudo_inverse: rel_tol must be in [0, 1)")
    if rel_tol == 0.0:
        rel_tol = max(a.shape) * EPS64
    u, s, v = thin_svd(a)
    sigma1 = s[0] if s.size else 0.0
    if sigma1 == 0.0:
        return np.zeros((a.shape[1], a.shape[0]), np.complex128)
    inv = np.where(s > rel_tol * sigma1, 1.0 / np.where(s > 0, s, 1.0), 0.0)
    return (v * inv) @ u.conj().T


# --------------------------------------------------------------------------- estimators
@dataclass
class SubspaceEstimate:
    """R/include/fastmusic/estimators.hpp:13-18."""
    basis: np.ndarray
    eigenvalues: np.ndarray
    method: str = "exact"
    attempts: int = 1
    extra: dict = field(default_factory=dict)


def clamp_nonnegative(v: np.ndarray) -> np.ndarray:
    """R/src/estimators.cpp:25-31."""
    out = np.array(v, np.float64)
    out[(out < 0.0) & (out >= -1e-10)] = 0.0
    return out


def rank_restricted_subspace(c, w, k, method):
    """R/src/estimators.cpp:37-50 — Nystrom rank-K recovery via two small SVDs."""
    uc, sc, vc = thin_svd(c)
    projected = (sc[:, None] * (vc.conj().T @ w @ vc)) * sc[None, :]
    ub, sb, _ = thin_svd(projected)
    u = uc @ ub
    return SubspaceEstimate(u[:, :k].copy(), clamp_nonnegative(sb[:k]), method)


def exact_signal_subspace(s, k):
    """R/src/estimators.cpp:73-85."""
    m = s.shape[0]
    if k < 1 or k >= m:
        raise ValueError("exact_signal_subspace: need 1 <= K < M")
    w, v = hermitian_eig(s)
    return SubspaceEstimate(v[:, :k].copy(), clamp_nonnegative(w[:k]), "exact")


def fast_music_1(s, k, p, seed):
    """R/src/estimators.cpp:87-102 — uniform column sampling + Nystrom weight."""
    m = s.shape[0]
    if k < 1 or k >= m:
        raise ValueError("fast_music_1: need 1 <= K < M")
    if p < k or p > m:
        raise ValueError("fast_music_1: need K <= p <= M")
    idx = sample_without_replacement(seed, m, p)
    c = s[:, idx]
    w = pseudo_inverse(s[np.ix_(idx, idx)])
    out = rank_restricted_subspace(c, w, k, "fast1")
    out.extra["indices"] = idx
    return out


def fast_music_2(s, k, p, t, seed, max_attempts=4):
    """R/src/estimators.cpp:104-139 — Gaussian sketch, t power rounds, Nystrom.

    Redraws with derive(seed, 0xF257 + attempt) on RankDeficiencyError."""
    m = s.shape[0]
    if k < 1 or k >= m:
        raise ValueError("fast_music_2: need 1 <= K < M")
    if p < k or p > m:
        raise ValueError("fast_music_2: need K <= p <= M")
    if t < 1 or t > 20:
        raise ValueError("fast_music_2: need 1 <= t <= 20")
    attempt = 0
    while True:
        draw_seed = seed if attempt == 0 else derive(seed, 0xF257 + attempt)
        try:
            pi = gaussian_matrix_real(m, p, draw_seed)
            c = (s.real @ pi) + 1j * (s.imag @ pi)
            v = None
            for _ in range(t):
                v = qr_orthonormal(c)
                c = s @ v
            w = pseudo_inverse(v.conj().T @ c)
            out = rank_restricted_subspace(c, w, k, "fast2")
            out.attempts = attempt + 1
            return out
        except RankDeficiencyError:
            if attempt + 1 >= max_attempts:
                raise
        attempt += 1


# --------------------------------------------------------------------------- spectrum
@dataclass(frozen=True)
class AngleGrid:
    """R/src/spectrum.cpp:18-33, generalised to [theta0, theta1].

    theta(i) = theta0 + (span * i) / (L - 1); theta0 = 0, span = pi reproduces
    the reference grid bit for bit."""
    size: int
    theta0: float = 0.0
    theta1: float = KPI

    def __post_init__(self):
        if self.size < 2:
            raise ValueError("AngleGrid: L >= 2 required")

    def thetas(self) -> np.ndarray:
        span = self.theta1 - self.theta0
        i = np.arange(self.size, dtype=np.float64)
        return self.theta0 + (span * i) / float(self.size - 1)


def norm2_sample_indices(s: np.ndarray, c: int, seed: int) -> np.ndarray:
    """EXTENSION, not in the reference (BASELINE config 3's wording): c column indices of S drawn
    without replacement with probability proportional to ||S(:, j)||^2 — Efraimidis-Spirakis: the c largest
    keys log(u_j) / w_j (ties: lower j; w_j = 0 never preferred), u_j = float32(j-th uniform01 of Rng(seed)).
    Returned ascending. Restates the library's k_norm2_select."""
    m = s.shape[0]
    w = np.sum(np.abs(s) ** 2, axis=0)
    u = uniform_stream(seed, m).astype(np.float32).astype(np.float64)
    keys = np.full(m, -np.inf)
    pos = w > 0
    keys[pos] = np.log(u[pos]) / w[pos]
    order = sorted(range(m), key=lambda j: (-keys[j], j))
    return np.sort(np.array(order[:c], dtype=np.int64))


def fast_music_1_norm2(s, k, c, seed, max_attempts=4, indices=None):
    """EXTENSION (see norm2_sample_indices): the fast2 tail with the sketch S(:, I) in place of S Omega and
    one power step — V = qr_orthonormal(S(:, I)), C = S V, W = pinv(V^H C), rank_restricted_subspace(C, W).
    Rank-deficient samples are redrawn with derive(seed, 0xF257 + attempt) like fast_music_2.
    `indices` fixes the selection (to check the tail on a given sample)."""
    m = s.shape[0]
    if k < 1 or k >= m:
        raise ValueError("fast_music_1_norm2: need 1 <= K < M")
    if c < k or c > m:
        raise ValueError("fast_music_1_norm2: need K <= p <= M")
    attempt = 0
    while True:
        draw_seed = seed if attempt == 0 else derive(seed, 0xF257 + attempt)
        try:
            idx = indices if indices is not None else norm2_sample_indices(s, c, draw_seed)
            v = qr_orthonormal(s[:, idx])
            cc = s @ v
            w = pseudo_inverse(v.conj().T @ cc)
            out = rank_restricted_subspace(cc, w, k, "fast1_norm2")
            out.attempts = attempt + 1
            out.indices = idx
            return out
        except RankDeficiencyError:
            if attempt + 1 >= max_attempts or indices is not None:
                raise
        attempt += 1


def block_lanczos_subspace(s, k, block, max_iterations):
    """R/src/estimators.cpp:154-222 — block Krylov with full reorthogonalisation; converged when the top-K
    Ritz values change by <= 1e-10 relative on two consecutive checks."""
    s = hermitian(s)
    m = s.shape[0]
    if k < 1 or k >= m:
        raise ValueError("block_lanczos_subspace: need 1 <= K < M")
    if block < k:
        raise ValueError("block_lanczos_subspace: need block >= K")
    if max_iterations < 1:
        raise ValueError("block_lanczos_subspace: iters >= 1")
    tol = 1e-10
    q = qr_orthonormal(gaussian_matrix_real(m, min(block, m), 0x6C616E637A6F).astype(np.complex128))
    basis = q
    h = np.zeros((0, 0), np.complex128)
    prev = None
    last_change = float("inf")
    stable = 0
    for _ in range(max_iterations):
        w = s @ q
        old, new = h.shape[0], w.shape[1]
        strip = basis.conj().T @ w
        hn = np.zeros((old + new, old + new), np.complex128)
        hn[:old, :old] = h
        hn[:old, old:] = strip[:old]
        hn[old:, :old] = strip[:old].conj().T
        hn[old:, old:] = strip[old:]
        h = hn
        ev, vec = hermitian_eig(hermitian(h))
        vals = ev[:min(k, h.shape[0])]

        def estimate():
            return SubspaceEstimate(basis @ vec[:, :k], clamp_nonnegative(vals), "lanczos")

        if prev is not None and len(prev) == len(vals) == k:
            change = float(np.max(np.abs(vals - prev) / np.maximum(np.abs(vals), 1e-300)))
            last_change = change
            stable = stable + 1 if change <= tol else 0
            if stable >= 2:
                return estimate()
        prev = vals
        room = m - basis.shape[1]
        if room <= 0:
            return estimate()
        z = w - basis @ (basis.conj().T @ w)
        z = z - basis @ (basis.conj().T @ z)
        q = orthonormal_range(z[:, :min(z.shape[1], room)])
        if q.shape[1] == 0:
            return estimate()
        basis = np.hstack([basis, q])
    raise NonConvergenceError("block_lanczos_subspace: no convergence within iteration cap", last_change)


def baseline_grid(l: int) -> AngleGrid:
    """BASELINE grids: L points over [-90, 90] degrees."""
    return AngleGrid(l, -KPI / 2.0, KPI / 2.0)


def steering_matrix(grid: AngleGrid, m: int, d=0.5, lam=1.0) -> np.ndarray:
    """Columns a(theta_l) exactly as R/src/scene.cpp:72-82 (glibc sin/cos)."""
    th = grid.thetas()
    out = np.empty((m, grid.size), np.complex128)
    for l in range(grid.size):
        out[:, l] = steering_vector(th[l], m, d, lam)
    return out


def music_denominator(basis: np.ndarray, a_mat: np.ndarray) -> np.ndarray:
    """R/src/spectrum.cpp:50-68 denominator M - ||U^H a||^2 (before flooring)."""
    m = basis.shape[0]
    c = basis.conj().T @ a_mat
    return float(m) - np.sum(np.abs(c) ** 2, axis=0)


def music_spectrum(basis: np.ndarray, grid: AngleGrid, d=0.5, lam=1.0, a_mat=None):
    """R/src/spectrum.cpp:37-68 — P = 1/max(M - ||U^H a||^2, 1e-12 M)."""
    m = basis.shape[0]
    if m < 1:
        raise ValueError("music_spectrum: empty basis")
    if basis.shape[1] > 0:
        dev = np.max(np.abs(basis.conj().T @ basis - np.eye(basis.shape[1])))
        if dev > 1e-6:
            raise ValueError("music_spectrum: basis columns are not orthonormal")
    if a_mat is None:
        a_mat = steering_matrix(grid, m, d, lam)
    den = music_denominator(basis, a_mat)
    return 1.0 / np.maximum(den, 1e-12 * m)


@dataclass
class PeakSet:
    """R/include/fastmusic/spectrum.hpp:34-42 (+ the selected grid cells)."""
    cells: list
    angles: list
    heights: list
    baseline: float
    shortfall: bool


def local_maxima(v: np.ndarray):
    """R/src/spectrum.cpp:105-122 — strict maxima, plateaus -> leftmost index.

    Run-length form of the reference scan: a run of equal values [s, e] yields s
    iff 1 <= s, v[s] > v[s-1], e + 1 < n and v[e+1] < v[s]."""
    v = np.asarray(v)
    n = v.size
    if n < 3:
        return []
    change = np.flatnonzero(v[1:] != v[:-1]) + 1
    starts = np.concatenate(([0], change))
    ends = np.concatenate((change - 1, [n - 1]))
    s, e = starts, ends
    ok = (s >= 1) & (e + 1 < n)
    s, e = s[ok], e[ok]
    ok = (v[s] > v[s - 1]) & (v[e + 1] < v[s])
    return [(int(c), float(v[c])) for c in s[ok]]


def extract_peaks(values: np.ndarray, k: int, min_sep: int, grid: AngleGrid | None = None) -> PeakSet:
    """R/src/spectrum.cpp:124-188 — rank (height desc, cell asc), greedy
    separation |dc| >= min_sep, baseline = max over cells farther than min_sep
    from every selected peak, output sorted by cell."""
    if k < 1:
        raise ValueError("extract_peaks: K >= 1 required")
    cands = local_maxima(values)
    cands.sort(key=lambda c: (-c[1], c[0]))
    sel = []
    for c in cands:
        if len(sel) == k:
            break
        if all(abs(c[0] - s[0]) >= min_sep for s in sel):
            sel.append(c)
    v = np.asarray(values)
    mask = np.ones(v.size, bool)
    for c, _ in sel:
        mask[max(0, c - min_sep):c + min_sep + 1] = False
    p0 = max(0.0, float(np.max(v[mask]))) if mask.any() else 0.0
    sel.sort(key=lambda c: c[0])
    cells = [c for c, _ in sel]
    th = grid.thetas() if grid is not None else None
    return PeakSet(cells, [float(th[c]) for c in cells] if th is not None else [],
                   [h for _, h in sel], p0, len(sel) < k)


# --------------------------------------------------------------------------- configs
@dataclass
class PathConfig:
    name: str
    method: str          # fast2 | fast1 | exact
    spec: SceneSpec
    frames: int
    grid_size: int
    p: int = 0
    t: int = 1
    base_seed: int = 0
    min_sep_cells: int = 3


def baseline_configs():
    """The five BASELINE.json configs (SURVEY.md §8d mapping F6/F7)."""
    c1 = PathConfig("c1", "fast2", SceneSpec(64, 200, 3, fixed_angles_deg=(-20.0, 5.0, 31.0),
                                               snr_lo_db=20.0, snr_hi_db=20.0),
                    1, 1801, p=8, t=1, base_seed=1)
    c2 = PathConfig("c2", "fast2", SceneSpec(256, 512, 8, -60.0, 60.0, 3.0, 10.0, 30.0),
                    1024, 3601, p=16, t=2, base_seed=2)
    c3 = PathConfig("c3", "fast1", SceneSpec(256, 512, 8, -60.0, 60.0, 3.0, 10.0, 30.0),
                    1024, 3601, p=32, base_seed=2)
    c4 = PathConfig("c4", "fast2", SceneSpec(1024, 2048, 16, -70.0, 70.0, 1.0, 20.0, 20.0),
                    256, 18001, p=32, t=2, base_seed=4)
    c5 = PathConfig("c5", "exact", SceneSpec(256, 512, 8, -60.0, 60.0, 3.0, 20.0, 20.0),
                    512, 3601, base_seed=2)
    # extension: config 3 with BASELINE's own sampling wording (norm^2-weighted; not in the reference, F6)
    c3n = PathConfig("c3n", "fast1_norm2", SceneSpec(256, 512, 8, -60.0, 60.0, 3.0, 10.0, 30.0),
                     1024, 3601, p=32, base_seed=2)
    # the paper's accurate baseline (block-Lanczos, block = K, cap 200 as R/include/fastmusic/bench.hpp:61-62)
    # on the c2 frames
    c2lz = PathConfig("c2lz", "lanczos", SceneSpec(256, 512, 8, -60.0, 60.0, 3.0, 10.0, 30.0),
                      1024, 3601, p=0, t=200, base_seed=2)
    return {c.name: c for c in (c1, c2, c3, c4, c5, c3n, c2lz)}


def frame_inputs(cfg: PathConfig, f: int):
    """Per-frame host draws: Omega (fast2) or sampled indices (fast1)."""
    s = frame_seed(cfg.base_seed, f)
    if cfg.method == "fast2":
        return {"seed": derive(s, 4)}
    if cfg.method in ("fast1", "fast1_norm2"):
        return {"seed": derive(s, 3)}
    return {}


def run_frame(cfg: PathConfig, x: np.ndarray, f: int, grid: AngleGrid | None = None, a_mat=None):
    """Full reference path for one frame: covariance -> subspace -> spectrum -> peaks."""
    grid = grid or baseline_grid(cfg.grid_size)
    k = cfg.spec.k
    s = spatial_covariance(x)
    fin = frame_inputs(cfg, f)
    if cfg.method == "fast2":
        est = fast_music_2(s, k, cfg.p, cfg.t, fin["seed"])
    elif cfg.method == "fast1":
        est = fast_music_1(s, k, cfg.p, fin["seed"])
    elif cfg.method == "fast1_norm2":
        est = fast_music_1_norm2(s, k, cfg.p, fin["seed"])
    elif cfg.method == "lanczos":  # block = p (0 selects K, R/include/fastmusic/bench.hpp:61), cap t
        est = block_lanczos_subspace(s, k, cfg.p or k, cfg.t)
    else:
        est = exact_signal_subspace(s, k)
    spec = music_spectrum(est.basis, grid, a_mat=a_mat)
    peaks = extract_peaks(spec, k, cfg.min_sep_cells, grid)
    return est, spec, peaks


# --------------------------------------------------------------------------- ToA path
@dataclass
class ToaSpec:
    """Seeded beat-signal frames (the reference's discrete beat model, R/include/fastmusic/scene.hpp:57-66:
    Y(m, n) = sum_k alpha_k rho_k kappa_k^n vartheta_k^m + noise) parametrised directly by the per-sample beat
    phase w_k (kappa_k = exp(j w_k) = delay_shift, R/src/scene.cpp:91) instead of an FMCW chirp."""
    m: int = 256
    n: int = 512
    k: int = 8
    w_lo: float = 0.2
    w_hi: float = 2.9
    min_sep: float = 0.05
    theta_lo_deg: float = -60.0
    theta_hi_deg: float = 60.0
    snr_db: float = 20.0


def generate_toa_frame(fseed: int, spec: ToaSpec):
    """One frame X (M x N complex64) and its sorted beat phases. Draws: Rng(derive(fseed, 1)) uniforms for the
    beat phases (rejection sampling with min separation, the angle pattern of R/src/bench.cpp:191-214), then the K
    angles, then the K gain phases (alpha_k rho_k = exp(j 2 pi u)); noise from Rng(derive(fseed, 2)) normals,
    row-major (re, im), variance sigma^2 = K / 10^(SNR/10) (R/src/bench.cpp:262-264)."""
    u = uniform_stream(derive(fseed, 1), 100000)
    pos = 0
    w = []
    while len(w) < spec.k:
        if pos >= u.size - 2 * spec.k:
            raise RuntimeError("generate_toa_frame: cannot place targets at this separation")
        c = spec.w_lo + (spec.w_hi - spec.w_lo) * u[pos]
        pos += 1
        if all(abs(c - x) >= spec.min_sep for x in w):
            w.append(c)
    w = np.sort(np.array(w))
    lo, hi = spec.theta_lo_deg * KPI / 180.0, spec.theta_hi_deg * KPI / 180.0
    th = lo + (hi - lo) * u[pos:pos + spec.k]
    ph = 2.0 * KPI * u[pos + spec.k:pos + 2 * spec.k]
    mm = np.arange(spec.m, dtype=np.float64)[:, None]
    nn = np.arange(spec.n, dtype=np.float64)[None, :]
    x = np.zeros((spec.m, spec.n), np.complex128)
    for k in range(spec.k):
        x += np.exp(1j * (ph[k] + KPI * np.sin(th[k]) * mm + w[k] * nn))
    sigma2 = spec.k / 10.0 ** (spec.snr_db / 10.0)
    z = normal_stream(derive(fseed, 2), 2 * spec.m * spec.n).reshape(spec.m, spec.n, 2)
    x += np.sqrt(sigma2 / 2.0) * (z[..., 0] + 1j * z[..., 1])
    return x.astype(np.complex64), w


def generate_toa_batch(base_seed: int, frames, spec: ToaSpec):
    xs, ws = zip(*(generate_toa_frame(frame_seed(base_seed, f), spec) for f in frames))
    return np.stack(xs), np.stack(ws)


def beat_grid(l: int, w0: float, w1: float) -> np.ndarray:
    """Beat phases w_l = w0 + ((w1 - w0) l) / (L - 1) (the AngleGrid formula, R/src/spectrum.cpp:26-28)."""
    return np.array([w0 + ((w1 - w0) * i) / (l - 1) for i in range(l)], np.float64)


def beat_steering_matrix(w: np.ndarray, n: int) -> np.ndarray:
    """Columns b_n(w) = exp(-j w n): the steering of T = Y^H Y / M, whose range is spanned by the conjugated
    beat vectors conj(kappa_k^n) (std::polar(1, -w n) as R/src/scene.cpp:79)."""
    out = np.empty((n, w.size), np.complex128)
    for l in range(w.size):
        ang = -w[l] * np.arange(n, dtype=np.float64)
        out[:, l] = np.cos(ang) + 1j * np.sin(ang)
    return out


def toa_spectrum(basis: np.ndarray, w: np.ndarray, b_mat=None) -> np.ndarray:
    """music_spectrum (R/src/spectrum.cpp:50-68) on the beat grid: P = 1 / max(N - ||U^H b(w)||^2, 1e-12 N)."""
    n = basis.shape[0]
    if b_mat is None:
        b_mat = beat_steering_matrix(w, n)
    return 1.0 / np.maximum(music_denominator(basis, b_mat), 1e-12 * n)


@dataclass
class ToaConfig:
    name: str = "toa"
    spec: ToaSpec = field(default_factory=ToaSpec)
    frames: int = 1024
    grid_size: int = 3601
    w0: float = 0.0
    w1: float = KPI
    p: int = 16
    t: int = 2
    base_seed: int = 6
    min_sep_cells: int = 3
    method: str = "fast2"


def run_toa_frame(cfg: ToaConfig, x: np.ndarray, f: int, b_mat=None):
    """ToA path for one frame: T = temporal_covariance(Y) (R/src/scene.cpp:161-163) -> fast_music_2 on T
    (R/src/estimators.cpp:104-139, Omega of dimension N from derive(frame seed, 4)) -> beat spectrum -> peaks."""
    t = temporal_covariance(x)
    seed = derive(frame_seed(cfg.base_seed, f), 4)
    est = fast_music_2(t, cfg.spec.k, cfg.p, cfg.t, seed)
    w = beat_grid(cfg.grid_size, cfg.w0, cfg.w1)
    spec = toa_spectrum(est.basis, w, b_mat)
    return est, spec, extract_peaks(spec, cfg.spec.k, cfg.min_sep_cells)


def spectrum_db_error(p_test: np.ndarray, p_ref: np.ndarray, dyn_db: float = 40.0) -> float:
    """max |10 log10(P/P_ref)| where P_ref >= max(P_ref) * 10^(-dyn/10) (BASELINE gate)."""
    p_ref = np.asarray(p_ref, np.float64)
    p_test = np.asarray(p_test, np.float64)
    mask = p_ref >= p_ref.max() * 10.0 ** (-dyn_db / 10.0)
    return float(np.max(np.abs(10.0 * np.log10(p_test[mask] / p_ref[mask]))))


def projector_error(a: np.ndarray, b: np.ndarray) -> float:
    """R/tests/test_estimators.cpp:41-43 — ||AA^H - BB^H||_2."""
    d = a @ a.conj().T - b @ b.conj().T
    return float(np.linalg.norm(d, 2))
