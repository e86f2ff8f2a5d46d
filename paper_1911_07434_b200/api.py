"""Python mirror of the reference estimator API, executed on the B200 through the C ABI.

Names, argument meaning and error behaviour follow R/include/fastmusic/{estimators,
spectrum,scene,types}.hpp so the parity tests read like the reference's own tests:
``fast_music_2(S, K, Fast2Params(p, t, seed))`` -> ``SubspaceEstimate``; parameter
violations raise ``ValueError`` (std::invalid_argument), rank-deficient sketches raise
``RankDeficiencyError`` after the reference's redraw policy, solver failures raise
``NonConvergenceError``.  ``BatchPlan`` drives the batched complex64 pipeline on
device tensors (torch is used only for device memory and streams).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import LIB, ptr

KPI = 3.14159265358979323846


class NonConvergenceError(RuntimeError):
    def __init__(self, what, residual=float("nan")):
        super().__init__(what)
        self.residual = residual


class RankDeficiencyError(RuntimeError):
    def __init__(self, what, column=-1):
        super().__init__(what)
        self.column = column


class SingularMatrixError(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


def _check(st: int, column: int = -1):
    if st == _capi.FM_OK:
        return
    msg = _capi.last_error()
    if st == _capi.FM_EINVAL:
        raise ValueError(msg)
    if st == _capi.FM_ERANK:
        raise RankDeficiencyError(msg, column)
    if st == _capi.FM_ENOCONV:
        raise NonConvergenceError(msg)
    if st == _capi.FM_ESINGULAR:
        raise SingularMatrixError(msg)
    if st == _capi.FM_ENOTSUP:
        raise NotImplementedError(msg)
    if st == _capi.FM_EIO:
        raise OSError(msg)
    raise CudaError(msg)


# ------------------------------------------------------------------ types
@dataclass
class Fast1Params:
    """R/include/fastmusic/estimators.hpp:20-23."""
    p: int = 0
    seed: int = 0


@dataclass
class Fast2Params:
    """R/include/fastmusic/estimators.hpp:25-29."""
    p: int = 0
    iterations: int = 1
    seed: int = 0


METHOD_NAMES = ("exact", "fast1", "fast2", "lanczos", "matrix_inverse", "propagator", "fft")


def method_name(method) -> str:
    """R/src/linalg.cpp:14-26 — the reference's names, by enum value or name."""
    if isinstance(method, str):
        return method if method in METHOD_NAMES else "unknown"
    return METHOD_NAMES[method] if 0 <= int(method) < len(METHOD_NAMES) else "unknown"


def method_from_name(name: str) -> int:
    """R/src/linalg.cpp:28-34 — Method enum value (types.hpp:45-53); ValueError('unknown method name: ...')."""
    if name not in METHOD_NAMES:
        raise ValueError("unknown method name: " + str(name))
    return METHOD_NAMES.index(name)


def is_finite(a) -> bool:
    """R/src/linalg.cpp:36-38."""
    return bool(np.all(np.isfinite(np.asarray(a))))


def ensure_finite(a, what: str) -> None:
    """R/src/linalg.cpp:40-44 — ValueError('<what>: non-finite entries')."""
    if not is_finite(a):
        raise ValueError(f"{what}: non-finite entries")


@dataclass
class EigResult:
    """R/include/fastmusic/types.hpp:78-83 — eigenvalues descending, column i pairs with eigenvalue i."""
    eigenvalues: np.ndarray
    eigenvectors: np.ndarray


@dataclass
class SvdResult:
    """R/include/fastmusic/types.hpp:85-90 — thin SVD, singular values descending."""
    u: np.ndarray
    sigma: np.ndarray
    v: np.ndarray


@dataclass
class SubspaceEstimate:
    """R/include/fastmusic/estimators.hpp:13-18."""
    basis: np.ndarray
    eigenvalues: np.ndarray
    method: str = "exact"
    cost_seconds: float = 0.0


@dataclass(frozen=True)
class AngleGrid:
    """R/include/fastmusic/spectrum.hpp:12-25, generalised to [theta0, theta1]."""
    size: int
    theta0: float = 0.0
    theta1: float = KPI

    def __post_init__(self):
        if self.size < 2:
            raise ValueError("AngleGrid: L >= 2 required")

    def spacing(self) -> float:
        return (self.theta1 - self.theta0) / float(self.size - 1)

    def theta(self, i) -> float:
        return self.theta0 + ((self.theta1 - self.theta0) * float(i)) / float(self.size - 1)

    def thetas(self) -> np.ndarray:
        return self.theta0 + ((self.theta1 - self.theta0) * np.arange(self.size, dtype=np.float64)) / float(self.size - 1)

    def nearest(self, theta: float) -> int:
        i = int(np.rint((theta - self.theta0) / self.spacing()))
        return min(max(i, 0), self.size - 1)


def baseline_grid(l: int) -> AngleGrid:
    return AngleGrid(l, -KPI / 2.0, KPI / 2.0)


@dataclass
class PseudoSpectrum:
    grid: AngleGrid
    values: np.ndarray
    method: str = "exact"
    degenerate: bool = False


@dataclass
class PeakSet:
    angles: list
    heights: list
    baseline: float = 0.0
    shortfall: bool = False
    cells: list = field(default_factory=list)


# ------------------------------------------------------------------ helpers
def _cmat(a) -> np.ndarray:
    """complex128, column-major (Eigen::MatrixXcd storage)."""
    return np.asfortranarray(np.asarray(a, dtype=np.complex128))


def hermitian(a) -> np.ndarray:
    """HermitianMatrix ctor (R/src/linalg.cpp:46-52): square, finite, 0.5 (A + A^H)."""
    a = np.asarray(a, dtype=np.complex128)
    if a.ndim != 2 or a.shape[0] != a.shape[1] or a.shape[0] < 1:
        raise ValueError("HermitianMatrix: input must be square and non-empty")
    if not np.all(np.isfinite(a)):
        raise ValueError("HermitianMatrix: non-finite entries")
    return _cmat(0.5 * (a + a.conj().T))


# ------------------------------------------------------------------ RNG (host, bit-exact)
def derive(seed: int, tag: int) -> int:
    return int(LIB.fm_rng_derive(seed & (2**64 - 1), tag & (2**64 - 1)))


def normals(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    _check(LIB.fm_rng_normals(seed, n, ptr(out)))
    return out


def sample_without_replacement(seed: int, m: int, p: int) -> np.ndarray:
    out = np.empty(max(p, 1), np.int64)
    _check(LIB.fm_sample_without_replacement(seed, m, p, ptr(out)))
    return out[:p]


def gaussian_matrix_real(m: int, p: int, seed: int) -> np.ndarray:
    out = np.empty((m, p), np.float64)
    _check(LIB.fm_gaussian_matrix_real(m, p, seed, ptr(out)))
    return out


def draw_omega_batch(seeds, m: int, p: int) -> np.ndarray:
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    out = np.empty((seeds.size, m, p), np.float32)
    _check(LIB.fm_draw_omega_batch(seeds.size, ptr(seeds), m, p, ptr(out)))
    return out


def draw_indices_batch(seeds, m: int, p: int) -> np.ndarray:
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    out = np.empty((seeds.size, p), np.int32)
    _check(LIB.fm_draw_indices_batch(seeds.size, ptr(seeds), m, p, ptr(out)))
    return out


def draw_uniforms_batch(seeds, m: int) -> np.ndarray:
    """fast1_norm2 draws: u[f][j] = float32(Rng(seeds[f]).uniform01()), j < m."""
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    out = np.empty((seeds.size, m), np.float32)
    _check(LIB.fm_draw_uniforms_batch(seeds.size, ptr(seeds), m, ptr(out)))
    return out


def generate_frames(m, n, k, base_seed, f0, frames, theta_lo_deg=-60.0, theta_hi_deg=60.0, min_sep_deg=3.0,
                    snr_lo_db=10.0, snr_hi_db=30.0, fixed_angles_deg=None, d=0.5, lam=1.0, threads=0, out=None):
    """Synthetic BASELINE frames; returns (x complex64 [frames, m, n], angles, snr)."""
    x = out if out is not None else np.empty((frames, m, n), np.complex64)
    ang = np.empty((frames, k), np.float64)
    snr = np.empty(frames, np.float64)
    fixed = None
    if fixed_angles_deg is not None:
        fixed = np.array([a * KPI / 180.0 for a in fixed_angles_deg], np.float64)
    sd = _capi.SceneDesc(m, n, k, theta_lo_deg * KPI / 180.0, theta_hi_deg * KPI / 180.0,
                         min_sep_deg * KPI / 180.0, snr_lo_db, snr_hi_db, ptr(fixed), d, lam)
    _check(LIB.fm_generate_frames(C.byref(sd), base_seed, f0, frames, ptr(x), ptr(ang), ptr(snr), threads))
    return x, ang, snr


# ------------------------------------------------------------------ reference single-matrix API
def steering_vector(theta: float, m: int, d: float, lam: float) -> np.ndarray:
    """R/src/scene.cpp:72-82."""
    if m < 1 or d <= 0 or lam <= 0:
        raise ValueError("steering_vector: need M >= 1, d > 0, lambda > 0")
    step = 2.0 * KPI * d * np.sin(theta) / lam
    ph = step * np.arange(m, dtype=np.float64)
    return np.cos(ph) + 1j * np.sin(ph)


def spatial_covariance(y) -> np.ndarray:
    """R/src/scene.cpp:157-159 — on the GPU in fp64."""
    y = _cmat(y)
    if y.ndim != 2 or y.shape[0] < 1 or y.shape[1] < 1:
        raise ValueError("covariance: empty signal matrix")
    s = np.empty((y.shape[0], y.shape[0]), np.complex128, order="F")
    _check(LIB.fm_z_spatial_covariance(y.shape[0], y.shape[1], ptr(y), ptr(s)))
    return s


def temporal_covariance(y) -> np.ndarray:
    """R/src/scene.cpp:161-163 (T = Y^H Y / M, N x N) — on the GPU in fp64."""
    y = _cmat(y)
    if y.ndim != 2 or y.shape[0] < 1 or y.shape[1] < 1:
        raise ValueError("covariance: empty signal matrix")
    t = np.empty((y.shape[1], y.shape[1]), np.complex128, order="F")
    _check(LIB.fm_z_temporal_covariance(y.shape[0], y.shape[1], ptr(y), ptr(t)))
    return t


def temporal_covariance_batch(x, out=None, status=None, stream=None, work=None):
    """Batched T_f = X_f^H X_f / M on the device (torch tensors: x complex64 [frames, M, N] or its float32
    view) -> complex64 [frames, N, N]; per-frame FM_FRAME_* bits in `status` (int32 [frames]). X is read in its
    stored order (no transpose pass). `work`: optional complex64 scratch used only for odd N, frames * M * (N + 1)
    elements (else allocated per call)."""
    import torch
    frames, m = x.shape[0], x.shape[1]
    n = x.shape[2] if x.dtype == torch.complex64 else x.shape[2] // 2
    if out is None:
        out = torch.empty((frames, n, n), dtype=torch.complex64, device=x.device)
    if status is None:
        status = torch.empty((frames,), dtype=torch.int32, device=x.device)
    s = None if stream is None else C.c_void_p(stream.cuda_stream)
    if work is not None and (n % 2) and work.numel() * work.element_size() < 8 * frames * m * (n + 1):
        raise ValueError("temporal_covariance_batch: work too small")
    _check(LIB.fm_temporal_covariance_batch(ptr(x), frames, m, n, ptr(out), ptr(status), ptr(work), s))
    return out, status


def block_lanczos_batch(s, k: int, block: int, max_iterations: int, stream=None):
    """Batched block_lanczos_subspace on device covariance matrices (torch complex64 [frames, M, M], Hermitian):
    returns (basis complex128 [frames, M, K], eigenvalues [frames, K], status int32 [frames], iterations int32
    [frames] = 10000 * Krylov iterations + Jacobi sweeps) as device tensors."""
    import torch
    if s.dtype != torch.complex64 or s.dim() != 3 or s.shape[1] != s.shape[2]:
        raise ValueError("block_lanczos_batch: need a complex64 [frames, M, M] device tensor")
    s = s.contiguous()  # row-major per frame (a transposed view would read S^T = conj(S))
    frames, m = s.shape[0], s.shape[1]
    dev = s.device
    basis = torch.empty((frames, k, m, 2), dtype=torch.float64, device=dev)
    eig = torch.empty((frames, k), dtype=torch.float64, device=dev)
    status = torch.empty((frames,), dtype=torch.int32, device=dev)
    iters = torch.empty((frames,), dtype=torch.int32, device=dev)
    q = None if stream is None else C.c_void_p(stream.cuda_stream)
    _check(LIB.fm_block_lanczos_batch(ptr(s), frames, m, k, block, max_iterations, ptr(basis), ptr(eig), ptr(status),
                                      ptr(iters), q))
    b = torch.view_as_complex(basis).transpose(1, 2)
    return b, eig, status, iters


def _est_out(m, k):
    return np.empty((m, k), np.complex128, order="F"), np.empty(k, np.float64), C.c_double(0.0)


def hermitian_eig(s) -> EigResult:
    """R/src/linalg.cpp:77-89 — full decomposition of a Hermitian matrix by one-sided Jacobi on the GPU (fp64)."""
    s = hermitian(s)
    m = s.shape[0]
    v = np.empty((m, m), np.complex128, order="F")
    e = np.empty(m, np.float64)
    _check(LIB.fm_z_hermitian_eig(m, ptr(s), ptr(e), ptr(v)))
    return EigResult(e, v)


def exact_signal_subspace(s, k: int) -> SubspaceEstimate:
    """R/src/estimators.cpp:73-85 — batched one-sided Jacobi on the GPU (fp64 here)."""
    s = hermitian(s)
    m = s.shape[0]
    if k < 1 or k >= m:
        raise ValueError("exact_signal_subspace: need 1 <= K < M")
    b, e, cost = _est_out(m, k)
    _check(LIB.fm_z_exact_signal_subspace(m, ptr(s), k, ptr(b), ptr(e), C.byref(cost)))
    return SubspaceEstimate(b, e, "exact", cost.value)


def block_lanczos_subspace(s, k: int, block: int, max_iterations: int) -> SubspaceEstimate:
    """R/src/estimators.cpp:154-222 — block Krylov with full reorthogonalisation, fp64 on the GPU.
    NonConvergenceError(residual = last relative Ritz-value change) at the iteration cap."""
    s = hermitian(s)
    m = s.shape[0]
    if k < 1 or k >= m:
        raise ValueError("block_lanczos_subspace: need 1 <= K < M")
    if block < k:
        raise ValueError("block_lanczos_subspace: need block >= K")
    if max_iterations < 1:
        raise ValueError("block_lanczos_subspace: iters >= 1")
    b, e, cost = _est_out(m, k)
    last = C.c_double(0.0)
    st = LIB.fm_z_block_lanczos_subspace(m, ptr(s), k, block, max_iterations, ptr(b), ptr(e), C.byref(cost),
                                         C.byref(last))
    if st == _capi.FM_ENOCONV:
        raise NonConvergenceError(_capi.last_error(), last.value)
    _check(st)
    return SubspaceEstimate(b, e, "lanczos", cost.value)


def fast_music_1(s, k: int, params: Fast1Params) -> SubspaceEstimate:
    """R/src/estimators.cpp:87-102."""
    s = hermitian(s)
    m = s.shape[0]
    if k < 1 or k >= m:
        raise ValueError("fast_music_1: need 1 <= K < M")
    if params.p < k or params.p > m:
        raise ValueError("fast_music_1: need K <= p <= M")
    b, e, cost = _est_out(m, k)
    _check(LIB.fm_z_fast_music_1(m, ptr(s), k, params.p, params.seed & (2**64 - 1), ptr(b), ptr(e), C.byref(cost)))
    return SubspaceEstimate(b, e, "fast1", cost.value)


def fast_music_2(s, k: int, params: Fast2Params) -> SubspaceEstimate:
    """R/src/estimators.cpp:104-139 (redraws with derive(seed, 0xF257 + attempt))."""
    s = hermitian(s)
    m = s.shape[0]
    if k < 1 or k >= m:
        raise ValueError("fast_music_2: need 1 <= K < M")
    if params.p < k or params.p > m:
        raise ValueError("fast_music_2: need K <= p <= M")
    if params.iterations < 1 or params.iterations > 20:
        raise ValueError("fast_music_2: need 1 <= t <= 20")
    b, e, cost = _est_out(m, k)
    col = C.c_int64(-1)
    st = LIB.fm_z_fast_music_2(m, ptr(s), k, params.p, params.iterations, params.seed & (2**64 - 1), ptr(b), ptr(e),
                               C.byref(cost), C.byref(col))
    _check(st, col.value)
    return SubspaceEstimate(b, e, "fast2", cost.value)


def music_spectrum(estimate: SubspaceEstimate, grid: AngleGrid, d: float, lam: float) -> PseudoSpectrum:
    """R/src/spectrum.cpp:50-68."""
    u = _cmat(estimate.basis)
    if u.ndim != 2 or u.shape[0] < 1:
        raise ValueError("music_spectrum: empty basis")
    vals = np.empty(grid.size, np.float64)
    _check(LIB.fm_z_music_spectrum(u.shape[0], u.shape[1], ptr(u) if u.size else None, grid.size, grid.theta0,
                                   grid.theta1, d, lam, ptr(vals)))
    return PseudoSpectrum(grid, vals, estimate.method)


def extract_peaks(p: PseudoSpectrum, k: int, min_separation_cells: int) -> PeakSet:
    """R/src/spectrum.cpp:182-188."""
    if k < 1:
        raise ValueError("extract_peaks: K >= 1 required")
    v = np.ascontiguousarray(p.values, np.float64)
    cells = np.empty(k, np.int64)
    heights = np.empty(k, np.float64)
    count, base, short = C.c_int64(0), C.c_double(0.0), C.c_int32(0)
    _check(LIB.fm_z_extract_peaks(ptr(v), v.size, k, min_separation_cells, ptr(cells), ptr(heights), C.byref(count),
                                  C.byref(base), C.byref(short)))
    n = count.value
    cl = [int(c) for c in cells[:n]]
    return PeakSet([p.grid.theta(c) for c in cl], [float(h) for h in heights[:n]], base.value, bool(short.value), cl)


# ------------------------------------------------------------------ frame I/O (R/src/io.cpp:66-131)
def _paths(paths):
    import os
    enc = [os.fsencode(q) for q in paths]
    return (C.c_char_p * max(1, len(enc)))(*enc), len(enc)


def write_matrix_binary(path, a) -> None:
    """write_matrix_binary, R/src/io.cpp:71-86 (FMCX: complex64 row-major; complex128 input is cast per part)."""
    a = np.asarray(a)
    if a.ndim != 2:
        raise ValueError("write_matrix_binary: 2-D matrix required")
    if a.dtype == np.complex64:
        c = np.ascontiguousarray(a)
        _check(LIB.fm_fmcx_write(str(path).encode(), a.shape[0], a.shape[1], ptr(c) if c.size else None))
    else:
        z = _cmat(a)
        _check(LIB.fm_z_fmcx_write(str(path).encode(), a.shape[0], a.shape[1], ptr(z) if z.size else None))


def read_matrix_binary(path) -> np.ndarray:
    """read_matrix_binary, R/src/io.cpp:88-109; returns the complex64 payload as a (rows, cols) array."""
    r, c = C.c_int64(0), C.c_int64(0)
    _check(LIB.fm_fmcx_read_header(str(path).encode(), C.byref(r), C.byref(c)))
    out = np.empty((r.value, c.value), np.complex64)
    _check(LIB.fm_fmcx_read(str(path).encode(), r.value, c.value, ptr(out) if out.size else None))
    return out


def read_frames(paths, m: int, n: int, out=None, threads: int = 0) -> np.ndarray:
    """Batch ingest: one M x N FMCX file per frame into x[f] (complex64 [frames, m, n]; pass a pinned
    buffer as `out` to feed BatchPlan.estimate_host without another copy)."""
    arr, cnt = _paths(paths)
    x = out if out is not None else np.empty((cnt, m, n), np.complex64)
    if x.dtype != np.complex64 or x.shape != (cnt, m, n) or not x.flags.c_contiguous:
        raise ValueError("read_frames: out must be C-contiguous complex64 [frames, m, n]")
    _check(LIB.fm_fmcx_read_frames(C.cast(arr, C.c_void_p), cnt, m, n, ptr(x), threads))
    return x


def write_frames(paths, x, threads: int = 0) -> None:
    """One FMCX file per frame of x (complex64 [frames, m, n])."""
    x = np.ascontiguousarray(x, np.complex64)
    arr, cnt = _paths(paths)
    if x.ndim != 3 or x.shape[0] != cnt:
        raise ValueError("write_frames: x must be [len(paths), m, n]")
    _check(LIB.fm_fmcx_write_frames(C.cast(arr, C.c_void_p), cnt, x.shape[1], x.shape[2], ptr(x), threads))


def write_matrix_csv(path, a) -> None:
    """write_matrix_csv, R/src/io.cpp:111-122."""
    z = _cmat(a)
    if z.ndim != 2:
        raise ValueError("write_matrix_csv: 2-D matrix required")
    _check(LIB.fm_z_write_matrix_csv(str(path).encode(), z.shape[0], z.shape[1], ptr(z) if z.size else None))


def write_spectrum_csv(path, spectrum: PseudoSpectrum) -> None:
    """write_spectrum_csv, R/src/io.cpp:124-131."""
    v = np.ascontiguousarray(spectrum.values, np.float64)
    if v.size != spectrum.grid.size:
        raise ValueError("write_spectrum_csv: values / grid size mismatch")
    _check(LIB.fm_write_spectrum_csv(str(path).encode(), spectrum.grid.size, spectrum.grid.theta0,
                                     spectrum.grid.theta1, ptr(v)))


# ------------------------------------------------------------------ batched plan
class BatchPlan:
    """fm_plan over device tensors (torch for allocation / streams only)."""

    def __init__(self, m, n, k, method="fast2", p=0, t=1, grid_size=3601, theta0=-KPI / 2, theta1=KPI / 2, d=0.5,
                 lam=1.0, min_sep_cells=3, max_frames=1, device=0, exact_jacobi=False, temporal=False):
        """exact_jacobi: the exact method runs the full Jacobi eigensolver on every frame (FM_PLAN_EXACT_JACOBI)
        instead of the certified subspace iteration. temporal: the ToA path (FM_PLAN_TEMPORAL) -- the pipeline runs
        on T = X^H X / M (N x N); theta0 / theta1 span the beat phase per sample w (radians), the spectrum scans
        exp(-j w n); K, p, omega, indices, basis and the covariance export refer to dimension N."""
        flags = (_capi.PLAN_EXACT_JACOBI if exact_jacobi else 0) | (_capi.PLAN_TEMPORAL if temporal else 0)
        self.desc = _capi.PlanDesc(m, n, k, _capi.METHOD[method], p, t, grid_size, theta0, theta1, d, lam,
                                   min_sep_cells, max_frames, flags)
        self.method, self.m, self.n, self.k, self.p, self.t, self.L = method, m, n, k, p, t, grid_size
        self.temporal = temporal
        self.dim = n if temporal else m  # dimension of the covariance the subspace is estimated on
        self.max_frames, self.device = max_frames, device
        h = C.c_void_p()
        _check(LIB.fm_plan_create(C.byref(self.desc), device, C.byref(h)))
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            LIB.fm_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        self.close()

    def workspace_bytes(self) -> int:
        b = C.c_int64(0)
        _check(LIB.fm_plan_workspace_bytes(self.handle, C.byref(b)))
        return b.value

    def set_profiling(self, on: bool = True):
        _check(LIB.fm_plan_set_profiling(self.handle, 1 if on else 0))

    def stage_times_ms(self):
        """Summed {covariance, subspace, autocorr, spectrum_peaks} ms and the number of batches
        recorded since profiling was enabled / last read (call after synchronising)."""
        ms = np.zeros(4, np.float32)
        runs = C.c_int32(0)
        _check(LIB.fm_plan_stage_times(self.handle, ptr(ms), C.byref(runs)))
        return dict(zip(("covariance", "subspace", "autocorr", "spectrum_peaks"), ms.astype(float))), runs.value

    def set_concurrency(self, subbatches: int):
        """Run each batch as `subbatches` concurrent frame ranges (0 = automatic)."""
        _check(LIB.fm_plan_set_concurrency(self.handle, subbatches))

    def set_graphs(self, on: bool = True):
        """Replay identical batches (same frames and buffers) from a captured CUDA graph (one launch per batch)."""
        _check(LIB.fm_plan_set_graphs(self.handle, 1 if on else 0))

    def launches_per_batch(self) -> int:
        return int(LIB.fm_plan_launches_per_batch(self.handle))

    def outputs(self, frames, spectrum=True, basis=False, covariance=False):
        import torch
        dev = torch.device("cuda", self.device)
        o = {
            "peak_cells": torch.empty((frames, self.k), dtype=torch.int32, device=dev),
            "peak_heights": torch.empty((frames, self.k), dtype=torch.float64, device=dev),
            "baseline": torch.empty((frames,), dtype=torch.float64, device=dev),
            "peak_count": torch.empty((frames,), dtype=torch.int32, device=dev),
            "status": torch.empty((frames,), dtype=torch.int32, device=dev),
        }
        if spectrum:
            o["spectrum"] = torch.empty((frames, self.L), dtype=torch.float32, device=dev)
        if basis:
            o["basis"] = torch.empty((frames, self.k, self.dim, 2), dtype=torch.float64, device=dev)
            o["eigenvalues"] = torch.empty((frames, self.k), dtype=torch.float64, device=dev)
        if covariance:
            o["covariance"] = torch.empty((frames, self.dim, self.dim, 2), dtype=torch.float32, device=dev)
        return o

    def _io(self, x, omega, indices, out):
        return _capi.BatchIO(ptr(x), ptr(omega), ptr(indices), ptr(out.get("spectrum")), ptr(out["peak_cells"]),
                             ptr(out["peak_heights"]), ptr(out["baseline"]), ptr(out["peak_count"]),
                             ptr(out["status"]), ptr(out.get("basis")), ptr(out.get("eigenvalues")),
                             ptr(out.get("covariance")))

    def run(self, frames, x, omega=None, indices=None, out=None, stream=None):
        """x: device float32 view of complex64 [frames, M, N]; omega float32 [frames, M, p]; indices int32."""
        io = self._io(x, omega, indices, out)
        s = None if stream is None else C.c_void_p(stream.cuda_stream)
        _check(LIB.fm_run_batch(self.handle, frames, C.byref(io), s))
        return out

    def rerun(self, frame_list, x, omega=None, indices=None, out=None, stream=None):
        """Subspace + spectrum + peaks again for the listed frames (ascending indices of the last batch) on the
        kept covariance; x / omega / indices / out are the whole batch's buffers."""
        fl = np.ascontiguousarray(np.asarray(frame_list, np.int32))
        io = self._io(x, omega, indices, out)
        s = None if stream is None else C.c_void_p(stream.cuda_stream)
        _check(LIB.fm_rerun_frames(self.handle, fl.size, ptr(fl) if fl.size else None, C.byref(io), s))
        return out

    def estimate_host(self, x_host, draw_seeds, spectrum=None, heights=None, baseline=None, stream=None):
        """End-to-end from host buffers (pinned recommended): returns dict of host arrays."""
        frames = x_host.shape[0]
        cells = np.empty((frames, self.k), np.int32)
        count = np.empty(frames, np.int32)
        status = np.empty(frames, np.int32)
        attempts = np.empty(frames, np.int32)
        seeds = None if draw_seeds is None else np.ascontiguousarray(draw_seeds, np.uint64)
        ho = _capi.HostOut(ptr(spectrum), ptr(cells), ptr(heights), ptr(baseline), ptr(count), ptr(status),
                           ptr(attempts))
        s = None if stream is None else C.c_void_p(stream.cuda_stream)
        _check(LIB.fm_estimate_batch_host(self.handle, frames, ptr(x_host), ptr(seeds), C.byref(ho), s))
        return {"peak_cells": cells, "peak_count": count, "status": status, "attempts": attempts,
                "spectrum": spectrum, "peak_heights": heights, "baseline": baseline}
