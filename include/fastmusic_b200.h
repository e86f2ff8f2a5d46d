/* fastmusic_b200 — C ABI of the B200-native Fast-MUSIC hot path (arXiv 1911.07434).
 *
 * Plain pointers and sizes only. Every entry point replaces a reference C++ function
 * (R/ = reference proj/ tree); the reference has no FFI of its own, so these are the
 * symbols a maintainer binds (ctypes / cgo / JNI stubs in INTEGRATION.md) and the
 * C++ facade (include/fastmusic_b200/fastmusic.hpp) re-exposes them under the
 * reference names with the reference's exceptions.
 *
 * Matrices crossing the single-matrix ("_z", complex128) entry points are column-major
 * interleaved (re, im) doubles exactly like Eigen::MatrixXcd::data() in the reference.
 * Batched entry points take DEVICE pointers and a cudaStream_t passed as void*.
 */
#ifndef FASTMUSIC_B200_H
#define FASTMUSIC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; the facade maps them onto the reference exceptions
 * (R/include/fastmusic/types.hpp:17-43): EINVAL -> std::invalid_argument,
 * ERANK -> RankDeficiencyError, ENOCONV -> NonConvergenceError,
 * ESINGULAR -> SingularMatrixError. */
typedef int32_t fm_status;
#define FM_OK 0
#define FM_EINVAL 1
#define FM_ERANK 2
#define FM_ENOCONV 3
#define FM_ESINGULAR 4
#define FM_ECUDA 5
#define FM_ENOTSUP 6
#define FM_EIO 7 /* file I/O (std::runtime_error in the reference's io.cpp) */

/* Per-frame status bits written by the batched kernels. */
#define FM_FRAME_OK 0
#define FM_FRAME_RANK 1
#define FM_FRAME_NOCONV 2
#define FM_FRAME_RANGE 4     /* max |x| outside [2^-50, 2^50]: R would leave the complex64 range */
#define FM_FRAME_NONFINITE 8

/* Method enum values follow R/include/fastmusic/types.hpp:46-54 for the three hot-path methods. */
#define FM_METHOD_EXACT 0
#define FM_METHOD_FAST1 1
#define FM_METHOD_FAST2 2
/* block_lanczos_subspace (R/src/estimators.cpp:154-222, Method::Lanczos = 3): fm_plan_desc.p is the block
 * (0 selects K, R/include/fastmusic/bench.hpp:61; block <= 16), .t the iteration cap (>= 1; the reference's bench
 * uses 200). The whole Krylov loop runs on the device, one CTA per frame (lanczos_batch.cu); a frame that hits the
 * cap, or needs more than 72 basis columns, is flagged FM_FRAME_NOCONV. No per-frame draws. */
#define FM_METHOD_LANCZOS 3
/* Extension (BASELINE config 3's wording, not in the reference): p columns of R drawn without
 * replacement with probability proportional to their squared norm (Efraimidis-Spirakis keys log(u_j) / w_j,
 * u_j host uniforms from the reference RNG), orthonormalised, one product R V, Nystrom tail as fast2. */
#define FM_METHOD_FAST1_NORM2 16

int32_t fm_abi_version(void);
const char* fm_status_string(fm_status s);
/* Message of the last failure on the calling thread (never NULL). */
const char* fm_last_error(void);
/* Device name and SM count; FM_ECUDA if no device. */
fm_status fm_device_info(int32_t device, char* name, int32_t name_len, int32_t* sm_count);

/* ------------------------------------------------------------------ host random streams
 * Bit-exact restatements of the reference generators (run on the host; the draws are
 * copied to the device, as the BASELINE contract requires). */
/* Rng::derive, R/src/linalg.cpp:70-75 */
uint64_t fm_rng_derive(uint64_t seed, uint64_t tag);
/* first n outputs of Rng(seed).normal(), R/include/fastmusic/rng.hpp:28-39 */
fm_status fm_rng_normals(uint64_t seed, int64_t n, double* out);
/* Rng(seed).sample_without_replacement(m, p), R/src/linalg.cpp:54-68 */
fm_status fm_sample_without_replacement(uint64_t seed, int64_t m, int64_t p, int64_t* out);
/* gaussian_matrix_real(m, p, seed) row-major, R/src/linalg.cpp:180-192 */
fm_status fm_gaussian_matrix_real(int64_t m, int64_t p, uint64_t seed, double* out);
/* Batched per-frame draws (threaded): omega (frames x m x p float, row-major per frame)
 * from seeds[f] (fast2), or indices (frames x p int32) from seeds[f] (fast1). */
fm_status fm_draw_omega_batch(int64_t frames, const uint64_t* seeds, int64_t m, int64_t p, float* omega);
fm_status fm_draw_indices_batch(int64_t frames, const uint64_t* seeds, int64_t m, int64_t p, int32_t* indices);
/* FM_METHOD_FAST1_NORM2 draws: u[f][j] = (float) Rng(seeds[f]).uniform01(), j < m (frames x m) */
fm_status fm_draw_uniforms_batch(int64_t frames, const uint64_t* seeds, int64_t m, float* u);

/* Synthetic BASELINE frames: frame f of a batch uses seed derive(base_seed, f0 + f).
 * x: frames x m x n complex64 interleaved row-major. angles (frames x k rad) / snr (frames)
 * may be NULL. fixed_angles (k rad) may be NULL. Threaded over frames. */
typedef struct fm_scene_desc {
    int64_t m, n, k;
    double theta_lo, theta_hi, min_sep; /* radians */
    double snr_lo_db, snr_hi_db;
    const double* fixed_angles; /* k entries or NULL */
    double d, lambda;
} fm_scene_desc;
fm_status fm_generate_frames(const fm_scene_desc* scene, uint64_t base_seed, int64_t f0, int64_t frames, float* x,
                             double* angles, double* snr_db, int32_t threads);

/* ------------------------------------------------------------------ batched plan (device) */
typedef struct fm_plan_desc {
    int64_t m;              /* antennas M */
    int64_t n;              /* snapshots N (even) */
    int64_t k;              /* sources K, 1 <= K < M, K <= 64 */
    int32_t method;         /* FM_METHOD_* */
    int64_t p;              /* sketch width (fast1/fast2), K <= p <= min(M, 64) */
    int32_t t;              /* power iterations (fast2), 1..20 */
    int64_t grid_size;      /* L >= 2 */
    double theta0, theta1;  /* grid span, theta_l = theta0 + ((theta1-theta0) * l) / (L-1) */
    double d, lambda;       /* ULA spacing and wavelength */
    int64_t min_sep_cells;  /* peak separation (R/include/fastmusic/bench.hpp:71 default 3) */
    int64_t max_frames;     /* workspace capacity */
    int32_t flags;          /* FM_PLAN_* bits (0 = defaults) */
} fm_plan_desc;
/* exact method: full Jacobi eigensolver on every frame instead of the certified subspace iteration */
#define FM_PLAN_EXACT_JACOBI 1
/* ToA path (SURVEY.md §8(f)4, R/PAPER.md §II-B "the estimation of ToAs may be similarly accomplished with T"):
 * the pipeline runs on the temporal covariance T = X^H X / M (N x N, temporal_covariance R/src/scene.cpp:161-163)
 * instead of R. X keeps its M x N layout; K, p and the per-frame draws (omega frames x N x p, indices < N, basis
 * frames x K x N, covariance export frames x N x N) refer to the N-dimensional problem (1 <= K < N, p <= N). The
 * grid is the beat phase per sample, w_l = theta0 + (theta1 - theta0) l / (L - 1) in radians (w = mu tau T_s, the
 * delay_shift of R/src/scene.cpp:91; d and lambda are ignored), and the spectrum scans the steering of T's range,
 * b_n(w) = exp(-j w n). */
#define FM_PLAN_TEMPORAL 2
typedef struct fm_plan_s* fm_plan;

/* Validates like the reference (R/src/estimators.cpp:74-76,88-92,105-112) and allocates
 * device workspace + the shared grid table on `device`. */
fm_status fm_plan_create(const fm_plan_desc* desc, int32_t device, fm_plan* out);
fm_status fm_plan_destroy(fm_plan plan);
fm_status fm_plan_workspace_bytes(fm_plan plan, int64_t* bytes);

typedef struct fm_batch_io {
    const float* x;          /* frames x M x N complex64, row-major (FMCX order) */
    const float* omega;      /* fast2: frames x M x p, row-major; fast1_norm2: frames x M uniforms; else NULL */
    const int32_t* indices;  /* fast1: frames x p sorted column indices; else NULL */
    float* spectrum;         /* frames x L fp32 pseudo-spectrum, or NULL */
    int32_t* peak_cells;     /* frames x K grid cells ascending (-1 past count) */
    double* peak_heights;    /* frames x K */
    double* baseline;        /* frames */
    int32_t* peak_count;     /* frames (shortfall <=> count < K) */
    int32_t* status;         /* frames FM_FRAME_* bits (zeroed by the call) */
    double* basis;           /* frames x K x M complex128 column-major, or NULL */
    double* eigenvalues;     /* frames x K, or NULL */
    float* covariance;       /* frames x M x M complex64 export of R, or NULL */
} fm_batch_io;

/* Device-resident batched pipeline: covariance -> subspace -> spectrum -> peaks, enqueued
 * on `stream` (cudaStream_t, may be NULL). Asynchronous; per-frame status in io->status.
 * Frames whose Nystrom tail is singular (H = V^H C or S(I, I) singular, e.g. N < p) are finished by an
 * exact-algebra fallback with the reference's truncating pseudo-inverse; frames with max |x| outside the fp16
 * operand range are recomputed with a power-of-two prescale. Neither sets a status bit. */
fm_status fm_run_batch(fm_plan plan, int64_t frames, const fm_batch_io* io, void* stream);
/* Re-run subspace + spectrum + peaks for the listed frames (HOST int32 list of ascending frame indices of the
 * batch `io` describes) on the covariance kept from the last fm_run_batch / fm_estimate_batch_host; io->omega /
 * io->indices carry the new draws (fast2 redraws use derive(seed, 0xF257 + attempt), R/src/estimators.cpp:114-137).
 * Other frames' outputs are untouched. Asynchronous on `stream`. */
fm_status fm_rerun_frames(fm_plan plan, int64_t count, const int32_t* h_frames, const fm_batch_io* io, void* stream);
/* Stage timing: when enabled, every fm_run_batch records CUDA events on its stream between
 * its stages; once the stream is synchronised, fm_plan_stage_times returns the summed
 * {covariance, subspace, autocorrelation, spectrum+peaks} ms over the batches recorded since
 * profiling was enabled (or last read), their count in *runs, and restarts the count. */
fm_status fm_plan_set_profiling(fm_plan plan, int32_t on);
fm_status fm_plan_stage_times(fm_plan plan, float* ms4, int32_t* runs);
/* Split each fm_run_batch into `subbatches` (<= 16) frame ranges run concurrently on plan-owned streams forked
 * from / joined into the caller's stream (0 = automatic: 1 on the p <= 16 plane path, else 2 when frames >= 512). */
fm_status fm_plan_set_concurrency(fm_plan plan, int32_t subbatches);
/* CUDA-graph replay (on != 0): the first fm_run_batch with a given (frames, io) on a non-NULL stream is captured
 * into a graph and every later identical call replays it with one launch (small batches are otherwise bound by
 * the host's launch rate). Not used while profiling. Captured graphs are dropped by fm_plan_set_concurrency. */
fm_status fm_plan_set_graphs(fm_plan plan, int32_t on);
/* Per-frame peak records for the cross-GPU gather: rec[f] = {cells[f][0..k), count[f], status[f]}
 * (int32, row stride k + 2), one kernel on `stream`; device pointers. */
fm_status fm_pack_peak_records(const int32_t* cells, const int32_t* count, const int32_t* status, int64_t frames,
                               int64_t k, int32_t* rec, void* stream);
/* Number of kernel launches one fm_run_batch enqueues (per sub-batch). */
int32_t fm_plan_launches_per_batch(fm_plan plan);

/* End-to-end, host buffers (the reference-facing call): H2D of x and of the per-frame draws
 * (generated here from draw_seeds[f], exactly as the reference draws them), pipeline, fast2
 * redraws (<= 4 attempts, R/src/estimators.cpp:114-137), D2H of peaks/spectrum/status.
 * Host outputs may be NULL except peak_cells/peak_count/status. Synchronous. */
typedef struct fm_host_out {
    float* spectrum;         /* frames x L or NULL */
    int32_t* peak_cells;     /* frames x K */
    double* peak_heights;    /* frames x K or NULL */
    double* baseline;        /* frames or NULL */
    int32_t* peak_count;     /* frames */
    int32_t* status;         /* frames */
    int32_t* attempts;       /* frames (fast2 draws used) or NULL */
} fm_host_out;
fm_status fm_estimate_batch_host(fm_plan plan, int64_t frames, const float* h_x, const uint64_t* draw_seeds,
                                 fm_host_out* out, void* stream);

/* Batched temporal covariance (temporal_covariance R/src/scene.cpp:140-153,161-163), DEVICE
 * pointers: x frames x M x N complex64 row-major -> t_out frames x N x N complex64 row-major, T = X^H X / M (the
 * tensor-core covariance kernel reading X in its stored order; same precision contract as fm_run_batch's R).
 * status: frames FM_FRAME_* bits (RANGE / NONFINITE), zeroed by the call. work: device scratch used only for odd N
 * (frames x M x (N + 1) complex64), or NULL for a stream-ordered allocation. Asynchronous on `stream`. */
fm_status fm_temporal_covariance_batch(const float* x, int64_t frames, int64_t m, int64_t n, float* t_out,
                                       int32_t* status, float* work, void* stream);

/* ------------------------------------------------------------------ frame I/O (host)
 * FMCX binary matrix, R/include/fastmusic/io.hpp:17-21 / R/src/io.cpp:66-109: little-endian "FMCX",
 * u32 version 1, u32 rows, u32 cols, rows*cols complex64 row-major — one M x N file is one frame of
 * fm_batch_io.x. Errors: FM_EIO for open failure / bad magic / unsupported version / truncated payload
 * (the reference's std::runtime_error), FM_EINVAL for non-finite entries on write (ensure_finite) or a
 * dimension mismatch on read. */
/* write_matrix_binary from a row-major complex64 matrix */
fm_status fm_fmcx_write(const char* path, int64_t rows, int64_t cols, const float* a);
fm_status fm_fmcx_read_header(const char* path, int64_t* rows, int64_t* cols);
/* read_matrix_binary into row-major complex64; rows/cols must match the header */
fm_status fm_fmcx_read(const char* path, int64_t rows, int64_t cols, float* a);
/* the same two on a column-major complex128 CxMat (R/src/io.cpp:71-109 exactly) */
fm_status fm_z_fmcx_write(const char* path, int64_t rows, int64_t cols, const double* a);
fm_status fm_z_fmcx_read(const char* path, int64_t rows, int64_t cols, double* a);
/* Batch ingest: frame f of x (frames x m x n complex64, e.g. the pinned buffer handed to
 * fm_estimate_batch_host) from / to paths[f]; threaded over frames (threads <= 0: all cores). */
fm_status fm_fmcx_read_frames(const char* const* paths, int64_t frames, int64_t m, int64_t n, float* x,
                              int32_t threads);
fm_status fm_fmcx_write_frames(const char* const* paths, int64_t frames, int64_t m, int64_t n, const float* x,
                               int32_t threads);
/* write_matrix_csv, R/src/io.cpp:111-122 (column-major complex128) */
fm_status fm_z_write_matrix_csv(const char* path, int64_t rows, int64_t cols, const double* a);
/* write_spectrum_csv, R/src/io.cpp:124-131 on theta_l = theta0 + ((theta1-theta0)*l)/(L-1) */
fm_status fm_write_spectrum_csv(const char* path, int64_t grid_size, double theta0, double theta1,
                                const double* values);

/* ------------------------------------------------------------------ reference single-matrix API
 * complex128, column-major; computed on the GPU in fp64 (facade path of
 * include/fastmusic_b200/fastmusic.hpp). cost_seconds = CUDA-event time of the subspace
 * kernels (R/src/estimators.cpp:19-23 semantics). */
/* spatial_covariance, R/src/scene.cpp:157-159 (+ HermitianMatrix symmetrisation) */
fm_status fm_z_spatial_covariance(int64_t m, int64_t n, const double* y, double* s_out);
/* temporal_covariance, R/src/scene.cpp:140-153,161-163: T = Y^H Y / M (N x N), fp64 on the GPU */
fm_status fm_z_temporal_covariance(int64_t m, int64_t n, const double* y, double* t_out);
/* hermitian_eig, R/src/linalg.cpp:77-89: full spectral decomposition of the Hermitian S (column-major complex128,
 * symmetrised like HermitianMatrix), eigenvalues[m] descending (signed), eigenvectors m x m column-major complex128,
 * column i pairing with eigenvalue i. One-sided Jacobi on the GPU (the exact estimator's solver with K = M);
 * FM_ENOCONV at the sweep cap. */
fm_status fm_z_hermitian_eig(int64_t m, const double* s, double* eigenvalues, double* eigenvectors);
/* exact_signal_subspace, R/src/estimators.cpp:73-85 */
fm_status fm_z_exact_signal_subspace(int64_t m, const double* s, int64_t k, double* basis, double* eigenvalues,
                                     double* cost_seconds);
/* fast_music_1, R/src/estimators.cpp:87-102 */
fm_status fm_z_fast_music_1(int64_t m, const double* s, int64_t k, int64_t p, uint64_t seed, double* basis,
                            double* eigenvalues, double* cost_seconds);
/* fast_music_2, R/src/estimators.cpp:104-139; *deficient_column set on FM_ERANK */
fm_status fm_z_fast_music_2(int64_t m, const double* s, int64_t k, int64_t p, int32_t t, uint64_t seed,
                            double* basis, double* eigenvalues, double* cost_seconds, int64_t* deficient_column);
/* block_lanczos_subspace, R/src/estimators.cpp:154-222 (block Krylov, full reorthogonalisation, top-K Ritz
 * values stable to 1e-10 relative on two consecutive checks); fp64 on the GPU: the device Krylov loop of
 * lanczos_batch.cu for block <= 16 and bases up to 72 columns, else the host-driven loop (any M and block).
 * FM_ENOCONV at the iteration cap with the last relative change in *last_change (may be NULL). */
fm_status fm_z_block_lanczos_subspace(int64_t m, const double* s, int64_t k, int64_t block, int32_t max_iterations,
                                      double* basis, double* eigenvalues, double* cost_seconds, double* last_change);
/* Batched block_lanczos_subspace on DEVICE covariance matrices: s frames x M x M complex64
 * (row-major, Hermitian), the whole Krylov loop of R/src/estimators.cpp:154-222 in fp64 on the device, one CTA per
 * frame (lanczos_batch.cu). basis: frames x K x M complex128 (column-major per frame), eigenvalues frames x K,
 * status frames FM_FRAME_* (NOCONV: iteration cap, or more than 72 basis columns needed), iterations (may be NULL):
 * frames x (10000 * Krylov iterations + Jacobi sweeps). block <= 16. Asynchronous on `stream`. */
fm_status fm_block_lanczos_batch(const float* s, int64_t frames, int64_t m, int64_t k, int64_t block,
                                 int32_t max_iterations, double* basis, double* eigenvalues, int32_t* status,
                                 int32_t* iterations, void* stream);
/* music_spectrum, R/src/spectrum.cpp:50-68 on theta_l = theta0 + ((theta1-theta0)*l)/(L-1) */
fm_status fm_z_music_spectrum(int64_t m, int64_t kb, const double* basis, int64_t grid_size, double theta0,
                              double theta1, double d, double lambda, double* values);
/* extract_peaks, R/src/spectrum.cpp:182-188 (any L >= 1, K >= 1, any finite values); cells ascending */
fm_status fm_z_extract_peaks(const double* values, int64_t grid_size, int64_t k, int64_t min_sep, int64_t* cells,
                             double* heights, int64_t* count, double* baseline, int32_t* shortfall);

#ifdef __cplusplus
}
#endif

#endif /* FASTMUSIC_B200_H */
