// C ABI of the B200 Fast-MUSIC path (include/fastmusic_b200.h): plans, the batched
// device pipeline, the host-buffer end-to-end entry, the fp64 single-matrix entry points
// behind the reference-named C++ facade, host random draws and the synthetic frame
// generator. No CPU compute fallback: every numeric stage below launches a kernel.

#ifndef FM_COV_F16
#define FM_COV_F16 1  // multi-tile covariance from fp16 planes converted once per batch
#endif
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/fastmusic_b200.h"
#include "fm_common.cuh"
#include "host_rng.hpp"

// ------------------------------------------------------------------ kernel launchers (other TUs)
cudaError_t fm_launch_cov_tc(const float* d_x, float* d_r, int32_t* d_status, int64_t frames, int64_t m, int64_t n,
                             cudaStream_t stream, void* planes_hi = nullptr, void* planes_lo = nullptr,
                             float* scale = nullptr, int64_t n_true = 0, const FmCovRescue* rescue = nullptr,
                             int64_t t_rows = 0, void* xplanes = nullptr);
size_t fm_final_fallback_scratch_bytes(int ctas);
template <typename TS>
cudaError_t fm_launch_lanczos_batch(const void* S, const double* q0, double* basis_ws, double* w_ws, double* z_ws,
                                    double* out_basis, double* out_eig, int32_t* status, double* last_change,
                                    int32_t* iters, int frames, int m, int k, int b0, int max_iter, cudaStream_t s);
int fm_lanczos_batch_bmax();
int fm_lanczos_batch_nbmax();
std::vector<double> fm_lanczos_start_block(int64_t m, int b);
int fm_final_fallback_ctas();
cudaError_t fm_launch_final_fallback(const void* C, const void* V, const void* H, void* basis, double* eig,
                                     int32_t* status, void* scratch, int frames, int m, int p, int k,
                                     cudaStream_t s);
template <typename T>
cudaError_t fm_launch_rmul(const void*, const void*, const void*, void*, const int32_t*, int, int, int, bool,
                           cudaStream_t);
template <typename T>
cudaError_t fm_launch_gather(const void*, const int32_t*, void*, void*, const int32_t*, int, int, int, cudaStream_t);
template <typename T>
cudaError_t fm_launch_qr(const void*, void*, void*, void*, int32_t*, int32_t*, const int32_t*, int, int, int, bool,
                         cudaStream_t);
template <typename T>
cudaError_t fm_launch_nystrom(const void*, const void*, const void*, const void*, const void*, void*, double*,
                              int32_t*, const int32_t*, int, int, int, int, bool, cudaStream_t);
cudaError_t fm_launch_cholqr(const void* C, void* work, void* Vout, void* Rt, int32_t* status, const int32_t* fmap,
                             int frames, int m, int p, bool final_mode, const void* Vin, void* Hout, cudaStream_t s);
template <typename T>
cudaError_t fm_launch_nystrom_warp(const void* H, const void* work, const void* Rt, void* basis, double* eig,
                                   int32_t* status, int frames, int m, int p, int k, cudaStream_t s);
cudaError_t fm_launch_cholqr_warp(const void* C, void* work, void* Vout, void* Rt, void* Hout, const void* Vin,
                                  int32_t* status, int frames, int m, int p, bool final_mode, cudaStream_t s);
cudaError_t fm_launch_nystrom_warp2(const void* H, const void* work, const void* Rt, void* basis, double* eig,
                                    int32_t* status, int frames, int m, int p, int k, cudaStream_t s);
cudaError_t fm_launch_rmul_tc(const float* d_r, const float* d_omega, const float* d_v, float* d_c, int64_t frames,
                              int64_t m, int64_t p, cudaStream_t stream);
cudaError_t fm_launch_orth_split(const void* C, void* Vout, void* Lw, int32_t* permw, int32_t* status, int frames,
                                 int m, int p, cudaStream_t s, const void* gpart = nullptr);
cudaError_t fm_launch_rmul_planes(const void* planes_hi, const void* planes_lo, const float* d_scale,
                                  const float* d_omega, const float* d_v, float* d_c, int64_t frames, int64_t m,
                                  int64_t p, cudaStream_t stream, bool hi_only, int gram = 0, double* gpart = nullptr,
                                  double* hpart = nullptr);
cudaError_t fm_launch_final_split(const void* C, const void* V, void* Hw, void* Gw, void* Tw, void* basis, double* eig,
                                  int32_t* status, int frames, int m, int p, int k, cudaStream_t s,
                                  double* eig_next = nullptr, const void* gpart = nullptr,
                                  const void* hpart = nullptr);
cudaError_t fm_launch_autocorr(const void* basis, void* t, int frames, int m, int k, cudaStream_t s,
                               const int32_t* only = nullptr);
cudaError_t fm_launch_exact_residual(const void* R, const void* basis, double* cert, int frames, int m, int k,
                                     cudaStream_t s);
cudaError_t fm_launch_exact_check(const double* cert, const double* spec64, const int32_t* iter_status, int32_t* status,
                                  int frames, int m, int L, cudaStream_t s);
cudaError_t fm_launch_spectrum_one(const void* t, const void* zgrid, int frames, int m, int L, float* spec32,
                                   double* spec64, cudaStream_t s, const int32_t* only = nullptr);
size_t fm_peaks_workspace_bytes(int frames, int L, int K);
cudaError_t fm_launch_peaks_only(const double* values, int frames, int L, int K, int min_sep, int32_t* cells,
                                 double* heights, double* baseline, int32_t* count, void* gws, cudaStream_t s,
                                 const int32_t* only = nullptr);
cudaError_t fm_launch_orthocheck(const void* basis, int frames, int m, int k, double* dev, cudaStream_t s);
int fm_spectrum_tc_pairs_pad(int L, int half);
int fm_spectrum_tc_canon_off(int row, int k);
cudaError_t fm_launch_spectrum_tc(const void* t, const int8_t* zk, int8_t* tk, double* tscale, int frames, int m, int L,
                                  float* spec32, double* spec64, cudaStream_t s, int half);
cudaError_t fm_launch_spectrum_multi(const void* t, const void* zgrid, int frames, int m, int L, float* spec32,
                                     double* spec64, cudaStream_t s);
template <typename T>
cudaError_t fm_launch_jacobi_eig(const void* R, void* work, void* basis, double* eig, int32_t* status, int frames,
                                 int m, int k, cudaStream_t s, int only_flagged = 0, void* work32 = nullptr);

namespace {

constexpr double kPi = 3.14159265358979323846;
thread_local std::string g_err = "";

fm_status fail(fm_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

}  // namespace

// last-error setter shared with the host-only translation units (io.cpp)
fm_status fm_set_error(fm_status s, const std::string& msg) { return fail(s, msg); }

fm_status fm_fail_cuda(cudaError_t e, const char* expr, const char* file, int line) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e), cudaGetErrorString(e),
                  file, line, expr);
    g_err = buf;
    return e == cudaErrorInvalidValue ? FM_EINVAL : FM_ECUDA;
}

// ------------------------------------------------------------------ small kernels local to the ABI layer
namespace {

__global__ void k_clear_bits(int32_t* status, int frames, int32_t bits) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f < frames) status[f] &= ~bits;
}

// rec[f] = {cells[f][0..k), count[f], status[f]} (the gather record of shard.py), thread per record entry
__global__ void k_pack_records(const int32_t* __restrict__ cells, const int32_t* __restrict__ count,
                               const int32_t* __restrict__ status, int64_t frames, int k, int32_t* __restrict__ rec) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= frames * (k + 2)) return;
    const int64_t f = e / (k + 2);
    const int c = static_cast<int>(e % (k + 2));
    rec[e] = c < k ? cells[f * k + c] : (c == k ? count[f] : status[f]);
}

// Odd N: rows of X (N complex) -> rows of N + 1 complex with a zero last snapshot (the TMA row pitch of
// the covariance kernel must be a multiple of 16 bytes; a zero snapshot adds nothing to X X^H).
__global__ void k_pad_rows(const float2* __restrict__ x, float2* __restrict__ xp, int64_t rows, int n) {
    const int64_t row = blockIdx.x;
    if (row >= rows) return;
    const float2* src = x + row * n;
    float2* dst = xp + row * (n + 1);
    for (int j = threadIdx.x; j <= n; j += blockDim.x) dst[j] = j < n ? src[j] : make_float2(0.f, 0.f);
}

// FM_METHOD_FAST1_NORM2 column selection (extension: BASELINE config 3's "columns of R sampled with
// probability proportional to squared column norm"; not in the reference). One CTA per frame:
// w_j = sum_i |R_ij|^2 (R Hermitian: the row norms; from the fp16 hi/lo planes the common factor s_f^2 is
// dropped, which leaves the order of the keys unchanged), Efraimidis-Spirakis keys log(u_j) / w_j (the
// p largest, ties to the lower index, give a weighted sample without replacement), bitonic sort in shared
// memory, Omega = E_I (M x p row-major, I ascending) for the fast2 product kernel.
__global__ void k_norm2_select(const float* __restrict__ R, const __half* __restrict__ hi, const __half* __restrict__ lo,
                               const float* __restrict__ u, float* __restrict__ omega, int m, int p, int n2) {
    extern __shared__ uint8_t nsm[];
    double* key = reinterpret_cast<double*>(nsm);
    int* idx = reinterpret_cast<int*>(key + n2);
    const int f = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    // row norms: one warp per row, coalesced (the row is 2M reals: fp16 hi + lo planes, or fp32)
    for (int j = warp; j < m; j += nw) {
        const size_t row = (static_cast<size_t>(f) * m + j) * 2 * m;
        double w = 0.0;
        if (hi && (m & 3) == 0) {  // 16-byte rows: 8 halves per load from each plane
            const uint4* h4 = reinterpret_cast<const uint4*>(hi + row);
            const uint4* l4 = reinterpret_cast<const uint4*>(lo + row);
            for (int e = lane; e < m / 4; e += 32) {
                const uint4 a = h4[e], b = l4[e];
                const __half2* ha = reinterpret_cast<const __half2*>(&a);
                const __half2* hb = reinterpret_cast<const __half2*>(&b);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float2 x = __half22float2(ha[q]), y = __half22float2(hb[q]);
                    const double v0 = static_cast<double>(x.x) + static_cast<double>(y.x);
                    const double v1 = static_cast<double>(x.y) + static_cast<double>(y.y);
                    w += v0 * v0 + v1 * v1;
                }
            }
        } else if (hi) {
            for (int e = lane; e < 2 * m; e += 32) {
                const double v = static_cast<double>(__half2float(hi[row + e])) + static_cast<double>(__half2float(lo[row + e]));
                w += v * v;
            }
        } else {
            for (int e = lane; e < 2 * m; e += 32) {
                const double v = R[row + e];
                w += v * v;
            }
        }
        w = fmk::warp_sum(w);
        if (lane == 0) key[j] = w > 0.0 ? log(static_cast<double>(u[static_cast<size_t>(f) * m + j])) / w : -INFINITY;
    }
    for (int j = threadIdx.x; j < n2; j += blockDim.x) {
        if (j >= m) key[j] = -INFINITY;
        idx[j] = j < m ? j : 0x7fffffff;
    }
    __syncthreads();
    // bitonic sort: key descending, index ascending
    for (int k2 = 2; k2 <= n2; k2 <<= 1)
        for (int jj = k2 >> 1; jj > 0; jj >>= 1) {
            for (int i = threadIdx.x; i < n2; i += blockDim.x) {
                const int o = i ^ jj;
                if (o > i) {
                    const bool o_first = key[o] > key[i] || (key[o] == key[i] && idx[o] < idx[i]);
                    if (((i & k2) == 0) ? o_first : !o_first) {
                        const double tk = key[i];
                        key[i] = key[o];
                        key[o] = tk;
                        const int ti = idx[i];
                        idx[i] = idx[o];
                        idx[o] = ti;
                    }
                }
            }
            __syncthreads();
        }
    // the p selected indices ascending: rank of each among the first p
    float* om = omega + static_cast<size_t>(f) * m * p;
    for (int e = threadIdx.x; e < m * p; e += blockDim.x) om[e] = 0.f;
    __syncthreads();
    for (int a = threadIdx.x; a < p; a += blockDim.x) {
        int rank = 0;
        for (int b = 0; b < p; ++b) rank += idx[b] < idx[a] ? 1 : 0;
        om[static_cast<size_t>(idx[a]) * p + rank] = 1.f;
    }
}

// fp64 covariance for the single-matrix facade path (R/src/scene.cpp:138-159 +
// R/src/linalg.cpp:46-52): y column-major M x N; output S column-major, exactly Hermitian.
__global__ void k_cov_z(const fmk::c64* __restrict__ y, fmk::c64* __restrict__ s, int m, int n) {
    const int i = blockIdx.y * blockDim.y + threadIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m || j >= m || j > i) return;
    fmk::c64 acc = fmk::mk(0.0, 0.0);
    for (int q = 0; q < n; ++q) {
        const fmk::c64 a = y[static_cast<size_t>(q) * m + i], b = y[static_cast<size_t>(q) * m + j];
        acc.re += a.re * b.re + a.im * b.im;
        acc.im += a.im * b.re - a.re * b.im;
    }
    const double inv = 1.0 / static_cast<double>(n);
    acc.re *= inv;
    acc.im *= inv;
    if (i == j) acc.im = 0.0;
    s[static_cast<size_t>(j) * m + i] = acc;              // S(i, j)
    s[static_cast<size_t>(i) * m + j] = fmk::conj(acc);   // S(j, i)
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaError_t alloc(size_t count) {
        n = count;
        return count ? cudaMalloc(&p, sizeof(T) * count) : cudaSuccess;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

// Per-element phase step of grid point th: the ULA steering exp(j 2 pi d m sin(th) / lambda) exactly as
// R/src/scene.cpp:76, or (ToA path, `beat`) th is a beat phase w per sample (delay_shift = exp(j mu tau T_s),
// R/src/scene.cpp:91) and the steering of T = X^H X / M is conj(kappa^n) = exp(-j w n): T's range is spanned by
// the conjugated beat vectors.
inline double grid_step(double th, double d, double lambda, bool beat) {
    return beat ? -th : 2.0 * kPi * d * std::sin(th) / lambda;
}

std::vector<double> zgrid_host(int64_t L, double theta0, double theta1, double d, double lambda, bool beat) {
    // theta_l = theta0 + (span * l) / (L - 1)  (R/src/spectrum.cpp:26-28 for theta0 = 0, span = pi)
    std::vector<double> z(static_cast<size_t>(2 * L));
    const double span = theta1 - theta0;
    for (int64_t l = 0; l < L; ++l) {
        const double th = theta0 + (span * static_cast<double>(l)) / static_cast<double>(L - 1);
        const double step = grid_step(th, d, lambda, beat);
        z[2 * l] = std::cos(step);
        z[2 * l + 1] = std::sin(step);
    }
    return z;
}

// Digits of the cos / sin table for the tcgen05 spectrum (spectrum_tc.cu): for pair q < nq and delta < m,
// z = (cos, sin)(delta phi_q) (angle in fp64, glibc) as 5 signed base-128 digits of z / 2, in the zK layout
// [pair tile of 48][K block of 32][plane = s * 2 + cs][canonical 48 x 32 tile] (zero padding past nq and m).
std::vector<int8_t> zdig_host_k(int64_t L, double theta0, double theta1, double d, double lambda, int64_t m,
                                bool beat, bool half) {
    constexpr int kS = 5;
    const int64_t nq = half ? L : (L + 1) / 2, nqp = fm_spectrum_tc_pairs_pad(static_cast<int>(L), half ? 1 : 0),
                  mk = (m + 31) / 32 * 32;
    std::vector<int8_t> z(static_cast<size_t>(kS * 2 * nqp * mk), 0);
    const double span = theta1 - theta0;
    for (int64_t q = 0; q < nq; ++q) {
        const double th = theta0 + (span * static_cast<double>(q)) / static_cast<double>(L - 1);
        const double step = grid_step(th, d, lambda, beat);
        for (int64_t dl = 0; dl < m; ++dl) {
            const double ang = static_cast<double>(dl) * step;
            double r[2] = {0.5 * std::cos(ang), 0.5 * std::sin(ang)};
            for (int sl = 0; sl < kS; ++sl)
                for (int cs = 0; cs < 2; ++cs) {
                    const double x = 128.0 * r[cs];
                    const double dg = std::nearbyint(x);
                    r[cs] = x - dg;
                    const int64_t kb = dl / 32, plane = sl * 2 + cs;
                    z[static_cast<size_t>(((q / 48 * (mk / 32) + kb) * 10 + plane) * 48 * 32 +
                                          fm_spectrum_tc_canon_off(static_cast<int>(q % 48), static_cast<int>(dl % 32)))] =
                        static_cast<int8_t>(dg);
                }
        }
    }
    return z;
}

int hw_threads(int32_t req) {
    if (req > 0) return req;
    const unsigned h = std::thread::hardware_concurrency();
    return h ? static_cast<int>(h) : 1;
}

template <typename F>
void parallel_for(int64_t count, int threads, F&& fn) {
    threads = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(threads, count)));
    if (threads <= 1) {
        for (int64_t i = 0; i < count; ++i) fn(i);
        return;
    }
    std::atomic<int64_t> next{0};
    std::vector<std::thread> pool;
    for (int w = 0; w < threads; ++w)
        pool.emplace_back([&] {
            for (;;) {
                const int64_t i = next.fetch_add(1);
                if (i >= count) return;
                fn(i);
            }
        });
    for (auto& th : pool) th.join();
}

}  // namespace

// ------------------------------------------------------------------ misc
extern "C" int32_t fm_abi_version(void) { return 2; }

extern "C" const char* fm_status_string(fm_status s) {
    switch (s) {
        case FM_OK: return "ok";
        case FM_EINVAL: return "invalid argument";
        case FM_ERANK: return "rank deficiency";
        case FM_ENOCONV: return "no convergence";
        case FM_ESINGULAR: return "singular matrix";
        case FM_ECUDA: return "cuda error";
        case FM_ENOTSUP: return "not supported";
        case FM_EIO: return "i/o error";
    }
    return "unknown";
}

extern "C" const char* fm_last_error(void) { return g_err.c_str(); }

extern "C" fm_status fm_device_info(int32_t device, char* name, int32_t name_len, int32_t* sm_count) {
    cudaDeviceProp prop;
    FM_CUDA_OK(cudaGetDeviceProperties(&prop, device));
    if (name && name_len > 0) {
        std::strncpy(name, prop.name, static_cast<size_t>(name_len - 1));
        name[name_len - 1] = '\0';
    }
    if (sm_count) *sm_count = prop.multiProcessorCount;
    return FM_OK;
}

// ------------------------------------------------------------------ host random streams
extern "C" uint64_t fm_rng_derive(uint64_t seed, uint64_t tag) { return fmhost::Rng::derive(seed, tag); }

extern "C" fm_status fm_rng_normals(uint64_t seed, int64_t n, double* out) {
    if (n < 0 || (n > 0 && !out)) return fail(FM_EINVAL, "fm_rng_normals: bad arguments");
    fmhost::Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.normal();
    return FM_OK;
}

extern "C" fm_status fm_sample_without_replacement(uint64_t seed, int64_t m, int64_t p, int64_t* out) {
    if (p < 1 || p > m) return fail(FM_EINVAL, "sample_without_replacement: need 1 <= p <= m");
    fmhost::Rng r(seed);
    const auto v = r.sample_without_replacement(m, p);
    std::copy(v.begin(), v.end(), out);
    return FM_OK;
}

extern "C" fm_status fm_gaussian_matrix_real(int64_t m, int64_t p, uint64_t seed, double* out) {
    if (m < 1 || p < 1) return fail(FM_EINVAL, "gaussian_matrix: need M, p >= 1");
    fmhost::gaussian_matrix_real(m, p, seed, out);
    return FM_OK;
}

extern "C" fm_status fm_draw_omega_batch(int64_t frames, const uint64_t* seeds, int64_t m, int64_t p, float* omega) {
    if (frames < 0 || m < 1 || p < 1) return fail(FM_EINVAL, "fm_draw_omega_batch: bad arguments");
    parallel_for(frames, hw_threads(0), [&](int64_t f) {
        fmhost::gaussian_matrix_real(m, p, seeds[f], omega + static_cast<size_t>(f) * m * p);
    });
    return FM_OK;
}

extern "C" fm_status fm_draw_uniforms_batch(int64_t frames, const uint64_t* seeds, int64_t m, float* u) {
    if (frames < 0 || m < 1 || (frames > 0 && (!seeds || !u))) return fail(FM_EINVAL, "fm_draw_uniforms_batch: bad arguments");
    parallel_for(frames, hw_threads(0), [&](int64_t f) {
        fmhost::Rng r(seeds[f]);
        for (int64_t j = 0; j < m; ++j) u[static_cast<size_t>(f) * m + j] = static_cast<float>(r.uniform01());
    });
    return FM_OK;
}

extern "C" fm_status fm_draw_indices_batch(int64_t frames, const uint64_t* seeds, int64_t m, int64_t p,
                                           int32_t* indices) {
    if (frames < 0 || p < 1 || p > m) return fail(FM_EINVAL, "fm_draw_indices_batch: need 1 <= p <= m");
    parallel_for(frames, hw_threads(0), [&](int64_t f) {
        fmhost::Rng r(seeds[f]);
        const auto v = r.sample_without_replacement(m, p);
        for (int64_t i = 0; i < p; ++i) indices[static_cast<size_t>(f) * p + i] = static_cast<int32_t>(v[i]);
    });
    return FM_OK;
}

// ------------------------------------------------------------------ synthetic frames
// Model: angles/SNR from Rng(derive(s_f,1)); sources then noise from
// Rng(derive(s_f,2)); X = sum_k a_k s_k^T + noise in fp64, rounded to complex64.
extern "C" fm_status fm_generate_frames(const fm_scene_desc* sc, uint64_t base_seed, int64_t f0, int64_t frames,
                                        float* x, double* angles, double* snr_db, int32_t threads) {
    if (!sc || !x || sc->m < 1 || sc->n < 1 || sc->k < 1 || frames < 0)
        return fail(FM_EINVAL, "fm_generate_frames: bad arguments");
    const int64_t m = sc->m, n = sc->n, k = sc->k;
    std::atomic<int> bad{0};
    parallel_for(frames, hw_threads(threads), [&](int64_t fi) {
        const uint64_t s_f = fmhost::Rng::derive(base_seed, static_cast<uint64_t>(f0 + fi));
        std::vector<double> ang;
        fmhost::Rng ra(fmhost::Rng::derive(s_f, 1));
        if (sc->fixed_angles) {
            ang.assign(sc->fixed_angles, sc->fixed_angles + k);
        } else {
            int attempts = 0;
            while (static_cast<int64_t>(ang.size()) < k) {
                if (++attempts > 100000) {
                    bad = 1;
                    return;
                }
                const double th = sc->theta_lo + ra.uniform01() * (sc->theta_hi - sc->theta_lo);
                bool ok = true;
                for (double a : ang)
                    if (std::abs(th - a) < sc->min_sep) {
                        ok = false;
                        break;
                    }
                if (ok) ang.push_back(th);
            }
        }
        std::sort(ang.begin(), ang.end());
        const double snr = sc->snr_lo_db + (sc->snr_hi_db - sc->snr_lo_db) * ra.uniform01();
        const double sigma2 = static_cast<double>(k) / std::pow(10.0, snr / 10.0);
        fmhost::Rng rn(fmhost::Rng::derive(s_f, 2));
        const double inv_sqrt2 = 1.0 / std::sqrt(2.0);
        std::vector<double> src(static_cast<size_t>(2 * k * n));
        for (int64_t i = 0; i < k * n; ++i) {
            const double re = rn.normal();
            const double im = rn.normal();
            src[2 * i] = re * inv_sqrt2;
            src[2 * i + 1] = im * inv_sqrt2;
        }
        std::vector<double> st(static_cast<size_t>(2 * k * m));
        for (int64_t q = 0; q < k; ++q) {
            const double step = 2.0 * kPi * sc->d * std::sin(ang[q]) / sc->lambda;
            for (int64_t i = 0; i < m; ++i) {
                const double ph = step * static_cast<double>(i);
                st[2 * (q * m + i)] = std::cos(ph);
                st[2 * (q * m + i) + 1] = std::sin(ph);
            }
        }
        const double scale = std::sqrt(sigma2 / 2.0);
        float* xf = x + static_cast<size_t>(fi) * 2 * m * n;
        for (int64_t i = 0; i < m; ++i) {
            for (int64_t j = 0; j < n; ++j) {
                double ar_acc = 0.0, ai_acc = 0.0;
                for (int64_t q = 0; q < k; ++q) {
                    const double ar = st[2 * (q * m + i)], ai = st[2 * (q * m + i) + 1];
                    const double sr = src[2 * (q * n + j)], si = src[2 * (q * n + j) + 1];
                    ar_acc += ar * sr - ai * si;
                    ai_acc += ar * si + ai * sr;
                }
                const double nr = rn.normal();
                const double ni = rn.normal();
                ar_acc += scale * nr;
                ai_acc += scale * ni;
                xf[2 * (i * n + j)] = static_cast<float>(ar_acc);
                xf[2 * (i * n + j) + 1] = static_cast<float>(ai_acc);
            }
        }
        if (angles) std::copy(ang.begin(), ang.end(), angles + fi * k);
        if (snr_db) snr_db[fi] = snr;
    });
    if (bad) return fail(FM_EINVAL, "random_scene: cannot place targets at this separation");
    return FM_OK;
}

// ------------------------------------------------------------------ plan
struct fm_plan_s {
    fm_plan_desc d{};
    int device = 0;
    // workspace
    float* R = nullptr;       // frames x M x M complex64
    float* C = nullptr;       // frames x p x M complex64
    float* V = nullptr;       // frames x p x M complex64
    double* work = nullptr;   // frames x 2 x p x M complex128
    double* Rt = nullptr;     // frames x p x p complex128
    double* H = nullptr;      // frames x p x p complex128 (fast1)
    double* basis = nullptr;  // frames x K x M complex128
    double* eig = nullptr;    // frames x K
    double* t = nullptr;      // frames x M complex128
    double* spec64 = nullptr; // frames x L (fp64 spectrum for peak picking)
    double* zgrid = nullptr;  // L complex128
    uint8_t* peak_ws = nullptr;  // peak-picking workspace when a frame's does not fit in shared memory (long grids)
    int8_t* zk = nullptr;     // int8 digits of the grid's cos / sin table (zdig_host_k)
    bool zk_half = false;     // grid not mirror-symmetric: every point evaluated as its own pair
    int8_t* tdig = nullptr;   // per batch: int8 digits of t (frames padded per sub-batch)
    double* tscale = nullptr; // per batch: power-of-two scale of each frame's t
    size_t tdig_rows = 0;     // frame rows of tdig / tscale (sub-batch i uses rows f0 + 64 i ..)
    int32_t* scratch_status = nullptr;  // frames
    float* x_pad = nullptr;             // odd X row length: frames x rows x (row length + 1) complex64
    // ToA path (FM_PLAN_TEMPORAL): d describes the N-dimensional problem on T = X^H X / M (d.m = N, d.n = M);
    // X itself is xrows x xlen per frame (M x N). Spatial plans: xrows = d.m, xlen = d.n.
    bool temporal = false;
    int64_t xrows = 0, xlen = 0;
    // multi-tile spatial frames (M > 256): X as fp16 Re / Im planes, converted once per batch (cov_tc.cu kF16)
    uint16_t* xplanes = nullptr;
    int64_t xplane_len = 0;  // halves per plane row (X row length rounded up to 64)
    float* rscale = nullptr;            // frames: s_f of the fp16 hi/lo R planes (plane mode)
    // covariance rescue pass (cov_tc.cu): per-frame max |x|, out-of-range list, counts (one per sub-batch), prescale
    uint32_t* amax = nullptr;
    int32_t* rlist = nullptr;
    int32_t* rcount = nullptr;
    float* xscale = nullptr;
    void* fb_scratch = nullptr;         // final-step fallback (final_fallback.cu) work matrices
    size_t peak_ws_frame = 0;           // bytes of peak_ws per frame (0: frames fit in shared memory)
    bool last_planes = false;           // R of the last run is stored as planes (fm_rerun_frames)
    // exact method via certified subspace iteration (pe > 0): plan-owned Omega, R U product, gap
    int pe = 0;
    float* omega_e = nullptr;   // frames x M x pe fp32
    double* cert = nullptr;     // frames: sin-theta bound of the iteration's basis (exact.cu)
    float* work32 = nullptr;    // exact method: fp32 Jacobi stage, frames x MP x MP complex64
    double* gpart = nullptr;    // frames x 2 x p x p complex: G halves from the product epilogue (plane path)
    double* hpart = nullptr;    // frames x 2 x p x p complex: H = V^H C halves (last product)
    // block-Lanczos (FM_METHOD_LANCZOS, lanczos_batch.cu): shared start block, per-frame Krylov basis and blocks
    double* lz_q0 = nullptr;     // M x block complex128
    double* lz_basis = nullptr;  // frames x nbmax x M complex128
    double* lz_w = nullptr;      // frames x M x bmax complex128
    double* lz_z = nullptr;      // frames x M x bmax complex128
    int lz_block = 0;
    // host-path staging
    float* x_dev = nullptr;
    float* omega_dev = nullptr;
    int32_t* idx_dev = nullptr;
    float* spec_dev = nullptr;
    int32_t* cells_dev = nullptr;
    double* heights_dev = nullptr;
    double* base_dev = nullptr;
    int32_t* count_dev = nullptr;
    int32_t* status_dev = nullptr;
    float* omega_pinned = nullptr;
    int32_t* status_pinned = nullptr;
    // host path: chunked H2D on a plan-owned copy stream; [0..kHostChunks) chunk-ready, [kHostChunks] fork
    static constexpr int kHostChunks = 8;
    cudaStream_t copy_s = nullptr;
    cudaEvent_t copy_ev[kHostChunks + 1] = {};
    size_t bytes = 0;
    // optional per-stage CUDA events (covariance | subspace | autocorr | spectrum+peaks),
    // one set of 5 per recorded batch (ring of kMaxProf batches), summed by fm_plan_stage_times
    static constexpr int kMaxProf = 4096;
    bool profiling = false;
    std::vector<cudaEvent_t> ev;
    int prof_runs = 0;
    int cur = 0;
    // concurrent sub-batches: plan-owned streams forked from / joined into the caller's stream
    int nsub = 0;  // 0 = automatic
    std::vector<cudaStream_t> sub;
    std::vector<cudaEvent_t> sub_ev;  // [0] fork, [1..] joins
    std::vector<void*> allocs;
    // CUDA-graph replay of whole batches (fm_plan_set_graphs): one graph per (frames, io) seen, replayed with a
    // single launch -- the enqueue cost of a small batch (~40 launches) would otherwise exceed its GPU time
    struct GraphEntry {
        int64_t frames;
        fm_batch_io io;
        cudaGraphExec_t exec;
    };
    bool use_graphs = false;
    std::vector<GraphEntry> graphs;

    template <typename T>
    cudaError_t get(T** p, size_t count) {
        if (count == 0) {
            *p = nullptr;
            return cudaSuccess;
        }
        void* q = nullptr;
        cudaError_t e = cudaMalloc(&q, sizeof(T) * count);
        if (e != cudaSuccess) return e;
        allocs.push_back(q);
        bytes += sizeof(T) * count;
        *p = static_cast<T*>(q);
        return cudaSuccess;
    }
    ~fm_plan_s() {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        for (void* q : allocs) cudaFree(q);
        for (cudaEvent_t e : ev)
            if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : sub_ev)
            if (e) cudaEventDestroy(e);
        for (cudaStream_t q : sub)
            if (q) cudaStreamDestroy(q);
        for (cudaEvent_t e : copy_ev)
            if (e) cudaEventDestroy(e);
        for (auto& g : graphs)
            if (g.exec) cudaGraphExecDestroy(g.exec);
        if (copy_s) cudaStreamDestroy(copy_s);
        if (omega_pinned) cudaFreeHost(omega_pinned);
        if (status_pinned) cudaFreeHost(status_pinned);
        cudaSetDevice(prev);
    }
};

// Exact method via certified subspace iteration: p_e = 2K rounded up to a multiple of 4 (>= K + 4),
// t = kExactIters power steps, Omega from kExactSeed; needs the tensor-core / tiled paths (even M,
// p_e <= 32, p_e <= M). Otherwise (or with the FM_PLAN_EXACT_JACOBI flag) every frame runs the Jacobi solver.
constexpr uint64_t kExactSeed = 0x4558414354ull;
constexpr int kExactIters = 3;
static int exact_fast_p(const fm_plan_desc& d) {
    if (d.method != FM_METHOD_EXACT || (d.flags & FM_PLAN_EXACT_JACOBI)) return 0;
    const int pe = std::max<int>(static_cast<int>((2 * d.k + 3) / 4 * 4), static_cast<int>((d.k + 4 + 3) / 4 * 4));
    if (pe > 32 || pe > d.m || (d.m % 2) || (d.k % 4)) return 0;
    return pe;
}

static fm_status validate_desc(const fm_plan_desc* d) {
    if (!d) return fail(FM_EINVAL, "fm_plan_create: null descriptor");
    if (d->m < 2) return fail(FM_EINVAL, "plan: need M >= 2");
    if (d->n < 1) return fail(FM_EINVAL, "plan: need N >= 1");
    const char* who = d->method == FM_METHOD_FAST2         ? "fast_music_2"
                      : d->method == FM_METHOD_FAST1       ? "fast_music_1"
                      : d->method == FM_METHOD_FAST1_NORM2 ? "fast_music_1_norm2"
                      : d->method == FM_METHOD_LANCZOS     ? "block_lanczos_subspace"
                                                           : "exact_signal_subspace";
    if (d->k < 1 || d->k >= d->m) return fail(FM_EINVAL, std::string(who) + ": need 1 <= K < M");
    if (d->k > 64) return fail(FM_ENOTSUP, "plan: K <= 64 supported");
    if (d->method == FM_METHOD_FAST1 || d->method == FM_METHOD_FAST2 || d->method == FM_METHOD_FAST1_NORM2) {
        if (d->p < d->k || d->p > d->m) return fail(FM_EINVAL, std::string(who) + ": need K <= p <= M");
        if (d->p > 64) return fail(FM_ENOTSUP, "plan: p <= 64 supported");
    } else if (d->method == FM_METHOD_LANCZOS) {  // p = block (0 selects K, R/include/fastmusic/bench.hpp:61)
        const int64_t block = d->p > 0 ? d->p : d->k;
        if (block < d->k) return fail(FM_EINVAL, "block_lanczos_subspace: need block >= K");
        if (d->t < 1) return fail(FM_EINVAL, "block_lanczos_subspace: iters >= 1");
        if (std::min<int64_t>(block, d->m) > fm_lanczos_batch_bmax())
            return fail(FM_ENOTSUP, "plan: block_lanczos_subspace block <= 16 supported");
    } else if (d->method != FM_METHOD_EXACT) {
        return fail(FM_EINVAL, "plan: unknown method");
    }
    if (d->method == FM_METHOD_FAST2 && (d->t < 1 || d->t > 20))
        return fail(FM_EINVAL, "fast_music_2: need 1 <= t <= 20");
    if (d->grid_size < 2) return fail(FM_EINVAL, "AngleGrid: L >= 2 required");
    if (d->d <= 0.0 || d->lambda <= 0.0) return fail(FM_EINVAL, "steering_vector: need M >= 1, d > 0, lambda > 0");
    if (d->min_sep_cells < 0) return fail(FM_EINVAL, "plan: min_sep_cells >= 0");
    if (d->max_frames < 1) return fail(FM_EINVAL, "plan: max_frames >= 1");
    if (d->m > 4096) return fail(FM_ENOTSUP, "plan: M <= 4096 supported");
    return FM_OK;
}

extern "C" fm_status fm_plan_create(const fm_plan_desc* desc, int32_t device, fm_plan* out) {
    if (!out) return fail(FM_EINVAL, "fm_plan_create: null out");
    *out = nullptr;
    if (!desc) return fail(FM_EINVAL, "fm_plan_create: null descriptor");
    fm_plan_desc vd = *desc;  // ToA path: validated as the N-dimensional problem on T (K < N, p <= N)
    if (desc->flags & FM_PLAN_TEMPORAL) std::swap(vd.m, vd.n);
    fm_status st = validate_desc(&vd);
    if (st != FM_OK) return st;
    FM_CUDA_OK(cudaSetDevice(device));
    auto* pl = new fm_plan_s();
    pl->d = *desc;
    pl->device = device;
    pl->temporal = (desc->flags & FM_PLAN_TEMPORAL) != 0;
    pl->xrows = desc->m;
    pl->xlen = desc->n;
    if (pl->temporal) {  // the pipeline runs on T = X^H X / M: dimension N, M "snapshots" (validated below)
        pl->d.m = desc->n;
        pl->d.n = desc->m;
    }
    desc = &pl->d;  // everything below sizes the N-dimensional problem in temporal mode
    const size_t B = static_cast<size_t>(desc->max_frames), M = desc->m, K = desc->k, L = desc->grid_size;
    pl->pe = exact_fast_p(*desc);
    const size_t P = desc->method == FM_METHOD_EXACT     ? static_cast<size_t>(pl->pe)
                     : desc->method == FM_METHOD_LANCZOS ? static_cast<size_t>(1)
                                                         : static_cast<size_t>(desc->p);
    cudaError_t e = cudaSuccess;
    auto chk = [&](cudaError_t x) {
        if (e == cudaSuccess) e = x;
    };
    chk(pl->get(&pl->R, B * M * M * 2));
    chk(pl->get(&pl->C, B * P * M * 2));
    chk(pl->get(&pl->V, B * P * M * 2));
    const size_t MP = (M + 15) / 16 * 16;  // Jacobi pads columns to blocks of 16
    const size_t work_elems = desc->method == FM_METHOD_EXACT ? B * MP * MP * 2 : B * 2 * P * M * 2;
    chk(pl->get(&pl->work, work_elems));
    chk(pl->get(&pl->Rt, B * P * P * 2));
    chk(pl->get(&pl->H, B * P * P * 2));
    chk(pl->get(&pl->basis, B * K * M * 2));
    chk(pl->get(&pl->eig, B * K));
    chk(pl->get(&pl->t, B * M * 2));
    chk(pl->get(&pl->spec64, B * L));
    chk(pl->get(&pl->zgrid, L * 2));
    chk(pl->get(&pl->scratch_status, B));
    chk(pl->get(&pl->rscale, B));
    chk(pl->get(&pl->amax, B));
    chk(pl->get(&pl->rlist, B));
    chk(pl->get(&pl->rcount, 64));
    chk(pl->get(&pl->xscale, B));
    if (desc->method == FM_METHOD_LANCZOS) {
        pl->lz_block = static_cast<int>(std::min<int64_t>(desc->p > 0 ? desc->p : desc->k, desc->m));
        chk(pl->get(&pl->lz_q0, M * pl->lz_block * 2));
        chk(pl->get(&pl->lz_basis, B * static_cast<size_t>(fm_lanczos_batch_nbmax()) * M * 2));
        chk(pl->get(&pl->lz_w, B * M * static_cast<size_t>(fm_lanczos_batch_bmax()) * 2));
        chk(pl->get(&pl->lz_z, B * M * static_cast<size_t>(fm_lanczos_batch_bmax()) * 2));
        if (e == cudaSuccess) {
            const auto q0 = fm_lanczos_start_block(static_cast<int64_t>(M), pl->lz_block);
            e = cudaMemcpy(pl->lz_q0, q0.data(), sizeof(double) * q0.size(), cudaMemcpyHostToDevice);
        }
    } else if (desc->method != FM_METHOD_EXACT) {
        uint8_t* fb = nullptr;
        chk(pl->get(&fb, fm_final_fallback_scratch_bytes(fm_final_fallback_ctas())));
        pl->fb_scratch = fb;
    }
    if (pl->xlen & 1) chk(pl->get(&pl->x_pad, B * static_cast<size_t>(pl->xrows) * (static_cast<size_t>(pl->xlen) + 1) * 2));
    if (FM_COV_F16 && !pl->temporal && desc->m > 256 && desc->m % 2 == 0) {
        pl->xplane_len = ((pl->xlen + (pl->xlen & 1)) + 63) / 64 * 64;
        chk(pl->get(&pl->xplanes, B * static_cast<size_t>(pl->xrows) * pl->xplane_len * 2));
    }
    if (desc->method == FM_METHOD_FAST1_NORM2) chk(pl->get(&pl->omega_e, B * M * P));  // selection Omega = E_I
    if ((desc->method == FM_METHOD_FAST2 || desc->method == FM_METHOD_FAST1_NORM2) && M <= 256 && P <= 16) {
        chk(pl->get(&pl->gpart, B * 2 * P * P * 2));  // Gram halves from the product epilogue (plane path)
        chk(pl->get(&pl->hpart, B * 2 * P * P * 2));
    }
    if (pl->pe > 0) {
        chk(pl->get(&pl->omega_e, B * M * pl->pe));
        chk(pl->get(&pl->cert, B));
    }
    if (e == cudaSuccess) e = cudaMemset(pl->amax, 0, sizeof(uint32_t) * B);
    if (e != cudaSuccess) {
        delete pl;
        return fm_fail_cuda(e, "fm_plan_create workspace", __FILE__, __LINE__);
    }
    if (desc->method == FM_METHOD_EXACT && e == cudaSuccess) {
        const size_t mp = (M + 15) / 16 * 16;
        e = pl->get(&pl->work32, B * mp * mp * 2);
        if (e != cudaSuccess) {
            delete pl;
            return fm_fail_cuda(e, "fm_plan_create jacobi workspace", __FILE__, __LINE__);
        }
    }
    if (pl->pe > 0) {  // fixed Gaussian start blocks, one per frame slot
        std::vector<float> om(B * M * pl->pe);
        for (size_t f = 0; f < B; ++f)
            fmhost::gaussian_matrix_real(static_cast<int64_t>(M), pl->pe,
                                         fmhost::Rng::derive(kExactSeed, static_cast<uint64_t>(f)),
                                         om.data() + f * M * pl->pe);
        e = cudaMemcpy(pl->omega_e, om.data(), sizeof(float) * om.size(), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            delete pl;
            return fm_fail_cuda(e, "fm_plan_create exact omega", __FILE__, __LINE__);
        }
    }
    const auto z = zgrid_host(desc->grid_size, desc->theta0, desc->theta1, desc->d, desc->lambda, pl->temporal);
    e = cudaMemcpy(pl->zgrid, z.data(), sizeof(double) * z.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        delete pl;
        return fm_fail_cuda(e, "fm_plan_create zgrid", __FILE__, __LINE__);
    }
    {  // the tensor-core spectrum for every grid: mirror pairs when symmetric, single points otherwise
        pl->zk_half = !(desc->theta0 == -desc->theta1);
        const size_t mk = (static_cast<size_t>(desc->m) + 31) / 32 * 32;
        const auto zkh = zdig_host_k(desc->grid_size, desc->theta0, desc->theta1, desc->d, desc->lambda, desc->m,
                                     pl->temporal, pl->zk_half);
        e = pl->get(&pl->zk, zkh.size());
        if (e == cudaSuccess) e = cudaMemcpy(pl->zk, zkh.data(), zkh.size(), cudaMemcpyHostToDevice);
        pl->tdig_rows = B + 128 * 16;
        if (e == cudaSuccess) e = pl->get(&pl->tdig, pl->tdig_rows * 5 * 2 * mk);
        if (e == cudaSuccess) e = pl->get(&pl->tscale, pl->tdig_rows);
        if (e != cudaSuccess) {
            delete pl;
            return fm_fail_cuda(e, "fm_plan_create spectrum digits", __FILE__, __LINE__);
        }
    }
    if (const size_t pws = fm_peaks_workspace_bytes(static_cast<int>(B), static_cast<int>(L), static_cast<int>(K))) {
        pl->peak_ws_frame = pws / B;
        e = pl->get(&pl->peak_ws, pws);
        if (e != cudaSuccess) {
            delete pl;
            return fm_fail_cuda(e, "fm_plan_create peak workspace", __FILE__, __LINE__);
        }
    }
    *out = pl;
    return FM_OK;
}

extern "C" fm_status fm_plan_destroy(fm_plan plan) {
    delete plan;
    return FM_OK;
}

extern "C" fm_status fm_plan_workspace_bytes(fm_plan plan, int64_t* bytes) {
    if (!plan || !bytes) return fail(FM_EINVAL, "fm_plan_workspace_bytes: null");
    *bytes = static_cast<int64_t>(plan->bytes);
    return FM_OK;
}

extern "C" fm_status fm_plan_set_profiling(fm_plan plan, int32_t on) {
    if (!plan) return fail(FM_EINVAL, "fm_plan_set_profiling: null plan");
    FM_CUDA_OK(cudaSetDevice(plan->device));
    plan->profiling = on != 0;
    plan->prof_runs = 0;
    return FM_OK;
}

// Sum over the batches recorded since profiling was (re)enabled; *runs gets their count.
extern "C" fm_status fm_plan_stage_times(fm_plan plan, float* ms, int32_t* runs) {
    if (!plan || !ms) return fail(FM_EINVAL, "fm_plan_stage_times: null argument");
    const int n = std::min(plan->prof_runs, fm_plan_s::kMaxProf);
    for (int i = 0; i < 4; ++i) ms[i] = 0.f;
    for (int r = 0; r < n; ++r)
        for (int i = 0; i < 4; ++i) {
            float t = 0.f;
            FM_CUDA_OK(cudaEventElapsedTime(&t, plan->ev[static_cast<size_t>(r) * 5 + i],
                                            plan->ev[static_cast<size_t>(r) * 5 + i + 1]));
            ms[i] += t;
        }
    if (runs) *runs = n;
    plan->prof_runs = 0;
    return FM_OK;
}

// Tensor-core products (rmul_tc.cu) need an even M (16-byte TMA row pitch) and p <= 32 (p % 4 == 0);
// other shapes use the SIMT k_rmul.
static bool tc_rmul(int m, int p) { return (m % 2) == 0 && p >= 4 && p <= 32 && (p % 4) == 0; }

// R as fp16 hi/lo planes of R / s_f (cov_tc.cu kEpi = 2 -> rmul_planes_kernel): M <= 256 (one tile per
// frame), tensor-core products. fast2 / fast1_norm2 only: the exact method's Jacobi fallback and fast1's gather
// read complex64 R.
static bool plane_mode(const fm_plan_s* pl) {
    return (pl->d.method == FM_METHOD_FAST2 || pl->d.method == FM_METHOD_FAST1_NORM2) && pl->d.m <= 256 &&
           tc_rmul(static_cast<int>(pl->d.m), static_cast<int>(pl->d.p));
}
struct Planes {  // per-sub-batch view; hi == nullptr: complex64 R
    void* hi = nullptr;
    void* lo = nullptr;
    float* scale = nullptr;
};
static Planes planes_view(fm_plan pl, int64_t f0) {
    Planes v;
    const size_t plane = static_cast<size_t>(pl->d.max_frames) * pl->d.m * 2 * pl->d.m;  // halves per plane
    __half* base = reinterpret_cast<__half*>(pl->R);
    v.hi = base + static_cast<size_t>(f0) * pl->d.m * 2 * pl->d.m;
    v.lo = base + plane + static_cast<size_t>(f0) * pl->d.m * 2 * pl->d.m;
    v.scale = pl->rscale + f0;
    return v;
}

// Gram epilogue (plane path, p <= 16): the products also form G = C^H C (and H = V^H C on the last one), so the
// orthonormalisation / final stage skip their Gram kernels.
static bool gram_epilogue(const fm_plan_s* pl) {
    return plane_mode(pl) && pl->d.p <= 16 && (pl->d.p % 4) == 0 && pl->gpart != nullptr;
}

extern "C" int32_t fm_plan_launches_per_batch(fm_plan plan) {
    if (!plan) return 0;
    const auto& d = plan->d;
    const int t = d.t;
    // covariance + rescue list + rescue covariance + autocorr + spectrum + peaks (+ odd-N pad)
    int n = 1 + 2 + 3 + (plan->x_pad ? 1 : 0);
    if (plan->zk) n += 1;  // int8 spectrum: + the digit split of t (k_slice_tk)
    const bool tiled = d.p <= 32 && (d.p % 4) == 0;
    const int gepi = gram_epilogue(plan) ? 1 : 0;
    const int fin = (tiled ? 3 - gepi : 2) + 1;  // gram, small-warp, (fallback), basis | cholqr, nystrom, (fallback)
    const int orth = tiled ? 3 - gepi : 1;      // gram, pivoted chol, rows solve | cholqr
    if (d.method == FM_METHOD_FAST2) n += 1 + t * (orth + 1) + fin;  // rmul, t x (orth, rmul), final
    else if (d.method == FM_METHOD_FAST1_NORM2) n += 1 + 1 + (orth + 1) + fin;  // select, rmul, orth, rmul, final
    else if (d.method == FM_METHOD_FAST1) n += 1 + fin;      // gather, final
    else if (d.method == FM_METHOD_LANCZOS) n += 1;          // the whole Krylov loop in one launch
    else if (plan->pe > 0) n += 1 + 1 + kExactIters * (3 + 1) + 3 + 1 + 6;  // see run_post_cov
    else n += 1;                                              // jacobi
    return n;
}

// FM_DEBUG_SYNC=1: synchronise after every launch so a fault is attributed to its kernel.
static bool debug_sync() {
    static const bool on = [] {
        const char* e = std::getenv("FM_DEBUG_SYNC");
        return e && e[0] == '1';
    }();
    return on;
}
#define FM_LAUNCH(expr)                                                  \
    do {                                                                 \
        FM_CUDA_OK(expr);                                                \
        if (debug_sync()) FM_CUDA_OK(cudaStreamSynchronize(s));          \
    } while (0)

static void mark(fm_plan pl, int i, cudaStream_t s) {
    if (!pl->profiling) return;
    if (i == 0) {
        pl->cur = pl->prof_runs % fm_plan_s::kMaxProf;
        const size_t need = static_cast<size_t>(pl->cur + 1) * 5;
        while (pl->ev.size() < need) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            pl->ev.push_back(e);
        }
        pl->prof_runs++;
    }
    cudaEventRecord(pl->ev[static_cast<size_t>(pl->cur) * 5 + i], s);
}

// Per-sub-batch view of the plan workspace (pointers offset to the sub-batch's first frame).
struct WorkView {
    float* C;
    float* V;
    double* work;
    double* Rt;
    double* H;
    double* basis;
    double* eig;
    double* t;
    double* spec64;
    int32_t* scratch;
    float* omega_e;
    double* cert;
    float* work32;
    double* gpart;
    double* hpart;
    uint8_t* peak_ws;
    double* lz_basis;
    double* lz_w;
    double* lz_z;
    FmCovRescue resc;
    size_t dslot;  // first frame row of this sub-batch's region in tdig / tscale
};

static WorkView work_view(fm_plan pl, int64_t f0, int sub = 0) {
    const auto& d = pl->d;
    const size_t M = d.m, P = d.method == FM_METHOD_EXACT ? pl->pe : d.p, K = d.k;
    const size_t MP = (M + 15) / 16 * 16;
    const size_t wsz = d.method == FM_METHOD_EXACT ? MP * MP * 2 : 2 * P * M * 2;
    WorkView w;
    w.omega_e = pl->omega_e ? pl->omega_e + f0 * M * P : nullptr;
    w.cert = pl->cert ? pl->cert + f0 : nullptr;
    w.work32 = pl->work32 ? pl->work32 + f0 * ((M + 15) / 16 * 16) * ((M + 15) / 16 * 16) * 2 : nullptr;
    w.dslot = static_cast<size_t>(f0) + 128 * static_cast<size_t>(sub);
    w.gpart = pl->gpart ? pl->gpart + f0 * 2 * P * P * 2 : nullptr;
    w.hpart = pl->hpart ? pl->hpart + f0 * 2 * P * P * 2 : nullptr;
    w.C = pl->C + f0 * P * M * 2;
    w.V = pl->V + f0 * P * M * 2;
    w.work = pl->work + f0 * wsz;
    w.Rt = pl->Rt + f0 * P * P * 2;
    w.H = pl->H + f0 * P * P * 2;
    w.basis = pl->basis + f0 * K * M * 2;
    w.eig = pl->eig + f0 * K;
    w.t = pl->t + f0 * M * 2;
    w.spec64 = pl->spec64 + f0 * static_cast<size_t>(d.grid_size);
    w.scratch = pl->scratch_status + f0;
    w.peak_ws = pl->peak_ws ? pl->peak_ws + f0 * pl->peak_ws_frame : nullptr;
    const size_t nbm = static_cast<size_t>(fm_lanczos_batch_nbmax()), bm = static_cast<size_t>(fm_lanczos_batch_bmax());
    w.lz_basis = pl->lz_basis ? pl->lz_basis + f0 * nbm * M * 2 : nullptr;
    w.lz_w = pl->lz_w ? pl->lz_w + f0 * M * bm * 2 : nullptr;
    w.lz_z = pl->lz_z ? pl->lz_z + f0 * M * bm * 2 : nullptr;
    w.resc = FmCovRescue{pl->amax + f0, pl->rlist + f0, pl->rcount + std::min(sub, 63), pl->xscale + f0};
    return w;
}

static fm_batch_io io_view(fm_plan pl, const fm_batch_io* io, int64_t f0) {
    const auto& d = pl->d;
    const size_t M = d.m, N = d.n, P = d.p, K = d.k, L = d.grid_size;
    fm_batch_io o = *io;
    o.x = io->x + f0 * M * N * 2;
    if (io->omega) o.omega = io->omega + f0 * M * (d.method == FM_METHOD_FAST1_NORM2 ? 1 : P);
    if (io->indices) o.indices = io->indices + f0 * P;
    if (io->spectrum) o.spectrum = io->spectrum + f0 * L;
    o.peak_cells = io->peak_cells + f0 * K;
    o.peak_heights = io->peak_heights + f0 * K;
    o.baseline = io->baseline + f0;
    o.peak_count = io->peak_count + f0;
    o.status = io->status + f0;
    if (io->basis) o.basis = io->basis + f0 * K * M * 2;
    if (io->eigenvalues) o.eigenvalues = io->eigenvalues + f0 * K;
    if (io->covariance) o.covariance = io->covariance + f0 * M * M * 2;
    return o;
}

static fm_status run_post_cov(fm_plan pl, int64_t frames, const fm_batch_io* io, const float* R, cudaStream_t s,
                              const WorkView& w, bool prof, const Planes& pv, bool fresh = true) {
    const auto& d = pl->d;
    const int F = static_cast<int>(frames), M = static_cast<int>(d.m), P = static_cast<int>(d.p),
              K = static_cast<int>(d.k);
    double* basis = io->basis ? io->basis : w.basis;
    double* eig = io->eigenvalues ? io->eigenvalues : w.eig;
    if (!fresh) {  // a rerun keeps the batch's status words: drop the stage flags of the previous pass
        k_clear_bits<<<(F + 255) / 256, 256, 0, s>>>(io->status, F, FM_FRAME_RANK | FM_FRAME_NOCONV);
        FM_CUDA_OK(cudaGetLastError());
    }
    const bool warp_path = P <= 32;              // block-per-frame small-matrix kernels (smallmat.cu)
    const bool tiled = P <= 32 && (P % 4) == 0;  // register-tiled Gram + split final stage
    // Gram epilogue (plane path, p <= 16): the products also form G = C^H C (and H = V^H C on the last one),
    // so the orthonormalisation / final stage skip their Gram kernels.
    const bool gepi = pv.hi && w.gpart && P <= 16 && tiled;
    auto orth = [&](bool final_mode, const void* vin) -> fm_status {
        if (tiled && !final_mode) {
            FM_LAUNCH(fm_launch_orth_split(w.C, w.V, w.Rt, reinterpret_cast<int32_t*>(w.H), io->status, F, M, P, s,
                                           gepi ? w.gpart : nullptr));
            return FM_OK;
        }
        if (warp_path)
            FM_LAUNCH(fm_launch_cholqr_warp(w.C, w.work, final_mode ? nullptr : w.V, w.Rt, w.H, vin,
                                            final_mode ? w.scratch : io->status, F, M, P, final_mode, s));
        else
            FM_LAUNCH(fm_launch_cholqr(w.C, w.work, final_mode ? nullptr : w.V, final_mode ? w.Rt : nullptr,
                                       final_mode ? w.scratch : io->status, nullptr, F, M, P, final_mode,
                                       vin, w.H, s));
        return FM_OK;
    };
    auto nystrom = [&]() -> fm_status {
        if (warp_path)
            FM_LAUNCH(fm_launch_nystrom_warp2(w.H, w.work, w.Rt, basis, eig, io->status, F, M, P, K, s));
        else
            FM_LAUNCH(fm_launch_nystrom_warp<float>(w.H, w.work, w.Rt, basis, eig, io->status, F, M, P, K, s));
        return FM_OK;
    };
    // frames the fast Nystrom tail flagged (singular H, rank-deficient C, Jacobi cap): exact reference algebra
    // with a truncating pinv (final_fallback.cu); unflagged frames return at once.
    auto fallback = [&](const void* v, const void* h) -> fm_status {
        FM_LAUNCH(fm_launch_final_fallback(w.C, v, h, basis, eig, io->status, pl->fb_scratch, F, M, P, K, s));
        return FM_OK;
    };
    fm_status st = FM_OK;
    // C = R Omega (omega) or C = R V: fp16 planes -> rmul_planes_kernel, complex64 R -> tf32 kernel / SIMT.
    // Range-finder products (all but the last) read only the hi plane of R (R to 2^-12 s_f): they only shape
    // span(V); the last product, which feeds the Nystrom step, reads both planes. Measured over 1024 c2 frames
    // vs the fp64 oracle: worst spectrum error 0.00556 -> 0.00557 dB, no peak changes, step 1.191 -> 1.140 ms.
    auto rmul = [&](const float* omega, const float* v, float* c, int p, bool range_only = false,
                    int gram = 0) -> fm_status {
        if (pv.hi)
            FM_LAUNCH(fm_launch_rmul_planes(pv.hi, pv.lo, pv.scale, omega, v, c, F, M, p, s, range_only,
                                            gepi ? gram : 0, w.gpart, w.hpart));
        else if (tc_rmul(M, p))
            FM_LAUNCH(fm_launch_rmul_tc(R, omega, v, c, F, M, p, s));
        else
            FM_LAUNCH(fm_launch_rmul<float>(R, omega, v, c, nullptr, F, M, p, omega != nullptr, s));
        return FM_OK;
    };
    if (d.method == FM_METHOD_FAST2 || d.method == FM_METHOD_FAST1_NORM2) {
        const float* omega = io->omega;
        int tt = d.t;
        if (d.method == FM_METHOD_FAST1_NORM2) {  // Omega = E_I from the norm^2-weighted selection, one power step
            int n2 = 1;
            while (n2 < static_cast<int>(M)) n2 <<= 1;
            const int smem = n2 * static_cast<int>(sizeof(double) + sizeof(int));
            if (smem > 48 * 1024) FM_CUDA_OK(cudaFuncSetAttribute(k_norm2_select, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            k_norm2_select<<<F, 256, smem, s>>>(pv.hi ? nullptr : R, static_cast<const __half*>(pv.hi),
                                                static_cast<const __half*>(pv.lo), io->omega, w.omega_e, M, P, n2);
            FM_LAUNCH(cudaGetLastError());
            omega = w.omega_e;
            tt = 1;
        }
        // the first t products only shape the range (V); the last one feeds the Nystrom step
        if ((st = rmul(omega, nullptr, w.C, P, tt > 0, 1)) != FM_OK) return st;
        for (int it = 0; it < tt; ++it) {
            if ((st = orth(false, nullptr)) != FM_OK) return st;
            if ((st = rmul(nullptr, w.V, w.C, P, it + 1 < tt, it + 1 < tt ? 1 : 2)) != FM_OK) return st;
        }
        if (tiled) {
            FM_LAUNCH(fm_launch_final_split(w.C, w.V, w.H, w.Rt, w.work, basis, eig, io->status, F, M, P, K, s,
                                            nullptr, gepi ? w.gpart : nullptr, gepi ? w.hpart : nullptr));
        } else {
            if ((st = orth(true, w.V)) != FM_OK) return st;
            if ((st = nystrom()) != FM_OK) return st;
        }
        if ((st = fallback(w.V, nullptr)) != FM_OK) return st;
    } else if (d.method == FM_METHOD_FAST1) {
        FM_LAUNCH(fm_launch_gather<float>(R, io->indices, w.C, w.H, nullptr, F, M, P, s));
        if (tiled) {
            FM_LAUNCH(fm_launch_final_split(w.C, nullptr, w.H, w.Rt, w.work, basis, eig, io->status, F, M, P, K, s));
        } else {
            if ((st = orth(true, nullptr)) != FM_OK) return st;
            if ((st = nystrom()) != FM_OK) return st;
        }
        if ((st = fallback(nullptr, w.H)) != FM_OK) return st;
    } else if (d.method == FM_METHOD_LANCZOS) {
        FM_LAUNCH(fm_launch_lanczos_batch<float>(R, pl->lz_q0, w.lz_basis, w.lz_w, w.lz_z, basis, eig, io->status,
                                                 nullptr, nullptr, F, M, K, pl->lz_block, d.t, s));
    } else if (pl->pe > 0) {
        // exact_signal_subspace as certified subspace iteration: C = R Omega, kExactIters x {V = orth(C),
        // C = R V}, Nystrom/Rayleigh step -> U; then the fp64 residual bound (exact.cu) -- checked against the
        // spectrum after the peaks below; frames not certified rerun the Jacobi eigensolver.
        const int PE = pl->pe;
        k_clear_bits<<<(F + 255) / 256, 256, 0, s>>>(w.scratch, F, ~0);
        FM_CUDA_OK(cudaGetLastError());
        if ((st = rmul(w.omega_e, nullptr, w.C, PE)) != FM_OK) return st;
        for (int it = 0; it < kExactIters; ++it) {
            FM_LAUNCH(fm_launch_orth_split(w.C, w.V, w.Rt, reinterpret_cast<int32_t*>(w.H), w.scratch, F, M, PE, s));
            if ((st = rmul(nullptr, w.V, w.C, PE)) != FM_OK) return st;
        }
        FM_LAUNCH(fm_launch_final_split(w.C, w.V, w.H, w.Rt, w.work, basis, eig, w.scratch, F, M, PE, K, s));
        FM_LAUNCH(fm_launch_exact_residual(R, basis, w.cert, F, M, K, s));
    } else {
        FM_LAUNCH(fm_launch_jacobi_eig<float>(R, w.work, basis, eig, io->status, F, M, K, s, 0, w.work32));
    }
    if (prof) mark(pl, 2, s);
    FM_LAUNCH(fm_launch_autocorr(basis, w.t, F, M, K, s));
    if (prof) mark(pl, 3, s);
    // the spectrum on the INT8 tensor cores (tcgen05 kind::i8) with fp64-exact digit splitting (spectrum_tc.cu):
    // mirror-symmetric grids (theta0 = -theta1) as pairs (theta, -theta) sharing one evaluation, other grids point
    // by point; the fp64 power recurrence only when the digit workspace does not cover the batch
    const bool dig_fits = w.dslot + (static_cast<size_t>(F) + 127) / 128 * 128 <= pl->tdig_rows;
    if (pl->zk && dig_fits) {
        const size_t mk = (static_cast<size_t>(M) + 31) / 32 * 32;
        FM_LAUNCH(fm_launch_spectrum_tc(w.t, pl->zk, pl->tdig + w.dslot * 5 * 2 * mk, pl->tscale + w.dslot, F, M,
                                        static_cast<int>(d.grid_size), io->spectrum, w.spec64, s,
                                        pl->zk_half ? 1 : 0));
    } else {
        FM_LAUNCH(fm_launch_spectrum_multi(w.t, pl->zgrid, F, M, static_cast<int>(d.grid_size), io->spectrum, w.spec64,
                                           s));
    }
    FM_LAUNCH(fm_launch_peaks_only(w.spec64, F, static_cast<int>(d.grid_size), K, static_cast<int>(d.min_sep_cells),
                                   io->peak_cells, io->peak_heights, io->baseline, io->peak_count, w.peak_ws, s));
    if (pl->pe > 0) {
        // exact method: the certificate against this spectrum's deepest denominator; frames it does not cover (or
        // that the iteration flagged) are recomputed by the Jacobi eigensolver, then their spectrum and peaks
        FM_LAUNCH(fm_launch_exact_check(w.cert, w.spec64, w.scratch, io->status, F, M, static_cast<int>(d.grid_size), s));
        FM_LAUNCH(fm_launch_jacobi_eig<float>(R, w.work, basis, eig, io->status, F, M, K, s, 1, w.work32));
        FM_LAUNCH(fm_launch_autocorr(basis, w.t, F, M, K, s, io->status));
        FM_LAUNCH(fm_launch_spectrum_one(w.t, pl->zgrid, F, M, static_cast<int>(d.grid_size), io->spectrum, w.spec64, s,
                                         io->status));
        FM_LAUNCH(fm_launch_peaks_only(w.spec64, F, static_cast<int>(d.grid_size), K, static_cast<int>(d.min_sep_cells),
                                       io->peak_cells, io->peak_heights, io->baseline, io->peak_count, w.peak_ws, s,
                                       io->status));
        k_clear_bits<<<(F + 255) / 256, 256, 0, s>>>(io->status, F, fmk::kFrameRefine);
        FM_CUDA_OK(cudaGetLastError());
    }
    if (prof) mark(pl, 4, s);
    return FM_OK;
}

static fm_status check_io(fm_plan pl, int64_t frames, const fm_batch_io* io) {
    if (!pl || !io) return fail(FM_EINVAL, "fm_run_batch: null plan/io");
    if (frames < 1 || frames > pl->d.max_frames) return fail(FM_EINVAL, "fm_run_batch: frames outside [1, max_frames]");
    if (!io->x || !io->peak_cells || !io->peak_heights || !io->baseline || !io->peak_count || !io->status)
        return fail(FM_EINVAL, "fm_run_batch: x, peak outputs and status are required");
    if (pl->d.method == FM_METHOD_FAST2 && !io->omega) return fail(FM_EINVAL, "fm_run_batch: fast2 needs omega");
    if (pl->d.method == FM_METHOD_FAST1_NORM2 && !io->omega)
        return fail(FM_EINVAL, "fm_run_batch: fast1_norm2 needs the uniforms in io->omega");
    if (pl->d.method == FM_METHOD_FAST1 && !io->indices) return fail(FM_EINVAL, "fm_run_batch: fast1 needs indices");
    return FM_OK;
}

static int auto_subbatches(fm_plan pl, int64_t frames) {
    if (pl->nsub > 0) return static_cast<int>(std::min<int64_t>(std::min(pl->nsub, 16), frames));
    // Two concurrent sub-batches for large batches, except on the p <= 16 plane path (Gram halves in the products),
    // whose kernels no longer gain from the overlap: c2 1.036 / 1.043 ms for 1 / 2; c3 1.408 / 1.286, c5 0.964 /
    // 0.952, c3n 2.181 / 2.069.
    if (pl->gpart) return 1;
    return frames >= 512 ? 2 : 1;
}

// fm_run_batch on frames [ws0, ws0 + frames) of the plan workspace (the host path keeps every chunk's R in place
// so that fm_rerun_frames can redo any frame of the batch).
static fm_status run_batch_at(fm_plan pl, int64_t ws0, int64_t frames, const fm_batch_io* io, cudaStream_t s) {
    FM_CUDA_OK(cudaMemsetAsync(io->status, 0, sizeof(int32_t) * frames, s));
    const int nsub = auto_subbatches(pl, frames);
    const bool planes = plane_mode(pl) && !io->covariance;
    pl->last_planes = planes;
    const int64_t nx = pl->x_pad ? pl->xlen + 1 : pl->xlen;  // X row length fed to the covariance kernel
    const int64_t trows = pl->temporal ? pl->xrows : 0;     // temporal mode: contraction over X's rows
    auto xpl = [&](int64_t f0) -> void* {  // this frame range's region of the plane workspace (both planes)
        return pl->xplanes ? static_cast<void*>(pl->xplanes + f0 * pl->xrows * pl->xplane_len * 2) : nullptr;
    };
    const size_t MM2 = static_cast<size_t>(pl->d.m) * pl->d.m * 2;
    auto xin = [&](const float* x, int64_t f0, int64_t nf, cudaStream_t q) -> const float* {
        if (!pl->x_pad) return x;
        float* xp = pl->x_pad + f0 * pl->xrows * nx * 2;
        k_pad_rows<<<static_cast<unsigned>(nf * pl->xrows), 128, 0, q>>>(reinterpret_cast<const float2*>(x),
                                                                        reinterpret_cast<float2*>(xp), nf * pl->xrows,
                                                                        static_cast<int>(pl->xlen));
        return xp;
    };
    if (nsub <= 1) {
        float* R = io->covariance ? io->covariance : pl->R + ws0 * MM2;
        const Planes pv = planes ? planes_view(pl, ws0) : Planes{};
        const WorkView w = work_view(pl, ws0);
        mark(pl, 0, s);
        FM_LAUNCH(fm_launch_cov_tc(xin(io->x, ws0, frames, s), R, io->status, frames, pl->d.m, nx, s, pv.hi, pv.lo,
                                   pv.scale, pl->d.n, &w.resc, trows, xpl(ws0)));
        mark(pl, 1, s);
        return run_post_cov(pl, frames, io, R, s, w, true, pv);
    }
    while (static_cast<int>(pl->sub.size()) < nsub) {
        cudaStream_t q;
        FM_CUDA_OK(cudaStreamCreateWithFlags(&q, cudaStreamNonBlocking));
        pl->sub.push_back(q);
    }
    while (static_cast<int>(pl->sub_ev.size()) < nsub + 1) {
        cudaEvent_t e;
        FM_CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        pl->sub_ev.push_back(e);
    }
    FM_CUDA_OK(cudaEventRecord(pl->sub_ev[0], s));
    const int64_t chunk = (frames + nsub - 1) / nsub;
    for (int i = 0; i < nsub; ++i) {
        const int64_t f0 = i * chunk;
        const int64_t nf = std::min<int64_t>(chunk, frames - f0);
        if (nf <= 0) break;
        cudaStream_t q = pl->sub[i];
        FM_CUDA_OK(cudaStreamWaitEvent(q, pl->sub_ev[0], 0));
        const fm_batch_io o = io_view(pl, io, f0);
        float* R = io->covariance ? o.covariance : pl->R + (ws0 + f0) * MM2;
        const Planes pv = planes ? planes_view(pl, ws0 + f0) : Planes{};
        const WorkView w = work_view(pl, ws0 + f0, i);
        if (i == 0) mark(pl, 0, q);
        {
            cudaStream_t s = q;  // FM_LAUNCH synchronises `s` in debug mode
            FM_LAUNCH(fm_launch_cov_tc(xin(o.x, ws0 + f0, nf, q), R, o.status, nf, pl->d.m, nx, q, pv.hi, pv.lo,
                                       pv.scale, pl->d.n, &w.resc, trows, xpl(ws0 + f0)));
        }
        if (i == 0) mark(pl, 1, q);
        fm_status st = run_post_cov(pl, nf, &o, R, q, w, i == 0, pv);
        if (st != FM_OK) return st;
        FM_CUDA_OK(cudaEventRecord(pl->sub_ev[1 + i], q));
        FM_CUDA_OK(cudaStreamWaitEvent(s, pl->sub_ev[1 + i], 0));
    }
    return FM_OK;
}

extern "C" fm_status fm_run_batch(fm_plan pl, int64_t frames, const fm_batch_io* io, void* stream) {
    fm_status st = check_io(pl, frames, io);
    if (st != FM_OK) return st;
    FM_CUDA_OK(cudaSetDevice(pl->device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!pl->use_graphs || !s || pl->profiling || debug_sync()) return run_batch_at(pl, 0, frames, io, s);
    for (auto& g : pl->graphs)
        if (g.frames == frames && std::memcmp(&g.io, io, sizeof(fm_batch_io)) == 0) {
            FM_CUDA_OK(cudaGraphLaunch(g.exec, s));
            return FM_OK;
        }
    // first batch with these buffers: capture the whole enqueue sequence (sub-batch forks included) once
    FM_CUDA_OK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    st = run_batch_at(pl, 0, frames, io, s);
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(s, &graph);
    if (st != FM_OK) {
        if (graph) cudaGraphDestroy(graph);
        return st;
    }
    FM_CUDA_OK(ce);
    cudaGraphExec_t exec = nullptr;
    const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    FM_CUDA_OK(ie);
    pl->graphs.push_back({frames, *io, exec});
    FM_CUDA_OK(cudaGraphLaunch(exec, s));
    return FM_OK;
}

extern "C" fm_status fm_plan_set_graphs(fm_plan plan, int32_t on) {
    if (!plan) return fail(FM_EINVAL, "fm_plan_set_graphs: null plan");
    plan->use_graphs = on != 0;
    return FM_OK;
}

extern "C" fm_status fm_plan_set_concurrency(fm_plan plan, int32_t subbatches) {
    if (!plan || subbatches < 0) return fail(FM_EINVAL, "fm_plan_set_concurrency: bad arguments");
    if (plan->nsub != subbatches) {  // captured graphs hold the old split
        for (auto& g : plan->graphs)
            if (g.exec) cudaGraphExecDestroy(g.exec);
        plan->graphs.clear();
    }
    plan->nsub = subbatches;
    return FM_OK;
}

// Subspace + spectrum + peaks again for the listed frames of the last batch, on its kept covariance; the
// frames are grouped into runs of consecutive indices, each run one pass over the post-covariance pipeline.
static fm_status rerun_list(fm_plan pl, const int32_t* list, int64_t count, const fm_batch_io* io, cudaStream_t s) {
    const size_t MM2 = static_cast<size_t>(pl->d.m) * pl->d.m * 2;
    int64_t i = 0;
    while (i < count) {
        int64_t j = i + 1;
        while (j < count && list[j] == list[j - 1] + 1) ++j;
        const int64_t f0 = list[i], nf = j - i;
        const fm_batch_io o = io_view(pl, io, f0);
        const float* R = io->covariance ? o.covariance : pl->R + f0 * MM2;
        const Planes pv = pl->last_planes && !io->covariance ? planes_view(pl, f0) : Planes{};
        fm_status st = run_post_cov(pl, nf, &o, R, s, work_view(pl, f0), false, pv, false);
        if (st != FM_OK) return st;
        i = j;
    }
    return FM_OK;
}

extern "C" fm_status fm_pack_peak_records(const int32_t* cells, const int32_t* count, const int32_t* status,
                                          int64_t frames, int64_t k, int32_t* rec, void* stream) {
    if (frames < 0 || k < 1 || k > (1 << 20) || (frames > 0 && (!cells || !count || !status || !rec)))
        return fail(FM_EINVAL, "fm_pack_peak_records: bad arguments");
    if (frames == 0) return FM_OK;
    const int64_t n = frames * (k + 2);
    k_pack_records<<<static_cast<unsigned>((n + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        cells, count, status, frames, static_cast<int>(k), rec);
    FM_CUDA_OK(cudaGetLastError());
    return FM_OK;
}

extern "C" fm_status fm_rerun_frames(fm_plan pl, int64_t count, const int32_t* h_frames, const fm_batch_io* io,
                                     void* stream) {
    if (!pl || !io || count < 0 || (count > 0 && !h_frames))
        return fail(FM_EINVAL, "fm_rerun_frames: bad arguments");
    for (int64_t i = 0; i < count; ++i)
        if (h_frames[i] < 0 || h_frames[i] >= pl->d.max_frames || (i > 0 && h_frames[i] <= h_frames[i - 1]))
            return fail(FM_EINVAL, "fm_rerun_frames: frame list must be ascending indices within max_frames");
    if (count == 0) return FM_OK;
    FM_CUDA_OK(cudaSetDevice(pl->device));
    return rerun_list(pl, h_frames, count, io, static_cast<cudaStream_t>(stream));
}

extern "C" fm_status fm_estimate_batch_host(fm_plan pl, int64_t frames, const float* h_x, const uint64_t* draw_seeds,
                                            fm_host_out* out, void* stream) {
    if (!pl || !h_x || !out || !out->peak_cells || !out->peak_count || !out->status)
        return fail(FM_EINVAL, "fm_estimate_batch_host: null argument");
    if (frames < 1 || frames > pl->d.max_frames) return fail(FM_EINVAL, "fm_estimate_batch_host: frames out of range");
    const auto& d = pl->d;
    if (d.method != FM_METHOD_EXACT && d.method != FM_METHOD_LANCZOS && !draw_seeds)
        return fail(FM_EINVAL, "fm_estimate_batch_host: seeds required");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    FM_CUDA_OK(cudaSetDevice(pl->device));
    const size_t B = static_cast<size_t>(d.max_frames), M = d.m, N = d.n, P = d.p, K = d.k, L = d.grid_size;
    if (!pl->x_dev) {
        cudaError_t e = cudaSuccess;
        auto chk = [&](cudaError_t x) {
            if (e == cudaSuccess) e = x;
        };
        chk(pl->get(&pl->x_dev, B * M * N * 2));
        chk(pl->get(&pl->omega_dev, d.method == FM_METHOD_FAST2 ? B * M * P : d.method == FM_METHOD_FAST1_NORM2 ? B * M : 0));
        chk(pl->get(&pl->idx_dev, d.method == FM_METHOD_FAST1 ? B * P : 0));
        chk(pl->get(&pl->spec_dev, B * L));
        chk(pl->get(&pl->cells_dev, B * K));
        chk(pl->get(&pl->heights_dev, B * K));
        chk(pl->get(&pl->base_dev, B));
        chk(pl->get(&pl->count_dev, B));
        chk(pl->get(&pl->status_dev, B));
        if (d.method == FM_METHOD_FAST2) chk(cudaMallocHost(&pl->omega_pinned, sizeof(float) * B * M * P));
        if (d.method == FM_METHOD_FAST1_NORM2) chk(cudaMallocHost(&pl->omega_pinned, sizeof(float) * B * M));
        chk(cudaMallocHost(&pl->status_pinned, sizeof(int32_t) * B));
        chk(cudaStreamCreateWithFlags(&pl->copy_s, cudaStreamNonBlocking));
        for (cudaEvent_t& ev : pl->copy_ev) chk(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        if (e != cudaSuccess) return fm_fail_cuda(e, "fm_estimate_batch_host staging", __FILE__, __LINE__);
    }
    // The host path is PCIe-bound (X is 8 B per snapshot element): X crosses in chunks of >= kChunkMin
    // frames on the plan's copy stream, the Omega / index draw runs on the host while chunk 0 copies,
    // and chunk c computes on the caller's stream while chunk c+1 copies. Frames are independent, so
    // per-chunk runs give the same per-frame results as one run over the batch.
    constexpr int64_t kChunkMin = 128;
    // measured c2 (1024 frames): 1 chunk 21.3 ms, 2: 20.8, 4: 20.56, 8: 22.4; the plain 1.07 GB pinned H2D alone
    // takes 20.3 ms
    constexpr int64_t max_ch = 4;
    const int64_t nch = std::max<int64_t>(1, std::min<int64_t>(max_ch, frames / kChunkMin));
    const int64_t cs = (frames + nch - 1) / nch;
    cudaStream_t cp = pl->copy_s;
    FM_CUDA_OK(cudaEventRecord(pl->copy_ev[fm_plan_s::kHostChunks], s));  // staging free once s is here
    FM_CUDA_OK(cudaStreamWaitEvent(cp, pl->copy_ev[fm_plan_s::kHostChunks], 0));
    std::vector<int32_t> idx_host;
    for (int64_t c = 0; c < nch; ++c) {
        const int64_t f0 = c * cs, fc = std::min(cs, frames - f0);
        const size_t xo = static_cast<size_t>(f0) * M * N * 2;
        FM_CUDA_OK(cudaMemcpyAsync(pl->x_dev + xo, h_x + xo, sizeof(float) * fc * M * N * 2, cudaMemcpyHostToDevice, cp));
        if (c == 0 && (d.method == FM_METHOD_FAST2 || d.method == FM_METHOD_FAST1_NORM2)) {
            const size_t per = d.method == FM_METHOD_FAST2 ? M * P : M;
            if (d.method == FM_METHOD_FAST2) fm_draw_omega_batch(frames, draw_seeds, d.m, d.p, pl->omega_pinned);
            else fm_draw_uniforms_batch(frames, draw_seeds, d.m, pl->omega_pinned);
            FM_CUDA_OK(cudaMemcpyAsync(pl->omega_dev, pl->omega_pinned, sizeof(float) * frames * per,
                                       cudaMemcpyHostToDevice, cp));
        } else if (c == 0 && d.method == FM_METHOD_FAST1) {
            idx_host.resize(static_cast<size_t>(frames) * P);
            fm_status st = fm_draw_indices_batch(frames, draw_seeds, d.m, d.p, idx_host.data());
            if (st != FM_OK) return st;
            FM_CUDA_OK(cudaMemcpyAsync(pl->idx_dev, idx_host.data(), sizeof(int32_t) * idx_host.size(),
                                       cudaMemcpyHostToDevice, cp));
        }
        FM_CUDA_OK(cudaEventRecord(pl->copy_ev[c], cp));
    }
    auto chunk_io = [&](int64_t f0) {
        fm_batch_io io{};
        io.x = pl->x_dev + static_cast<size_t>(f0) * M * N * 2;
        io.omega = pl->omega_dev ? pl->omega_dev + static_cast<size_t>(f0) * M * (d.method == FM_METHOD_FAST2 ? P : 1)
                                 : nullptr;
        io.indices = pl->idx_dev ? pl->idx_dev + static_cast<size_t>(f0) * P : nullptr;
        io.spectrum = out->spectrum ? pl->spec_dev + static_cast<size_t>(f0) * L : nullptr;
        io.peak_cells = pl->cells_dev + static_cast<size_t>(f0) * K;
        io.peak_heights = pl->heights_dev + static_cast<size_t>(f0) * K;
        io.baseline = pl->base_dev + f0;
        io.peak_count = pl->count_dev + f0;
        io.status = pl->status_dev + f0;
        return io;
    };
    for (int64_t c = 0; c < nch; ++c) {
        const int64_t f0 = c * cs, fc = std::min(cs, frames - f0);
        FM_CUDA_OK(cudaStreamWaitEvent(s, pl->copy_ev[c], 0));
        const fm_batch_io io = chunk_io(f0);
        fm_status st = run_batch_at(pl, f0, fc, &io, s);  // R of every chunk kept in place for the redraws
        if (st != FM_OK) return st;
    }
    fm_batch_io io{};
    io.x = pl->x_dev;
    io.omega = pl->omega_dev;
    io.indices = pl->idx_dev;
    io.spectrum = out->spectrum ? pl->spec_dev : nullptr;
    io.peak_cells = pl->cells_dev;
    io.peak_heights = pl->heights_dev;
    io.baseline = pl->base_dev;
    io.peak_count = pl->count_dev;
    io.status = pl->status_dev;
    fm_status st = FM_OK;
    std::vector<int32_t> attempts(static_cast<size_t>(frames), 1);
    if (d.method == FM_METHOD_FAST2 || d.method == FM_METHOD_FAST1_NORM2) {
        // R/src/estimators.cpp:114-137: up to 3 sub-seeded redraws per rank-deficient frame.
        const size_t per = d.method == FM_METHOD_FAST2 ? M * P : M;
        std::vector<uint64_t> seeds(draw_seeds, draw_seeds + frames);
        std::vector<int32_t> redo;
        for (int attempt = 1; attempt < 4; ++attempt) {
            FM_CUDA_OK(cudaMemcpyAsync(pl->status_pinned, pl->status_dev, sizeof(int32_t) * frames,
                                       cudaMemcpyDeviceToHost, s));
            FM_CUDA_OK(cudaStreamSynchronize(s));
            redo.clear();
            for (int64_t f = 0; f < frames; ++f) {
                if (pl->status_pinned[f] & FM_FRAME_RANK) {
                    redo.push_back(static_cast<int32_t>(f));
                    attempts[f] = attempt + 1;
                    const uint64_t ds = fmhost::Rng::derive(draw_seeds[f], 0xF257u + static_cast<uint64_t>(attempt));
                    float* dst = pl->omega_pinned + static_cast<size_t>(f) * per;
                    if (d.method == FM_METHOD_FAST2) fmhost::gaussian_matrix_real(d.m, d.p, ds, dst);
                    else fm_draw_uniforms_batch(1, &ds, d.m, dst);
                    FM_CUDA_OK(cudaMemcpyAsync(pl->omega_dev + static_cast<size_t>(f) * per, dst, sizeof(float) * per,
                                               cudaMemcpyHostToDevice, s));
                }
            }
            if (redo.empty()) break;
            // only the flagged frames again, on their kept covariance (R/src/estimators.cpp:114-137 redraws the
            // failing frame alone)
            st = rerun_list(pl, redo.data(), static_cast<int64_t>(redo.size()), &io, s);
            if (st != FM_OK) return st;
        }
    }
    FM_CUDA_OK(cudaMemcpyAsync(out->peak_cells, pl->cells_dev, sizeof(int32_t) * frames * K, cudaMemcpyDeviceToHost, s));
    FM_CUDA_OK(cudaMemcpyAsync(out->peak_count, pl->count_dev, sizeof(int32_t) * frames, cudaMemcpyDeviceToHost, s));
    FM_CUDA_OK(cudaMemcpyAsync(out->status, pl->status_dev, sizeof(int32_t) * frames, cudaMemcpyDeviceToHost, s));
    if (out->peak_heights)
        FM_CUDA_OK(cudaMemcpyAsync(out->peak_heights, pl->heights_dev, sizeof(double) * frames * K,
                                   cudaMemcpyDeviceToHost, s));
    if (out->baseline)
        FM_CUDA_OK(cudaMemcpyAsync(out->baseline, pl->base_dev, sizeof(double) * frames, cudaMemcpyDeviceToHost, s));
    if (out->spectrum)
        FM_CUDA_OK(cudaMemcpyAsync(out->spectrum, pl->spec_dev, sizeof(float) * frames * L, cudaMemcpyDeviceToHost, s));
    FM_CUDA_OK(cudaStreamSynchronize(s));
    if (out->attempts) std::copy(attempts.begin(), attempts.end(), out->attempts);
    return FM_OK;
}

// ------------------------------------------------------------------ fp64 single-matrix entry points
namespace {

struct ZCtx {
    cudaStream_t s = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    ZCtx() {
        cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
    }
    ~ZCtx() {
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
        if (s) cudaStreamDestroy(s);
    }
};

// column-major complex128 Hermitian S -> row-major R (= conj of the column-major buffer)
std::vector<double> to_rowmajor_hermitian(const double* s, int64_t m) {
    std::vector<double> r(static_cast<size_t>(2 * m * m));
    for (int64_t e = 0; e < m * m; ++e) {
        r[2 * e] = s[2 * e];
        r[2 * e + 1] = -s[2 * e + 1];
    }
    return r;
}

bool all_finite(const double* a, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
        if (!std::isfinite(a[i])) return false;
    return true;
}

fm_status check_hermitian_input(const double* s, int64_t m, const char* who) {
    if (!s || m < 1) return fail(FM_EINVAL, std::string(who) + ": null or empty matrix");
    if (!all_finite(s, 2 * m * m)) return fail(FM_EINVAL, std::string(who) + ": non-finite entries");
    return FM_OK;
}

}  // namespace

extern "C" fm_status fm_z_spatial_covariance(int64_t m, int64_t n, const double* y, double* s_out) {
    if (m < 1 || n < 1) return fail(FM_EINVAL, "covariance: empty signal matrix");
    if (!y || !s_out) return fail(FM_EINVAL, "covariance: null pointer");
    if (!all_finite(y, 2 * m * n)) return fail(FM_EINVAL, "covariance: non-finite entries");
    ZCtx c;
    DevBuf<double> dy, ds;
    FM_CUDA_OK(dy.alloc(2 * m * n));
    FM_CUDA_OK(ds.alloc(2 * m * m));
    FM_CUDA_OK(cudaMemcpyAsync(dy.p, y, sizeof(double) * 2 * m * n, cudaMemcpyHostToDevice, c.s));
    dim3 blk(16, 16), grd(static_cast<unsigned>((m + 15) / 16), static_cast<unsigned>((m + 15) / 16));
    k_cov_z<<<grd, blk, 0, c.s>>>(reinterpret_cast<const fmk::c64*>(dy.p), reinterpret_cast<fmk::c64*>(ds.p),
                                  static_cast<int>(m), static_cast<int>(n));
    FM_CUDA_OK(cudaGetLastError());
    FM_CUDA_OK(cudaMemcpyAsync(s_out, ds.p, sizeof(double) * 2 * m * m, cudaMemcpyDeviceToHost, c.s));
    FM_CUDA_OK(cudaStreamSynchronize(c.s));
    return FM_OK;
}

// ------------------------------------------------------------------ temporal covariance
// temporal_covariance, R/src/scene.cpp:140-153,161-163: T = Y^H Y / M (N x N, lower rankUpdate of Y^H,
// mirrored, symmetrised) — the spatial kernels applied to Y^H.
extern "C" fm_status fm_z_temporal_covariance(int64_t m, int64_t n, const double* y, double* t_out) {
    if (m < 1 || n < 1) return fail(FM_EINVAL, "covariance: empty signal matrix");
    if (!y || !t_out) return fail(FM_EINVAL, "covariance: null pointer");
    if (!all_finite(y, 2 * m * n)) return fail(FM_EINVAL, "covariance: non-finite entries");
    std::vector<double> yh(static_cast<size_t>(2 * m * n));  // Y^H, N x M column-major
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            const size_t s = (static_cast<size_t>(j) * m + i) * 2, d = (static_cast<size_t>(i) * n + j) * 2;
            yh[d] = y[s];
            yh[d + 1] = -y[s + 1];
        }
    return fm_z_spatial_covariance(n, m, yh.data(), t_out);
}

// T = X^H X / M read straight from X's stored order (cov_tc.cu temporal mode: TMA boxes of 16 antenna rows x 128
// snapshots, transposed by the converter warps); odd N pads each row with one zero snapshot into `work` first (the
// TMA row pitch must be a multiple of 16 B), which adds nothing to T.
extern "C" fm_status fm_temporal_covariance_batch(const float* x, int64_t frames, int64_t m, int64_t n,
                                                  float* t_out, int32_t* status, float* work, void* stream) {
    if (frames < 1 || m < 1 || n < 1) return fail(FM_EINVAL, "temporal_covariance: empty signal matrix");
    if (!x || !t_out || !status) return fail(FM_EINVAL, "temporal_covariance: null pointer");
    if (frames * n > 0x7fffffff || frames * m > 0x7fffffff) return fail(FM_EINVAL, "temporal_covariance: batch too large");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t np = n + (n & 1);
    const float* xin = x;
    float* pad = nullptr;
    FM_CUDA_OK(cudaMemsetAsync(status, 0, sizeof(int32_t) * frames, s));
    if (n & 1) {
        pad = work;
        if (!pad) FM_CUDA_OK(cudaMallocAsync(reinterpret_cast<void**>(&pad), sizeof(float) * 2 * frames * m * np, s));
        k_pad_rows<<<static_cast<unsigned>(frames * m), 128, 0, s>>>(reinterpret_cast<const float2*>(x),
                                                                    reinterpret_cast<float2*>(pad), frames * m,
                                                                    static_cast<int>(n));
        xin = pad;
    }
    cudaError_t e = cudaGetLastError();
    // rescue-pass workspace (out-of-range frames recomputed with a power-of-two prescale, cov_tc.cu)
    FmCovRescue rs{};
    void* rbuf = nullptr;
    const size_t rbytes = sizeof(uint32_t) * frames + sizeof(int32_t) * frames + sizeof(float) * frames + 16;
    if (e == cudaSuccess) e = cudaMallocAsync(&rbuf, rbytes, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(rbuf, 0, rbytes, s);
    if (e == cudaSuccess) {
        rs.amax = static_cast<uint32_t*>(rbuf);
        rs.list = reinterpret_cast<int32_t*>(rs.amax + frames);
        rs.xscale = reinterpret_cast<float*>(rs.list + frames);
        rs.count = reinterpret_cast<int32_t*>(rs.xscale + frames);
        e = fm_launch_cov_tc(xin, t_out, status, frames, n, np, s, nullptr, nullptr, nullptr, m, &rs, m);
    }
    if (rbuf) cudaFreeAsync(rbuf, s);
    if (pad && !work) cudaFreeAsync(pad, s);
    if (e != cudaSuccess) return fm_fail_cuda(e, "fm_temporal_covariance_batch", __FILE__, __LINE__);
    return FM_OK;
}

static fm_status z_nystrom_common(int64_t m, const double* s, int64_t k, int64_t p, int32_t t, uint64_t seed,
                                  bool fast2, double* basis, double* eigenvalues, double* cost_seconds,
                                  int64_t* deficient_column) {
    ZCtx c;
    const int M = static_cast<int>(m), P = static_cast<int>(p), K = static_cast<int>(k);
    const auto rrow = to_rowmajor_hermitian(s, m);
    DevBuf<double> dR, dOm, dC, dV, dW, dRt, dH, dB, dE;
    DevBuf<int32_t> dSt, dScr, dDef, dIdx;
    FM_CUDA_OK(dR.alloc(2 * m * m));
    FM_CUDA_OK(dOm.alloc(m * p));
    FM_CUDA_OK(dC.alloc(2 * m * p));
    FM_CUDA_OK(dV.alloc(2 * m * p));
    FM_CUDA_OK(dW.alloc(4 * m * p));
    FM_CUDA_OK(dRt.alloc(2 * p * p));
    FM_CUDA_OK(dH.alloc(2 * p * p));
    FM_CUDA_OK(dB.alloc(2 * m * k));
    FM_CUDA_OK(dE.alloc(k));
    FM_CUDA_OK(dSt.alloc(1));
    FM_CUDA_OK(dScr.alloc(1));
    FM_CUDA_OK(dDef.alloc(1));
    FM_CUDA_OK(dIdx.alloc(p));
    FM_CUDA_OK(cudaMemcpyAsync(dR.p, rrow.data(), sizeof(double) * rrow.size(), cudaMemcpyHostToDevice, c.s));
    FM_CUDA_OK(cudaEventRecord(c.e0, c.s));
    int32_t st_host = 0, def_host = -1;
    if (fast2) {
        std::vector<double> om(static_cast<size_t>(m * p));
        for (int attempt = 0;; ++attempt) {
            const uint64_t ds = attempt == 0 ? seed : fmhost::Rng::derive(seed, 0xF257u + static_cast<uint64_t>(attempt));
            fmhost::gaussian_matrix_real(m, p, ds, om.data());
            FM_CUDA_OK(cudaMemcpyAsync(dOm.p, om.data(), sizeof(double) * om.size(), cudaMemcpyHostToDevice, c.s));
            FM_CUDA_OK(cudaMemsetAsync(dSt.p, 0, sizeof(int32_t), c.s));
            FM_CUDA_OK(cudaMemsetAsync(dDef.p, 0xff, sizeof(int32_t), c.s));
            FM_CUDA_OK(fm_launch_rmul<double>(dR.p, dOm.p, nullptr, dC.p, nullptr, 1, M, P, true, c.s));
            for (int it = 0; it < t; ++it) {
                FM_CUDA_OK(fm_launch_qr<double>(dC.p, dW.p, dV.p, nullptr, dSt.p, dDef.p, nullptr, 1, M, P, false, c.s));
                FM_CUDA_OK(fm_launch_rmul<double>(dR.p, nullptr, dV.p, dC.p, nullptr, 1, M, P, false, c.s));
            }
            FM_CUDA_OK(cudaMemcpyAsync(&st_host, dSt.p, sizeof(int32_t), cudaMemcpyDeviceToHost, c.s));
            FM_CUDA_OK(cudaMemcpyAsync(&def_host, dDef.p, sizeof(int32_t), cudaMemcpyDeviceToHost, c.s));
            FM_CUDA_OK(cudaStreamSynchronize(c.s));
            if (!(st_host & FM_FRAME_RANK)) break;
            if (attempt + 1 >= 4) {
                if (deficient_column) *deficient_column = def_host;
                char msg[160];
                std::snprintf(msg, sizeof msg, "qr_orthonormal: rank deficient sketch; column %d is dependent",
                              def_host);
                return fail(FM_ERANK, msg);
            }
        }
        FM_CUDA_OK(fm_launch_qr<double>(dC.p, dW.p, nullptr, dRt.p, dScr.p, nullptr, nullptr, 1, M, P, true, c.s));
        FM_CUDA_OK(fm_launch_nystrom<double>(dV.p, dC.p, nullptr, dW.p, dRt.p, dB.p, dE.p, dSt.p, nullptr, 1, M, P, K,
                                             true, c.s));
    } else {
        fmhost::Rng r(seed);
        const auto idx = r.sample_without_replacement(m, p);
        std::vector<int32_t> idx32(idx.begin(), idx.end());
        FM_CUDA_OK(cudaMemcpyAsync(dIdx.p, idx32.data(), sizeof(int32_t) * p, cudaMemcpyHostToDevice, c.s));
        FM_CUDA_OK(cudaMemsetAsync(dSt.p, 0, sizeof(int32_t), c.s));
        FM_CUDA_OK(fm_launch_gather<double>(dR.p, dIdx.p, dC.p, dH.p, nullptr, 1, M, P, c.s));
        FM_CUDA_OK(fm_launch_qr<double>(dC.p, dW.p, nullptr, dRt.p, dScr.p, nullptr, nullptr, 1, M, P, true, c.s));
        FM_CUDA_OK(fm_launch_nystrom<double>(nullptr, nullptr, dH.p, dW.p, dRt.p, dB.p, dE.p, dSt.p, nullptr, 1, M, P,
                                             K, false, c.s));
    }
    FM_CUDA_OK(cudaEventRecord(c.e1, c.s));
    FM_CUDA_OK(cudaMemcpyAsync(basis, dB.p, sizeof(double) * 2 * m * k, cudaMemcpyDeviceToHost, c.s));
    FM_CUDA_OK(cudaMemcpyAsync(eigenvalues, dE.p, sizeof(double) * k, cudaMemcpyDeviceToHost, c.s));
    FM_CUDA_OK(cudaMemcpyAsync(&st_host, dSt.p, sizeof(int32_t), cudaMemcpyDeviceToHost, c.s));
    FM_CUDA_OK(cudaStreamSynchronize(c.s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c.e0, c.e1);
    if (cost_seconds) *cost_seconds = ms * 1e-3;
    if (st_host & FM_FRAME_NOCONV) return fail(FM_ENOCONV, "thin_svd: Jacobi SVD did not converge");
    return FM_OK;
}

extern "C" fm_status fm_z_fast_music_2(int64_t m, const double* s, int64_t k, int64_t p, int32_t t, uint64_t seed,
                                       double* basis, double* eigenvalues, double* cost_seconds,
                                       int64_t* deficient_column) {
    fm_status st = check_hermitian_input(s, m, "fast_music_2");
    if (st != FM_OK) return st;
    if (k < 1 || k >= m) return fail(FM_EINVAL, "fast_music_2: need 1 <= K < M");
    if (p < k || p > m) return fail(FM_EINVAL, "fast_music_2: need K <= p <= M");
    if (t < 1 || t > 20) return fail(FM_EINVAL, "fast_music_2: need 1 <= t <= 20");
    if (!basis || !eigenvalues) return fail(FM_EINVAL, "fast_music_2: null output");
    return z_nystrom_common(m, s, k, p, t, seed, true, basis, eigenvalues, cost_seconds, deficient_column);
}

extern "C" fm_status fm_z_fast_music_1(int64_t m, const double* s, int64_t k, int64_t p, uint64_t seed, double* basis,
                                       double* eigenvalues, double* cost_seconds) {
    fm_status st = check_hermitian_input(s, m, "fast_music_1");
    if (st != FM_OK) return st;
    if (k < 1 || k >= m) return fail(FM_EINVAL, "fast_music_1: need 1 <= K < M");
    if (p < k || p > m) return fail(FM_EINVAL, "fast_music_1: need K <= p <= M");
    if (!basis || !eigenvalues) return fail(FM_EINVAL, "fast_music_1: null output");
    return z_nystrom_common(m, s, k, p, 1, seed, false, basis, eigenvalues, cost_seconds, nullptr);
}

// The K leading (signed-descending) eigenpairs of the Hermitian S by the Jacobi eigensolver; K = M gives the full
// decomposition (hermitian_eig).
static fm_status z_leading_eigenpairs(int64_t m, const double* s, int64_t k, double* basis, double* eigenvalues,
                                      double* cost_seconds) {
    const int64_t mp = (m + 15) / 16 * 16;
    ZCtx c;
    const auto rrow = to_rowmajor_hermitian(s, m);
    DevBuf<double> dR, dW, dB, dE;
    DevBuf<int32_t> dSt;
    FM_CUDA_OK(dR.alloc(2 * m * m));
    FM_CUDA_OK(dW.alloc(2 * mp * mp));
    FM_CUDA_OK(dB.alloc(2 * m * k));
    FM_CUDA_OK(dE.alloc(k));
    FM_CUDA_OK(dSt.alloc(1));
    FM_CUDA_OK(cudaMemcpyAsync(dR.p, rrow.data(), sizeof(double) * rrow.size(), cudaMemcpyHostToDevice, c.s));
    FM_CUDA_OK(cudaMemsetAsync(dSt.p, 0, sizeof(int32_t), c.s));
    FM_CUDA_OK(cudaEventRecord(c.e0, c.s));
    FM_CUDA_OK(fm_launch_jacobi_eig<double>(dR.p, dW.p, dB.p, dE.p, dSt.p, 1, static_cast<int>(m),
                                            static_cast<int>(k), c.s));
    FM_CUDA_OK(cudaEventRecord(c.e1, c.s));
    int32_t st_host = 0;
    FM_CUDA_OK(cudaMemcpyAsync(basis, dB.p, sizeof(double) * 2 * m * k, cudaMemcpyDeviceToHost, c.s));
    FM_CUDA_OK(cudaMemcpyAsync(eigenvalues, dE.p, sizeof(double) * k, cudaMemcpyDeviceToHost, c.s));
    FM_CUDA_OK(cudaMemcpyAsync(&st_host, dSt.p, sizeof(int32_t), cudaMemcpyDeviceToHost, c.s));
    FM_CUDA_OK(cudaStreamSynchronize(c.s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c.e0, c.e1);
    if (cost_seconds) *cost_seconds = ms * 1e-3;
    if (st_host & FM_FRAME_NOCONV) return fail(FM_ENOCONV, "hermitian_eig: eigensolver did not converge");
    return FM_OK;
}

extern "C" fm_status fm_z_exact_signal_subspace(int64_t m, const double* s, int64_t k, double* basis,
                                                double* eigenvalues, double* cost_seconds) {
    fm_status st = check_hermitian_input(s, m, "exact_signal_subspace");
    if (st != FM_OK) return st;
    if (k < 1 || k >= m) return fail(FM_EINVAL, "exact_signal_subspace: need 1 <= K < M");
    if (!basis || !eigenvalues) return fail(FM_EINVAL, "exact_signal_subspace: null output");
    return z_leading_eigenpairs(m, s, k, basis, eigenvalues, cost_seconds);
}

extern "C" fm_status fm_z_hermitian_eig(int64_t m, const double* s, double* eigenvalues, double* eigenvectors) {
    fm_status st = check_hermitian_input(s, m, "hermitian_eig");
    if (st != FM_OK) return st;
    if (!eigenvalues || !eigenvectors) return fail(FM_EINVAL, "hermitian_eig: null output");
    if (m == 1) {  // nothing to rotate: the entry itself
        eigenvalues[0] = s[0];
        eigenvectors[0] = 1.0;
        eigenvectors[1] = 0.0;
        return FM_OK;
    }
    return z_leading_eigenpairs(m, s, m, eigenvectors, eigenvalues, nullptr);
}

extern "C" fm_status fm_z_music_spectrum(int64_t m, int64_t kb, const double* basis, int64_t L, double theta0,
                                         double theta1, double d, double lambda, double* values) {
    if (m < 1) return fail(FM_EINVAL, "music_spectrum: empty basis");
    if (L < 2) return fail(FM_EINVAL, "AngleGrid: L >= 2 required");
    if (d <= 0.0 || lambda <= 0.0) return fail(FM_EINVAL, "steering_vector: need M >= 1, d > 0, lambda > 0");
    if (kb < 0 || (kb > 0 && !basis) || !values) return fail(FM_EINVAL, "music_spectrum: bad arguments");
    ZCtx c;
    DevBuf<double> dB, dT, dZ, dOut, dDev;
    FM_CUDA_OK(dB.alloc(std::max<int64_t>(2 * m * kb, 2)));
    FM_CUDA_OK(dT.alloc(2 * m));
    FM_CUDA_OK(dZ.alloc(2 * L));
    FM_CUDA_OK(dOut.alloc(L));
    FM_CUDA_OK(dDev.alloc(1));
    if (kb > 0)
        FM_CUDA_OK(cudaMemcpyAsync(dB.p, basis, sizeof(double) * 2 * m * kb, cudaMemcpyHostToDevice, c.s));
    const auto z = zgrid_host(L, theta0, theta1, d, lambda, false);
    FM_CUDA_OK(cudaMemcpyAsync(dZ.p, z.data(), sizeof(double) * z.size(), cudaMemcpyHostToDevice, c.s));
    if (kb > 0) {
        double dev = 0.0;
        FM_CUDA_OK(fm_launch_orthocheck(dB.p, 1, static_cast<int>(m), static_cast<int>(kb), dDev.p, c.s));
        FM_CUDA_OK(cudaMemcpyAsync(&dev, dDev.p, sizeof(double), cudaMemcpyDeviceToHost, c.s));
        FM_CUDA_OK(cudaStreamSynchronize(c.s));
        if (!(dev <= 1e-6)) return fail(FM_EINVAL, "music_spectrum: basis columns are not orthonormal");
    }
    FM_CUDA_OK(fm_launch_autocorr(dB.p, dT.p, 1, static_cast<int>(m), static_cast<int>(kb), c.s));
    FM_CUDA_OK(fm_launch_spectrum_one(dT.p, dZ.p, 1, static_cast<int>(m), static_cast<int>(L), nullptr, dOut.p, c.s));
    FM_CUDA_OK(cudaMemcpyAsync(values, dOut.p, sizeof(double) * L, cudaMemcpyDeviceToHost, c.s));
    FM_CUDA_OK(cudaStreamSynchronize(c.s));
    return FM_OK;
}

extern "C" fm_status fm_z_extract_peaks(const double* values, int64_t L, int64_t k, int64_t min_sep, int64_t* cells,
                                        double* heights, int64_t* count, double* baseline, int32_t* shortfall) {
    if (k < 1) return fail(FM_EINVAL, "extract_peaks: K >= 1 required");
    if (!values || L < 1 || !cells || !heights || !count || !baseline || !shortfall)
        return fail(FM_EINVAL, "extract_peaks: bad arguments");
    if (L > 0x7fffffff || k > 0x7fffffff) return fail(FM_EINVAL, "extract_peaks: grid or K too large");
    ZCtx c;
    DevBuf<double> dV, dH, dBase;
    DevBuf<int32_t> dC, dN;
    DevBuf<uint8_t> dWs;
    FM_CUDA_OK(dV.alloc(L));
    FM_CUDA_OK(dH.alloc(k));
    FM_CUDA_OK(dBase.alloc(1));
    FM_CUDA_OK(dC.alloc(k));
    FM_CUDA_OK(dN.alloc(1));
    FM_CUDA_OK(dWs.alloc(fm_peaks_workspace_bytes(1, static_cast<int>(L), static_cast<int>(k))));
    FM_CUDA_OK(cudaMemcpyAsync(dV.p, values, sizeof(double) * L, cudaMemcpyHostToDevice, c.s));
    FM_CUDA_OK(fm_launch_peaks_only(dV.p, 1, static_cast<int>(L), static_cast<int>(k), static_cast<int>(min_sep), dC.p,
                                    dH.p, dBase.p, dN.p, dWs.p, c.s));
    std::vector<int32_t> c32(static_cast<size_t>(k));
    int32_t n = 0;
    FM_CUDA_OK(cudaMemcpyAsync(c32.data(), dC.p, sizeof(int32_t) * k, cudaMemcpyDeviceToHost, c.s));
    FM_CUDA_OK(cudaMemcpyAsync(heights, dH.p, sizeof(double) * k, cudaMemcpyDeviceToHost, c.s));
    FM_CUDA_OK(cudaMemcpyAsync(baseline, dBase.p, sizeof(double), cudaMemcpyDeviceToHost, c.s));
    FM_CUDA_OK(cudaMemcpyAsync(&n, dN.p, sizeof(int32_t), cudaMemcpyDeviceToHost, c.s));
    FM_CUDA_OK(cudaStreamSynchronize(c.s));
    for (int64_t i = 0; i < k; ++i) cells[i] = c32[static_cast<size_t>(i)];
    *count = n;
    *shortfall = n < k ? 1 : 0;
    return FM_OK;
}
