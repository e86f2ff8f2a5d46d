// Shared device helpers for the Fast-MUSIC B200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

// Covariance rescue-pass workspace (cov_tc.cu): per-frame max |x| of pass 1 (float bits; zero between batches),
// the list of out-of-range frames, its count (device), and their power-of-two prescale.
struct FmCovRescue {
    uint32_t* amax;
    int32_t* list;
    int32_t* count;
    float* xscale;
};

namespace fmk {

// Per-frame status bits (written by kernels; mapped to the reference's
// exceptions by the host layer, R/include/fastmusic/types.hpp:18-43).
enum FrameStatus : int32_t {
    kFrameOk = 0,
    kFrameRank = 1,      // sketch lost column rank  -> RankDeficiencyError (host redraws)
    kFrameNoConv = 2,    // Jacobi sweep cap hit     -> NonConvergenceError
    kFrameRange = 4,     // input outside fp16 operand range of the tensor-core covariance
    kFrameNonFinite = 8, // NaN/Inf in the input frame
    kFrameRefine = 16    // internal: exact method, subspace iteration not certified -> Jacobi
};

template <typename T> struct cplx { T re, im; };
using c32 = cplx<float>;
using c64 = cplx<double>;

template <typename T> __host__ __device__ __forceinline__ cplx<T> mk(T r, T i) { return {r, i}; }
template <typename T> __host__ __device__ __forceinline__ cplx<T> operator+(cplx<T> a, cplx<T> b) { return {a.re + b.re, a.im + b.im}; }
template <typename T> __host__ __device__ __forceinline__ cplx<T> operator-(cplx<T> a, cplx<T> b) { return {a.re - b.re, a.im - b.im}; }
template <typename T> __host__ __device__ __forceinline__ cplx<T> operator*(cplx<T> a, cplx<T> b) {
    return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
template <typename T> __host__ __device__ __forceinline__ cplx<T> operator*(T s, cplx<T> a) { return {s * a.re, s * a.im}; }
template <typename T> __host__ __device__ __forceinline__ cplx<T> conj(cplx<T> a) { return {a.re, -a.im}; }
template <typename T> __host__ __device__ __forceinline__ T norm2(cplx<T> a) { return a.re * a.re + a.im * a.im; }
// acc += conj(a) * b
template <typename T> __host__ __device__ __forceinline__ void cmac_conj(cplx<T>& acc, cplx<T> a, cplx<T> b) {
    acc.re = fma(a.re, b.re, fma(a.im, b.im, acc.re));
    acc.im = fma(a.re, b.im, fma(-a.im, b.re, acc.im));
}
// acc += a * b
template <typename T> __host__ __device__ __forceinline__ void cmac(cplx<T>& acc, cplx<T> a, cplx<T> b) {
    acc.re = fma(a.re, b.re, fma(-a.im, b.im, acc.re));
    acc.im = fma(a.re, b.im, fma(a.im, b.re, acc.im));
}
template <typename T> __device__ __forceinline__ cplx<double> to64(cplx<T> a) { return {double(a.re), double(a.im)}; }

template <typename T> struct eps_of;
template <> struct eps_of<float> { static constexpr double value = 1.1920928955078125e-07; };
template <> struct eps_of<double> { static constexpr double value = 2.220446049250313e-16; };

// Rank of a batched CholQR factor by Eigen's ColPivHouseholderQR::rank() rule as the reference applies it
// (R/src/linalg.cpp:127-141): nonzero-pivot cut, then |R_kk| > p eps max|R_jj| -- with the reference's eps_64.
// The pivots come from the pivoted Cholesky of the fp64 Gram, d_k = |R_kk|^2, which resolves |R_kk| / |R_00|
// only down to ~sqrt(p eps_64) (~6e-8 at p = 16); that floors the threshold. Sketches with condition numbers up
// to ~1e7 (per-source 40 dB at M = 256) therefore pass, as they do in the fp64 reference.
__device__ __forceinline__ int cholqr_rank(const double* d, int p, int m) {
    const double eps = 2.220446049250313e-16;
    const double thr_helper = fmax(d[0], 0.0) * eps * eps / static_cast<double>(m);  // maxColNorm^2 = d[0]
    int nonzero = p;
    double maxpivot = 0.0;
    for (int k = 0; k < p; ++k) {
        if (nonzero == p && d[k] < thr_helper * static_cast<double>(m - k)) nonzero = k;
        maxpivot = fmax(maxpivot, sqrt(fmax(d[k], 0.0)));
    }
    const double rel = fmax(eps * static_cast<double>(p), sqrt(eps * static_cast<double>(p)));
    const double thr = maxpivot * rel;
    int rank = 0;
    for (int k = 0; k < nonzero; ++k) rank += sqrt(fmax(d[k], 0.0)) > thr ? 1 : 0;
    return rank;
}

// 2^-e for the power of two 2^e nearest below sqrt(v) (v > 0 normal double): exact rescaling factor.
__device__ __forceinline__ double pow2_inv_sqrt_scale(double v) {
    int e2 = ((__double2hiint(v) >> 20) & 0x7ff) - 1023;  // v = 1.x 2^e2
    int eh = e2 >> 1;                                     // floor(e2 / 2)
    eh = eh < -500 ? -500 : (eh > 500 ? 500 : eh);
    return __hiloint2double((1023 - eh) << 20, 0);
}

// One-sided Jacobi rotation of the column pair (x, y), al = |x|^2, be = |y|^2, g = x^H y, g2 = |g|^2 > 0:
// c, s (fp64) and s e with e = g / |g|, so that x' = c x - conj(s e) y, y' = s e x + c y are orthogonal.
// The angle is seeded in fp32 (short MUFU latency) from quantities normalised by a power of two near |g|
// (exact), so data of any scale neither underflows nor overflows the fp32 seed; c and 1/|g| are refined to
// fp64 by a Newton step (unitary to ~5e-15).
__device__ __forceinline__ void jacobi_rotation(double al, double be, c64 ga, double g2, double& cs, c64& se) {
    const double sc = pow2_inv_sqrt_scale(g2);
    const double g2n = g2 * sc * sc;  // [1, 4)
    const float igf = rsqrtf(static_cast<float>(g2n));
    const float zeta = static_cast<float>((be - al) * sc) * (0.5f * igf);
    const float tf = copysignf(1.0f, zeta) / (fabsf(zeta) + sqrtf(fmaf(zeta, zeta, 1.0f)));
    const double t = tf;
    const double x1 = fma(t, t, 1.0);
    double c = static_cast<double>(rsqrtf(static_cast<float>(x1)));
    c = c * fma(-0.5 * x1, c * c, 1.5);
    double ig = static_cast<double>(igf);
    ig = ig * fma(-0.5 * g2n, ig * ig, 1.5);
    ig *= sc;  // 1 / |g|
    const double sn = c * t;
    cs = c;
    se = mk(sn * ga.re * ig, sn * ga.im * ig);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace fmk

#define FM_CUDA_OK(expr)                                                     \
    do {                                                                     \
        cudaError_t _e = (expr);                                             \
        if (_e != cudaSuccess) return fm_fail_cuda(_e, #expr, __FILE__, __LINE__); \
    } while (0)
