// Certificate of the exact method's subspace iteration (exact_signal_subspace, R/src/estimators.cpp:73-85 ->
// hermitian_eig, R/src/linalg.cpp:77-89): a frame's top-K basis U from the iteration is accepted only if its
// distance to the true top-K eigenvectors of R provably moves the MUSIC spectrum by less than a tenth of the
// 0.05 dB gate; every other frame is recomputed by the full Jacobi eigensolver (jacobi.cu).
//
// Bound (Davis-Kahan sin-theta, Courant-Fischer):
//   mu_k = u_k^H R u_k (Rayleigh quotients), E = R U - U diag(mu) (fp64 products of the complex64 R),
//   lambda_{K+1}(R) <= lambda_max(P_perp R P_perp) <= tr(R) - tr(U^H R U)       (R PSD, U orthonormal),
//   delta = min_k mu_k - (tr(R) - sum_k mu_k);  if delta > 0:  ||sin Theta(U, U_true)||_2 <= s = ||E||_F / delta.
// For a steering vector a (||a||^2 = M) the denominator d = a^H (I - U U^H) a then moves by at most
//   |d - d_true| <= 2 s ||a|| sqrt(d_true) + s^2 ||a||^2,
// so with d_min = 1 / max_theta P(theta) the relative error over the whole grid is bounded by
//   2 s sqrt(M / d_min) + s^2 M / d_min  (first-order in s; checked against kRelTol = 1.16e-3 = 0.005 dB).
// Products and sums are fp64 (the only rounding is fp64's), so the bound is rigorous for the complex64 R the
// batch path eigendecomposes; the covariance's own fp16-operand error is the separate, measured part of the gate.

#include <cuda_runtime.h>

#include <cstdint>

#include "fm_common.cuh"

namespace fmk {
namespace exact {

constexpr int kT = 256;
constexpr int kMaxK = 16;
constexpr double kRelTol = 1.1579e-3;  // 10^(0.005 / 10) - 1: a tenth of the 0.05 dB gate

// One CTA per frame. R: frames x M x M complex64 row-major; basis: frames x K x M complex128 (column k of U
// contiguous). cert[f] = s (or +inf when delta <= 0 or K > kMaxK).
__global__ void __launch_bounds__(kT) k_exact_residual(const c32* __restrict__ R, const c64* __restrict__ basis,
                                                       double* __restrict__ cert, int m, int k) {
    extern __shared__ c64 xsm[];
    c64* U = xsm;          // [k][m]
    c64* RU = U + k * m;   // [k][m]
    __shared__ double red[kT / 32][2 * kMaxK + 2];
    __shared__ double mu[kMaxK];
    const int f = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (k > kMaxK) {
        if (tid == 0) cert[f] = INFINITY;
        return;
    }
    const c64* Uf = basis + static_cast<size_t>(f) * k * m;
    for (int e = tid; e < k * m; e += kT) U[e] = Uf[e];
    __syncthreads();
    const c32* Rf = R + static_cast<size_t>(f) * m * m;
    double tr = 0.0;
    // (R U)(r, :) by one warp per row: lanes split the columns c (coalesced row reads, all of a 256-column chunk
    // issued before the fp64 FMAs consume them), fp64 accumulation
    for (int r = warp; r < m; r += kT / 32) {
        c64 acc[kMaxK];
#pragma unroll
        for (int q = 0; q < kMaxK; ++q) acc[q] = mk(0.0, 0.0);
        const c32* row = Rf + static_cast<size_t>(r) * m;
        for (int c0 = 0; c0 < m; c0 += 256) {
            c32 a32[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int c = c0 + lane + 32 * j;
                a32[j] = c < m ? row[c] : mk(0.f, 0.f);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int c = c0 + lane + 32 * j;
                if (c >= m) break;
                const c64 a = to64(a32[j]);
                if (c == r) tr += a.re;
#pragma unroll
                for (int q = 0; q < kMaxK; ++q)
                    if (q < k) cmac(acc[q], a, U[q * m + c]);
            }
        }
#pragma unroll
        for (int q = 0; q < kMaxK; ++q) {
            if (q < k) {
                const double re = warp_sum(acc[q].re), im = warp_sum(acc[q].im);
                if (lane == 0) RU[q * m + r] = mk(re, im);
            }
        }
    }
    tr = warp_sum(tr);
    if (lane == 0) red[warp][2 * kMaxK] = tr;
    __syncthreads();
    // Rayleigh quotients mu_q = Re(u_q^H (R U)_q)
    for (int q = warp; q < k; q += kT / 32) {
        double s = 0.0;
        for (int r = lane; r < m; r += 32) {
            const c64 u = U[q * m + r], v = RU[q * m + r];
            s += u.re * v.re + u.im * v.im;
        }
        s = warp_sum(s);
        if (lane == 0) mu[q] = s;
    }
    __syncthreads();
    // ||E||_F^2 with E = R U - U diag(mu)
    double e2 = 0.0;
    for (int idx = tid; idx < k * m; idx += kT) {
        const int q = idx / m;
        const c64 u = U[idx], v = RU[idx];
        const double dr = v.re - mu[q] * u.re, di = v.im - mu[q] * u.im;
        e2 += dr * dr + di * di;
    }
    e2 = warp_sum(e2);
    if (lane == 0) red[warp][2 * kMaxK + 1] = e2;
    __syncthreads();
    if (tid == 0) {
        double trace = 0.0, en = 0.0, msum = 0.0, mmin = INFINITY;
        for (int w = 0; w < kT / 32; ++w) {
            trace += red[w][2 * kMaxK];
            en += red[w][2 * kMaxK + 1];
        }
        for (int q = 0; q < k; ++q) {
            msum += mu[q];
            mmin = fmin(mmin, mu[q]);
        }
        const double delta = mmin - (trace - msum);
        cert[f] = delta > 0.0 ? sqrt(en) / delta : INFINITY;
    }
}

// After the spectrum: d_min = 1 / max P; frames whose bound exceeds kRelTol (or that the iteration flagged) get
// kFrameRefine for the Jacobi rerun. One warp per frame.
__global__ void k_exact_check(const double* __restrict__ cert, const double* __restrict__ spec64,
                              const int32_t* __restrict__ iter_status, int32_t* __restrict__ status, int frames, int m,
                              int L) {
    const int f = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (f >= frames) return;
    const double* p = spec64 + static_cast<size_t>(f) * L;
    double pmax = 0.0;
    for (int l = lane; l < L; l += 32) pmax = fmax(pmax, p[l]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pmax = fmax(pmax, __shfl_xor_sync(0xffffffffu, pmax, o));
    if (lane == 0) {
        const double s = cert[f];
        const double q = pmax > 0.0 ? static_cast<double>(m) * pmax : INFINITY;  // M / d_min
        const double rel = 2.0 * s * sqrt(q) + s * s * q;
        if (iter_status[f] != 0 || !(rel <= kRelTol)) atomicOr(&status[f], kFrameRefine);
    }
}

}  // namespace exact
}  // namespace fmk

cudaError_t fm_launch_exact_residual(const void* R, const void* basis, double* cert, int frames, int m, int k,
                                     cudaStream_t s) {
    const size_t smem = sizeof(fmk::c64) * 2 * static_cast<size_t>(k) * m;
    if (smem > 200 * 1024) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(fmk::exact::k_exact_residual, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    fmk::exact::k_exact_residual<<<frames, fmk::exact::kT, smem, s>>>(static_cast<const fmk::c32*>(R),
                                                                      static_cast<const fmk::c64*>(basis), cert, m, k);
    return cudaGetLastError();
}

cudaError_t fm_launch_exact_check(const double* cert, const double* spec64, const int32_t* iter_status, int32_t* status,
                                  int frames, int m, int L, cudaStream_t s) {
    fmk::exact::k_exact_check<<<(frames + 7) / 8, 256, 0, s>>>(cert, spec64, iter_status, status, frames, m, L);
    return cudaGetLastError();
}
