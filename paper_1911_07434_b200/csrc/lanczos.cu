// Block-Lanczos signal subspace: block_lanczos_subspace, R/src/estimators.cpp:154-222
// (orthonormal_range :143-149), the paper's accurate baseline. Block Krylov iteration with full
// reorthogonalisation; converged when the top-K Ritz values change by <= 1e-10 relative on two consecutive
// checks; NonConvergenceError(last change) at the iteration cap.
//
// fp64 on the GPU, one matrix per call (the reference's single-matrix API): S q by the fp64 product kernel
// (fm_launch_rmul<double>), projections / corrections by the small complex128 GEMM kernels below, the
// start block and every expansion by the pivoted Householder QR (k_qr, Eigen ColPivHouseholderQR rank rule),
// the Ritz problem by the fp64 Jacobi eigensolver (k_jacobi_eig). The host only assembles the projected
// matrix h from the strips (copies, no arithmetic beyond the Hermitian average the reference applies) and
// runs the reference's control flow. The 1e-10 tolerance needs fp64 end to end, which is why this is not a
// batched complex64 plan method.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <limits>
#include <string>
#include <vector>

#include "../../include/fastmusic_b200.h"
#include "fm_common.cuh"
#include "host_rng.hpp"

fm_status fm_set_error(fm_status s, const std::string& msg);  // capi.cu
fm_status fm_fail_cuda(cudaError_t e, const char* expr, const char* file, int line);
template <typename T>
cudaError_t fm_launch_rmul(const void*, const void*, const void*, void*, const int32_t*, int, int, int, bool,
                           cudaStream_t);
template <typename T>
cudaError_t fm_launch_jacobi_eig(const void* R, void* work, void* basis, double* eig, int32_t* status, int frames,
                                 int m, int k, cudaStream_t s, int only_flagged, void* work32 = nullptr);
template <typename TS>
cudaError_t fm_launch_lanczos_batch(const void* S, const double* q0, double* basis_ws, double* w_ws, double* z_ws,
                                    double* out_basis, double* out_eig, int32_t* status, double* last_change,
                                    int32_t* iters, int frames, int m, int k, int b0, int max_iter, cudaStream_t s);
int fm_lanczos_batch_bmax();
int fm_lanczos_batch_nbmax();
int32_t fm_lanczos_batch_cap_flag();
std::vector<double> fm_lanczos_start_block(int64_t m, int b);
template <typename T>
cudaError_t fm_launch_qr_rank(const void* C, void* work, void* Vout, int32_t* status, int32_t* rank_out, int m, int p,
                              cudaStream_t s);

namespace {

using fmk::c64;
using fmk::mk;

// G = A^H B: A (m x na), B (m x nb) column-major complex128 -> G (na x nb) column-major. Warp per entry.
__global__ void k_zgemm_ah_b(const c64* __restrict__ A, const c64* __restrict__ B, c64* __restrict__ G, int m,
                             int na, int nb) {
    const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (e >= na * nb) return;
    const int i = e % na, j = e / na;
    const c64* a = A + static_cast<size_t>(i) * m;
    const c64* b = B + static_cast<size_t>(j) * m;
    double re = 0.0, im = 0.0;
    for (int r = lane; r < m; r += 32) {  // conj(a) b
        re += a[r].re * b[r].re + a[r].im * b[r].im;
        im += a[r].re * b[r].im - a[r].im * b[r].re;
    }
    re = fmk::warp_sum(re);
    im = fmk::warp_sum(im);
    if (lane == 0) G[e] = mk(re, im);
}

// Z = W - A G: W, Z (m x nb), A (m x na), G (na x nb), column-major; in place (Z == W) is fine.
__global__ void k_zgemm_sub(const c64* W, const c64* __restrict__ A, const c64* __restrict__ G, c64* Z, int m,
                            int na, int nb) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
    if (r >= m || j >= nb) return;
    double re = W[static_cast<size_t>(j) * m + r].re, im = W[static_cast<size_t>(j) * m + r].im;
    for (int c = 0; c < na; ++c) {
        const c64 a = A[static_cast<size_t>(c) * m + r], g = G[static_cast<size_t>(j) * na + c];
        re -= a.re * g.re - a.im * g.im;
        im -= a.re * g.im + a.im * g.re;
    }
    Z[static_cast<size_t>(j) * m + r] = mk(re, im);
}

// U = A V: A (m x na), V (na x k) column-major -> U (m x k).
__global__ void k_zgemm_ab(const c64* __restrict__ A, const c64* __restrict__ V, c64* __restrict__ U, int m, int na,
                           int k) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
    if (r >= m || j >= k) return;
    double re = 0.0, im = 0.0;
    for (int c = 0; c < na; ++c) {
        const c64 a = A[static_cast<size_t>(c) * m + r], v = V[static_cast<size_t>(j) * na + c];
        re += a.re * v.re - a.im * v.im;
        im += a.re * v.im + a.im * v.re;
    }
    U[static_cast<size_t>(j) * m + r] = mk(re, im);
}

template <typename T>
struct Buf {
    T* p = nullptr;
    cudaError_t alloc(size_t n) { return n ? cudaMalloc(&p, sizeof(T) * n) : cudaSuccess; }
    ~Buf() {
        if (p) cudaFree(p);
    }
};

struct Stream {
    cudaStream_t s = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    ~Stream() {
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
        if (s) cudaStreamDestroy(s);
    }
};

}  // namespace

#define LZ_CUDA(x)                                                              \
    do {                                                                        \
        cudaError_t e_ = (x);                                                   \
        if (e_ != cudaSuccess) return fm_fail_cuda(e_, #x, __FILE__, __LINE__); \
    } while (0)

extern "C" fm_status fm_z_block_lanczos_subspace(int64_t m, const double* s, int64_t k, int64_t block,
                                                 int32_t max_iterations, double* basis, double* eigenvalues,
                                                 double* cost_seconds, double* last_change) {
    if (m < 1 || !s) return fm_set_error(FM_EINVAL, "HermitianMatrix: input must be square and non-empty");
    for (int64_t i = 0; i < 2 * m * m; ++i)
        if (!std::isfinite(s[i])) return fm_set_error(FM_EINVAL, "HermitianMatrix: non-finite entries");
    if (k < 1 || k >= m) return fm_set_error(FM_EINVAL, "block_lanczos_subspace: need 1 <= K < M");
    if (block < k) return fm_set_error(FM_EINVAL, "block_lanczos_subspace: need block >= K");
    if (max_iterations < 1) return fm_set_error(FM_EINVAL, "block_lanczos_subspace: iters >= 1");
    if (!basis || !eigenvalues) return fm_set_error(FM_EINVAL, "block_lanczos_subspace: null output");
    const int M = static_cast<int>(m), K = static_cast<int>(k);
    const int b0 = static_cast<int>(std::min<int64_t>(block, m));
    const int64_t bc = std::max<int64_t>(64, b0);  // block-column capacity of the work buffers
    constexpr double kTol = 1e-10;
    constexpr uint64_t kStartSeed = 0x6C616E637A6FULL;  // R/src/estimators.cpp:162

    Stream st;
    LZ_CUDA(cudaStreamCreateWithFlags(&st.s, cudaStreamNonBlocking));
    LZ_CUDA(cudaEventCreate(&st.e0));
    LZ_CUDA(cudaEventCreate(&st.e1));
    cudaStream_t q_ = st.s;
    const size_t mm = static_cast<size_t>(m) * m;
    // S row-major Hermitian (HermitianMatrix symmetrisation, R/src/linalg.cpp:46-52) for the product kernel
    std::vector<double> srow(2 * mm);
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < m; ++j) {
            const double* a = s + 2 * (j * m + i);  // S(i, j)
            const double* b = s + 2 * (i * m + j);  // S(j, i)
            srow[2 * (i * m + j)] = 0.5 * (a[0] + b[0]);
            srow[2 * (i * m + j) + 1] = 0.5 * (a[1] - b[1]);
        }
    Buf<double> dS, dBasis, dQ, dW, dZ, dStrip, dStrip2, dQrWork, dH, dJW, dVec, dVal, dU;
    Buf<int32_t> dSt, dRank;
    const int64_t mpad = (m + 15) / 16 * 16;
    LZ_CUDA(dS.alloc(2 * mm));
    LZ_CUDA(dBasis.alloc(2 * mm));
    LZ_CUDA(dQ.alloc(2 * m * bc));
    LZ_CUDA(dW.alloc(2 * m * bc));
    LZ_CUDA(dZ.alloc(2 * m * bc));
    LZ_CUDA(dStrip.alloc(2 * m * bc));
    LZ_CUDA(dStrip2.alloc(2 * m * bc));
    LZ_CUDA(dQrWork.alloc(4 * m * bc));
    LZ_CUDA(dH.alloc(2 * mm));
    LZ_CUDA(dJW.alloc(2 * mpad * mpad));
    LZ_CUDA(dVec.alloc(2 * m * K));
    LZ_CUDA(dVal.alloc(K));
    LZ_CUDA(dU.alloc(2 * m * K));
    LZ_CUDA(dSt.alloc(1));
    LZ_CUDA(dRank.alloc(1));
    LZ_CUDA(cudaMemcpyAsync(dS.p, srow.data(), sizeof(double) * srow.size(), cudaMemcpyHostToDevice, q_));
    LZ_CUDA(cudaEventRecord(st.e0, q_));

    // Device-resident Krylov loop (lanczos_batch.cu, one CTA): used whenever the block and the basis fit its shared
    // memory; a frame that outgrows it (kFrameCap) falls through to the host-driven loop below.
    if (b0 <= fm_lanczos_batch_bmax()) {
        const auto q0 = fm_lanczos_start_block(m, b0);
        Buf<double> dQ0, dLB, dLW, dLZ, dOut, dEig, dLast;
        Buf<int32_t> dFl;
        LZ_CUDA(dQ0.alloc(q0.size()));
        LZ_CUDA(dLB.alloc(2 * m * static_cast<size_t>(fm_lanczos_batch_nbmax())));
        LZ_CUDA(dLW.alloc(2 * m * static_cast<size_t>(fm_lanczos_batch_bmax())));
        LZ_CUDA(dLZ.alloc(2 * m * static_cast<size_t>(fm_lanczos_batch_bmax())));
        LZ_CUDA(dOut.alloc(2 * m * K));
        LZ_CUDA(dEig.alloc(K));
        LZ_CUDA(dLast.alloc(1));
        LZ_CUDA(dFl.alloc(1));
        LZ_CUDA(cudaMemcpyAsync(dQ0.p, q0.data(), sizeof(double) * q0.size(), cudaMemcpyHostToDevice, q_));
        LZ_CUDA(cudaMemsetAsync(dFl.p, 0, sizeof(int32_t), q_));
        LZ_CUDA(fm_launch_lanczos_batch<double>(dS.p, dQ0.p, dLB.p, dLW.p, dLZ.p, dOut.p, dEig.p, dFl.p, dLast.p,
                                                nullptr, 1, M, K, b0, max_iterations, q_));
        LZ_CUDA(cudaEventRecord(st.e1, q_));
        int32_t fl = 0;
        double chg = 0.0;
        LZ_CUDA(cudaMemcpyAsync(&fl, dFl.p, sizeof(int32_t), cudaMemcpyDeviceToHost, q_));
        LZ_CUDA(cudaMemcpyAsync(&chg, dLast.p, sizeof(double), cudaMemcpyDeviceToHost, q_));
        LZ_CUDA(cudaMemcpyAsync(basis, dOut.p, sizeof(double) * 2 * m * K, cudaMemcpyDeviceToHost, q_));
        LZ_CUDA(cudaMemcpyAsync(eigenvalues, dEig.p, sizeof(double) * K, cudaMemcpyDeviceToHost, q_));
        LZ_CUDA(cudaStreamSynchronize(q_));
        if (!(fl & fm_lanczos_batch_cap_flag())) {
            float ms = 0.f;
            LZ_CUDA(cudaEventElapsedTime(&ms, st.e0, st.e1));
            if (cost_seconds) *cost_seconds = 1e-3 * ms;
            if (last_change) *last_change = chg;
            if (fl & fmk::kFrameNoConv) {
                char msg[160];
                std::snprintf(msg, sizeof msg,
                              "block_lanczos_subspace: no convergence within iteration cap (last change %.3g)", chg);
                return fm_set_error(FM_ENOCONV, msg);
            }
            return FM_OK;
        }
        LZ_CUDA(cudaEventRecord(st.e0, q_));
    }

    // q = qr_orthonormal(gaussian_matrix(m, min(block, m), kStartSeed)): real Gaussian cast to complex
    {
        std::vector<double> g(static_cast<size_t>(m) * b0), gc(2 * static_cast<size_t>(m) * b0, 0.0);
        fmhost::gaussian_matrix_real(m, b0, kStartSeed, g.data());  // row-major m x b0
        for (int64_t i = 0; i < m; ++i)
            for (int j = 0; j < b0; ++j) gc[2 * (static_cast<size_t>(j) * m + i)] = g[static_cast<size_t>(i) * b0 + j];
        LZ_CUDA(cudaMemcpyAsync(dZ.p, gc.data(), sizeof(double) * gc.size(), cudaMemcpyHostToDevice, q_));
    }
    int32_t st_host = 0, rank_host = 0;
    LZ_CUDA(cudaMemsetAsync(dSt.p, 0, sizeof(int32_t), q_));
    LZ_CUDA(fm_launch_qr_rank<double>(dZ.p, dQrWork.p, dQ.p, dSt.p, dRank.p, M, b0, q_));
    LZ_CUDA(cudaMemcpyAsync(&st_host, dSt.p, sizeof(int32_t), cudaMemcpyDeviceToHost, q_));
    LZ_CUDA(cudaStreamSynchronize(q_));
    if (st_host & FM_FRAME_RANK)  // R/src/linalg.cpp:134-139
        return fm_set_error(FM_ERANK, "qr_orthonormal: rank deficient start block");
    LZ_CUDA(cudaMemcpyAsync(dBasis.p, dQ.p, sizeof(double) * 2 * m * b0, cudaMemcpyDeviceToDevice, q_));
    int nb = b0, nw = b0;  // basis columns, newest block width
    std::vector<double> h;  // projected matrix, nh x nh column-major complex
    int nh = 0;
    std::vector<double> prev, vals(K), strip;
    double change_last = std::numeric_limits<double>::infinity();
    int stable = 0;

    auto finish = [&](int nbasis) -> fm_status {  // ritz_estimate: basis * eigvecs(:, 0:K), clamp_nonnegative
        const dim3 grd(static_cast<unsigned>((m + 127) / 128), static_cast<unsigned>(K));
        k_zgemm_ab<<<grd, 128, 0, q_>>>(reinterpret_cast<const c64*>(dBasis.p), reinterpret_cast<const c64*>(dVec.p),
                                        reinterpret_cast<c64*>(dU.p), M, nbasis, K);
        LZ_CUDA(cudaGetLastError());
        LZ_CUDA(cudaEventRecord(st.e1, q_));
        LZ_CUDA(cudaMemcpyAsync(basis, dU.p, sizeof(double) * 2 * m * K, cudaMemcpyDeviceToHost, q_));
        LZ_CUDA(cudaStreamSynchronize(q_));
        for (int i = 0; i < K; ++i) eigenvalues[i] = (vals[i] < 0.0 && vals[i] >= -1e-10) ? 0.0 : vals[i];
        float ms = 0.f;
        cudaEventElapsedTime(&ms, st.e0, st.e1);
        if (cost_seconds) *cost_seconds = ms * 1e-3;
        if (last_change) *last_change = change_last;
        return FM_OK;
    };

    for (int iter = 0; iter < max_iterations; ++iter) {
        // w = S q
        LZ_CUDA(fm_launch_rmul<double>(dS.p, nullptr, dQ.p, dW.p, nullptr, 1, M, nw, false, q_));
        // strip = basis^H w ((old + new) x new); the newest block is basis(:, old:nb)
        {
            const int ne = nb * nw;
            k_zgemm_ah_b<<<(ne + 7) / 8, 256, 0, q_>>>(reinterpret_cast<const c64*>(dBasis.p),
                                                       reinterpret_cast<const c64*>(dW.p),
                                                       reinterpret_cast<c64*>(dStrip.p), M, nb, nw);
            LZ_CUDA(cudaGetLastError());
            strip.assign(2 * static_cast<size_t>(ne), 0.0);
            LZ_CUDA(cudaMemcpyAsync(strip.data(), dStrip.p, sizeof(double) * strip.size(), cudaMemcpyDeviceToHost, q_));
            LZ_CUDA(cudaStreamSynchronize(q_));
        }
        // grow h (R/src/estimators.cpp:176-181)
        const int old = nh, nn = nb;
        std::vector<double> hn(2 * static_cast<size_t>(nn) * nn, 0.0);
        for (int j = 0; j < old; ++j)
            for (int i = 0; i < old; ++i) {
                hn[2 * (static_cast<size_t>(j) * nn + i)] = h[2 * (static_cast<size_t>(j) * old + i)];
                hn[2 * (static_cast<size_t>(j) * nn + i) + 1] = h[2 * (static_cast<size_t>(j) * old + i) + 1];
            }
        for (int j = 0; j < nw; ++j)
            for (int i = 0; i < nb; ++i) {
                const double re = strip[2 * (static_cast<size_t>(j) * nb + i)];
                const double im = strip[2 * (static_cast<size_t>(j) * nb + i) + 1];
                hn[2 * (static_cast<size_t>(old + j) * nn + i)] = re;  // h(i, old + j)
                hn[2 * (static_cast<size_t>(old + j) * nn + i) + 1] = im;
                if (i < old) {  // h(old + j, i) = conj(strip(i, j))
                    hn[2 * (static_cast<size_t>(i) * nn + old + j)] = re;
                    hn[2 * (static_cast<size_t>(i) * nn + old + j) + 1] = -im;
                }
            }
        h.swap(hn);
        nh = nn;
        // ritz = hermitian_eig(HermitianMatrix(h)): row-major 0.5 (h + h^H) for the Jacobi kernel
        std::vector<double> hr(2 * static_cast<size_t>(nh) * nh);
        for (int i = 0; i < nh; ++i)
            for (int j = 0; j < nh; ++j) {
                const double* a = &h[2 * (static_cast<size_t>(j) * nh + i)];  // h(i, j)
                const double* b = &h[2 * (static_cast<size_t>(i) * nh + j)];  // h(j, i)
                hr[2 * (static_cast<size_t>(i) * nh + j)] = 0.5 * (a[0] + b[0]);
                hr[2 * (static_cast<size_t>(i) * nh + j) + 1] = 0.5 * (a[1] - b[1]);
            }
        const int kk = std::min(K, nh);
        LZ_CUDA(cudaMemcpyAsync(dH.p, hr.data(), sizeof(double) * hr.size(), cudaMemcpyHostToDevice, q_));
        LZ_CUDA(cudaMemsetAsync(dSt.p, 0, sizeof(int32_t), q_));
        LZ_CUDA(fm_launch_jacobi_eig<double>(dH.p, dJW.p, dVec.p, dVal.p, dSt.p, 1, nh, kk, q_, 0));
        vals.assign(K, 0.0);
        LZ_CUDA(cudaMemcpyAsync(vals.data(), dVal.p, sizeof(double) * kk, cudaMemcpyDeviceToHost, q_));
        LZ_CUDA(cudaMemcpyAsync(&st_host, dSt.p, sizeof(int32_t), cudaMemcpyDeviceToHost, q_));
        LZ_CUDA(cudaStreamSynchronize(q_));
        if (st_host & FM_FRAME_NOCONV) return fm_set_error(FM_ENOCONV, "hermitian_eig: eigensolver did not converge");
        vals.resize(kk);
        if (static_cast<int>(prev.size()) == kk && kk == K) {  // R/src/estimators.cpp:194-203
            double change = 0.0;
            for (int i = 0; i < K; ++i) {
                const double denom = std::max(std::abs(vals[i]), 1e-300);
                change = std::max(change, std::abs(vals[i] - prev[i]) / denom);
            }
            change_last = change;
            stable = change <= kTol ? stable + 1 : 0;
            if (stable >= 2) return finish(nb);
        }
        prev = vals;
        // expand (R/src/estimators.cpp:205-217)
        const int room = M - nb;
        if (room <= 0) return finish(nb);
        {
            const dim3 grd(static_cast<unsigned>((m + 127) / 128), static_cast<unsigned>(nw));
            const c64* B = reinterpret_cast<const c64*>(dBasis.p);
            // z = w - basis (basis^H w)  (basis^H w is the strip)
            k_zgemm_sub<<<grd, 128, 0, q_>>>(reinterpret_cast<const c64*>(dW.p), B,
                                             reinterpret_cast<const c64*>(dStrip.p), reinterpret_cast<c64*>(dZ.p), M,
                                             nb, nw);
            // z -= basis (basis^H z)
            k_zgemm_ah_b<<<(nb * nw + 7) / 8, 256, 0, q_>>>(B, reinterpret_cast<const c64*>(dZ.p),
                                                            reinterpret_cast<c64*>(dStrip2.p), M, nb, nw);
            k_zgemm_sub<<<grd, 128, 0, q_>>>(reinterpret_cast<const c64*>(dZ.p), B,
                                             reinterpret_cast<const c64*>(dStrip2.p), reinterpret_cast<c64*>(dZ.p), M,
                                             nb, nw);
            LZ_CUDA(cudaGetLastError());
        }
        const int nz = std::min(nw, room);
        LZ_CUDA(cudaMemsetAsync(dSt.p, 0, sizeof(int32_t), q_));
        LZ_CUDA(fm_launch_qr_rank<double>(dZ.p, dQrWork.p, dQ.p, dSt.p, dRank.p, M, nz, q_));
        LZ_CUDA(cudaMemcpyAsync(&rank_host, dRank.p, sizeof(int32_t), cudaMemcpyDeviceToHost, q_));
        LZ_CUDA(cudaStreamSynchronize(q_));
        if (rank_host == 0) return finish(nb);
        LZ_CUDA(cudaMemcpyAsync(dBasis.p + 2 * static_cast<size_t>(nb) * m, dQ.p, sizeof(double) * 2 * m * rank_host,
                                cudaMemcpyDeviceToDevice, q_));
        nb += rank_host;
        nw = rank_host;
    }
    if (last_change) *last_change = change_last;
    char msg[160];
    std::snprintf(msg, sizeof msg, "block_lanczos_subspace: no convergence within iteration cap (last change %.3g)",
                  change_last);
    return fm_set_error(FM_ENOCONV, msg);
}
