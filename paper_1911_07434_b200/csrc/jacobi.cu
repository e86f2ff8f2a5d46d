// K5 — exact-MUSIC signal subspace: full Hermitian eigendecomposition by batched,
// block-cyclic one-sided (Hestenes) Jacobi, one CTA per frame.
//
// Replaces exact_signal_subspace R/src/estimators.cpp:73-85 -> hermitian_eig
// R/src/linalg.cpp:77-89 (Eigen SelfAdjointEigenSolver, eigenvalues descending).
//
// A = R (+ mu I) is orthogonalised column by column: for every column pair (i, j)
//   alpha = ||a_i||^2, beta = ||a_j||^2, gamma = a_i^H a_j,
//   zeta = (beta - alpha) / 2|gamma|, t = sgn(zeta) / (|zeta| + sqrt(1 + zeta^2)),
//   a_i' = c a_i - s e^{-i phi} a_j,  a_j' = s e^{i phi} a_i + c a_j   (e^{i phi} = gamma / |gamma|),
// until a sweep performs no rotation (|gamma| <= tol sqrt(alpha beta)). At convergence
// A = R V = U Sigma with U = V for PSD R, so the eigenpairs are (||a_c||, a_c / ||a_c||).
// Columns are processed in blocks of 16 staged in shared memory (block I stays resident
// while every block J >= I streams through), so each sweep touches the frame's A (kept in
// global / L2) ~ (nb + nb^2/2) block-times instead of once per column pair.
// fp64 facade path: a Gershgorin shift mu makes indefinite Hermitian input PSD (eigenvectors
// unchanged; lambda = sigma - mu), so the signed descending order of the reference is kept.
// Batch path (complex64 R): fp32 sweeps to fp32 convergence, then fp64 sweeps polish the fp32-converged columns
// (kModePolish: A starts from the fp32 A, widened exactly) -- the fp32 stage alone leaves the column orthogonality
// at ~1e-6, which moves the MUSIC spectrum by up to ~0.08 dB at c5; after the polish the columns are the exact
// singular vectors of a matrix within ~eps_32 |R| of R, like the rest of the complex64 path.

#include <cuda_runtime.h>

#include <cstdint>

#include "fm_common.cuh"

namespace fmk {
namespace jac {

constexpr int kNT = 256;
constexpr int kNW = kNT / 32;
constexpr int kB = 16;  // columns per block

template <typename T>
__device__ __forceinline__ bool pair_rotate(cplx<T>* ai, cplx<T>* aj, int mp, int lane, T tol) {
    T al = 0, be = 0;
    cplx<T> ga = mk<T>(0, 0);
    for (int r = lane; r < mp; r += 32) {
        const cplx<T> x = ai[r], y = aj[r];
        al = fma(x.re, x.re, fma(x.im, x.im, al));
        be = fma(y.re, y.re, fma(y.im, y.im, be));
        cmac_conj(ga, x, y);
    }
    al = warp_sum(al);
    be = warp_sum(be);
    ga.re = warp_sum(ga.re);
    ga.im = warp_sum(ga.im);
    const T g = sqrt(ga.re * ga.re + ga.im * ga.im);
    if (!(g > tol * sqrt(al * be)) || g == T(0)) return false;
    const T zeta = (be - al) / (T(2) * g);
    const T t = (zeta >= T(0) ? T(1) : T(-1)) / (fabs(zeta) + sqrt(T(1) + zeta * zeta));
    const T c = T(1) / sqrt(T(1) + t * t);
    const T s = c * t;
    const T er = ga.re / g, ei = ga.im / g;
    for (int r = lane; r < mp; r += 32) {
        const cplx<T> x = ai[r], y = aj[r];
        // conj(e) y and e x
        const T eyr = er * y.re + ei * y.im, eyi = er * y.im - ei * y.re;
        const T exr = er * x.re - ei * x.im, exi = er * x.im + ei * x.re;
        ai[r] = mk<T>(c * x.re - s * eyr, c * x.im - s * eyi);
        aj[r] = mk<T>(s * exr + c * y.re, s * exi + c * y.im);
    }
    return true;
}

constexpr int kModeOnlyFlagged = 1;  // frames with kFrameRefine only (the exact method's uncertified frames)
constexpr int kModePolish = 2;       // A starts from A0 (fp32 stage), R (complex64) only sets the scale
constexpr int kModeNoStatus = 4;     // do not flag non-convergence (the fp32 stage; the polish decides)

template <typename T>
__global__ void __launch_bounds__(kNT) k_jacobi_eig(const void* __restrict__ Rv, const cplx<float>* __restrict__ A0,
                                                    cplx<T>* __restrict__ work, c64* __restrict__ basis,
                                                    double* __restrict__ eig, int32_t* __restrict__ status, int m,
                                                    int k, int mode) {
    const int only_flagged = mode & kModeOnlyFlagged;
    const bool polish = (mode & kModePolish) != 0;
    extern __shared__ uint8_t dsm[];
    const int mp = (m + kB - 1) / kB * kB;
    const int nb = mp / kB;
    cplx<T>* sI = reinterpret_cast<cplx<T>*>(dsm);
    cplx<T>* sJ = sI + kB * mp;
    __shared__ double s_sig[1024];
    __shared__ int s_rot;
    __shared__ double s_mu;
    const int f = blockIdx.x;
    if (only_flagged && !(status[f] & kFrameRefine)) return;  // certified by the subspace iteration
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // R: cplx<T> (mode 0) or the batch's complex64 R (polish: only its diagonal, for the scale)
    const cplx<T>* Rf = static_cast<const cplx<T>*>(Rv) + static_cast<size_t>(f) * m * m;
    const cplx<float>* Rf32 = static_cast<const cplx<float>*>(Rv) + static_cast<size_t>(f) * m * m;
    auto rdiag = [&](int c) -> double {
        return polish ? static_cast<double>(Rf32[static_cast<size_t>(c) * m + c].re)
                      : static_cast<double>(Rf[static_cast<size_t>(c) * m + c].re);
    };
    cplx<T>* A = work + static_cast<size_t>(f) * mp * mp;
    const T tol = T(4) * static_cast<T>(eps_of<T>::value) * sqrt(static_cast<T>(mp));

    // Gershgorin shift (fp64 facade path only): mu = max(0, -min_i (R_ii - sum_{j!=i} |R_ij|))
    if (threadIdx.x == 0) s_mu = 0.0;
    __syncthreads();
    if (sizeof(T) == 8 && !polish) {
        for (int c = warp; c < m; c += kNW) {
            double off = 0.0;
            for (int r = lane; r < m; r += 32)
                if (r != c) off += sqrt(norm2(to64(Rf[static_cast<size_t>(c) * m + r])));
            off = warp_sum(off);
            if (lane == 0) {
                const double lo = static_cast<double>(Rf[static_cast<size_t>(c) * m + c].re) - off;
                if (lo < 0.0) {
                    // atomic max on a non-negative double via its bit pattern
                    unsigned long long* p = reinterpret_cast<unsigned long long*>(&s_mu);
                    atomicMax(p, __double_as_longlong(-lo));
                }
            }
        }
        __syncthreads();
    }
    // power-of-two normalisation (exact): A = 2^-e (R + mu I) with max_c |R_cc| + mu in [1, 2) -- the column
    // products below then stay inside the fp32 range for inputs of any scale; lambda is scaled back at the end
    __shared__ double s_dmax;
    if (threadIdx.x == 0) s_dmax = 0.0;
    __syncthreads();
    for (int c = threadIdx.x; c < m; c += kNT) {
        const double v = fabs(rdiag(c)) + s_mu;
        if (v > 0.0 && v < 1e300) atomicMax(reinterpret_cast<unsigned long long*>(&s_dmax), __double_as_longlong(v));
    }
    __syncthreads();
    const double nsc = s_dmax > 0.0 ? pow2_inv_sqrt_scale(s_dmax * s_dmax) : 1.0;  // 2^-e
    const T mu = static_cast<T>(s_mu);
    // A[c][r] = R(r, c) = conj(R[c][r]) (row-major Hermitian R), padded with zeros
    if (polish) {  // the fp32 stage's columns (already scaled by nsc), widened exactly
        const cplx<float>* A0f = A0 + static_cast<size_t>(f) * mp * mp;
        for (int e = threadIdx.x; e < mp * mp; e += kNT)
            A[e] = mk<T>(static_cast<T>(A0f[e].re), static_cast<T>(A0f[e].im));
    } else {
        for (int e = threadIdx.x; e < mp * mp; e += kNT) {
            const int c = e / mp, r = e % mp;
            cplx<T> v = mk<T>(0, 0);
            if (c < m && r < m) v = conj(Rf[static_cast<size_t>(c) * m + r]);
            if (c == r && c < m) v.re += mu;
            A[static_cast<size_t>(c) * mp + r] = mk<T>(static_cast<T>(v.re * nsc), static_cast<T>(v.im * nsc));
        }
    }
    __syncthreads();

    bool converged = false;
    for (int sweep = 0; sweep < 40 && !converged; ++sweep) {
        if (threadIdx.x == 0) s_rot = 0;
        bool rot = false;
        for (int I = 0; I < nb; ++I) {
            __syncthreads();
            for (int e = threadIdx.x; e < kB * mp; e += kNT) sI[e] = A[static_cast<size_t>(I) * kB * mp + e];
            __syncthreads();
            // intra-block pairs: round-robin over 16 columns (15 rounds x 8 pairs)
            for (int rnd = 0; rnd < kB - 1; ++rnd) {
                int i, j;
                if (warp == 0) {
                    i = rnd;
                    j = kB - 1;
                } else {
                    i = (rnd + warp) % (kB - 1);
                    j = (rnd - warp + (kB - 1)) % (kB - 1);
                }
                rot |= pair_rotate(sI + i * mp, sI + j * mp, mp, lane, tol);
                __syncthreads();
            }
            for (int J = I + 1; J < nb; ++J) {
                for (int e = threadIdx.x; e < kB * mp; e += kNT) sJ[e] = A[static_cast<size_t>(J) * kB * mp + e];
                __syncthreads();
                // cross pairs (i, (i + rnd) % 16): 16 rounds x 16 disjoint pairs, 2 per warp
                for (int rnd = 0; rnd < kB; ++rnd) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int i = warp + kNW * h;
                        const int j = (i + rnd) % kB;
                        rot |= pair_rotate(sI + i * mp, sJ + j * mp, mp, lane, tol);
                    }
                    __syncthreads();
                }
                for (int e = threadIdx.x; e < kB * mp; e += kNT) A[static_cast<size_t>(J) * kB * mp + e] = sJ[e];
                __syncthreads();
            }
            for (int e = threadIdx.x; e < kB * mp; e += kNT) A[static_cast<size_t>(I) * kB * mp + e] = sI[e];
        }
        if (rot && lane == 0) s_rot = 1;
        __syncthreads();
        converged = (s_rot == 0);
        __syncthreads();
    }
    // eigenvalues sigma_c = ||a_c|| (minus the shift), top-K descending
    for (int c = warp; c < mp; c += kNW) {
        double s = 0.0;
        const cplx<T>* a = A + static_cast<size_t>(c) * mp;
        for (int r = lane; r < mp; r += 32) s += norm2(to64(a[r]));
        s = warp_sum(s);
        if (lane == 0) s_sig[c] = c < m ? sqrt(s) : -1.0;
    }
    __syncthreads();
    __shared__ int s_sel[64];
    if (threadIdx.x == 0) {
        for (int q = 0; q < k; ++q) {
            int best = -1;
            for (int c = 0; c < m; ++c) {
                bool used = false;
                for (int z = 0; z < q; ++z) used |= (s_sel[z] == c);
                if (!used && (best < 0 || s_sig[c] > s_sig[best])) best = c;
            }
            s_sel[q] = best;
        }
    }
    __syncthreads();
    c64* Bf = basis + static_cast<size_t>(f) * m * k;
    for (int e = threadIdx.x; e < m * k; e += kNT) {
        const int q = e / m, r = e % m;
        const int c = s_sel[q];
        const double s = s_sig[c];
        const double inv = s > 0.0 ? 1.0 / s : 0.0;
        const c64 a = to64(A[static_cast<size_t>(c) * mp + r]);
        Bf[static_cast<size_t>(q) * m + r] = mk(a.re * inv, a.im * inv);
    }
    if (threadIdx.x < k) {
        double lam = s_sig[s_sel[threadIdx.x]] / nsc - static_cast<double>(mu);
        if (lam < 0.0 && lam >= -1e-10) lam = 0.0;
        eig[static_cast<size_t>(f) * k + threadIdx.x] = lam;
    }
    if (threadIdx.x == 0 && !converged && !(mode & kModeNoStatus)) atomicOr(&status[f], kFrameNoConv);
}

}  // namespace jac
}  // namespace fmk

using namespace fmk;

cudaError_t fm_gen_hermitian_eig(const void* R, void* work, void* basis, double* eig, int32_t* status, int m, int k,
                                 cudaStream_t s);

template <typename T>
static cudaError_t launch_jac(const void* R, const void* a0, void* wk, void* basis, double* eig, int32_t* status,
                              int frames, int m, int k, int mode, cudaStream_t s) {
    const int mp = (m + jac::kB - 1) / jac::kB * jac::kB;
    const size_t smem = 2 * jac::kB * static_cast<size_t>(mp) * sizeof(cplx<T>);
    if (mp > 1024 || k > 64 || smem > 200 * 1024) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(jac::k_jacobi_eig<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    jac::k_jacobi_eig<T><<<frames, jac::kNT, smem, s>>>(R, static_cast<const cplx<float>*>(a0), static_cast<cplx<T>*>(wk),
                                                        static_cast<c64*>(basis), eig, status, m, k, mode);
    return cudaGetLastError();
}

// T = double: fp64 on cplx<double> R (facade, Lanczos). T = float: complex64 R, fp32 sweeps into work32 (frames x
// mp x mp complex64) then the fp64 polish into work (frames x mp x mp complex128).
template <typename T>
cudaError_t fm_launch_jacobi_eig(const void* R, void* work, void* basis, double* eig, int32_t* status, int frames,
                                 int m, int k, cudaStream_t s, int only_flagged, void* work32) {
    const int of = only_flagged ? jac::kModeOnlyFlagged : 0;
    if (sizeof(T) == 8) {
        const int mp = (m + jac::kB - 1) / jac::kB * jac::kB;
        if (mp > 384 || k > 64) {  // beyond the shared-memory block staging: global-memory Jacobi (general.cu)
            if (only_flagged) return cudaErrorInvalidValue;
            for (int f = 0; f < frames; ++f) {
                cudaError_t e = fm_gen_hermitian_eig(static_cast<const c64*>(R) + static_cast<size_t>(f) * m * m,
                                                     static_cast<c64*>(work) + static_cast<size_t>(f) * mp * mp,
                                                     static_cast<c64*>(basis) + static_cast<size_t>(f) * m * k,
                                                     eig + static_cast<size_t>(f) * k, status + f, m, k, s);
                if (e != cudaSuccess) return e;
            }
            return cudaSuccess;
        }
        return launch_jac<double>(R, nullptr, work, basis, eig, status, frames, m, k, of, s);
    }
    if (!work32) return cudaErrorInvalidValue;
    cudaError_t e = launch_jac<float>(R, nullptr, work32, basis, eig, status, frames, m, k, of | jac::kModeNoStatus, s);
    if (e != cudaSuccess) return e;
    return launch_jac<double>(R, work32, work, basis, eig, status, frames, m, k, of | jac::kModePolish, s);
}

template cudaError_t fm_launch_jacobi_eig<float>(const void*, void*, void*, double*, int32_t*, int, int, int,
                                                 cudaStream_t, int, void*);
template cudaError_t fm_launch_jacobi_eig<double>(const void*, void*, void*, double*, int32_t*, int, int, int,
                                                  cudaStream_t, int, void*);
