// Size-general fp64 small-matrix path for the single-matrix facade: the reference API accepts any M, K < M and
// K <= p <= M (R/src/estimators.cpp:73-139, R/src/linalg.cpp:77-163), while the shared-memory kernels of the
// facade stage whole p x p / block-of-columns working sets (jacobi.cu: M <= 384, subspace.cu k_nystrom: p <= 64).
// Beyond those sizes the same algebra runs here on matrices kept in global memory (L2-resident up to M ~ 2000):
//
//   gen_jacobi        one-sided (Hestenes) Jacobi on the columns of A (optionally accumulating V, A V = U S),
//                     parallel circle ordering: the np/2 disjoint pairs of a round are rotated by one warp each
//                     across the whole GPU, one launch per round, a device flag per sweep for convergence;
//   gen_hermitian_eig hermitian_eig R/src/linalg.cpp:77-89 as jacobi.cu computes it (Gershgorin shift to PSD,
//                     power-of-two normalisation, top-K columns by norm, eigenvalues descending);
//   gen_nystrom       rank_restricted_subspace R/src/estimators.cpp:37-50 with pseudo_inverse R/src/linalg.cpp:
//                     143-163 (Jacobi SVD, cutoff p eps s1), as subspace.cu k_nystrom computes it for p <= 64.
// Only the facade (frames = 1) and the host-driven block-Lanczos loop come here; the batched plan keeps its caps.

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "fm_common.cuh"

namespace fmk {
namespace gen {

constexpr int kNT = 256;
constexpr int kNW = kNT / 32;

__device__ __forceinline__ c64 warp_sum_c(c64 v) {
    v.re = warp_sum(v.re);
    v.im = warp_sum(v.im);
    return v;
}

// One round of the circle ordering over np (even) column slots; slots >= ncols are padding (never rotate).
// Rotation as subspace.cu block_jacobi_svd: a_i' = c a_i - s conj(e) a_j, a_j' = s e a_i + c a_j.
__global__ void __launch_bounds__(kNT) k_round(c64* __restrict__ A, int rows, int lda, int ncols, int np,
                                               c64* __restrict__ V, int ldv, int vrows, int rnd, double tol,
                                               int* __restrict__ flag) {
    const int q = blockIdx.x * kNW + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (q >= np / 2) return;
    int i, j;
    if (q == 0) {
        i = rnd;
        j = np - 1;
    } else {
        i = (rnd + q) % (np - 1);
        j = (rnd - q + (np - 1)) % (np - 1);
    }
    if (i > j) {
        const int t = i;
        i = j;
        j = t;
    }
    if (j >= ncols) return;
    c64* ai = A + static_cast<size_t>(i) * lda;
    c64* aj = A + static_cast<size_t>(j) * lda;
    double al = 0.0, be = 0.0;
    c64 ga = mk(0.0, 0.0);
    for (int r = lane; r < rows; r += 32) {
        const c64 x = ai[r], y = aj[r];
        al += norm2(x);
        be += norm2(y);
        cmac_conj(ga, x, y);
    }
    al = warp_sum(al);
    be = warp_sum(be);
    ga = warp_sum_c(ga);
    const double g = sqrt(norm2(ga));
    if (g == 0.0 || !(g > tol * sqrt(al * be))) return;
    const double zeta = (be - al) / (2.0 * g);
    const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
    const double c = 1.0 / sqrt(1.0 + t * t);
    const double s = c * t;
    const c64 e = mk(ga.re / g, ga.im / g);
    auto rot = [&](c64* xi, c64* xj, int n) {
        for (int r = lane; r < n; r += 32) {
            const c64 x = xi[r], y = xj[r];
            const c64 ey = mk(e.re * y.re + e.im * y.im, e.re * y.im - e.im * y.re);  // conj(e) y
            const c64 ex = mk(e.re * x.re - e.im * x.im, e.re * x.im + e.im * x.re);  // e x
            xi[r] = mk(c * x.re - s * ey.re, c * x.im - s * ey.im);
            xj[r] = mk(s * ex.re + c * y.re, s * ex.im + c * y.im);
        }
    };
    rot(ai, aj, rows);
    if (V) rot(V + static_cast<size_t>(i) * ldv, V + static_cast<size_t>(j) * ldv, vrows);
    if (lane == 0) *flag = 1;
}

__global__ void k_identity(c64* __restrict__ V, int n, int ldv) {
    const size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= static_cast<size_t>(n) * ldv) return;
    const int c = static_cast<int>(e / ldv), r = static_cast<int>(e % ldv);
    V[e] = mk(r == c ? 1.0 : 0.0, 0.0);
}

// sig[c] = ||a_c|| (warp per column)
__global__ void __launch_bounds__(kNT) k_colnorm(const c64* __restrict__ A, int rows, int lda, int ncols,
                                                 double* __restrict__ sig) {
    const int c = blockIdx.x * kNW + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (c >= ncols) return;
    double s = 0.0;
    for (int r = lane; r < rows; r += 32) s += norm2(A[static_cast<size_t>(c) * lda + r]);
    s = warp_sum(s);
    if (lane == 0) sig[c] = sqrt(s);
}

// order[0..cnt) = indices of the cnt largest sig (descending; ties keep the lower index), one CTA. sig >= 0 is
// consumed (selected entries set to -1).
__global__ void __launch_bounds__(1024) k_select(double* __restrict__ sig, int n, int cnt, int* __restrict__ order) {
    __shared__ double sv[32];
    __shared__ int si[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int q = 0; q < cnt; ++q) {
        double bv = -2.0;
        int bi = 0x7fffffff;
        for (int c = threadIdx.x; c < n; c += blockDim.x) {
            const double v = sig[c];
            if (v > bv) {  // ascending c per thread: first max kept
                bv = v;
                bi = c;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > bv || (ov == bv && oi < bi)) {
                bv = ov;
                bi = oi;
            }
        }
        if (lane == 0) {
            sv[warp] = bv;
            si[warp] = bi;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double v = sv[0];
            int ix = si[0];
            for (int w = 1; w < nw; ++w)
                if (sv[w] > v || (sv[w] == v && si[w] < ix)) {
                    v = sv[w];
                    ix = si[w];
                }
            order[q] = ix;
            sig[ix] = -1.0;
        }
        __syncthreads();
    }
}

// Gershgorin shift mu = max(0, -min_i (R_ii - sum_{j != i} |R_ij|)) and max_i |R_ii| + mu (row-major Hermitian R),
// warp per row; sc[0] = mu, sc[1] = max |R_ii| (mu added by k_load).
__global__ void __launch_bounds__(kNT) k_shift(const c64* __restrict__ R, int m, double* __restrict__ sc) {
    const int c = blockIdx.x * kNW + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (c >= m) return;
    double off = 0.0;
    for (int r = lane; r < m; r += 32)
        if (r != c) off += sqrt(norm2(R[static_cast<size_t>(c) * m + r]));
    off = warp_sum(off);
    if (lane == 0) {
        const double d = R[static_cast<size_t>(c) * m + c].re;
        const double lo = d - off;
        if (lo < 0.0) atomicMax(reinterpret_cast<unsigned long long*>(&sc[0]), __double_as_longlong(-lo));
        const double a = fabs(d);
        if (a > 0.0 && a < 1e300) atomicMax(reinterpret_cast<unsigned long long*>(&sc[1]), __double_as_longlong(a));
    }
}

// A[c][r] = 2^-e conj(R[c][r]) (+ mu on the diagonal): column-major R + mu I, normalised so that max_c |R_cc| + mu
// lies in [1, 4) (as jacobi.cu).
__global__ void k_load(const c64* __restrict__ R, int m, const double* __restrict__ sc, c64* __restrict__ A) {
    const size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= static_cast<size_t>(m) * m) return;
    const double mu = sc[0], dmax = sc[1] + mu;
    const double nsc = dmax > 0.0 ? pow2_inv_sqrt_scale(dmax * dmax) : 1.0;
    const int c = static_cast<int>(e / m), r = static_cast<int>(e % m);
    c64 v = conj(R[e]);
    if (c == r) v.re += mu;
    A[e] = mk(v.re * nsc, v.im * nsc);
}

// basis[:, q] = a_{order[q]} / sig, lambda_q = sig / nsc - mu (clamp_nonnegative tolerance of jacobi.cu)
__global__ void k_eig_out(const c64* __restrict__ A, int m, int k, const int* __restrict__ order,
                          const double* __restrict__ sig, const double* __restrict__ sc, c64* __restrict__ basis,
                          double* __restrict__ eig) {
    const size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= static_cast<size_t>(m) * k) return;
    const int q = static_cast<int>(e / m), r = static_cast<int>(e % m);
    const int c = order[q];
    const double s = sig[c];
    const double inv = s > 0.0 ? 1.0 / s : 0.0;
    const c64 a = A[static_cast<size_t>(c) * m + r];
    basis[e] = mk(a.re * inv, a.im * inv);
    if (r == 0) {
        const double mu = sc[0], dmax = sc[1] + mu;
        const double nsc = dmax > 0.0 ? pow2_inv_sqrt_scale(dmax * dmax) : 1.0;
        double lam = s / nsc - mu;
        if (lam < 0.0 && lam >= -1e-10) lam = 0.0;
        eig[q] = lam;
    }
}

// C (rows x cols, column-major ldc) = op(A) op(B), op = N or H; thread per entry, fp64 complex.
__global__ void k_zgemm(const c64* __restrict__ A, int lda, bool ha, const c64* __restrict__ B, int ldb, bool hb,
                        c64* __restrict__ C, int ldc, int rows, int cols, int inner) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
    if (i >= rows) return;
    c64 acc = mk(0.0, 0.0);
    for (int c = 0; c < inner; ++c) {
        const c64 a = ha ? conj(A[static_cast<size_t>(i) * lda + c]) : A[static_cast<size_t>(c) * lda + i];
        const c64 b = hb ? conj(B[static_cast<size_t>(c) * ldb + j]) : B[static_cast<size_t>(j) * ldb + c];
        cmac(acc, a, b);
    }
    C[static_cast<size_t>(j) * ldc + i] = acc;
}

// W(i, j) = sum_c [s_c > cutoff] v(i, c) conj(a(j, c)) / s_c^2 (pinv of H from H V = U S, u = a / s),
// cutoff = p eps s1 with s1 = max s (subspace.cu k_nystrom).
__global__ void k_pinv(const c64* __restrict__ Aa, const c64* __restrict__ Vv, const double* __restrict__ sig,
                       const double* __restrict__ s1p, int p, double eps, c64* __restrict__ W) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
    if (i >= p) return;
    const double s1 = *s1p;
    const double cutoff = static_cast<double>(p) * eps * s1;
    c64 acc = mk(0.0, 0.0);
    if (s1 > 0.0)
        for (int c = 0; c < p; ++c) {
            const double s = sig[c];
            if (s > cutoff) {
                const c64 vi = Vv[static_cast<size_t>(c) * p + i];
                const c64 aj = Aa[static_cast<size_t>(c) * p + j];
                const double w = 1.0 / (s * s);
                acc.re += w * (vi.re * aj.re + vi.im * aj.im);
                acc.im += w * (vi.im * aj.re - vi.re * aj.im);
            }
        }
    W[static_cast<size_t>(j) * p + i] = acc;
}

__global__ void k_max(const double* __restrict__ v, int n, double* __restrict__ out) {
    __shared__ double s[32];
    double m = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, v[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) m = fmax(m, s[w]);
        *out = fmax(m, s[0]);
    }
}

// basis[:, q] = Q a_{order[q]} / sig (Q: m x p column-major), lambda_q = sig (clamped)
__global__ void k_nys_out(const c64* __restrict__ Q, const c64* __restrict__ Aa, int m, int p, int k,
                          const int* __restrict__ order, const double* __restrict__ sig, c64* __restrict__ basis,
                          double* __restrict__ eig) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x, q = blockIdx.y;
    if (r >= m) return;
    const int c = order[q];
    const double s = sig[c];
    const double inv = s > 0.0 ? 1.0 / s : 0.0;
    c64 acc = mk(0.0, 0.0);
    for (int u = 0; u < p; ++u) cmac(acc, Q[static_cast<size_t>(u) * m + r], Aa[static_cast<size_t>(c) * p + u]);
    basis[static_cast<size_t>(q) * m + r] = mk(acc.re * inv, acc.im * inv);
    if (r == 0) {
        double lam = s;
        if (lam < 0.0 && lam >= -1e-10) lam = 0.0;
        eig[q] = lam;
    }
}

__global__ void k_set_status(int32_t* status, int32_t bits) { atomicOr(status, bits); }

}  // namespace gen
}  // namespace fmk

using namespace fmk;

namespace {

// Run sweeps until one performs no rotation (cap 60). flag: one device int of scratch.
cudaError_t gen_jacobi(c64* A, int rows, int lda, int ncols, c64* V, int ldv, double tol, int* flag, bool* converged,
                       cudaStream_t s) {
    const int np = ncols + (ncols & 1);
    const unsigned blocks = static_cast<unsigned>((np / 2 + gen::kNW - 1) / gen::kNW);
    *converged = false;
    if (V) {
        const size_t n = static_cast<size_t>(ncols) * ldv;
        gen::k_identity<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(V, ncols, ldv);
    }
    for (int sweep = 0; sweep < 60; ++sweep) {
        cudaError_t e = cudaMemsetAsync(flag, 0, sizeof(int), s);
        if (e != cudaSuccess) return e;
        for (int rnd = 0; rnd < np - 1; ++rnd)
            gen::k_round<<<blocks, gen::kNT, 0, s>>>(A, rows, lda, ncols, np, V, ldv, ncols, rnd, tol, flag);
        int h = 1;
        e = cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return e;
        if (h == 0) {
            *converged = true;
            break;
        }
    }
    return cudaGetLastError();
}

template <typename T>
struct Scratch {
    T* p = nullptr;
    cudaError_t alloc(size_t n) { return cudaMalloc(reinterpret_cast<void**>(&p), sizeof(T) * (n ? n : 1)); }
    ~Scratch() {
        if (p) cudaFree(p);
    }
};

}  // namespace

// Top-K eigenpairs of the row-major Hermitian m x m R (complex128) for any m: basis m x k column-major, eigenvalues
// descending (R/src/linalg.cpp:77-89 through the same Hestenes formulation as jacobi.cu). work >= m * m complex128.
cudaError_t fm_gen_hermitian_eig(const void* R, void* work, void* basis, double* eig, int32_t* status, int m, int k,
                                 cudaStream_t s) {
    if (m < 1 || k < 1 || k > m) return cudaErrorInvalidValue;
    Scratch<double> sc, sig;
    Scratch<int> order, flag;
    cudaError_t e = sc.alloc(2);
    if (e == cudaSuccess) e = sig.alloc(m);
    if (e == cudaSuccess) e = order.alloc(k);
    if (e == cudaSuccess) e = flag.alloc(1);
    if (e == cudaSuccess) e = cudaMemsetAsync(sc.p, 0, 2 * sizeof(double), s);
    if (e != cudaSuccess) return e;
    auto Rp = static_cast<const c64*>(R);
    auto A = static_cast<c64*>(work);
    const unsigned wblocks = static_cast<unsigned>((m + gen::kNW - 1) / gen::kNW);
    gen::k_shift<<<wblocks, gen::kNT, 0, s>>>(Rp, m, sc.p);
    const size_t mm = static_cast<size_t>(m) * m;
    gen::k_load<<<static_cast<unsigned>((mm + 255) / 256), 256, 0, s>>>(Rp, m, sc.p, A);
    bool conv = false;
    const double tol = 4.0 * 2.220446049250313e-16 * sqrt(static_cast<double>(m));
    e = gen_jacobi(A, m, m, m, nullptr, 0, tol, flag.p, &conv, s);
    if (e != cudaSuccess) return e;
    gen::k_colnorm<<<wblocks, gen::kNT, 0, s>>>(A, m, m, m, sig.p);
    Scratch<double> sig2;
    e = sig2.alloc(m);
    if (e == cudaSuccess) e = cudaMemcpyAsync(sig2.p, sig.p, sizeof(double) * m, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return e;
    gen::k_select<<<1, 1024, 0, s>>>(sig2.p, m, k, order.p);
    const size_t mk_ = static_cast<size_t>(m) * k;
    gen::k_eig_out<<<static_cast<unsigned>((mk_ + 255) / 256), 256, 0, s>>>(A, m, k, order.p, sig.p, sc.p,
                                                                            static_cast<c64*>(basis), eig);
    if (!conv && status) gen::k_set_status<<<1, 1, 0, s>>>(status, kFrameNoConv);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // scratch freed on return
    return e;
}

// Nystrom tail of one frame for any p (subspace.cu k_nystrom's algebra on global memory): V, C m x p column-major
// (fast2: H = V^H C) or H p x p given (fast1); work[1] = Q (m x p), Rt p x p; basis m x k, eig k.
cudaError_t fm_gen_nystrom(const void* V, const void* C, const void* H, const void* work, const void* Rt, void* basis,
                           double* eig, int32_t* status, int m, int p, int k, bool fast2, cudaStream_t s) {
    if (p < 1 || k < 1 || k > p) return cudaErrorInvalidValue;
    const size_t pp = static_cast<size_t>(p) * p;
    Scratch<c64> a, v, w, t;
    Scratch<double> sig, sig2, s1;
    Scratch<int> order, flag;
    cudaError_t e = a.alloc(pp);
    if (e == cudaSuccess) e = v.alloc(pp);
    if (e == cudaSuccess) e = w.alloc(pp);
    if (e == cudaSuccess) e = t.alloc(pp);
    if (e == cudaSuccess) e = sig.alloc(p);
    if (e == cudaSuccess) e = sig2.alloc(p);
    if (e == cudaSuccess) e = s1.alloc(1);
    if (e == cudaSuccess) e = order.alloc(p);
    if (e == cudaSuccess) e = flag.alloc(1);
    if (e != cudaSuccess) return e;
    const dim3 gp(static_cast<unsigned>((p + 127) / 128), static_cast<unsigned>(p));
    if (fast2)
        gen::k_zgemm<<<gp, 128, 0, s>>>(static_cast<const c64*>(V), m, true, static_cast<const c64*>(C), m, false, a.p,
                                        p, p, p, m);
    else
        e = cudaMemcpyAsync(a.p, H, sizeof(c64) * pp, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return e;
    const double tol = 8.0 * 2.220446049250313e-16 * p;  // block_jacobi_svd's rotation threshold
    bool ok1 = false, ok2 = false;
    e = gen_jacobi(a.p, p, p, p, v.p, p, tol, flag.p, &ok1, s);
    if (e != cudaSuccess) return e;
    const unsigned wblocks = static_cast<unsigned>((p + gen::kNW - 1) / gen::kNW);
    gen::k_colnorm<<<wblocks, gen::kNT, 0, s>>>(a.p, p, p, p, sig.p);
    gen::k_max<<<1, 1024, 0, s>>>(sig.p, p, s1.p);
    gen::k_pinv<<<gp, 128, 0, s>>>(a.p, v.p, sig.p, s1.p, p, 2.220446049250313e-16, w.p);
    auto Rtp = static_cast<const c64*>(Rt);
    gen::k_zgemm<<<gp, 128, 0, s>>>(Rtp, p, false, w.p, p, false, t.p, p, p, p, p);  // T = Rt W
    gen::k_zgemm<<<gp, 128, 0, s>>>(t.p, p, false, Rtp, p, true, a.p, p, p, p, p);   // B' = T Rt^H
    e = gen_jacobi(a.p, p, p, p, nullptr, 0, tol, flag.p, &ok2, s);
    if (e != cudaSuccess) return e;
    gen::k_colnorm<<<wblocks, gen::kNT, 0, s>>>(a.p, p, p, p, sig.p);
    e = cudaMemcpyAsync(sig2.p, sig.p, sizeof(double) * p, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return e;
    gen::k_select<<<1, 1024, 0, s>>>(sig2.p, p, k, order.p);
    const c64* Q = static_cast<const c64*>(work) + static_cast<size_t>(p) * m;
    const dim3 gb(static_cast<unsigned>((m + 127) / 128), static_cast<unsigned>(k));
    gen::k_nys_out<<<gb, 128, 0, s>>>(Q, a.p, m, p, k, order.p, sig.p, static_cast<c64*>(basis), eig);
    if (!(ok1 && ok2) && status) gen::k_set_status<<<1, 1, 0, s>>>(status, kFrameNoConv);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    return e;
}
