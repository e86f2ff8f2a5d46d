// Exact-algebra fallback of the batched Nystrom tail for frames the fast path flags (kFrameNoConv): a singular
// or near-singular H = V^H C (fast2) / S(I, I) (fast1), a numerically rank-deficient C, or a Jacobi sweep cap.
//
// The fast path (smallmat.cu k_small_warp) inverts H through its Cholesky factor, which has no answer for a
// singular H. The reference never fails there: pseudo_inverse truncates (R/src/linalg.cpp:143-163, "pinv never
// aborts", R/src/estimators.cpp:97) and R/tests/test_estimators.cpp:117-126 pins that. This kernel restates the
// reference algebra with Hermitian eigendecompositions in fp64:
//   W = pinv(H)                      H = Q diag(l) Q^H, 1 / l_i kept for |l_i| > p eps |l|_max (linalg.cpp:143-163)
//   thin_svd(C) = U_c S_c V_c^H      from G = C^H C = V_c S_c^2 V_c^H (linalg.cpp:108-125)
//   B = S_c V_c^H W V_c S_c          (rank_restricted_subspace, estimators.cpp:37-50)
//   B = U_B S_B U_B^H                (thin_svd(B): B is Hermitian, singular values |l_B|, descending)
//   basis = U_c U_B(:, 1:K) = C T,   T = V_c S_c^+ U_B(:, 1:K);  eigenvalues = S_B(1:K) (clamp, :25-31)
// The cut-offs use the epsilon of the batch data (complex64 R, fp32-level C and H): eigen-directions below
// p eps_32 of the largest are representation noise of the fp32 data and are dropped, as the reference drops its
// fp64 noise at p eps_64. Directions of C with s_j <= p eps_32 s_max get S_c^+ = 0 (their rows of B vanish).
//
// One CTA per frame (grid-stride over frames); unflagged frames return at once. The p x p work matrices live in
// a global scratch slice per CTA (this path is rare; L1 / L2 hold it). Cyclic two-sided complex Jacobi with
// round-robin parallel ordering: the p / 2 disjoint rotations of a round are applied to columns, then to rows.

#include <cuda_runtime.h>

#include <cstdint>

#include "fm_common.cuh"

namespace fmk {
namespace fbk {

constexpr int kT = 128;
constexpr int kMaxP = 64;

// Eigen-decomposition of the Hermitian n x n A (column-major, ld n) in place: A -> diag(l), V <- eigenvectors
// (V initialised to I here). rot: scratch for kMaxP / 2 rotations. Returns sweeps (0: cap hit).
__device__ int herm_jacobi(c64* A, c64* V, int n, double* rc, double* rs, c64* re, int* pi, int* pj) {
    const int tid = threadIdx.x;
    for (int e = tid; e < n * n; e += kT) V[e] = mk((e % n) == (e / n) ? 1.0 : 0.0, 0.0);
    const int np = (n + 1) & ~1;  // round-robin over an even count (a dummy index when n is odd)
    __shared__ double s_off, s_dia;
    __syncthreads();
    for (int sweep = 1; sweep <= 60; ++sweep) {
        // convergence: off-diagonal Frobenius norm vs diagonal
        if (tid == 0) {
            double off = 0.0, dia = 0.0;
            for (int j = 0; j < n; ++j)
                for (int i = 0; i < n; ++i) {
                    const double v = norm2(A[j * n + i]);
                    if (i == j) dia += v;
                    else off += v;
                }
            s_off = off;
            s_dia = dia;
        }
        __syncthreads();
        if (!(s_off > 1e-30 * s_dia) || s_off == 0.0) return sweep;
        for (int rnd = 0; rnd < np - 1; ++rnd) {
            // pairs of this round: slot 0 = (rnd, np - 1), slot s = (rnd + s, rnd - s) mod (np - 1)
            if (tid < np / 2) {
                const int sl = tid;
                int i = (rnd + sl) % (np - 1), j = (rnd - sl + (np - 1)) % (np - 1);
                if (sl == 0) j = np - 1;
                if (i > j) {
                    const int t = i;
                    i = j;
                    j = t;
                }
                pi[sl] = i;
                pj[sl] = j;
                rc[sl] = 1.0;
                rs[sl] = 0.0;
                re[sl] = mk(1.0, 0.0);
                if (j < n) {
                    const c64 b = A[j * n + i];  // A(i, j)
                    const double ab = sqrt(norm2(b));
                    const double a = A[i * n + i].re, d = A[j * n + j].re;
                    if (ab > 1e-300 && ab > 1e-17 * sqrt(fabs(a * d))) {
                        const double tau = (d - a) / (2.0 * ab);
                        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                        const double c = 1.0 / sqrt(1.0 + t * t);
                        rc[sl] = c;
                        rs[sl] = t * c;
                        re[sl] = mk(b.re / ab, b.im / ab);  // e^{i phi}
                    }
                }
            }
            __syncthreads();
            // columns: A <- A J, V <- V J, J = [[c, s e], [-s conj(e), c]] on (i, j)
            for (int e = tid; e < (np / 2) * n; e += kT) {
                const int sl = e / n, r = e % n;
                const int i = pi[sl], j = pj[sl];
                if (j >= n || rs[sl] == 0.0) continue;
                const double c = rc[sl], s = rs[sl];
                const c64 ph = re[sl];
                for (int w = 0; w < 2; ++w) {
                    c64* M = w ? V : A;
                    const c64 x = M[i * n + r], y = M[j * n + r];
                    const c64 sey = s * (conj(ph) * y);
                    const c64 sex = s * (ph * x);
                    M[i * n + r] = mk(c * x.re - sey.re, c * x.im - sey.im);
                    M[j * n + r] = mk(sex.re + c * y.re, sex.im + c * y.im);
                }
            }
            __syncthreads();
            // rows: A <- J^H A
            for (int e = tid; e < (np / 2) * n; e += kT) {
                const int sl = e / n, col = e % n;
                const int i = pi[sl], j = pj[sl];
                if (j >= n || rs[sl] == 0.0) continue;
                const double c = rc[sl], s = rs[sl];
                const c64 ph = re[sl];
                const c64 x = A[col * n + i], y = A[col * n + j];
                const c64 sey = s * (ph * y);
                const c64 sex = s * (conj(ph) * x);
                A[col * n + i] = mk(c * x.re - sey.re, c * x.im - sey.im);
                A[col * n + j] = mk(sex.re + c * y.re, sex.im + c * y.im);
            }
            __syncthreads();
        }
        __syncthreads();
    }
    return 0;
}

// Descending order of |d_i| (ties: lower index first) -> ord.
__device__ void order_desc_abs(const double* d, int n, int* ord) {
    for (int i = threadIdx.x; i < n; i += kT) {
        int rank = 0;
        for (int q = 0; q < n; ++q)
            if (q != i && (fabs(d[q]) > fabs(d[i]) || (fabs(d[q]) == fabs(d[i]) && q < i))) ++rank;
        ord[rank] = i;
    }
    __syncthreads();
}

// C, V: frames x p x m complex64 column-major (C(:, q) contiguous). Hin (fast1, V == nullptr): frames x p x p
// complex128 column-major S(I, I). basis: frames x K x m complex128 column-major; eig: frames x K.
__global__ void __launch_bounds__(kT) k_final_fallback(const c32* __restrict__ C, const c32* __restrict__ Vb,
                                                       const c64* __restrict__ Hin, c64* __restrict__ basis,
                                                       double* __restrict__ eig, int32_t* __restrict__ status,
                                                       c64* __restrict__ scratch, int frames, int m, int p, int k) {
    __shared__ double rc[kMaxP / 2], rs[kMaxP / 2];
    __shared__ c64 re[kMaxP / 2];
    __shared__ int pi[kMaxP / 2], pj[kMaxP / 2];
    __shared__ double sg[kMaxP], lh[kMaxP], lb[kMaxP], sinv[kMaxP];
    __shared__ int ord[kMaxP];
    __shared__ int s_ok;
    const int tid = threadIdx.x;
    const int pp = p * p;
    c64* A = scratch + static_cast<size_t>(blockIdx.x) * 4 * kMaxP * kMaxP;
    c64* Vm = A + pp;
    c64* X = Vm + pp;  // V_c, later T
    c64* Y = X + pp;   // W
    const double eps = static_cast<double>(p) * eps_of<float>::value;
    // one parallel pass over this CTA's status words first: a CTA without flagged frames exits after one load
    int any = 0;
    for (int f = blockIdx.x + tid * gridDim.x; f < frames; f += kT * gridDim.x) any |= status[f] & kFrameNoConv;
    if (!__syncthreads_or(any)) return;
    for (int f = blockIdx.x; f < frames; f += gridDim.x) {
        if (!(status[f] & kFrameNoConv)) continue;  // block-uniform
        const c32* Cf = C + static_cast<size_t>(f) * m * p;
        // ---- G = C^H C -> V_c, s_c
        for (int e = tid; e < pp; e += kT) {
            const int i = e % p, j = e / p;
            c64 acc = mk(0.0, 0.0);
            for (int r = 0; r < m; ++r) cmac_conj(acc, to64(Cf[static_cast<size_t>(i) * m + r]), to64(Cf[static_cast<size_t>(j) * m + r]));
            A[e] = acc;
        }
        __syncthreads();
        for (int e = tid; e < pp; e += kT) {  // exactly Hermitian
            const int i = e % p, j = e / p;
            if (i < j) {
                const c64 a = A[j * p + i], b = A[i * p + j];
                const c64 h = mk(0.5 * (a.re + b.re), 0.5 * (a.im - b.im));
                A[j * p + i] = h;
                A[i * p + j] = conj(h);
            } else if (i == j) {
                A[e].im = 0.0;
            }
        }
        __syncthreads();
        int sw = herm_jacobi(A, Vm, p, rc, rs, re, pi, pj);
        for (int i = tid; i < p; i += kT) sg[i] = sqrt(fmax(A[i * p + i].re, 0.0));
        for (int e = tid; e < pp; e += kT) X[e] = Vm[e];
        __syncthreads();
        if (tid == 0) {
            double smax = 0.0;
            for (int i = 0; i < p; ++i) smax = fmax(smax, sg[i]);
            for (int i = 0; i < p; ++i) sinv[i] = sg[i] > eps * smax ? 1.0 / sg[i] : 0.0;
            s_ok = sw > 0;
        }
        __syncthreads();
        // ---- H (Hermitian part) -> Q, l; W = Q diag(l^+) Q^H into Y
        if (Vb) {
            const c32* Vf = Vb + static_cast<size_t>(f) * m * p;
            for (int e = tid; e < pp; e += kT) {
                const int i = e % p, j = e / p;
                c64 acc = mk(0.0, 0.0);
                for (int r = 0; r < m; ++r) cmac_conj(acc, to64(Vf[static_cast<size_t>(i) * m + r]), to64(Cf[static_cast<size_t>(j) * m + r]));
                A[e] = acc;
            }
        } else {
            const c64* Hf = Hin + static_cast<size_t>(f) * pp;
            for (int e = tid; e < pp; e += kT) A[e] = Hf[e];
        }
        __syncthreads();
        for (int e = tid; e < pp; e += kT) {
            const int i = e % p, j = e / p;
            if (i < j) {
                const c64 a = A[j * p + i], b = A[i * p + j];
                const c64 h = mk(0.5 * (a.re + b.re), 0.5 * (a.im - b.im));
                A[j * p + i] = h;
                A[i * p + j] = conj(h);
            } else if (i == j) {
                A[e].im = 0.0;
            }
        }
        __syncthreads();
        sw = herm_jacobi(A, Vm, p, rc, rs, re, pi, pj);
        for (int i = tid; i < p; i += kT) lh[i] = A[i * p + i].re;
        __syncthreads();
        if (tid == 0) {
            double lmax = 0.0;
            for (int i = 0; i < p; ++i) lmax = fmax(lmax, fabs(lh[i]));
            for (int i = 0; i < p; ++i) lh[i] = fabs(lh[i]) > eps * lmax ? 1.0 / lh[i] : 0.0;
            s_ok = s_ok && sw > 0;
        }
        __syncthreads();
        for (int e = tid; e < pp; e += kT) {  // W(i, j) = sum_q Q(i, q) l_q^+ conj(Q(j, q))
            const int i = e % p, j = e / p;
            c64 acc = mk(0.0, 0.0);
            for (int q = 0; q < p; ++q) {
                const double w = lh[q];
                if (w != 0.0) cmac(acc, w * Vm[q * p + i], conj(Vm[q * p + j]));
            }
            Y[e] = acc;
        }
        __syncthreads();
        // ---- B = S V_c^H W V_c S: Vm <- W V_c, then A <- V_c^H Vm scaled
        for (int e = tid; e < pp; e += kT) {
            const int i = e % p, j = e / p;
            c64 acc = mk(0.0, 0.0);
            for (int q = 0; q < p; ++q) cmac(acc, Y[q * p + i], X[j * p + q]);
            Vm[e] = acc;
        }
        __syncthreads();
        for (int e = tid; e < pp; e += kT) {
            const int i = e % p, j = e / p;
            c64 acc = mk(0.0, 0.0);
            for (int q = 0; q < p; ++q) cmac_conj(acc, X[i * p + q], Vm[j * p + q]);
            A[e] = (sg[i] * sg[j]) * acc;
        }
        __syncthreads();
        for (int e = tid; e < pp; e += kT) {
            const int i = e % p, j = e / p;
            if (i < j) {
                const c64 a = A[j * p + i], b = A[i * p + j];
                const c64 h = mk(0.5 * (a.re + b.re), 0.5 * (a.im - b.im));
                A[j * p + i] = h;
                A[i * p + j] = conj(h);
            } else if (i == j) {
                A[e].im = 0.0;
            }
        }
        __syncthreads();
        sw = herm_jacobi(A, Vm, p, rc, rs, re, pi, pj);
        for (int i = tid; i < p; i += kT) lb[i] = A[i * p + i].re;
        __syncthreads();
        order_desc_abs(lb, p, ord);
        // ---- T = V_c S^+ U_B(:, ord[0..K)) into Y (p x K), eigenvalues
        for (int e = tid; e < p * k; e += kT) {
            const int i = e % p, kk = e / p, col = ord[kk];
            c64 acc = mk(0.0, 0.0);
            for (int q = 0; q < p; ++q) cmac(acc, sinv[q] * X[q * p + i], Vm[col * p + q]);
            Y[kk * p + i] = acc;
        }
        for (int kk = tid; kk < k; kk += kT) {
            double v = fabs(lb[ord[kk]]);
            eig[static_cast<size_t>(f) * k + kk] = v;
        }
        __syncthreads();
        // ---- basis = C T (fp64 accumulation)
        c64* Bf = basis + static_cast<size_t>(f) * m * k;
        for (int e = tid; e < m * k; e += kT) {
            const int r = e % m, kk = e / m;
            c64 acc = mk(0.0, 0.0);
            for (int q = 0; q < p; ++q) cmac(acc, to64(Cf[static_cast<size_t>(q) * m + r]), Y[kk * p + q]);
            Bf[static_cast<size_t>(kk) * m + r] = acc;
        }
        if (tid == 0) {
            if (s_ok && sw > 0) atomicAnd(&status[f], ~static_cast<int32_t>(kFrameNoConv));
        }
        __syncthreads();
    }
}

}  // namespace fbk
}  // namespace fmk

// Scratch bytes for `ctas` CTAs of k_final_fallback.
size_t fm_final_fallback_scratch_bytes(int ctas) {
    return sizeof(fmk::c64) * 4 * fmk::fbk::kMaxP * fmk::fbk::kMaxP * static_cast<size_t>(ctas);
}
int fm_final_fallback_ctas() { return 148; }

cudaError_t fm_launch_final_fallback(const void* C, const void* V, const void* H, void* basis, double* eig,
                                     int32_t* status, void* scratch, int frames, int m, int p, int k,
                                     cudaStream_t s) {
    if (p < 1 || p > fmk::fbk::kMaxP || k > p || frames < 1 || !scratch) return cudaErrorInvalidValue;
    const int grid = frames < fm_final_fallback_ctas() ? frames : fm_final_fallback_ctas();
    fmk::fbk::k_final_fallback<<<grid, fmk::fbk::kT, 0, s>>>(
        static_cast<const fmk::c32*>(C), static_cast<const fmk::c32*>(V), static_cast<const fmk::c64*>(H),
        static_cast<fmk::c64*>(basis), eig, status, static_cast<fmk::c64*>(scratch), frames, m, p, k);
    return cudaGetLastError();
}
