// K2/K3/K4 — randomized range finder, orthonormalisation and Nystrom rank restriction,
// batched over frames (one CTA per frame for the small-matrix stages).
//
// Reference lines replaced:
//   fast_music_2            R/src/estimators.cpp:104-139  (C = S Omega, t x {V = orth(C); C = S V},
//                                                          W = pinv(V^H C), rank-restricted recovery)
//   fast_music_1            R/src/estimators.cpp:87-102   (C = S(:,I), W = pinv(S(I,I)))
//   rank_restricted_subspace R/src/estimators.cpp:37-50   (+ clamp_nonnegative :25-31)
//   qr_orthonormal          R/src/linalg.cpp:127-141      (column-pivoted Householder, Eigen rank rule)
//   pseudo_inverse          R/src/linalg.cpp:143-163      (SVD, cutoff max(r,c)*eps*sigma1)
//   thin_svd / JacobiSVD    R/src/linalg.cpp:93-125
//
// Layouts (HBM / L2): R  B x M x M complex<T> row-major (K1 output, Hermitian);
//   Omega B x M x p real<T> row-major (the reference fill order, R/src/linalg.cpp:186-190);
//   C, V  B x p x M complex<T> column-major (column c contiguous);
//   work  B x 2 x p x M complex<double> (Householder vectors | explicit Q);
//   Rt    B x p x p complex<double> (R factor with the column pivoting undone).
// Arithmetic: products C = R V in T (fp32 for the batched c64 path, fp64 for the
// reference-facade path); every small-matrix step (Householder QR, Gram H, Jacobi SVD,
// pinv, B' = Rt W Rt^H, basis U = Q Z_K) in fp64. Rank / pinv cutoffs
// use the reference formulas with the machine epsilon of the data type T.

#include <cuda_runtime.h>

#include <cstdint>

#include "fm_common.cuh"

namespace fmk {
namespace sub {

constexpr int kNT = 256;  // threads per block
constexpr int kNW = kNT / 32;

__device__ __forceinline__ int frame_of(const int32_t* map) { return map ? map[blockIdx.y] : blockIdx.y; }
__device__ __forceinline__ int frame_of_x(const int32_t* map) { return map ? map[blockIdx.x] : blockIdx.x; }

// ------------------------------------------------------------------ C = R * rhs
// C[c][m] = sum_j R[m][j] rhs[j][c] = sum_j conj(R[j][m]) rhs[j][c]  (R Hermitian; the
// conj-transpose read makes the R loads coalesced across threads m).
// rhs: REAL -> Omega row-major M x p (real); else V column-major p x M (complex).
template <typename T, int PC, bool REAL>
__global__ void __launch_bounds__(kNT) k_rmul(const cplx<T>* __restrict__ R, const T* __restrict__ omega,
                                               const cplx<T>* __restrict__ V, cplx<T>* __restrict__ C,
                                               const int32_t* __restrict__ fmap, int m, int p) {
    constexpr int JC = 32;
    __shared__ cplx<T> rhs_s[JC][PC];
    const int f = frame_of(fmap);
    const int row = blockIdx.x * kNT + threadIdx.x;
    const int c0 = blockIdx.z * PC;  // column slice (p > PC)
    const cplx<T>* Rf = R + static_cast<size_t>(f) * m * m;
    cplx<T> acc[PC];
#pragma unroll
    for (int c = 0; c < PC; ++c) acc[c] = mk<T>(0, 0);
    for (int j0 = 0; j0 < m; j0 += JC) {
        const int jn = min(JC, m - j0);
        __syncthreads();
        for (int e = threadIdx.x; e < JC * PC; e += kNT) {
            const int jj = e / PC, c = e % PC;
            cplx<T> v = mk<T>(0, 0);
            if (jj < jn && c0 + c < p) {
                if (REAL) {
                    v.re = omega[static_cast<size_t>(f) * m * p + static_cast<size_t>(j0 + jj) * p + c0 + c];
                } else {
                    v = V[static_cast<size_t>(f) * m * p + static_cast<size_t>(c0 + c) * m + j0 + jj];
                }
            }
            rhs_s[jj][c] = v;
        }
        __syncthreads();
        if (row < m) {
            const cplx<T>* col = Rf + static_cast<size_t>(j0) * m + row;
            // batches of 8 independent R loads in flight per thread before the MACs
            for (int jj = 0; jj < jn; jj += 8) {
                cplx<T> r[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) r[u] = jj + u < jn ? col[static_cast<size_t>(jj + u) * m] : mk<T>(0, 0);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
#pragma unroll
                    for (int c = 0; c < PC; ++c) {
                        if (REAL) {
                            acc[c].re = fma(r[u].re, rhs_s[jj + u][c].re, acc[c].re);
                            acc[c].im = fma(-r[u].im, rhs_s[jj + u][c].re, acc[c].im);
                        } else {
                            cmac_conj(acc[c], r[u], rhs_s[jj + u][c]);
                        }
                    }
                }
            }
        }
    }
    if (row < m) {
        cplx<T>* Cf = C + static_cast<size_t>(f) * m * p;
#pragma unroll
        for (int c = 0; c < PC; ++c)
            if (c0 + c < p) Cf[static_cast<size_t>(c0 + c) * m + row] = acc[c];
    }
}

// ------------------------------------------------------------------ fast1 gather
// C = R(:, I) (column-major p x M), H = R(I, I) (p x p, fp64).
template <typename T>
__global__ void __launch_bounds__(kNT) k_gather(const cplx<T>* __restrict__ R, const int32_t* __restrict__ idx,
                                                 cplx<T>* __restrict__ C, c64* __restrict__ H,
                                                 const int32_t* __restrict__ fmap, int m, int p) {
    const int f = frame_of_x(fmap);
    const cplx<T>* Rf = R + static_cast<size_t>(f) * m * m;
    const int32_t* ix = idx + static_cast<size_t>(f) * p;
    cplx<T>* Cf = C + static_cast<size_t>(f) * m * p;
    for (int e = threadIdx.x; e < m * p; e += kNT) {
        const int c = e / m, row = e % m;
        // column I_c of R: R[row][I_c] = conj(R[I_c][row]) -> coalesced read of row I_c
        Cf[static_cast<size_t>(c) * m + row] = conj(Rf[static_cast<size_t>(ix[c]) * m + row]);
    }
    c64* Hf = H + static_cast<size_t>(f) * p * p;
    for (int e = threadIdx.x; e < p * p; e += kNT) {
        const int i = e % p, j = e / p;  // column-major H[j][i] = H(i, j)
        Hf[static_cast<size_t>(j) * p + i] = to64(Rf[static_cast<size_t>(ix[i]) * m + ix[j]]);
    }
}

// ------------------------------------------------------------------ block helpers
__device__ __forceinline__ c64 warp_sum_c(c64 v) {
    v.re = warp_sum(v.re);
    v.im = warp_sum(v.im);
    return v;
}

// ------------------------------------------------------------------ pivoted Householder QR
// R/src/linalg.cpp:127-141 (ColPivHouseholderQR + rank()). One CTA per frame, fp64.
// Column-major A = work[f][0] (p x M), explicit Q = work[f][1]. Warp w owns columns
// j == w (mod 8) for the reductions and the trailing updates.
// OUT: MODE 0 -> V (T, column-major) for the power iteration;
//      MODE 1 -> Q (fp64, in work[f][1]) and Rt (p x p, pivoting undone) for the Nystrom tail.
template <typename T, int MODE>
__global__ void __launch_bounds__(kNT) k_qr(const cplx<T>* __restrict__ Cin, c64* __restrict__ work,
                                             cplx<T>* __restrict__ Vout, c64* __restrict__ Rt,
                                             int32_t* __restrict__ status, int32_t* __restrict__ defcol,
                                             const int32_t* __restrict__ fmap, int m, int p,
                                             int32_t* __restrict__ rank_out = nullptr) {
    extern __shared__ uint8_t qsm[];  // p entries each (any p: 36 p bytes of dynamic shared memory)
    c64* rdiag = reinterpret_cast<c64*>(qsm);
    double* nrm2 = reinterpret_cast<double*>(rdiag + p);
    double* tau = nrm2 + p;
    int* perm = reinterpret_cast<int*>(tau + p);
    __shared__ int s_pivot;
    __shared__ double s_maxcol;
    const int f = frame_of_x(fmap);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    c64* A = work + static_cast<size_t>(f) * 2 * p * m;
    c64* Q = A + static_cast<size_t>(p) * m;
    const cplx<T>* Cf = Cin + static_cast<size_t>(f) * m * p;
    const double eps = eps_of<T>::value;

    // load + initial column norms
    for (int j = warp; j < p; j += kNW) {
        double s = 0.0;
        for (int r = lane; r < m; r += 32) {
            const c64 v = to64(Cf[static_cast<size_t>(j) * m + r]);
            A[static_cast<size_t>(j) * m + r] = v;
            s += norm2(v);
        }
        s = warp_sum(s);
        if (lane == 0) nrm2[j] = s;
    }
    for (int j = threadIdx.x; j < p; j += kNT) perm[j] = j;
    __syncthreads();
    if (threadIdx.x == 0) {
        double mx = 0.0;
        for (int j = 0; j < p; ++j) mx = fmax(mx, nrm2[j]);
        s_maxcol = sqrt(mx);
    }
    __syncthreads();
    const double thr_helper = (s_maxcol * eps) * (s_maxcol * eps) / static_cast<double>(m);
    int nonzero = p;  // tracked by thread 0 only

    for (int k = 0; k < p; ++k) {
        if (threadIdx.x == 0) {
            int piv = k;
            double best = nrm2[k];
            for (int j = k + 1; j < p; ++j)
                if (nrm2[j] > best) {
                    best = nrm2[j];
                    piv = j;
                }
            if (nonzero == p && best < thr_helper * static_cast<double>(m - k)) nonzero = k;
            s_pivot = piv;
            const int tp = perm[k];
            perm[k] = perm[piv];
            perm[piv] = tp;
            nrm2[piv] = nrm2[k];
            nrm2[k] = best;
        }
        __syncthreads();
        const int piv = s_pivot;
        if (piv != k) {
            for (int r = threadIdx.x; r < m; r += kNT) {
                const c64 a = A[static_cast<size_t>(k) * m + r];
                A[static_cast<size_t>(k) * m + r] = A[static_cast<size_t>(piv) * m + r];
                A[static_cast<size_t>(piv) * m + r] = a;
            }
        }
        __syncthreads();
        // Householder for x = A[k:, k]; H x = alpha e_k, alpha = -phase(x0) ||x||.
        if (threadIdx.x == 0) {
            const double xn = sqrt(fmax(nrm2[k], 0.0));
            const c64 x0 = A[static_cast<size_t>(k) * m + k];
            const double ax0 = sqrt(norm2(x0));
            if (xn == 0.0) {
                rdiag[k] = mk(0.0, 0.0);
                tau[k] = 0.0;
            } else {
                const c64 ph = ax0 > 0.0 ? mk(x0.re / ax0, x0.im / ax0) : mk(1.0, 0.0);
                rdiag[k] = mk(-ph.re * xn, -ph.im * xn);
                A[static_cast<size_t>(k) * m + k] = mk(x0.re + ph.re * xn, x0.im + ph.im * xn);  // v_k
                tau[k] = 1.0 / (xn * (xn + ax0));  // 2 / (v^H v)
            }
        }
        __syncthreads();
        const double tk = tau[k];
        const c64* v = A + static_cast<size_t>(k) * m;
        for (int j = k + 1 + warp; j < p; j += kNW) {
            c64* a = A + static_cast<size_t>(j) * m;
            c64 w = mk(0.0, 0.0);
            for (int r = k + lane; r < m; r += 32) cmac_conj(w, v[r], a[r]);
            w = warp_sum_c(w);
            double s = 0.0;
            const c64 tw = mk(tk * w.re, tk * w.im);
            for (int r = k + lane; r < m; r += 32) {
                const c64 vr = v[r];
                c64 ar = a[r];
                ar.re -= vr.re * tw.re - vr.im * tw.im;
                ar.im -= vr.re * tw.im + vr.im * tw.re;
                a[r] = ar;
                if (r > k) s += norm2(ar);
            }
            s = warp_sum(s);
            if (lane == 0) nrm2[j] = s;
        }
        __syncthreads();
    }

    // rank (Eigen ColPivHouseholderQR::rank) with the data-type epsilon
    if (threadIdx.x == 0) {
        double maxpivot = 0.0;
        for (int k = 0; k < p; ++k) maxpivot = fmax(maxpivot, sqrt(norm2(rdiag[k])));
        const double thr = maxpivot * eps * static_cast<double>(p);
        int rank = 0;
        for (int k = 0; k < nonzero; ++k) rank += sqrt(norm2(rdiag[k])) > thr ? 1 : 0;
        if (rank_out) rank_out[f] = rank;
        if (rank < p) {
            atomicOr(&status[f], kFrameRank);
            if (defcol) defcol[f] = perm[rank];
        }
    }

    // explicit Q: column j = H_0 H_1 ... H_j e_j  (columns independent: one warp each)
    for (int j = warp; j < p; j += kNW) {
        c64* q = Q + static_cast<size_t>(j) * m;
        for (int r = lane; r < m; r += 32) q[r] = mk(r == j ? 1.0 : 0.0, 0.0);
        __syncwarp();
        for (int k = j; k >= 0; --k) {
            const c64* v = A + static_cast<size_t>(k) * m;
            c64 w = mk(0.0, 0.0);
            for (int r = k + lane; r < m; r += 32) cmac_conj(w, v[r], q[r]);
            w = warp_sum_c(w);
            const c64 tw = mk(tau[k] * w.re, tau[k] * w.im);
            for (int r = k + lane; r < m; r += 32) {
                const c64 vr = v[r];
                q[r].re -= vr.re * tw.re - vr.im * tw.im;
                q[r].im -= vr.re * tw.im + vr.im * tw.re;
            }
            __syncwarp();
        }
        if (MODE == 0) {
            cplx<T>* vo = Vout + static_cast<size_t>(f) * m * p + static_cast<size_t>(j) * m;
            for (int r = lane; r < m; r += 32) vo[r] = mk<T>(static_cast<T>(q[r].re), static_cast<T>(q[r].im));
        }
    }
    if (MODE == 1) {
        // Rt[:, perm[j]] = R[:, j]  (C = Q R P^T), column-major p x p
        c64* Rf = Rt + static_cast<size_t>(f) * p * p;
        for (int e = threadIdx.x; e < p * p; e += kNT) {
            const int i = e % p, j = e / p;
            c64 val = mk(0.0, 0.0);
            if (i == j) val = rdiag[i];
            else if (j > i) val = A[static_cast<size_t>(j) * m + i];
            Rf[static_cast<size_t>(perm[j]) * p + i] = val;
        }
    }
}

// ------------------------------------------------------------------ pivoted Cholesky QR (fp32 batch path)
// Same factorisation as the reference's column-pivoted QR (R/src/linalg.cpp:127-141) in exact
// arithmetic: the pivoted Cholesky factor of G = C^H C (fp64; products of fp32 data are exact)
// is R with |R_kk| = sqrt(Schur pivot), so Eigen's rank rule (nonzero-pivot cut + |R_kk| >
// eps*p*maxpivot, eps of the data type) is applied to the same quantities. Far fewer block
// barriers than Householder: one Gram pass, a p x p factorisation + inverse in one warp, a
// row-parallel product with L^-H.
//   MODE 0: V = C P L^-H (complex64, column-major) for the power iteration, rank flags.
//   MODE 1: CholQR2 -> Q (fp64, work[f][1]) and Rt = Q^H C for the Nystrom tail.
constexpr int kRC = 64;   // rows per staged Gram chunk
constexpr int kRCP = 65;  // padded column stride (16-B elements): conflict-free column reads

// G(i, j) = sum_r conj(X_i[r]) Y_j[r] over column-major X, Y (p x m), staged kRC rows at a time.
// HERM: X == Y, only i <= j computed and mirrored.
template <bool HERM, typename XT, typename YT>
__device__ void block_gram(const XT* __restrict__ X, const YT* __restrict__ Y, int m, int p, c64* chunk, c64* G) {
    const int ne = HERM ? p * (p + 1) / 2 : p * p;
    constexpr int kMaxE = 16;  // entries per thread (p <= 64: 4096 / 256)
    c64 acc[kMaxE];
    int cnt = 0;
    for (int e = threadIdx.x; e < ne && cnt < kMaxE; e += blockDim.x) acc[cnt++] = mk(0.0, 0.0);
    c64* cy = HERM ? chunk : chunk + p * kRCP;
    for (int r0 = 0; r0 < m; r0 += kRC) {
        const int rn = min(kRC, m - r0);
        __syncthreads();
        for (int e = threadIdx.x; e < p * kRC; e += blockDim.x) {
            const int c = e / kRC, r = e % kRC;
            chunk[c * kRCP + r] = r < rn ? to64(X[static_cast<size_t>(c) * m + r0 + r]) : mk(0.0, 0.0);
            if (!HERM) cy[c * kRCP + r] = r < rn ? to64(Y[static_cast<size_t>(c) * m + r0 + r]) : mk(0.0, 0.0);
        }
        __syncthreads();
        int q = 0;
        for (int e = threadIdx.x; e < ne && q < kMaxE; e += blockDim.x, ++q) {
            int i, j;
            if (HERM) {
                i = 0;
                int rem = e;
                while (rem >= p - i) { rem -= p - i; ++i; }
                j = i + rem;
            } else {
                i = e % p;
                j = e / p;
            }
            const c64* xi = chunk + i * kRCP;
            const c64* yj = cy + j * kRCP;
            c64 a = acc[q];
            for (int r = 0; r < rn; ++r) cmac_conj(a, xi[r], yj[r]);
            acc[q] = a;
        }
    }
    int q = 0;
    for (int e = threadIdx.x; e < ne && q < kMaxE; e += blockDim.x, ++q) {
        int i, j;
        if (HERM) {
            i = 0;
            int rem = e;
            while (rem >= p - i) { rem -= p - i; ++i; }
            j = i + rem;
            G[i * p + j] = conj(acc[q]);  // G(j, i)
        } else {
            i = e % p;
            j = e / p;
        }
        G[j * p + i] = acc[q];  // column-major G(i, j)
    }
    __syncthreads();
}

// In-place Cholesky of the Hermitian p x p matrix A (column-major) by warp 0: A_perm = L L^H,
// then A <- L^-1 (lower triangular). Optional diagonal pivoting; d[k] = Schur pivot at step k.
__device__ void warp_cholesky_inv(c64* A, int p, bool pivot, int* perm, double* d) {
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    for (int k = 0; k < p; ++k) {
        int piv = k;
        if (pivot) {
            double best = -1.0;
            int bi = p;
            for (int j = k + lane; j < p; j += 32) {
                const double v = A[j * p + j].re;
                if (v > best || (v == best && j < bi)) { best = v; bi = j; }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
            }
            piv = bi;
        }
        if (piv != k) {  // symmetric swap of rows/cols k and piv
            for (int i = lane; i < p; i += 32) {
                const c64 t = A[k * p + i]; A[k * p + i] = A[piv * p + i]; A[piv * p + i] = t;
            }
            __syncwarp();
            for (int i = lane; i < p; i += 32) {
                const c64 t = A[i * p + k]; A[i * p + k] = A[i * p + piv]; A[i * p + piv] = t;
            }
            if (lane == 0) { const int t = perm[k]; perm[k] = perm[piv]; perm[piv] = t; }
            __syncwarp();
        }
        const double dk = A[k * p + k].re;
        if (lane == 0) d[k] = dk;
        const double lkk = dk > 0.0 ? sqrt(dk) : 0.0;
        const double inv = lkk > 0.0 ? 1.0 / lkk : 0.0;
        __syncwarp();
        for (int i = k + lane; i < p; i += 32) {
            const c64 v = A[k * p + i];
            A[k * p + i] = i == k ? mk(lkk, 0.0) : mk(v.re * inv, v.im * inv);
        }
        __syncwarp();
        const int nt = p - k - 1;  // Schur update of the trailing block (lower + mirror)
        for (int e = lane; e < nt * nt; e += 32) {
            const int i = k + 1 + e % nt, j = k + 1 + e / nt;
            if (j > i) continue;
            const c64 li = A[k * p + i], lj = A[k * p + j];
            c64 a = A[j * p + i];
            a.re -= li.re * lj.re + li.im * lj.im;  // li * conj(lj)
            a.im -= li.im * lj.re - li.re * lj.im;
            A[j * p + i] = a;
            A[i * p + j] = conj(a);
        }
        __syncwarp();
    }
    // L^-1 by forward substitution, one lane per column c (columns independent).
    for (int c = lane; c < p; c += 32) {
        const double lcc = A[c * p + c].re;
        const double icc = lcc > 0.0 ? 1.0 / lcc : 0.0;
        c64 x[64];
        x[c] = mk(icc, 0.0);
        for (int i = c + 1; i < p; ++i) {
            c64 acc = mk(0.0, 0.0);
            for (int q = c; q < i; ++q) cmac(acc, A[q * p + i], x[q]);  // L(i,q) Linv(q,c)
            const double lii = A[i * p + i].re;
            const double ii = lii > 0.0 ? -1.0 / lii : 0.0;
            x[i] = mk(acc.re * ii, acc.im * ii);
        }
        __syncwarp(__activemask());
        for (int i = 0; i < c; ++i) A[c * p + i] = mk(0.0, 0.0);
        for (int i = c; i < p; ++i) A[c * p + i] = x[i];
    }
    __syncwarp();
}

// Out[j][r] = sum_{i <= j} X[perm[i]][r] conj(Linv(j, i))   (rows of X P L^-H), 16 columns at a time.
template <typename XT, typename OT>
__device__ void rows_apply_linvh(const XT* __restrict__ X, const int* perm, const c64* Linv, int m, int p,
                                 OT* __restrict__ Out) {
    for (int r = threadIdx.x; r < m; r += blockDim.x) {
        for (int jb = 0; jb < p; jb += 16) {
            const int jn = min(16, p - jb);
            c64 acc[16];
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) acc[jj] = mk(0.0, 0.0);
            for (int i = 0; i < jb + jn; ++i) {
                const c64 x = to64(X[static_cast<size_t>(perm ? perm[i] : i) * m + r]);
                const c64* lcol = Linv + i * p + jb;  // Linv(jb.., i)
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) {
                    if (jj < jn && i <= jb + jj) cmac(acc[jj], x, conj(lcol[jj]));
                }
            }
#pragma unroll
            for (int jj = 0; jj < 16; ++jj)
                if (jj < jn) {
                    OT o;
                    o.re = static_cast<decltype(o.re)>(acc[jj].re);
                    o.im = static_cast<decltype(o.im)>(acc[jj].im);
                    Out[static_cast<size_t>(jb + jj) * m + r] = o;
                }
        }
    }
}

template <int MODE>
__global__ void __launch_bounds__(kNT) k_cholqr(const c32* __restrict__ Cin, c64* __restrict__ work,
                                                 c32* __restrict__ Vout, c64* __restrict__ Rt,
                                                 int32_t* __restrict__ status, const int32_t* __restrict__ fmap,
                                                 int m, int p, const c32* __restrict__ Vin, c64* __restrict__ Hout) {
    extern __shared__ uint8_t dsm[];
    c64* G = reinterpret_cast<c64*>(dsm);  // p x p
    c64* chunk = G + p * p;                // 2 x p x kRC
    __shared__ int perm[64];
    __shared__ double d[64];
    const int f = frame_of_x(fmap);
    const c32* Cf = Cin + static_cast<size_t>(f) * m * p;
    for (int j = threadIdx.x; j < p; j += kNT) perm[j] = j;
    block_gram<true>(Cf, Cf, m, p, chunk, G);
    warp_cholesky_inv(G, p, true, perm, d);
    __syncthreads();
    if (MODE == 0 && threadIdx.x == 0) {
        // Eigen ColPivHouseholderQR::rank() on the pivoted-Cholesky diagonal, data eps = fp32
        if (cholqr_rank(d, p, m) < p) atomicOr(&status[f], kFrameRank);
    }
    if (MODE == 0) {
        rows_apply_linvh(Cf, perm, G, m, p, Vout + static_cast<size_t>(f) * m * p);
        return;
    }
    // MODE 1: Q1 = C P L1^-H -> work[f][0]; Q = Q1 L2^-H -> work[f][1]; Rt = Q^H C.
    c64* Q1 = work + static_cast<size_t>(f) * 2 * p * m;
    c64* Q = Q1 + static_cast<size_t>(p) * m;
    rows_apply_linvh(Cf, perm, G, m, p, Q1);
    __syncthreads();
    block_gram<true>(static_cast<const c64*>(Q1), static_cast<const c64*>(Q1), m, p, chunk, G);
    warp_cholesky_inv(G, p, false, nullptr, d);
    __syncthreads();
    rows_apply_linvh(static_cast<const c64*>(Q1), nullptr, G, m, p, Q);
    __syncthreads();
    block_gram<false>(static_cast<const c64*>(Q), Cf, m, p, chunk, G);
    c64* Rf = Rt + static_cast<size_t>(f) * p * p;
    for (int e = threadIdx.x; e < p * p; e += kNT) Rf[e] = G[e];
    if (Vin) {  // fast2: H = V^H C with V the last power-iteration basis (W = pinv(H))
        block_gram<false>(Vin + static_cast<size_t>(f) * m * p, Cf, m, p, chunk, G);
        c64* Hf = Hout + static_cast<size_t>(f) * p * p;
        for (int e = threadIdx.x; e < p * p; e += kNT) Hf[e] = G[e];
    }
}

// ------------------------------------------------------------------ one-sided Jacobi SVD
// n x n complex fp64, column-major in smem (a[c*n + r]); v accumulates right rotations.
// Round-robin (circle) ordering, one warp per column pair. Returns false on sweep cap.
__device__ bool block_jacobi_svd(c64* a, c64* v, int n, double* sig, int* order, int* sweeps_out = nullptr) {
    __shared__ int s_rot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) v[e] = mk((e % n) == (e / n) ? 1.0 : 0.0, 0.0);
    const int np = (n + 1) & ~1;
    bool converged = false;
    for (int sweep = 0; sweep < 40; ++sweep) {
        if (threadIdx.x == 0) s_rot = 0;
        __syncthreads();
        for (int rnd = 0; rnd < np - 1; ++rnd) {
            for (int idx = warp; idx < np / 2; idx += blockDim.x / 32) {
                int i, j;
                if (idx == 0) {
                    i = rnd;
                    j = np - 1;
                } else {
                    i = (rnd + idx) % (np - 1);
                    j = (rnd - idx + (np - 1)) % (np - 1);
                }
                if (i > j) {
                    const int t = i;
                    i = j;
                    j = t;
                }
                if (j >= n) continue;
                c64* ai = a + i * n;
                c64* aj = a + j * n;
                double al = 0.0, be = 0.0;
                c64 ga = mk(0.0, 0.0);
                for (int r = lane; r < n; r += 32) {
                    al += norm2(ai[r]);
                    be += norm2(aj[r]);
                    cmac_conj(ga, ai[r], aj[r]);
                }
                al = warp_sum(al);
                be = warp_sum(be);
                ga = warp_sum_c(ga);
                const double g = sqrt(norm2(ga));
                if (g == 0.0 || g <= 8.0 * 2.220446049250313e-16 * n * sqrt(al * be)) continue;
                const double zeta = (be - al) / (2.0 * g);
                const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / sqrt(1.0 + t * t);
                const double s = c * t;
                const c64 e = mk(ga.re / g, ga.im / g);  // e^{i phi}
                // a_i' = c a_i - s e^{-i phi} a_j ;  a_j' = s e^{i phi} a_i + c a_j
                for (int r = lane; r < n; r += 32) {
                    const c64 x = ai[r], y = aj[r];
                    const c64 ey = mk(e.re * y.re + e.im * y.im, e.re * y.im - e.im * y.re);  // conj(e) y
                    const c64 ex = mk(e.re * x.re - e.im * x.im, e.re * x.im + e.im * x.re);  // e x
                    ai[r] = mk(c * x.re - s * ey.re, c * x.im - s * ey.im);
                    aj[r] = mk(s * ex.re + c * y.re, s * ex.im + c * y.im);
                }
                c64* vi = v + i * n;
                c64* vj = v + j * n;
                for (int r = lane; r < n; r += 32) {
                    const c64 x = vi[r], y = vj[r];
                    const c64 ey = mk(e.re * y.re + e.im * y.im, e.re * y.im - e.im * y.re);
                    const c64 ex = mk(e.re * x.re - e.im * x.im, e.re * x.im + e.im * x.re);
                    vi[r] = mk(c * x.re - s * ey.re, c * x.im - s * ey.im);
                    vj[r] = mk(s * ex.re + c * y.re, s * ex.im + c * y.im);
                }
                if (lane == 0) s_rot = 1;
            }
            __syncthreads();
        }
        const bool done = (s_rot == 0);
        __syncthreads();  // every warp has read s_rot before thread 0 resets it next sweep
        if (done) {
            converged = true;
            if (sweeps_out && threadIdx.x == 0) *sweeps_out = sweep + 1;
            break;
        }
    }
    // singular values and descending order (stable: ties keep the lower index)
    for (int c = warp; c < n; c += blockDim.x / 32) {
        double s = 0.0;
        for (int r = lane; r < n; r += 32) s += norm2(a[c * n + r]);
        s = warp_sum(s);
        if (lane == 0) sig[c] = sqrt(s);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int c = 0; c < n; ++c) order[c] = c;
        for (int x = 0; x < n; ++x) {
            int best = x;
            for (int y = x + 1; y < n; ++y)
                if (sig[order[y]] > sig[order[best]]) best = y;
            const int t = order[x];
            order[x] = order[best];
            order[best] = t;
        }
    }
    __syncthreads();
    return converged;
}

__device__ int32_t* g_dbg_sweeps = nullptr;  // optional per-frame Jacobi sweep counts (debug)

// ------------------------------------------------------------------ warp-per-frame Nystrom tail
// Hermitian eigendecomposition of an n x n matrix (n <= 64, column-major in the warp's shared
// slice) by cyclic two-sided Jacobi with the parallel (circle) ordering: the n/2 disjoint
// rotations of a round commute, so all column rotations are applied, then all row rotations.
// Rotation (R/tests/oracle_jacobi.hpp form): b = a_pq, phi = arg b, tau = (a_qq - a_pp) / 2|b|,
// t = sgn(tau) / (|tau| + sqrt(1 + tau^2)), c = 1/sqrt(1+t^2), s = t c e^{i phi}.
// Warp-synchronous: no block barriers. Returns sweeps used (0 = no convergence in 30).
__device__ int warp_jacobi_eigh(c64* A, c64* Z, int n, double* rc, double* rs, c64* re) {
    const int lane = threadIdx.x & 31;
    for (int e = lane; e < n * n; e += 32) Z[e] = mk((e % n) == (e / n) ? 1.0 : 0.0, 0.0);
    const int np = (n + 1) & ~1;
    const int npairs = np / 2;
    double dmax = 0.0;  // scale for an absolute floor on negligible off-diagonals
    for (int c = 0; c < n; ++c) dmax = fmax(dmax, fabs(A[c * n + c].re));
    const double floor2 = (1e-18 * dmax) * (1e-18 * dmax);
    __syncwarp();
    for (int sweep = 0; sweep < 30; ++sweep) {
        bool any = false;
        for (int rnd = 0; rnd < np - 1; ++rnd) {
            // rotation parameters, one lane per pair
            for (int t = lane; t < npairs; t += 32) {
                int i, j;
                if (t == 0) { i = rnd; j = np - 1; }
                else { i = (rnd + t) % (np - 1); j = (rnd - t + (np - 1)) % (np - 1); }
                if (i > j) { const int x = i; i = j; j = x; }
                double c = 1.0, sm = 0.0;
                c64 ph = mk(1.0, 0.0);
                if (j < n) {
                    const c64 b = A[j * n + i];  // a(i, j)
                    const double app = A[i * n + i].re, aqq = A[j * n + j].re;
                    const double ab2 = norm2(b);
                    if (ab2 > floor2 && ab2 > 1e-30 * fabs(app * aqq)) {
                        const double ab = sqrt(ab2);
                        const double tau = (aqq - app) / (2.0 * ab);
                        const double tt = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                        c = 1.0 / sqrt(1.0 + tt * tt);
                        sm = tt * c;
                        ph = mk(b.re / ab, b.im / ab);
                    }
                }
                rc[t] = c;
                rs[t] = sm;
                re[t] = ph;
            }
            __syncwarp();
            bool rot = false;
            for (int t = 0; t < npairs; ++t) rot |= rs[t] != 0.0;
            any |= rot;
            if (!rot) continue;
            // columns: a(r,i) = c a_ri - conj(s) a_rj ; a(r,j) = s a_ri + c a_rj  (A and Z)
            for (int e = lane; e < npairs * n * 2; e += 32) {
                const int which = e / (npairs * n);  // 0: A, 1: Z
                const int t = (e / n) % npairs, r = e % n;
                int i, j;
                if (t == 0) { i = rnd; j = np - 1; }
                else { i = (rnd + t) % (np - 1); j = (rnd - t + (np - 1)) % (np - 1); }
                if (i > j) { const int x = i; i = j; j = x; }
                if (j >= n || rs[t] == 0.0) continue;
                c64* M = which ? Z : A;
                const double c = rc[t], sm = rs[t];
                const c64 s = mk(sm * re[t].re, sm * re[t].im);
                const c64 x = M[i * n + r], y = M[j * n + r];
                M[i * n + r] = mk(c * x.re - (s.re * y.re + s.im * y.im), c * x.im - (s.re * y.im - s.im * y.re));
                M[j * n + r] = mk(s.re * x.re - s.im * x.im + c * y.re, s.re * x.im + s.im * x.re + c * y.im);
            }
            __syncwarp();
            // rows: a(i,r) = c a_ir - s a_jr ; a(j,r) = conj(s) a_ir + c a_jr
            for (int e = lane; e < npairs * n; e += 32) {
                const int t = e / n, r = e % n;
                int i, j;
                if (t == 0) { i = rnd; j = np - 1; }
                else { i = (rnd + t) % (np - 1); j = (rnd - t + (np - 1)) % (np - 1); }
                if (i > j) { const int x = i; i = j; j = x; }
                if (j >= n || rs[t] == 0.0) continue;
                const double c = rc[t], sm = rs[t];
                const c64 s = mk(sm * re[t].re, sm * re[t].im);
                const c64 x = A[r * n + i], y = A[r * n + j];
                A[r * n + i] = mk(c * x.re - (s.re * y.re - s.im * y.im), c * x.im - (s.re * y.im + s.im * y.re));
                A[r * n + j] = mk(s.re * x.re + s.im * x.im + c * y.re, s.re * x.im - s.im * x.re + c * y.im);
            }
            __syncwarp();
        }
        if (!any) return sweep + 1;
    }
    return 0;
}

// Descending order of the real diagonal (ties: lower index first), computed by lane 0.
__device__ void warp_order_desc(const c64* A, int n, bool by_abs, int* order) {
    if ((threadIdx.x & 31) == 0) {
        for (int c = 0; c < n; ++c) order[c] = c;
        for (int x = 0; x < n; ++x) {
            int best = x;
            for (int y = x + 1; y < n; ++y) {
                const double vy = A[order[y] * n + order[y]].re, vb = A[order[best] * n + order[best]].re;
                if ((by_abs ? fabs(vy) > fabs(vb) : vy > vb)) best = y;
            }
            const int t = order[x]; order[x] = order[best]; order[best] = t;
        }
    }
    __syncwarp();
}

// One warp per frame: W = pinv(Herm(H)) (cutoff p*eps_T*max|lambda|), B' = Rt W Rt^H,
// eig(B') descending, U = Q Z_K, lambda = clamp(Z_K eigenvalues). R/src/estimators.cpp:37-50,
// R/src/linalg.cpp:143-163. Q (fp64, work[f][1]), Rt, H (p x p column-major) from k_cholqr<1> /
// k_gather.
template <typename T>
__global__ void __launch_bounds__(128) k_nystrom_warp(const c64* __restrict__ Hin, const c64* __restrict__ work,
                                                     const c64* __restrict__ Rt, c64* __restrict__ basis,
                                                     double* __restrict__ eig, int32_t* __restrict__ status,
                                                     int frames, int m, int p, int k) {
    extern __shared__ uint8_t dsm[];
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int f = blockIdx.x * (blockDim.x >> 5) + wib;
    const size_t per_warp = sizeof(c64) * (3 * p * p + 2 * 64) + sizeof(double) * 2 * 64 + sizeof(int) * 64;
    uint8_t* base = dsm + wib * ((per_warp + 15) & ~size_t(15));
    c64* A = reinterpret_cast<c64*>(base);
    c64* Z = A + p * p;
    c64* Tm = Z + p * p;
    c64* re = Tm + p * p;
    c64* zk = re + 64;
    double* rc = reinterpret_cast<double*>(zk + 64);
    double* rs = rc + 64;
    int* order = reinterpret_cast<int*>(rs + 64);
    if (f >= frames) return;
    const double eps = eps_of<T>::value;
    const c64* Hf = Hin + static_cast<size_t>(f) * p * p;
    for (int e = lane; e < p * p; e += 32) {
        const int i = e % p, j = e / p;
        const c64 a = Hf[j * p + i], b = Hf[i * p + j];
        A[e] = mk(0.5 * (a.re + b.re), 0.5 * (a.im - b.im));  // Herm(H)(i, j)
    }
    __syncwarp();
    const int sw1 = warp_jacobi_eigh(A, Z, p, rc, rs, re);
    warp_order_desc(A, p, true, order);
    const double lmax = fabs(A[order[0] * p + order[0]].re);
    const double cutoff = static_cast<double>(p) * eps * lmax;
    // W = Z diag(1/lambda) Z^H over |lambda| > cutoff -> Tm
    for (int e = lane; e < p * p; e += 32) {
        const int i = e % p, j = e / p;
        c64 acc = mk(0.0, 0.0);
        if (lmax > 0.0)
            for (int c = 0; c < p; ++c) {
                const double l = A[c * p + c].re;
                if (fabs(l) > cutoff) {
                    const c64 zi = Z[c * p + i], zj = Z[c * p + j];
                    const double w = 1.0 / l;
                    acc.re += w * (zi.re * zj.re + zi.im * zj.im);
                    acc.im += w * (zi.im * zj.re - zi.re * zj.im);
                }
            }
        Tm[e] = acc;
    }
    __syncwarp();
    // A = Rt W ; then B' = A Rt^H -> Z (scratch), copied back to A
    const c64* Rf = Rt + static_cast<size_t>(f) * p * p;
    for (int e = lane; e < p * p; e += 32) {
        const int i = e % p, j = e / p;
        c64 acc = mk(0.0, 0.0);
        for (int c = 0; c < p; ++c) cmac(acc, Rf[c * p + i], Tm[j * p + c]);
        A[e] = acc;
    }
    __syncwarp();
    for (int e = lane; e < p * p; e += 32) {
        const int i = e % p, j = e / p;
        c64 acc = mk(0.0, 0.0);
        for (int c = 0; c < p; ++c) cmac(acc, A[c * p + i], conj(Rf[c * p + j]));
        Tm[e] = acc;
    }
    __syncwarp();
    for (int e = lane; e < p * p; e += 32) {  // Hermitian part of B'
        const int i = e % p, j = e / p;
        const c64 a = Tm[j * p + i], b = Tm[i * p + j];
        A[e] = mk(0.5 * (a.re + b.re), 0.5 * (a.im - b.im));
    }
    __syncwarp();
    const int sw2 = warp_jacobi_eigh(A, Z, p, rc, rs, re);
    warp_order_desc(A, p, false, order);
    // basis U(:, kk) = Q Z(:, order[kk])
    const c64* Qf = work + static_cast<size_t>(f) * 2 * p * m + static_cast<size_t>(p) * m;
    c64* Bf = basis + static_cast<size_t>(f) * m * k;
    for (int kk = 0; kk < k; ++kk) {
        const int c = order[kk];
        for (int q = lane; q < p; q += 32) zk[q] = Z[c * p + q];
        __syncwarp();
        for (int r = lane; r < m; r += 32) {
            c64 acc = mk(0.0, 0.0);
            for (int q = 0; q < p; ++q) cmac(acc, Qf[static_cast<size_t>(q) * m + r], zk[q]);
            Bf[static_cast<size_t>(kk) * m + r] = acc;
        }
        __syncwarp();
    }
    for (int kk = lane; kk < k; kk += 32) {
        double lam = A[order[kk] * p + order[kk]].re;
        if (lam < 0.0 && lam >= -1e-10) lam = 0.0;
        eig[static_cast<size_t>(f) * k + kk] = lam;
    }
    if (lane == 0 && (sw1 == 0 || sw2 == 0)) atomicOr(&status[f], kFrameNoConv);
    if (lane == 0 && g_dbg_sweeps) g_dbg_sweeps[f] = sw1 | (sw2 << 8);
}

// ------------------------------------------------------------------ Nystrom tail
// MODE_FAST2: H = V^H C (V, C: the last power-iteration sketch); MODE_FAST1: H from k_gather.
// W = pinv(H)  (cutoff p*eps_T*sigma1)            R/src/linalg.cpp:143-163
// B' = Rt W Rt^H; SVD(B') = Ub Sb ..;  U = Q Ub(:,1:K); lambda = clamp(Sb(1:K))
//                                                  R/src/estimators.cpp:37-50, :25-31
// Output basis column-major K x M fp64, eigenvalues K fp64.
template <typename T, bool FAST2>
__global__ void __launch_bounds__(kNT) k_nystrom(const cplx<T>* __restrict__ V, const cplx<T>* __restrict__ C,
                                                  const c64* __restrict__ Hin, const c64* __restrict__ work,
                                                  const c64* __restrict__ Rt, c64* __restrict__ basis,
                                                  double* __restrict__ eig, int32_t* __restrict__ status,
                                                  const int32_t* __restrict__ fmap, int m, int p, int k,
                                                  int32_t* __restrict__ dbg) {
    __shared__ int s_sw[2];
    extern __shared__ uint8_t dsm[];
    c64* sa = reinterpret_cast<c64*>(dsm);  // p x p
    c64* sv = sa + p * p;                   // p x p
    c64* sw = sv + p * p;                   // p x p (W)
    c64* st = sv;                           // p x p temp (aliases sv once W is formed)
    double* sig = reinterpret_cast<double*>(sw + p * p);
    int* order = reinterpret_cast<int*>(sig + p);
    const int f = frame_of_x(fmap);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double eps = eps_of<T>::value;

    // H (column-major)
    if (FAST2) {
        const cplx<T>* Vf = V + static_cast<size_t>(f) * m * p;
        const cplx<T>* Cf = C + static_cast<size_t>(f) * m * p;
        for (int e = warp; e < p * p; e += kNW) {
            const int i = e % p, j = e / p;
            c64 s = mk(0.0, 0.0);
            for (int r = lane; r < m; r += 32)
                cmac_conj(s, to64(Vf[static_cast<size_t>(i) * m + r]), to64(Cf[static_cast<size_t>(j) * m + r]));
            s = warp_sum_c(s);
            if (lane == 0) sa[j * p + i] = s;
        }
    } else {
        const c64* Hf = Hin + static_cast<size_t>(f) * p * p;
        for (int e = threadIdx.x; e < p * p; e += kNT) sa[e] = Hf[e];
    }
    __syncthreads();
    bool ok = block_jacobi_svd(sa, sv, p, sig, order, &s_sw[0]);
    // W = V diag(1/s) U^H, U_c = a_c / s_c
    const double s1 = sig[order[0]];
    const double cutoff = static_cast<double>(p) * eps * s1;
    for (int e = threadIdx.x; e < p * p; e += kNT) {
        const int i = e % p, j = e / p;  // W(i, j)
        c64 acc = mk(0.0, 0.0);
        if (s1 > 0.0) {
            for (int c = 0; c < p; ++c) {
                const double s = sig[c];
                if (s > cutoff) {
                    // v(i,c) * conj(a(j,c)) / s^2   (u = a / s)
                    const c64 vi = sv[c * p + i];
                    const c64 aj = sa[c * p + j];
                    const double w = 1.0 / (s * s);
                    acc.re += w * (vi.re * aj.re + vi.im * aj.im);
                    acc.im += w * (vi.im * aj.re - vi.re * aj.im);
                }
            }
        }
        sw[j * p + i] = acc;
    }
    __syncthreads();
    // T = Rt W ; B' = T Rt^H
    const c64* Rf = Rt + static_cast<size_t>(f) * p * p;
    for (int e = threadIdx.x; e < p * p; e += kNT) {
        const int i = e % p, j = e / p;
        c64 acc = mk(0.0, 0.0);
        for (int c = 0; c < p; ++c) cmac(acc, Rf[c * p + i], sw[j * p + c]);
        st[j * p + i] = acc;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < p * p; e += kNT) {
        const int i = e % p, j = e / p;
        c64 acc = mk(0.0, 0.0);
        for (int c = 0; c < p; ++c) cmac(acc, st[c * p + i], conj(Rf[c * p + j]));
        sa[j * p + i] = acc;
    }
    __syncthreads();
    ok = block_jacobi_svd(sa, sv, p, sig, order, &s_sw[1]) && ok;
    if (dbg && threadIdx.x == 0) dbg[f] = s_sw[0] | (s_sw[1] << 8);
    // basis U[:, kk] = Q * (a[:, order[kk]] / sig)
    const c64* Qf = work + static_cast<size_t>(f) * 2 * p * m + static_cast<size_t>(p) * m;
    c64* Bf = basis + static_cast<size_t>(f) * m * k;
    for (int e = threadIdx.x; e < m * k; e += kNT) {
        const int kk = e / m, r = e % m;
        const int c = order[kk];
        const double s = sig[c];
        const double inv = s > 0.0 ? 1.0 / s : 0.0;
        c64 acc = mk(0.0, 0.0);
        for (int q = 0; q < p; ++q) cmac(acc, Qf[static_cast<size_t>(q) * m + r], sa[c * p + q]);
        Bf[static_cast<size_t>(kk) * m + r] = mk(acc.re * inv, acc.im * inv);
    }
    if (threadIdx.x < k) {
        double lam = sig[order[threadIdx.x]];
        if (lam < 0.0 && lam >= -1e-10) lam = 0.0;
        eig[static_cast<size_t>(f) * k + threadIdx.x] = lam;
    }
    if (threadIdx.x == 0 && !ok) atomicOr(&status[f], kFrameNoConv);
}

}  // namespace sub
}  // namespace fmk

// ------------------------------------------------------------------ launchers (host)
using namespace fmk;

cudaError_t fm_gen_nystrom(const void* V, const void* C, const void* H, const void* work, const void* Rt, void* basis,
                           double* eig, int32_t* status, int m, int p, int k, bool fast2, cudaStream_t s);

template <typename T>
cudaError_t fm_launch_rmul(const void* R, const void* omega, const void* V, void* C, const int32_t* fmap, int frames,
                           int m, int p, bool real_rhs, cudaStream_t s) {
    constexpr int kMaxPC = sizeof(T) == 4 ? 64 : 32;
    const int slices = (p + kMaxPC - 1) / kMaxPC;
    dim3 grid((m + sub::kNT - 1) / sub::kNT, frames, slices);
    auto Rp = static_cast<const cplx<T>*>(R);
    auto Op = static_cast<const T*>(omega);
    auto Vp = static_cast<const cplx<T>*>(V);
    auto Cp = static_cast<cplx<T>*>(C);
#define FM_RMUL(PC)                                                                                   \
    if (p <= PC || (PC == kMaxPC)) {                                                                  \
        if (real_rhs) sub::k_rmul<T, PC, true><<<grid, sub::kNT, 0, s>>>(Rp, Op, Vp, Cp, fmap, m, p);  \
        else sub::k_rmul<T, PC, false><<<grid, sub::kNT, 0, s>>>(Rp, Op, Vp, Cp, fmap, m, p);         \
        return cudaGetLastError();                                                                    \
    }
    FM_RMUL(8)
    FM_RMUL(16)
    FM_RMUL(32)
    if constexpr (kMaxPC == 64) { FM_RMUL(64) }
#undef FM_RMUL
    return cudaErrorInvalidValue;
}

template <typename T>
cudaError_t fm_launch_gather(const void* R, const int32_t* idx, void* C, void* H, const int32_t* fmap, int frames,
                             int m, int p, cudaStream_t s) {
    sub::k_gather<T><<<frames, sub::kNT, 0, s>>>(static_cast<const cplx<T>*>(R), idx, static_cast<cplx<T>*>(C),
                                                 static_cast<c64*>(H), fmap, m, p);
    return cudaGetLastError();
}

// pivoted Householder QR: dynamic shared memory of the per-column arrays (rdiag, nrm2, tau, perm)
static size_t qr_smem(int p) { return static_cast<size_t>(p) * (sizeof(c64) + 2 * sizeof(double) + sizeof(int)); }
template <typename K>
static cudaError_t qr_attr(K kern, size_t smem) {
    if (smem > 200 * 1024) return cudaErrorInvalidValue;
    if (smem <= 48 * 1024) return cudaSuccess;
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
}

template <typename T>
cudaError_t fm_launch_qr(const void* C, void* work, void* Vout, void* Rt, int32_t* status, int32_t* defcol,
                         const int32_t* fmap, int frames, int m, int p, bool final_mode, cudaStream_t s) {
    if (p < 1 || m < p) return cudaErrorInvalidValue;
    const size_t smem = qr_smem(p);
    auto kern = final_mode ? sub::k_qr<T, 1> : sub::k_qr<T, 0>;
    cudaError_t e = qr_attr(kern, smem);
    if (e != cudaSuccess) return e;
    if (final_mode)
        kern<<<frames, sub::kNT, smem, s>>>(static_cast<const cplx<T>*>(C), static_cast<c64*>(work), nullptr,
                                            static_cast<c64*>(Rt), status, defcol, fmap, m, p, nullptr);
    else
        kern<<<frames, sub::kNT, smem, s>>>(static_cast<const cplx<T>*>(C), static_cast<c64*>(work),
                                            static_cast<cplx<T>*>(Vout), nullptr, status, defcol, fmap, m, p, nullptr);
    return cudaGetLastError();
}

// One matrix: Q (first p columns, column-major) and the Eigen ColPivHouseholderQR rank (orthonormal_range of
// the block-Lanczos expansion, R/src/estimators.cpp:143-149: Q(:, 0:rank) spans the range).
template <typename T>
cudaError_t fm_launch_qr_rank(const void* C, void* work, void* Vout, int32_t* status, int32_t* rank_out, int m, int p,
                              cudaStream_t s) {
    if (p < 1 || m < p) return cudaErrorInvalidValue;
    const size_t smem = qr_smem(p);
    cudaError_t e = qr_attr(sub::k_qr<T, 0>, smem);
    if (e != cudaSuccess) return e;
    sub::k_qr<T, 0><<<1, sub::kNT, smem, s>>>(static_cast<const cplx<T>*>(C), static_cast<c64*>(work),
                                           static_cast<cplx<T>*>(Vout), nullptr, status, nullptr, nullptr, m, p,
                                           rank_out);
    return cudaGetLastError();
}
template cudaError_t fm_launch_qr_rank<double>(const void*, void*, void*, int32_t*, int32_t*, int, int, cudaStream_t);

cudaError_t fm_launch_cholqr(const void* C, void* work, void* Vout, void* Rt, int32_t* status, const int32_t* fmap,
                             int frames, int m, int p, bool final_mode, const void* Vin, void* Hout, cudaStream_t s) {
    if (p > 64 || p < 1 || m < p) return cudaErrorInvalidValue;
    const size_t smem = sizeof(c64) * (p * p + 2 * p * sub::kRCP);
    auto kern = final_mode ? sub::k_cholqr<1> : sub::k_cholqr<0>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    kern<<<frames, sub::kNT, smem, s>>>(static_cast<const c32*>(C), static_cast<c64*>(work), static_cast<c32*>(Vout),
                                        static_cast<c64*>(Rt), status, fmap, m, p, static_cast<const c32*>(Vin),
                                        static_cast<c64*>(Hout));
    return cudaGetLastError();
}


template <typename T>
cudaError_t fm_launch_nystrom(const void* V, const void* C, const void* H, const void* work, const void* Rt,
                              void* basis, double* eig, int32_t* status, const int32_t* fmap, int frames, int m,
                              int p, int k, bool fast2, cudaStream_t s) {
    const size_t smem = 3 * sizeof(c64) * p * p + sizeof(double) * p + sizeof(int) * p;
    if (smem > 200 * 1024) {  // p > 64: the same algebra on global memory (general.cu), fp64 facade only
        if (sizeof(T) != 8 || fmap) return cudaErrorInvalidValue;
        for (int f = 0; f < frames; ++f) {
            const size_t mp_ = static_cast<size_t>(m) * p, pp = static_cast<size_t>(p) * p;
            cudaError_t e = fm_gen_nystrom(V ? static_cast<const c64*>(V) + f * mp_ : nullptr,
                                           C ? static_cast<const c64*>(C) + f * mp_ : nullptr,
                                           H ? static_cast<const c64*>(H) + f * pp : nullptr,
                                           static_cast<const c64*>(work) + f * 2 * mp_,
                                           static_cast<const c64*>(Rt) + f * pp,
                                           static_cast<c64*>(basis) + static_cast<size_t>(f) * m * k, eig + f * k,
                                           status + f, m, p, k, fast2, s);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }
    auto kern = fast2 ? sub::k_nystrom<T, true> : sub::k_nystrom<T, false>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    kern<<<frames, sub::kNT, smem, s>>>(static_cast<const cplx<T>*>(V), static_cast<const cplx<T>*>(C),
                                        static_cast<const c64*>(H), static_cast<const c64*>(work),
                                        static_cast<const c64*>(Rt), static_cast<c64*>(basis), eig, status, fmap, m,
                                        p, k, nullptr);
    return cudaGetLastError();
}

template cudaError_t fm_launch_rmul<float>(const void*, const void*, const void*, void*, const int32_t*, int, int, int,
                                           bool, cudaStream_t);
template cudaError_t fm_launch_rmul<double>(const void*, const void*, const void*, void*, const int32_t*, int, int,
                                            int, bool, cudaStream_t);
template cudaError_t fm_launch_gather<float>(const void*, const int32_t*, void*, void*, const int32_t*, int, int, int,
                                             cudaStream_t);
template cudaError_t fm_launch_gather<double>(const void*, const int32_t*, void*, void*, const int32_t*, int, int, int,
                                              cudaStream_t);
template cudaError_t fm_launch_qr<float>(const void*, void*, void*, void*, int32_t*, int32_t*, const int32_t*, int, int,
                                         int, bool, cudaStream_t);
template cudaError_t fm_launch_qr<double>(const void*, void*, void*, void*, int32_t*, int32_t*, const int32_t*, int,
                                          int, int, bool, cudaStream_t);
template cudaError_t fm_launch_nystrom<float>(const void*, const void*, const void*, const void*, const void*, void*,
                                              double*, int32_t*, const int32_t*, int, int, int, int, bool,
                                              cudaStream_t);
template cudaError_t fm_launch_nystrom<double>(const void*, const void*, const void*, const void*, const void*, void*,
                                               double*, int32_t*, const int32_t*, int, int, int, int, bool,
                                               cudaStream_t);


template <typename T>
cudaError_t fm_launch_nystrom_warp(const void* H, const void* work, const void* Rt, void* basis, double* eig,
                                   int32_t* status, int frames, int m, int p, int k, cudaStream_t s) {
    if (p > 64 || k > p) return cudaErrorInvalidValue;
    const int wpb = 4;
    const size_t per_warp = sizeof(c64) * (3 * p * p + 2 * 64) + sizeof(double) * 2 * 64 + sizeof(int) * 64;
    const size_t smem = wpb * ((per_warp + 15) & ~size_t(15));
    if (smem > 200 * 1024) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(sub::k_nystrom_warp<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    sub::k_nystrom_warp<T><<<(frames + wpb - 1) / wpb, 32 * wpb, smem, s>>>(
        static_cast<const c64*>(H), static_cast<const c64*>(work), static_cast<const c64*>(Rt),
        static_cast<c64*>(basis), eig, status, frames, m, p, k);
    return cudaGetLastError();
}
template cudaError_t fm_launch_nystrom_warp<float>(const void*, const void*, const void*, void*, double*, int32_t*,
                                                   int, int, int, int, cudaStream_t);
