// Batched block-Lanczos signal subspace: block_lanczos_subspace, R/src/estimators.cpp:154-222
// (orthonormal_range :143-149), the paper's accurate baseline, for a whole batch of frames in ONE launch.
//
// One CTA per frame runs the reference's control flow on the device, in fp64 (the 1e-10 Ritz-value tolerance needs
// fp64 end to end; S is read as stored: complex64 R of the batch plan, or complex128 for the facade):
//   W = S Q                       thread per row, S read down its columns (S Hermitian: S(i, j) = conj S(j, i), so
//                                 the reads are coalesced), Q broadcast from the frame's basis columns
//   strip = basis^H W             warp per entry
//   h grows by the strip          kept raw in shared memory (A), the new corner symmetrised as HermitianMatrix does
//   Ritz values                   Householder tridiagonalisation of a copy, then the top-K eigenvalues by Sturm
//                                 multisection (16 probes per eigenvalue and round): per iteration O(n^3 / threads)
//                                 with ~5 barriers per column, instead of sweeps of rotations
//   Ritz vectors (once, at exit)  tridiagonalisation keeping the reflectors, inverse iteration on the real tridiagonal
//                                 for the K Ritz values, Gram-Schmidt, phases and reflectors back (ritz_vectors)
//   convergence                   |vals - prev| / max(|vals|, 1e-300) <= 1e-10 on two consecutive checks
//   z = W - basis (basis^H W),    twice (the reference's two Gram-Schmidt passes)
//   q = orthonormal_range(z)      column-pivoted CGS2 with Eigen's ColPivHouseholderQR rank rule
//   basis += q                    until convergence, an empty expansion, a full basis (room <= 0) or the cap
// Ritz vectors U = basis V(:, top-K) and clamp_nonnegative(vals) (R/src/estimators.cpp:25-31) are written out.
// The start block is the plan's orthonormal basis of span(gaussian_matrix(M, block, 0x6C616E637A6F)): the Krylov
// space and hence every Ritz value depend only on that span (R/src/estimators.cpp:161-163).
// Capacity: block <= kBMax, basis <= kNBMax columns (A and V live in shared memory); a frame that would need more
// is flagged kFrameCap (the facade then reruns it with the host-driven lanczos.cu path, the batch marks it NOCONV).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <algorithm>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/fastmusic_b200.h"
#include "fm_common.cuh"
#include "host_rng.hpp"

namespace fmk {
namespace lzb {

constexpr int kThreads = 256;
constexpr int kBMax = 16;   // block columns per expansion
constexpr int kNBMax = 72;  // basis columns: A, V complex128 72 x 72 each in shared memory
constexpr int kLd = kNBMax + 1;
static_assert(16 * kLd * 16 + 8 * 16 * 5 * kNBMax + 16 * kNBMax <= 16 * kLd * kNBMax,
              "exit-time Ritz-vector scratch (Z, solver rows, phases) fits in A");  // their leading dimension: 1168 B, so rows walked across columns are bank-conflict free
constexpr double kTol = 1e-10;  // R/src/estimators.cpp:160

#ifdef FM_LZ_TIMELINE  // experiment only: clock64 per phase of block 0 (tools/lz_timeline.py)
__device__ long long g_lz_tl[16];
#define LZ_T0() long long lz_t0_ = clock64()
#define LZ_MARK(slot)                                                 \
    do {                                                              \
        __syncthreads();                                              \
        if (blockIdx.x == 0 && threadIdx.x == 0) {                    \
            const long long now_ = clock64();                         \
            g_lz_tl[slot] += now_ - lz_t0_;                           \
            lz_t0_ = now_;                                            \
        }                                                             \
    } while (0)
#else
#define LZ_T0()
#define LZ_MARK(slot)
#endif

struct Args {
    const void* S;        // frames x M x M (row-major, full Hermitian), complex64 or complex128
    const double* q0;     // M x b0 complex128 column-major (shared start block)
    double* basis;        // frames x kNBMax x M complex128 (column-major per frame)
    double* W;            // frames x M x kBMax complex128 (row-major)
    double* Z;            // frames x M x kBMax complex128 (row-major)
    double* out_basis;    // frames x K x M complex128 (column-major per frame)
    double* out_eig;      // frames x K
    int32_t* status;      // frames (FM_FRAME_NOCONV / kFrameCap bits OR-ed in)
    double* last_change;  // frames, or nullptr
    int32_t* iters;       // frames, or nullptr (iterations run)
    int m, k, b0, max_iter;
};

constexpr int32_t kFrameCap = 1 << 20;  // basis / block beyond the kernel's shared-memory capacity

template <typename TS>
__device__ __forceinline__ c64 ld_s(const TS* p);
template <>
__device__ __forceinline__ c64 ld_s<float>(const float* p) {
    const float2 v = *reinterpret_cast<const float2*>(p);
    return mk(static_cast<double>(v.x), static_cast<double>(v.y));
}
template <>
__device__ __forceinline__ c64 ld_s<double>(const double* p) {
    const double2 v = *reinterpret_cast<const double2*>(p);
    return mk(v.x, v.y);
}

__device__ __forceinline__ c64 warp_csum(c64 v) {
    v.re = warp_sum(v.re);
    v.im = warp_sum(v.im);
    return v;
}

// strip(r, c) = sum_i conj(B(i, r)) X(i, c) for r < ncols, c < bq: warp per basis column r, lanes over rows, all bq
// columns of X at once (X row-major [i][kBMax]), then a warp reduction per column.
__device__ __forceinline__ void block_ah_x(const c64* B, const c64* X, c64* strip, int M, int ncols, int bq, int warp,
                                           int lane) {
    constexpr int kWarps = kThreads / 32;
    for (int r = warp; r < ncols; r += kWarps) {
        c64 acc[kBMax];
#pragma unroll
        for (int c = 0; c < kBMax; ++c) acc[c] = mk(0.0, 0.0);
        for (int i = lane; i < M; i += 32) {
            const c64 b = B[static_cast<size_t>(r) * M + i];
#pragma unroll
            for (int c = 0; c < kBMax; ++c)
                if (c < bq) cmac_conj(acc[c], b, X[i * kBMax + c]);
        }
#pragma unroll
        for (int c = 0; c < kBMax; ++c)
            if (c < bq) {
                const c64 v = warp_csum(acc[c]);
                if (lane == 0) strip[r * kBMax + c] = v;
            }
    }
}

// Y = X - B strip (rows i, columns c < bq; X, Y row-major [i][kBMax], may alias): thread per row, basis columns
// outer so every B element is loaded once.
__device__ __forceinline__ void block_sub(const c64* B, const c64* X, c64* Y, const c64* strip, int M, int ncols,
                                          int bq) {
    for (int i = threadIdx.x; i < M; i += kThreads) {
        c64 acc[kBMax];
#pragma unroll
        for (int c = 0; c < kBMax; ++c) acc[c] = c < bq ? X[i * kBMax + c] : mk(0.0, 0.0);
        int r = 0;
        for (; r + 4 <= ncols; r += 4) {
            c64 bv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) bv[u] = B[static_cast<size_t>(r + u) * M + i];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int c = 0; c < kBMax; ++c)
                    if (c < bq) acc[c] = acc[c] - bv[u] * strip[(r + u) * kBMax + c];
        }
        for (; r < ncols; ++r) {
            const c64 b = B[static_cast<size_t>(r) * M + i];
#pragma unroll
            for (int c = 0; c < kBMax; ++c)
                if (c < bq) acc[c] = acc[c] - b * strip[r * kBMax + c];
        }
#pragma unroll
        for (int c = 0; c < kBMax; ++c)
            if (c < bq) Y[i * kBMax + c] = acc[c];
    }
}


// Householder tridiagonalisation of the Hermitian n x n block of T (column-major, leading dim kLd; destroyed):
// T -> Q^H T Q real symmetric tridiagonal, diagonal d[i] and off-diagonal |e[i]| (the phases of a complex Hermitian
// tridiagonal are a diagonal unitary similarity away). Step k: unit v on rows k+1.., p = T v, w = p - (v^H p) v,
// T22 -= 2 (v w^H + w v^H). Scratch: vv, pp (kNBMax each).
// keep (optional): the unit Householder vector of step k is left in column k below the diagonal and the complex
// sub-diagonal entry in alph[k] (the back-transformation of the Ritz vectors needs both).
__device__ void tridiagonalize(c64* T, int n, double* d, double* e, c64* vv, c64* pp, double* red,
                               c64* alph = nullptr) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int kWarps = kThreads / 32;
    for (int k = 0; k + 2 < n; ++k) {
        const int L = n - k - 1;
        const c64* x = T + (k + 1) + kLd * k;  // column k below the diagonal
        // ||x||^2 and x0 (one warp)
        if (warp == 0) {
            double s2 = 0.0;
            for (int i = lane; i < L; i += 32) s2 += norm2(x[i]);
            s2 = warp_sum(s2);
            if (lane == 0) red[0] = s2;
        }
        __syncthreads();
        const double xn = sqrt(red[0]);
        const c64 x0 = x[0];
        const double ax0 = sqrt(norm2(x0));
        if (xn == 0.0 || (L == 1 && x0.im == 0.0)) {  // nothing to annihilate
            if (tid == 0) {
                d[k] = T[k + kLd * k].re;
                e[k] = sqrt(norm2(x0));
                if (alph) alph[k] = x0;
            }
            if (alph)
                for (int i = tid; i < L; i += kThreads) T[(k + 1 + i) + kLd * k] = mk(0.0, 0.0);  // H_k = I
            __syncthreads();
            continue;
        }
        const c64 ph = ax0 > 0.0 ? mk(x0.re / ax0, x0.im / ax0) : mk(1.0, 0.0);
        const c64 alpha = mk(-ph.re * xn, -ph.im * xn);          // x -> alpha e1
        // v = (x - alpha e1) / ||x - alpha e1||,  ||x - alpha e1||^2 = 2 xn (xn + |x0|)
        const double vnorm = sqrt(2.0 * xn * (xn + ax0));
        for (int i = tid; i < L; i += kThreads) {
            c64 v = x[i];
            if (i == 0) v = v - alpha;
            vv[i] = mk(v.re / vnorm, v.im / vnorm);
        }
        __syncthreads();
        // p = T22 v (T22 = T[k+1.., k+1..]); warp per row group, lanes over columns
        for (int i = warp; i < L; i += kWarps) {
            c64 acc = mk(0.0, 0.0);
            for (int j = lane; j < L; j += 32) cmac(acc, T[(k + 1 + i) + kLd * (k + 1 + j)], vv[j]);
            acc.re = warp_sum(acc.re);
            acc.im = warp_sum(acc.im);
            if (lane == 0) pp[i] = acc;
        }
        __syncthreads();
        if (warp == 0) {  // K = v^H p (real for Hermitian T22)
            double kr = 0.0;
            for (int i = lane; i < L; i += 32) kr += vv[i].re * pp[i].re + vv[i].im * pp[i].im;
            kr = warp_sum(kr);
            if (lane == 0) red[1] = kr;
        }
        __syncthreads();
        const double kk = red[1];
        for (int i = tid; i < L; i += kThreads) pp[i] = pp[i] - kk * vv[i];  // w
        __syncthreads();
        for (int it = tid; it < L * L; it += kThreads) {  // T22 -= 2 (v w^H + w v^H)
            const int i = it % L, j = it / L;
            const c64 a = vv[i] * conj(pp[j]) + pp[i] * conj(vv[j]);
            c64& t = T[(k + 1 + i) + kLd * (k + 1 + j)];
            t = t - 2.0 * a;
        }
        if (tid == 0) {
            d[k] = T[k + kLd * k].re;
            e[k] = xn;  // |alpha|
            if (alph) alph[k] = alpha;
        }
        __syncthreads();
        if (alph)
            for (int i = tid; i < L; i += kThreads) T[(k + 1 + i) + kLd * k] = vv[i];
    }
    if (tid == 0) {
        if (n >= 2) {
            d[n - 2] = T[(n - 2) + kLd * (n - 2)].re;
            e[n - 2] = sqrt(norm2(T[(n - 1) + kLd * (n - 2)]));
            if (alph) alph[n - 2] = T[(n - 1) + kLd * (n - 2)];
        }
        d[n - 1] = T[(n - 1) + kLd * (n - 1)].re;
    }
    __syncthreads();
}

// Eigenvectors of the Hermitian matrix tridiagonalize(..., alph) reduced (T holds the Householder vectors) for
// its kk eigenvalues lam (descending): inverse iteration on the real tridiagonal (LU with partial pivoting, as
// LAPACK dgttrf / dgttrs, two solves from a fixed start), modified Gram-Schmidt over the kk vectors (vectors of
// close eigenvalues come out mixed; their span is what the projector needs), the diagonal phases taking the real
// tridiagonal to the complex one, then the reflectors in reverse (one warp per vector). Z: n x kk, leading dim kLd.
// Scratch: 5 * kNBMax doubles per vector.
__device__ void ritz_vectors(const c64* T, const double* d, const double* e, const c64* alph, int n, int kk,
                             const double* lam, c64* Z, double* scr) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int kWarps = kThreads / 32;
    if (tid < kk) {  // one thread per eigenvalue: the tridiagonal solves are serial in n
        double* dd = scr + tid * 5 * kNBMax;
        double* du = dd + kNBMax;
        double* du2 = du + kNBMax;
        double* dl = du2 + kNBMax;
        double* x = dl + kNBMax;
        double tnorm = 0.0;
        for (int i = 0; i < n; ++i) tnorm = fmax(tnorm, fabs(d[i]) + (i > 0 ? e[i - 1] : 0.0) + (i + 1 < n ? e[i] : 0.0));
        const double tiny = fmax(2.220446049250313e-16 * tnorm, 1e-300);
        const double l = lam[tid];
        for (int i = 0; i < n; ++i) {
            dd[i] = d[i] - l;
            if (i + 1 < n) {
                du[i] = e[i];
                dl[i] = e[i];
            }
            du2[i] = 0.0;
            x[i] = 1.0 + 0.001 * static_cast<double>((i * 7 + tid * 3) % 11);  // fixed, non-degenerate start
        }
        int piv = 0;  // bit i: rows i, i + 1 interchanged at step i (n <= 72 -> two words)
        unsigned long long pv0 = 0ull, pv1 = 0ull;
        for (int i = 0; i + 1 < n; ++i) {
            if (fabs(dd[i]) >= fabs(dl[i])) {
                if (dd[i] == 0.0) dd[i] = tiny;
                const double fact = dl[i] / dd[i];
                dl[i] = fact;
                dd[i + 1] -= fact * du[i];
            } else {
                const double fact = dd[i] / dl[i];
                dd[i] = dl[i];
                dl[i] = fact;
                const double tmp = du[i];
                du[i] = dd[i + 1];
                dd[i + 1] = tmp - fact * dd[i + 1];
                if (i + 2 < n) {
                    du2[i] = du[i + 1];
                    du[i + 1] = -fact * du[i + 1];
                }
                if (i < 64) pv0 |= 1ull << i;
                else pv1 |= 1ull << (i - 64);
            }
        }
        if (dd[n - 1] == 0.0) dd[n - 1] = tiny;
        for (int i = 0; i < n; ++i)
            if (fabs(dd[i]) < tiny) dd[i] = dd[i] < 0.0 ? -tiny : tiny;
        (void)piv;
        for (int rep = 0; rep < 2; ++rep) {
            for (int i = 0; i + 1 < n; ++i) {  // L solve with the interchanges
                const bool sw = i < 64 ? (pv0 >> i) & 1ull : (pv1 >> (i - 64)) & 1ull;
                if (!sw) {
                    x[i + 1] -= dl[i] * x[i];
                } else {
                    const double t = x[i];
                    x[i] = x[i + 1];
                    x[i + 1] = t - dl[i] * x[i];
                }
            }
            x[n - 1] /= dd[n - 1];  // U solve (diag dd, super du, second super du2)
            if (n >= 2) x[n - 2] = (x[n - 2] - du[n - 2] * x[n - 1]) / dd[n - 2];
            for (int i = n - 3; i >= 0; --i) x[i] = (x[i] - du[i] * x[i + 1] - du2[i] * x[i + 2]) / dd[i];
            double nr = 0.0;
            for (int i = 0; i < n; ++i) nr = fmax(nr, fabs(x[i]));
            const double s = nr > 0.0 ? 1.0 / nr : 1.0;
            for (int i = 0; i < n; ++i) x[i] *= s;
        }
        for (int i = 0; i < n; ++i) Z[i + kLd * tid] = mk(x[i], 0.0);
    }
    __syncthreads();
    if (warp == 0) {  // modified Gram-Schmidt over the kk real vectors (one warp, lanes over rows)
        for (int j = 0; j < kk; ++j) {
            for (int q = 0; q < j; ++q) {
                double dot = 0.0;
                for (int i = lane; i < n; i += 32) dot += Z[i + kLd * q].re * Z[i + kLd * j].re;
                dot = warp_sum(dot);
                for (int i = lane; i < n; i += 32) Z[i + kLd * j].re -= dot * Z[i + kLd * q].re;
                __syncwarp();
            }
            double nr = 0.0;
            for (int i = lane; i < n; i += 32) nr += Z[i + kLd * j].re * Z[i + kLd * j].re;
            nr = warp_sum(nr);
            const double s = nr > 0.0 ? 1.0 / sqrt(nr) : 0.0;
            for (int i = lane; i < n; i += 32) Z[i + kLd * j].re *= s;
            __syncwarp();
        }
    }
    __syncthreads();
    for (int j = warp; j < kk; j += kWarps) {  // phases, then Q = H_0 ... H_{n-3} applied from the right end
        c64* z = Z + kLd * j;
        if (lane == 0) {
            c64 ph = mk(1.0, 0.0);
            for (int i = 0; i < n; ++i) {
                const double zr = z[i].re;
                z[i] = mk(zr * ph.re, zr * ph.im);
                if (i + 1 < n) {
                    const double a = sqrt(norm2(alph[i]));
                    if (a > 0.0) ph = ph * mk(alph[i].re / a, alph[i].im / a);
                }
            }
        }
        __syncwarp();
        for (int k = n - 3; k >= 0; --k) {
            const int L = n - k - 1;
            const c64* v = T + (k + 1) + kLd * k;
            c64 acc = mk(0.0, 0.0);
            for (int i = lane; i < L; i += 32) cmac_conj(acc, v[i], z[k + 1 + i]);
            acc = warp_csum(acc);
            for (int i = lane; i < L; i += 32) z[k + 1 + i] = z[k + 1 + i] - 2.0 * (v[i] * acc);
            __syncwarp();
        }
    }
    __syncthreads();
}

// Number of eigenvalues of the symmetric tridiagonal (d, e) below x (Sturm sequence, with the LAPACK pivmin guard).
__device__ __forceinline__ int sturm_below(const double* d, const double* e, int n, double x, double pivmin) {
    int cnt = 0;
    double q = d[0] - x;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
    for (int i = 1; i < n; ++i) {
        q = (d[i] - x) - e[i - 1] * e[i - 1] / q;
        if (fabs(q) < pivmin) q = -pivmin;
        cnt += q < 0.0;
    }
    return cnt;
}

// The kk largest eigenvalues of (d, e), descending, to the bisection limit (relative 1e-17 of the spectrum span):
// 16 threads per eigenvalue, each round evaluates 15 interior points and keeps the sub-interval holding it.
__device__ void top_eigenvalues(const double* d, const double* e, int n, int kk, double* out, double* lohi) {
    const int tid = threadIdx.x;
    __shared__ double s_lo[kBMax], s_hi[kBMax];
    __shared__ int s_cnt[kBMax][16];
    if (tid == 0) {  // Gershgorin bounds
        double lo = INFINITY, hi = -INFINITY, emax = 0.0;
        for (int i = 0; i < n; ++i) {
            const double r = (i > 0 ? e[i - 1] : 0.0) + (i + 1 < n ? e[i] : 0.0);
            lo = fmin(lo, d[i] - r);
            hi = fmax(hi, d[i] + r);
            if (i + 1 < n) emax = fmax(emax, e[i] * e[i]);
        }
        const double w = fmax(hi - lo, 1e-300);
        lohi[0] = lo - 1e-14 * w;
        lohi[1] = hi + 1e-14 * w;
        lohi[2] = fmax(2.2250738585072014e-308, 2.220446049250313e-16 * emax);  // pivmin (LAPACK dstebz)
    }
    __syncthreads();
    const int j = tid >> 4, u = tid & 15;  // eigenvalue j (0 = largest), probe u
    if (j < kk && u == 0) {
        s_lo[j] = lohi[0];
        s_hi[j] = lohi[1];
    }
    __syncthreads();
    const double pivmin = lohi[2];
    for (int round = 0; round < 20; ++round) {  // 16^20 >> 2^64: converged well before
        if (j < kk) {
            const double lo = s_lo[j], hi = s_hi[j];
            const double x = lo + (hi - lo) * (u + 1) / 16.0;
            s_cnt[j][u] = u < 15 ? sturm_below(d, e, n, x, pivmin) : n;
        }
        __syncthreads();
        if (j < kk && u == 0) {
            // the (n - 1 - j)-th smallest eigenvalue (0-based) lies where the count first exceeds n - 1 - j
            const int target = n - 1 - j;
            const double lo = s_lo[j], hi = s_hi[j];
            int b = 0;
            while (b < 15 && s_cnt[j][b] <= target) ++b;
            const double nlo = b == 0 ? lo : lo + (hi - lo) * b / 16.0;
            const double nhi = lo + (hi - lo) * (b + 1) / 16.0;
            s_lo[j] = nlo;
            s_hi[j] = b == 15 ? hi : nhi;
        }
        __syncthreads();
    }
    if (j < kk && u == 0) out[j] = 0.5 * (s_lo[j] + s_hi[j]);
    __syncthreads();
}

template <typename TS>
__global__ void __launch_bounds__(kThreads, 1) k_lanczos_batch(Args a) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    c64* A = reinterpret_cast<c64*>(smem_raw);
    c64* V = A + kLd * kNBMax;
    c64* strip = V + kLd * kNBMax;                // kNBMax x kBMax, row-major [r][c]
    double* vals = reinterpret_cast<double*>(strip + kNBMax * kBMax);  // [kBMax]
    double* prev = vals + kBMax;                                   // [kBMax]
    double* nrm = prev + kBMax;                                    // [kBMax] column norms^2 (orthonormal_range)
    int* top = reinterpret_cast<int*>(nrm + kBMax);                // [kBMax]
    int* ctl = top + kBMax;  // [0] any rotation, [1] ncols, [2] bq, [3] done, [4] stable, [5] have_prev, [6] flags,
                             // [7] rank, [8] pivot, [9] iterations
    double* dctl = reinterpret_cast<double*>(ctl + 16);  // [0] last change, [1] thr helper, [2] max pivot, [3] amax,
                                                         // [4..5] tridiagonalisation, [6..8] bisection bounds
    double* td = dctl + 16;                               // [kNBMax] tridiagonal diagonal
    double* te = td + kNBMax;                             // [kNBMax] |off-diagonal|
    c64* tv = reinterpret_cast<c64*>(te + kNBMax);        // [kNBMax] Householder vector
    c64* tp = tv + kNBMax;                                // [kNBMax] T v / w

    const int f = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int kWarps = kThreads / 32;
    const int M = a.m, K = a.k;
    const TS* S = reinterpret_cast<const TS*>(a.S) + static_cast<size_t>(f) * M * M * 2;
    c64* B = reinterpret_cast<c64*>(a.basis) + static_cast<size_t>(f) * kNBMax * M;
    c64* W = reinterpret_cast<c64*>(a.W) + static_cast<size_t>(f) * M * kBMax;
    c64* Z = reinterpret_cast<c64*>(a.Z) + static_cast<size_t>(f) * M * kBMax;
    const c64* Q0 = reinterpret_cast<const c64*>(a.q0);

    for (int i = tid; i < M * a.b0; i += kThreads) B[i] = Q0[i];
    if (tid == 0) {
        ctl[1] = a.b0;
        ctl[2] = a.b0;
        ctl[3] = 0;
        ctl[4] = 0;
        ctl[5] = 0;
        ctl[6] = 0;
        ctl[9] = 0;
        ctl[10] = 0;
        dctl[0] = INFINITY;
    }
    __syncthreads();

    LZ_T0();
    for (int it = 0; it < a.max_iter; ++it) {
        const int ncols = ctl[1], bq = ctl[2], old = ncols - bq;
        // ---- W = S Q (Q = basis columns [old, ncols))
        for (int i = tid; i < M; i += kThreads) {
            c64 acc[kBMax];
#pragma unroll
            for (int c = 0; c < kBMax; ++c) acc[c] = mk(0.0, 0.0);
            const c64* Qc = B + static_cast<size_t>(old) * M;
            // eight independent S loads in flight per thread (one CTA per SM: the S stream is latency-bound; a
            // double-buffered variant with the next group's loads in flight measured slower, tools/lz_timeline.py)
            int j0 = 0;
            for (; j0 + 8 <= M; j0 += 8) {
                c64 sv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) sv[u] = ld_s<TS>(S + (static_cast<size_t>(j0 + u) * M + i) * 2);
#pragma unroll
                for (int u = 0; u < 8; ++u)
#pragma unroll
                    for (int c = 0; c < kBMax; ++c)
                        if (c < bq) cmac_conj(acc[c], sv[u], Qc[static_cast<size_t>(c) * M + j0 + u]);
            }
            for (int j = j0; j < M; ++j) {
                const c64 sji = ld_s<TS>(S + (static_cast<size_t>(j) * M + i) * 2);  // S(j, i) = conj S(i, j)
#pragma unroll
                for (int c = 0; c < kBMax; ++c)
                    if (c < bq) cmac_conj(acc[c], sji, Qc[static_cast<size_t>(c) * M + j]);  // conj(S(j,i)) Q(j,c)
            }
#pragma unroll
            for (int c = 0; c < kBMax; ++c)
                if (c < bq) W[i * kBMax + c] = acc[c];
        }
        __syncthreads();
        LZ_MARK(0);  // W = S Q
        // ---- strip = basis^H W (ncols x bq)
        block_ah_x(B, W, strip, M, ncols, bq, warp, lane);
        __syncthreads();
        LZ_MARK(1);  // strip
        // ---- extend h (raw, in A) by the strip: A[:old, new] = strip[:old], A[new, new] = Herm(strip[new])
        for (int e = tid; e < old * bq; e += kThreads) {
            const int x = e % old, c = e / old;
            const c64 v = strip[x * kBMax + c];
            A[x + kLd * (old + c)] = v;
            A[(old + c) + kLd * x] = conj(v);
        }
        for (int e = tid; e < bq * bq; e += kThreads) {
            const int r = e % bq, c = e / bq;
            const c64 hrc = strip[(old + r) * kBMax + c], hcr = strip[(old + c) * kBMax + r];
            A[(old + r) + kLd * (old + c)] = 0.5 * (hrc + conj(hcr));  // HermitianMatrix(h), R/src/linalg.cpp:51
        }
        __syncthreads();
        // ---- Ritz values of h: tridiagonalise a copy (in V), top-K by multisection
        for (int e = tid; e < ncols * ncols; e += kThreads) {
            const int x = e % ncols, c = e / ncols;
            V[x + kLd * c] = A[x + kLd * c];
        }
        __syncthreads();
        const int kk0 = min(K, ncols);
        if (tid == 0) ctl[11] = ncols;  // size of the h the Ritz values below belong to
        LZ_MARK(2);  // extend + copy
        tridiagonalize(V, ncols, td, te, tv, tp, dctl + 4);
        LZ_MARK(3);  // tridiagonalise
        top_eigenvalues(td, te, ncols, kk0, vals, dctl + 6);
        LZ_MARK(4);  // bisection
        if (tid == 0) {
            const int kk = kk0;
            int done = 0;
            if (ctl[5] && kk == K) {
                double change = 0.0;
                for (int j = 0; j < K; ++j) change = fmax(change, fabs(vals[j] - prev[j]) / fmax(fabs(vals[j]), 1e-300));
                dctl[0] = change;
                ctl[4] = change <= kTol ? ctl[4] + 1 : 0;
                if (ctl[4] >= 2) done = 1;
            }
            if (!done) {
                for (int j = 0; j < kk; ++j) prev[j] = vals[j];
                ctl[5] = (kk == K);
                if (M - ncols <= 0) done = 1;  // the basis spans the space: Ritz pairs exact
            }
            ctl[3] = done;
            ctl[9] = it + 1;
        }
        __syncthreads();
        if (ctl[3]) break;
        // ---- z = W - B (B^H W); z -= B (B^H z)
        block_sub(B, W, Z, strip, M, ncols, bq);
        __syncthreads();
        block_ah_x(B, Z, strip, M, ncols, bq, warp, lane);
        __syncthreads();
        block_sub(B, Z, Z, strip, M, ncols, bq);
        __syncthreads();
        LZ_MARK(5);  // two Gram-Schmidt passes
        // ---- q = orthonormal_range(z(:, 1:bz)): column-pivoted CGS2, Eigen ColPivHouseholderQR::rank() rule
        // (nonzero pivots while |R_kk|^2 >= (maxColNorm eps)^2 / rows (rows - k), then |R_kk| > eps size maxpivot)
        const int room = M - ncols;
        const int bz = min(bq, room);
        unsigned remaining = (bz >= 32 ? 0xffffffffu : ((1u << bz) - 1u));
        int rank = 0;
        for (int step = 0; step < bz; ++step) {
            for (int c = warp; c < bz; c += kWarps) {
                if (!((remaining >> c) & 1u)) continue;
                double s2 = 0.0;
                for (int i = lane; i < M; i += 32) s2 += norm2(Z[i * kBMax + c]);
                s2 = warp_sum(s2);
                if (lane == 0) nrm[c] = s2;
            }
            __syncthreads();
            if (tid == 0) {
                int p = -1;
                double best = -1.0;
                for (int c = 0; c < bz; ++c)
                    if (((remaining >> c) & 1u) && nrm[c] > best) {
                        best = nrm[c];
                        p = c;
                    }
                if (step == 0) dctl[1] = best * (2.220446049250313e-16 * 2.220446049250313e-16) / M;  // thr helper
                const double rkk = sqrt(best);
                if (step == 0) dctl[2] = rkk;
                const bool ok = best >= dctl[1] * (M - step) && rkk > 2.220446049250313e-16 * bz * dctl[2] && best > 0.0;
                ctl[8] = ok ? p : -1;
            }
            __syncthreads();
            const int p = ctl[8];
            if (p < 0) break;
            const double inv = 1.0 / sqrt(nrm[p]);
            c64* qn = B + static_cast<size_t>(ncols + rank) * M;
            if (ncols + rank < kNBMax)
                for (int i = tid; i < M; i += kThreads) qn[i] = inv * Z[i * kBMax + p];
            remaining &= ~(1u << p);
            ++rank;
            __syncthreads();
            if (ncols + rank > kNBMax) break;
            for (int pass = 0; pass < 2; ++pass) {  // CGS2 of the remaining columns against q
                for (int c = warp; c < bz; c += kWarps) {
                    if (!((remaining >> c) & 1u)) continue;
                    c64 acc = mk(0.0, 0.0);
                    for (int i = lane; i < M; i += 32) cmac_conj(acc, qn[i], Z[i * kBMax + c]);
                    acc = warp_csum(acc);
                    if (lane == 0) strip[c] = acc;
                }
                __syncthreads();
                for (int e = tid; e < M * bz; e += kThreads) {
                    const int i = e / bz, c = e - i * bz;
                    if ((remaining >> c) & 1u) Z[i * kBMax + c] = Z[i * kBMax + c] - qn[i] * strip[c];
                }
                __syncthreads();
            }
        }
        LZ_MARK(6);  // orthonormal_range
        if (tid == 0) {
            if (rank == 0) ctl[3] = 1;  // invariant Krylov space: the Ritz pairs are exact
            else if (ncols + rank > kNBMax) {
                ctl[6] |= kFrameCap;
                ctl[3] = 1;
            } else {
                ctl[1] = ncols + rank;
                ctl[2] = rank;
            }
        }
        __syncthreads();
        if (ctl[3]) break;
    }
    LZ_MARK(8);  // exit
    // ---- outputs (the estimate of the last Ritz problem); the iteration cap without convergence -> NOCONV
    const bool capped = !ctl[3];
    const int hn = ctl[11];  // the h of the last Ritz values (the basis may hold one more block after the cap)
    const int kk = min(K, hn);
    // Ritz vectors of h for those values: tridiagonalise a copy keeping the reflectors, inverse iteration, back-
    // transformation (ritz_vectors); Z and the solver scratch live in A's space once h is copied out
    for (int e = tid; e < hn * hn; e += kThreads) {
        const int x = e % hn, c = e / hn;
        V[x + kLd * c] = A[x + kLd * c];
    }
    __syncthreads();
    c64* Zs = A;                                                  // kLd x kk
    double* scr = reinterpret_cast<double*>(A + kLd * kBMax);     // kBMax x 5 x kNBMax
    c64* alph = reinterpret_cast<c64*>(scr + kBMax * 5 * kNBMax);  // kNBMax
    tridiagonalize(V, hn, td, te, tv, tp, dctl + 4, alph);
    ritz_vectors(V, td, te, alph, hn, kk, vals, Zs, scr);
    LZ_MARK(7);  // Ritz vectors
    double* ob = a.out_basis + static_cast<size_t>(f) * K * M * 2;
    for (int e = tid; e < M * K; e += kThreads) {
        const int j = e / M, i = e - j * M;
        c64 u = mk(0.0, 0.0);
        if (j < kk)
            for (int r = 0; r < hn; ++r) u = u + B[static_cast<size_t>(r) * M + i] * Zs[r + kLd * j];
        ob[2 * e] = u.re;
        ob[2 * e + 1] = u.im;
    }
    if (tid < K) {
        double v = tid < kk ? vals[tid] : 0.0;
        if (v < 0.0 && v >= -1e-10) v = 0.0;  // clamp_nonnegative, R/src/estimators.cpp:25-31
        a.out_eig[static_cast<size_t>(f) * K + tid] = v;
    }
    if (tid == 0) {
        int flags = ctl[6] | (capped ? kFrameNoConv : 0) | ((ctl[6] & kFrameCap) ? kFrameNoConv : 0);
        if (flags) atomicOr(&a.status[f], flags);
        if (a.last_change) a.last_change[f] = dctl[0];
        if (a.iters) a.iters[f] = ctl[9] * 10000;  // Krylov iterations
    }
}

}  // namespace lzb
}  // namespace fmk

// Start block of block_lanczos_subspace (R/src/estimators.cpp:161-163): an orthonormal basis of
// span(gaussian_matrix(M, b, 0x6C616E637A6F)) (the Krylov space, hence every Ritz value, depends only on the span),
// M x b complex128 column-major, by two passes of modified Gram-Schmidt in fp64.
std::vector<double> fm_lanczos_start_block(int64_t m, int b) {
    constexpr uint64_t kStartSeed = 0x6C616E637A6FULL;
    std::vector<double> g(static_cast<size_t>(m * b));
    fmhost::gaussian_matrix_real(m, b, kStartSeed, g.data());  // row-major M x b
    std::vector<double> q(static_cast<size_t>(2 * m * b), 0.0);
    for (int c = 0; c < b; ++c) {
        std::vector<double> v(static_cast<size_t>(m));
        for (int64_t i = 0; i < m; ++i) v[i] = g[static_cast<size_t>(i * b + c)];
        for (int pass = 0; pass < 2; ++pass)
            for (int r = 0; r < c; ++r) {
                double dot = 0.0;
                for (int64_t i = 0; i < m; ++i) dot += q[2 * (static_cast<size_t>(r) * m + i)] * v[i];
                for (int64_t i = 0; i < m; ++i) v[i] -= dot * q[2 * (static_cast<size_t>(r) * m + i)];
            }
        double nrm = 0.0;
        for (int64_t i = 0; i < m; ++i) nrm += v[i] * v[i];
        nrm = std::sqrt(nrm);
        for (int64_t i = 0; i < m; ++i) q[2 * (static_cast<size_t>(c) * m + i)] = v[i] / nrm;
    }
    return q;
}

size_t fm_lanczos_batch_smem() {
    using namespace fmk::lzb;
    return sizeof(fmk::c64) * (2 * kLd * kNBMax + kNBMax * kBMax) +
           sizeof(double) * 3 * kBMax + sizeof(int) * (kBMax + 16) + sizeof(double) * (16 + 2 * kNBMax) +
           sizeof(fmk::c64) * 2 * kNBMax + 64;
}
int fm_lanczos_batch_bmax() { return fmk::lzb::kBMax; }
int fm_lanczos_batch_nbmax() { return fmk::lzb::kNBMax; }
int32_t fm_lanczos_batch_cap_flag() { return fmk::lzb::kFrameCap; }

// S: frames x M x M Hermitian (row-major, full), element type TS (float: complex64, double: complex128).
// Workspace: basis frames x kNBMax x M, W / Z frames x M x kBMax (complex128 each).
template <typename TS>
cudaError_t fm_launch_lanczos_batch(const void* S, const double* q0, double* basis_ws, double* w_ws, double* z_ws,
                                    double* out_basis, double* out_eig, int32_t* status, double* last_change,
                                    int32_t* iters, int frames, int m, int k, int b0, int max_iter, cudaStream_t s) {
    using namespace fmk::lzb;
    if (frames < 1) return cudaSuccess;
    if (b0 < 1 || b0 > kBMax || k < 1 || k > b0 || m < 2) return cudaErrorInvalidValue;
    const size_t smem = fm_lanczos_batch_smem();
    static bool attr[2] = {false, false};
    if (!attr[sizeof(TS) == 8]) {
        cudaError_t e = cudaFuncSetAttribute(k_lanczos_batch<TS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        attr[sizeof(TS) == 8] = true;
    }
    Args a{S, q0, basis_ws, w_ws, z_ws, out_basis, out_eig, status, last_change, iters, m, k, b0, max_iter};
    k_lanczos_batch<TS><<<frames, kThreads, smem, s>>>(a);
    return cudaGetLastError();
}

template cudaError_t fm_launch_lanczos_batch<float>(const void*, const double*, double*, double*, double*, double*,
                                                    double*, int32_t*, double*, int32_t*, int, int, int, int, int,
                                                    cudaStream_t);
template cudaError_t fm_launch_lanczos_batch<double>(const void*, const double*, double*, double*, double*, double*,
                                                     double*, int32_t*, double*, int32_t*, int, int, int, int, int,
                                                     cudaStream_t);

fm_status fm_set_error(fm_status s, const std::string& msg);  // capi.cu
fm_status fm_fail_cuda(cudaError_t e, const char* expr, const char* file, int line);

// Batched block_lanczos_subspace on device-resident covariance matrices (see the header).
extern "C" fm_status fm_block_lanczos_batch(const float* s, int64_t frames, int64_t m, int64_t k, int64_t block,
                                            int32_t max_iterations, double* basis, double* eigenvalues,
                                            int32_t* status, int32_t* iterations, void* stream) {
    if (frames < 1 || m < 2 || !s || !basis || !eigenvalues || !status)
        return fm_set_error(FM_EINVAL, "block_lanczos_batch: empty batch or null pointer");
    if (k < 1 || k >= m) return fm_set_error(FM_EINVAL, "block_lanczos_subspace: need 1 <= K < M");
    if (block < k) return fm_set_error(FM_EINVAL, "block_lanczos_subspace: need block >= K");
    if (max_iterations < 1) return fm_set_error(FM_EINVAL, "block_lanczos_subspace: iters >= 1");
    const int b0 = static_cast<int>(std::min<int64_t>(block, m));
    if (b0 > fmk::lzb::kBMax) return fm_set_error(FM_ENOTSUP, "block_lanczos_batch: block <= 16 supported");
    if (frames > 0x7fffffff || m > 0x7fff) return fm_set_error(FM_EINVAL, "block_lanczos_batch: batch too large");
    cudaStream_t q = static_cast<cudaStream_t>(stream);
    const auto q0 = fm_lanczos_start_block(m, b0);
    const size_t nb = fmk::lzb::kNBMax, bm = fmk::lzb::kBMax;
    const size_t doubles = q0.size() + 2 * static_cast<size_t>(frames) * m * (nb + 2 * bm);
    double* ws = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&ws), sizeof(double) * doubles, q);
    if (e == cudaSuccess) e = cudaMemcpyAsync(ws, q0.data(), sizeof(double) * q0.size(), cudaMemcpyHostToDevice, q);
    if (e == cudaSuccess) e = cudaMemsetAsync(status, 0, sizeof(int32_t) * frames, q);
    if (e == cudaSuccess) {
        double* lb = ws + q0.size();
        double* lw = lb + 2 * static_cast<size_t>(frames) * m * nb;
        double* lz = lw + 2 * static_cast<size_t>(frames) * m * bm;
        e = fm_launch_lanczos_batch<float>(s, ws, lb, lw, lz, basis, eigenvalues, status, nullptr, iterations,
                                           static_cast<int>(frames), static_cast<int>(m), static_cast<int>(k), b0,
                                           max_iterations, q);
    }
    if (ws) cudaFreeAsync(ws, q);
    if (e != cudaSuccess) return fm_fail_cuda(e, "fm_block_lanczos_batch", __FILE__, __LINE__);
    return FM_OK;
}

// Debug / test hook: the Ritz-value kernel path on one Hermitian matrix (h n x n complex128 column-major, n <= 72):
// Householder tridiagonalisation + Sturm multisection, the kk largest eigenvalues descending into out (device).
namespace fmk {
namespace lzb {
__global__ void __launch_bounds__(kThreads, 1) k_ritz_probe(const c64* h, int n, int kk, double* out) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    c64* T = reinterpret_cast<c64*>(smem_raw);
    double* d = reinterpret_cast<double*>(T + kLd * kNBMax);
    double* e = d + kNBMax;
    c64* vv = reinterpret_cast<c64*>(e + kNBMax);
    c64* pp = vv + kNBMax;
    double* red = reinterpret_cast<double*>(pp + kNBMax);
    for (int i = threadIdx.x; i < n * n; i += kThreads) T[(i % n) + kLd * (i / n)] = h[i];
    __syncthreads();
    tridiagonalize(T, n, d, e, vv, pp, red);
    top_eigenvalues(d, e, n, kk, out, red + 4);
}
}  // namespace lzb
}  // namespace fmk

extern "C" fm_status fm_debug_ritz_values(const double* h, int32_t n, int32_t kk, double* out) {
    using namespace fmk::lzb;
    if (n < 2 || n > kNBMax || kk < 1 || kk > kBMax || kk > n) return fm_set_error(FM_EINVAL, "ritz probe: bad size");
    const size_t smem = sizeof(fmk::c64) * (kLd * kNBMax + 2 * kNBMax) + sizeof(double) * (2 * kNBMax + 16);
    double *dh = nullptr, *dout = nullptr;
    cudaMalloc(&dh, sizeof(double) * 2 * n * n);
    cudaMalloc(&dout, sizeof(double) * kk);
    cudaMemcpy(dh, h, sizeof(double) * 2 * n * n, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k_ritz_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k_ritz_probe<<<1, kThreads, smem>>>(reinterpret_cast<const fmk::c64*>(dh), n, kk, dout);
    cudaError_t err = cudaMemcpy(out, dout, sizeof(double) * kk, cudaMemcpyDeviceToHost);
    cudaFree(dh);
    cudaFree(dout);
    if (err != cudaSuccess) return fm_fail_cuda(err, "fm_debug_ritz_values", __FILE__, __LINE__);
    return FM_OK;
}

#ifdef FM_LZ_TIMELINE
extern "C" int fm_debug_lz_timeline(long long* host, int zero) {
    if (zero) {
        static long long z[16] = {};
        return static_cast<int>(cudaMemcpyToSymbol(fmk::lzb::g_lz_tl, z, sizeof(z)));
    }
    return static_cast<int>(cudaMemcpyFromSymbol(host, fmk::lzb::g_lz_tl, sizeof(long long) * 16));
}
#endif
