// Batched block-Lanczos signal subspace: block_lanczos_subspace, R/src/estimators.cpp:154-222
// (orthonormal_range :143-149), the paper's accurate baseline, for a whole batch of frames in ONE launch.
//
// One CTA per frame runs the reference's control flow on the device, in fp64 (the 1e-10 Ritz-value tolerance needs
// fp64 end to end; S is read as stored: complex64 R of the batch plan, or complex128 for the facade):
//   W = S Q                       thread per row, S read down its columns (S Hermitian: S(i, j) = conj S(j, i), so
//                                 the reads are coalesced), Q broadcast from the frame's basis columns
//   strip = basis^H W             warp per entry
//   h grows by the strip          kept in its Ritz basis: A = V^H h V with V the accumulated Jacobi rotations, so the
//                                 new strip only needs V_old^H strip and the Hermitian new corner (warm start)
//   Ritz values                   two-sided cyclic Jacobi on A (parallel round-robin pairs, complex rotations), V
//                                 accumulated in shared memory; top-K of diag(A)
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
#include <vector>

#include "../../include/fastmusic_b200.h"
#include "fm_common.cuh"
#include "host_rng.hpp"

namespace fmk {
namespace lzb {

constexpr int kThreads = 256;
constexpr int kBMax = 16;   // block columns per expansion
constexpr int kNBMax = 72;  // basis columns: A, V complex128 72 x 72 each in shared memory
constexpr int kMaxSweeps = 60;
constexpr double kTol = 1e-10;  // R/src/estimators.cpp:160

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

// Round-robin pairing (circle method) over n2 (even) slots: step r in [0, n2 - 1), pair t in [0, n2 / 2).
__device__ __forceinline__ void rr_pair(int r, int t, int n2, int& p, int& q) {
    const int L = n2 - 1;
    int a, b;
    if (t == 0) {
        a = r;
        b = L;
    } else {
        a = (r + t) % L;
        b = (r - t + L) % L;
    }
    p = min(a, b);
    q = max(a, b);
}

struct Rot {
    int p, q;
    double c, s;
    c64 e;  // phase of A(p, q)
    double t_g;  // t |A(p, q)| (diagonal update)
};

// Two-sided cyclic Jacobi on the Hermitian n x n leading block of A (column-major, leading dim kNBMax),
// accumulating the rotations into V's n x n block. Returns the number of sweeps (kMaxSweeps + 1: no convergence).
// Rotation threshold: |A(p, q)| <= 2^-52 max_i |A(i, i)| is at the rounding level of the matrix (a purely relative
// test, |A(p, q)| <= eps sqrt|A(p, p) A(q, q)|, keeps re-rotating the rounding noise that rotations of large entries
// leave between pairs of small ones, and never ends); the top-K Ritz values it decides are then exact to that level.
__device__ int jacobi_sweeps(c64* A, c64* V, int n, Rot* rot, int* s_any, double* s_amax) {
    const int n2 = n + (n & 1);
    const int np = n2 / 2;
    const int tid = threadIdx.x;
    for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
        if (tid == 0) {
            *s_any = 0;
            double am = 0.0;
            for (int x = 0; x < n; ++x) am = fmax(am, fabs(A[x + kNBMax * x].re));
            *s_amax = am;
        }
        __syncthreads();
        const double thr = 2.220446049250313e-16 * *s_amax;
        for (int r = 0; r < n2 - 1; ++r) {
            if (tid < np) {
                int p, q;
                rr_pair(r, tid, n2, p, q);
                Rot o;
                o.p = p;
                o.q = q;
                o.c = 1.0;
                o.s = 0.0;
                o.e = mk(1.0, 0.0);
                o.t_g = 0.0;
                if (q < n) {
                    const c64 apq = A[p + kNBMax * q];
                    const double g = sqrt(norm2(apq));
                    const double app = A[p + kNBMax * p].re, aqq = A[q + kNBMax * q].re;
                    // skip rotations below the relative accuracy of the pair (and denormal-size entries)
                    if (g > 1e-290 && g > thr) {
                        const double tau = (aqq - app) / (2.0 * g);
                        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                        o.c = 1.0 / sqrt(1.0 + t * t);
                        o.s = t * o.c;
                        o.e = mk(apq.re / g, apq.im / g);
                        o.t_g = t * g;
                        *s_any = 1;
                    } else {
                        o.q = -1;  // inactive
                    }
                } else {
                    o.q = -1;
                }
                rot[tid] = o;
            }
            __syncthreads();
            // columns: A <- A J, V <- V J with J = [[c, s e], [-s conj(e), c]] on (p, q)
            for (int it = tid; it < np * n; it += kThreads) {
                const int t = it / n, row = it - t * n;
                const Rot o = rot[t];
                if (o.q < 0) continue;
                const c64 ep = mk(o.s * o.e.re, o.s * o.e.im);  // s e
                {
                    const c64 ap = A[row + kNBMax * o.p], aq = A[row + kNBMax * o.q];
                    A[row + kNBMax * o.p] = o.c * ap - conj(ep) * aq;
                    A[row + kNBMax * o.q] = ep * ap + o.c * aq;
                }
                {
                    const c64 vp = V[row + kNBMax * o.p], vq = V[row + kNBMax * o.q];
                    V[row + kNBMax * o.p] = o.c * vp - conj(ep) * vq;
                    V[row + kNBMax * o.q] = ep * vp + o.c * vq;
                }
            }
            __syncthreads();
            // rows: A <- J^H A (J^H = [[c, -s e], [s conj(e), c]])
            for (int it = tid; it < np * n; it += kThreads) {
                const int t = it / n, col = it - t * n;
                const Rot o = rot[t];
                if (o.q < 0) continue;
                const c64 ep = mk(o.s * o.e.re, o.s * o.e.im);
                const c64 ap = A[o.p + kNBMax * col], aq = A[o.q + kNBMax * col];
                A[o.p + kNBMax * col] = o.c * ap - ep * aq;
                A[o.q + kNBMax * col] = conj(ep) * ap + o.c * aq;
            }
            __syncthreads();
            if (tid < np) {  // the pair's closed form: zero off-diagonal, real diagonal
                const Rot o = rot[tid];
                if (o.q >= 0) {
                    A[o.p + kNBMax * o.q] = mk(0.0, 0.0);
                    A[o.q + kNBMax * o.p] = mk(0.0, 0.0);
                    A[o.p + kNBMax * o.p].im = 0.0;
                    A[o.q + kNBMax * o.q].im = 0.0;
                }
            }
            __syncthreads();
        }
        if (*s_any == 0) return sweep + 1;
        __syncthreads();
    }
    return kMaxSweeps + 1;
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

template <typename TS>
__global__ void __launch_bounds__(kThreads, 1) k_lanczos_batch(Args a) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    c64* A = reinterpret_cast<c64*>(smem_raw);
    c64* V = A + kNBMax * kNBMax;
    c64* strip = V + kNBMax * kNBMax;                // kNBMax x kBMax, row-major [r][c]
    Rot* rot = reinterpret_cast<Rot*>(strip + kNBMax * kBMax);
    double* vals = reinterpret_cast<double*>(rot + kNBMax / 2);  // [kBMax]
    double* prev = vals + kBMax;                                   // [kBMax]
    double* nrm = prev + kBMax;                                    // [kBMax] column norms^2 (orthonormal_range)
    int* top = reinterpret_cast<int*>(nrm + kBMax);                // [kBMax]
    int* ctl = top + kBMax;  // [0] any rotation, [1] ncols, [2] bq, [3] done, [4] stable, [5] have_prev, [6] flags,
                             // [7] rank, [8] pivot, [9] iterations
    double* dctl = reinterpret_cast<double*>(ctl + 16);  // [0] last change, [1] thr helper, [2] max pivot, [3] amax

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

    for (int it = 0; it < a.max_iter; ++it) {
        const int ncols = ctl[1], bq = ctl[2], old = ncols - bq;
        // ---- W = S Q (Q = basis columns [old, ncols))
        for (int i = tid; i < M; i += kThreads) {
            c64 acc[kBMax];
#pragma unroll
            for (int c = 0; c < kBMax; ++c) acc[c] = mk(0.0, 0.0);
            const c64* Qc = B + static_cast<size_t>(old) * M;
            // eight independent S loads in flight per thread (one CTA per SM: the S stream is latency-bound)
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
        // ---- strip = basis^H W (ncols x bq)
        block_ah_x(B, W, strip, M, ncols, bq, warp, lane);
        __syncthreads();
        // ---- extend A = V^H h V by the new block (warm start) and V by the identity
        for (int e = tid; e < old * bq; e += kThreads) {
            const int x = e % old, c = e / old;
            c64 acc = mk(0.0, 0.0);
            for (int r = 0; r < old; ++r) cmac_conj(acc, V[r + kNBMax * x], strip[r * kBMax + c]);
            A[x + kNBMax * (old + c)] = acc;
            A[(old + c) + kNBMax * x] = conj(acc);
        }
        for (int e = tid; e < bq * bq; e += kThreads) {
            const int r = e % bq, c = e / bq;
            const c64 hrc = strip[(old + r) * kBMax + c], hcr = strip[(old + c) * kBMax + r];
            A[(old + r) + kNBMax * (old + c)] = 0.5 * (hrc + conj(hcr));  // HermitianMatrix(h), R/src/linalg.cpp:51
        }
        for (int e = tid; e < ncols * bq; e += kThreads) {
            const int x = e % ncols, c = e / ncols;
            V[x + kNBMax * (old + c)] = mk(x == old + c ? 1.0 : 0.0, 0.0);
            if (x < old) V[(old + c) + kNBMax * x] = mk(0.0, 0.0);
        }
        __syncthreads();
        const int sweeps = jacobi_sweeps(A, V, ncols, rot, &ctl[0], &dctl[3]);
        if (tid == 0) ctl[10] += sweeps;
        // ---- Ritz values: top-K of diag(A), descending (ties: lower index)
        if (tid == 0) {
            const int kk = min(K, ncols);
            for (int j = 0; j < kk; ++j) {
                int best = -1;
                double bv = 0.0;
                for (int x = 0; x < ncols; ++x) {
                    bool used = false;
                    for (int u = 0; u < j; ++u) used |= (top[u] == x);
                    if (used) continue;
                    const double v = A[x + kNBMax * x].re;
                    if (best < 0 || v > bv) {
                        best = x;
                        bv = v;
                    }
                }
                top[j] = best;
                vals[j] = bv;
            }
            if (sweeps > kMaxSweeps) ctl[6] |= kFrameNoConv;
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
    // ---- outputs (the estimate of the last Ritz problem); the iteration cap without convergence -> NOCONV
    const bool capped = !ctl[3];
    const int ncols = ctl[1];
    const int kk = min(K, ncols);
    double* ob = a.out_basis + static_cast<size_t>(f) * K * M * 2;
    for (int e = tid; e < M * K; e += kThreads) {
        const int j = e / M, i = e - j * M;
        c64 u = mk(0.0, 0.0);
        if (j < kk)
            for (int r = 0; r < ncols; ++r) u = u + B[static_cast<size_t>(r) * M + i] * V[r + kNBMax * top[j]];
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
        if (a.iters) a.iters[f] = ctl[9] * 10000 + ctl[10];  // iterations, total Jacobi sweeps
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
    return sizeof(fmk::c64) * (2 * kNBMax * kNBMax + kNBMax * kBMax) + sizeof(Rot) * (kNBMax / 2) +
           sizeof(double) * 3 * kBMax + sizeof(int) * (kBMax + 16) + sizeof(double) * 4 + 64;
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
