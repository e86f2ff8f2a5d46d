// K3/K4 for the batched complex64 path — block-per-frame small-matrix kernels (p <= 32)
// designed around short critical paths: every phase is spread over the whole CTA.
//
// k_cholqr_blk (R/src/linalg.cpp:127-141 qr_orthonormal; Eigen ColPivHouseholderQR rank rule)
//   G = C^H C in fp64 (products of fp32 data are exact in fp64) -> masked outer-product
//   pivoted Cholesky over all threads (pivot = largest remaining Schur diagonal = Eigen's
//   largest remaining column norm, so |R_kk| = sqrt(pivot_k) is the pivoted-QR diagonal in
//   exact arithmetic) -> rows of C P R^-1 by forward substitution (thread per row).
//   MODE 0: V (complex64) for the power iteration + rank flag (fp32 epsilon).
//   MODE 1: CholQR2 -> Q (fp64) + Rt = Q^H C + H = V^H C for the Nystrom tail.
// k_nystrom_blk (R/src/estimators.cpp:37-50 rank_restricted_subspace + :25-31 clamp;
//                R/src/linalg.cpp:143-163 pseudo_inverse)
//   H (Hermitian PD) = L_H L_H^H, so W = pinv(H) = L_H^-H L_H^-1 and B' = Rt W Rt^H = Y Y^H with
//   Y = Rt L_H^-H. The top-K eigenvectors of B' are the top-K left singular vectors of Y:
//   one-sided Jacobi on Y's columns (one warp per column pair per round), eigenvalues = s^2.
//   B' is never formed. A Cholesky pivot below p*eps_32*max is flagged (degenerate pinv).

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "fm_common.cuh"

namespace fmk {
namespace smb {

constexpr int kNT = 256;
// latency-bound small-matrix kernels: frames (warps) per CTA and register caps (tuning switches)
#ifndef FM_GRAM_RG32
#define FM_GRAM_RG32 4
#endif
#ifndef FM_JACOBI_TOL32
#define FM_JACOBI_TOL32 1e-6f  // fp32 Jacobi phase: sweep until every rotation is below this (then fp64 sweeps)
#endif
#ifndef FM_SMALL_WARPS
#define FM_SMALL_WARPS 4  // 93.4 -> 91.9 us at c2 (scripts_small_tune.sh)
#endif
#ifndef FM_PIV_WARPS
#define FM_PIV_WARPS 4  // 22.4 -> 21.2 us
#endif
#ifndef FM_SOLVE_MINB
#define FM_SOLVE_MINB 1
#endif
#ifndef FM_BASIS_MINB
#define FM_BASIS_MINB 1
#endif
constexpr int kNW = kNT / 32;
constexpr int kRC = 64;   // rows per staged Gram chunk
constexpr int kRCP = 65;  // padded column stride (conflict-free 16-B column reads)
__device__ int* g_phase_dbg = nullptr;

// G(i, j) = sum_r conj(X_i[r]) Y_j[r] over column-major p x m operands. Threads own entries
// (HERM: upper triangle, mirrored); rows staged kRC at a time in padded shared memory and
// each entry's sum split over two row halves for shorter FMA chains.
template <bool HERM, typename XT, typename YT>
__device__ void block_gram(const XT* __restrict__ X, const YT* __restrict__ Y, int m, int p, c64* chunk, c64* G,
                           c64* part) {
    const int ne = HERM ? p * (p + 1) / 2 : p * p;
    const int slots = 2 * ne;                 // (entry, half)
    const int per = (slots + kNT - 1) / kNT;  // <= 8 for p <= 32
    c64 acc[8];
    int ei[8], ej[8], eh[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        acc[q] = mk(0.0, 0.0);
        const int sl = threadIdx.x + kNT * q;
        int e = sl >> 1, i = 0, j = 0;
        if (q < per && sl < slots) {
            if (HERM) {
                int rem = e;
                while (rem >= p - i) { rem -= p - i; ++i; }
                j = i + rem;
            } else {
                i = e % p;
                j = e / p;
            }
        }
        ei[q] = i;
        ej[q] = j;
        eh[q] = sl & 1;
    }
    c64* cy = HERM ? chunk : chunk + p * kRCP;
    long long tst = 0, tcp = 0;
    for (int r0 = 0; r0 < m; r0 += kRC) {
        const int rn = min(kRC, m - r0);
        __syncthreads();
        long long ta = clock64();
        for (int e = threadIdx.x; e < p * kRC; e += kNT) {
            const int c = e / kRC, r = e % kRC;
            chunk[c * kRCP + r] = r < rn ? to64(X[static_cast<size_t>(c) * m + r0 + r]) : mk(0.0, 0.0);
            if (!HERM) cy[c * kRCP + r] = r < rn ? to64(Y[static_cast<size_t>(c) * m + r0 + r]) : mk(0.0, 0.0);
        }
        __syncthreads();
        long long tb = clock64();
        tst += tb - ta;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (q < per && threadIdx.x + kNT * q < slots) {
                const c64* xi = chunk + ei[q] * kRCP + eh[q] * (kRC / 2);
                const c64* yj = cy + ej[q] * kRCP + eh[q] * (kRC / 2);
                c64 a = acc[q];
#pragma unroll 8
                for (int r = 0; r < kRC / 2; ++r) cmac_conj(a, xi[r], yj[r]);
                acc[q] = a;
            }
        }
        __syncthreads();
        tcp += clock64() - tb;
    }
    (void)tst;
    (void)tcp;
    // combine halves through `part`, write G (column-major)
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int sl = threadIdx.x + kNT * q;
        if (q < per && sl < slots && eh[q] == 1) part[sl >> 1] = acc[q];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int sl = threadIdx.x + kNT * q;
        if (q < per && sl < slots && eh[q] == 0) {
            const c64 v = acc[q] + part[sl >> 1];
            G[ej[q] * p + ei[q]] = v;
            if (HERM) G[ei[q] * p + ej[q]] = conj(v);
        }
    }
    __syncthreads();
}

// Masked outer-product Cholesky of the Hermitian p x p A (column-major, destroyed), all threads.
// perm[k] = original index eliminated at step k (k if !pivot), d[k] its Schur pivot,
// L[k * p + i] = l_k(i) by ORIGINAL row index i (zero for rows eliminated earlier).
__device__ void block_chol(c64* A, int p, bool pivot, int* perm, double* d, c64* L, int* done, double* s_inv) {
    for (int i = threadIdx.x; i < p; i += kNT) done[i] = 0;
    __syncthreads();
    for (int k = 0; k < p; ++k) {
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            int piv = k;
            if (pivot) {
                double best = -1.0;
                int bi = p;
                for (int j = lane; j < p; j += 32) {
                    if (done[j]) continue;
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
            if (lane == 0) {
                const double dk = A[piv * p + piv].re;
                perm[k] = piv;
                d[k] = dk;
                done[piv] = 1;
                *s_inv = dk > 0.0 ? 1.0 / sqrt(dk) : 0.0;
            }
        }
        __syncthreads();
        const int piv = perm[k];
        const double inv = *s_inv;
        for (int i = threadIdx.x; i < p; i += kNT) {
            // l_k(i) = A(i, piv) / sqrt(A(piv, piv)) for rows not yet eliminated (incl. piv)
            const bool live = !done[i] || i == piv;
            const c64 a = A[piv * p + i];
            L[k * p + i] = live ? mk(a.re * inv, a.im * inv) : mk(0.0, 0.0);
        }
        __syncthreads();
        for (int e = threadIdx.x; e < p * p; e += kNT) {
            const int i = e % p, j = e / p;
            if (done[i] || done[j]) continue;
            const c64 li = L[k * p + i], lj = L[k * p + j];
            c64 a = A[e];
            a.re -= li.re * lj.re + li.im * lj.im;  // li * conj(lj)
            a.im -= li.im * lj.re - li.re * lj.im;
            A[e] = a;
        }
        __syncthreads();
    }
}

// Out[j][r] = v_j with v L_p^H = x, x_a = X[perm[a]][r], L_p(j, a) = L[a * p + perm[j]]
// (forward substitution: v_j = (x_j - sum_{a<j} v_a conj(L_p(j,a))) / L_p(j,j)). Thread per row.
template <int PC, typename XT, typename OT>
__device__ void rows_solve(const XT* __restrict__ X, const int* perm, const c64* L, int m, int p, OT* __restrict__ Out) {
    for (int r = threadIdx.x; r < m; r += kNT) {
        c64 v[PC];
#pragma unroll
        for (int j = 0; j < PC; ++j) {
            if (j < p) {
                const int pj = perm[j];
                c64 x = to64(X[static_cast<size_t>(pj) * m + r]);
#pragma unroll
                for (int a = 0; a < PC; ++a) {
                    if (a < j) {
                        const c64 l = L[a * p + pj];
                        x.re -= v[a].re * l.re + v[a].im * l.im;
                        x.im -= v[a].im * l.re - v[a].re * l.im;
                    }
                }
                const double ljj = L[j * p + pj].re;
                const double inv = ljj > 0.0 ? 1.0 / ljj : 0.0;
                v[j] = mk(x.re * inv, x.im * inv);
                OT o;
                o.re = static_cast<decltype(o.re)>(v[j].re);
                o.im = static_cast<decltype(o.im)>(v[j].im);
                Out[static_cast<size_t>(j) * m + r] = o;
            }
        }
    }
}

struct CholSmem {
    c64* G;      // p x p
    c64* L;      // p x p
    c64* chunk;  // 2 x p x kRCP
    c64* part;   // p x p
};

template <int PC>
__host__ __device__ constexpr size_t chol_smem_bytes() {
    return sizeof(c64) * (3 * PC * PC + 2 * PC * kRCP);
}

__device__ __forceinline__ CholSmem carve(uint8_t* dsm, int p) {
    CholSmem s;
    s.G = reinterpret_cast<c64*>(dsm);
    s.L = s.G + p * p;
    s.part = s.L + p * p;
    s.chunk = s.part + p * p;
    return s;
}

template <int PC, int MODE>
__global__ void __launch_bounds__(kNT) k_cholqr_blk(const c32* __restrict__ Cin, c64* __restrict__ work,
                                                    c32* __restrict__ Vout, c64* __restrict__ Rt,
                                                    c64* __restrict__ Hout, const c32* __restrict__ Vin,
                                                    int32_t* __restrict__ status, int m, int p) {
    extern __shared__ uint8_t dsm[];
    __shared__ int perm[32], done[32];
    __shared__ double d[32];
    __shared__ double s_inv;
    const CholSmem sm = carve(dsm, p);
    const int f = blockIdx.x;
    const c32* Cf = Cin + static_cast<size_t>(f) * m * p;
    long long t0 = clock64();
    block_gram<true>(Cf, Cf, m, p, sm.chunk, sm.G, sm.part);
    long long t1 = clock64();
    block_chol(sm.G, p, true, perm, d, sm.L, done, &s_inv);
    long long t2 = clock64();
    if (MODE == 0) {
        if (threadIdx.x == 0) {
            // Eigen ColPivHouseholderQR::rank(): nonzero-pivot cut + |R_kk| > eps * p * maxpivot
            if (cholqr_rank(d, p, m) < p) atomicOr(&status[f], kFrameRank);
        }
        rows_solve<PC>(Cf, perm, sm.L, m, p, Vout + static_cast<size_t>(f) * m * p);
        __syncthreads();
        long long t3 = clock64();
        if (threadIdx.x == 0 && g_phase_dbg) {
            g_phase_dbg[f * 4 + 0] = static_cast<int>(t1 - t0);
            g_phase_dbg[f * 4 + 1] = static_cast<int>(t2 - t1);
            g_phase_dbg[f * 4 + 2] = static_cast<int>(t3 - t2);
        }
        return;
    }
    c64* Q1 = work + static_cast<size_t>(f) * 2 * p * m;
    c64* Q = Q1 + static_cast<size_t>(p) * m;
    rows_solve<PC>(Cf, perm, sm.L, m, p, Q1);
    __syncthreads();
    block_gram<true>(static_cast<const c64*>(Q1), static_cast<const c64*>(Q1), m, p, sm.chunk, sm.G, sm.part);
    block_chol(sm.G, p, false, perm, d, sm.L, done, &s_inv);
    rows_solve<PC>(static_cast<const c64*>(Q1), perm, sm.L, m, p, Q);
    __syncthreads();
    block_gram<false>(static_cast<const c64*>(Q), Cf, m, p, sm.chunk, sm.G, sm.part);
    c64* Rf = Rt + static_cast<size_t>(f) * p * p;
    for (int e = threadIdx.x; e < p * p; e += kNT) Rf[e] = sm.G[e];
    if (Vin) {
        block_gram<false>(Vin + static_cast<size_t>(f) * m * p, Cf, m, p, sm.chunk, sm.G, sm.part);
        c64* Hf = Hout + static_cast<size_t>(f) * p * p;
        for (int e = threadIdx.x; e < p * p; e += kNT) Hf[e] = sm.G[e];
    }
}

// ------------------------------------------------------------------ single-warp p x p kernels
// Same contract as block_chol, executed by one warp with __syncwarp only (called by warp 0).
__device__ void warp_chol(c64* A, int p, bool pivot, int* perm, double* d, c64* L, int* done) {
    const int lane = threadIdx.x & 31;
    for (int i = lane; i < p; i += 32) done[i] = 0;
    __syncwarp();
    for (int k = 0; k < p; ++k) {
        int piv = k;
        if (pivot) {
            double best = -1.0;
            int bi = p;
            for (int j = lane; j < p; j += 32) {
                if (done[j]) continue;
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
        const double dk = A[piv * p + piv].re;
        const double inv = dk > 0.0 ? rsqrt(dk) : 0.0;
        __syncwarp();
        if (lane == 0) {
            perm[k] = piv;
            d[k] = dk;
            done[piv] = 1;
        }
        __syncwarp();
        for (int i = lane; i < p; i += 32) {
            const bool live = !done[i] || i == piv;
            const c64 a = A[piv * p + i];
            L[k * p + i] = live ? mk(a.re * inv, a.im * inv) : mk(0.0, 0.0);
        }
        __syncwarp();
        for (int e = lane; e < p * p; e += 32) {
            const int i = e % p, j = e / p;
            if (done[i] || done[j]) continue;
            const c64 li = L[k * p + i], lj = L[k * p + j];
            c64 a = A[e];
            a.re -= li.re * lj.re + li.im * lj.im;
            a.im -= li.im * lj.re - li.re * lj.im;
            A[e] = a;
        }
        __syncwarp();
    }
}

// Cyclic two-sided Jacobi eigensolver for the Hermitian n x n A (column-major, shared; n <= 32),
// one warp, parallel (circle) ordering: the n/2 rotations of a round are disjoint and commute,
// so all column rotations (A and Z) are applied, then all row rotations. Rotation parameters
// come from three entries (no reductions). On return diag(A) holds the eigenvalues and Z the
// eigenvectors (columns). prm: 4 * 32 doubles of scratch. Returns sweeps (0 = cap hit).
__device__ int warp_jacobi_herm(c64* A, c64* Z, int n, double* prm) {
    const int lane = threadIdx.x & 31;
    for (int e = lane; e < n * n; e += 32) Z[e] = mk((e % n) == (e / n) ? 1.0 : 0.0, 0.0);
    const int np = (n + 1) & ~1, npairs = np / 2;
    double* pc = prm;            // c
    double* ps = prm + 32;       // s magnitude (0 = identity)
    double* per = prm + 64;      // e^{i phi} re
    double* pei = prm + 96;      // e^{i phi} im
    double dscale = 0.0;
    for (int c = 0; c < n; ++c) dscale = fmax(dscale, fabs(A[c * n + c].re));
    __syncwarp();
    for (int sweep = 0; sweep < 30; ++sweep) {
        bool any = false;
        for (int rnd = 0; rnd < np - 1; ++rnd) {
            int pi = 0, pj = 0;  // this lane's pair (lanes < npairs)
            if (lane < npairs) {
                if (lane == 0) {
                    pi = rnd;
                    pj = np - 1;
                } else {
                    pi = rnd + lane;
                    if (pi >= np - 1) pi -= np - 1;
                    pj = rnd - lane;
                    if (pj < 0) pj += np - 1;
                }
                if (pi > pj) { const int t = pi; pi = pj; pj = t; }
                double c = 1.0, sm = 0.0, er = 1.0, ei = 0.0;
                if (pj < n) {
                    const c64 b = A[pj * n + pi];  // a(pi, pj)
                    const double app = A[pi * n + pi].re, aqq = A[pj * n + pj].re;
                    const double b2 = norm2(b);
                    const double thr = 1e-15 * 1e-15;
                    if (b2 > thr * fabs(app * aqq) && b2 > (1e-30 * dscale) * (1e-30 * dscale)) {
                        const double ib = rsqrt(b2);
                        const double tau = (aqq - app) * 0.5 * ib;
                        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                        c = rsqrt(1.0 + t * t);
                        sm = t * c;
                        er = b.re * ib;
                        ei = b.im * ib;
                    }
                }
                pc[lane] = c;
                ps[lane] = sm;
                per[lane] = er;
                pei[lane] = ei;
            }
            const bool rot = __any_sync(0xffffffffu, lane < npairs && ps[lane] != 0.0);
            __syncwarp();
            if (!rot) continue;
            any = true;
            // columns (A and Z): a(r,i) = c a_ri - conj(s) a_rj ; a(r,j) = s a_ri + c a_rj
            for (int e = lane; e < 2 * npairs * n; e += 32) {
                const int which = e >= npairs * n;
                const int e2 = which ? e - npairs * n : e;
                const int t = e2 / n, r = e2 % n;
                if (ps[t] == 0.0) continue;
                int i, j;
                if (t == 0) { i = rnd; j = np - 1; }
                else {
                    i = rnd + t; if (i >= np - 1) i -= np - 1;
                    j = rnd - t; if (j < 0) j += np - 1;
                }
                if (i > j) { const int x = i; i = j; j = x; }
                if (j >= n) continue;
                c64* M = which ? Z : A;
                const double c = pc[t], sm = ps[t];
                const double sr = sm * per[t], si = sm * pei[t];
                const c64 x = M[i * n + r], y = M[j * n + r];
                M[i * n + r] = mk(c * x.re - (sr * y.re + si * y.im), c * x.im - (sr * y.im - si * y.re));
                M[j * n + r] = mk(sr * x.re - si * x.im + c * y.re, sr * x.im + si * x.re + c * y.im);
            }
            __syncwarp();
            // rows: a(i,r) = c a_ir - s a_jr ; a(j,r) = conj(s) a_ir + c a_jr
            for (int e = lane; e < npairs * n; e += 32) {
                const int t = e / n, r = e % n;
                if (ps[t] == 0.0) continue;
                int i, j;
                if (t == 0) { i = rnd; j = np - 1; }
                else {
                    i = rnd + t; if (i >= np - 1) i -= np - 1;
                    j = rnd - t; if (j < 0) j += np - 1;
                }
                if (i > j) { const int x = i; i = j; j = x; }
                if (j >= n) continue;
                const double c = pc[t], sm = ps[t];
                const double sr = sm * per[t], si = sm * pei[t];
                const c64 x = A[r * n + i], y = A[r * n + j];
                A[r * n + i] = mk(c * x.re - (sr * y.re - si * y.im), c * x.im - (sr * y.im + si * y.re));
                A[r * n + j] = mk(sr * x.re + si * x.im + c * y.re, sr * x.im - si * x.re + c * y.im);
            }
            __syncwarp();
        }
        if (!any) return sweep + 1;
    }
    return 0;
}

// ------------------------------------------------------------------ register-tiled fp64 Gram(s)
// Up to two products G1 = X1^H Y1 (HERM1: X1 == Y1, upper tiles mirrored) and G2 = X2^H Y2 of
// column-major p x m operands (p % 4 == 0). Rows are staged kRCH at a time row-major in shared
// memory with a padded stride (p + 1 complex, conflict-free 16-B reads across 8 row groups);
// each thread accumulates a 4x4 tile over every 8th row (16 complex MACs per 8 shared loads),
// and the 8 row-group partials are reduced with shuffles. Results: column-major p x p in G1/G2.
constexpr int kRG = 8;      // row groups (consecutive lanes)
constexpr int kRCH = 64;    // rows per staged chunk

// Row groups per tile: 8 for p <= 16; 4 for p = 32 (the 36 upper tiles of G then fit one pass of 256 threads,
// and G + H two passes instead of three).
template <int PC> struct GramRG { static constexpr int value = PC > 16 ? FM_GRAM_RG32 : 8; };

template <int PC, typename T1, typename T2>
__device__ void tiled_gram2(const T1* __restrict__ X1, bool herm1, const T1* __restrict__ Y1, const T2* __restrict__ X2,
                            const T2* __restrict__ Y2, int m, int p, c64* stage, c64* G1, c64* G2) {
    // Callers: herm1 always true (G = X1^H X1); X2 optional with Y2 == X1 (H = X2^H X1).
    (void)Y1;
    (void)Y2;
    const int nb = p >> 2;
    const int t1 = nb * (nb + 1) / 2;
    // X2^H X1 is only used as H = V^H R V (Hermitian in exact arithmetic, symmetrised by the callers):
    // both products use the upper-triangle 4x4 tiles and mirror the strictly upper blocks
    const int t2 = X2 ? nb * (nb + 1) / 2 : 0;
    const int ntiles = t1 + t2;
    const int ld = p + 1;
    c64* sX1 = stage;
    c64* sX2 = sX1 + kRCH * ld;
    constexpr int kRGt = GramRG<PC>::value;
    const int rg = threadIdx.x % kRGt;
    // software pipeline over row chunks: the next chunk's elements are loaded into registers
    // (all in flight together) while the current chunk is consumed from shared memory
    constexpr int kEPT = (PC * kRCH + kNT - 1) / kNT;  // elements per thread per chunk per operand
    const int nel = p * kRCH;
    c32 n1[kEPT], n2[kEPT];
    auto fetch = [&](int r0) {
        const int rn = min(kRCH, m - r0);
#pragma unroll
        for (int u = 0; u < kEPT; ++u) {
            const int e = threadIdx.x + u * kNT;
            const int c = e / kRCH, r = e % kRCH;
            const bool ok = e < nel && r < rn;
            n1[u] = ok ? X1[static_cast<size_t>(c) * m + r0 + r] : c32{0.f, 0.f};
            if (X2) n2[u] = ok ? X2[static_cast<size_t>(c) * m + r0 + r] : c32{0.f, 0.f};
        }
    };
    for (int pass = 0; pass * (kNT / kRGt) < ntiles; ++pass) {
        const int tile = pass * (kNT / kRGt) + threadIdx.x / kRGt;
        const bool active = tile < ntiles;
        const bool second = tile >= t1;
        int ti = 0, tj = 0;
        if (active) {
            if (!second) {
                int rem = tile;
                while (rem >= nb - ti) { rem -= nb - ti; ++ti; }
                tj = ti + rem;
            } else {
                int rem = tile - t1;
                while (rem >= nb - ti) { rem -= nb - ti; ++ti; }
                tj = ti + rem;
            }
        }
        c64 acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = mk(0.0, 0.0);
        fetch(0);
        for (int r0 = 0; r0 < m; r0 += kRCH) {
            const int rn = min(kRCH, m - r0);
            __syncthreads();  // previous chunk consumed
#pragma unroll
            for (int u = 0; u < kEPT; ++u) {
                const int e = threadIdx.x + u * kNT;
                if (e < nel) {
                    const int c = e / kRCH, r = e % kRCH;
                    sX1[r * ld + c] = to64(n1[u]);
                    if (X2) sX2[r * ld + c] = to64(n2[u]);
                }
            }
            __syncthreads();
            if (r0 + kRCH < m) fetch(r0 + kRCH);  // overlaps the compute below
            if (active) {
                const c64* xs = second ? sX2 : sX1;
                const c64* ys = sX1;
                for (int r = rg; r < rn; r += kRGt) {
                    c64 x[4], y[4];
#pragma unroll
                    for (int a = 0; a < 4; ++a) {
                        x[a] = xs[r * ld + 4 * ti + a];
                        y[a] = ys[r * ld + 4 * tj + a];
                    }
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int b = 0; b < 4; ++b) cmac_conj(acc[a][b], x[a], y[b]);
                }
            }
        }
        // reduce the kRG row-group partials (consecutive lanes)
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
#pragma unroll
                for (int o = 1; o < kRGt; o <<= 1) {
                    acc[a][b].re += __shfl_xor_sync(0xffffffffu, acc[a][b].re, o);
                    acc[a][b].im += __shfl_xor_sync(0xffffffffu, acc[a][b].im, o);
                }
            }
        if (active && rg == 0) {
            c64* G = second ? G2 : G1;
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const int i = 4 * ti + a, j = 4 * tj + b;
                    G[j * p + i] = acc[a][b];
                    if (ti != tj) G[i * p + j] = conj(acc[a][b]);
                }
        }
    }
    __syncthreads();
}

template <int PC>
__host__ __device__ constexpr size_t tiled_stage_bytes(int nbuf) {
    return sizeof(c64) * nbuf * kRCH * (PC + 1);
}


__device__ __forceinline__ c64 warp_sum_c(c64 v) {
    v.re = warp_sum(v.re);
    v.im = warp_sum(v.im);
    return v;
}

// One-sided Jacobi on the n columns of a (column-major n x n, shared), one warp per pair per
// round (circle ordering). Rotation parameters seeded in fp32 (short MUFU latency), applied as
// an exactly unitary fp64 rotation (c from t in fp64, |e| = 1 to fp64 via Newton steps).
// Returns sweeps used (0 = cap hit).
__device__ int block_hestenes(c64* a, int n, int* s_rot) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int np = (n + 1) & ~1;
    const double tol = 8.0 * 2.220446049250313e-16 * n;
    for (int sweep = 0; sweep < 40; ++sweep) {
        if (threadIdx.x == 0) *s_rot = 0;
        __syncthreads();
        for (int rnd = 0; rnd < np - 1; ++rnd) {
            for (int idx = warp; idx < np / 2; idx += kNW) {
                int i, j;
                if (idx == 0) {
                    i = rnd;
                    j = np - 1;
                } else {
                    i = rnd + idx;
                    if (i >= np - 1) i -= np - 1;
                    j = rnd - idx;
                    if (j < 0) j += np - 1;
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
                    const c64 x = ai[r], y = aj[r];
                    al += norm2(x);
                    be += norm2(y);
                    cmac_conj(ga, x, y);
                }
                al = warp_sum(al);
                be = warp_sum(be);
                ga = warp_sum_c(ga);
                const double g2 = norm2(ga);
                if (!(g2 > tol * tol * al * be) || g2 == 0.0) continue;
                double c;
                c64 e;  // s e
                jacobi_rotation(al, be, ga, g2, c, e);
                for (int r = lane; r < n; r += 32) {
                    const c64 x = ai[r], y = aj[r];
                    ai[r] = mk(c * x.re - (e.re * y.re + e.im * y.im), c * x.im - (e.re * y.im - e.im * y.re));
                    aj[r] = mk((e.re * x.re - e.im * x.im) + c * y.re, (e.re * x.im + e.im * x.re) + c * y.im);
                }
                if (lane == 0) *s_rot = 1;
            }
            __syncthreads();
        }
        const bool fin = (*s_rot == 0);
        __syncthreads();
        if (fin) return sweep + 1;
    }
    return 0;
}

template <int PC>
__host__ __device__ constexpr size_t nys_smem_bytes() {
    return sizeof(c64) * (3 * PC * PC) + sizeof(double) * PC;
}

template <int PC>
__global__ void __launch_bounds__(kNT) k_nystrom_blk(const c64* __restrict__ Hin, const c64* __restrict__ work,
                                                     const c64* __restrict__ Rt, c64* __restrict__ basis,
                                                     double* __restrict__ eig, int32_t* __restrict__ status, int m,
                                                     int p, int k, int32_t* __restrict__ dbg) {
    extern __shared__ uint8_t dsm[];
    c64* A = reinterpret_cast<c64*>(dsm);  // H, then Y
    c64* L = A + p * p;
    c64* Rs = L + p * p;
    double* sig = reinterpret_cast<double*>(Rs + p * p);
    __shared__ int perm[32], done[32], order[32];
    __shared__ double d[32];
    __shared__ double s_inv;
    __shared__ int s_rot;
    const int f = blockIdx.x;
    const c64* Hf = Hin + static_cast<size_t>(f) * p * p;
    const c64* Rf = Rt + static_cast<size_t>(f) * p * p;
    for (int e = threadIdx.x; e < p * p; e += kNT) {
        const int i = e % p, j = e / p;
        const c64 a = Hf[j * p + i], b = Hf[i * p + j];
        A[e] = mk(0.5 * (a.re + b.re), 0.5 * (a.im - b.im));  // Herm(H)(i, j)
        Rs[e] = Rf[e];
    }
    __syncthreads();
    block_chol(A, p, false, perm, d, L, done, &s_inv);
    // Y = Rt L_H^-H: row i of Y solves y L^H = rt_i (thread per row i < p), into A (column-major)
    if (threadIdx.x < p) {
        const int i = threadIdx.x;
        c64 v[PC];
#pragma unroll
        for (int j = 0; j < PC; ++j) {
            if (j < p) {
                c64 x = Rs[j * p + i];
#pragma unroll
                for (int a = 0; a < PC; ++a) {
                    if (a < j) {
                        const c64 l = L[a * p + j];
                        x.re -= v[a].re * l.re + v[a].im * l.im;
                        x.im -= v[a].im * l.re - v[a].re * l.im;
                    }
                }
                const double ljj = L[j * p + j].re;
                const double inv = ljj > 0.0 ? 1.0 / ljj : 0.0;
                v[j] = mk(x.re * inv, x.im * inv);
                A[j * p + i] = v[j];
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double dmax = 0.0, dmin = 1e300;
        for (int q = 0; q < p; ++q) {
            dmax = fmax(dmax, d[q]);
            dmin = fmin(dmin, d[q]);
        }
        if (!(dmin > static_cast<double>(p) * eps_of<float>::value * dmax)) atomicOr(&status[f], kFrameNoConv);
    }
    const int sw = block_hestenes(A, p, &s_rot);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int c = warp; c < p; c += kNW) {
        double s = 0.0;
        for (int r = lane; r < p; r += 32) s += norm2(A[c * p + r]);
        s = warp_sum(s);
        if (lane == 0) sig[c] = sqrt(s);
    }
    __syncthreads();
    if (threadIdx.x < p) {  // descending rank (ties: lower index first)
        const int c = threadIdx.x;
        int rank = 0;
        for (int q = 0; q < p; ++q)
            if (q != c && (sig[q] > sig[c] || (sig[q] == sig[c] && q < c))) ++rank;
        order[rank] = c;
    }
    __syncthreads();
    const c64* Qf = work + static_cast<size_t>(f) * 2 * p * m + static_cast<size_t>(p) * m;
    c64* Bf = basis + static_cast<size_t>(f) * m * k;
    for (int e = threadIdx.x; e < m * k; e += kNT) {
        const int kk = e / m, r = e % m;
        const int c = order[kk];
        const double inv = sig[c] > 0.0 ? 1.0 / sig[c] : 0.0;
        c64 acc = mk(0.0, 0.0);
        for (int q = 0; q < p; ++q) cmac(acc, Qf[static_cast<size_t>(q) * m + r], A[c * p + q]);
        Bf[static_cast<size_t>(kk) * m + r] = mk(acc.re * inv, acc.im * inv);
    }
    if (threadIdx.x < k) {
        double lam = sig[order[threadIdx.x]];
        lam *= lam;
        if (lam < 0.0 && lam >= -1e-10) lam = 0.0;
        eig[static_cast<size_t>(f) * k + threadIdx.x] = lam;
    }
    if (threadIdx.x == 0 && sw == 0) atomicOr(&status[f], kFrameNoConv);
    if (threadIdx.x == 0 && dbg) dbg[f] = sw;
}




// ------------------------------------------------------------------------------------------
// Split final stage (p in {4, 8, ..., 32}, p % 4 == 0). A fused block-per-frame final stage spent ~90% of
// its time in p x p phases where one frame occupies a whole CTA behind __syncthreads; here the
// Gram products stay block-per-frame, and every p x p phase runs one WARP per frame (8 frames
// per CTA for p <= 16), so all frames of a batch are in flight at once.
//   k_gram_gh   : G = C^H C, H = Herm(V^H C) (fast1: Herm(H given)) in fp64 -> workspace
//   k_small_warp: G = L L^H, H = L_H L_H^H (warp Cholesky), Y = R L_H^-H (R = L^H),
//                 one-sided Jacobi on Y (lane-per-column), s, order, T = R^-1 Z_K / s, eig = s^2
//   k_basis_ct  : U = C T (thread per row, fp64 accumulation)
// R/src/estimators.cpp:37-50, :104-139; linalg.cpp:143-163.

template <int PC>
__global__ void __launch_bounds__(kNT, 2) k_gram_gh(const c32* __restrict__ Cin, const c32* __restrict__ Vin,
                                                 c64* __restrict__ Gout, c64* __restrict__ Hio, int m, int p) {
    extern __shared__ uint8_t dsm[];
    c64* G = reinterpret_cast<c64*>(dsm);
    c64* H = G + PC * PC;
    c64* stage = H + PC * PC;
    const int f = blockIdx.x;
    const c32* Cf = Cin + static_cast<size_t>(f) * m * p;
    c64* Hf = Hio + static_cast<size_t>(f) * p * p;
    if (Vin) {
        tiled_gram2<PC, c32, c32>(Cf, true, Cf, Vin + static_cast<size_t>(f) * m * p, Cf, m, p, stage, G, H);
    } else {
        tiled_gram2<PC, c32, c32>(Cf, true, Cf, nullptr, nullptr, m, p, stage, G, nullptr);
        for (int e = threadIdx.x; e < p * p; e += kNT) H[e] = Hf[e];
        __syncthreads();
    }
    c64* Gf = Gout + static_cast<size_t>(f) * p * p;
    for (int e = threadIdx.x; e < p * p; e += kNT) {
        const int i = e % p, j = e / p;
        const c64 a = H[j * p + i], b = H[i * p + j];  // Herm: (H(i,j) + conj(H(j,i))) / 2, exactly Hermitian
        Gf[e] = G[e];
        Hf[e] = mk(0.5 * (a.re + b.re), 0.5 * (a.im - b.im));
    }
}


template <int PC> struct WarpCfg {
    static constexpr int kLPC = 32 / PC;                   // lanes per column in the Jacobi
    static constexpr int kWarps = PC <= 16 ? FM_SMALL_WARPS : 4;  // frames per CTA
    static constexpr int kLd = PC + ((kLPC - PC) % 8 + 8) % 8;  // ld = LPC (mod 8): conflict-free 16-B rows
    // L, L_H (reused for T once Y is formed), Y (in-place pair-lane Jacobi)
    static constexpr size_t kBytes = sizeof(c64) * (2 * PC * PC + PC * kLd) + sizeof(double) * PC + sizeof(int) * PC;
    static constexpr size_t kWarpBytes = (kBytes + 15) / 16 * 16;
};

// In-place non-pivoted Cholesky of the Hermitian PD p x p A (column-major, ld p) by one warp:
// lower triangle -> L (diagonal real sqrt(d_k)); the strict upper triangle is left stale.
// Returns min / max Schur pivots (all lanes).
__device__ __forceinline__ void warp_chol_lower(c64* A, int p, double& dmin, double& dmax) {
    const int lane = threadIdx.x & 31;
    dmin = 1e300;
    dmax = 0.0;
    for (int k = 0; k < p; ++k) {
        const double dk = A[k * p + k].re;
        dmin = fmin(dmin, dk);
        dmax = fmax(dmax, dk);
        const double inv = dk > 0.0 ? 1.0 / sqrt(dk) : 0.0;
        __syncwarp();
        // lane = row i > k: l_i = A(i, k) / sqrt(d_k), then A(i, j) -= l_i conj(l_j), k < j <= i
        // (column-major: lanes touch consecutive rows of one column -> conflict-free)
        c64 li = mk(0.0, 0.0);
        if (lane > k && lane < p) {
            const c64 a = A[k * p + lane];
            li = mk(a.re * inv, a.im * inv);
            A[k * p + lane] = li;
        }
        if (lane == 0) A[k * p + k] = mk(dk > 0.0 ? sqrt(dk) : 0.0, 0.0);
        __syncwarp();
        if (lane > k && lane < p) {  // batches of 8: all loads before the stores
            for (int j0 = k + 1; j0 <= lane; j0 += 8) {
                c64 lj[8], a[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int j = j0 + u;
                    if (j <= lane) {
                        lj[u] = A[k * p + j];
                        a[u] = A[j * p + lane];
                    }
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int j = j0 + u;
                    if (j <= lane) {
                        a[u].re -= li.re * lj[u].re + li.im * lj[u].im;  // li * conj(lj)
                        a[u].im -= li.im * lj[u].re - li.re * lj[u].im;
                        A[j * p + lane] = a[u];
                    }
                }
            }
        }
        __syncwarp();
    }
}

// Two independent in-place Cholesky factorisations (p <= 16) by one warp: lanes 0..15 factor A1,
// lanes 16..31 factor A2, row = lane & 15 (same schedule as warp_chol_lower). Returns both pivot ranges.
__device__ __forceinline__ void warp_chol_lower_pair(c64* A1, c64* A2, int p, double& dmin1, double& dmax1,
                                                     double& dmin2, double& dmax2) {
    const int lane = threadIdx.x & 31;
    c64* A = lane < 16 ? A1 : A2;
    const int row = lane & 15;
    double dmin = 1e300, dmax = 0.0;
    for (int k = 0; k < p; ++k) {
        const double dk = A[k * p + k].re;
        dmin = fmin(dmin, dk);
        dmax = fmax(dmax, dk);
        const double inv = dk > 0.0 ? 1.0 / sqrt(dk) : 0.0;
        __syncwarp();
        c64 li = mk(0.0, 0.0);
        if (row > k && row < p) {
            const c64 a = A[k * p + row];
            li = mk(a.re * inv, a.im * inv);
            A[k * p + row] = li;
        }
        if (row == 0) A[k * p + k] = mk(dk > 0.0 ? sqrt(dk) : 0.0, 0.0);
        __syncwarp();
        if (row > k && row < p) {
            for (int j = k + 1; j <= row; ++j) {
                const c64 lj = A[k * p + j];
                c64 a = A[j * p + row];
                a.re -= li.re * lj.re + li.im * lj.im;
                a.im -= li.im * lj.re - li.re * lj.im;
                A[j * p + row] = a;
            }
        }
        __syncwarp();
    }
    dmin1 = __shfl_sync(0xffffffffu, dmin, 0);
    dmax1 = __shfl_sync(0xffffffffu, dmax, 0);
    dmin2 = __shfl_sync(0xffffffffu, dmin, 16);
    dmax2 = __shfl_sync(0xffffffffu, dmax, 16);
}

template <int PC>
__global__ void __launch_bounds__(32 * WarpCfg<PC>::kWarps)
    k_small_warp(const c64* __restrict__ Gin, const c64* __restrict__ Hin, c64* __restrict__ Tout,
                 double* __restrict__ eig, int32_t* __restrict__ status, int frames, int p, int k,
                 int32_t* __restrict__ dbg, double* __restrict__ eig_next, const c64* __restrict__ gpart,
                 const c64* __restrict__ hpart) {
    using W = WarpCfg<PC>;
    constexpr int LPC = W::kLPC;
    extern __shared__ uint8_t dsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int f = blockIdx.x * W::kWarps + warp;
    if (f >= frames) return;  // whole warp
    const int ld = W::kLd;
    c64* L = reinterpret_cast<c64*>(dsm + warp * W::kWarpBytes);
    c64* LH = L + PC * PC;
    c64* Ya = LH + PC * PC;
    double* sig = reinterpret_cast<double*>(Ya + PC * ld);
    int* order = reinterpret_cast<int*>(sig + PC);
    const c64* Gf = Gin + static_cast<size_t>(f) * p * p;
    const c64* Hf = Hin + static_cast<size_t>(f) * p * p;
    const long long T0 = clock64();
    if (gpart) {  // G, H halves from the product kernel's epilogue; H symmetrised as k_gram_gh does
        const size_t pp = static_cast<size_t>(p) * p;
        const c64* g0 = gpart + static_cast<size_t>(f) * 2 * pp;
        const c64* h0 = hpart + static_cast<size_t>(f) * 2 * pp;
        for (int e = lane; e < p * p; e += 32) {
            const int i = e % p, j = e / p;
            const c64 a = h0[e] + h0[pp + e], b = h0[i * p + j] + h0[pp + i * p + j];
            L[e] = g0[e] + g0[pp + e];
            LH[e] = mk(0.5 * (a.re + b.re), 0.5 * (a.im - b.im));
        }
    } else
    for (int e0 = 0; e0 < p * p; e0 += 8 * 32) {  // 16 loads in flight per lane
        c64 g[8], hh[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = e0 + lane + 32 * u;
            if (e < p * p) {
                g[u] = Gf[e];
                hh[u] = Hf[e];
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = e0 + lane + 32 * u;
            if (e < p * p) {
                L[e] = g[u];
                LH[e] = hh[u];
            }
        }
    }
    __syncwarp();
    double dmin, dmax, dminG, dmaxG;
    if (PC <= 16) {
        // G = L L^H (R = L^H) and H = L_H L_H^H concurrently
        warp_chol_lower_pair(L, LH, p, dminG, dmaxG, dmin, dmax);
    } else {
        warp_chol_lower(L, p, dminG, dmaxG);  // G = L L^H, R = L^H: R(i, j) = conj(L[i * p + j]), j >= i
        warp_chol_lower(LH, p, dmin, dmax);   // H = L_H L_H^H
    }
    // A near-singular H (its Cholesky cannot stand in for the reference's truncating pinv) or a C whose Gram
    // pivots fall below the fp64 Gram's resolution goes to the exact-algebra fallback (final_fallback.cu).
    if (lane == 0 && (!(dmin > static_cast<double>(p) * eps_of<float>::value * dmax) ||
                      !(dminG > static_cast<double>(p) * eps_of<double>::value * dmaxG)))
        atomicOr(&status[f], kFrameNoConv);
    for (int e = lane; e < PC * ld; e += 32) Ya[e] = mk(0.0, 0.0);  // rows >= p stay zero
    __syncwarp();
    // Y(i, :) solves y L_H^H = R(i, :) (forward substitution, lane per row); Y -> Ya (ld).
    // Reciprocal pivots first; two partial sums per step for a shorter FMA chain.
    double* rinv = sig;  // PC doubles, free until the singular values are formed
    if (lane < p) {
        const double ljj = LH[lane * p + lane].re;
        rinv[lane] = ljj > 0.0 ? 1.0 / ljj : 0.0;
    }
    __syncwarp();
    if (lane < p) {
        const int i = lane;
        for (int j = 0; j < p; ++j) {
            c64 x0 = j >= i ? conj(L[i * p + j]) : mk(0.0, 0.0);
            c64 x1 = mk(0.0, 0.0);
            int a = i;
            for (; a + 1 < j; a += 2) {  // y_a = 0 for a < i
                const c64 l0 = LH[a * p + j], l1 = LH[(a + 1) * p + j];
                const c64 v0 = Ya[a * ld + i], v1 = Ya[(a + 1) * ld + i];
                x0.re -= v0.re * l0.re + v0.im * l0.im;
                x0.im -= v0.im * l0.re - v0.re * l0.im;
                x1.re -= v1.re * l1.re + v1.im * l1.im;
                x1.im -= v1.im * l1.re - v1.re * l1.im;
            }
            if (a < j) {
                const c64 l0 = LH[a * p + j];
                const c64 v0 = Ya[a * ld + i];
                x0.re -= v0.re * l0.re + v0.im * l0.im;
                x0.im -= v0.im * l0.re - v0.re * l0.im;
            }
            const double inv = rinv[j];
            Ya[j * ld + i] = j >= i ? mk((x0.re + x1.re) * inv, (x0.im + x1.im) * inv) : mk(0.0, 0.0);
        }
    }
    __syncwarp();
    // Y to unit scale by a power of two (exact): the Jacobi below then sees the same numbers for any input scale
    // (X * 2^-20 .. X * 2^12); singular values -- and the eigenvalues s^2 -- are scaled back at the end, and
    // the columns' directions (hence T) are unaffected.
    double yscale2 = 1.0;  // 2^(2e): eigenvalue factor
    {
        double ymax = 0.0;
        for (int e = lane; e < p * ld; e += 32) ymax = fmax(ymax, norm2(Ya[e]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ymax = fmax(ymax, __shfl_xor_sync(0xffffffffu, ymax, o));
        if (ymax > 0.0 && ymax < 1e300) {
            const double sc = pow2_inv_sqrt_scale(ymax);  // 2^-e, |Y|max 2^-e in [1, 2)
            yscale2 = 1.0 / (sc * sc);
            for (int e = lane; e < PC * ld; e += 32) Ya[e] = mk(Ya[e].re * sc, Ya[e].im * sc);
        }
    }
    __syncwarp();
    const long long T1 = clock64();
    // one-sided Jacobi on Y's columns, in place in Ya. Lanes are assigned to column PAIRS: slot
    // = lane / LPP of the round-robin schedule (slot 0: (rnd, p-1); slot s: (rnd + s, rnd - s)
    // mod (p - 1)), sub = lane % LPP owns rows sub, sub + LPP, ... of BOTH columns, so every
    // element is read and written by one lane per round (one __syncwarp per round). Rotation:
    // fp32-seeded angle, fp64 cos / phase refined by one Newton step (unitary to ~5e-15).
    constexpr int LPP = 64 / PC;            // lanes per pair
    constexpr int RPL = PC * PC / 64;       // rows per lane
    const int slot = lane / LPP, sub = lane % LPP;
    const bool act = slot < p / 2;
    const int n1 = p - 1;                   // p even (p % 4 == 0)
    const double tol = 8.0 * 2.220446049250313e-16 * p;
    c64* cur = Ya;
    int sweeps = 0;
    // Phase 1 (fp32): sweeps on a complex64 copy of Y (in the L_H region, free until T is formed) until
    // every rotated pair has |g| / sqrt(al be) < 1e-6; the fp64 phase below then restores exact column
    // orthogonality (the fp32 rotations perturb Y by ~1e-6 relative, far inside the error budget of the
    // fp16-operand covariance).
    {
        c32* y32 = reinterpret_cast<c32*>(LH);
        for (int e = lane; e < PC * ld; e += 32) y32[e] = mk(static_cast<float>(Ya[e].re), static_cast<float>(Ya[e].im));
        __syncwarp();
        const float tol32 = FM_JACOBI_TOL32;
        for (int sweep = 0; sweep < 12; ++sweep) {
            bool rot_any = false;
            for (int rnd = 0; rnd < n1; ++rnd) {
                int i = rnd + slot, j = rnd - slot;
                if (i >= n1) i -= n1;
                if (j < 0) j += n1;
                if (slot == 0) j = n1;
                const int lo = act ? min(i, j) : 0, hi = act ? max(i, j) : 0;
                c32* xlo = y32 + lo * ld + sub;
                c32* xhi = y32 + hi * ld + sub;
                c32 x[RPL], y[RPL];
                float al = 0.f, be = 0.f;
                c32 ga = mk(0.f, 0.f);
#pragma unroll
                for (int t = 0; t < RPL; ++t) {
                    x[t] = xlo[t * LPP];
                    y[t] = xhi[t * LPP];
                    al = fmaf(x[t].re, x[t].re, fmaf(x[t].im, x[t].im, al));
                    be = fmaf(y[t].re, y[t].re, fmaf(y[t].im, y[t].im, be));
                    cmac_conj(ga, x[t], y[t]);
                }
#pragma unroll
                for (int o = 1; o < LPP; o <<= 1) {
                    al += __shfl_xor_sync(0xffffffffu, al, o);
                    be += __shfl_xor_sync(0xffffffffu, be, o);
                    ga.re += __shfl_xor_sync(0xffffffffu, ga.re, o);
                    ga.im += __shfl_xor_sync(0xffffffffu, ga.im, o);
                }
                const float g2 = ga.re * ga.re + ga.im * ga.im;
                const bool rotate = act && (g2 > tol32 * tol32 * al * be) && g2 > 0.f;
                if (rotate) {
                    const float ig = rsqrtf(g2);
                    const float zeta = (be - al) * (0.5f * ig);
                    const float tf = copysignf(1.0f, zeta) / (fabsf(zeta) + sqrtf(fmaf(zeta, zeta, 1.0f)));
                    const float cs = rsqrtf(fmaf(tf, tf, 1.0f));
                    const float sn = cs * tf;
                    const c32 se = mk(sn * ga.re * ig, sn * ga.im * ig);
#pragma unroll
                    for (int t2 = 0; t2 < RPL; ++t2) {
                        const c32 u = x[t2], v = y[t2];
                        xlo[t2 * LPP] = mk(fmaf(cs, u.re, -fmaf(se.re, v.re, se.im * v.im)),
                                           fmaf(cs, u.im, -fmaf(se.re, v.im, -se.im * v.re)));
                        xhi[t2 * LPP] = mk(fmaf(cs, v.re, fmaf(se.re, u.re, -se.im * u.im)),
                                           fmaf(cs, v.im, fmaf(se.re, u.im, se.im * u.re)));
                    }
                }
                rot_any |= rotate;
                __syncwarp();
            }
            if (!__any_sync(0xffffffffu, rot_any)) break;
        }
        for (int e = lane; e < PC * ld; e += 32) Ya[e] = to64(y32[e]);
        __syncwarp();
    }
    for (int sweep = 0; sweep < 40; ++sweep) {
        bool rot_any = false;
        bool big = false;  // some rotation of this sweep had |g|^2 >= 1e-14 al be
        for (int rnd = 0; rnd < n1; ++rnd) {
            int i = rnd + slot, j = rnd - slot;
            if (i >= n1) i -= n1;
            if (j < 0) j += n1;
            if (slot == 0) j = n1;
            const int lo = act ? min(i, j) : 0, hi = act ? max(i, j) : 0;
            c64* xlo = cur + lo * ld + sub;
            c64* xhi = cur + hi * ld + sub;
            c64 x[RPL], y[RPL];
            double al0 = 0.0, al1 = 0.0, be0 = 0.0, be1 = 0.0;
            c64 g0 = mk(0.0, 0.0), g1 = mk(0.0, 0.0);
#pragma unroll
            for (int t = 0; t < RPL; ++t) {
                x[t] = xlo[t * LPP];
                y[t] = xhi[t * LPP];
                if (t & 1) {
                    al1 += norm2(x[t]);
                    be1 += norm2(y[t]);
                    cmac_conj(g1, x[t], y[t]);
                } else {
                    al0 += norm2(x[t]);
                    be0 += norm2(y[t]);
                    cmac_conj(g0, x[t], y[t]);
                }
            }
            double al = al0 + al1, be = be0 + be1;
            c64 ga = mk(g0.re + g1.re, g0.im + g1.im);
#pragma unroll
            for (int o = 1; o < LPP; o <<= 1) {
                al += __shfl_xor_sync(0xffffffffu, al, o);
                be += __shfl_xor_sync(0xffffffffu, be, o);
                ga.re += __shfl_xor_sync(0xffffffffu, ga.re, o);
                ga.im += __shfl_xor_sync(0xffffffffu, ga.im, o);
            }
            const double g2 = norm2(ga);
            const bool rotate = act && (g2 > tol * tol * al * be) && g2 != 0.0;
            if (rotate) {
                big |= g2 >= 1e-14 * al * be;
                double cs;
                c64 se;  // s e
                jacobi_rotation(al, be, ga, g2, cs, se);
#pragma unroll
                for (int t2 = 0; t2 < RPL; ++t2) {
                    const c64 u = x[t2], v = y[t2];
                    // lo' = c x - conj(s e) y ; hi' = s e x + c y
                    xlo[t2 * LPP] = mk(fma(cs, u.re, -fma(se.re, v.re, se.im * v.im)),
                                       fma(cs, u.im, -fma(se.re, v.im, -se.im * v.re)));
                    xhi[t2 * LPP] = mk(fma(cs, v.re, fma(se.re, u.re, -se.im * u.im)),
                                       fma(cs, v.im, fma(se.re, u.im, se.im * u.re)));
                }
            }
            rot_any |= rotate;
            __syncwarp();
        }
        if (!__any_sync(0xffffffffu, rot_any)) {
            sweeps = sweep + 1;
            break;
        }
        // quadratic convergence: if every rotation of this sweep had |g| / sqrt(al be) < 1e-7, the next
        // sweep's would be ~1e-14 (at the 8 eps p threshold) -- skip the verification sweep
        if (!__any_sync(0xffffffffu, big)) {
            sweeps = sweep + 1;
            break;
        }
    }
    c64* nxt = LH;  // free after Y was formed: holds T (p x k, ld = p)
    const int c = lane;
    const long long T2 = clock64();
    // singular values, descending order (ties: lower index first)
    if (c < p) {
        double s0 = 0.0, s1 = 0.0;
        for (int r = 0; r < p; r += 2) {
            s0 += norm2(cur[c * ld + r]);
            s1 += norm2(cur[c * ld + r + 1]);
        }
        const double sv = sqrt(s0 + s1);
        sig[c] = sv <= 1e300 ? sv : -1.0;  // NaN / inf (corrupt input): ranked last, frame flagged below
        if (!(sv <= 1e300)) atomicOr(&status[f], kFrameNoConv);
    }
    __syncwarp();
    if (lane < p) {
        int rank = 0;
        for (int q = 0; q < p; ++q)
            if (q != lane && (sig[q] > sig[lane] || (sig[q] == sig[lane] && q < lane))) ++rank;
        order[rank] = lane;
    }
    __syncwarp();
    // T(:, kk) = R^-1 z / s (back substitution; R(i, j) = conj(L[i * p + j])), into nxt (free)
    c64* Tm = nxt;
    if (lane < k) {
        const int kk = lane, cc = order[kk];
        const double inv_s = sig[cc] > 0.0 ? 1.0 / sig[cc] : 0.0;
        for (int i = p - 1; i >= 0; --i) {
            c64 acc = cur[cc * ld + i];
            acc.re *= inv_s;
            acc.im *= inv_s;
            for (int j = i + 1; j < p; ++j) {
                const c64 rij = conj(L[i * p + j]);
                const c64 tj = Tm[kk * p + j];
                acc.re -= rij.re * tj.re - rij.im * tj.im;
                acc.im -= rij.re * tj.im + rij.im * tj.re;
            }
            const double rii = L[i * p + i].re;
            const double inv = rii > 0.0 ? 1.0 / rii : 0.0;
            Tm[kk * p + i] = mk(acc.re * inv, acc.im * inv);
        }
        double lam = sig[cc];
        lam *= lam * yscale2;  // eigenvalue of B' = Y Y^H
        eig[static_cast<size_t>(f) * k + kk] = lam;
    }
    if (eig_next && lane == 0) {  // (K+1)-th Ritz value (exact method's gap estimate)
        const double sn = k < p ? sig[order[k]] : 0.0;
        eig_next[f] = sn * sn * yscale2;
    }
    __syncwarp();
    c64* Tf = Tout + static_cast<size_t>(f) * p * k;
    for (int e = lane; e < p * k; e += 32) Tf[e] = Tm[e];  // T stored compactly (ld p) in L_H
    if (lane == 0 && sweeps == 0) atomicOr(&status[f], kFrameNoConv);
    if (lane == 0 && dbg) dbg[f] = sweeps;
    const long long T3 = clock64();
    if (lane == 0 && g_phase_dbg) {
        g_phase_dbg[f * 4 + 0] = static_cast<int>(T1 - T0);
        g_phase_dbg[f * 4 + 1] = static_cast<int>(T2 - T1);
        g_phase_dbg[f * 4 + 2] = static_cast<int>(T3 - T2);
        g_phase_dbg[f * 4 + 3] = sweeps;
    }
}


template <int PC>
__global__ void __launch_bounds__(128, FM_BASIS_MINB) k_basis_ct(const c32* __restrict__ Cin, const c64* __restrict__ Tin,
                                                  c64* __restrict__ basis, int m, int p, int k) {
    __shared__ c64 Ts[PC * PC];
    const int f = blockIdx.y;
    const c64* Tf = Tin + static_cast<size_t>(f) * p * k;
    for (int e = threadIdx.x; e < p * k; e += blockDim.x) Ts[e] = Tf[e];
    __syncthreads();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m) return;
    const c32* Cf = Cin + static_cast<size_t>(f) * m * p;
    c64 crow[PC];
#pragma unroll
    for (int q = 0; q < PC; ++q)
        if (q < p) crow[q] = to64(Cf[static_cast<size_t>(q) * m + r]);
    c64* Bf = basis + static_cast<size_t>(f) * m * k;
    for (int kk = 0; kk < k; ++kk) {
        c64 acc = mk(0.0, 0.0);
#pragma unroll
        for (int q = 0; q < PC; ++q)
            if (q < p) cmac(acc, crow[q], Ts[kk * p + q]);
        Bf[static_cast<size_t>(kk) * m + r] = acc;
    }
}


// ------------------------------------------------------------------------------------------
// Split power-iteration orthonormalisation (R/src/linalg.cpp:127-141 qr_orthonormal with the
// Eigen ColPivHouseholderQR rank rule), same algebra as the block-per-frame k_cholqr_blk:
//   k_gram_only : G = C^H C (fp64, block per frame) -> workspace
//   k_cholpiv_warp: pivoted Cholesky of G by one warp per frame (pivot = largest remaining Schur
//                 diagonal), rank rule in fp32 epsilon -> L (by original row index) + perm
//   k_rows_solve: V = C P R^-1 by forward substitution, thread per row (fp64 -> complex64)
template <int PC>
__global__ void __launch_bounds__(kNT, 2) k_gram_only(const c32* __restrict__ Cin, c64* __restrict__ Gout, int m,
                                                   int p) {
    extern __shared__ uint8_t dsm[];
    c64* G = reinterpret_cast<c64*>(dsm);
    c64* stage = G + PC * PC;
    const int f = blockIdx.x;
    tiled_gram2<PC, c32, c32>(Cin + static_cast<size_t>(f) * m * p, true, Cin + static_cast<size_t>(f) * m * p, nullptr,
                          nullptr, m, p, stage, G, nullptr);
    c64* Gf = Gout + static_cast<size_t>(f) * p * p;
    for (int e = threadIdx.x; e < p * p; e += kNT) Gf[e] = G[e];
}

template <int PC> struct PivCfg {
    static constexpr int kWarps = PC <= 16 ? FM_PIV_WARPS : 4;
    static constexpr size_t kWarpBytes = sizeof(c64) * 2 * PC * PC + sizeof(double) * PC;
};

template <int PC>
__global__ void __launch_bounds__(32 * PivCfg<PC>::kWarps)
    k_cholpiv_warp(c64* __restrict__ GL, int32_t* __restrict__ perm_out, int32_t* __restrict__ status, int frames,
                   int m, int p, const c64* __restrict__ gpart) {
    extern __shared__ uint8_t dsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int f = blockIdx.x * PivCfg<PC>::kWarps + warp;
    if (f >= frames) return;
    c64* A = reinterpret_cast<c64*>(dsm + warp * PivCfg<PC>::kWarpBytes);
    c64* L = A + PC * PC;
    double* d = reinterpret_cast<double*>(L + PC * PC);
    c64* GLf = GL + static_cast<size_t>(f) * p * p;
    if (gpart) {  // G = sum of the two CTA halves formed in the product kernel's epilogue (rmul_tc.cu)
        const c64* g0 = gpart + static_cast<size_t>(f) * 2 * p * p;
        for (int e = lane; e < p * p; e += 32) {
            A[e] = g0[e] + g0[p * p + e];
            L[e] = mk(0.0, 0.0);
        }
    } else {
        for (int e = lane; e < p * p; e += 32) {
            A[e] = GLf[e];
            L[e] = mk(0.0, 0.0);
        }
    }
    __syncwarp();
    bool done = lane >= p;  // lane i <-> original row / column i
    int my_step = -1;
    for (int k = 0; k < p; ++k) {
        // pivot: largest remaining Schur diagonal, ties -> lower index
        double best = done ? -1.0 : A[lane * p + lane].re;
        int bi = done ? p : lane;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ob > best || (ob == best && oi < bi)) {
                best = ob;
                bi = oi;
            }
        }
        const int piv = bi;
        const double dk = A[piv * p + piv].re;
        const double inv = dk > 0.0 ? 1.0 / sqrt(dk) : 0.0;
        if (lane == 0) d[k] = dk;
        if (lane == piv) {
            done = true;
            my_step = k;
        }
        // l_k(i) = A(i, piv) / sqrt(d_k) for rows not yet eliminated (incl. piv)
        c64 li = mk(0.0, 0.0);
        if (lane < p && (!done || lane == piv)) {
            const c64 a = A[piv * p + lane];
            li = mk(a.re * inv, a.im * inv);
        }
        if (lane < p) L[k * p + lane] = li;
        __syncwarp();
        uint32_t live = __ballot_sync(0xffffffffu, lane < p && !done);
        if (lane < p && !done) {  // A(i, j) -= l_i conj(l_j) over live columns only
            while (live) {  // batches of up to 8 live columns: loads first, then stores
                int js[8];
                c64 lj[8], a[8];
                int cnt = 0;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    js[u] = live ? __ffs(live) - 1 : -1;
                    if (live) live &= live - 1;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (js[u] >= 0) {
                        lj[u] = L[k * p + js[u]];
                        a[u] = A[js[u] * p + lane];
                        ++cnt;
                    }
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (js[u] >= 0) {
                        a[u].re -= li.re * lj[u].re + li.im * lj[u].im;
                        a[u].im -= li.im * lj[u].re - li.re * lj[u].im;
                        A[js[u] * p + lane] = a[u];
                    }
                (void)cnt;
            }
        }
        __syncwarp();
    }
    if (lane < p) perm_out[static_cast<size_t>(f) * p + my_step] = lane;
    for (int e = lane; e < p * p; e += 32) GLf[e] = L[e];
    if (lane == 0) {  // Eigen ColPivHouseholderQR rank rule
        if (cholqr_rank(d, p, m) < p) atomicOr(&status[f], kFrameRank);
    }
}

template <int PC>
__global__ void __launch_bounds__(128, FM_SOLVE_MINB) k_rows_solve(const c32* __restrict__ Cin, const c64* __restrict__ Lin,
                                                    const int32_t* __restrict__ perm_in, c32* __restrict__ Vout, int m,
                                                    int p) {
    __shared__ c64 Lp[PC * PC];  // Lp[a * PC + j] = conj-free L_p(j, a) = L[a * p + perm[j]], a < j
    __shared__ double rinv[PC];  // 1 / L_p(j, j)
    __shared__ int perm[PC];
    const int f = blockIdx.y;
    for (int e = threadIdx.x; e < p; e += blockDim.x) perm[e] = perm_in[static_cast<size_t>(f) * p + e];
    __syncthreads();
    const c64* Lf = Lin + static_cast<size_t>(f) * p * p;
    for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
        const int a = e / p, j = e % p;
        Lp[a * PC + j] = Lf[a * p + perm[j]];
    }
    for (int j = threadIdx.x; j < p; j += blockDim.x) {
        const double ljj = Lf[j * p + perm[j]].re;
        rinv[j] = ljj > 0.0 ? 1.0 / ljj : 0.0;
    }
    __syncthreads();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m) return;
    const c32* X = Cin + static_cast<size_t>(f) * m * p;
    c32* Out = Vout + static_cast<size_t>(f) * m * p;
    c32 xin[PC];  // all inputs in flight before the (serial) substitution
#pragma unroll
    for (int j = 0; j < PC; ++j) xin[j] = j < p ? X[static_cast<size_t>(perm[j]) * m + r] : c32{0.f, 0.f};
    c64 v[PC];
#pragma unroll
    for (int j = 0; j < PC; ++j) {
        if (j < p) {
            c64 x = to64(xin[j]);
            c64 x1 = mk(0.0, 0.0);
#pragma unroll
            for (int a = 0; a < PC; ++a) {
                if (a < j) {
                    const c64 l = Lp[a * PC + j];
                    c64& acc = (a & 1) ? x1 : x;
                    acc.re -= v[a].re * l.re + v[a].im * l.im;
                    acc.im -= v[a].im * l.re - v[a].re * l.im;
                }
            }
            const double inv = rinv[j];
            v[j] = mk((x.re + x1.re) * inv, (x.im + x1.im) * inv);
            Out[static_cast<size_t>(j) * m + r] = mk(static_cast<float>(v[j].re), static_cast<float>(v[j].im));
        }
    }
}

}  // namespace smb
}  // namespace fmk

using namespace fmk;

static int32_t* g_sweep_dbg = nullptr;
extern "C" int32_t fm_debug_set_sweep_buffer(int32_t* d) {
    g_sweep_dbg = d;
    return 0;
}
extern "C" int32_t fm_debug_set_phase_buffer(int32_t* d) {
    return cudaMemcpyToSymbol(smb::g_phase_dbg, &d, sizeof(d)) == cudaSuccess ? 0 : 1;
}

cudaError_t fm_launch_cholqr_warp(const void* C, void* work, void* Vout, void* Rt, void* Hout, const void* Vin,
                                  int32_t* status, int frames, int m, int p, bool final_mode, cudaStream_t s) {
    if (p > 32 || p < 1 || m < p) return cudaErrorInvalidValue;
    auto go = [&](auto kern, size_t smem) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        kern<<<frames, smb::kNT, smem, s>>>(static_cast<const c32*>(C), static_cast<c64*>(work),
                                            static_cast<c32*>(Vout), static_cast<c64*>(Rt), static_cast<c64*>(Hout),
                                            static_cast<const c32*>(Vin), status, m, p);
        return cudaGetLastError();
    };
    if (p <= 8) return final_mode ? go(smb::k_cholqr_blk<8, 1>, smb::chol_smem_bytes<8>())
                                  : go(smb::k_cholqr_blk<8, 0>, smb::chol_smem_bytes<8>());
    if (p <= 16) return final_mode ? go(smb::k_cholqr_blk<16, 1>, smb::chol_smem_bytes<16>())
                                   : go(smb::k_cholqr_blk<16, 0>, smb::chol_smem_bytes<16>());
    return final_mode ? go(smb::k_cholqr_blk<32, 1>, smb::chol_smem_bytes<32>())
                      : go(smb::k_cholqr_blk<32, 0>, smb::chol_smem_bytes<32>());
}

// Split orthonormalisation: G -> Lw (in place), perm -> permw, V = C P R^-1 -> Vout.
// gpart != nullptr: G halves already formed by the product kernel (rmul_planes_kernel GM >= 1), no Gram launch.
cudaError_t fm_launch_orth_split(const void* C, void* Vout, void* Lw, int32_t* permw, int32_t* status, int frames,
                                 int m, int p, cudaStream_t s, const void* gpart) {
    if (p > 32 || (p & 3) || m < p || frames < 1) return cudaErrorInvalidValue;
    auto go = [&](auto gram, auto piv, auto solve, int pc, int pw, size_t pbytes) {
        const size_t gsm = sizeof(c64) * pc * pc + sizeof(c64) * 3 * 64 * (pc + 1);
        cudaError_t e = cudaSuccess;
        if (!gpart) {
            e = cudaFuncSetAttribute(gram, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(gsm));
            if (e != cudaSuccess) return e;
            gram<<<frames, smb::kNT, gsm, s>>>(static_cast<const c32*>(C), static_cast<c64*>(Lw), m, p);
            e = cudaGetLastError();
            if (e != cudaSuccess) return e;
        }
        e = cudaFuncSetAttribute(piv, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(pw * pbytes));
        if (e != cudaSuccess) return e;
        piv<<<(frames + pw - 1) / pw, 32 * pw, pw * pbytes, s>>>(static_cast<c64*>(Lw), permw, status, frames, m, p,
                                                                 static_cast<const c64*>(gpart));
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        solve<<<dim3((m + 127) / 128, frames), 128, 0, s>>>(static_cast<const c32*>(C), static_cast<const c64*>(Lw),
                                                            permw, static_cast<c32*>(Vout), m, p);
        return cudaGetLastError();
    };
    using namespace smb;
    if (p <= 8)
        return go(k_gram_only<8>, k_cholpiv_warp<8>, k_rows_solve<8>, 8, PivCfg<8>::kWarps, PivCfg<8>::kWarpBytes);
    if (p <= 16)
        return go(k_gram_only<16>, k_cholpiv_warp<16>, k_rows_solve<16>, 16, PivCfg<16>::kWarps,
                  PivCfg<16>::kWarpBytes);
    return go(k_gram_only<32>, k_cholpiv_warp<32>, k_rows_solve<32>, 32, PivCfg<32>::kWarps, PivCfg<32>::kWarpBytes);
}

// Split final stage: G -> Gw, Herm(H) -> Hw (in place for fast1), T -> Tw (p x k per frame).
// gpart / hpart != nullptr: G and H halves already formed by the product kernel (GM = 2), no Gram launch.
cudaError_t fm_launch_final_split(const void* C, const void* V, void* Hw, void* Gw, void* Tw, void* basis, double* eig,
                                  int32_t* status, int frames, int m, int p, int k, cudaStream_t s,
                                  double* eig_next, const void* gpart, const void* hpart) {
    if (p > 32 || (p & 3) || k > p || m < p || frames < 1) return cudaErrorInvalidValue;
    auto go = [&](auto gram, auto small, auto bas, int pc, int warps, size_t warp_bytes) {
        const size_t gsm = sizeof(c64) * 2 * pc * pc + sizeof(c64) * 3 * 64 * (pc + 1);
        cudaError_t e = cudaSuccess;
        if (!gpart) {
            e = cudaFuncSetAttribute(gram, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(gsm));
            if (e != cudaSuccess) return e;
            gram<<<frames, smb::kNT, gsm, s>>>(static_cast<const c32*>(C), static_cast<const c32*>(V),
                                               static_cast<c64*>(Gw), static_cast<c64*>(Hw), m, p);
            if ((e = cudaGetLastError()) != cudaSuccess) return e;
        }
        const size_t wsm = warp_bytes * warps;
        e = cudaFuncSetAttribute(small, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(wsm));
        if (e != cudaSuccess) return e;
        small<<<(frames + warps - 1) / warps, 32 * warps, wsm, s>>>(static_cast<const c64*>(Gw),
                                                                    static_cast<const c64*>(Hw), static_cast<c64*>(Tw),
                                                                    eig, status, frames, p, k, g_sweep_dbg, eig_next,
                                                                    static_cast<const c64*>(gpart),
                                                                    static_cast<const c64*>(hpart));
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        bas<<<dim3((m + 127) / 128, frames), 128, 0, s>>>(static_cast<const c32*>(C), static_cast<const c64*>(Tw),
                                                          static_cast<c64*>(basis), m, p, k);
        return cudaGetLastError();
    };
    using namespace smb;
    if (p <= 8)
        return go(k_gram_gh<8>, k_small_warp<8>, k_basis_ct<8>, 8, WarpCfg<8>::kWarps, WarpCfg<8>::kWarpBytes);
    if (p <= 16)
        return go(k_gram_gh<16>, k_small_warp<16>, k_basis_ct<16>, 16, WarpCfg<16>::kWarps, WarpCfg<16>::kWarpBytes);
    // p in (16, 32]: one warp per frame (a two-warp variant measured slower: c3 1.29 -> 1.48 ms, the per-round
    // barrier between the two warps costs more than the halved row work)
    return go(k_gram_gh<32>, k_small_warp<32>, k_basis_ct<32>, 32, WarpCfg<32>::kWarps, WarpCfg<32>::kWarpBytes);
}

cudaError_t fm_launch_nystrom_warp2(const void* H, const void* work, const void* Rt, void* basis, double* eig,
                                    int32_t* status, int frames, int m, int p, int k, cudaStream_t s) {
    if (p > 32 || k > p) return cudaErrorInvalidValue;
    auto go = [&](auto kern, size_t smem) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        kern<<<frames, smb::kNT, smem, s>>>(static_cast<const c64*>(H), static_cast<const c64*>(work),
                                            static_cast<const c64*>(Rt), static_cast<c64*>(basis), eig, status, m, p,
                                            k, g_sweep_dbg);
        return cudaGetLastError();
    };
    if (p <= 8) return go(smb::k_nystrom_blk<8>, smb::nys_smem_bytes<8>());
    if (p <= 16) return go(smb::k_nystrom_blk<16>, smb::nys_smem_bytes<16>());
    return go(smb::k_nystrom_blk<32>, smb::nys_smem_bytes<32>());
}
