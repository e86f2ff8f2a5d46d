// K6 + K7 — MUSIC pseudo-spectrum over the angle grid and peak picking, batched.
//
// Reference lines replaced:
//   music_spectrum / denominator_spectrum   R/src/spectrum.cpp:37-68
//   steering_vector                         R/src/scene.cpp:72-82
//   extract_peaks (local_maxima, ranked_maxima, select_separated,
//                  baseline_outside, to_peak_set)  R/src/spectrum.cpp:97-188
//
// Formulation. For an orthonormal basis U (M x K) and a ULA steering vector with
// a_m = z^m, z = exp(j * 2 pi d sin(theta) / lambda), the reference denominator
//     d(theta) = M - ||U^H a||^2 = M - a^H (U U^H) a
// is a trigonometric polynomial in z whose coefficients are the diagonal sums of the
// signal projector:   t_delta = sum_m (U U^H)_{m, m+delta} = sum_k sum_m U_mk conj(U_{m+delta,k})
//     d = (M - t_0) - 2 Re( sum_{delta=1}^{M-1} t_delta z^delta ).
// The t_delta (M complex per frame) are computed once per frame (k_autocorr) and every
// grid point costs M-1 complex Horner steps in fp64 instead of the K*M complex MACs of
// U^H a — and fp64 removes the cancellation M - ||U^H a||^2 that makes an fp32/TF32 GEMM
// of U^H A miss the 0.05 dB gate. The reference floor 1e-12*M is kept.
//
// Layout: basis B x K x M complex<double> (column-major per frame); t B x M complex<double>;
// zgrid L complex<double> (host-computed exp(j*step_l) with the reference's step formula);
// spectrum out B x L (fp32 and/or fp64); peaks B x K int32 cells + fp64 heights, baseline,
// count (shortfall = count < K).

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "fm_common.cuh"

namespace fmk {
namespace spec {

constexpr int kNT = 256;
#ifndef FM_FFT_MINB
#define FM_FFT_MINB 4  // four CTAs per SM (64 registers): 60.7 -> 52.7 us at c2 (scripts_fft_minb.sh)
#endif
constexpr int kNW = kNT / 32;

// t_delta, delta = 0..M-1, for frame blockIdx.x. Thread i owns lags i and M-1-i, so every
// thread performs M+1 products per basis column (the triangle of lags is load-balanced).
__global__ void __launch_bounds__(kNT) k_autocorr(const c64* __restrict__ basis, c64* __restrict__ t, int m, int k,
                                                  const int32_t* __restrict__ only) {
    if (only && !(only[blockIdx.x] & kFrameRefine)) return;
    extern __shared__ c64 col[];  // one basis column (M complex)
    const int f = blockIdx.x;
    const c64* Uf = basis + static_cast<size_t>(f) * m * k;
    const int nh = (m + 1) / 2;
    for (int i0 = 0; i0 < nh; i0 += blockDim.x) {
        const int i = i0 + threadIdx.x;
        const int d1 = i, d2 = m - 1 - i;
        c64 a1 = mk(0.0, 0.0), a2 = mk(0.0, 0.0);
        for (int kk = 0; kk < k; ++kk) {
            __syncthreads();
            for (int r = threadIdx.x; r < m; r += blockDim.x) col[r] = Uf[static_cast<size_t>(kk) * m + r];
            __syncthreads();
            if (i < nh) {
                for (int r = 0; r + d1 < m; ++r) {  // U_r * conj(U_{r+delta})
                    const c64 a = col[r], b = col[r + d1];
                    a1.re = fma(a.re, b.re, fma(a.im, b.im, a1.re));
                    a1.im = fma(a.im, b.re, fma(-a.re, b.im, a1.im));
                }
                if (d2 != d1) {
                    for (int r = 0; r + d2 < m; ++r) {
                        const c64 a = col[r], b = col[r + d2];
                        a2.re = fma(a.re, b.re, fma(a.im, b.im, a2.re));
                        a2.im = fma(a.im, b.re, fma(-a.re, b.im, a2.im));
                    }
                }
            }
        }
        if (i < nh) {
            t[static_cast<size_t>(f) * m + d1] = a1;
            if (d2 != d1) t[static_cast<size_t>(f) * m + d2] = a2;
        }
    }
}

// t_delta by the correlation theorem: with A_k = FFT_N(u_k) (zero-padded, N >= 2M - 1 so the
// circular correlation has no wrap), sum_r u_k[r] conj(u_k[r + delta]) = (1/N) FFT_N(|A_k|^2)[delta],
// hence t = (1/N) FFT_N(P), P = sum_k |A_k|^2 (real). O(K N log N) instead of O(K M^2).
// One CTA per frame; `cnt` columns are transformed in lock-step in shared memory by a self-
// sorting Stockham FFT: radix-8 passes (8-point DFTs in registers) plus one radix-4/2 pass,
// twiddles exp(-2 pi i t k / (R p)) = w1(k)^t from per-pass sincospi tables. Shared indices are
// padded by one slot per 8 (conflict-free stride-8 stores). fp64 throughout.
__device__ __forceinline__ int fpad(int i) { return i + (i >> 3); }
__device__ __forceinline__ c64 cmul(c64 a, c64 b) { return mk(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re); }
__device__ __forceinline__ c64 cadd(c64 a, c64 b) { return mk(a.re + b.re, a.im + b.im); }
__device__ __forceinline__ c64 csub(c64 a, c64 b) { return mk(a.re - b.re, a.im - b.im); }
__device__ __forceinline__ c64 mul_mi(c64 a) { return mk(a.im, -a.re); }  // a * (-i)

template <int R>
__device__ __forceinline__ void dft_r(c64 (&x)[R]) {
    if constexpr (R == 2) {
        const c64 a = x[0], b = x[1];
        x[0] = cadd(a, b);
        x[1] = csub(a, b);
    } else if constexpr (R == 4) {
        const c64 a0 = cadd(x[0], x[2]), a1 = csub(x[0], x[2]), a2 = cadd(x[1], x[3]), a3 = mul_mi(csub(x[1], x[3]));
        x[0] = cadd(a0, a2);
        x[1] = cadd(a1, a3);
        x[2] = csub(a0, a2);
        x[3] = csub(a1, a3);
    } else {
        constexpr double r2 = 0.70710678118654752440;
        const c64 a0 = cadd(x[0], x[4]), a1 = csub(x[0], x[4]), a2 = cadd(x[2], x[6]), a3 = mul_mi(csub(x[2], x[6]));
        const c64 b0 = cadd(x[1], x[5]), b1 = csub(x[1], x[5]), b2 = cadd(x[3], x[7]), b3 = mul_mi(csub(x[3], x[7]));
        const c64 e0 = cadd(a0, a2), e2 = csub(a0, a2), e1 = cadd(a1, a3), e3 = csub(a1, a3);
        const c64 o0 = cadd(b0, b2), o2 = csub(b0, b2), o1 = cadd(b1, b3), o3 = csub(b1, b3);
        const c64 w1 = mk(r2 * (o1.re + o1.im), r2 * (o1.im - o1.re));    // (1 - i)/sqrt2 * o1
        const c64 w2 = mul_mi(o2);                                        // -i * o2
        const c64 w3 = mk(r2 * (o3.im - o3.re), -r2 * (o3.re + o3.im));   // (-1 - i)/sqrt2 * o3
        x[0] = cadd(e0, o0);
        x[4] = csub(e0, o0);
        x[1] = cadd(e1, w1);
        x[5] = csub(e1, w1);
        x[2] = cadd(e2, w2);
        x[6] = csub(e2, w2);
        x[3] = cadd(e3, w3);
        x[7] = csub(e3, w3);
    }
}

// One Stockham pass of radix R with input stride p over cnt transforms (in place: all loads
// of the pass complete before any store). Each thread holds at most 8 values.
template <int R>
__device__ void fft_pass(c64* a, int logn, int cnt, int p, const c64* twp) {
    constexpr int LR = R == 8 ? 3 : (R == 4 ? 2 : 1);
    constexpr int GPT = 8 / R;
    const int nfft = 1 << logn, lt = logn - LR, T = 1 << lt;
    const int total = cnt << lt;
    c64 x[GPT][R];
#pragma unroll
    for (int g = 0; g < GPT; ++g) {
        const int e = threadIdx.x + g * blockDim.x;
        if (e < total) {
            const int q = e >> lt, i = e & (T - 1);
#pragma unroll
            for (int t = 0; t < R; ++t) x[g][t] = a[fpad((q << logn) + i + t * T)];
        }
    }
    __syncthreads();
#pragma unroll
    for (int g = 0; g < GPT; ++g) {
        const int e = threadIdx.x + g * blockDim.x;
        if (e < total) {
            const int q = e >> lt, i = e & (T - 1);
            const int k = i & (p - 1);
            const c64 w1 = twp[k];
            c64 w = w1;
#pragma unroll
            for (int t = 1; t < R; ++t) {
                x[g][t] = cmul(x[g][t], w);
                if (t + 1 < R) w = cmul(w, w1);
            }
            dft_r<R>(x[g]);
            const int j = ((i - k) << LR) + k;
#pragma unroll
            for (int t = 0; t < R; ++t) a[fpad((q << logn) + j + t * p)] = x[g][t];
        }
    }
    __syncthreads();
}

// Full transform of cnt sequences: radix-8 passes, then a radix-4 or radix-2 pass.
__device__ void fft_stockham(c64* a, int logn, int cnt, const c64* tw) {
    int p = 1, off = 0;
    for (int l = logn; l >= 3; l -= 3) {
        fft_pass<8>(a, logn, cnt, p, tw + off);
        off += p;
        p <<= 3;
    }
    const int rem = logn % 3;
    if (rem == 2) fft_pass<4>(a, logn, cnt, p, tw + off);
    else if (rem == 1) fft_pass<2>(a, logn, cnt, p, tw + off);
}

__global__ void __launch_bounds__(kNT, FM_FFT_MINB) k_autocorr_fft(const c64* __restrict__ basis, c64* __restrict__ t, int m, int k,
                                                   int logn, int grp, const int32_t* __restrict__ only) {
    if (only && !(only[blockIdx.x] & kFrameRefine)) return;
    extern __shared__ c64 fsm[];
    const int nfft = 1 << logn;
    c64* tw = fsm;                                         // < nfft entries: per-pass w1 tables
    double* P = reinterpret_cast<double*>(tw + nfft);      // nfft
    c64* buf = reinterpret_cast<c64*>(P + nfft);           // fpad(grp * nfft)
    const int f = blockIdx.x;
    const c64* Uf = basis + static_cast<size_t>(f) * m * k;
    {  // twiddle tables: pass with stride p and radix R holds exp(-2 pi i k / (R p)), k < p
        int p = 1, off = 0;
        for (int l = logn; l > 0;) {
            const int lr = l >= 3 ? 3 : l;
            const int rp = p << lr;
            for (int kk = threadIdx.x; kk < p; kk += blockDim.x) {
                double sn, cs;
                sincospi(-2.0 * static_cast<double>(kk) / static_cast<double>(rp), &sn, &cs);
                tw[off + kk] = mk(cs, sn);
            }
            off += p;
            p = rp;
            l -= lr;
        }
    }
    for (int j = threadIdx.x; j < nfft; j += blockDim.x) P[j] = 0.0;
    for (int k0 = 0; k0 < k; k0 += grp) {
        const int cnt = min(grp, k - k0);
        __syncthreads();  // previous group's P accumulation done with buf; tables ready
        for (int e0 = 0; e0 < (cnt << logn); e0 += 8 * blockDim.x) {  // 8 loads in flight per thread
            c64 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = e0 + threadIdx.x + u * blockDim.x;
                const int q = e >> logn, r = e & (nfft - 1);
                v[u] = (e < (cnt << logn) && r < m) ? Uf[static_cast<size_t>(k0 + q) * m + r] : mk(0.0, 0.0);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = e0 + threadIdx.x + u * blockDim.x;
                if (e < (cnt << logn)) buf[fpad(e)] = v[u];
            }
        }
        __syncthreads();
        fft_stockham(buf, logn, cnt, tw);
        for (int j = threadIdx.x; j < nfft; j += blockDim.x) {
            double acc = P[j];
            for (int q = 0; q < cnt; ++q) acc += norm2(buf[fpad((q << logn) + j)]);
            P[j] = acc;
        }
    }
    __syncthreads();
    for (int r = threadIdx.x; r < nfft; r += blockDim.x) buf[fpad(r)] = mk(P[r], 0.0);
    __syncthreads();
    fft_stockham(buf, logn, 1, tw);
    const double inv = 1.0 / static_cast<double>(nfft);
    for (int d = threadIdx.x; d < m; d += blockDim.x) {
        const c64 v = buf[fpad(d)];
        t[static_cast<size_t>(f) * m + d] = mk(v.re * inv, v.im * inv);
    }
}

struct PeakOut {
    int32_t* cells;     // B x K
    double* heights;    // B x K
    double* baseline;   // B
    int32_t* count;     // B
};

// Spectrum only (fp64 Horner over z), one CTA per frame, any grid: the facade's music_spectrum, and the exact
// method's recomputation of the frames the Jacobi solver redid (only != nullptr: frames with kFrameRefine).
__global__ void __launch_bounds__(kNT) k_spectrum_one(const c64* __restrict__ t, const c64* __restrict__ zgrid, int m,
                                                      int L, float* __restrict__ spec32, double* __restrict__ spec64,
                                                      const int32_t* __restrict__ only) {
    extern __shared__ c64 st1[];
    const int f = blockIdx.x;
    if (only && !(only[f] & kFrameRefine)) return;
    for (int r = threadIdx.x; r < m; r += kNT) st1[r] = t[static_cast<size_t>(f) * m + r];
    __syncthreads();
    const double c0 = static_cast<double>(m) - st1[0].re;
    const double floor_v = 1e-12 * static_cast<double>(m);
    for (int l = threadIdx.x; l < L; l += kNT) {
        const c64 z = zgrid[l];
        double pr = 0.0, pi = 0.0;
        if (m > 1) {
            pr = st1[m - 1].re;
            pi = st1[m - 1].im;
            for (int dlt = m - 2; dlt >= 1; --dlt) {
                const double nr = fma(pr, z.re, fma(-pi, z.im, st1[dlt].re));
                const double ni = fma(pr, z.im, fma(pi, z.re, st1[dlt].im));
                pr = nr;
                pi = ni;
            }
            pr = pr * z.re - pi * z.im;  // Re(p * z)
        }
        const double P = 1.0 / fmax(c0 - 2.0 * pr, floor_v);
        spec64[static_cast<size_t>(f) * L + l] = P;
        if (spec32) spec32[static_cast<size_t>(f) * L + l] = static_cast<float>(P);
    }
}

// Spectrum for kFPB frames at once: thread = grid point l, the block's kFPB frames share one
// fp64 power sequence z_l^delta (4 DFMA per step) and each frame adds Re(t_delta z^delta)
// (2 DFMA) from a shared-memory broadcast of its coefficients: ~2.25 DFMA per (frame, point,
// delta) versus 4 for a per-frame Horner. The z^delta recurrence error (~delta * eps64) is far
// below the fp64 cancellation budget of d = (M - t_0) - 2 Re sum_delta t_delta z^delta.
constexpr int kFPB = 16;  // frames per block (8 when 16 x M coefficients exceed shared memory)

template <int kFPB>
__global__ void __launch_bounds__(kNT) k_spectrum_multi(const c64* __restrict__ t, const c64* __restrict__ zgrid,
                                                        int frames, int m, int L, float* __restrict__ spec32,
                                                        double* __restrict__ spec64) {
    extern __shared__ c64 st[];  // kFPB x m coefficients, delta-major: st[delta * kFPB + f]
    const int f0 = blockIdx.y * kFPB;
    const int nf = min(kFPB, frames - f0);
    for (int e = threadIdx.x; e < kFPB * m; e += kNT) {
        const int f = e / m, dl = e % m;
        st[dl * kFPB + f] = f < nf ? t[static_cast<size_t>(f0 + f) * m + dl] : mk(0.0, 0.0);
    }
    __syncthreads();
    // two grid points per thread (l0, l0 + half): 2 power sequences share every coefficient load
    const int half = (L + 1) / 2;
    const int l0 = blockIdx.x * kNT + threadIdx.x;
    if (l0 >= half) return;
    const int l1 = l0 + half;
    const bool has1 = l1 < L;
    const c64 za = zgrid[l0];
    const c64 zb = has1 ? zgrid[l1] : mk(1.0, 0.0);
    double acc0[kFPB], acc1[kFPB];
#pragma unroll
    for (int f = 0; f < kFPB; ++f) acc0[f] = acc1[f] = 0.0;
    double ar = 1.0, ai = 0.0, br = 1.0, bi = 0.0;
    for (int dl = 1; dl < m; ++dl) {
        const double nar = fma(ar, za.re, -ai * za.im);
        const double nai = fma(ar, za.im, ai * za.re);
        const double nbr = fma(br, zb.re, -bi * zb.im);
        const double nbi = fma(br, zb.im, bi * zb.re);
        ar = nar;
        ai = nai;
        br = nbr;
        bi = nbi;
        const c64* row = st + dl * kFPB;
#pragma unroll
        for (int f = 0; f < kFPB; ++f) {
            const c64 c = row[f];
            acc0[f] = fma(c.re, ar, fma(-c.im, ai, acc0[f]));
            acc1[f] = fma(c.re, br, fma(-c.im, bi, acc1[f]));
        }
    }
    const double floor_v = 1e-12 * static_cast<double>(m);
#pragma unroll
    for (int f = 0; f < kFPB; ++f) {
        if (f < nf) {
            const double c0 = static_cast<double>(m) - st[f].re;
            const double P0 = 1.0 / fmax(c0 - 2.0 * acc0[f], floor_v);
            const size_t o = static_cast<size_t>(f0 + f) * L;
            if (spec32) spec32[o + l0] = static_cast<float>(P0);
            spec64[o + l0] = P0;
            if (has1) {
                const double P1 = 1.0 / fmax(c0 - 2.0 * acc1[f], floor_v);
                if (spec32) spec32[o + l1] = static_cast<float>(P1);
                spec64[o + l1] = P1;
            }
        }
    }
}

// Peaks, one 128-thread CTA per frame (R/src/spectrum.cpp:97-188, any L >= 1 and K >= 1):
//  1. values -> shared memory (coalesced, 8 loads in flight per thread), or read in place from global memory when
//     the frame's workspace does not fit (long grids / large K: the workspace then lives in `gws`);
//  2. strict interior maxima (leftmost-plateau rule, local_maxima :105-122), 32 consecutive cells per warp step,
//     compacted in cell order (ballots -> per-warp counts -> prefix); the exact capacity floor((L-1)/2) holds them
//     all (strict maxima are never adjacent);
//  3. warp 0 runs the greedy (ranked_maxima + select_separated :124-148) as K argmax rounds over the list: the
//     best (height desc, cell asc) candidate not yet excluded is the reference walk's next acceptance (a candidate
//     that clashes with an accepted pick stays rejected), then candidates with |c - s| < min_sep (and c == s) are
//     excluded; no sort. The argmax starts at -inf, so any finite spectrum (dB scale, negative values) works;
//  4. baseline_outside (:150-164) = max over cells with |l - s| > min_sep for every pick (bitmask), init 0 (fmax
//     drops NaN like std::max(p0, NaN)); picks in ascending cell order (to_peak_set :166-178).
constexpr int kPRT = 128;
constexpr int kPCL = 8;  // register-held candidates per lane (256 per frame)

struct PeakLayout {
    int cap, nmask, ngroups;
    size_t o_sv, o_selh, o_cl, o_near, o_bal, o_sel, o_ex, bytes;
};
__host__ __device__ inline PeakLayout peak_layout(int L, int K, bool with_values) {
    PeakLayout p;
    p.cap = L > 2 ? (L - 1) / 2 : 1;
    p.nmask = (L + 31) / 32;
    p.ngroups = L > 2 ? (L - 2 + 31) / 32 : 0;
    size_t o = 0;
    p.o_sv = o;
    if (with_values) o += sizeof(double) * static_cast<size_t>(L);
    p.o_selh = o;
    o += sizeof(double) * static_cast<size_t>(K);
    p.o_cl = o;
    o += sizeof(int) * static_cast<size_t>(p.cap);
    p.o_near = o;
    o += sizeof(uint32_t) * static_cast<size_t>(p.nmask);
    p.o_bal = o;
    o += sizeof(uint32_t) * static_cast<size_t>(p.ngroups + 1);
    p.o_sel = o;
    o += sizeof(int) * static_cast<size_t>(K);
    p.o_ex = o;
    o += static_cast<size_t>(p.cap);
    p.bytes = (o + 15) & ~size_t(15);
    return p;
}
constexpr size_t kPeakSmemMax = 220 * 1024;

__device__ __forceinline__ bool better_w(double h1, int c1, double h2, int c2) {
    return h1 > h2 || (h1 == h2 && c1 < c2);
}

template <bool kInSmem, int NT = kPRT>
__global__ void __launch_bounds__(NT) k_peaks_rounds(const double* __restrict__ values, int L, int K, int min_sep,
                                                      PeakOut out, uint8_t* __restrict__ gws,
                                                      const int32_t* __restrict__ only) {
    extern __shared__ __align__(16) uint8_t prs[];
    const PeakLayout lay = peak_layout(L, K, kInSmem);
    const int f = blockIdx.x;
    if (only && !(only[f] & kFrameRefine)) return;
    uint8_t* base = kInSmem ? prs : gws + static_cast<size_t>(f) * lay.bytes;
    const double* v = values + static_cast<size_t>(f) * L;
    double* svw = reinterpret_cast<double*>(base + lay.o_sv);
    const double* sv = kInSmem ? svw : v;
    double* s_selh = reinterpret_cast<double*>(base + lay.o_selh);
    int* cl = reinterpret_cast<int*>(base + lay.o_cl);
    uint32_t* near = reinterpret_cast<uint32_t*>(base + lay.o_near);
    uint32_t* bal_s = reinterpret_cast<uint32_t*>(base + lay.o_bal);
    int* s_sel = reinterpret_cast<int*>(base + lay.o_sel);
    uint8_t* ex = base + lay.o_ex;
    const int nmask = lay.nmask;
    __shared__ int s_cnt[NT / 32];
    __shared__ int s_nsel;
    __shared__ double s_wmax[NT / 32];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (kInSmem) {
        for (int l0 = tid; l0 < L; l0 += 8 * NT) {
            double tmp[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int l = l0 + u * NT;
                tmp[u] = l < L ? __ldcs(v + l) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int l = l0 + u * NT;
                if (l < L) svw[l] = tmp[u];
            }
        }
    }
    for (int w = tid; w < nmask; w += NT) near[w] = 0u;
    __syncthreads();
    auto is_max = [&](int l) -> bool {
        if (l < 1 || l >= L - 1) return false;
        const double x = sv[l], xm = sv[l - 1], xp = sv[l + 1];
        if (!(x > xm)) return false;
        if (xp < x) return true;
        if (!(xp == x)) return false;
        int r = l + 1;  // plateau: leftmost cell is the maximum if the run then falls
        while (r + 1 < L && sv[r + 1] == x) ++r;
        return (r + 1 < L) && sv[r + 1] < x;
    };
    const int ngroups = lay.ngroups;
    const int gpw = (ngroups + NT / 32 - 1) / (NT / 32);
    const int g0 = warp * gpw, g1 = min(ngroups, g0 + gpw);
    int cnt = 0;
    for (int gb = g0; gb < g1; gb += 4) {  // four groups' loads in flight
        double xv[4], xm[4], xp[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int l = 1 + 32 * (gb + u) + lane;
            const bool in = gb + u < g1 && l < L - 1;
            xv[u] = in ? sv[l] : 0.0;
            xm[u] = in ? sv[l - 1] : 0.0;
            xp[u] = in ? sv[l + 1] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (gb + u >= g1) break;  // warp-uniform
            const int l = 1 + 32 * (gb + u) + lane;
            bool mx = l < L - 1 && xv[u] > xm[u] && xp[u] <= xv[u];
            if (mx && xp[u] == xv[u]) mx = is_max(l);  // plateau
            const uint32_t bal = __ballot_sync(0xffffffffu, mx);
            if (lane == 0) bal_s[gb + u] = bal;
            cnt += __popc(bal);
        }
    }
    if (lane == 0) s_cnt[warp] = cnt;
    __syncthreads();
    int off = 0, nc = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) {
        off += w < warp ? s_cnt[w] : 0;
        nc += s_cnt[w];
    }
    for (int g = g0; g < g1; ++g) {
        const uint32_t bal = bal_s[g];
        if ((bal >> lane) & 1u) {
            const int pos = off + __popc(bal & ((1u << lane) - 1u));
            cl[pos] = 1 + 32 * g + lane;
            ex[pos] = 0;
        }
        off += __popc(bal);
    }
    __syncthreads();
    if (warp == 0 && nc <= 32 * kPCL) {  // greedy rounds, candidates in registers (any MUSIC spectrum: < M maxima);
        // lane holds list entries lane + 32 u (ascending cells within the lane)
        double hv[kPCL];
        int cv[kPCL];
        uint32_t live = 0u;
#pragma unroll
        for (int u = 0; u < kPCL; ++u) {
            const int j = lane + 32 * u;
            cv[u] = j < nc ? cl[j] : 0x7fffffff;
            hv[u] = j < nc ? sv[cv[u]] : -INFINITY;
            if (j < nc) live |= 1u << u;
        }
        int nsel = 0;
        for (; nsel < K; ++nsel) {
            double h = -INFINITY;
            int c = 0x7fffffff;
#pragma unroll
            for (int u = 0; u < kPCL; ++u)
                if (((live >> u) & 1u) && (c == 0x7fffffff || better_w(hv[u], cv[u], h, c))) {
                    h = hv[u];
                    c = cv[u];
                }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double oh = __shfl_xor_sync(0xffffffffu, h, o);
                const int oc = __shfl_xor_sync(0xffffffffu, c, o);
                if (oc != 0x7fffffff && (c == 0x7fffffff || better_w(oh, oc, h, c))) {
                    h = oh;
                    c = oc;
                }
            }
            if (c == 0x7fffffff) break;
            if (lane == 0) {
                s_sel[nsel] = c;
                s_selh[nsel] = h;
            }
#pragma unroll
            for (int u = 0; u < kPCL; ++u)  // clash: |c_u - s| < min_sep, and c_u == s
                if (abs(cv[u] - c) < min_sep || cv[u] == c) live &= ~(1u << u);
            for (int d = lane - min_sep; d <= min_sep; d += 32) {
                const int l = c + d;
                if (l >= 0 && l < L) atomicOr(&near[l >> 5], 1u << (l & 31));
            }
        }
        if (lane == 0) s_nsel = nsel;
    } else if (warp == 0) {  // greedy rounds over the compacted list
        int nsel = 0;
        for (; nsel < K; ++nsel) {
            double h = -INFINITY;
            int c = 0x7fffffff, jb = -1;
            for (int j = lane; j < nc; j += 32)
                if (!ex[j]) {
                    const int cj = cl[j];
                    const double hj = sv[cj];
                    if (jb < 0 || better_w(hj, cj, h, c)) {
                        h = hj;
                        c = cj;
                        jb = j;
                    }
                }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double oh = __shfl_xor_sync(0xffffffffu, h, o);
                const int oc = __shfl_xor_sync(0xffffffffu, c, o);
                const int oj = __shfl_xor_sync(0xffffffffu, jb, o);
                if (oj >= 0 && (jb < 0 || better_w(oh, oc, h, c))) {
                    h = oh;
                    c = oc;
                    jb = oj;
                }
            }
            if (jb < 0) break;
            if (lane == 0) {
                s_sel[nsel] = c;
                s_selh[nsel] = h;
            }
            // clash band around the pick: the list is in cell order, so walk outwards from its index
            for (int d = lane;; d += 32) {
                bool any = false;
                const int jl = jb - d, jr = jb + d;
                if (jl >= 0 && (c - cl[jl] < min_sep || jl == jb)) {
                    ex[jl] = 1;
                    any = true;
                }
                if (jr < nc && cl[jr] - c < min_sep) {
                    ex[jr] = 1;
                    any = true;
                }
                if (!__any_sync(0xffffffffu, any)) break;
            }
            for (int d = lane - min_sep; d <= min_sep; d += 32) {
                const int l = c + d;
                if (l >= 0 && l < L) atomicOr(&near[l >> 5], 1u << (l & 31));
            }
            __syncwarp();
        }
        if (lane == 0) s_nsel = nsel;
    }
    __syncthreads();
    double p0 = 0.0;
    for (int l = tid; l < L; l += NT)
        if (!((near[l >> 5] >> (l & 31)) & 1u)) p0 = fmax(p0, sv[l]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) p0 = fmax(p0, __shfl_xor_sync(0xffffffffu, p0, o));
    if (lane == 0) s_wmax[warp] = p0;
    __syncthreads();
    const int nsel = s_nsel;
    for (int xk = tid; xk < K; xk += NT) {
        if (xk < nsel) {
            const int c = s_sel[xk];
            int rank = 0;
            for (int y = 0; y < nsel; ++y) rank += s_sel[y] < c ? 1 : 0;
            out.cells[static_cast<size_t>(f) * K + rank] = c;
            out.heights[static_cast<size_t>(f) * K + rank] = s_selh[xk];
        } else {
            out.cells[static_cast<size_t>(f) * K + xk] = -1;
            out.heights[static_cast<size_t>(f) * K + xk] = 0.0;
        }
    }
    if (tid == 0) {
        double b = 0.0;
        for (int w = 0; w < NT / 32; ++w) b = fmax(b, s_wmax[w]);
        out.baseline[f] = b;
        out.count[f] = nsel;
    }
}

// max |U^H U - I| per frame (music_spectrum precondition, R/src/spectrum.cpp:55-61).
__global__ void __launch_bounds__(kNT) k_orthocheck(const c64* __restrict__ basis, int m, int k,
                                                    double* __restrict__ dev) {
    __shared__ double s_w[kNW];
    const int f = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const c64* Uf = basis + static_cast<size_t>(f) * m * k;
    double mx = 0.0;
    for (int e = warp; e < k * k; e += kNW) {
        const int i = e % k, j = e / k;
        c64 s = mk(0.0, 0.0);
        for (int r = lane; r < m; r += 32) cmac_conj(s, Uf[static_cast<size_t>(i) * m + r], Uf[static_cast<size_t>(j) * m + r]);
        s.re = warp_sum(s.re);
        s.im = warp_sum(s.im);
        if (i == j) s.re -= 1.0;
        mx = fmax(mx, sqrt(norm2(s)));
    }
    if (lane == 0) s_w[warp] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = 0.0;
        for (int w = 0; w < kNW; ++w) b = fmax(b, s_w[w]);
        dev[f] = b;
    }
}

}  // namespace spec
}  // namespace fmk

using namespace fmk;

cudaError_t fm_launch_autocorr(const void* basis, void* t, int frames, int m, int k, cudaStream_t s,
                               const int32_t* only) {
    int logn = 1;
    while ((1 << logn) < 2 * m - 1) ++logn;
    if (logn <= 12) {  // FFT in shared memory (M <= 2048)
        const int nfft = 1 << logn;
        const size_t fixed = sizeof(c64) * nfft + sizeof(double) * nfft;
        const size_t per = sizeof(c64) * (nfft + nfft / 8);  // padded
        const size_t budget = 96 * 1024;
        int grp = static_cast<int>(std::max<size_t>(1, budget > fixed ? (budget - fixed) / per : 1));
        grp = std::min(grp, std::max(1, 8 * spec::kNT / nfft));  // <= 8 values per thread per pass
        grp = std::max(1, std::min(grp, k));
        const size_t smem = fixed + per * grp + sizeof(c64);
        if (smem <= 200 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(spec::k_autocorr_fft, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(smem));
            if (e != cudaSuccess) return e;
            spec::k_autocorr_fft<<<frames, spec::kNT, smem, s>>>(static_cast<const c64*>(basis), static_cast<c64*>(t),
                                                                 m, k, logn, grp, only);
            return cudaGetLastError();
        }
    }
    // direct lag sums (large M)
    const size_t smem = sizeof(c64) * m;
    if (smem > 220 * 1024) return cudaErrorInvalidValue;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(spec::k_autocorr, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    const int threads = std::min(spec::kNT, std::max(32, ((m + 1) / 2 + 31) / 32 * 32));
    spec::k_autocorr<<<frames, threads, smem, s>>>(static_cast<const c64*>(basis), static_cast<c64*>(t), m, k, only);
    return cudaGetLastError();
}

// Facade music_spectrum: spectrum only, any grid, one CTA per frame.
cudaError_t fm_launch_spectrum_one(const void* t, const void* zgrid, int frames, int m, int L, float* spec32,
                                   double* spec64, cudaStream_t s, const int32_t* only) {
    const size_t smem = sizeof(c64) * m;
    if (smem > 220 * 1024) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(spec::k_spectrum_one, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    spec::k_spectrum_one<<<frames, spec::kNT, smem, s>>>(static_cast<const c64*>(t), static_cast<const c64*>(zgrid), m, L,
                                                         spec32, spec64, only);
    return cudaGetLastError();
}

// Any grid (the plan's path when theta0 != -theta1): kFPB frames per CTA share one fp64 power sequence.
cudaError_t fm_launch_spectrum_multi(const void* t, const void* zgrid, int frames, int m, int L, float* spec32,
                                     double* spec64, cudaStream_t s) {
    auto go = [&](auto kern, int fpb) {
        const size_t smem = sizeof(c64) * fpb * m;
        if (smem > 200 * 1024) return cudaErrorInvalidValue;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        dim3 grid(((L + 1) / 2 + spec::kNT - 1) / spec::kNT, (frames + fpb - 1) / fpb);
        kern<<<grid, spec::kNT, smem, s>>>(static_cast<const c64*>(t), static_cast<const c64*>(zgrid), frames, m, L,
                                           spec32, spec64);
        return cudaGetLastError();
    };
    if (sizeof(c64) * 16 * m <= 200 * 1024) return go(spec::k_spectrum_multi<16>, 16);
    if (sizeof(c64) * 8 * m <= 200 * 1024) return go(spec::k_spectrum_multi<8>, 8);
    return go(spec::k_spectrum_multi<4>, 4);
}

// Global workspace bytes fm_launch_peaks_only needs for `frames` frames (0: the frame fits in shared memory).
size_t fm_peaks_workspace_bytes(int frames, int L, int K) {
    if (spec::peak_layout(L, K, true).bytes <= spec::kPeakSmemMax) return 0;
    return static_cast<size_t>(frames) * spec::peak_layout(L, K, false).bytes;
}

// extract_peaks on B x L fp64 values (R/src/spectrum.cpp:182-188), any L >= 1, K >= 1. gws: device workspace of
// fm_peaks_workspace_bytes(frames, L, K) bytes when that is non-zero.
cudaError_t fm_launch_peaks_only(const double* values, int frames, int L, int K, int min_sep, int32_t* cells,
                                 double* heights, double* baseline, int32_t* count, void* gws, cudaStream_t s,
                                 const int32_t* only) {
    if (K < 1 || L < 1 || frames < 1) return cudaErrorInvalidValue;
    spec::PeakOut out{cells, heights, baseline, count};
    const spec::PeakLayout lay = spec::peak_layout(L, K, true);
    if (lay.bytes <= spec::kPeakSmemMax) {
#ifndef FM_PEAKS_LONG_NT
#define FM_PEAKS_LONG_NT 512
#endif
        if (L > 8192) {  // long grids (c4's 18001 cells): one frame per SM by shared memory -> more warps per frame
            constexpr int NT = FM_PEAKS_LONG_NT;
            cudaError_t e = cudaFuncSetAttribute(spec::k_peaks_rounds<true, NT>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(lay.bytes));
            if (e != cudaSuccess) return e;
            spec::k_peaks_rounds<true, NT><<<frames, NT, lay.bytes, s>>>(values, L, K, min_sep, out, nullptr, only);
            return cudaGetLastError();
        }
        cudaError_t e = cudaFuncSetAttribute(spec::k_peaks_rounds<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(lay.bytes));
        if (e != cudaSuccess) return e;
        spec::k_peaks_rounds<true><<<frames, spec::kPRT, lay.bytes, s>>>(values, L, K, min_sep, out, nullptr, only);
    } else {
        if (!gws) return cudaErrorInvalidValue;
        spec::k_peaks_rounds<false><<<frames, spec::kPRT, 0, s>>>(values, L, K, min_sep, out,
                                                                 static_cast<uint8_t*>(gws), only);
    }
    return cudaGetLastError();
}

cudaError_t fm_launch_orthocheck(const void* basis, int frames, int m, int k, double* dev, cudaStream_t s) {
    spec::k_orthocheck<<<frames, spec::kNT, 0, s>>>(static_cast<const c64*>(basis), m, k, dev);
    return cudaGetLastError();
}
