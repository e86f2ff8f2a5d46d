// MUSIC pseudo-spectrum on the 5th-gen INT8 tensor cores, mirror-symmetric grids (theta_0 = -theta_{L-1}) as
// pairs (theta, -theta) sharing one evaluation, any other grid (half mode: the ToA beat grid, asymmetric spans) with
// every point a pair of its own and the mirror values dropped:
// tcgen05.mma kind::i8 with TMEM int32 accumulators, operands streamed by bulk async copies
// (R/src/spectrum.cpp:37-68 music_spectrum; steering R/src/scene.cpp:72-82).
//
// With t_delta the projector's diagonal sums (k_autocorr_fft) and z_q = e^{j phi_q}:
//   A(f, q) = sum_delta Re t_delta cos(delta phi_q),  B(f, q) = sum_delta Im t_delta sin(delta phi_q),
//   d(theta_q) = c0 - 2 (A - B),  d(-theta_q) = c0 - 2 (A + B),  P = 1 / max(d, 1e-12 M),
// evaluated exactly to fp64 level by digit splitting (Ozaki scheme): t / scale_f and the plan's cos / sin / 2 as
// five signed base-128 digits (|digit| <= 64), the 15 digit products with a + b <= 4 summed exactly in int32 per
// group g = a + b, the groups combined exactly in int64 and rounded once to fp64 (weights 128^-(g+2)).
//
// Tiles: 128 frames (M: the frames' t digits, A operand) x 48 mirror pairs (N: the z digits, B operand) per CTA;
// the K loop walks delta in blocks of 32 (one kind::i8 MMA each). Both operands are stored pre-tiled in the UMMA
// canonical K-major layout (no swizzle: 8-row x 16-byte core matrices, LBO 128 B along K, SBO 256 B along rows),
// so a stage -- the 10 A planes (5 digits x Re / Im, 40 KB) and 10 B planes (5 digits x cos / sin, 15 KB) of one
// K block -- is two contiguous bulk copies. One thread issues the 30 MMAs per K block (15 digit pairs x A / B) into
// 10 TMEM accumulators of 48 columns (480 of 512); the epilogue warps drain TMEM (one frame per lane), stage both
// mirror cells in the idle pipeline smem and write coalesced rows of cells.
//
// Layouts (device, int8): tK [frame tile][K block][plane = s * 2 + ri][128 x 32 canonical] (k_slice_tk, per batch),
// zK [pair tile][K block][plane = s * 2 + cs][48 x 32 canonical] (plan table, capi.cu zdig_host_k).

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "fm_common.cuh"
#include "tc_common.cuh"

namespace fmk {
namespace spectc {

using namespace fmk::tc;

constexpr int kS = 5;                  // digit slices per operand
constexpr int kPlanes = 2 * kS;        // x (Re / Im, cos / sin)
constexpr int kM = 128;                // frames per tile
constexpr int kN = 48;                 // mirror pairs per tile
constexpr int kK = 32;                 // delta per K block (one MMA)
#ifndef STC_STAGES
#define STC_STAGES 3
#endif
constexpr int kStages = STC_STAGES;
constexpr int kAPlane = kM * kK;       // 4 KB (one plane of one K block, canonical layout)
constexpr int kBPlane = kN * kK;       // 1.5 KB
constexpr int kStageBytes = kPlanes * (kAPlane + kBPlane);  // 56320
#ifndef STC_EPI_SPLIT
#define STC_EPI_SPLIT 3
#endif
constexpr int kSplit = STC_EPI_SPLIT;  // epilogue warps per TMEM lane quarter (column split)
constexpr int kThreads = 64 + 128 * kSplit;  // w0 TMA, w1 MMA, w2.. epilogue
constexpr int kTmemCols = 512;
constexpr int kSmem = 1024 + kStages * kStageBytes + 256;
#ifdef STC_TIMELINE
__device__ long long g_stc_tl[4096 * 8];  // micro-benchmark only (tools/micro/spec_tc_bench.cu)
#define STC_STAMP(slot) g_stc_tl[(blockIdx.y * gridDim.x + blockIdx.x) * 8 + (slot)] = clock64()
#else
#define STC_STAMP(slot)
#endif
constexpr int kRow = 2 * kN + 1;       // epilogue staging row (doubles; odd: 2-wavefront 8-byte stores)
static_assert(4 * 32 * kRow * 8 <= kStages * kStageBytes, "epilogue staging fits the pipeline smem");

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}

// Byte offset of (row, k) in one canonical K-major plane tile of 32-byte rows: core matrices of 8 rows x 16 B.
__host__ __device__ __forceinline__ int canon_off(int row, int k) {
    return (row >> 3) * 256 + (k >> 4) * 128 + (row & 7) * 16 + (k & 15);
}
// UMMA descriptor of a canonical K-major tile without swizzle: LBO = 128 B (next core matrix along K), SBO = 256 B
// (next 8-row group).
__device__ __forceinline__ uint64_t desc_canon(uint32_t saddr) {
    return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>(128 >> 4) << 16) |
           (static_cast<uint64_t>(256 >> 4) << 32) | (1ull << 46);
}
// kind::i8: D = S32 (2), A = B = signed int8 (1), K-major, N = kN, M = kM.
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((static_cast<uint32_t>(kN) >> 3) << 17) |
                            ((static_cast<uint32_t>(kM) >> 4) << 24);

__device__ __forceinline__ void umma_i8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(kIdesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar)
                 : "memory");
}

// t digits for the tensor-core kernel in the tK layout (frames of this call; rows f >= frames and delta = 0 or
// >= m zero), scale[f] = power of two >= 2 max |t_delta| (delta >= 1). Thread j writes deltas 4 j .. 4 j + 3 of
// all 10 planes as 32-bit words.
__global__ void __launch_bounds__(256) k_slice_tk(const c64* __restrict__ t, int8_t* __restrict__ tk,
                                                  double* __restrict__ tscale, int frames, int m, int nkb) {
    __shared__ double red[8];
    const int f = blockIdx.x, tid = threadIdx.x;
    const int row = f % kM;
    int8_t* tile = tk + static_cast<size_t>(f / kM) * nkb * kPlanes * kAPlane;
    const c64* tf = t + static_cast<size_t>(f) * m;
    double mx = 0.0;
    if (f < frames)
        for (int d = 1 + tid; d < m; d += 256) mx = fmax(mx, fmax(fabs(tf[d].re), fabs(tf[d].im)));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((tid & 31) == 0) red[tid >> 5] = mx;
    __syncthreads();
    mx = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) mx = fmax(mx, red[w]);
    int e = 0;
    frexp(2.0 * mx, &e);  // 2 mx < 2^e
    const double scale = mx > 0.0 ? ldexp(1.0, e) : 1.0;
    if (tid == 0 && f < frames) tscale[f] = scale;
    const double inv = 1.0 / scale;  // exact (power of two)
    for (int d0 = 4 * tid; d0 < kK * nkb; d0 += 4 * 256) {
        uint32_t w[kPlanes] = {};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int d = d0 + u;
            const bool live = f < frames && d >= 1 && d < m;
            double r[2] = {live ? tf[d].re * inv : 0.0, live ? tf[d].im * inv : 0.0};
#pragma unroll
            for (int sl = 0; sl < kS; ++sl)
#pragma unroll
                for (int ri = 0; ri < 2; ++ri) {
                    const double x = 128.0 * r[ri];
                    const double dg = rint(x);
                    r[ri] = x - dg;
                    w[sl * 2 + ri] |= (static_cast<uint32_t>(static_cast<int>(dg)) & 0xFFu) << (8 * u);
                }
        }
        const int kb = d0 / kK;
        int8_t* base = tile + static_cast<size_t>(kb) * kPlanes * kAPlane + canon_off(row, d0 % kK);
#pragma unroll
        for (int pl = 0; pl < kPlanes; ++pl) *reinterpret_cast<uint32_t*>(base + pl * kAPlane) = w[pl];
    }
}

__global__ void __launch_bounds__(kThreads, 1)
    k_spectrum_tc(const int8_t* __restrict__ tk, const int8_t* __restrict__ zk, const double* __restrict__ tscale, const c64* __restrict__ t, int frames, int m, int nkb, int L,
                  float* __restrict__ spec32, double* __restrict__ spec64, int half) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + kStages;
    uint64_t* acc_full = bars + 2 * kStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int f0 = blockIdx.y * kM, q0 = blockIdx.x * kN;
    if (threadIdx.x == 0) {
        STC_STAMP(0);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(smem_u32(&full[s]), 1);
            mbar_init(smem_u32(&empty[s]), 1);
        }
        mbar_init(smem_u32(acc_full), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // warp-uniform: MMA operands in uniform registers

    if (warp == 0) {
        if (lane == 0) {  // producer: per K block, the A planes (40 KB) and the B planes (15 KB), one bulk copy each
            const int8_t* ta = tk + static_cast<size_t>(blockIdx.y) * nkb * kPlanes * kAPlane;
            const int8_t* zb = zk + static_cast<size_t>(blockIdx.x) * nkb * kPlanes * kBPlane;
            for (int kb = 0; kb < nkb; ++kb) {
                const int s = kb % kStages;
                mbar_wait(smem_u32(&empty[s]), ((kb / kStages) & 1) ^ 1);
                const uint32_t fb = smem_u32(&full[s]);
                mbar_arrive_expect_tx(fb, kStageBytes);
                const uint32_t st = smem_u32(smem + s * kStageBytes);
                bulk_g2s(st, ta + static_cast<size_t>(kb) * kPlanes * kAPlane, kPlanes * kAPlane, fb);
                bulk_g2s(st + kPlanes * kAPlane, zb + static_cast<size_t>(kb) * kPlanes * kBPlane, kPlanes * kBPlane, fb);
            }
        }
    } else if (warp == 1) {
        {  // MMA issuer: the warp stays converged (operands in uniform registers), one elected lane issues;
           // accumulator (group g, A | B) at columns (2 g + x) kN
            STC_STAMP(1);
            for (int kb = 0; kb < nkb; ++kb) {
                const int s = kb % kStages;
                mbar_wait(smem_u32(&full[s]), (kb / kStages) & 1);
                tc_fence_after();
                if (kb == 0) STC_STAMP(2);
                const uint32_t st = smem_u32(smem + s * kStageBytes);
                const uint32_t sb = st + kPlanes * kAPlane;
                if (elect_one()) {
#pragma unroll
                for (int a = 0; a < kS; ++a)
#pragma unroll
                    for (int b = 0; a + b < kS; ++b) {
                        const int g = a + b;
                        const uint32_t acc = (kb > 0 || a > 0) ? 1u : 0u;  // group g's first product: (a = 0, b = g)
#pragma unroll
                        for (int x = 0; x < 2; ++x)  // x = 0: Re t x cos (A), x = 1: Im t x sin (B)
                            umma_i8(tmem + static_cast<uint32_t>((2 * g + x) * kN),
                                    desc_canon(st + (2 * a + x) * kAPlane), desc_canon(sb + (2 * b + x) * kBPlane), acc);
                    }
                    umma_commit(smem_u32(&empty[s]));
                }
                __syncwarp();
            }
            if (elect_one()) umma_commit(smem_u32(acc_full));
            __syncwarp();
            STC_STAMP(5);
        }
    } else {
        // epilogue: warp w drains TMEM lanes 32 (w % 4) .. (frames f0 + 32 (w % 4) + lane). The five int32 groups
        // are combined exactly in int64 (Horner in 128: |group g| <= 5 * 64^2 * m), converted once to fp64, and
        // both mirror cells staged in the (now idle) pipeline smem, [frame][97] doubles per warp, so the rows go
        // out as coalesced runs of cells: q0 .. q0 + 47 and L - q0 - 48 .. L - 1 - q0.
        const int quarter = warp & 3, part = (warp - 2) >> 2;  // lane quarter, column part
        mbar_wait(smem_u32(acc_full), 0);
        tc_fence_after();
        if (warp == 2 && lane == 0) STC_STAMP(3);
        const uint32_t taddr = tmem + (static_cast<uint32_t>(32 * quarter) << 16);
        const int f = f0 + 32 * quarter + lane;
        const bool live = f < frames;
        const double sc = live ? ldexp(2.0 * tscale[f], -42) : 0.0;  // 128^-6 of the Horner value
        const double c0 = live ? static_cast<double>(m) - t[static_cast<size_t>(f) * m].re : 0.0;
        const double floor_v = 1e-12 * static_cast<double>(m);
        double* stg = reinterpret_cast<double*>(smem) + quarter * 32 * kRow;
        constexpr int kCols = kN / kSplit;
        static_assert(kCols % 8 == 0, "column part in chunks of 8");
#pragma unroll 1
        for (int c = part * kCols; c < (part + 1) * kCols; c += 8) {
            uint32_t v[2 * kS][8];
#pragma unroll
            for (int i = 0; i < 2 * kS; ++i) tmem_ld8(taddr + static_cast<uint32_t>(i * kN + c), v[i]);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                long long ha = static_cast<int32_t>(v[0][j]), hb = static_cast<int32_t>(v[1][j]);
#pragma unroll
                for (int g = 1; g < kS; ++g) {
                    ha = ha * 128 + static_cast<int32_t>(v[2 * g][j]);
                    hb = hb * 128 + static_cast<int32_t>(v[2 * g + 1][j]);
                }
                const double a = static_cast<double>(ha) * sc, b = static_cast<double>(hb) * sc;
                stg[lane * kRow + c + j] = __drcp_rn(fmax(c0 - 2.0 * (a - b), floor_v));
                stg[lane * kRow + kN + (kN - 1 - c - j)] = __drcp_rn(fmax(c0 - 2.0 * (a + b), floor_v));
            }
        }
        if (kSplit > 1)
            named_bar_sync(1 + quarter, 32 * kSplit);
        else
            __syncwarp();
        const int nq = half ? L : (L + 1) / 2;  // half: every grid point is a "pair" of its own, mirrors dropped
        const int fw = f0 + 32 * quarter;
        constexpr int kRows = (32 + kSplit - 1) / kSplit;
#pragma unroll 1
        for (int r = part * kRows; r < min(32, (part + 1) * kRows) && fw + r < frames; ++r) {
            const size_t o = static_cast<size_t>(fw + r) * L;
#pragma unroll
            for (int i = lane; i < 2 * kN; i += 32) {
                const int q = i < kN ? q0 + i : q0 + (2 * kN - 1 - i);  // pair of this slot
                if (q >= nq || (half && i >= kN)) continue;
                const int cell = i < kN ? q : L - 1 - q;
                if (i >= kN && cell == q) continue;  // centre cell of an odd grid: written once
                const double P = stg[r * kRow + i];
                if (spec32) spec32[o + cell] = static_cast<float>(P);
                spec64[o + cell] = P;
            }
        }
        if (warp == 2 && lane == 0) STC_STAMP(4);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

}  // namespace spectc
}  // namespace fmk

// Plan-side geometry of the tensor-core spectrum: pairs padded to kN, delta to 32.
// half = 0: mirror-symmetric grid, (L + 1) / 2 pairs (theta_q, -theta_q); half = 1: any grid, all L points as pairs whose
// mirror half is discarded (twice the symmetric work per point, still on the tensor cores)
int fm_spectrum_tc_pairs_pad(int L, int half) {
    return ((half ? L : (L + 1) / 2) + fmk::spectc::kN - 1) / fmk::spectc::kN * fmk::spectc::kN;
}
int fm_spectrum_tc_canon_off(int row, int k) { return fmk::spectc::canon_off(row, k); }
int fm_spectrum_tc_frames_pad(int frames) { return (frames + fmk::spectc::kM - 1) / fmk::spectc::kM * fmk::spectc::kM; }

// zk: the plan's zK table (capi.cu zdig_host_k); tk / tscale: workspace of fm_spectrum_tc_frames_pad(frames) rows
// (x 10 planes x mk bytes, mk = M rounded up to 32) and doubles.
cudaError_t fm_launch_spectrum_tc(const void* t, const int8_t* zk, int8_t* tk, double* tscale, int frames, int m, int L,
                                  float* spec32, double* spec64, cudaStream_t s, int half) {
    using namespace fmk::spectc;
    const int nkb = (m + kK - 1) / kK;
    const int fpad = fm_spectrum_tc_frames_pad(frames), nqp = fm_spectrum_tc_pairs_pad(L, half);
    k_slice_tk<<<fpad, 256, 0, s>>>(static_cast<const fmk::c64*>(t), tk, tscale, frames, m, nkb);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_spectrum_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    const dim3 grid(nqp / kN, fpad / kM);
    k_spectrum_tc<<<grid, kThreads, kSmem, s>>>(tk, zk, tscale, static_cast<const fmk::c64*>(t), frames, m, nkb, L,
                                                spec32, spec64, half);
    return cudaGetLastError();
}
