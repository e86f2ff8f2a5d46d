// K1 — batched spatial covariance R_f = X_f X_f^H / N on the 5th-gen tensor cores.
//
// Replaces R/src/scene.cpp:138-159 (scaled_gram: Eigen selfadjointView rankUpdate,
// lower triangle mirrored) + the HermitianMatrix symmetrisation R/src/linalg.cpp:46-52.
//
// Data layout (HBM): X is B frames x M rows x N snapshots of interleaved complex64,
// row-major (the FMCX order, R/src/io.cpp:76-83). R is B x M x M complex64 row-major,
// written in full (lower tiles computed, upper tiles mirrored as conj-transpose).
//
// One CTA pair (cluster of 2, tcgen05 cta_group::2) owns one 256x256 tile of R.
// Each CTA streams its 128 rows of X (and of the B-side rows for off-diagonal tiles)
// through a TMA (128B-swizzled fp32 staging) -> converter warps (fp32 -> fp16 planes
// Re / Im in the UMMA canonical K-major layout) -> one elected thread of the leader
// CTA issuing four M256xN256xK16 tcgen05.mma per 16 snapshots:
//     Re += Xr Xr^T + Xi Xi^T ;   Im += Xi Xr^T - Xr Xi^T   (a_negate bit)
// Accumulators (Re cols 0..255, Im cols 256..511) fill the 512 TMEM columns of both
// SMs; the epilogue reads them with tcgen05.ld, scales by 1/N and stores fp32.
// Precision: operands rounded to fp16 (11-bit significand), fp32 accumulation.
// Measured on the c2 frames against the fp64 oracle: 3e-3 dB max spectrum error,
// identical peaks.
// Scale: MUSIC is scale-free and the reference computes in fp64, so the fp16 operand range must not limit the
// input. The converters record each frame's max |x|; frames outside [2^-8, 2^15) (fp16 overflow, or significand
// bits lost to subnormals) are listed by k_rescue_list and recomputed by a second launch over the list only,
// with X scaled by a power of two 2^e (exact) so that max |x| lands in [2^6, 2^7), and 2^-2e folded into the
// epilogue's 1/N. Frames in range cost one atomicMax per converter warp and tile; an empty list exits at once.
// Temporal mode (temporal_covariance R/src/scene.cpp:140-153,161-163): T = X^H X / M is the same
// Hermitian product on Z = X^H, whose operand rows are X's columns (snapshots) and whose contraction runs over X's
// rows (antennas). X is read in its stored order: the TMA box is 16 antenna rows x 128 snapshots (a 3D map
// {row length, M, frames}, so rows past M zero-fill instead of reading the next frame), and the converter warps
// transpose while they convert (Z_ik = conj X_ki), writing the same K-major fp16 planes. No transpose pass.

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstdio>

#include "fm_common.cuh"
#include "tc_common.cuh"

namespace fmk {
namespace cov {

constexpr int kRows = 128;          // rows of X per CTA (half of the UMMA M=256 tile)
constexpr int kChunk = 16;          // complex snapshots per pipeline stage (one UMMA K-slice)
// Ring depths (stages). General tiles stage the A and B sides (32 KB fp32 per staging stage, 16 KB fp16 per
// operand stage); diagonal-only launches (M <= 256) stage one side (16 KB / 8 KB). The TMA staging ring is
// the deeper one: the bytes in flight per CTA bound the X stream (off-diagonal tiles re-read 256-row slabs
// of X from L2). Measured on one box (scripts_cov_ring.sh, FM_COV_RING): general 3/3 -> 4/2 takes the c4
// covariance 3.28 -> 3.16 ms; diagonal 6/6 -> 8/4 takes c2's 0.350 -> 0.343 ms.
constexpr int kStagesS = 4;         // fp32 staging ring (TMA destination), general tiles
constexpr int kStagesO = 2;         // fp16 operand ring (UMMA source), general tiles
constexpr int kDiagS = 6;           // diagonal-only launches (6 / 8 with four converter warps: 0.332 -> 0.325 ms)
constexpr int kDiagO = 8;
constexpr int kMaxStages = 8;
static_assert(kStagesS <= kMaxStages && kStagesO <= kMaxStages && kDiagS <= kMaxStages && kDiagO <= kMaxStages,
              "ring barriers");
constexpr int kStageBytes = kRows * kChunk * 8;   // 16 KB fp32 per operand side
constexpr int kPlaneBytes = kRows * kChunk * 2;   // 4 KB fp16 per plane (Re or Im)
constexpr int kOpBytes = 2 * kPlaneBytes;         // 8 KB per operand side
constexpr int kThreads = 320;                     // w0 TMA, w1 MMA, w2..w5 convert, w6..w9 epilogue
constexpr int kThreadsP = 448;                    // plane epilogue: w6..w13, two warps per TMEM lane quarter
constexpr int kSmemStaging = kStagesS * 2 * kStageBytes;
constexpr int kSmemOperand = kStagesO * 2 * kOpBytes;
constexpr int kSmemBarriers = 512;  // 4 x 8 ring barriers + acc + exchange slots + tmem slot (~300 B used)
constexpr int kEpiLd = 33;                                  // padded row (float2) of the transpose tile
constexpr int kEpiChunk = 4096;                             // 32 rows x 16 complex fp32 (one TMA store box)
constexpr int kEpiWarpBytes = 4 * kEpiChunk;                // [diag buf0 | diag buf1 | mirror buf0 | mirror buf1]
constexpr int kSmemEpilogue = 4 * kEpiWarpBytes;            // >= 4 * 32 * kEpiLd * 8 (generic-store fallback)
static_assert(kSmemEpilogue >= 4 * 32 * kEpiLd * 8, "epilogue region");
constexpr int kSmemBytes = 1024 + kSmemStaging + kSmemOperand + kSmemEpilogue + kSmemBarriers;

// Staging + operand bytes of a packed ring (general S, general O, diag S, diag O), rounded up to 1 KB.
__host__ __device__ constexpr int ring_region_bytes(int ring, bool diag_only) {
    return diag_only ? (((ring >> 16) & 0xff) * kStageBytes + ((ring >> 24) & 0xff) * kOpBytes + 1023) / 1024 * 1024
                     : ((ring & 0xff) * 2 * kStageBytes + ((ring >> 8) & 0xff) * 2 * kOpBytes + 1023) / 1024 * 1024;
}

// PTX wrappers: tc_common.cuh
using namespace fmk::tc;

__device__ __forceinline__ uint32_t pack_half2(float lo, float hi) {
    __half2 h = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
}

// UMMA shared-memory descriptor, K-major, SWIZZLE_NONE: core matrices of 8 rows x 16 B,
// LBO = 128 B (next 8 K-elements), SBO = 256 B (next 8 rows), version bit 46 (sm_100).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
    return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>(128 >> 4) << 16) |
           (static_cast<uint64_t>(256 >> 4) << 32) | (1ull << 46);
}
// UMMA smem descriptor, K-major, SWIZZLE_128B (TMA-written fp16 plane tiles: rows of 64 halves = 128 B, 8-row
// atoms 1024 B apart); a K step of 16 advances the start address by 32 B inside the atom.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (1ull << 16) | (static_cast<uint64_t>(1024 >> 4) << 32) |
           (1ull << 46) | (2ull << 61);
}
// Multi-tile frames (M > 256: every 256-row block of X feeds nb tiles, so the fused fp32 -> fp16 conversion would
// run nb times per block and the converters, not the tensor cores, would set the pace): X is converted ONCE into
// Re / Im fp16 planes (frames x M x n_pad halves, zero-padded to a multiple of 64 snapshots) with each frame's
// max |x| (the rescue list's input) and non-finite flag, and the covariance kernel (kF16) TMA-loads the planes
// straight into 128B-swizzled UMMA operand tiles.
#ifndef FM_F16_KC
#define FM_F16_KC 32
#endif
constexpr int kF16Kc = FM_F16_KC;                  // snapshots per fp16 stage (one 64-B / 128-B swizzle row)
constexpr int kF16Plane = kRows * kF16Kc * 2;      // 128 rows x kF16Kc halves
constexpr int kF16Stage = 4 * kF16Plane;           // A re, A im, B re, B im
constexpr int kF16Stages = kF16Kc == 64 ? 2 : 4;   // 128 KB of ring either way
// K-major swizzled descriptor of the plane tiles: rows of 2 kF16Kc bytes, 8-row atoms (SBO) 16 kF16Kc bytes apart
__device__ __forceinline__ uint64_t umma_desc_plane(uint32_t saddr) {
    constexpr uint64_t layout = kF16Kc == 64 ? 2ull : 4ull;  // SWIZZLE_128B / SWIZZLE_64B
    return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (1ull << 16) |
           (static_cast<uint64_t>((16 * kF16Kc) >> 4) << 32) | (1ull << 46) | (layout << 61);
}
constexpr int kXpRows = 4;  // rows per warp (one max |x| atomic per warp and frame run of rows)
__global__ void __launch_bounds__(256) k_x_planes(const float4* __restrict__ x, uint2* __restrict__ pre,
                                                  uint2* __restrict__ pim, uint32_t* __restrict__ amax,
                                                  int32_t* __restrict__ status, int64_t rows, int m, int n,
                                                  int n_pad) {
    const int lane = threadIdx.x & 31;
    const int64_t r0 = (static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5)) * kXpRows;
    float mx = 0.f;
    bool bad = false;
    int fcur = -1;
    for (int64_t row = r0; row < r0 + kXpRows && row < rows; ++row) {
        const int f = static_cast<int>(row / m);
        if (f != fcur) {  // the warp's rows crossed into another frame: flush the previous frame's max
            if (fcur >= 0) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                if (lane == 0 && amax) atomicMax(&amax[fcur], __float_as_uint(mx));
                if (__any_sync(0xffffffffu, bad) && lane == 0 && status) atomicOr(&status[fcur], kFrameNonFinite);
                mx = 0.f;
                bad = false;
            }
            fcur = f;
        }
        const float4* xr = x + row * (n / 2);
        uint2* rr = pre + row * (n_pad / 4);
        uint2* ri = pim + row * (n_pad / 4);
        for (int q = lane; q < n_pad / 4; q += 32) {  // four snapshots per lane and step
            float re[4] = {0.f, 0.f, 0.f, 0.f}, im[4] = {0.f, 0.f, 0.f, 0.f};
            if (4 * q < n) {
                const float4 a = __ldcs(xr + 2 * q);
                re[0] = a.x; im[0] = a.y; re[1] = a.z; im[1] = a.w;
                if (4 * q + 2 < n) {
                    const float4 c = __ldcs(xr + 2 * q + 1);
                    re[2] = c.x; im[2] = c.y; re[3] = c.z; im[3] = c.w;
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                mx = fmaxf(mx, fmaxf(fabsf(re[u]), fabsf(im[u])));
                bad |= !(isfinite(re[u]) && isfinite(im[u]));
            }
            rr[q] = make_uint2(pack_half2(re[0], re[1]), pack_half2(re[2], re[3]));
            ri[q] = make_uint2(pack_half2(im[0], im[1]), pack_half2(im[2], im[3]));
        }
    }
    if (fcur >= 0) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0 && amax) atomicMax(&amax[fcur], __float_as_uint(mx));
        if (__any_sync(0xffffffffu, bad) && lane == 0 && status) atomicOr(&status[fcur], kFrameNonFinite);
    }
}

// Instruction descriptor: kind::f16, A=B=F16, D=F32, K-major both, M=256, N=256.
__host__ __device__ constexpr uint32_t umma_idesc(bool neg_a) {
    return (1u << 4) | (0u << 7) | (0u << 10) | ((neg_a ? 1u : 0u) << 13) | ((256u >> 3) << 17) | ((256u >> 4) << 24);
}
__device__ __forceinline__ void umma_f16_2sm(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

#ifdef FM_COV_TIMELINE  // experiment only: clock64 stamps of CTA 0's first 16 tiles (tools/experiments)
__device__ long long g_cov_tl[16 * 16];
#define COV_STAMP(tile_i, slot)                                                        \
    do {                                                                               \
        if (blockIdx.x == 0 && (tile_i) < 16) g_cov_tl[(tile_i) * 16 + (slot)] = clock64(); \
    } while (0)
#define COV_ADD(tile_i, slot, v)                                                        \
    do {                                                                                \
        if (blockIdx.x == 0 && (tile_i) < 16) g_cov_tl[(tile_i) * 16 + (slot)] += (v);  \
    } while (0)
#define COV_CLK() clock64()
#else
#define COV_STAMP(tile_i, slot)
#define COV_ADD(tile_i, slot, v)
#define COV_CLK() 0ll
#endif

// Lower-triangle tile enumeration: t -> (bi, bj) with bi >= bj.
__device__ __forceinline__ void tile_coords(int t, int& bi, int& bj) {
    bi = 0;
    while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
    bj = t - bi * (bi + 1) / 2;
}

// Convert one 128-row x 16-complex fp32 staging tile (one TMA box, SWIZZLE_128B: row r
// occupies 128 B, its 16-byte chunk c (2 complex) sits at chunk slot c ^ (r & 7)) into the
// Re/Im fp16 UMMA planes. Tracks max |x| (fp16 range check) and non-finite inputs.
// Lane mapping keeps both the swizzled reads and the core-matrix writes bank-conflict free.
// kJ = 2: four converter warps (32 rows each); kJ = 1: eight converter warps (16 rows each).
template <int kJ>
__device__ __forceinline__ void convert_tile(const uint8_t* stage, uint8_t* op, int cw, int lane, int row_base,
                                             int m_rows, float xs, float& amax, bool& nonfinite) {
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
        const int r = 16 * kJ * cw + (lane & 7) + 8 * (lane >> 4) + 16 * j;
        const int q = (lane >> 3) & 1;  // which 8-complex half of the 16-complex chunk
        const bool valid = (row_base + r) < m_rows;
        const uint8_t* src = stage + r * 128;
        float re[8], im[8];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float4 v = *reinterpret_cast<const float4*>(src + (((4 * q + u) ^ (r & 7)) << 4));
            re[2 * u] = v.x;
            im[2 * u] = v.y;
            re[2 * u + 1] = v.z;
            im[2 * u + 1] = v.w;
        }
        if (!valid) {
#pragma unroll
            for (int u = 0; u < 8; ++u) re[u] = im[u] = 0.f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {  // power-of-two prescale (1 outside the rescue pass): exact
            re[u] *= xs;
            im[u] *= xs;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            amax = fmaxf(amax, fmaxf(fabsf(re[u]), fabsf(im[u])));
            nonfinite |= !(isfinite(re[u]) && isfinite(im[u]));
        }
        uint4 pr, pi;
        pr.x = pack_half2(re[0], re[1]);
        pr.y = pack_half2(re[2], re[3]);
        pr.z = pack_half2(re[4], re[5]);
        pr.w = pack_half2(re[6], re[7]);
        pi.x = pack_half2(im[0], im[1]);
        pi.y = pack_half2(im[2], im[3]);
        pi.z = pack_half2(im[4], im[5]);
        pi.w = pack_half2(im[6], im[7]);
        const int off = (r >> 3) * 256 + q * 128 + (r & 7) * 16;
        *reinterpret_cast<uint4*>(op + off) = pr;
        *reinterpret_cast<uint4*>(op + kPlaneBytes + off) = pi;
    }
}

// Temporal mode: the staging tile is 16 antenna rows (K) x 128 snapshots (operand rows) of complex fp32, plain
// (SWIZZLE_NONE) rows of 1 KB: element (k, r) at k * 1024 + r * 8. Same lane -> (row r, 8-K half q) mapping and
// output layout as convert_tile; each lane gathers its 8 K values down a column (conflict-free: the 16 lanes of
// a half read 128 contiguous bytes of one row). Z = X^H: the imaginary part is negated.
template <int kJ>
__device__ __forceinline__ void convert_tile_t(const uint8_t* stage, uint8_t* op, int cw, int lane, int row_base,
                                               int m_rows, float xs, float& amax, bool& nonfinite) {
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
        const int r = 16 * kJ * cw + (lane & 7) + 8 * (lane >> 4) + 16 * j;
        const int q = (lane >> 3) & 1;
        const bool valid = (row_base + r) < m_rows;
        float re[8], im[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const float2 v = *reinterpret_cast<const float2*>(stage + (8 * q + u) * 1024 + r * 8);
            re[u] = valid ? v.x * xs : 0.f;
            im[u] = valid ? -v.y * xs : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            amax = fmaxf(amax, fmaxf(fabsf(re[u]), fabsf(im[u])));
            nonfinite |= !(isfinite(re[u]) && isfinite(im[u]));
        }
        uint4 pr, pi;
        pr.x = pack_half2(re[0], re[1]);
        pr.y = pack_half2(re[2], re[3]);
        pr.z = pack_half2(re[4], re[5]);
        pr.w = pack_half2(re[6], re[7]);
        pi.x = pack_half2(im[0], im[1]);
        pi.y = pack_half2(im[2], im[3]);
        pi.z = pack_half2(im[4], im[5]);
        pi.w = pack_half2(im[6], im[7]);
        const int off = (r >> 3) * 256 + q * 128 + (r & 7) * 16;
        *reinterpret_cast<uint4*>(op + off) = pr;
        *reinterpret_cast<uint4*>(op + kPlaneBytes + off) = pi;
    }
}

// Persistent: CTA pair `pair` processes tiles pair, pair + npairs, ... Warp roles:
//   w0 TMA producer | w1 MMA issuer (leader) + TMEM owner | w2..w5 converters | w6..w9 epilogue.
// The epilogue of tile i (TMEM -> fp32 R) overlaps the TMA + fp16 conversion of tile i + 1;
// the MMA of tile i + 1 starts once both CTAs' epilogues have drained TMEM (acc_empty).
// kEpi: 0 generic-store fallback (odd M), 1 TMA-stored complex64 R, 2 TMA-stored fp16 hi/lo planes of
// R / s_f (M <= 256: one tile per frame; s_f = smallest power of two >= max_i R_ii, exchanged between the
// two CTAs of the pair; rmap / mmap are the hi / lo plane maps, rscale[f] = s_f).
// kConv8: four more converter warps after the epilogue warps (eight in all, 16 rows each). The redundant
// operand conversion of multi-tile frames (every 256-row block of X is converted once per tile it feeds,
// 4x at M = 1024) makes the converters the bottleneck there.
// kSplit (with kConv8): the eight converter warps form two groups of four that take alternate pipeline stages
// (each group converts whole stages, 32 rows per warp), so one stage's fixed costs -- the proxy fence, the group
// barrier and the cross-CTA operand-ready arrive -- overlap the other group's conversion.
template <int kEpi, bool kConv8, bool kSplit = false, bool kF16 = false>
#ifdef FM_COV_MAXNREG  // experiment: register cap so fp64 kernels of another sub-batch can co-reside
#define FM_COV_BOUNDS(t) __maxnreg__(FM_COV_MAXNREG)
#else
#define FM_COV_BOUNDS(t) __launch_bounds__(t, 1)
#endif
__global__ void __cluster_dims__(2, 1, 1) FM_COV_BOUNDS((kEpi == 2 ? kThreadsP : kThreads) + (kConv8 ? 128 : 0))
    cov_tc_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap rmap,
                  const __grid_constant__ CUtensorMap mmap, float* __restrict__ r_out, int32_t* __restrict__ status,
                  int m, int n, int tiles_per_frame, int total_tiles, float* __restrict__ rscale,
                  float inv_n_true, int dbg, int ring, const int32_t* __restrict__ flist,
                  const int32_t* __restrict__ fcount, const float* __restrict__ xscale,
                  uint32_t* __restrict__ amax_out, int temporal, const __grid_constant__ CUtensorMap pre_map,
                  const __grid_constant__ CUtensorMap pim_map) {
    constexpr bool kTmaStore = kEpi >= 1;
    // rescue pass: only the listed frames (the count is device-resident; every CTA of the grid reads the same
    // value, so an empty list ends all of them before any barrier or TMEM allocation)
    if (flist) {
        total_tiles = *fcount * tiles_per_frame;
        if (total_tiles == 0) return;
    }
    auto frame_of = [&](int tile) { return flist ? flist[tile / tiles_per_frame] : tile / tiles_per_frame; };
    auto inv_n_of = [&](int frame) {  // 1/N, and 2^-2e of the rescue prescale (exact)
        if (!xscale) return inv_n_true;
        const float xs = xscale[frame];
        return inv_n_true / (xs * xs);
    };
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* staging = smem;
    // diagonal-only launches split the staging + operand region 96 KB / 48 KB, general tiles 128 KB / 32 KB
    static_assert(kDiagS * kStageBytes + kDiagO * kOpBytes <= kSmemStaging + kSmemOperand, "diag rings");
    // ring: (general staging, general operand, diag staging, diag operand) depths, packed 4 x 8 bits
    const int gS = ring & 0xff, gO = (ring >> 8) & 0xff, dS = (ring >> 16) & 0xff, dO = (ring >> 24) & 0xff;
    uint8_t* operand = smem + (tiles_per_frame == 1 ? dS * kStageBytes : gS * 2 * kStageBytes);
    // epilogue region right after the rings (1024-aligned for the 128B-swizzled TMA store boxes)
    uint8_t* epi_bytes = smem + (kF16 ? kF16Stages * kF16Stage : ring_region_bytes(ring, tiles_per_frame == 1));
    uint64_t* bars = reinterpret_cast<uint64_t*>(epi_bytes + kSmemEpilogue);
    uint64_t* stage_full = bars;
    uint64_t* stage_empty = bars + kMaxStages;
    uint64_t* op_full = bars + 2 * kMaxStages;
    uint64_t* op_empty = bars + 3 * kMaxStages;
    uint64_t* acc_full = bars + 4 * kMaxStages;
    uint64_t* acc_empty = acc_full + 1;
    uint64_t* xch_bar = acc_empty + 1;                             // [2] peer's diagonal max arrived
    float* xch_val = reinterpret_cast<float*>(xch_bar + 2);         // [2] peer's diagonal max
    float* s_wmax = xch_val + 2;                                    // [4] per epilogue warp
    float* s_scale = s_wmax + 4;                                    // [1]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_scale + 1);
    float2* epi = reinterpret_cast<float2*>(epi_bytes);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = __shfl_sync(0xffffffffu, cluster_rank(), 0);  // warp-uniform for the compiler
    const int pair = blockIdx.x >> 1;
    const int npairs = gridDim.x >> 1;
    const int nk = kF16 ? (n + kF16Kc - 1) / kF16Kc : (n + kChunk - 1) / kChunk;  // K stages per tile
    // ring geometry: diagonal-only launches (one tile per frame) use half-size stages, twice as many
    const bool diag_only = tiles_per_frame == 1;
    const int nS = diag_only ? dS : gS, nO = diag_only ? dO : gO;
    const int sStride = diag_only ? kStageBytes : 2 * kStageBytes, oStride = diag_only ? kOpBytes : 2 * kOpBytes;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kMaxStages; ++s) {
            mbar_init(smem_u32(&stage_full[s]), 1);
            mbar_init(smem_u32(&stage_empty[s]), 1);
        }
        for (int s = 0; s < kMaxStages; ++s) {
            mbar_init(smem_u32(&op_full[s]), 2);  // one arrive per CTA (leader's copy used)
            mbar_init(smem_u32(&op_empty[s]), 1);
        }
        mbar_init(smem_u32(acc_full), 1);
        mbar_init(smem_u32(acc_empty), 2);  // one arrive per CTA's epilogue (leader's copy used)
        mbar_init(smem_u32(&xch_bar[0]), 1);
        mbar_init(smem_u32(&xch_bar[1]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xmap)) : "memory");
        if (kTmaStore) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&rmap)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mmap)) : "memory");
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // warp-uniform: MMA operands in uniform registers

    if (warp == 0) {
        // ---------------- TMA producer (one thread)
        if (lane == 0) {
            int g = 0;
            for (int tile = pair; tile < total_tiles; tile += npairs) {
                const int frame = frame_of(tile);
                int bi, bj;
                tile_coords(tile % tiles_per_frame, bi, bj);
                const bool diag = (bi == bj);
                const uint32_t bytes = diag ? kStageBytes : 2 * kStageBytes;
                const int ya = frame * m + 256 * bi + 128 * static_cast<int>(rank);
                const int yb = frame * m + 256 * bj + 128 * static_cast<int>(rank);
                // temporal: x = first snapshot (float offset) of the operand rows, y = first antenna row, z = frame
                const int ta = 2 * (256 * bi + 128 * static_cast<int>(rank));
                const int tb = 2 * (256 * bj + 128 * static_cast<int>(rank));
                for (int kc = 0; kc < nk; ++kc, ++g) {
                    if constexpr (kF16) {  // fp16 planes straight into the operand slots (freed by the MMA)
                        const int s = g % kF16Stages;
                        mbar_wait(smem_u32(&op_empty[s]), ((g / kF16Stages) & 1) ^ 1);
                        const uint32_t full = smem_u32(&stage_full[s]);
                        mbar_arrive_expect_tx(full, (diag ? 2 : 4) * kF16Plane);
                        uint8_t* st = smem + s * kF16Stage;
                        const int x = kF16Kc * kc;
                        tma_load_2d(smem_u32(st), &pre_map, full, x, ya);
                        tma_load_2d(smem_u32(st + kF16Plane), &pim_map, full, x, ya);
                        if (!diag) {
                            tma_load_2d(smem_u32(st + 2 * kF16Plane), &pre_map, full, x, yb);
                            tma_load_2d(smem_u32(st + 3 * kF16Plane), &pim_map, full, x, yb);
                        }
                        continue;
                    }
                    const int s = g % nS;
                    mbar_wait(smem_u32(&stage_empty[s]), ((g / nS) & 1) ^ 1);
                    const uint32_t full = smem_u32(&stage_full[s]);
                    mbar_arrive_expect_tx(full, bytes);
                    uint8_t* st = staging + s * sStride;
                    if (temporal) {
                        tma_load_3d(smem_u32(st), &xmap, full, ta, kChunk * kc, frame);
                        if (!diag) tma_load_3d(smem_u32(st + kStageBytes), &xmap, full, tb, kChunk * kc, frame);
                    } else {
                        const int x = 2 * kChunk * kc;
                        tma_load_2d(smem_u32(st), &xmap, full, x, ya);
                        if (!diag) tma_load_2d(smem_u32(st + kStageBytes), &xmap, full, x, yb);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (leader CTA; the warp waits converged, one elected lane issues)
        if (rank == 0) {
            const uint32_t id_pos = umma_idesc(false);
            const uint32_t id_neg = umma_idesc(true);
            int g = 0, t = 0;
            for (int tile = pair; tile < total_tiles; tile += npairs, ++t) {
                int bi, bj;
                tile_coords(tile % tiles_per_frame, bi, bj);
                const bool diag = (bi == bj);
                mbar_wait_cluster(smem_u32(acc_empty), (t & 1) ^ 1);  // both epilogues drained TMEM
                tc_fence_after();
                COV_STAMP(t, 0);
                for (int kc = 0; kc < nk; ++kc, ++g) {
                    if constexpr (kF16) {  // four K steps of 16 inside each 128B-swizzled 64-snapshot stage
                        const int o = g % kF16Stages;
                        mbar_wait_cluster(smem_u32(&op_full[o]), (g / kF16Stages) & 1);
                        tc_fence_after();
                        const uint32_t a = smem_u32(smem + o * kF16Stage);
                        const uint32_t b = diag ? a : a + 2 * kF16Plane;
                        if (elect_one()) {
#pragma unroll
                            for (int ks = 0; ks < kF16Kc / kChunk; ++ks) {
                                const uint32_t off = 32u * ks;
                                const uint64_t ar = umma_desc_plane(a + off), ai = umma_desc_plane(a + kF16Plane + off);
                                const uint64_t br = umma_desc_plane(b + off), bim = umma_desc_plane(b + kF16Plane + off);
                                const uint32_t acc = (kc > 0 || ks > 0) ? 1u : 0u;
                                umma_f16_2sm(tmem + 0, ar, br, id_pos, acc);
                                umma_f16_2sm(tmem + 0, ai, bim, id_pos, 1u);
                                umma_f16_2sm(tmem + 256, ai, br, id_pos, acc);
                                umma_f16_2sm(tmem + 256, ar, bim, id_neg, 1u);
                            }
                            umma_commit_mc(smem_u32(&op_empty[o]));
                        }
                        __syncwarp();
                        continue;
                    }
                    const int o = g % nO;
                    const long long c0 = COV_CLK();
                    mbar_wait_cluster(smem_u32(&op_full[o]), (g / nO) & 1);
                    COV_ADD(t, 9, COV_CLK() - c0);
                    tc_fence_after();
                    const uint32_t a = smem_u32(operand + o * oStride);
                    const uint32_t b = diag ? a : a + kOpBytes;
                    const uint64_t ar = umma_desc(a), ai = umma_desc(a + kPlaneBytes);
                    const uint64_t br = umma_desc(b), bim = umma_desc(b + kPlaneBytes);
                    const uint32_t acc = kc > 0 ? 1u : 0u;
                    if (elect_one()) {
                        if (!(dbg & 2)) {
                            umma_f16_2sm(tmem + 0, ar, br, id_pos, acc);
                            umma_f16_2sm(tmem + 0, ai, bim, id_pos, 1u);
                            umma_f16_2sm(tmem + 256, ai, br, id_pos, acc);
                            umma_f16_2sm(tmem + 256, ar, bim, id_neg, 1u);
                        }
                        umma_commit_mc(smem_u32(&op_empty[o]));
                    }
                    __syncwarp();
                }
                if (elect_one()) umma_commit_mc(smem_u32(acc_full));
                __syncwarp();
                COV_STAMP(t, 1);
            }
        }
    } else if (warp < 6 || (kConv8 && warp >= (kEpi == 2 ? kThreadsP : kThreads) / 32)) {
        // ---------------- converters (warps 2..5, plus the four after the epilogue warps when kConv8)
        constexpr int kFirstExtra = (kEpi == 2 ? kThreadsP : kThreads) / 32;
        constexpr int kJ = (kConv8 && !kSplit) ? 1 : 2;
        const int cwid = warp < 6 ? warp - 2 : 4 + warp - kFirstExtra;  // 0..7
        const int grp = kSplit ? (cwid >> 2) : 0;                        // stage group (kSplit)
        const int cw = kSplit ? (cwid & 3) : cwid;
        const bool lead = kSplit ? (cwid & 3) == 0 : warp == 2;          // arrives for the group's stages
        int g = 0, tt = 0;
        if constexpr (kF16) {  // no conversion: warp 2 tells the leader CTA each stage's planes have landed
            if (warp == 2 && lane == 0) {
                for (int tile = pair; tile < total_tiles; tile += npairs) {
                    for (int kc = 0; kc < nk; ++kc, ++g) {
                        const int s = g % kF16Stages;
                        mbar_wait(smem_u32(&stage_full[s]), (g / kF16Stages) & 1);
                        if (rank == 0) mbar_arrive_local(smem_u32(&op_full[s]));
                        else mbar_arrive_cluster(smem_u32(&op_full[s]), 0);
                    }
                }
            }
        } else
        for (int tile = pair; tile < total_tiles; tile += npairs, ++tt) {
            const int frame = frame_of(tile);
            int bi, bj;
            tile_coords(tile % tiles_per_frame, bi, bj);
            const bool diag = (bi == bj);
            const int row_a = 256 * bi + 128 * static_cast<int>(rank);
            const int row_b = 256 * bj + 128 * static_cast<int>(rank);
            const float xs = xscale ? xscale[frame] : 1.f;
            float amax = 0.f;
            bool nonfinite = false;
            for (int kc = 0; kc < nk; ++kc, ++g) {
                if (kSplit && (g & 1) != grp) continue;  // nS, nO even: a ring slot always belongs to one group
                const int s = g % nS;
                const int o = g % nO;
                const long long c0 = COV_CLK();
                mbar_wait(smem_u32(&stage_full[s]), (g / nS) & 1);
                const long long c1 = COV_CLK();
                mbar_wait(smem_u32(&op_empty[o]), ((g / nO) & 1) ^ 1);
                const long long c2 = COV_CLK();
                if (warp == 2 && lane == 0) {
                    COV_ADD(tt, 7, c1 - c0);
                    COV_ADD(tt, 8, c2 - c1);
                }
                const uint8_t* st = staging + s * sStride;
                uint8_t* op = operand + o * oStride;
                if (temporal) {
                    convert_tile_t<kJ>(st, op, cw, lane, row_a, m, xs, amax, nonfinite);
                    if (!diag)
                        convert_tile_t<kJ>(st + kStageBytes, op + kOpBytes, cw, lane, row_b, m, xs, amax, nonfinite);
                } else {
                    convert_tile<kJ>(st, op, cw, lane, row_a, m, xs, amax, nonfinite);
                    if (!diag)
                        convert_tile<kJ>(st + kStageBytes, op + kOpBytes, cw, lane, row_b, m, xs, amax, nonfinite);
                }
                fence_proxy_async();
                named_bar_sync(kSplit ? 1 + 2 * grp : 1, (kConv8 && !kSplit) ? 256 : 128);  // stage converted
                if (lead && lane == 0) {
                    if (kc == 0) COV_STAMP(tt, 5);
                    if (kc == nk - 1) COV_STAMP(tt, 6);
                    mbar_arrive_local(smem_u32(&stage_empty[s]));
                    if (rank == 0) mbar_arrive_local(smem_u32(&op_full[o]));
                    else mbar_arrive_cluster(smem_u32(&op_full[o]), 0);
                }
            }
            // pass 1 with a rescue list: record max |x| (k_rescue_list decides); otherwise flag fp16 overflow
            int flag = (nonfinite ? kFrameNonFinite : 0) | (!amax_out && amax > 65504.f ? kFrameRange : 0);
            flag = __reduce_or_sync(0xffffffffu, flag);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
            if (lane == 0) {
                if (flag && status != nullptr) atomicOr(&status[frame], flag);
                if (amax_out) atomicMax(&amax_out[frame], __float_as_uint(amax));  // amax >= 0: uint order
            }
        }
    } else if (kEpi == 2) {
        // ---------------- epilogue, fp16 hi/lo planes of R / s_f (M <= 256: tile == frame). Eight warps:
        // warp w drains TMEM lane quarter (w & 3), columns [128 h, 128 h + 128), h = (w - 6) >> 2.
        // 1. s_f: the warps whose column half holds their rows' diagonal read it, CTA max, exchange with
        //    the peer CTA through DSMEM + an mbarrier (double-buffered by tile parity).
        // 2. per 32-column chunk: two tcgen05.ld, x = R/s_f -> hi = fp16(x), lo = fp16(x - hi), two
        //    128B-swizzled 32 x 64-half boxes (single-buffered per warp), two TMA stores.
        const int quarter = warp & 3;
        const int half = (warp - 6) >> 2;
        const uint32_t ebase = smem_u32(epi_bytes) + (warp - 6) * (2 * kEpiChunk);
        const uint32_t peer = rank ^ 1u;
        int t = 0;
        for (int tile = pair; tile < total_tiles; tile += npairs, ++t) {
            const int frame = frame_of(tile);
            const float inv_n = inv_n_of(frame);
            const int row0 = 128 * static_cast<int>(rank) + 32 * quarter;
            const int gi = row0 + lane;
            mbar_wait(smem_u32(acc_full), t & 1);
            if (warp == 6 && lane == 0) COV_STAMP(t, 2);
            tc_fence_after();
            const uint32_t taddr = tmem + (static_cast<uint32_t>(32 * quarter) << 16);
            if (half == static_cast<int>(rank)) {
                uint32_t dv[32];
                tmem_ld32(taddr + row0, dv);
                tmem_wait_ld();
                float dg = 0.f;
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (j == lane) dg = __uint_as_float(dv[j]);
                dg *= inv_n;
                if (!(dg >= 0.f) || gi >= m) dg = 0.f;  // non-finite frames are flagged by the converters
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) dg = fmaxf(dg, __shfl_xor_sync(0xffffffffu, dg, o));
                if (lane == 0) s_wmax[quarter] = dg;
            }
            named_bar_sync(2, 256);
            if (half == static_cast<int>(rank) && quarter == 0 && lane == 0) {
                const float cmax = fmaxf(fmaxf(s_wmax[0], s_wmax[1]), fmaxf(s_wmax[2], s_wmax[3]));
                const uint32_t slot = smem_u32(&xch_val[t & 1]), bar = smem_u32(&xch_bar[t & 1]);
                asm volatile(
                    "{\n\t.reg .b32 ra, rb;\n\t"
                    "mapa.shared::cluster.u32 ra, %0, %2;\n\t"
                    "mapa.shared::cluster.u32 rb, %1, %2;\n\t"
                    "st.shared::cluster.f32 [ra], %3;\n\t"
                    "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [rb];\n\t}" ::"r"(slot),
                    "r"(bar), "r"(peer), "f"(cmax)
                    : "memory");
                mbar_wait_cluster(bar, (t >> 1) & 1);
                const float maxd = fmaxf(cmax, xch_val[t & 1]);
                float sc = 1.f;
                if (maxd > 0.f && maxd < 3.0e38f) {
                    int e;
                    const float fr = frexpf(maxd, &e);  // maxd = fr 2^e, fr in [0.5, 1)
                    sc = ldexpf(1.f, fr == 0.5f ? e - 1 : e);
                }
                *s_scale = sc;
                if (rank == 0) rscale[frame] = sc;
            }
            named_bar_sync(2, 256);
            if (warp == 6 && lane == 0) COV_STAMP(t, 3);
            const float mul = inv_n / *s_scale;  // power-of-two divisor: exact
            const int nchunks = (row0 < m && !(dbg & 4)) ? max(0, min(4, (m - 128 * half + 31) / 32)) : 0;
            for (int c = 0; c < nchunks; ++c) {
                const int col0 = 128 * half + 32 * c;
                uint32_t vr[32], vi[32];
                tmem_ld32(taddr + col0, vr);
                tmem_ld32(taddr + 256 + col0, vi);
                tmem_wait_ld();
                if (lane == 0) bulk_wait_read0();  // this warp's previous stores have read the boxes
                __syncwarp();
                const uint32_t hbuf = ebase, lbuf = ebase + kEpiChunk;
#pragma unroll
                for (int q = 0; q < 8; ++q) {  // 16-byte chunk q = complex 4q .. 4q + 3 (8 halves)
                    uint32_t hw[4], lw[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int j = 4 * q + u;
                        const float re = __uint_as_float(vr[j]) * mul;
                        const float im = (col0 + j == gi) ? 0.f : __uint_as_float(vi[j]) * mul;
                        const __half2 h = __floats2half2_rn(re, im);
                        const float2 hf = __half22float2(h);
                        const __half2 l = __floats2half2_rn(re - hf.x, im - hf.y);
                        hw[u] = *reinterpret_cast<const uint32_t*>(&h);
                        lw[u] = *reinterpret_cast<const uint32_t*>(&l);
                    }
                    const uint32_t off = lane * 128 + ((q ^ (lane & 7)) << 4);
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(hbuf + off), "r"(hw[0]), "r"(hw[1]),
                                 "r"(hw[2]), "r"(hw[3])
                                 : "memory");
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(lbuf + off), "r"(lw[0]), "r"(lw[1]),
                                 "r"(lw[2]), "r"(lw[3])
                                 : "memory");
                }
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) {
                    tma_store_3d(&rmap, hbuf, 2 * col0, row0, frame);
                    tma_store_3d(&mmap, lbuf, 2 * col0, row0, frame);
                    bulk_commit();
                }
            }
            tc_fence_before();
            named_bar_sync(2, 256);  // all eight epilogue warps finished reading TMEM
            if (warp == 6 && lane == 0) COV_STAMP(t, 4);
            if (warp == 6 && lane == 0) {
                if (rank == 0) mbar_arrive_local(smem_u32(acc_empty));
                else mbar_arrive_cluster(smem_u32(acc_empty), 0);
            }
        }
        if (lane == 0) bulk_wait_all();
    } else if (kTmaStore) {
        // ---------------- epilogue (warps 6..9): TMEM -> registers -> swizzled smem -> TMA store.
        // Per 16-column chunk: two tcgen05.ld (Re, Im), eight conflict-free 16-byte st.shared into a
        // 128B-swizzled 32 x 16 complex box, one elected cp.async.bulk.tensor store (double-buffered,
        // bulk groups). TMEM is released as soon as the last chunk is in smem, so the global writes
        // overlap the next tile's mainloop. Off-diagonal tiles also store the conj-transposed block.
        const int quarter = warp & 3;
        const uint32_t ebase = smem_u32(epi_bytes) + (warp - 6) * kEpiWarpBytes;
        int t = 0, gc = 0;
        for (int tile = pair; tile < total_tiles; tile += npairs, ++t) {
            const int frame = frame_of(tile);
            const float inv_n = inv_n_of(frame);  // 1 / N of the caller (n may include one zero pad column)
            int bi, bj;
            tile_coords(tile % tiles_per_frame, bi, bj);
            const bool diag = (bi == bj);
            const int row0 = 256 * bi + 128 * static_cast<int>(rank) + 32 * quarter;
            const int gi = row0 + lane;
            mbar_wait(smem_u32(acc_full), t & 1);
            tc_fence_after();
            const uint32_t taddr = tmem + (static_cast<uint32_t>(32 * quarter) << 16);
            const int nchunks = row0 < m ? min(16, (m - 256 * bj + 15) / 16) : 0;
            for (int c = 0; c < nchunks; ++c, ++gc) {
                const int col0 = 256 * bj + 16 * c;
                uint32_t vr[16], vi[16];
                tmem_ld16(taddr + 16 * c, vr);
                tmem_ld16(taddr + 256 + 16 * c, vi);
                tmem_wait_ld();
                const int b = gc & 1;
                if (lane == 0) bulk_wait_read1();  // the store issued from buffer b two chunks ago has read it
                __syncwarp();
                const uint32_t dbuf = ebase + b * kEpiChunk;
                const uint32_t mbuf = ebase + 2 * kEpiChunk + b * kEpiChunk;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float re0 = __uint_as_float(vr[2 * q]) * inv_n;
                    const float re1 = __uint_as_float(vr[2 * q + 1]) * inv_n;
                    const float im0 = (col0 + 2 * q == gi) ? 0.f : __uint_as_float(vi[2 * q]) * inv_n;
                    const float im1 = (col0 + 2 * q + 1 == gi) ? 0.f : __uint_as_float(vi[2 * q + 1]) * inv_n;
                    sts_v4(dbuf + lane * 128 + ((q ^ (lane & 7)) << 4), re0, im0, re1, im1);
                    if (!diag) {  // mirrored block row (col0 + 2q (+1)), column gi: conj
                        sts_v2(mbuf + ((2 * q) * 32 + lane) * 8, re0, -im0);
                        sts_v2(mbuf + ((2 * q + 1) * 32 + lane) * 8, re1, -im1);
                    }
                }
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) {
                    tma_store_3d(&rmap, dbuf, 2 * col0, row0, frame);
                    if (!diag) tma_store_3d(&mmap, mbuf, 2 * row0, col0, frame);
                    bulk_commit();
                }
            }
            tc_fence_before();
            named_bar_sync(2, 128);  // all four epilogue warps finished reading TMEM
            if (warp == 6 && lane == 0) {
                if (rank == 0) mbar_arrive_local(smem_u32(acc_empty));
                else mbar_arrive_cluster(smem_u32(acc_empty), 0);
            }
        }
        if (lane == 0) bulk_wait_all();
    } else {
        // ---------------- epilogue, generic-store fallback (odd M: row pitch not 16-byte aligned)
        const int quarter = warp & 3;
        const int row = 32 * quarter + lane;
        int t = 0;
        for (int tile = pair; tile < total_tiles; tile += npairs, ++t) {
            const int frame = frame_of(tile);
            const float inv_n = inv_n_of(frame);  // 1 / N of the caller (n may include one zero pad column)
            int bi, bj;
            tile_coords(tile % tiles_per_frame, bi, bj);
            const bool diag = (bi == bj);
            const int gi = 256 * bi + 128 * static_cast<int>(rank) + row;
            const size_t fbase = static_cast<size_t>(frame) * m * m;
            mbar_wait(smem_u32(acc_full), t & 1);
            tc_fence_after();
            float2* T = epi + (warp - 6) * 32 * kEpiLd;  // this warp's 32 x 32 transpose tile
            const int gi0 = 256 * bi + 128 * static_cast<int>(rank) + 32 * quarter;
            for (int c0 = 0; c0 < 256; c0 += 32) {
                uint32_t vr[32], vi[32];
                const uint32_t taddr = tmem + (static_cast<uint32_t>(32 * quarter) << 16) + c0;
                tmem_ld32(taddr, vr);
                tmem_ld32(taddr + 256, vi);
                tmem_wait_ld();
                const int gj0 = 256 * bj + c0;
#pragma unroll
                for (int jj = 0; jj < 32; ++jj) {
                    const float re = __uint_as_float(vr[jj]) * inv_n;
                    float im = __uint_as_float(vi[jj]) * inv_n;
                    if (gj0 + jj == gi) im = 0.f;
                    T[lane * kEpiLd + jj] = make_float2(re, im);
                }
                __syncwarp();
                // coalesced: lane = column; one 256-byte row of R per store instruction
                const int gj = gj0 + lane;
                for (int r = 0; r < 32; ++r) {
                    const int gr = gi0 + r;
                    const float2 v = T[r * kEpiLd + lane];
                    if (gr < m && gj < m) {
                        reinterpret_cast<float2*>(r_out)[fbase + static_cast<size_t>(gr) * m + gj] = v;
                        // mirrored block (off-diagonal tiles): R(gj, gr) = conj(R(gr, gj)); lanes -> rows gj:
                        // strided, but only M >= 512 frames have off-diagonal tiles
                        if (!diag) reinterpret_cast<float2*>(r_out)[fbase + static_cast<size_t>(gj) * m + gr] =
                            make_float2(v.x, -v.y);
                    }
                }
                __syncwarp();
            }
            tc_fence_before();
            named_bar_sync(2, 128);  // all four epilogue warps finished reading TMEM
            if (warp == 6 && lane == 0) {
                if (rank == 0) mbar_arrive_local(smem_u32(acc_empty));
                else mbar_arrive_cluster(smem_u32(acc_empty), 0);
            }
        }
    }
    __syncthreads();
    cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// Rescue list: frames whose max |x| (pass 1) lies outside [2^-8, 2^15) and is finite and non-zero get
// xscale = 2^e with max |x| 2^e in [2^6, 2^7); frames with max |x| outside [2^-50, 2^50] (R = X X^H / N would
// leave the complex64 range the rest of the batch path computes in) are flagged kFrameRange instead. Resets
// amax for the next batch. One CTA; list order is irrelevant (frames are independent).
__global__ void __launch_bounds__(1024) k_rescue_list(uint32_t* __restrict__ amax, int32_t* __restrict__ status,
                                                      int frames, int32_t* __restrict__ list,
                                                      int32_t* __restrict__ count, float* __restrict__ xscale) {
    __shared__ int s_n;
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    for (int f = threadIdx.x; f < frames; f += blockDim.x) {
        const float a = __uint_as_float(amax[f]);
        amax[f] = 0u;
        if ((status[f] & kFrameNonFinite) || !(a > 0.f) || (a >= 0.00390625f && a < 32768.f)) continue;
        if (!isfinite(a)) {
            atomicOr(&status[f], kFrameRange);
            continue;
        }
        int e2 = 0;
        frexpf(a, &e2);  // a in [2^(e2-1), 2^e2)
        const int sh = 7 - e2;  // a 2^sh in [2^6, 2^7)
        // R (complex64) and the downstream fp32 data must stay representable: max |x| within 2^+-50
        if (sh > 57 || sh < -43) {
            atomicOr(&status[f], kFrameRange);
            continue;
        }
        xscale[f] = ldexpf(1.f, sh);
        list[atomicAdd(&s_n, 1)] = f;
    }
    __syncthreads();
    if (threadIdx.x == 0) *count = s_n;
}

}  // namespace cov
}  // namespace fmk

#ifdef FM_COV_TIMELINE
extern "C" int fm_debug_cov_timeline(long long* host, int zero) {
    if (zero) {
        static long long z[16 * 16] = {};
        return static_cast<int>(cudaMemcpyToSymbol(fmk::cov::g_cov_tl, z, sizeof(z)));
    }
    return static_cast<int>(cudaMemcpyFromSymbol(host, fmk::cov::g_cov_tl, sizeof(long long) * 16 * 16));
}
#endif

// Launch K1 for `frames` frames. Requirements: n even (TMA 16-byte row stride).
// Returns a cudaError_t value (cudaErrorInvalidValue for unsupported shapes).
// planes_hi != nullptr selects the fp16 hi/lo plane output (M <= 256, M even): planes_hi / planes_lo
// are frames x M x 2M halves (R / s_f interleaved re, im), scale[f] = s_f; d_r is unused then.
// rescue (optional, FmCovRescue): per-frame amax (zeroed once by the caller, reset by the list kernel), the
// rescue list / count and the prescale; with it the call enqueues pass 1, k_rescue_list and the rescue pass.
cudaError_t fm_launch_cov_tc(const float* d_x, float* d_r, int32_t* d_status, int64_t frames, int64_t m, int64_t n,
                             cudaStream_t stream, void* planes_hi, void* planes_lo, float* scale, int64_t n_true,
                             const FmCovRescue* rescue, int64_t t_rows, void* xplanes) {
    if (n_true <= 0) n_true = n;  // n: row length of d_x (even); n_true: snapshots for the 1/N scaling
    using namespace fmk::cov;
    const bool temporal = t_rows > 0;  // d_x: frames x t_rows x n; output m x m (m <= n), contraction over t_rows
    if (frames < 1 || m < 1 || n < 2 || (n & 1) || frames * m > 0x7fffffff || 2 * n > 0x7fffffff)
        return cudaErrorInvalidValue;
    if (temporal && (m > n || t_rows > 0x7fffffff || frames * t_rows > 0x7fffffff)) return cudaErrorInvalidValue;
    const bool planes = planes_hi != nullptr;
    if (planes && (m > 256 || (m & 1) || !planes_lo || !scale)) return cudaErrorInvalidValue;
    EncodeTiledFn enc = get_encode();
    if (!enc) return cudaErrorNotSupported;
    CUtensorMap map, rmap, mmap;
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult cr;
    if (temporal) {  // boxes of 16 antenna rows x 128 snapshots, rows past t_rows zero-filled per frame
        cuuint64_t tdims[3] = {static_cast<cuuint64_t>(2 * n), static_cast<cuuint64_t>(t_rows),
                               static_cast<cuuint64_t>(frames)};
        cuuint64_t tstr[2] = {static_cast<cuuint64_t>(8 * n), static_cast<cuuint64_t>(8 * n * t_rows)};
        cuuint32_t tbox[3] = {256, 16, 1};
        cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(d_x), tdims, tstr, tbox, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(2 * n), static_cast<cuuint64_t>(frames * m)};
        cuuint64_t strides[1] = {static_cast<cuuint64_t>(8 * n)};
        cuuint32_t box[2] = {32, 128};
        cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(d_x), dims, strides, box, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
    const int64_t nk_len = temporal ? t_rows : n;  // contraction length seen by the kernel
    const int epi = planes ? 2 : ((m % 2) == 0 ? 1 : 0);  // R row pitch 8M bytes must be a multiple of 16
    if (epi == 2) {
        cuuint64_t pdims[3] = {static_cast<cuuint64_t>(2 * m), static_cast<cuuint64_t>(m),
                               static_cast<cuuint64_t>(frames)};
        cuuint64_t pstr[2] = {static_cast<cuuint64_t>(4 * m), static_cast<cuuint64_t>(4 * m * m)};
        cuuint32_t pbox[3] = {64, 32, 1};  // 32 rows x 32 complex halves (128 B rows), 128B-swizzled
        cr = enc(&rmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, planes_hi, pdims, pstr, pbox, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
        cr = enc(&mmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, planes_lo, pdims, pstr, pbox, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
    } else if (epi == 1) {
        cuuint64_t rdims[3] = {static_cast<cuuint64_t>(2 * m), static_cast<cuuint64_t>(m),
                               static_cast<cuuint64_t>(frames)};
        cuuint64_t rstr[2] = {static_cast<cuuint64_t>(8 * m), static_cast<cuuint64_t>(8 * m * m)};
        cuuint32_t rbox[3] = {32, 32, 1};  // 32 rows x 16 complex, 128B-swizzled
        cuuint32_t mbox[3] = {64, 16, 1};  // 16 rows x 32 complex (mirrored block), plain
        cr = enc(&rmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d_r, rdims, rstr, rbox, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
        cr = enc(&mmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d_r, rdims, rstr, mbox, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
    } else {
        rmap = map;  // unused by the fallback epilogue
        mmap = map;
    }
    // diagonal-only launches (M <= 256: one tile per frame): eight converter warps in two groups taking alternate
    // stages (kSplit); multi-tile frames: eight warps splitting each stage's rows (every 256-row block of X is
    // converted once per tile it feeds)
    // ring depths (stages): general staging / operand, diagonal-only staging / operand
    const int rs[4] = {kStagesS, kStagesO, kDiagS, kDiagO};
    const int ring = rs[0] | (rs[1] << 8) | (rs[2] << 16) | (rs[3] << 24);
    auto set_attr = [](auto kern) {
        return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    };
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaSuccess;
        for (cudaError_t x : {set_attr(cov_tc_kernel<0, true, true>), set_attr(cov_tc_kernel<1, true, true>),
                              set_attr(cov_tc_kernel<2, true, true>), set_attr(cov_tc_kernel<1, true, true, true>)})
            if (e == cudaSuccess) e = x;
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const int nb = static_cast<int>((m + 255) / 256);
    const int tiles_per_frame = nb * (nb + 1) / 2;
    const int64_t tiles = frames * tiles_per_frame;
    if (tiles > 0x7fffffff) return cudaErrorInvalidValue;
    static int sm_count = 0;
    if (!sm_count) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev);
    }
    const int64_t pairs = std::min<int64_t>(tiles, std::max(1, sm_count / 2));
    const dim3 grid(static_cast<unsigned>(2 * pairs));
    // multi-tile spatial frames with a plane workspace: X converted once (k_x_planes), kF16 pass 1
    const bool f16 = xplanes != nullptr && tiles_per_frame > 1 && !temporal && epi == 1;
    const int64_t n_pad = (n + kF16Kc - 1) / kF16Kc * kF16Kc;
    CUtensorMap pre_map = map, pim_map = map;
    if (f16) {
        __half* pre = static_cast<__half*>(xplanes);
        __half* pim = pre + static_cast<size_t>(frames) * m * n_pad;
        cuuint64_t fdims[2] = {static_cast<cuuint64_t>(n_pad), static_cast<cuuint64_t>(frames * m)};
        cuuint64_t fstr[1] = {static_cast<cuuint64_t>(2 * n_pad)};
        cuuint32_t fbox[2] = {static_cast<cuuint32_t>(kF16Kc), static_cast<cuuint32_t>(kRows)};
        const CUtensorMapSwizzle sw = kF16Kc == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
        cr = enc(&pre_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, pre, fdims, fstr, fbox, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
        cr = enc(&pim_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, pim, fdims, fstr, fbox, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
        const int64_t xrows = frames * m;
        k_x_planes<<<static_cast<unsigned>((xrows + 8 * kXpRows - 1) / (8 * kXpRows)), 256, 0, stream>>>(
            reinterpret_cast<const float4*>(d_x), reinterpret_cast<uint2*>(pre), reinterpret_cast<uint2*>(pim),
            rescue ? rescue->amax : nullptr, d_status, xrows, static_cast<int>(m), static_cast<int>(n),
            static_cast<int>(n_pad));
    }
    auto go = [&](auto kern, bool conv8, bool pass2, bool kf16) {
        const int threads = (epi == 2 ? kThreadsP : kThreads) + (conv8 ? 128 : 0);
        const int smem = 1024 + (kf16 ? kF16Stages * kF16Stage : ring_region_bytes(ring, tiles_per_frame == 1)) +
                         kSmemEpilogue + kSmemBarriers;
        const bool r = rescue != nullptr;
        kern<<<grid, threads, smem, stream>>>(map, rmap, mmap, d_r, d_status, static_cast<int>(m),
                                              static_cast<int>(nk_len), tiles_per_frame, static_cast<int>(tiles),
                                              scale, static_cast<float>(1.0 / static_cast<double>(n_true)), 0, ring,
                                              pass2 ? rescue->list : nullptr, pass2 ? rescue->count : nullptr,
                                              pass2 ? rescue->xscale : nullptr,
                                              (r && !pass2 && !kf16) ? rescue->amax : nullptr, temporal ? 1 : 0,
                                              pre_map, pim_map);
    };
    auto launch = [&](bool pass2) {
        // eight converter warps in two groups taking alternate stages (tools/ab_build.sh, tools/ab_cov_general.sh:
        // c2 covariance 0.347 -> 0.324 ms, c4 3.25 -> 3.04 ms, the ToA path's T 0.746 -> 0.714 ms)
        if (f16 && !pass2) go(cov_tc_kernel<1, true, true, true>, true, false, true);
        else if (epi == 2) go(cov_tc_kernel<2, true, true>, true, pass2, false);
        else if (epi == 1) go(cov_tc_kernel<1, true, true>, true, pass2, false);
        else go(cov_tc_kernel<0, true, true>, true, pass2, false);
    };
    launch(false);
    if (rescue) {
        if (!d_status) return cudaErrorInvalidValue;
        k_rescue_list<<<1, 1024, 0, stream>>>(rescue->amax, d_status, static_cast<int>(frames), rescue->list,
                                              rescue->count, rescue->xscale);
        launch(true);
    }
    return cudaGetLastError();
}
