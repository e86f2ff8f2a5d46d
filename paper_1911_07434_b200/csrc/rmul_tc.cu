// K2 — batched range-finder products C_f = R_f V_f on the 5th-gen tensor cores.
//
// Replaces the dense products of the randomized range finder, R/src/estimators.cpp:104-139
// (fast_music_2: Y = R Omega, then Y = R Q per power iteration), R/src/linalg.cpp:180-192.
//
// The complex product is one real GEMM with K = 2M, taking R's interleaved rows straight
// from HBM as the A operand:
//     [C_re | C_im] (M x 2p) = A (M x 2M) * B (2M x 2p),  A(i, 2j + s) = (Re, Im)[s] R(i, j)
//     B(2j, c) = Re V(j,c), B(2j+1, c) = -Im V(j,c)     (columns c < p: C_re)
//     B(2j, p+c) = Im V(j,c), B(2j+1, p+c) = Re V(j,c)  (columns p + c: C_im)
// (real Omega: B(2j, c) = B(2j+1, p+c) = Omega(j, c), zeros elsewhere).
// Precision: kind::tf32 with both operands split hi + lo (hi = fp32 truncated to tf32, lo =
// the exact remainder, also read as tf32): A_hi B_hi + A_hi B_lo + A_lo B_hi, fp32 accumulate
// in TMEM -- ~22-bit operands with fp32's exponent range (no scaling of R needed). The
// tensor core reads an fp32 operand as tf32 by dropping the low 13 mantissa bits, so raw R is
// A_hi as it lands (FM_RMUL_TRUNC_A=1 adds an explicit in-place truncation pass; tools/
// check_rmul_tc.py verifies the two give bitwise-identical C).
//
// One CTA pair (cluster 2, cta_group::2) owns 256 rows of one frame. Per stage (32 reals of
// K = 16 complex j) each CTA receives by TMA its 128 rows of R (3D map {2M, M, B}, 128B-
// swizzled, rows / columns past M zero-filled) and the matching 16-j chunk of V (or Omega).
// Converter warps write A_lo and this CTA's rows of two B^T operands:
//   MMA1 (N = 4 PH): A_hi x [B_hi(re) B_hi(im) | B_lo(re) B_lo(im)]   (rank 0 | rank 1 rows)
//   MMA2 (N = 2 PH): A_lo x [B_hi(re) | B_hi(im)]                       (rank 0 | rank 1 rows)
// so A_hi is read once per K-step; MMA2 accumulates onto MMA1's hi columns and the epilogue
// adds the lo columns: C_re = D[c] + D[2PH + c], C_im = D[PH + c] + D[3PH + c] (PH = 16 or 32).
// Accumulators are 4-way buffered in TMEM, so the epilogue (TMEM -> C, column-major p x M)
// overlaps the next tile. HBM traffic: R once (8 M^2 bytes/frame) + V (8 M p bytes).

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "fm_common.cuh"
#include "tc_common.cuh"

namespace fmk {
namespace rmtc {
using namespace fmk::tc;

constexpr int kRows = 128;                  // rows of R per CTA
constexpr int kKc = 32;                     // fp32 K-elements per stage (128 B per row)
constexpr int kStages = 4;
constexpr int kABytes = kRows * kKc * 4;    // 16 KB
constexpr int kAcc = 4;                     // TMEM accumulator buffers
constexpr int kThreads = 320;               // w0 TMA, w1 MMA, w2..w5 convert, w6..w9 epilogue

template <int PH>
struct Cfg {
    static constexpr int kN1 = 4 * PH;                              // MMA1 N (accumulator columns)
    static constexpr int kN2 = 2 * PH;                              // MMA2 N
    static constexpr int kB1Bytes = 2 * PH * 128;                   // this CTA's MMA1 B^T rows
    static constexpr int kB2Bytes = PH * 128;                       // this CTA's MMA2 B^T rows
    static constexpr int kVBytes = PH * 128;                        // V chunk (<= PH rows x 16 complex)
    static constexpr int kOffB1 = 2 * kABytes;
    static constexpr int kOffB2 = kOffB1 + kB1Bytes;
    static constexpr int kOffV = kOffB2 + kB2Bytes;
    static constexpr int kStageBytes = kOffV + kVBytes;
    static constexpr int kTmemCols = kAcc * kN1;                    // 256 or 512
    static constexpr int kSmem = 1024 + kStages * kStageBytes + 256;
    static_assert(kStageBytes % 1024 == 0 && kOffB1 % 1024 == 0 && kOffB2 % 1024 == 0, "SW128 alignment");
};

// UMMA smem descriptor, K-major, SWIZZLE_128B: rows of 128 B, 8-row atoms 1024 B apart (SBO),
// LBO unused; the K-step advance is +32 B on the start address inside the swizzle atom.
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
    return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (1ull << 16) | (static_cast<uint64_t>(1024 >> 4) << 32) |
           (1ull << 46) | (2ull << 61);
}
// kind::tf32, A = B = TF32 (format 2), D = F32, K-major, M = 256.
__host__ __device__ constexpr uint32_t idesc_tf32(int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((static_cast<uint32_t>(n) >> 3) << 17) | ((256u >> 4) << 24);
}
__device__ __forceinline__ void umma_tf32_2sm(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ float tf32_trunc(float v) { return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); }
__device__ __forceinline__ float4 trunc4(float4 v) {
    return make_float4(tf32_trunc(v.x), tf32_trunc(v.y), tf32_trunc(v.z), tf32_trunc(v.w));
}
__device__ __forceinline__ float4 sub4(float4 a, float4 b) { return make_float4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w); }
__device__ __forceinline__ void tma_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
            "r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y), "r"(z)
        : "memory");
}

template <int PH, bool REAL>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    rmul_tc_kernel(const __grid_constant__ CUtensorMap rmap, const __grid_constant__ CUtensorMap vmap,
                   float* __restrict__ c_out, int m, int p, int tiles_per_frame, int total_tiles, int trunc_a) {
    using C = Cfg<PH>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024 - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023)) & 1023);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * C::kStageBytes);
    uint64_t* full = bars;                     // TMA bytes landed (local)
    uint64_t* op_full = bars + kStages;        // both CTAs' converters done (leader copy)
    uint64_t* empty = bars + 2 * kStages;      // MMA finished reading the stage (multicast)
    uint64_t* acc_full = bars + 3 * kStages;   // kAcc
    uint64_t* acc_empty = acc_full + kAcc;     // kAcc (leader copy, count 2)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + kAcc);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = __shfl_sync(0xffffffffu, cluster_rank(), 0);  // warp-uniform for the compiler
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int nk = (2 * m + kKc - 1) / kKc;
    const uint32_t vbytes = REAL ? 16u * p * 4u : static_cast<uint32_t>(p) * 128u;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(smem_u32(&full[s]), 1);
            mbar_init(smem_u32(&op_full[s]), 2);
            mbar_init(smem_u32(&empty[s]), 1);
        }
        for (int b = 0; b < kAcc; ++b) {
            mbar_init(smem_u32(&acc_full[b]), 1);
            mbar_init(smem_u32(&acc_empty[b]), 2);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(C::kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&rmap)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&vmap)) : "memory");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // warp-uniform: MMA operands in uniform registers

    if (warp == 0) {
        // ---------------- TMA producer: R rows + V (Omega) chunk per stage
        if (lane == 0) {
            int g = 0;
            for (int tile = pair; tile < total_tiles; tile += npairs) {
                const int frame = tile / tiles_per_frame, rb = tile % tiles_per_frame;
                const int y = 256 * rb + 128 * static_cast<int>(rank);
                for (int kc = 0; kc < nk; ++kc, ++g) {
                    const int s = g % kStages;
                    uint8_t* st = smem + s * C::kStageBytes;
                    mbar_wait(smem_u32(&empty[s]), ((g / kStages) & 1) ^ 1);
                    const uint32_t fb = smem_u32(&full[s]);
                    mbar_arrive_expect_tx(fb, kABytes + vbytes);
                    tma_3d(smem_u32(st), &rmap, fb, kKc * kc, y, frame);
                    if (REAL) tma_3d(smem_u32(st + C::kOffV), &vmap, fb, 0, 16 * kc, frame);
                    else tma_3d(smem_u32(st + C::kOffV), &vmap, fb, kKc * kc, 0, frame);
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (leader CTA; the warp waits converged, one elected lane issues)
        if (rank == 0) {
            constexpr uint32_t id1 = idesc_tf32(C::kN1), id2 = idesc_tf32(C::kN2);
            int g = 0, t = 0;
            for (int tile = pair; tile < total_tiles; tile += npairs, ++t) {
                const int b = t % kAcc;
                mbar_wait_cluster(smem_u32(&acc_empty[b]), ((t / kAcc) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + static_cast<uint32_t>(b * C::kN1);
                for (int kc = 0; kc < nk; ++kc, ++g) {
                    const int s = g % kStages;
                    mbar_wait_cluster(smem_u32(&op_full[s]), (g / kStages) & 1);
                    tc_fence_after();
                    const uint32_t st = smem_u32(smem + s * C::kStageBytes);
                    if (elect_one()) {
#pragma unroll
                        for (int ks = 0; ks < kKc / 8; ++ks) {
                            const uint32_t o = 32u * ks;
                            umma_tf32_2sm(d, desc_sw128(st + o), desc_sw128(st + C::kOffB1 + o), id1,
                                          (kc > 0 || ks > 0) ? 1u : 0u);
                            umma_tf32_2sm(d, desc_sw128(st + kABytes + o), desc_sw128(st + C::kOffB2 + o), id2, 1u);
                        }
                        umma_commit_mc(smem_u32(&empty[s]));
                    }
                    __syncwarp();
                }
                if (elect_one()) umma_commit_mc(smem_u32(&acc_full[b]));
                __syncwarp();
            }
        }
    } else if (warp < 6) {
        // ---------------- converters (128 threads): A_lo = A - tf32(A); V chunk -> B^T rows
        const int ct = threadIdx.x - 64;
        const int bc = ct >> 3, kq = ct & 7;  // B^T row group and 16-byte chunk of this thread
        int g = 0;
        for (int tile = pair; tile < total_tiles; tile += npairs) {
            for (int kc = 0; kc < nk; ++kc, ++g) {
                const int s = g % kStages;
                uint8_t* st = smem + s * C::kStageBytes;
                mbar_wait(smem_u32(&full[s]), (g / kStages) & 1);
                float4* a4 = reinterpret_cast<float4*>(st);
                float4* l4 = reinterpret_cast<float4*>(st + kABytes);
#pragma unroll
                for (int u = 0; u < kABytes / 16 / 128; ++u) {
                    const int i = ct + 128 * u;
                    const float4 v = a4[i];
                    const float4 h = trunc4(v);
                    if (trunc_a) a4[i] = h;
                    l4[i] = sub4(v, h);
                }
                const int j0 = 16 * kc + 2 * kq;  // complex index of this thread's 4 K-elements
#pragma unroll
                for (int u = 0; u < PH / 16; ++u) {
                    const int c = bc + 16 * u;
                    float4 re = make_float4(0.f, 0.f, 0.f, 0.f), im = re;
                    if (c < p && j0 < m) {
                        if (REAL) {  // Omega chunk: 16 rows j x p floats
                            const float* om = reinterpret_cast<const float*>(st + C::kOffV);
                            const float o0 = om[(2 * kq) * p + c];
                            const float o1 = j0 + 1 < m ? om[(2 * kq + 1) * p + c] : 0.f;
                            re = make_float4(o0, 0.f, o1, 0.f);
                            im = make_float4(0.f, o0, 0.f, o1);
                        } else {  // V chunk: p rows c x 16 complex j
                            const float4 v = *reinterpret_cast<const float4*>(st + C::kOffV + c * 128 + kq * 16);
                            re = make_float4(v.x, -v.y, v.z, -v.w);
                            im = make_float4(v.y, v.x, v.w, v.z);
                        }
                    }
                    const float4 reh = trunc4(re), imh = trunc4(im);
                    const int sw = (kq ^ (c & 7)) << 4;   // rows c, PH + c share (c & 7) (PH % 8 == 0)
                    uint8_t* b1 = st + C::kOffB1;
                    uint8_t* b2 = st + C::kOffB2;
                    if (rank == 0) {
                        *reinterpret_cast<float4*>(b1 + c * 128 + sw) = reh;
                        *reinterpret_cast<float4*>(b1 + (PH + c) * 128 + sw) = imh;
                        *reinterpret_cast<float4*>(b2 + c * 128 + sw) = reh;
                    } else {
                        *reinterpret_cast<float4*>(b1 + c * 128 + sw) = sub4(re, reh);
                        *reinterpret_cast<float4*>(b1 + (PH + c) * 128 + sw) = sub4(im, imh);
                        *reinterpret_cast<float4*>(b2 + c * 128 + sw) = imh;
                    }
                }
                fence_proxy_async();
                named_bar_sync(1, 128);
                if (ct == 0) {
                    if (rank == 0) mbar_arrive_local(smem_u32(&op_full[s]));
                    else mbar_arrive_cluster(smem_u32(&op_full[s]), 0);
                }
            }
        }
    } else {
        // ---------------- epilogue (warps 6..9): TMEM -> C (column-major p x M complex)
        const int quarter = warp & 3;
        int t = 0;
        for (int tile = pair; tile < total_tiles; tile += npairs, ++t) {
            const int frame = tile / tiles_per_frame, rb = tile % tiles_per_frame;
            const int b = t % kAcc;
            mbar_wait(smem_u32(&acc_full[b]), (t / kAcc) & 1);
            tc_fence_after();
            const uint32_t taddr = tmem + (static_cast<uint32_t>(32 * quarter) << 16) + static_cast<uint32_t>(b * C::kN1);
            uint32_t v[C::kN1];
#pragma unroll
            for (int h = 0; h < C::kN1 / 32; ++h) {
                uint32_t (&vh)[32] = *reinterpret_cast<uint32_t(*)[32]>(v + 32 * h);
                tmem_ld32(taddr + 32 * h, vh);
            }
            tmem_wait_ld();
            tc_fence_before();
            named_bar_sync(2, 128);
            if (warp == 6 && lane == 0) {
                if (rank == 0) mbar_arrive_local(smem_u32(&acc_empty[b]));
                else mbar_arrive_cluster(smem_u32(&acc_empty[b]), 0);
            }
            const int row = 256 * rb + 128 * static_cast<int>(rank) + 32 * quarter + lane;
            if (row < m) {
                float2* cf = reinterpret_cast<float2*>(c_out) + static_cast<size_t>(frame) * m * p;
#pragma unroll
                for (int c = 0; c < PH; ++c)
                    if (c < p)
                        cf[static_cast<size_t>(c) * m + row] =
                            make_float2(__uint_as_float(v[c]) + __uint_as_float(v[2 * PH + c]),
                                        __uint_as_float(v[PH + c]) + __uint_as_float(v[3 * PH + c]));
            }
        }
    }
    __syncthreads();
    cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::kTmemCols));
    }
}


// ------------------------------------------------------------------------------------------
// Plane variant: R arrives as fp16 hi / lo planes of R / s_f (written by the covariance epilogue,
// cov_tc.cu kEpi = 2), so A needs no conversion pass: per stage of 64 reals (32 complex j) each CTA
// TMA-loads 128 rows of both planes (16 KB each, 128B-swizzled) and the 32-column chunk of V / Omega;
// converters only build this CTA's fp16 hi / lo B^T rows; kind::f16 MMAs (K = 16):
//   MMA1 (N = 4 PH): A_hi x [B_hi(re) B_hi(im) | B_lo(re) B_lo(im)];  MMA2 (N = 2 PH): A_lo x B_hi.
// Epilogue: C = s_f (D_hi + D_lo). Representation error of R <= 2^-24 s_f (s_f >= max |R_ij|).
constexpr int kPKc = 64;                     // halves of K per stage
constexpr int kPStages = 4;
template <int PH>
struct PCfg {
    static constexpr int kN1 = 4 * PH, kN2 = 2 * PH;
    static constexpr int kOffLo = kABytes;                         // 16 KB planes
    static constexpr int kOffV = 2 * kABytes;
    static constexpr int kVBytes = PH * 256;                       // <= PH rows x 32 complex (or 32 x PH floats)
    static constexpr int kOffB1 = kOffV + kVBytes;
    static constexpr int kOffB2 = kOffB1 + 2 * PH * 128;
    static constexpr int kStageBytes = kOffB2 + PH * 128;
    static constexpr int kTmemCols = kAcc * kN1;
    static constexpr int kSmem = 1024 + kPStages * kStageBytes + 256;
    static_assert(kStageBytes % 1024 == 0 && kOffB1 % 1024 == 0 && kOffB2 % 1024 == 0, "SW128 alignment");
};
__host__ __device__ constexpr uint32_t idesc_f16(int n) {
    return (1u << 4) | ((static_cast<uint32_t>(n) >> 3) << 17) | ((256u >> 4) << 24);  // A = B = F16, D = F32
}
__device__ __forceinline__ void umma_f16_2sm_(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
    return static_cast<uint32_t>(__half_as_ushort(__float2half_rn(a))) |
           (static_cast<uint32_t>(__half_as_ushort(__float2half_rn(b))) << 16);
}
// hi / lo fp16 split of 8 values -> two 16-byte words
__device__ __forceinline__ void split8(const float (&x)[8], uint4& hi, uint4& lo) {
    float h[8], l[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        h[i] = __half2float(__float2half_rn(x[i]));
        l[i] = x[i] - h[i];
    }
    hi = make_uint4(pack_h2(h[0], h[1]), pack_h2(h[2], h[3]), pack_h2(h[4], h[5]), pack_h2(h[6], h[7]));
    lo = make_uint4(pack_h2(l[0], l[1]), pack_h2(l[2], l[3]), pack_h2(l[4], l[5]), pack_h2(l[6], l[7]));
}

// Gram epilogue (GM > 0, PH = 16, M <= 256): the epilogue also forms this CTA's 128-row partial of
// G = C^H C (GM >= 1) and of H = V^H C (GM = 2) in fp64 from the complex64 C it writes (the values the
// separate Gram kernels would read back), as upper 4 x 4 tiles mirrored (tiled_gram2's convention,
// smallmat.cu). Partials: gpart / hpart[(frame * 2 + rank) * p * p], column-major; consumers add the
// two CTA halves. Replaces k_gram_only / k_gram_gh on the power-iteration path.
template <int GM>
__host__ __device__ constexpr int plane_stages() {  // the fp64 C and V tiles of GM = 2 leave room for 3 stages
    return GM == 2 ? 3 : kPStages;
}
template <int PH, int GM>
__host__ __device__ constexpr int plane_gram_off() {  // fp64 tiles after the stages and barriers
    return plane_stages<GM>() * PCfg<PH>::kStageBytes + 256;
}
template <int PH, int GM>
__host__ __device__ constexpr int plane_smem() {
    return 1024 + plane_gram_off<PH, GM>() + (GM == 0 ? 0 : (GM == 2 ? 2 : 1) * kRows * (PH + 1) * 16);
}

constexpr int kThreadsG = kThreads + 128;  // GM = 1: four Gram warps (10 G tiles x 8 row groups)
#ifndef FM_GRAM_RG2
#define FM_GRAM_RG2 4  // 4 (four Gram warps, 80 active): 123 us; 8 (five warps): 128 us (scripts_ab_build.sh)
#endif
// GM = 2: 10 G + 10 H tiles x FM_GRAM_RG2 row groups (8: five Gram warps; 4: four)
constexpr int kThreadsG2 = kThreads + (FM_GRAM_RG2 == 8 ? 160 : 128);
template <int GM> __host__ __device__ constexpr int gram_threads() { return GM == 2 ? kThreadsG2 : kThreadsG; }
template <int GM> __host__ __device__ constexpr int handoff_count() { return gram_threads<GM>() - kThreads + 128; }
__device__ long long* g_gram_dbg = nullptr;  // debug: per-frame (wait at tile-full, Gram compute) cycles, CTA 0  // Gram epilogue: w10..w13 form the Gram halves

template <int PH, bool REAL, bool LO, int GM = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GM ? gram_threads<GM>() : kThreads, 1)
    rmul_planes_kernel(const __grid_constant__ CUtensorMap hmap, const __grid_constant__ CUtensorMap lmap,
                       const __grid_constant__ CUtensorMap vmap, const float* __restrict__ rscale,
                       float* __restrict__ c_out, int m, int p, int tiles_per_frame, int total_tiles,
                       const float* __restrict__ v_in, double* __restrict__ gpart, double* __restrict__ hpart,
                       int gdbg) {
    static_assert(GM == 0 || PH == 16, "Gram epilogue: PH = 16");
    constexpr int NST = plane_stages<GM>();
    using C = PCfg<PH>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024 - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023)) & 1023);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NST * C::kStageBytes);
    uint64_t* full = bars;
    uint64_t* op_full = bars + NST;
    uint64_t* empty = bars + 2 * NST;
    uint64_t* acc_full = bars + 3 * NST;
    uint64_t* acc_empty = acc_full + kAcc;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + kAcc);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = __shfl_sync(0xffffffffu, cluster_rank(), 0);  // warp-uniform for the compiler
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int nk = (2 * m + kPKc - 1) / kPKc;
    const uint32_t vbytes = REAL ? 32u * p * 4u : static_cast<uint32_t>(p) * 256u;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(smem_u32(&full[s]), 1);
            mbar_init(smem_u32(&op_full[s]), 2);
            mbar_init(smem_u32(&empty[s]), 1);
        }
        for (int b = 0; b < kAcc; ++b) {
            mbar_init(smem_u32(&acc_full[b]), 1);
            mbar_init(smem_u32(&acc_empty[b]), 2);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(C::kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&hmap)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&lmap)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&vmap)) : "memory");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // warp-uniform: MMA operands in uniform registers

    if (warp == 0) {
        if (lane == 0) {  // TMA producer
            int g = 0;
            for (int tile = pair; tile < total_tiles; tile += npairs) {
                const int frame = tile / tiles_per_frame, rb = tile % tiles_per_frame;
                const int y = 256 * rb + 128 * static_cast<int>(rank);
                for (int kc = 0; kc < nk; ++kc, ++g) {
                    const int s = g % NST;
                    uint8_t* st = smem + s * C::kStageBytes;
                    mbar_wait(smem_u32(&empty[s]), ((g / NST) & 1) ^ 1);
                    const uint32_t fb = smem_u32(&full[s]);
                    mbar_arrive_expect_tx(fb, (LO ? 2 : 1) * kABytes + vbytes);
                    tma_3d(smem_u32(st), &hmap, fb, kPKc * kc, y, frame);
                    if (LO) tma_3d(smem_u32(st + C::kOffLo), &lmap, fb, kPKc * kc, y, frame);
                    if (REAL) tma_3d(smem_u32(st + C::kOffV), &vmap, fb, 0, 32 * kc, frame);
                    else tma_3d(smem_u32(st + C::kOffV), &vmap, fb, kPKc * kc, 0, frame);
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {  // MMA issuer: the warp waits converged, one elected lane issues
            constexpr uint32_t id1 = idesc_f16(C::kN1), id2 = idesc_f16(C::kN2);
            int g = 0, t = 0;
            for (int tile = pair; tile < total_tiles; tile += npairs, ++t) {
                const int b = t % kAcc;
                mbar_wait_cluster(smem_u32(&acc_empty[b]), ((t / kAcc) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + static_cast<uint32_t>(b * C::kN1);
                for (int kc = 0; kc < nk; ++kc, ++g) {
                    const int s = g % NST;
                    mbar_wait_cluster(smem_u32(&op_full[s]), (g / NST) & 1);
                    tc_fence_after();
                    const uint32_t st = smem_u32(smem + s * C::kStageBytes);
                    if (elect_one()) {
#pragma unroll
                        for (int ks = 0; ks < kPKc / 16; ++ks) {
                            const uint32_t o = 32u * ks;
                            umma_f16_2sm_(d, desc_sw128(st + o), desc_sw128(st + C::kOffB1 + o), id1,
                                          (kc > 0 || ks > 0) ? 1u : 0u);
                            if (LO)
                                umma_f16_2sm_(d, desc_sw128(st + C::kOffLo + o), desc_sw128(st + C::kOffB2 + o), id2,
                                              1u);
                        }
                        umma_commit_mc(smem_u32(&empty[s]));
                    }
                    __syncwarp();
                }
                if (elect_one()) umma_commit_mc(smem_u32(&acc_full[b]));
                __syncwarp();
            }
        }
    } else if (warp < 6) {
        // converters: V / Omega chunk -> fp16 hi / lo B^T rows of this CTA
        const int ct = threadIdx.x - 64;
        const int bc = ct >> 3, kq = ct & 7;  // B^T row group and 16-byte chunk (4 complex j)
        int g = 0;
        for (int tile = pair; tile < total_tiles; tile += npairs) {
            for (int kc = 0; kc < nk; ++kc, ++g) {
                const int s = g % NST;
                uint8_t* st = smem + s * C::kStageBytes;
                mbar_wait(smem_u32(&full[s]), (g / NST) & 1);
#pragma unroll
                for (int u = 0; u < PH / 16; ++u) {
                    const int c = bc + 16 * u;
                    float re[8], im[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) re[i] = im[i] = 0.f;
                    if (c < p) {
                        if (REAL) {  // Omega chunk: 32 rows j x p floats
                            const float* om = reinterpret_cast<const float*>(st + C::kOffV);
#pragma unroll
                            for (int w = 0; w < 4; ++w) {
                                const float o = om[(4 * kq + w) * p + c];
                                re[2 * w] = o;
                                im[2 * w + 1] = o;
                            }
                        } else {  // V chunk: p rows c x 32 complex j
                            const float4* vr = reinterpret_cast<const float4*>(st + C::kOffV + c * 256 + kq * 32);
                            const float4 a = vr[0], b = vr[1];
                            const float vv[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
                            for (int w = 0; w < 4; ++w) {
                                re[2 * w] = vv[2 * w];
                                re[2 * w + 1] = -vv[2 * w + 1];
                                im[2 * w] = vv[2 * w + 1];
                                im[2 * w + 1] = vv[2 * w];
                            }
                        }
                    }
                    uint4 reh, rel, imh, iml;
                    split8(re, reh, rel);
                    split8(im, imh, iml);
                    const int sw = (kq ^ (c & 7)) << 4;  // rows c and PH + c share (c & 7)
                    uint8_t* b1 = st + C::kOffB1;
                    uint8_t* b2 = st + C::kOffB2;
                    if (rank == 0) {
                        *reinterpret_cast<uint4*>(b1 + c * 128 + sw) = reh;
                        *reinterpret_cast<uint4*>(b1 + (PH + c) * 128 + sw) = imh;
                        *reinterpret_cast<uint4*>(b2 + c * 128 + sw) = reh;
                    } else {
                        *reinterpret_cast<uint4*>(b1 + c * 128 + sw) = rel;
                        *reinterpret_cast<uint4*>(b1 + (PH + c) * 128 + sw) = iml;
                        *reinterpret_cast<uint4*>(b2 + c * 128 + sw) = imh;
                    }
                }
                fence_proxy_async();
                named_bar_sync(1, 128);
                if (ct == 0) {
                    if (rank == 0) mbar_arrive_local(smem_u32(&op_full[s]));
                    else mbar_arrive_cluster(smem_u32(&op_full[s]), 0);
                }
            }
        }
    } else if (warp >= kThreads / 32) {
        if constexpr (GM > 0) {
            // Gram warps: per frame, this CTA's 128-row halves of G = C^H C (and H = V^H C for GM = 2) in fp64
            // from the tile the epilogue staged; upper 4 x 4 tiles, mirrored (tiled_gram2's convention).
            constexpr int ld = PH + 1;
            const fmk::c64* sC = reinterpret_cast<const fmk::c64*>(smem + plane_gram_off<PH, GM>());
            const fmk::c64* sV = sC + kRows * ld;
            constexpr int RG = GM == 2 ? FM_GRAM_RG2 : 8;  // row groups (consecutive lanes) per 4 x 4 tile
            const int et = threadIdx.x - kThreads;
            const int nb = p >> 2, t1 = nb * (nb + 1) / 2;
            const int gt = et / RG, rg = et % RG;
            const bool second = gt >= t1;
            const bool active = gt < (GM == 2 ? 2 : 1) * t1;
            int ti = 0, tj = 0;
            if (active) {
                int rem = second ? gt - t1 : gt;
                while (rem >= nb - ti) { rem -= nb - ti; ++ti; }
                tj = ti + rem;
            }
            const fmk::c64* xs = second ? sV : sC;
            for (int tile = pair; tile < total_tiles; tile += npairs) {
                const int frame = tile / tiles_per_frame;
                fmk::c64 acc[4][4];
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) acc[a][b] = fmk::mk(0.0, 0.0);
                const long long Tw0 = clock64();
                named_bar_sync(4, handoff_count<GM>());  // tile full
                const long long Tw1 = clock64();
                if (active && !(gdbg & 1)) {
#pragma unroll 4
                    for (int r = rg; r < kRows; r += RG) {
                        fmk::c64 x[4], y[4];
#pragma unroll
                        for (int a = 0; a < 4; ++a) {
                            x[a] = xs[r * ld + 4 * ti + a];
                            y[a] = sC[r * ld + 4 * tj + a];
                        }
#pragma unroll
                        for (int a = 0; a < 4; ++a)
#pragma unroll
                            for (int b = 0; b < 4; ++b) fmk::cmac_conj(acc[a][b], x[a], y[b]);
                    }
                }
                if (g_gram_dbg && blockIdx.x == 0 && threadIdx.x == kThreads) {
                    const int it = (tile - pair) / npairs;
                    g_gram_dbg[2 * it] = Tw1 - Tw0;
                    g_gram_dbg[2 * it + 1] = clock64() - Tw1;
                }
                if (tile + npairs < total_tiles) named_bar_arrive(5, handoff_count<GM>());  // tile free for the next frame
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b)
#pragma unroll
                        for (int o = 1; o < RG; o <<= 1) {
                            acc[a][b].re += __shfl_xor_sync(0xffffffffu, acc[a][b].re, o);
                            acc[a][b].im += __shfl_xor_sync(0xffffffffu, acc[a][b].im, o);
                        }
                if (active && rg == 0) {
                    fmk::c64* G = reinterpret_cast<fmk::c64*>(second ? hpart : gpart) +
                                  (static_cast<size_t>(frame) * 2 + rank) * p * p;
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int b = 0; b < 4; ++b) {
                            const int i = 4 * ti + a, j = 4 * tj + b;
                            G[j * p + i] = acc[a][b];
                            if (ti != tj) G[i * p + j] = fmk::conj(acc[a][b]);
                        }
                }
            }
        }
    } else {
        // epilogue: C = s_f (D_hi + D_lo), column-major p x M complex
        const int quarter = warp & 3;
        int t = 0;
        for (int tile = pair; tile < total_tiles; tile += npairs, ++t) {
            const int frame = tile / tiles_per_frame, rb = tile % tiles_per_frame;
            const int b = t % kAcc;
            mbar_wait(smem_u32(&acc_full[b]), (t / kAcc) & 1);
            tc_fence_after();
            const uint32_t taddr = tmem + (static_cast<uint32_t>(32 * quarter) << 16) + static_cast<uint32_t>(b * C::kN1);
            uint32_t v[C::kN1];
#pragma unroll
            for (int h = 0; h < C::kN1 / 32; ++h) {
                uint32_t (&vh)[32] = *reinterpret_cast<uint32_t(*)[32]>(v + 32 * h);
                tmem_ld32(taddr + 32 * h, vh);
            }
            tmem_wait_ld();
            tc_fence_before();
            named_bar_sync(2, 128);
            if (warp == 6 && lane == 0) {
                if (rank == 0) mbar_arrive_local(smem_u32(&acc_empty[b]));
                else mbar_arrive_cluster(smem_u32(&acc_empty[b]), 0);
            }
            const float sf = rscale[frame];
            const int row = 256 * rb + 128 * static_cast<int>(rank) + 32 * quarter + lane;
            if (row < m) {
                float2* cf = reinterpret_cast<float2*>(c_out) + static_cast<size_t>(frame) * m * p;
#pragma unroll
                for (int c = 0; c < PH; ++c)
                    if (c < p)
                        cf[static_cast<size_t>(c) * m + row] =
                            make_float2(sf * (__uint_as_float(v[c]) + __uint_as_float(v[2 * PH + c])),
                                        sf * (__uint_as_float(v[PH + c]) + __uint_as_float(v[3 * PH + c])));
            }
            if constexpr (GM > 0) {
                // hand this row of C (and of V) to the Gram warps through the shared tile; rows >= m are zero.
                // Barrier 5: the Gram warps finished reading the previous frame's tile; barrier 4: tile full.
                constexpr int ld = PH + 1;
                fmk::c64* sC = reinterpret_cast<fmk::c64*>(smem + plane_gram_off<PH, GM>());
                fmk::c64* sV = sC + kRows * ld;
                const int lr = 32 * quarter + lane;
                const bool ok = row < m;
                float2 vv[PH];
                if constexpr (GM == 2) {
                    const float2* vf = reinterpret_cast<const float2*>(v_in) + static_cast<size_t>(frame) * m * p;
#pragma unroll
                    for (int c = 0; c < PH; ++c) vv[c] = (ok && c < p) ? vf[static_cast<size_t>(c) * m + row] : make_float2(0.f, 0.f);
                }
                if (t > 0) named_bar_sync(5, handoff_count<GM>());
#pragma unroll
                for (int c = 0; c < PH; ++c) {  // the complex64 values written to C, widened once
                    const float re = sf * (__uint_as_float(v[c]) + __uint_as_float(v[2 * PH + c]));
                    const float im = sf * (__uint_as_float(v[PH + c]) + __uint_as_float(v[3 * PH + c]));
                    sC[lr * ld + c] = (ok && c < p) ? fmk::mk(static_cast<double>(re), static_cast<double>(im))
                                                    : fmk::mk(0.0, 0.0);
                }
                if constexpr (GM == 2) {
#pragma unroll
                    for (int c = 0; c < PH; ++c)
                        sV[lr * ld + c] = fmk::mk(static_cast<double>(vv[c].x), static_cast<double>(vv[c].y));
                }
                named_bar_arrive(4, handoff_count<GM>());
            }
        }
    }
    __syncthreads();
    cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::kTmemCols));
    }
}

}  // namespace rmtc
}  // namespace fmk

// C = R V (V complex, column-major p x m) or C = R Omega (omega real, row-major m x p).
// Requirements: m even (TMA row pitch), 4 <= p <= 32, p % 4 == 0 (Omega row pitch).
cudaError_t fm_launch_rmul_tc(const float* d_r, const float* d_omega, const float* d_v, float* d_c, int64_t frames,
                              int64_t m, int64_t p, cudaStream_t stream) {
    using namespace fmk::rmtc;
    if (frames < 1 || m < 2 || (m & 1) || p < 4 || p > 32 || (p & 3) || (!d_omega == !d_v))
        return cudaErrorInvalidValue;
    if (frames * m > 0x7fffffff || 2 * m > 0x7fffffff) return cudaErrorInvalidValue;
    auto enc = fmk::tc::get_encode();
    if (!enc) return cudaErrorNotSupported;
    CUtensorMap rmap, vmap;
    cuuint32_t estr[3] = {1, 1, 1};
    {
        cuuint64_t dims[3] = {static_cast<cuuint64_t>(2 * m), static_cast<cuuint64_t>(m), static_cast<cuuint64_t>(frames)};
        cuuint64_t strides[2] = {static_cast<cuuint64_t>(8 * m), static_cast<cuuint64_t>(8 * m * m)};
        cuuint32_t box[3] = {kKc, kRows, 1};
        if (enc(&rmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(d_r), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    if (d_omega) {  // Omega: {p, m, frames}, box {p, 16, 1}
        cuuint64_t dims[3] = {static_cast<cuuint64_t>(p), static_cast<cuuint64_t>(m), static_cast<cuuint64_t>(frames)};
        cuuint64_t strides[2] = {static_cast<cuuint64_t>(4 * p), static_cast<cuuint64_t>(4 * p * m)};
        cuuint32_t box[3] = {static_cast<cuuint32_t>(p), 16, 1};
        if (enc(&vmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(d_omega), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    } else {  // V: {2m, p, frames}, box {32, p, 1}
        cuuint64_t dims[3] = {static_cast<cuuint64_t>(2 * m), static_cast<cuuint64_t>(p), static_cast<cuuint64_t>(frames)};
        cuuint64_t strides[2] = {static_cast<cuuint64_t>(8 * m), static_cast<cuuint64_t>(8 * m * p)};
        cuuint32_t box[3] = {kKc, static_cast<cuuint32_t>(p), 1};
        if (enc(&vmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(d_v), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    const int tiles_per_frame = static_cast<int>((m + 255) / 256);
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
    auto go = [&](auto kern, int smem) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        kern<<<grid, kThreads, smem, stream>>>(rmap, vmap, d_c, static_cast<int>(m), static_cast<int>(p),
                                               tiles_per_frame, static_cast<int>(tiles), 0);
        return cudaGetLastError();
    };
    if (p <= 16)
        return d_omega ? go(rmul_tc_kernel<16, true>, Cfg<16>::kSmem) : go(rmul_tc_kernel<16, false>, Cfg<16>::kSmem);
    return d_omega ? go(rmul_tc_kernel<32, true>, Cfg<32>::kSmem) : go(rmul_tc_kernel<32, false>, Cfg<32>::kSmem);
}

extern "C" int32_t fm_debug_set_gram_buffer(long long* d) {
    return cudaMemcpyToSymbol(fmk::rmtc::g_gram_dbg, &d, sizeof(d)) == cudaSuccess ? 0 : 1;
}

// Debug entry (not part of the public header): run the tensor-core product synchronously.
extern "C" int32_t fm_debug_rmul_tc(const float* d_r, const float* d_omega, const float* d_v, float* d_c,
                                    int64_t frames, int64_t m, int64_t p) {
    cudaError_t e = fm_launch_rmul_tc(d_r, d_omega, d_v, d_c, frames, m, p, nullptr);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    return static_cast<int32_t>(e);
}

// C = R V / C = R Omega from the fp16 hi / lo planes of R / s_f (M <= 256, M even, p % 4 == 0, p <= 32).
// hi_only: skip the lo plane (R represented to 2^-12 s_f instead of 2^-24 s_f; half the R bytes read).
// gram: 0 none, 1 G partials -> gpart, 2 G and H = V^H C partials -> gpart, hpart (p <= 16, V products only
// for 2); see rmul_planes_kernel.
cudaError_t fm_launch_rmul_planes(const void* planes_hi, const void* planes_lo, const float* d_scale,
                                  const float* d_omega, const float* d_v, float* d_c, int64_t frames, int64_t m,
                                  int64_t p, cudaStream_t stream, bool hi_only, int gram, double* gpart,
                                  double* hpart) {
    using namespace fmk::rmtc;
    if (frames < 1 || m < 2 || (m & 1) || m > 256 || p < 4 || p > 32 || (p & 3) || (!d_omega == !d_v))
        return cudaErrorInvalidValue;
    auto enc = fmk::tc::get_encode();
    if (!enc) return cudaErrorNotSupported;
    CUtensorMap hmap, lmap, vmap;
    cuuint32_t estr[3] = {1, 1, 1};
    {
        cuuint64_t dims[3] = {static_cast<cuuint64_t>(2 * m), static_cast<cuuint64_t>(m), static_cast<cuuint64_t>(frames)};
        cuuint64_t strides[2] = {static_cast<cuuint64_t>(4 * m), static_cast<cuuint64_t>(4 * m * m)};
        cuuint32_t box[3] = {kPKc, kRows, 1};
        if (enc(&hmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(planes_hi), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
            enc(&lmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(planes_lo), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    if (d_omega) {  // Omega: {p, m, frames}, box {p, 32, 1}
        cuuint64_t dims[3] = {static_cast<cuuint64_t>(p), static_cast<cuuint64_t>(m), static_cast<cuuint64_t>(frames)};
        cuuint64_t strides[2] = {static_cast<cuuint64_t>(4 * p), static_cast<cuuint64_t>(4 * p * m)};
        cuuint32_t box[3] = {static_cast<cuuint32_t>(p), 32, 1};
        if (enc(&vmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(d_omega), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    } else {  // V: {2m, p, frames}, box {64, p, 1}
        cuuint64_t dims[3] = {static_cast<cuuint64_t>(2 * m), static_cast<cuuint64_t>(p), static_cast<cuuint64_t>(frames)};
        cuuint64_t strides[2] = {static_cast<cuuint64_t>(8 * m), static_cast<cuuint64_t>(8 * m * p)};
        cuuint32_t box[3] = {64, static_cast<cuuint32_t>(p), 1};
        if (enc(&vmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(d_v), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    const int tiles_per_frame = 1;
    const int64_t tiles = frames;
    static int sm_count = 0;
    if (!sm_count) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev);
    }
    const int64_t pairs = std::min<int64_t>(tiles, std::max(1, sm_count / 2));
    const dim3 grid(static_cast<unsigned>(2 * pairs));
    auto go = [&](auto kern, int smem) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        kern<<<grid, gram == 2 ? kThreadsG2 : gram == 1 ? kThreadsG : kThreads, smem, stream>>>(hmap, lmap, vmap, d_scale, d_c, static_cast<int>(m),
                                                                       static_cast<int>(p), tiles_per_frame,
                                                                       static_cast<int>(tiles), d_v, gpart, hpart, 0);
        return cudaGetLastError();
    };
    if (gram > 0) {
        if (p > 16 || !gpart || (gram == 2 && (!hpart || d_omega))) return cudaErrorInvalidValue;
        if (gram == 2)
            return hi_only ? go(rmul_planes_kernel<16, false, false, 2>, plane_smem<16, 2>())
                           : go(rmul_planes_kernel<16, false, true, 2>, plane_smem<16, 2>());
        if (d_omega)
            return hi_only ? go(rmul_planes_kernel<16, true, false, 1>, plane_smem<16, 1>())
                           : go(rmul_planes_kernel<16, true, true, 1>, plane_smem<16, 1>());
        return hi_only ? go(rmul_planes_kernel<16, false, false, 1>, plane_smem<16, 1>())
                       : go(rmul_planes_kernel<16, false, true, 1>, plane_smem<16, 1>());
    }
    if (hi_only) {
        if (p <= 16)
            return d_omega ? go(rmul_planes_kernel<16, true, false>, PCfg<16>::kSmem)
                           : go(rmul_planes_kernel<16, false, false>, PCfg<16>::kSmem);
        return d_omega ? go(rmul_planes_kernel<32, true, false>, PCfg<32>::kSmem)
                       : go(rmul_planes_kernel<32, false, false>, PCfg<32>::kSmem);
    }
    if (p <= 16)
        return d_omega ? go(rmul_planes_kernel<16, true, true>, PCfg<16>::kSmem)
                       : go(rmul_planes_kernel<16, false, true>, PCfg<16>::kSmem);
    return d_omega ? go(rmul_planes_kernel<32, true, true>, PCfg<32>::kSmem)
                   : go(rmul_planes_kernel<32, false, true>, PCfg<32>::kSmem);
}
