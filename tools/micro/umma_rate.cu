// Microbenchmark: tcgen05.mma issue rate per shape from fixed shared-memory operands (canonical K-major layout, no
// swizzle; or SWIZZLE_128B), one CTA per SM, one issuing thread, 8 accumulators round-robin.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/micro/umma_rate.cu -o /tmp/ur && /tmp/ur
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t a, int lbo, int sbo, int layout) {
    return static_cast<uint64_t>((a >> 4) & 0x3FFFu) | (static_cast<uint64_t>(lbo >> 4) << 16) |
           (static_cast<uint64_t>(sbo >> 4) << 32) | (1ull << 46) | (static_cast<uint64_t>(layout) << 61);
}
template <int KIND>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
    if (KIND == 0)
        asm volatile("{.reg .pred p; setp.ne.b32 p, 1, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;}" ::"r"(d), "l"(a), "l"(b), "r"(idesc));
    else
        asm volatile("{.reg .pred p; setp.ne.b32 p, 1, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(d), "l"(a), "l"(b), "r"(idesc));
}
__device__ __forceinline__ bool lane0() { return (threadIdx.x & 31) == 0; }
template <int KIND>
__global__ void k(int N, int iters, int layout, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 64 * 1024; i += blockDim.x) sm[i] = static_cast<uint8_t>(i * 7);
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = slot;
    // i8: c=S32(2), a=b=S8(1); f16: c=F32(1), a=b=BF16(1)
    const uint32_t idesc = (KIND == 0 ? (2u << 4) | (1u << 7) | (1u << 10) : (1u << 4) | (1u << 7) | (1u << 10)) |
                           ((static_cast<uint32_t>(N) >> 3) << 17) | ((128u >> 4) << 24);
    const int span = (512 / N < 8 ? 512 / N : 8) * N;  // columns cycled through (accumulators x N)
    if (warp == 0) {  // whole warp converged; one elected lane issues (uniform operands)
        const uint32_t a = su32(sm), b = su32(sm + 32768);
        const int lbo = layout == 0 ? 128 : 16, sbo = layout == 0 ? 256 : 1024;
        const uint64_t da = desc(a, lbo, sbo, layout), db = desc(b, lbo, sbo, layout);
        long long t0 = clock64();
        uint32_t col = 0;
        for (int i = 0; i < iters; ++i) {
            uint32_t pred;
            asm volatile("{.reg .pred e; elect.sync _|e, 0xffffffff; selp.u32 %0, 1, 0, e;}" : "=r"(pred));
            if (pred) mma<KIND>(tmem + col, da, db, idesc);
            __syncwarp();
            col += N;
            if (col >= static_cast<uint32_t>(span)) col = 0;
        }
        if (lane0()) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
        asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0; @!P bra W;}" ::"r"(su32(&bar)));
        long long t1 = clock64();
        if (lane0()) out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}
int main() {
    long long* d;
    cudaMalloc(&d, 8 * 148);
    cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    const int iters = 4000;
    for (int kind = 0; kind < 2; ++kind)
        for (int layout : {0, 2})
            for (int N : {16, 32, 48, 64, 96, 128, 192, 256}) {
                for (int rep = 0; rep < 2; ++rep) {
                    if (kind == 0) k<0><<<148, 128, 64 * 1024>>>(N, iters, layout, d);
                    else k<1><<<148, 128, 64 * 1024>>>(N, iters, layout, d);
                }
                cudaError_t e = cudaDeviceSynchronize();
                long long h[148];
                cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
                double avg = 0;
                for (int i = 0; i < 148; ++i) avg += h[i];
                avg /= 148.0 * iters;
                printf("%s layout %s M128 N%3d K32B: %.1f cyc/mma (floor 128N/256 = %.0f) %s\n", kind ? "f16" : "i8 ",
                       layout ? "SW128" : "none ", N, avg, 128.0 * N / 256, cudaGetErrorString(e));
            }
    return 0;
}
