// Microbenchmark: tcgen05.mma cta_group::2 kind::f16 M256 N256 K16 (the covariance MMA) issue rate from fixed
// shared-memory operands (canonical K-major, no swizzle), with `noise` warps per CTA streaming ld/st.shared
// traffic concurrently (the converters' load), to separate the MMA floor from shared-memory contention.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/micro/umma2_rate.cu -o /tmp/u2 && /tmp/u2
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
    return static_cast<uint64_t>((a >> 4) & 0x3FFFu) | (static_cast<uint64_t>(128 >> 4) << 16) |
           (static_cast<uint64_t>(256 >> 4) << 32) | (1ull << 46);
}
__device__ __forceinline__ uint32_t crank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ bool elect() {
    uint32_t p;
    asm volatile("{.reg .pred e; elect.sync _|e, 0xffffffff; selp.u32 %0, 1, 0, e;}" : "=r"(p));
    return p;
}
__global__ void __cluster_dims__(2, 1, 1) k(int iters, int noise, int nmma, long long* out, float* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    __shared__ volatile int done;
    for (int i = threadIdx.x; i < 96 * 1024; i += blockDim.x) sm[i] = static_cast<uint8_t>(i * 7);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = crank();
    if (threadIdx.x == 0) {
        done = 0;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;");
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = slot;
    const uint32_t idesc = (1u << 4) | ((256u >> 3) << 17) | ((256u >> 4) << 24);
    if (warp == 0) {
        if (rank == 0) {
            const uint32_t a = su32(sm), b = su32(sm + 16384);
            long long t0 = clock64();
            for (int i = 0; i < iters; ++i) {
                if (elect()) {
                    for (int j = 0; j < nmma; ++j) {
                        const uint64_t da = desc(a + 4096 * (j & 1)), db = desc(b + 4096 * (j >> 1));
                        asm volatile("{.reg .pred p; setp.ne.b32 p, 1, 0; tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(tmem + 256 * (j >> 1)),
                                     "l"(da), "l"(db), "r"(idesc));
                    }
                }
                __syncwarp();
            }
            if (elect())
                asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(su32(&bar)), "h"(static_cast<uint16_t>(3)));
            __syncwarp();
            asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0; @!P bra W;}" ::"r"(su32(&bar)));
            long long t1 = clock64();
            if (lane == 0) out[blockIdx.x >> 1] = t1 - t0;
        } else {
            asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0; @!P bra W;}" ::"r"(su32(&bar)));
        }
        if (lane == 0) done = 1;
    } else if (warp <= noise) {
        // noise: a converter-like stream of 16-byte shared loads + stores over a 64 KB region
        float acc = 0.f;
        const int w = warp - 1;
        uint32_t base = su32(sm + 32768);
        int it = 0;
        while (!done) {
            for (int u = 0; u < 16; ++u) {
                const uint32_t off = ((it * 16 + u) * 512 + w * 2048 + lane * 16) & 0xFFF0u;
                float4 v;
                asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(base + off));
                acc += v.x + v.w;
                asm volatile("st.shared.v2.f32 [%0], {%1,%2};" ::"r"(base + ((off + 8192) & 0xFFF0u)), "f"(v.y), "f"(v.z));
            }
            ++it;
        }
        if (acc == 12345.f) sink[0] = acc;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}
int main() {
    long long* d;
    float* s;
    cudaMalloc(&d, 8 * 148);
    cudaMalloc(&s, 4);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    const int iters = 500;
    for (int noise : {0, 2, 4, 8})
        for (int nmma : {4}) {
            for (int rep = 0; rep < 2; ++rep) k<<<148, 320, 96 * 1024>>>(iters, noise, nmma, d, s);
            cudaError_t e = cudaDeviceSynchronize();
            long long h[74];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < 74; ++i) avg += h[i];
            avg /= 74.0 * iters * nmma;
            printf("cta_group::2 M256 N256 K16 f16: %.1f cyc/mma with %d noise warps (floor 128) %s\n", avg, noise,
                   cudaGetErrorString(e));
        }
    return 0;
}
