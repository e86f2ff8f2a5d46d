// Microbenchmark: legacy warp-level int8 MMA (mma.sync m16n8k32 s8.s8.s32) throughput on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void imma_thr(int* out, int n) {
    unsigned a0 = threadIdx.x * 0x01010101u, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 ^ 0x55u, b1 = b0 + 7;
    int c[8][4];
    for (int u = 0; u < 8; ++u) c[u][0] = c[u][1] = c[u][2] = c[u][3] = 0;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
            asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+r"(c[u][0]), "+r"(c[u][1]), "+r"(c[u][2]), "+r"(c[u][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    int s = 0;
    for (int u = 0; u < 8; ++u) s += c[u][0] + c[u][1] + c[u][2] + c[u][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    int* d;
    cudaMalloc(&d, 1 << 26);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int n = 4096;
    for (int warps : {4, 8, 16}) {
        imma_thr<<<sms * 2, 32 * warps>>>(d, 16);
        cudaEventRecord(e0);
        imma_thr<<<sms * 2, 32 * warps>>>(d, n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = 2.0 * 16 * 8 * 32 * 8.0 * n * (sms * 2.0 * warps);
        printf("IMMA m16n8k32 s8 (%d warps/CTA, 2 CTA/SM): %.1f TOP/s\n", warps, ops / ms / 1e9);
    }
    return 0;
}
