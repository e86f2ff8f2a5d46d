// Microbenchmark: FP64 tensor-core MMA (mma.sync m8n8k4 f64) throughput vs DFMA on this GPU, and
// F2F.F64.F32 conversion throughput.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_thr(double* out, int n) {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
    double c[8][2];
    for (int u = 0; u < 8; ++u) c[u][0] = c[u][1] = 0.0;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[u][0]), "+d"(c[u][1]) : "d"(a), "d"(b));
    }
    double s = 0.0;
    for (int u = 0; u < 8; ++u) s += c[u][0] + c[u][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void f2f_thr(double* out, int n) {
    float x0 = threadIdx.x * 1e-3f, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    for (int i = 0; i < n; ++i) {
        s0 += (double)x0; s1 += (double)x1; s2 += (double)x2; s3 += (double)x3;
        x0 += 1.0f; x1 += 1.0f; x2 += 1.0f; x3 += 1.0f;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}
int main() {
    double* d;
    cudaMalloc(&d, 1 << 26);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int n = 4096;
    for (int warps : {4, 8, 16}) {
        dmma_thr<<<sms * 2, 32 * warps>>>(d, 16);
        cudaEventRecord(e0);
        dmma_thr<<<sms * 2, 32 * warps>>>(d, n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * 8 * 8 * 4 * 8.0 * n * (sms * 2.0 * warps);
        printf("DMMA m8n8k4 (%d warps/CTA, 2 CTA/SM): %.2f TFLOP/s\n", warps, flops / ms / 1e9);
    }
    f2f_thr<<<sms * 4, 256>>>(d, 16);
    cudaEventRecord(e0);
    f2f_thr<<<sms * 4, 256>>>(d, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("F2F.F64.F32 (+DADD): %.1f Gconv/s = %.1f per SM per clk at 1.965 GHz\n", 4.0 * n * sms * 4 * 256 / ms / 1e6,
           4.0 * n * sms * 4 * 256 / (ms * 1e-3) / sms / 1.965e9);
    return 0;
}
