// Microbenchmark: FP64 vs FP32 FMA latency/throughput and __syncthreads cost on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dep_chain_f64(double* out, int n, long long* cyc) {
    double a = threadIdx.x * 1e-3, b = 1.0000001, c = 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) a = fma(a, b, c);
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void dep_chain_f32(float* out, int n, long long* cyc) {
    float a = threadIdx.x * 1e-3f, b = 1.0000001f, c = 1e-9f;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) a = fmaf(a, b, c);
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void thr_f64(double* out, int n) {
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double b = 1.0000001, c = 1e-9;
    for (int i = 0; i < n; ++i) {
        a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
        a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void thr_f32(float* out, int n) {
    float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const float b = 1.0000001f, c = 1e-9f;
    for (int i = 0; i < n; ++i) {
        a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
        a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void sync_cost(int n, long long* cyc) {
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    double* d; float* f; long long* cyc;
    cudaMalloc(&d, 1 << 26); cudaMalloc(&f, 1 << 26); cudaMalloc(&cyc, 1 << 20);
    long long h;
    const int n = 4096;
    dep_chain_f64<<<1, 32>>>(d, n, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.2f cycles\n", (double)h / n);
    dep_chain_f32<<<1, 32>>>(f, n, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("FFMA dependent latency: %.2f cycles\n", (double)h / n);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int blocks = 148 * 8, threads = 256, iters = 20000;
    thr_f64<<<blocks, threads>>>(d, 100); cudaEventRecord(e0);
    thr_f64<<<blocks, threads>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * (double)iters * blocks * threads;
    printf("FP64 FMA throughput: %.2f TFLOP/s\n", flops / ms / 1e9);
    thr_f32<<<blocks, threads>>>(f, 100); cudaEventRecord(e0);
    thr_f32<<<blocks, threads>>>(f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FP32 FMA throughput: %.2f TFLOP/s\n", flops / ms / 1e9);
    for (int nt : {64, 256}) for (int bps : {1, 2, 4}) {
        sync_cost<<<148 * bps, nt>>>(1000, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("__syncthreads: %d threads, %d blocks/SM: %.1f cycles\n", nt, bps, (double)h / 1000);
    }
    return 0;
}
