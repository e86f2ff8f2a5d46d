// Microbenchmark: the product kernel's fp64 Gram (G and H upper 8x8 blocks of 16x16 from a 128-row complex64
// tile in shared memory) on DMMA, 4 warps, isolated from the rest of the product kernel.
#include <cstdio>
#include <cuda_runtime.h>
struct c32 { float re, im; };
__device__ __forceinline__ void dmma_884(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__global__ void k(const c32* in, double* out, long long* cyc, int reps, int slots) {
    __shared__ c32 sC[128 * 17], sV[128 * 17];
    for (int e = threadIdx.x; e < 128 * 17; e += blockDim.x) { sC[e] = in[e]; sV[e] = in[e + 128 * 17]; }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane >> 2, r4 = lane & 3;
    double acc[2][8][2] = {};  // [slot][(term, k parity)][fragment]
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll 4
        for (int k0 = 0; k0 < 128; k0 += 4) {
            const int r = k0 + r4;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                if (u >= slots) continue;
                const int bi = (warp + u) & 1, bj = 1;
                const c32 xa = (u ? sV : sC)[r * 17 + 8 * bi + q];
                const c32 yb = sC[r * 17 + 8 * bj + q];
                const double xr = xa.re, xi = xa.im, yr = yb.re, yi = yb.im;
                const int par = (k0 >> 2) & 1;
                dmma_884(acc[u][0 + par], xr, yr);
                dmma_884(acc[u][2 + par], xi, yi);
                dmma_884(acc[u][4 + par], xr, yi);
                dmma_884(acc[u][6 + par], -xi, yr);
            }
        }
    }
    long long t1 = clock64();
    if (lane == 0) cyc[blockIdx.x * 4 + warp] = (t1 - t0) / reps;
    double t = 0; for (int u = 0; u < 2; ++u) for (int i = 0; i < 8; ++i) t += acc[u][i][0] + acc[u][i][1];
    out[blockIdx.x * 128 + threadIdx.x] = t;
}
int main() {
    c32* in; double* out; long long* cyc;
    cudaMalloc(&in, sizeof(c32) * 128 * 17 * 2); cudaMemset(in, 0, sizeof(c32) * 128 * 17 * 2);
    cudaMalloc(&out, sizeof(double) * 148 * 128); cudaMalloc(&cyc, sizeof(long long) * 148 * 4);
    for (int slots = 1; slots <= 2; ++slots) {
        k<<<148, 128>>>(in, out, cyc, 50, slots);
        cudaDeviceSynchronize();
        long long h[4]; cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
        printf("slots %d: cycles per frame-Gram per warp %lld %lld %lld %lld (DMMA per warp %d)\n", slots, h[0], h[1], h[2], h[3], slots * 128);
    }
    return 0;
}
