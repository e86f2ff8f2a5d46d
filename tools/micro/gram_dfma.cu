// Microbenchmark: fp64 Gram on DFMA, 4 warps, lane = (4x4 tile, sub-row), the product kernel's GM = 2 assignment.
#include <cstdio>
#include <cuda_runtime.h>
struct c32 { float re, im; };
struct c64 { double re, im; };
__device__ __forceinline__ void cmac_conj(c64& acc, c64 a, c64 b) {
    acc.re = fma(a.re, b.re, fma(a.im, b.im, acc.re));
    acc.im = fma(a.re, b.im, fma(-a.im, b.re, acc.im));
}
template <int S, typename T>
__global__ void k(const T* in, double* out, long long* cyc, int reps, int ntiles) {
    extern __shared__ __align__(16) unsigned char dsm_[]; T* sC = reinterpret_cast<T*>(dsm_); T* sV = sC + 128 * 17;
    for (int e = threadIdx.x; e < 128 * 17; e += blockDim.x) { sC[e] = in[e]; sV[e] = in[e + 128 * 17]; }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int per = (ntiles + 3) / 4, tl = lane / S, sub = lane % S, tix = warp * per + tl;
    const bool active = tl < per && tix < ntiles;
    const int ti = tix % 4, tj = (tix / 4) % 4;
    const bool second = tix >= 10;
    c64 acc[4][4] = {};
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
        if (active) {
#pragma unroll 2
            for (int r = sub; r < 128; r += S) {
                c64 x[4], y[4];
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    const T xa = (second ? sV : sC)[r * 17 + 4 * ti + a], yb = sC[r * 17 + 4 * tj + a];
                    x[a] = {double(xa.re), double(xa.im)};
                    y[a] = {double(yb.re), double(yb.im)};
                }
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) cmac_conj(acc[a][b], x[a], y[b]);
            }
        }
    }
    long long t1 = clock64();
    if (lane == 0) cyc[blockIdx.x * 16 + warp] = (t1 - t0) / reps;
    double t = 0; for (int a = 0; a < 4; ++a) for (int b = 0; b < 4; ++b) t += acc[a][b].re + acc[a][b].im;
    out[blockIdx.x * 512 + threadIdx.x] = t;
}
template <int S, typename T> void run(const char* nm, int ntiles, int nt) {
    T* in; double* out; long long* cyc;
    cudaMalloc(&in, sizeof(T) * 128 * 17 * 2); cudaMemset(in, 0, sizeof(T) * 128 * 17 * 2);
    cudaMalloc(&out, sizeof(double) * 148 * 512); cudaMalloc(&cyc, sizeof(long long) * 148 * 16);
    cudaFuncSetAttribute(k<S, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80000); k<S, T><<<148, nt, sizeof(T) * 128 * 17 * 2>>>(in, out, cyc, 50, ntiles);
    cudaDeviceSynchronize();
    long long h[4]; cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    printf("%s S=%d tiles=%d: cycles per frame-Gram per warp %lld %lld %lld %lld\n", nm, S, ntiles, h[0], h[1], h[2], h[3]);
}
int main() {
    run<4, c32>("c32", 26, 128); run<4, c64>("c64", 26, 128);
    run<8, c32>("c32", 10, 128); run<8, c64>("c64", 10, 128);
    run<4, c32>("c32", 20, 128);
    return 0;
}
