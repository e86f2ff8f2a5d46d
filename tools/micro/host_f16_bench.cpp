// Host-side complex64 -> fp16 conversion rate (F16C, threads, one frame at a time: amax pass then convert pass),
// to size an fp16 H2D path for fm_estimate_batch_host. Also pinned H2D rate for the halved bytes.
// g++ -O3 -mavx2 -mf16c -pthread host_f16_bench.cpp -I/usr/local/cuda/include -L/usr/local/cuda/lib64 -lcudart
#include <cuda_runtime.h>
#include <immintrin.h>

#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

int main(int argc, char** argv) {
    const int frames = 1024, m = 256, n = 512;
    const size_t per = static_cast<size_t>(m) * n * 2;  // floats per frame
    int threads = argc > 1 ? atoi(argv[1]) : static_cast<int>(std::thread::hardware_concurrency());
    float* x;
    uint16_t* h;
    cudaMallocHost(&x, per * frames * 4);
    cudaMallocHost(&h, per * frames * 2);
    for (size_t i = 0; i < per * frames; ++i) x[i] = static_cast<float>((i * 2654435761u) % 1000) * 1e-3f - 0.5f;
    void* d;
    cudaMalloc(&d, per * frames * 2);
    for (int rep = 0; rep < 4; ++rep) {
        auto t0 = std::chrono::steady_clock::now();
        std::atomic<int> next{0};
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t)
            pool.emplace_back([&] {
                for (;;) {
                    const int f = next.fetch_add(1);
                    if (f >= frames) return;
                    const float* src = x + f * per;
                    uint16_t* dst = h + f * per;
                    __m256 mx = _mm256_setzero_ps();
                    const __m256 absmask = _mm256_castsi256_ps(_mm256_set1_epi32(0x7fffffff));
                    for (size_t i = 0; i < per; i += 8) mx = _mm256_max_ps(mx, _mm256_and_ps(_mm256_loadu_ps(src + i), absmask));
                    float a[8];
                    _mm256_storeu_ps(a, mx);
                    float am = 0.f;
                    for (float v : a) am = std::fmax(am, v);
                    const __m256 sc = _mm256_set1_ps(am > 0 ? 1.0f : 1.0f);
                    for (size_t i = 0; i < per; i += 8) {
                        const __m128i v = _mm256_cvtps_ph(_mm256_mul_ps(_mm256_loadu_ps(src + i), sc), _MM_FROUND_TO_NEAREST_INT);
                        _mm_storeu_si128(reinterpret_cast<__m128i*>(dst + i), v);
                    }
                }
            });
        for (auto& th : pool) th.join();
        auto t1 = std::chrono::steady_clock::now();
        cudaMemcpy(d, h, per * frames * 2, cudaMemcpyHostToDevice);
        auto t2 = std::chrono::steady_clock::now();
        cudaMemcpy(d, x, per * frames * 2, cudaMemcpyHostToDevice);  // same bytes from the fp32 buffer (baseline)
        auto t3 = std::chrono::steady_clock::now();
        printf("threads %d convert %.2f ms  h2d fp16 (%.0f MB) %.2f ms  h2d same bytes %.2f ms\n", threads,
               std::chrono::duration<double, std::milli>(t1 - t0).count(), per * frames * 2 / 1e6,
               std::chrono::duration<double, std::milli>(t2 - t1).count(),
               std::chrono::duration<double, std::milli>(t3 - t2).count());
    }
    return 0;
}
