// Microbenchmark of the tcgen05 spectrum (csrc/spectrum_tc.cu) at the c2 shape (1024 frames, M = 256, L = 3601) on
// random digits: kernel time by CUDA events and, with -DSTC_TIMELINE, per-CTA phase stamps (clock64):
// 0 start, 1 MMA issuer ready (TMEM allocated), 2 first stage full, 5 last MMA issued, 3 accumulators ready
// (epilogue), 4 epilogue done.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSTC_TIMELINE -I include \
//        -I paper_1911_07434_b200/csrc tools/micro/spec_tc_bench.cu -lcuda -o /tmp/stb && /tmp/stb
#include "../../paper_1911_07434_b200/csrc/spectrum_tc.cu"

#include <algorithm>
#include <cstdio>
#include <vector>

int main(int argc, char** argv) {
    const int frames = argc > 1 ? atoi(argv[1]) : 1024, m = argc > 2 ? atoi(argv[2]) : 256, L = argc > 3 ? atoi(argv[3]) : 3601;
    const int mk = (m + 31) / 32 * 32, nqp = fm_spectrum_tc_pairs_pad(L, 0), fpad = fm_spectrum_tc_frames_pad(frames);
    std::vector<double> th(2 * static_cast<size_t>(frames) * m);
    for (size_t i = 0; i < th.size(); ++i) th[i] = std::sin(0.37 * i) * 0.3;
    std::vector<int8_t> zh(static_cast<size_t>(10) * nqp * mk);
    for (size_t i = 0; i < zh.size(); ++i) zh[i] = static_cast<int8_t>((i * 2654435761u >> 7) % 129) - 64;
    void* t; int8_t *zk, *tk; double *ts, *s64; float* s32;
    cudaMalloc(&t, th.size() * 8);
    cudaMemcpy(t, th.data(), th.size() * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&zk, zh.size());
    cudaMemcpy(zk, zh.data(), zh.size(), cudaMemcpyHostToDevice);
    cudaMalloc(&tk, static_cast<size_t>(10) * fpad * mk);
    cudaMalloc(&ts, 8 * fpad);
    cudaMalloc(&s64, 8ull * frames * L);
    cudaMalloc(&s32, 4ull * frames * L);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 5; ++i) fm_launch_spectrum_tc(t, zk, tk, ts, frames, m, L, s32, s64, 0, 0);
    cudaEventRecord(a);
    const int reps = 50;
    for (int i = 0; i < reps; ++i) fm_launch_spectrum_tc(t, zk, tk, ts, frames, m, L, s32, s64, 0, 0);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("status %s  slice+spectrum %.2f us per call (frames %d m %d L %d, grid %d x %d)\n", cudaGetErrorString(e),
           1000 * ms / reps, frames, m, L, nqp / fmk::spectc::kN, fpad / fmk::spectc::kM);
#ifdef STC_TIMELINE
    const int ctas = nqp / fmk::spectc::kN * fpad / fmk::spectc::kM;
    std::vector<long long> tl(static_cast<size_t>(ctas) * 8);
    cudaMemcpyFromSymbol(tl.data(), fmk::spectc::g_stc_tl, tl.size() * 8);
    double acc[5] = {0, 0, 0, 0, 0};
    for (int c = 0; c < ctas; ++c) {
        const long long* r = &tl[c * 8];
        acc[0] += r[1] - r[0];  // prologue
        acc[1] += r[2] - r[1];  // first TMA stage
        acc[2] += r[5] - r[2];  // MMA issue
        acc[3] += r[3] - r[2];  // first stage -> accumulators ready
        acc[4] += r[4] - r[3];  // epilogue
    }
    printf("avg cycles per CTA: prologue %.0f  first-stage %.0f  mma-issue %.0f  mainloop %.0f  epilogue %.0f\n",
           acc[0] / ctas, acc[1] / ctas, acc[2] / ctas, acc[3] / ctas, acc[4] / ctas);
#endif
    return 0;
}
