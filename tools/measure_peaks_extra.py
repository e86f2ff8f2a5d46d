"""Peaks SURVEY.md §8(d) asks to be measured next to MEASURED_PEAKS.json: dense TF32, FP16 and INT8 tensor
throughput (cuBLAS through torch, 8192^3, best of 10 and sustained over 3 s) and the FP32 FFMA rate
(cuBLAS SGEMM with TF32 off). Writes one JSON object to stdout.

  python tools/measure_peaks_extra.py > profiles/rNN_measured_peaks_extra.json
"""
import json
import time

import torch


def gemm_rate(a, b, fn, flops, burst=10, sustain_s=3.0):
    for _ in range(3):
        fn(a, b)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(burst):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, flops / (e0.elapsed_time(e1) * 1e-3))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n, t0 = 0, time.time()
    e0.record()
    while time.time() - t0 < sustain_s:
        for _ in range(10):
            fn(a, b)
        n += 10
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return best / 1e12, n * flops / (e0.elapsed_time(e1) * 1e-3) / 1e12


def main():
    dev = torch.device("cuda:0")
    n = 8192
    fl = 2.0 * n ** 3
    out = {"gpu_name": torch.cuda.get_device_name(0), "torch": torch.__version__, "n": n,
           "how": "torch.matmul / torch._int_mm over n^3, CUDA events: best of 10 (burst), back to back for 3 s (sustained)"}
    a32 = torch.randn(n, n, device=dev)
    b32 = torch.randn(n, n, device=dev)
    torch.backends.cuda.matmul.allow_tf32 = True
    out["tf32_tflops"], out["tf32_tflops_sustained"] = gemm_rate(a32, b32, torch.matmul, fl)
    torch.backends.cuda.matmul.allow_tf32 = False
    m = 4096  # SGEMM on the CUDA cores is ~25x slower: smaller problem, same method
    out["ffma_tflops"], out["ffma_tflops_sustained"] = gemm_rate(a32[:m, :m].contiguous(), b32[:m, :m].contiguous(),
                                                                 torch.matmul, 2.0 * m ** 3)
    a16, b16 = a32.half(), b32.half()
    out["fp16_tflops"], out["fp16_tflops_sustained"] = gemm_rate(a16, b16, torch.matmul, fl)
    ab, bb = a32.bfloat16(), b32.bfloat16()
    out["bf16_tflops"], out["bf16_tflops_sustained"] = gemm_rate(ab, bb, torch.matmul, fl)
    try:
        a8 = torch.randint(-127, 127, (n, n), device=dev, dtype=torch.int8)
        b8 = torch.randint(-127, 127, (n, n), device=dev, dtype=torch.int8).t().contiguous().t()
        out["int8_tops"], out["int8_tops_sustained"] = gemm_rate(a8, b8, torch._int_mm, fl)
    except Exception as e:  # noqa: BLE001
        out["int8_tops"] = None
        out["int8_error"] = str(e)[:200]
    a64 = torch.randn(m, m, device=dev, dtype=torch.float64)
    b64 = torch.randn(m, m, device=dev, dtype=torch.float64)
    out["fp64_tflops"], out["fp64_tflops_sustained"] = gemm_rate(a64, b64, torch.matmul, 2.0 * m ** 3)
    src = torch.empty(1 << 30, dtype=torch.bfloat16, device=dev)
    dst = torch.empty_like(src)
    best = 0.0
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dst.copy_(src)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, 2 * src.numel() * 2 / (e0.elapsed_time(e1) * 1e-3))
    out["hbm_copy_gbs"] = best / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
