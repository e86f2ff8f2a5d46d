"""Throughput of the batched temporal covariance at the c2 frame shape: 1024 frames of
M=256 x N=512 -> T (512 x 512) per frame. CUDA events on the launch stream; X (1 GiB) exceeds L2.
Prints one JSON line: frames/s, achieved HBM GB/s on the algorithmic bytes (X read 8MN + T write 8N^2),
and tensor TFLOP/s on the HERK flops (8 N^2 M, complex MAC = 8 flops, full square as computed)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1911_07434_b200 as fm  # noqa: E402


def main():
    B, M, N = int(os.environ.get("FRAMES", 1024)), 256, 512
    x = torch.empty((B, M, N), dtype=torch.complex64)
    fm.generate_frames(M, N, 8, 5, 0, B, out=x.numpy())
    xd = x.cuda()
    out = torch.empty((B, N, N), dtype=torch.complex64, device="cuda")
    st = torch.empty((B,), dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()
    work = None  # only odd N needs scratch (padded rows)
    for _ in range(3):
        fm.temporal_covariance_batch(xd, out, st, stream=s, work=work)
    torch.cuda.synchronize()
    steps = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        fm.temporal_covariance_batch(xd, out, st, stream=s, work=work)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    alg_bytes = B * (8 * M * N + 8 * N * N)
    flops = B * 8.0 * N * N * M
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = peaks.get("hbm_gbs") or peaks.get("hbm_copy_gbs")
    print(json.dumps({"what": "fm_temporal_covariance_batch", "frames": B, "work": work is not None, "m": M, "n": N, "ms": ms,
                      "frames_per_s": B / (ms / 1e3), "alg_gbs": alg_bytes / (ms / 1e3) / 1e9,
                      "alg_frac_hbm": alg_bytes / (ms / 1e3) / 1e9 / hbm if hbm else None,
                      "tflops": flops / (ms / 1e3) / 1e12, "status_ok": bool((st == 0).all().item())}))


if __name__ == "__main__":
    main()
