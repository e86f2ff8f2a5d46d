"""fm_estimate_batch_host — the reference-facing call from host buffers (C ABI, R/src/bench.cpp:59-86 frame
loop in batched form). It stages X in chunks on a copy stream while earlier chunks compute, draws Omega /
indices on the host and re-draws rank-deficient frames (R/src/estimators.cpp:114-137); every per-frame
output must be bitwise what the device-resident fm_run_batch gives on the same inputs."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

M, N, K, P = 64, 96, 3, 8


def _device_run(fm, method, x, seeds, grid):
    import torch
    frames = len(x)
    plan = fm.BatchPlan(M, N, K, method, p=P if method != "exact" else 0, t=1, grid_size=grid, max_frames=frames)
    xd = torch.from_numpy(np.ascontiguousarray(x).view(np.float32)).cuda()
    om = (torch.from_numpy(fm.draw_omega_batch(seeds, M, P)).cuda() if method == "fast2" else
          torch.from_numpy(fm.draw_uniforms_batch(seeds, M)).cuda() if method == "fast1_norm2" else None)
    ix = torch.from_numpy(fm.draw_indices_batch(seeds, M, P)).cuda() if method == "fast1" else None
    out = plan.outputs(frames, spectrum=True)
    plan.run(frames, xd, om, ix, out)
    torch.cuda.synchronize()
    res = {k: v.cpu().numpy() for k, v in out.items()}
    plan.close()
    return res


def _host_run(fm, method, x, seeds, grid, max_frames=None):
    frames = len(x)
    plan = fm.BatchPlan(M, N, K, method, p=P if method != "exact" else 0, t=1, grid_size=grid,
                        max_frames=max_frames or frames)
    spec = np.empty((frames, grid), np.float32)
    heights = np.empty((frames, K), np.float64)
    base = np.empty(frames, np.float64)
    xs = np.ascontiguousarray(x)
    res = plan.estimate_host(xs, None if method == "exact" else seeds, spectrum=spec, heights=heights, baseline=base)
    again = plan.estimate_host(xs, None if method == "exact" else seeds)  # staging reused, same answer
    assert np.array_equal(again["peak_cells"], res["peak_cells"])
    plan.close()
    return res


# 300 / 260 frames -> 2 chunks of 150 / 130; 130 -> 1 chunk; 5 frames in a larger plan
@pytest.mark.parametrize("method,frames,max_frames", [("fast2", 300, None), ("fast1", 260, None),
                                                      ("exact", 130, None), ("fast2", 5, 64),
                                                      ("fast1_norm2", 270, None)])
def test_host_path_matches_device_run(fm, method, frames, max_frames):
    x, _, _ = fm.generate_frames(M, N, K, 31, 0, frames)
    seeds = np.array([fm.derive(77, f) for f in range(frames)], np.uint64)
    dev = _device_run(fm, method, x, seeds, 721)
    host = _host_run(fm, method, x, seeds, 721, max_frames)
    assert np.all(host["status"] == 0)
    assert np.all(host["attempts"] == 1)
    assert np.array_equal(host["peak_cells"], dev["peak_cells"])
    assert np.array_equal(host["peak_count"], dev["peak_count"])
    assert np.array_equal(host["peak_heights"], dev["peak_heights"])
    assert np.array_equal(host["baseline"], dev["baseline"])
    assert np.array_equal(host["spectrum"], dev["spectrum"])


def test_host_path_redraws_rank_deficient_frames(fm):
    """An all-zero frame makes R Omega = 0: every draw is rank-deficient, so the host path spends all
    4 attempts on it and reports FM_FRAME_RANK, while the other frames (recomputed in the whole-batch
    rerun after the chunked pass) are unchanged."""
    from paper_1911_07434_b200 import _capi
    frames = 280
    x, _, _ = fm.generate_frames(M, N, K, 32, 0, frames)
    x[137] = 0
    seeds = np.array([fm.derive(78, f) for f in range(frames)], np.uint64)
    dev = _device_run(fm, "fast2", x, seeds, 721)
    host = _host_run(fm, "fast2", x, seeds, 721)
    assert host["status"][137] & _capi.FRAME_RANK
    assert host["attempts"][137] == 4
    ok = np.arange(frames) != 137
    assert np.all(host["status"][ok] == 0) and np.all(host["attempts"][ok] == 1)
    assert np.array_equal(host["peak_cells"][ok], dev["peak_cells"][ok])
    assert np.array_equal(host["spectrum"][ok], dev["spectrum"][ok])


def test_host_path_from_frame_files(fm, tmp_path):
    """SURVEY §8(f)1 ingest: one FMCX file per frame -> fm_fmcx_read_frames straight into pinned staging ->
    fm_estimate_batch_host; identical to the device run on the in-memory frames."""
    import torch
    frames = 260
    x, _, _ = fm.generate_frames(M, N, K, 33, 0, frames)
    paths = [tmp_path / f"frame_{f:04d}.fmcx" for f in range(frames)]
    fm.write_frames(paths, x)
    pinned = torch.empty((frames, M, N), dtype=torch.complex64).pin_memory().numpy()
    fm.read_frames(paths, M, N, out=pinned)
    assert np.array_equal(pinned, x)
    seeds = np.array([fm.derive(79, f) for f in range(frames)], np.uint64)
    dev = _device_run(fm, "fast2", x, seeds, 721)
    host = _host_run(fm, "fast2", pinned, seeds, 721)
    assert np.all(host["status"] == 0)
    assert np.array_equal(host["peak_cells"], dev["peak_cells"])
    assert np.array_equal(host["spectrum"], dev["spectrum"])


def test_coalesced_frame_stream_matches_per_batch_runs(fm):
    """bench.py's shard coalescing on real plans: one FrameStream launch over the shards of three consecutive
    batches (then a partial launch of one) packs the same per-frame records (fm_pack_peak_records) as three
    separate device runs."""
    import torch

    from paper_1911_07434_b200.shard import FrameStream, unshard_coalesced
    n, co = 40, 3
    x, _, _ = fm.generate_frames(M, N, K, 11, 0, co * n)
    seeds = np.array([fm.derive(fm.derive(11, f), 4) for f in range(co * n)], np.uint64)
    ref = _device_run(fm, "fast2", x, seeds, 721)
    xd = torch.from_numpy(np.ascontiguousarray(x).view(np.float32)).cuda()
    om = torch.from_numpy(fm.draw_omega_batch(seeds, M, P)).cuda()
    s = torch.cuda.Stream()
    fs = FrameStream(lambda i: fm.BatchPlan(M, N, K, "fast2", p=P, t=1, grid_size=721, max_frames=co * n),
                     co * n, co * n, K, 1, 2, [s, s], torch.device("cuda"))
    _, g = fs.step(xd, om)
    torch.cuda.synchronize()
    recs = [r.cpu().numpy() for r in unshard_coalesced(g, 1, n, co)]
    for i in range(co):
        sl = slice(i * n, (i + 1) * n)
        assert np.array_equal(recs[i][:, :K], ref["peak_cells"][sl])
        assert np.array_equal(recs[i][:, K], ref["peak_count"][sl])
        assert np.array_equal(recs[i][:, K + 1], ref["status"][sl])
    _, g = fs.step(xd, om, frames=n)  # partial launch: the first shard only
    torch.cuda.synchronize()
    assert np.array_equal(unshard_coalesced(g, 1, n, 1)[0].cpu().numpy()[:, :K], ref["peak_cells"][:n])
    fs.close()
