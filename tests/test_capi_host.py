"""CPU-side checks of the product library: it loads, exports every symbol the header
declares, its host RNG / draws / frame generator are bit-exact with the oracle and the
reference golden streams, and plan validation mirrors the reference messages."""
import ctypes
import json
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "fastmusic_b200.h")).read()
    return sorted(set(re.findall(r"\b(fm_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol(fm):
    from paper_1911_07434_b200 import _capi
    lib = ctypes.CDLL(_capi.LIB_PATH)
    declared = header_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_capi.EXPORTED) == declared


def test_product_rng_matches_reference_golden(fm):
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "rng_ref.json")))
    for st in g["streams"]:
        assert np.array_equal(fm.normals(st["seed"], len(st["normal"])), np.array(st["normal"]))


def test_product_draws_match_oracle(fm, oracle):
    for seed in (0, 1, 2**63 + 11, 987654321):
        assert fm.derive(seed, 0xF257 + 2) == oracle.derive(seed, 0xF257 + 2)
        assert np.array_equal(fm.gaussian_matrix_real(37, 9, seed), oracle.gaussian_matrix_real(37, 9, seed))
        assert np.array_equal(fm.sample_without_replacement(seed, 256, 32),
                              oracle.sample_without_replacement(seed, 256, 32))
    seeds = np.array([oracle.derive(5, f) for f in range(6)], np.uint64)
    om = fm.draw_omega_batch(seeds, 64, 8)
    for f, s in enumerate(seeds):
        assert np.array_equal(om[f], oracle.gaussian_matrix_real(64, 8, int(s)).astype(np.float32))
    ix = fm.draw_indices_batch(seeds, 256, 32)
    for f, s in enumerate(seeds):
        assert np.array_equal(ix[f], oracle.sample_without_replacement(int(s), 256, 32))


def test_frame_generator_matches_oracle(fm, oracle):
    cfgs = oracle.baseline_configs()
    spec = cfgs["c2"].spec
    xo, ao, so = oracle.generate_batch(2, range(3), spec)
    xp, ap, sp = fm.generate_frames(256, 512, 8, 2, 0, 3)
    assert np.array_equal(xo, xp) and np.array_equal(ao, ap) and np.array_equal(so, sp)
    c1 = cfgs["c1"]
    xo, ao, _ = oracle.generate_batch(1, [0], c1.spec)
    xp, ap, _ = fm.generate_frames(64, 200, 3, 1, 0, 1, fixed_angles_deg=(-20.0, 5.0, 31.0), snr_lo_db=20,
                                   snr_hi_db=20)
    assert np.array_equal(xo, xp) and np.array_equal(ao, ap)


def test_plan_validation_messages(fm):
    with pytest.raises(ValueError, match="fast_music_2: need 1 <= K < M"):
        fm.BatchPlan(16, 32, 16, "fast2", p=16, t=1)
    with pytest.raises(ValueError, match="fast_music_2: need K <= p <= M"):
        fm.BatchPlan(16, 32, 4, "fast2", p=2, t=1)
    with pytest.raises(ValueError, match="1 <= t <= 20"):
        fm.BatchPlan(16, 32, 4, "fast2", p=8, t=21)
    with pytest.raises(ValueError, match="fast_music_1: need K <= p <= M"):
        fm.BatchPlan(16, 32, 4, "fast1", p=17)
    with pytest.raises(ValueError, match="AngleGrid"):
        fm.BatchPlan(16, 32, 4, "exact", grid_size=1)


def test_facade_argument_validation_without_gpu(fm):
    s = np.eye(4, dtype=complex)
    with pytest.raises(ValueError):
        fm.fast_music_2(s, 3, fm.Fast2Params(2, 2, 0))
    with pytest.raises(ValueError):
        fm.fast_music_1(s, 3, fm.Fast1Params(5, 0))
    with pytest.raises(ValueError):
        fm.exact_signal_subspace(s, 4)
    with pytest.raises(ValueError):
        fm.hermitian(np.ones((2, 3)))
    with pytest.raises(ValueError):
        fm.AngleGrid(1)


def test_library_has_no_unresolved_internal_symbols():
    """A launcher whose declaration drifted from its definition links into the .so as an undefined
    C++ symbol and only fails at load time on the GPU box; catch it here."""
    import subprocess
    from paper_1911_07434_b200 import _capi
    out = subprocess.run(["nm", "-D", "--undefined-only", _capi.LIB_PATH], capture_output=True, text=True).stdout
    bad = [ln for ln in out.splitlines() if "fm_" in ln or "fmk" in ln]
    assert not bad, bad


def test_api_type_helpers(fm):
    """R/include/fastmusic/types.hpp:45-62 (R/src/linalg.cpp:14-44): method names round-trip through the enum
    order, unknown names and non-finite matrices raise with the reference's messages."""
    names = ["exact", "fast1", "fast2", "lanczos", "matrix_inverse", "propagator", "fft"]
    for i, n in enumerate(names):
        assert fm.method_from_name(n) == i and fm.method_name(i) == n
    assert fm.method_name(99) == "unknown"
    with pytest.raises(ValueError, match="unknown method name: nope"):
        fm.method_from_name("nope")
    good = np.ones((2, 2), complex)
    bad = good.copy()
    bad[1, 0] = np.inf
    assert fm.is_finite(good) and not fm.is_finite(bad)
    fm.ensure_finite(good, "thin_svd")
    with pytest.raises(ValueError, match="thin_svd: non-finite entries"):
        fm.ensure_finite(bad, "thin_svd")
    e = fm.EigResult(np.zeros(2), np.eye(2, dtype=complex))
    s = fm.SvdResult(np.eye(2, dtype=complex), np.ones(2), np.eye(2, dtype=complex))
    assert e.eigenvectors.shape == (2, 2) and s.sigma.shape == (2,)
