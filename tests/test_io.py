"""Frame / result file formats (host code of the library; no GPU): the reference's own io tests
(R/tests/test_io.cpp) re-run against the library, plus byte-for-byte checks against the oracle restatement
(oracle/io_oracle.py) and the batch frame reader that feeds fm_estimate_batch_host."""
import os
import struct

import numpy as np
import pytest

import paper_1911_07434_b200 as fm
from oracle import io_oracle as IO


def _rng_matrix(seed, rows, cols):
    # a(i, j) = Complex(rng.normal(), rng.normal()) row by row, as R/tests/test_io.cpp:52-55 fills it
    z = fm.normals(seed, 2 * rows * cols).reshape(rows, cols, 2)
    return z[..., 0] + 1j * z[..., 1]


def test_binary_round_trip_at_float32_precision(tmp_path):
    # R/tests/test_io.cpp:50-63
    a = _rng_matrix(5, 7, 3)
    path = tmp_path / "mat.bin"
    fm.write_matrix_binary(path, a)
    back = fm.read_matrix_binary(path)
    assert back.shape == (7, 3)
    assert np.linalg.norm(back - a) < 1e-6 * np.linalg.norm(a)
    assert os.path.getsize(path) == 4 + 4 + 4 + 4 + 7 * 3 * 8
    assert path.read_bytes() == IO.fmcx_bytes(a)


def test_binary_writer_complex64_and_128_agree(tmp_path):
    a = _rng_matrix(6, 5, 9)
    fm.write_matrix_binary(tmp_path / "z.bin", a)
    fm.write_matrix_binary(tmp_path / "c.bin", a.astype(np.complex64))
    assert (tmp_path / "z.bin").read_bytes() == (tmp_path / "c.bin").read_bytes() == IO.fmcx_bytes(a)


def test_binary_reader_on_oracle_files(tmp_path):
    a = _rng_matrix(7, 4, 11).astype(np.complex64)
    (tmp_path / "o.bin").write_bytes(IO.fmcx_bytes(a))
    assert np.array_equal(fm.read_matrix_binary(tmp_path / "o.bin"), IO.fmcx_parse(IO.fmcx_bytes(a)))
    assert np.array_equal(fm.read_matrix_binary(tmp_path / "o.bin"), a)


def test_binary_reader_rejects_bad_files(tmp_path):
    # R/tests/test_io.cpp:65-69 (bad magic) and the other runtime_error branches of R/src/io.cpp:88-109
    junk = tmp_path / "junk.bin"
    junk.write_bytes(b"NOPE furthermore")
    with pytest.raises(OSError, match="bad magic"):
        fm.read_matrix_binary(junk)
    v2 = tmp_path / "v2.bin"
    v2.write_bytes(b"FMCX" + struct.pack("<III", 2, 1, 1) + bytes(8))
    with pytest.raises(OSError, match="unsupported version"):
        fm.read_matrix_binary(v2)
    short_hdr = tmp_path / "short.bin"
    short_hdr.write_bytes(b"FMCX" + struct.pack("<I", 1))
    with pytest.raises(OSError, match="unsupported version"):
        fm.read_matrix_binary(short_hdr)
    trunc = tmp_path / "trunc.bin"
    trunc.write_bytes(IO.fmcx_bytes(np.ones((3, 3), np.complex64))[:-5])
    with pytest.raises(OSError, match="truncated payload"):
        fm.read_matrix_binary(trunc)
    with pytest.raises(OSError, match="cannot open for reading"):
        fm.read_matrix_binary(tmp_path / "missing.bin")
    with pytest.raises(OSError, match="cannot open for writing"):
        fm.write_matrix_binary(tmp_path / "no_such_dir" / "x.bin", np.ones((2, 2)))


def test_binary_writer_rejects_non_finite(tmp_path):
    # ensure_finite, R/src/linalg.cpp:40-44 -> std::invalid_argument
    a = np.ones((2, 2), np.complex128)
    a[1, 0] = complex(np.nan, 0)
    with pytest.raises(ValueError, match="non-finite"):
        fm.write_matrix_binary(tmp_path / "nan.bin", a)
    assert not (tmp_path / "nan.bin").exists()


def test_empty_matrix_round_trip(tmp_path):
    fm.write_matrix_binary(tmp_path / "e.bin", np.zeros((0, 4), np.complex64))
    assert os.path.getsize(tmp_path / "e.bin") == 16
    assert fm.read_matrix_binary(tmp_path / "e.bin").shape == (0, 4)


def test_matrix_and_spectrum_csv_writers(tmp_path):
    # R/tests/test_io.cpp:71-95
    mpath = tmp_path / "mat.csv"
    fm.write_matrix_csv(mpath, np.eye(2))
    lines = mpath.read_text().splitlines()
    assert "rows=2" in lines[0]
    assert lines[1] == "1,0,0,0"
    p = fm.PseudoSpectrum(fm.AngleGrid(3), np.array([0.5, 1.5, 0.25]))
    spath = tmp_path / "spec.csv"
    fm.write_spectrum_csv(spath, p)
    lines = spath.read_text().splitlines()
    assert lines[0] == "theta_deg,value"
    assert len(lines) == 4
    # byte-for-byte against the restated formatting
    assert spath.read_text() == IO.spectrum_csv_text(p.values, 0.0, np.pi)
    a = _rng_matrix(8, 3, 4) * 1e-7
    fm.write_matrix_csv(mpath, a)
    assert mpath.read_text() == IO.matrix_csv_text(a)
    g = fm.baseline_grid(181)
    v = np.abs(fm.normals(9, 181)) + 0.1
    fm.write_spectrum_csv(spath, fm.PseudoSpectrum(g, v))
    assert spath.read_text() == IO.spectrum_csv_text(v, g.theta0, g.theta1)


def test_batch_frame_files_round_trip(tmp_path):
    """The ingest path: frames written one FMCX file each, read back in parallel straight into the batch
    layout fm_estimate_batch_host takes (bitwise)."""
    m, n, frames = 16, 24, 37
    x, _, _ = fm.generate_frames(m, n, 3, 41, 0, frames)
    paths = [tmp_path / f"frame_{f:04d}.fmcx" for f in range(frames)]
    fm.write_frames(paths, x, threads=4)
    for f in (0, 17, 36):
        assert paths[f].read_bytes() == IO.fmcx_bytes(x[f])
    back = fm.read_frames(paths, m, n, threads=5)
    assert np.array_equal(back, x)
    out = np.zeros_like(x)
    assert fm.read_frames(paths, m, n, out=out) is out and np.array_equal(out, x)


def test_batch_frame_reader_errors(tmp_path):
    m, n = 8, 8
    x, _, _ = fm.generate_frames(m, n, 2, 42, 0, 6)
    paths = [tmp_path / f"f{f}.fmcx" for f in range(6)]
    fm.write_frames(paths, x)
    fm.write_matrix_binary(paths[3], x[3][:, :4])  # wrong shape in the middle of the batch
    with pytest.raises(ValueError, match=r"f3.fmcx: 8x4 matrix, expected 8x8"):
        fm.read_frames(paths, m, n, threads=3)
    paths[4].write_bytes(b"FMCX")
    with pytest.raises((ValueError, OSError)):
        fm.read_frames(paths, m, n, threads=1)
    with pytest.raises(OSError, match="cannot open for reading"):
        fm.read_frames([tmp_path / "nope.fmcx"], m, n)
