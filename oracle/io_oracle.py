"""ORACLE — test infrastructure only (never imported by the product package).

Restatement of the reference's matrix / spectrum file formats, R/src/io.cpp (header R/include/fastmusic/io.hpp:17-27),
used by tests/test_io.py to check the library's writers byte for byte and its readers on hand-made files.
The reference io.cpp needs Eigen (absent here), so it cannot be compiled as oracle/_ref; its own
tests (R/tests/test_io.cpp) are re-run against the library instead.
"""
from __future__ import annotations

import struct

import numpy as np

MAGIC = b"FMCX"  # R/src/io.cpp:13


def fmcx_bytes(a: np.ndarray) -> bytes:
    """write_matrix_binary, R/src/io.cpp:71-86: magic, u32 version 1, u32 rows, u32 cols, then row-major
    (float(re), float(im)) little-endian."""
    a = np.asarray(a)
    rows, cols = a.shape
    re = a.real.astype(np.float32)
    im = a.imag.astype(np.float32)
    payload = np.empty((rows, cols, 2), "<f4")
    payload[..., 0] = re
    payload[..., 1] = im
    return MAGIC + struct.pack("<III", 1, rows, cols) + payload.tobytes()


def fmcx_parse(data: bytes) -> np.ndarray:
    """read_matrix_binary, R/src/io.cpp:88-109 (ValueError stands in for the reference's runtime_error)."""
    if len(data) < 4 or data[:4] != MAGIC:
        raise ValueError("bad magic")
    if len(data) < 16:
        raise ValueError("unsupported version")
    version, rows, cols = struct.unpack("<III", data[4:16])
    if version != 1:
        raise ValueError("unsupported version")
    need = rows * cols * 8
    if len(data) - 16 < need:
        raise ValueError("truncated payload")
    f = np.frombuffer(data[16:16 + need], "<f4").reshape(rows, cols, 2)
    return (f[..., 0] + 1j * f[..., 1]).astype(np.complex64)


def _g17(v: float) -> str:
    # std::ostream << std::setprecision(17) << double (default floatfield) == printf("%.17g")
    return "%.17g" % v


def matrix_csv_text(a: np.ndarray) -> str:
    """write_matrix_csv, R/src/io.cpp:111-122."""
    a = np.asarray(a, np.complex128)
    rows, cols = a.shape
    out = [f"# rows={rows} cols={cols} re,im interleaved\n"]
    for i in range(rows):
        out.append(",".join(f"{_g17(a[i, j].real)},{_g17(a[i, j].imag)}" for j in range(cols)) + "\n")
    return "".join(out)


def spectrum_csv_text(values, theta0: float, theta1: float) -> str:
    """write_spectrum_csv, R/src/io.cpp:124-131 on theta_l = theta0 + ((theta1 - theta0) * l) / (L - 1)
    (R/src/spectrum.cpp:26-28 for the reference grid theta0 = 0, theta1 = pi)."""
    kpi = 3.14159265358979323846
    L = len(values)
    out = ["theta_deg,value\n"]
    for l in range(L):
        th = theta0 + ((theta1 - theta0) * float(l)) / float(L - 1)
        out.append(f"{_g17(th * 180.0 / kpi)},{_g17(float(values[l]))}\n")
    return "".join(out)
