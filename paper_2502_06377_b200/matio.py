"""Matrix files: the IBMI1 binary container and plain CSV (reference matio.py).

IBMI1 = 8-byte magic ``IBMI1\\0\\0\\0``, rows and cols as u64 little-endian,
then rows*cols float64 little-endian row-major (reference matio.py:3-47).
The host readers/writers here mirror the reference functions; the solve path
of the CLI instead streams IBMI1 files straight between disk and HBM through
``ibmi_load_ibmi1`` / ``ibmi_save_sigma_ibmi1`` (pinned slots, parallel
pread/pwrite) without a host copy of the matrix.
"""

from __future__ import annotations

import os

import numpy as np

from .exceptions import DimensionMismatch, IoError

MAGIC = b"IBMI1\x00\x00\x00"

__all__ = ["MAGIC", "read_header", "load_ibmi", "save_ibmi", "load_csv", "save_csv", "load_matrix", "save_matrix"]


def read_header(path) -> tuple[int, int]:
    """(rows, cols) of an IBMI1 file, validating magic and payload size."""
    with open(path, "rb") as fh:
        magic = fh.read(8)
        if magic != MAGIC:
            raise IoError(f"{path}: bad magic {magic!r}, expected {MAGIC!r}")
        hdr = fh.read(16)
    if len(hdr) != 16:
        raise IoError(f"{path}: truncated header")
    rows, cols = (int(v) for v in np.frombuffer(hdr, dtype="<u8"))
    if os.path.getsize(path) != 24 + 8 * rows * cols:
        raise IoError(f"{path}: expected {rows * cols} values for a {rows}x{cols} matrix")
    return rows, cols


def load_ibmi(path) -> np.ndarray:
    rows, cols = read_header(path)
    data = np.fromfile(path, dtype="<f8", offset=24)
    return data.reshape(rows, cols).astype(np.float64, copy=False)


def _matrix(a) -> np.ndarray:
    m = np.asarray(a, dtype=np.float64)
    if m.ndim != 2 or m.shape[0] < 1 or m.shape[1] < 1:
        raise DimensionMismatch(f"expected a nonempty 2-D matrix, got shape {m.shape}")
    return m


def save_ibmi(path, a) -> None:
    m = np.ascontiguousarray(_matrix(a), dtype="<f8")
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(np.asarray(m.shape, dtype="<u8").tobytes())
        m.tofile(fh)


def load_csv(path) -> np.ndarray:
    try:
        return np.loadtxt(path, delimiter=",", dtype=np.float64, ndmin=2)
    except ValueError as exc:
        raise IoError(f"{path}: malformed CSV matrix: {exc}") from exc


def save_csv(path, a) -> None:
    m = _matrix(a)
    with open(path, "w") as fh:
        for row in m:
            fh.write(",".join(repr(float(x)) for x in row) + "\n")


def is_csv(path) -> bool:
    return os.fspath(path).lower().endswith(".csv")


def load_matrix(path) -> np.ndarray:
    return load_csv(path) if is_csv(path) else load_ibmi(path)


def save_matrix(path, a) -> None:
    (save_csv if is_csv(path) else save_ibmi)(path, a)
