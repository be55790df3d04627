"""TNSR tensor files (the reference's on-disk format, proj/src/io.cpp:85-169).

Layout (SPEC.md io_cli TensorFileHeader): magic "TNSR", u16 version = 1,
u16 order N, N x u64 dims, then prod(dims) little-endian float64 values with
the first index fastest.  Errors are IoError with the reference's messages
(byte offsets included); writes are atomic (temp file + rename, io.cpp:31-68).
"""
from __future__ import annotations

import os
import struct
import tempfile

import numpy as np

from .api import ArgumentError, IoError

MAGIC = b"TNSR"
VERSION = 1


def read_tensor(path) -> np.ndarray:
    """read_tensor (io.cpp:85-149)."""
    path = os.fspath(path)
    try:
        f = open(path, "rb")
    except OSError:
        raise IoError(f"cannot open '{path}' for reading") from None
    with f:
        data = f.read()

    def need(offset, count, what):
        got = max(0, min(count, len(data) - offset))
        if got != count:
            raise IoError(f"'{path}': truncated {what} at byte offset {offset + got} "
                          f"(needed {count} bytes, got {got})")

    need(0, 4, "magic")
    if data[:4] != MAGIC:
        raise IoError(f"'{path}': bad magic at byte offset 0 (expected \"TNSR\")")
    need(4, 4, "header")
    version, order = struct.unpack_from("<HH", data, 4)
    if version != VERSION:
        raise IoError(f"'{path}': unsupported version {version} at byte offset 4")
    if order == 0:
        raise IoError(f"'{path}': zero order at byte offset 6")
    dims = []
    for n in range(order):
        off = 8 + 8 * n
        need(off, 8, "dimension")
        (v,) = struct.unpack_from("<Q", data, off)
        if v == 0 or v > (1 << 63) - 1:
            raise IoError(f"'{path}': invalid dimension {v} at byte offset {off}")
        dims.append(int(v))
    total = int(np.prod(dims, dtype=np.int64))
    payload = 8 + 8 * order
    nbytes = 8 * total
    got = max(0, min(nbytes, len(data) - payload))
    if got != nbytes:
        raise IoError(f"'{path}': truncated payload at byte offset {payload + got} "
                      f"(expected {nbytes} payload bytes, got {got})")
    if len(data) > payload + nbytes:
        raise IoError(f"'{path}': trailing bytes after payload at byte offset {payload + nbytes}")
    values = np.frombuffer(data, dtype="<f8", count=total, offset=payload).astype(np.float64)
    bad = np.flatnonzero(~np.isfinite(values))
    if bad.size:
        i = int(bad[0])
        raise IoError(f"'{path}': non-finite value at payload index {i} (byte offset {payload + 8 * i})")
    return values.reshape(dims, order="F")


def write_tensor(t, path) -> None:
    """write_tensor (io.cpp:151-169): atomic temp-file + rename."""
    a = np.asarray(t, dtype=np.float64)
    if a.ndim < 1:
        raise ArgumentError("write_tensor: empty tensor")
    if not np.all(np.isfinite(a)):
        raise ArgumentError("write_tensor: tensor contains non-finite entries")
    if a.ndim > 0xFFFF:
        raise ArgumentError("write_tensor: order does not fit the header")
    path = os.fspath(path)
    d = os.path.dirname(os.path.abspath(path))
    fd, tmp = tempfile.mkstemp(prefix=".tnsr.", dir=d)
    try:
        with os.fdopen(fd, "wb") as f:
            f.write(MAGIC)
            f.write(struct.pack("<HH", VERSION, a.ndim))
            for n in a.shape:
                f.write(struct.pack("<Q", int(n)))
            f.write(np.ravel(a, order="F").astype("<f8").tobytes())
        os.replace(tmp, path)
    except OSError as exc:
        try:
            os.unlink(tmp)
        except OSError:
            pass
        raise IoError(f"cannot write '{path}': {exc}") from None
