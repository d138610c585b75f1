"""BNDM band-matrix fixtures, on the host and straight to the device.

The on-disk format is the reference's (pkg/src/bandchol/core.py:254-283): the 16-byte
header ``'BNDM', u32 N, u32 k, u32 lead_dim`` (little-endian) followed by ``lead_dim*N``
little-endian float64 values -- the AB(lead_dim, N) column panels with the padding
entries zeroed.  ``load_matrix`` / ``save_matrix`` keep the reference's names and error
behaviour (``ShapeMismatch`` on a short file, a bad magic or a wrong payload size).
``load_matrix_device`` reads the payload into pinned host memory and copies it to a
CUDA tensor without an intermediate pageable copy, ready for ``dpbtrf_device``.
"""

from __future__ import annotations

import os
import struct

import numpy as np

from .core import BandedMatrix, check_matrix
from .errors import ShapeMismatch

MAGIC = b"BNDM"
HEADER = struct.Struct("<4sIII")


def save_matrix(matrix: BandedMatrix, path) -> None:
    """Write ``matrix`` as a BNDM fixture (padding bytes written as zeros)."""
    check_matrix(matrix)
    n, k, ld = matrix.dim, matrix.bandwidth, matrix.lead_dim
    clean = np.zeros(ld * n)
    clean.reshape(n, ld)[:, : k + 1] = np.asarray(matrix.data).reshape(n, ld)[:, : k + 1]
    with open(path, "wb") as fh:
        fh.write(HEADER.pack(MAGIC, n, k, ld))
        fh.write(clean.astype("<f8", copy=False).tobytes())


def _read_header(fh, size: int):
    head = fh.read(HEADER.size)
    if len(head) < HEADER.size:
        raise ShapeMismatch("fixture truncated before header end")
    magic, dim, bandwidth, lead_dim = HEADER.unpack(head)
    if magic != MAGIC:
        raise ShapeMismatch(f"bad fixture magic {magic!r}")
    expected = HEADER.size + 8 * lead_dim * dim
    if size != expected:
        raise ShapeMismatch(f"fixture payload is {size} bytes, expected {expected}")
    return dim, bandwidth, lead_dim


def load_matrix(path) -> BandedMatrix:
    """Read a BNDM fixture into a host ``BandedMatrix``."""
    with open(path, "rb") as fh:
        dim, bandwidth, lead_dim = _read_header(fh, os.fstat(fh.fileno()).st_size)
        data = np.frombuffer(fh.read(), dtype="<f8").astype(np.float64, copy=True)
    return BandedMatrix(dim, bandwidth, lead_dim, data)


def load_matrix_device(path, device: str = "cuda"):
    """Read a BNDM fixture straight into a CUDA float64 tensor.

    Returns ``(tensor, dim, bandwidth, lead_dim)``; the payload goes file -> pinned host
    buffer -> device (one DMA), the layout the kernels consume in place."""
    from .engine import _torch, pinned_empty

    torch = _torch()
    with open(path, "rb") as fh:
        dim, bandwidth, lead_dim = _read_header(fh, os.fstat(fh.fileno()).st_size)
        host = pinned_empty((lead_dim * dim,))
        view = memoryview(host.view(np.uint8))
        got = fh.readinto(view)
        if got != host.nbytes:
            raise ShapeMismatch(f"fixture payload short: {got} of {host.nbytes} bytes")
    if not np.little_endian:  # pragma: no cover - every supported host is little-endian
        host.byteswap(inplace=True)
    dev = torch.from_numpy(host).to(device, non_blocking=False)
    return dev, dim, bandwidth, lead_dim


__all__ = ["MAGIC", "HEADER", "save_matrix", "load_matrix", "load_matrix_device"]
