"""Packed lower band storage: the layout contract of the drop-in.

Same convention as the reference (`pkg/src/bandchol/core.py:1-19`, `:47-150`):
element (i, j), j <= i <= min(N-1, j+k), lives at flat offset
`j * lead_dim + (i - j)` of one contiguous float64 buffer; with
`lead_dim = k + 1` this is exactly LAPACK `AB(ldab, N)` lower storage.  The
GPU kernels read and write this buffer in place, so a reference
`bandchol.BandedMatrix` can be passed to every entry point of this package
unchanged (the functions only use `.dim`, `.bandwidth`, `.lead_dim`, `.data`).

Padding slots (rows past min(N-1, j+k) in panel j, and rows past k when
lead_dim > k+1) are never written by any kernel, as in the reference
(`pkg/tests/test_blocked.py:412-418`).
"""

from __future__ import annotations

import numpy as np
from numpy.lib.stride_tricks import as_strided

from .errors import InvalidBandwidth, OutOfBand, ShapeMismatch


def index_map(i: int, j: int, lead_dim: int) -> int:
    """Flat storage offset of in-band (i, j) (reference core.py:34-44)."""
    if i < j:
        raise OutOfBand(f"({i}, {j}) lies in the unstored upper triangle")
    if i - j >= lead_dim:
        raise OutOfBand(f"({i}, {j}) lies below the band for lead_dim={lead_dim}")
    return j * lead_dim + (i - j)


class BandedMatrix:
    """Symmetric banded matrix in packed lower-band storage (core.py:47-150)."""

    __slots__ = ("dim", "bandwidth", "lead_dim", "data")

    def __init__(self, dim: int, bandwidth: int, lead_dim: int | None = None,
                 data: np.ndarray | None = None):
        if dim < 1:
            raise ShapeMismatch(f"dimension must be positive, got {dim}")
        if bandwidth < 0 or bandwidth >= dim:
            raise InvalidBandwidth(f"bandwidth {bandwidth} invalid for dimension {dim}")
        if lead_dim is None:
            lead_dim = bandwidth + 1
        if lead_dim < bandwidth + 1:
            raise ShapeMismatch(f"lead_dim {lead_dim} < bandwidth+1 ({bandwidth + 1})")
        self.dim = int(dim)
        self.bandwidth = int(bandwidth)
        self.lead_dim = int(lead_dim)
        if data is None:
            data = np.zeros(self.lead_dim * self.dim)
        else:
            data = np.ascontiguousarray(data, dtype=np.float64)
            if data.shape != (self.lead_dim * self.dim,):
                raise ShapeMismatch(
                    f"data length {data.shape} != lead_dim*dim = {self.lead_dim * self.dim}")
        self.data = data

    @property
    def panel(self) -> np.ndarray:
        """(lead_dim, N) view; panel[d, j] = element (j+d, j)."""
        return self.data.reshape(self.dim, self.lead_dim).T

    def row_view(self, i: int) -> np.ndarray:
        """Strided view of stored row i: entries (i, l), l in [max(0,i-k), i]."""
        lo = max(0, i - self.bandwidth)
        length = i - lo + 1
        start = lo * self.lead_dim + (i - lo)
        step = self.lead_dim - 1
        stop = start + (length - 1) * step + 1
        item = self.data.itemsize
        return as_strided(self.data[start:stop], shape=(length,), strides=(step * item,))

    def offset(self, i: int, j: int) -> int:
        if not (0 <= j <= i < self.dim):
            raise OutOfBand(f"({i}, {j}) outside the stored lower triangle of dim {self.dim}")
        if i - j > self.bandwidth:
            raise OutOfBand(f"({i}, {j}) outside bandwidth {self.bandwidth}")
        return index_map(i, j, self.lead_dim)

    def get(self, i: int, j: int) -> float:
        """Mathematical value A(i, j): symmetric, zero outside the band."""
        if i < j:
            i, j = j, i
        if not (0 <= j and i < self.dim):
            raise OutOfBand(f"({i}, {j}) outside a {self.dim}x{self.dim} matrix")
        if i - j > self.bandwidth:
            return 0.0
        return float(self.data[index_map(i, j, self.lead_dim)])

    def set(self, i: int, j: int, value: float) -> None:
        self.data[self.offset(i, j)] = value

    def copy(self) -> "BandedMatrix":
        return BandedMatrix(self.dim, self.bandwidth, self.lead_dim, self.data.copy())

    def band_panel(self) -> np.ndarray:
        """Fresh (k+1, N) copy of the band with padding forced to zero."""
        p = self.panel[: self.bandwidth + 1].copy()
        for d in range(1, self.bandwidth + 1):
            p[d, self.dim - d:] = 0.0
        return p

    def to_dense(self) -> np.ndarray:
        n, k = self.dim, self.bandwidth
        dense = np.zeros((n, n))
        p = self.panel
        for d in range(0, k + 1):
            idx = np.arange(n - d)
            dense[idx + d, idx] = p[d, : n - d]
        return dense + np.tril(dense, -1).T

    @classmethod
    def from_dense(cls, dense: np.ndarray, bandwidth: int,
                   lead_dim: int | None = None) -> "BandedMatrix":
        dense = np.asarray(dense, dtype=np.float64)
        n = dense.shape[0]
        if dense.shape != (n, n):
            raise ShapeMismatch(f"dense input must be square, got {dense.shape}")
        m = cls(n, bandwidth, lead_dim)
        p = m.panel
        for d in range(0, bandwidth + 1):
            idx = np.arange(n - d)
            p[d, : n - d] = dense[idx + d, idx]
        return m


def check_matrix(matrix) -> tuple[int, int, int, np.ndarray]:
    """Validate a BandedMatrix-like object (ours or the reference's)."""
    try:
        n, k, ld, data = matrix.dim, matrix.bandwidth, matrix.lead_dim, matrix.data
    except AttributeError as exc:
        raise ShapeMismatch(f"not a banded matrix: {exc}") from None
    if n < 1 or k < 0 or k >= n or ld < k + 1:
        raise ShapeMismatch(f"bad band geometry N={n}, k={k}, lead_dim={ld}")
    if not isinstance(data, np.ndarray) or data.dtype != np.float64 or data.shape != (ld * n,):
        raise ShapeMismatch("data must be a float64 array of length lead_dim*dim")
    if not data.flags.c_contiguous:
        raise ShapeMismatch("data must be C-contiguous")
    return int(n), int(k), int(ld), data
