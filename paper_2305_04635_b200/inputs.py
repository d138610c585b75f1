"""Seeded host-side inputs: the reference generator and the five BASELINE configs.

`generate_spd` restates the reference generator (`pkg/src/bandchol/core.py:155-181`)
with the same numpy calls in the same order, so it produces the same bytes for
the same (dim, bandwidth, seed) -- pinned by `tests/test_inputs.py` against
SHA-256 fingerprints of the reference's own output (tests/golden/).

`generate_spd_wide` is the C3 construction.  The reference has no generator for
it; BASELINE.json describes it in words and SURVEY.md §8(d) pins one reading:
start from generate_spd, s = diagonal - 1 (the full-row abs-sum), draw
f = 10**U[0,4] from default_rng([seed, 2]), diagonal = 1 + (0.05 + f) * s.
It stays strictly diagonally dominant, hence SPD.

Right-hand sides (C2, C5): default_rng([seed, 1]).uniform(-1, 1, n).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import BandedMatrix


def generate_spd(dim: int, bandwidth: int, seed: int) -> BandedMatrix:
    """Diagonally dominant SPD band matrix, byte-identical to core.py:155-181."""
    m = BandedMatrix(dim, bandwidth)
    n, k = m.dim, m.bandwidth
    p = m.panel
    rng = np.random.default_rng(seed)
    if k:
        draw = rng.uniform(-1.0, 1.0, size=(k, n))
        for d in range(1, k + 1):
            p[d, : n - d] = draw[d - 1, : n - d]
        absval = np.abs(p[1: k + 1])
        rowsum = absval.sum(axis=0)
        for d in range(1, k + 1):
            rowsum[d:] += absval[d - 1, : n - d]
        p[0, :] = 1.0 + rowsum
    else:
        p[0, :] = 1.0
    return m


def generate_spd_wide(dim: int, bandwidth: int, seed: int) -> BandedMatrix:
    """C3: diagonal = 1 + (0.05 + 10**U[0,4]) * (row abs-sum); SURVEY.md §8(d)."""
    m = generate_spd(dim, bandwidth, seed)
    p = m.panel
    s = p[0, :] - 1.0
    f = 10.0 ** np.random.default_rng([seed, 2]).uniform(0.0, 4.0, dim)
    p[0, :] = 1.0 + (0.05 + f) * s
    return m


def make_rhs(dim: int, seed: int) -> np.ndarray:
    """One right-hand side uniform[-1, 1]."""
    return np.random.default_rng([seed, 1]).uniform(-1.0, 1.0, dim)


@dataclass(frozen=True)
class BandConfig:
    """One BASELINE.json config.  batch > 1 means seeds 0..batch-1."""
    name: str
    dim: int
    bandwidth: int
    batch: int = 1
    wide_diagonal: bool = False
    solve: bool = False

    def matrix(self, seed: int = 0) -> BandedMatrix:
        gen = generate_spd_wide if self.wide_diagonal else generate_spd
        return gen(self.dim, self.bandwidth, seed)

    def model_flops(self) -> int:
        """BASELINE flop model n*kd*(kd+3), times the batch."""
        return self.batch * self.dim * self.bandwidth * (self.bandwidth + 3)

    def band_bytes(self) -> int:
        """Algorithmic HBM bytes: the band read once and written once, 16*n*(kd+1)."""
        return self.batch * 16 * self.dim * (self.bandwidth + 1)


CONFIGS = {
    "C1": BandConfig("C1", 2000, 50),
    "C2": BandConfig("C2", 20000, 200, solve=True),
    "C3": BandConfig("C3", 50000, 500, wide_diagonal=True),
    "C4": BandConfig("C4", 20000, 2000),
    "C5": BandConfig("C5", 4096, 100, batch=1024, solve=True),
}
