"""CPU oracle for the band Cholesky path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module; it is the checker, never the thing
measured or shipped.  The product package (paper_2305_04635_b200) never imports
it and has no CPU fallback.

* `factor_reference`  -- bit-exact restatement of pkg/src/bandchol/reference.py:32-63
                         (C, exactly rounded sums; band_oracle.c).
* `factor_plain`      -- same recurrence, ordinary rounding, fast (large configs).
* `factor_plain_batched` -- factor_plain over a batch, one matrix per host thread.
* `factor_blocked_dense` -- numpy/scipy blocked restatement (blocked.py:259-284 algebra)
                         for C3/C4 full-L parity in seconds.
* `solve`             -- pkg/src/bandchol/core.py:216-240.
* `residual_norm`     -- pkg/src/bandchol/core.py:186-213 (numpy restatement, same ops);
                         `residual_fast` is the C version for the large configs.
* `max_scaled_diff`   -- the parity metric |x-y|/max(|y|,1) of
                         pkg/tests/test_acceptance.py:49.

Pinned against the reference's own outputs in tests/test_oracle.py
(fixtures: tests/golden/, generator script tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


class OracleFailure(Exception):
    """The oracle met a non-positive pivot / diagonal; `.column` says where."""

    def __init__(self, kind: str, column: int):
        self.kind = kind
        self.column = int(column)
        super().__init__(f"{kind} at column {column}")


def build() -> str:
    """Compile band_oracle.c into oracle/liboracle.so (make, gcc)."""
    subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or (
                os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "band_oracle.c"))):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        i64, dp = ctypes.c_int64, ctypes.POINTER(ctypes.c_double)
        L.bco_fsum.argtypes = [dp, i64]
        L.bco_fsum.restype = ctypes.c_double
        for name in ("bco_factor_reference", "bco_factor_plain"):
            getattr(L, name).argtypes = [i64, i64, i64, dp]
            getattr(L, name).restype = i64
        L.bco_solve.argtypes = [i64, i64, i64, dp, dp, dp]
        L.bco_solve.restype = i64
        L.bco_residual.argtypes = [i64, i64, i64, dp, i64, dp]
        L.bco_residual.restype = ctypes.c_double
        L.bco_max_scaled_diff.argtypes = [i64, i64, i64, dp, i64, dp]
        L.bco_max_scaled_diff.restype = ctypes.c_double
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def fsum(values) -> float:
    v = np.ascontiguousarray(values, dtype=np.float64)
    return float(lib().bco_fsum(_ptr(v), v.size))


def factor_reference(n: int, kd: int, ldab: int, data: np.ndarray) -> np.ndarray:
    """In place on `data`; raises OracleFailure('NotPositiveDefinite', col)."""
    r = lib().bco_factor_reference(n, kd, ldab, _ptr(data))
    if r >= 0:
        raise OracleFailure("NotPositiveDefinite", r)
    return data


def factor_plain(n: int, kd: int, ldab: int, data: np.ndarray) -> np.ndarray:
    r = lib().bco_factor_plain(n, kd, ldab, _ptr(data))
    if r >= 0:
        raise OracleFailure("NotPositiveDefinite", r)
    return data


def factor_plain_batched(n: int, kd: int, ldab: int, data: np.ndarray, threads: int | None = None) -> np.ndarray:
    """factor_plain on every row of `data` (batch, >= ldab*n), in place, one matrix per host
    thread (ctypes drops the GIL).  Returns the per-matrix failing column, -1 = success."""
    from concurrent.futures import ThreadPoolExecutor
    assert data.ndim == 2 and data.shape[1] >= ldab * n and data.flags.c_contiguous
    L = lib()
    rows = [data[b] for b in range(data.shape[0])]
    workers = threads or max(1, min(32, os.cpu_count() or 1))
    with ThreadPoolExecutor(workers) as ex:
        res = list(ex.map(lambda row: L.bco_factor_plain(n, kd, ldab, _ptr(row)), rows))
    return np.asarray(res, dtype=np.int64)


def factor_blocked_dense(n: int, kd: int, ldab: int, data: np.ndarray, nb: int = 256) -> np.ndarray:
    """Right-looking blocked band Cholesky in numpy/scipy (multithreaded BLAS), in place --
    an independent fast checker for the wide configs (C3, C4), where the C loops take
    minutes.  A dense (kd+nb)-square window slides down the band: POTRF of its leading
    nb x nb block, TRSM of the rows below, SYRK/GEMM of the trailing window, exactly the
    tile algebra of blocked.py:259-284 at tile size nb.  Entries outside the band stay
    exact zeros (they only ever meet zero products).  Raises OracleFailure at the first
    non-positive pivot (column found by an unblocked pass over the failing block)."""
    import scipy.linalg as sla

    band = data.reshape(n, ldab)  # band[j, d] = A(j+d, j)
    w = kd + nb

    def load(win, j0, r_lo, r_hi):
        # entries (i, j), j0 <= j <= i, r_lo <= i < r_hi, of the untouched band into the
        # window whose (0, 0) is global (j0, j0)
        for j in range(j0, min(n, r_hi)):
            lo, hi = max(r_lo, j), min(r_hi, n, j + kd + 1)
            if hi > lo:
                win[lo - j0: hi - j0, j - j0] = band[j, lo - j: hi - j]

    win = np.zeros((w, w))
    load(win, 0, 0, w)
    j0 = 0
    while j0 < n:
        b = min(nb, n - j0)
        rows = min(w, n - j0)          # live rows/cols of the window
        a11 = np.tril(win[:b, :b])
        try:
            l11 = np.linalg.cholesky(a11 + np.tril(a11, -1).T)
            ok = bool(np.all(np.diag(l11) > 0))
        except np.linalg.LinAlgError:
            ok = False
        if not ok:
            # locate the failing column like reference.py:56-57 (`pivot > 0`, NaN fails)
            t = a11.copy()
            for c in range(b):
                p = t[c, c]
                if not (p > 0.0):
                    raise OracleFailure("NotPositiveDefinite", j0 + c)
                t[c, c] = np.sqrt(p)
                t[c + 1:, c] /= t[c, c]
                t[c + 1:, c + 1:] -= np.tril(np.outer(t[c + 1:, c], t[c + 1:, c]))
            raise OracleFailure("NotPositiveDefinite", j0 + b - 1)
        win[:b, :b] = l11
        if rows > b:
            l21 = sla.solve_triangular(l11, win[b:rows, :b].T, lower=True).T
            win[b:rows, :b] = l21
            win[b:rows, b:rows] -= l21 @ l21.T
        for j in range(j0, j0 + b):  # the finished columns back to the band
            m = min(kd, n - 1 - j)
            band[j, : m + 1] = win[j - j0: j - j0 + m + 1, j - j0]
        nxt = np.zeros((w, w))
        nxt[: w - b, : w - b] = np.tril(win[b:, b:])
        win = nxt
        load(win, j0 + b, j0 + w, j0 + b + w)
        j0 += b
    return data


def solve(n: int, kd: int, ldab: int, factor: np.ndarray, rhs: np.ndarray) -> np.ndarray:
    b = np.ascontiguousarray(rhs, dtype=np.float64)
    x = np.empty(n)
    r = lib().bco_solve(n, kd, ldab, _ptr(factor), _ptr(b), _ptr(x))
    if r >= 0:
        raise OracleFailure("SingularFactor", r)
    return x


def band_panel(n: int, kd: int, ldab: int, data: np.ndarray) -> np.ndarray:
    """(kd+1, n) copy with padding zeroed (core.py:120-125)."""
    p = data.reshape(n, ldab).T[: kd + 1].copy()
    for d in range(1, kd + 1):
        p[d, n - d:] = 0.0
    return p


def residual_norm(n: int, kd: int, a_data: np.ndarray, a_ld: int,
                  l_data: np.ndarray, l_ld: int) -> float:
    """Numpy restatement of core.py:186-213 (same operations, same order)."""
    a = band_panel(n, kd, a_ld, a_data)
    l = band_panel(n, kd, l_ld, l_data)
    recon = np.zeros_like(a)
    for d in range(0, kd + 1):
        for s in range(0, kd + 1 - d):
            recon[d, s:] += l[d + s, : n - s] * l[s, : n - s]
    diff = a - recon
    weights = np.full((kd + 1, 1), 2.0)
    weights[0, 0] = 1.0
    num = float(np.sum(weights * diff * diff))
    den = float(np.sum(weights * a * a))
    if den == 0.0:
        return 0.0 if num == 0.0 else float("inf")
    return float(np.sqrt(num / den))


def residual_fast(n: int, kd: int, a_data: np.ndarray, a_ld: int,
                  l_data: np.ndarray, l_ld: int) -> float:
    return float(lib().bco_residual(n, kd, a_ld, _ptr(a_data), l_ld, _ptr(l_data)))


def max_scaled_diff(n: int, kd: int, x: np.ndarray, ldx: int, y: np.ndarray, ldy: int) -> float:
    """max over in-band entries of |x-y| / max(|y|,1) (test_acceptance.py:49)."""
    return float(lib().bco_max_scaled_diff(n, kd, ldx, _ptr(x), ldy, _ptr(y)))
