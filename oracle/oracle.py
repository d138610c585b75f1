"""CPU oracle for the band Cholesky path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module; it is the checker, never the thing
measured or shipped.  The product package (paper_2305_04635_b200) never imports
it and has no CPU fallback.

* `factor_reference`  -- bit-exact restatement of pkg/src/bandchol/reference.py:32-63
                         (C, exactly rounded sums; band_oracle.c).
* `factor_plain`      -- same recurrence, ordinary rounding, fast (large configs).
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
