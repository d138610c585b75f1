"""The C-ABI library loads and exports every symbol include/bandchol_b200.h declares.

No compute calls here (no GPU in the build container): only argument validation,
which returns before any CUDA work, and the workspace query.
"""

from __future__ import annotations

import ctypes
import os
import re

import pytest

from paper_2305_04635_b200 import _lib

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
HEADER = os.path.join(ROOT, "include", "bandchol_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(bcg_\w+)\s*\(", text)))


def test_library_built():
    assert os.path.exists(_lib.LIB_PATH), "run __graft_entry__.build()"


def test_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 8
    for name in syms:
        assert hasattr(lib, name), name
    assert set(syms) == set(_lib.SIGNATURES), "ctypes signatures out of sync with the header"


def test_version_and_argument_validation():
    lib = _lib.load()
    assert lib.bcg_version() >= 100
    # n < 1 -> -1, kd >= n -> -2, ldab < kd+1 -> -4 (LAPACK-style illegal argument codes)
    assert lib.bcg_dpbtrf(0, 0, None, 1, None, None, 0, None) == -1
    assert lib.bcg_dpbtrf(10, 10, None, 11, None, None, 0, None) == -2
    assert lib.bcg_dpbtrf(10, 3, None, 3, None, None, 0, None) == -4
    assert lib.bcg_dpbtrf(10, 3, None, 4, None, None, 0, None) == -3
    assert b"ab is NULL" in lib.bcg_last_error()
    assert lib.bcg_dpbtrf_batched(10, 3, ctypes.c_void_p(8), 4, 39, 1, None, None, 0, None) == -5
    assert lib.bcg_dpbtrs(10, 3, ctypes.c_void_p(8), 4, None, 10, 1, None, None) == -5
    assert lib.bcg_dpbsv_batched(10, 3, ctypes.c_void_p(8), 4, 40, ctypes.c_void_p(8), 9, 1, None, None, 0,
                                 None) == -7
    # multi-rhs batched: ldb < n, then a stride_b that cannot hold nrhs columns
    assert lib.bcg_dpbtrs_batched_nrhs(10, 3, ctypes.c_void_p(8), 4, 40, ctypes.c_void_p(8), 9, 100, 2, 1,
                                       None, None) == -7
    assert lib.bcg_dpbtrs_batched_nrhs(10, 3, ctypes.c_void_p(8), 4, 40, ctypes.c_void_p(8), 10, 19, 2, 1,
                                       None, None) == -8
    assert lib.bcg_band_residual_batched(10, 3, ctypes.c_void_p(8), 4, 39, ctypes.c_void_p(8), 4, 40, 1,
                                         ctypes.c_void_p(8), None, 0, None) == -5


def test_error_mapping():
    with pytest.raises(Exception) as err:
        _lib.check(-2, "bcg_dpbtrf")
    assert "illegal argument 2" in str(err.value)


def test_workspace_query_is_pure():
    lib = _lib.load()
    for (n, kd) in [(2000, 50), (20000, 200), (50000, 500), (20000, 2000)]:
        ws = lib.bcg_dpbtrf_workspace_size(n, kd, kd + 1)
        assert ws >= 0
    assert lib.bcg_dpbtrf_workspace_size(10, 10, 11) == 0
    # batched: one CTA per matrix up to the shared-memory window, the whole-GPU kernel beyond
    assert lib.bcg_dpbtrf_batched_workspace_size(4096, 100, 101, 1024) == 0
    assert lib.bcg_dpbtrf_batched_workspace_size(20000, 2000, 2001, 2) > 0
    assert lib.bcg_band_residual_batched_workspace_size(1024) == 1024 * 4 * 2 * 8
