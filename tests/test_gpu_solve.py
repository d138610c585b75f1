"""GPU parity of the streamed solve (band_sweep.cuh) through the C ABI, against the oracle.

The reference solve is solve_with_factor (pkg/src/bandchol/core.py:216-240); the oracle
restates it in C (oracle/band_oracle.c bco_solve).  Tolerance (pkg/tests/test_core.py:214-220):
  ||x_gpu - x_ref|| / ||x_ref|| <= 1e-10   for every right-hand side.
Covers: block-edge shapes and band widths (kd 0 .. the widest streamed ring, and the
wide-band fallback kernel), several right-hand sides per factor (one pass over L per group
of up to 16: nrhs 1..33), the batched multi-rhs entry point, failed members of a batched
factor + solve keeping b untouched (LAPACK dpbsv), and determinism.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import X_TOL

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2305_04635_b200 as bc  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2305_04635_b200.inputs import generate_spd, make_rhs  # noqa: E402


def _factor(n, k, seed):
    a = generate_spd(n, k, seed)
    oracle.factor_plain(n, k, k + 1, a.data)
    return a


def _rel(x, want):
    return np.linalg.norm(x - want) / max(np.linalg.norm(want), 1e-300)


@pytest.mark.parametrize("n,k", [(1, 0), (5, 0), (16, 3), (17, 16), (31, 30), (33, 1), (100, 15), (257, 16),
                                 (300, 17), (301, 31), (500, 32), (640, 63), (1000, 64), (777, 100), (4096, 100),
                                 (1500, 130), (3000, 255), (2000, 300), (20000, 200), (5000, 500)])
def test_solve_shapes(n, k):
    a = _factor(n, k, 11)
    for s in (0, 1):
        b = make_rhs(n, s)
        x = bc.solve_with_factor(a, b)
        assert _rel(x, oracle.solve(n, k, k + 1, a.data, b)) <= X_TOL, (n, k, s)


@pytest.mark.parametrize("nrhs", [1, 2, 3, 5, 8, 9, 16, 17, 33])
def test_multi_rhs_one_factor(nrhs):
    n, k = 3000, 100
    a = _factor(n, k, 9)
    B = np.stack([make_rhs(n, 40 + s) for s in range(nrhs)])
    X = bc.solve_many(a, B)
    for s in range(nrhs):
        assert _rel(X[s], oracle.solve(n, k, k + 1, a.data, B[s])) <= X_TOL, s


@pytest.mark.parametrize("n,k,nrhs", [(1000, 40, 4), (777, 100, 16), (4096, 100, 3), (513, 7, 16)])
def test_batched_multi_rhs(n, k, nrhs):
    batch = 5
    fac = np.stack([_factor(n, k, s).data for s in range(batch)])
    rhs = np.stack([np.stack([make_rhs(n, 100 * m + s) for s in range(nrhs)]) for m in range(batch)])
    X = bc.solve_batched(fac, rhs, n, k)
    for m in range(batch):
        for s in range(nrhs):
            assert _rel(X[m, s], oracle.solve(n, k, k + 1, fac[m], rhs[m, s])) <= X_TOL, (m, s)


def test_multi_rhs_padded_lead_dim_and_ldb():
    """ldab > kd + 1 and a right-hand-side stride larger than n, through the device API."""
    n, k, ld, R, ldb = 1000, 50, 57, 6, 1003
    a = bc.BandedMatrix(n, k, ld)
    a.data.reshape(n, ld)[:, : k + 1] = generate_spd(n, k, 3).data.reshape(n, k + 1)
    oracle.factor_plain(n, k, ld, a.data)
    B = np.zeros((R, ldb))
    for s in range(R):
        B[s, :n] = make_rhs(n, s)
    dab = torch.from_numpy(a.data).cuda()
    db = torch.from_numpy(B.copy()).cuda()
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    from paper_2305_04635_b200 import _lib
    rc = _lib.load().bcg_dpbtrs(n, k, dab.data_ptr(), ld, db.data_ptr(), ldb, R, info.data_ptr(),
                                torch.cuda.current_stream().cuda_stream)
    assert rc == 0 and int(info.item()) == 0
    got = db.cpu().numpy()
    for s in range(R):
        assert _rel(got[s, :n], oracle.solve(n, k, ld, a.data, B[s, :n])) <= X_TOL
        assert np.array_equal(got[s, n:], B[s, n:])  # the gap between columns is not written


def test_singular_factor_leaves_rhs():
    n, k = 900, 60
    a = _factor(n, k, 2)
    a.data[517 * (k + 1)] = 0.0
    b = make_rhs(n, 0)
    with pytest.raises(bc.SingularFactor):
        bc.solve_with_factor(a, b)
    dab = torch.from_numpy(a.data).cuda()
    db = torch.from_numpy(b.copy()).cuda()
    info = bc.dpbtrs_device(dab, n, k, k + 1, db)
    assert int(info.item()) == 518
    assert np.array_equal(db.cpu().numpy(), b)


@pytest.mark.parametrize("n,k", [(600, 30), (640, 100), (2000, 200)])
def test_dpbsv_failed_member_keeps_b(n, k):
    batch = 4
    data = np.stack([generate_spd(n, k, s).data for s in range(batch)])
    rhs = np.stack([make_rhs(n, s) for s in range(batch)])
    data[2, 333 * (k + 1)] = -5.0
    a0, b0 = data.copy(), rhs.copy()
    with pytest.raises(bc.NotPositiveDefinite) as err:
        bc.factor_solve_batched(data, rhs, n, k)
    assert err.value.matrix == 2 and err.value.column == 333
    assert np.array_equal(rhs[2], b0[2])  # LAPACK dpbsv: B unchanged when info > 0
    for s in (0, 1, 3):
        want = a0[s].copy()
        oracle.factor_plain(n, k, k + 1, want)
        assert _rel(rhs[s], oracle.solve(n, k, k + 1, want, b0[s])) <= X_TOL


def test_solve_deterministic():
    n, k = 4096, 100
    a = _factor(n, k, 5)
    b = make_rhs(n, 5)
    one = bc.solve_with_factor(a, b)
    two = bc.solve_with_factor(a, b)
    assert one.tobytes() == two.tobytes()
    B = np.stack([make_rhs(n, s) for s in range(16)])
    X1 = bc.solve_many(a, B)
    X2 = bc.solve_many(a, B)
    assert X1.tobytes() == X2.tobytes()
