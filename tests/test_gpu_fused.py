"""GPU parity of the fused factor + forward sweep and the backward-only sweep (the two halves
of bcg_dpbsv_batched's fused path: band_cta.cuh forward_head / forward_tail, band_sweep.cuh
with y0), through the C ABI.

Reference: factor_blocked_serial (pkg/src/bandchol/blocked.py:363-385) followed by
solve_with_factor (pkg/src/bandchol/core.py:216-240), whose forward loop (:231-235) produces
y and whose backward loop (:236-239) produces x.  Oracle: L from oracle.factor_plain, y from
a banded triangular solve of L y = b (scipy), x from oracle.solve.  Tolerances: L as everywhere
(1e-10 scaled), ||y - y_ref|| / ||y_ref|| and ||x - x_ref|| / ||x_ref|| <= 1e-10.
Covers block-edge shapes (n not a multiple of 16, kd = 32 .. the widest one-CTA window),
b left untouched by the first half, failed members (y only partly written, b untouched, info
kept by the second half), and the unfused fallback of bcg_dpbsv_batched (no workspace) giving
the same x.
"""

from __future__ import annotations

import numpy as np
import pytest
from scipy.linalg import solve_banded

from conftest import L_TOL, X_TOL

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2305_04635_b200 as bc  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2305_04635_b200 import _lib  # noqa: E402
from paper_2305_04635_b200.inputs import generate_spd, make_rhs  # noqa: E402


def _rel(x, want):
    return np.linalg.norm(x - want) / max(np.linalg.norm(want), 1e-300)


def _batch(n, k, batch, seed0=0):
    data = np.stack([generate_spd(n, k, seed0 + s).data for s in range(batch)])
    rhs = np.stack([make_rhs(n, seed0 + s) for s in range(batch)])
    return data, rhs


def _forward_ref(n, k, factor, b):
    """y with L y = b, L in lower band storage (column j at factor[j*(k+1):...])."""
    ab = factor.reshape(n, k + 1).T.copy()  # ab[d, j] = L(j + d, j)
    return solve_banded((k, 0), ab, b)


@pytest.mark.parametrize("n,k", [(33, 32), (100, 32), (640, 100), (777, 64), (1000, 37), (1500, 130), (4096, 100),
                                 (2001, 99)])
def test_fused_forward_then_backward(n, k):
    batch = 3
    data, rhs = _batch(n, k, batch, 20)
    assert _lib.load().bcg_dpbsv_batched_workspace_size(n, k, k + 1, batch) == batch * n * 8  # the fused path
    dab = torch.from_numpy(data.copy()).cuda()
    db = torch.from_numpy(rhs.copy()).cuda()
    dy = torch.full((batch, n), np.nan, dtype=torch.float64, device="cuda")
    info = bc.dpbtrf_fwd_batched_device(dab.view(-1), n, k, k + 1, db.view(-1), dy.view(-1), batch)
    assert int(info.abs().sum().item()) == 0
    assert np.array_equal(db.cpu().numpy(), rhs)  # b is only read
    L, y = dab.cpu().numpy(), dy.cpu().numpy()
    dx = torch.full((batch, n), np.nan, dtype=torch.float64, device="cuda")
    bc.dpbtrs_bwd_batched_device(dab.view(-1), n, k, k + 1, dy.view(-1), dx.view(-1), batch, info)
    x = dx.cpu().numpy()
    for s in range(batch):
        want = data[s].copy()
        oracle.factor_plain(n, k, k + 1, want)
        assert oracle.max_scaled_diff(n, k, L[s], k + 1, want, k + 1) <= L_TOL
        assert _rel(y[s], _forward_ref(n, k, want, rhs[s])) <= X_TOL, (n, k, s)
        assert _rel(x[s], oracle.solve(n, k, k + 1, want, rhs[s])) <= X_TOL, (n, k, s)


def test_fused_failed_member():
    n, k, batch = 900, 64, 4
    data, rhs = _batch(n, k, batch, 3)
    data[1, 500 * (k + 1)] = -2.0  # pivot of column 500 of member 1
    dab = torch.from_numpy(data.copy()).cuda()
    db = torch.from_numpy(rhs.copy()).cuda()
    dy = torch.zeros((batch, n), dtype=torch.float64, device="cuda")
    info = bc.dpbtrf_fwd_batched_device(dab.view(-1), n, k, k + 1, db.view(-1), dy.view(-1), batch)
    assert info.cpu().tolist() == [0, 501, 0, 0]
    dx = torch.full((batch, n), 7.0, dtype=torch.float64, device="cuda")
    bc.dpbtrs_bwd_batched_device(dab.view(-1), n, k, k + 1, dy.view(-1), dx.view(-1), batch, info)
    assert info.cpu().tolist() == [0, 501, 0, 0]  # the second half keeps the factorization's verdict
    x = dx.cpu().numpy()
    assert np.all(x[1] == 7.0)  # a failed member's x is left alone
    for s in (0, 2, 3):
        want = data[s].copy()
        oracle.factor_plain(n, k, k + 1, want)
        assert _rel(x[s], oracle.solve(n, k, k + 1, want, rhs[s])) <= X_TOL
    # the forward sweep of the failed member stopped with its factorization: the blocks before
    # the failing one hold the right y (the reference's y for the leading columns)
    lead = 496
    good = generate_spd(n, k, 3 + 1).data.copy()
    oracle.factor_plain(n, k, k + 1, good)
    y_ref = _forward_ref(n, k, good, rhs[1])
    assert _rel(dy.cpu().numpy()[1, :lead], y_ref[:lead]) <= X_TOL


def test_dpbsv_fused_equals_unfused():
    """bcg_dpbsv_batched with the y workspace (fused) and without (factorization, then the
    two-sweep solve): the same L bit for bit, x within the solve tolerance of each other."""
    n, k, batch = 2048, 100, 5
    data, rhs = _batch(n, k, batch, 40)
    lib = _lib.load()
    out = []
    for fused in (True, False):
        dab = torch.from_numpy(data.copy()).cuda()
        db = torch.from_numpy(rhs.copy()).cuda()
        info = torch.zeros(batch, dtype=torch.int32, device="cuda")
        ws = torch.empty(batch * n, dtype=torch.float64, device="cuda") if fused else None
        rc = lib.bcg_dpbsv_batched(n, k, dab.data_ptr(), k + 1, (k + 1) * n, db.data_ptr(), n, batch, info.data_ptr(),
                                   ws.data_ptr() if fused else None, batch * n * 8 if fused else 0, None)
        torch.cuda.synchronize()
        assert rc == 0 and int(info.abs().sum().item()) == 0
        out.append((dab.cpu().numpy(), db.cpu().numpy()))
    assert out[0][0].tobytes() == out[1][0].tobytes()
    for s in range(batch):
        assert _rel(out[0][1][s], out[1][1][s]) <= X_TOL


def test_fused_deterministic():
    n, k, batch = 4096, 100, 8
    data, rhs = _batch(n, k, batch, 7)
    runs = []
    for _ in range(2):
        a, b = data.copy(), rhs.copy()
        bc.factor_solve_batched(a, b, n, k)
        runs.append((a.tobytes(), b.tobytes()))
    assert runs[0] == runs[1]


def test_split_entry_points_reject_unsupported_geometry():
    lib = _lib.load()
    d = torch.zeros(64, dtype=torch.float64, device="cuda")
    i = torch.zeros(1, dtype=torch.int32, device="cuda")
    # kd < 32: the lock-step one-CTA kernel has no fused forward sweep
    assert lib.bcg_dpbtrf_fwd_batched(40, 8, d.data_ptr(), 9, 360, d.data_ptr(), 40, 1, i.data_ptr(), d.data_ptr(), None) < 0
    assert lib.bcg_dpbsv_batched_workspace_size(40, 8, 9, 1) == 0
