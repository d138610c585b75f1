"""The pipelined one-CTA factorization (kd >= 32: pivot / worker / light warp roles,
mbarrier dataflow) on the paths the golden cases do not reach: failing pivots at the first,
a middle, a block-boundary and the last column (negative and NaN), failures inside a batch
(every matrix keeps its own info, the others stay exact), the fused solve with a failing
member, and shapes whose last block is short or whose window copies take the element-wise
path (odd ldab with an odd tail)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import L_TOL, X_TOL

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2305_04635_b200 as bc  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2305_04635_b200.inputs import generate_spd, make_rhs  # noqa: E402


@pytest.mark.parametrize("n,k,col,bad", [(300, 32, 0, -1.0), (300, 32, 150, -1.0), (300, 32, 299, -1.0),
                                         (777, 64, 400, float("nan")), (1000, 100, 15, -1.0),
                                         (1000, 100, 16, -1.0), (1000, 100, 999, float("nan")),
                                         (4096, 100, 2000, -3.0)])
def test_pipelined_failure_column(n, k, col, bad):
    a = generate_spd(n, k, 3)
    a.set(col, col, bad)
    with pytest.raises(bc.NotPositiveDefinite) as err:
        bc.factor_blocked_serial(a)
    assert err.value.column == col


def test_pipelined_batch_failures_are_per_matrix():
    n, k, B = 1500, 100, 9
    data = np.stack([generate_spd(n, k, s).data for s in range(B)])
    fails = {2: 0, 5: 731, 7: 1499}
    for m, c in fails.items():
        data[m, c * (k + 1)] = -1.0
    dev = torch.from_numpy(data.copy()).cuda()
    info = bc.dpbtrf_batched_device(dev, n, k, k + 1, B)
    got = info.cpu().numpy()
    out = dev.cpu().numpy()
    for m in range(B):
        if m in fails:
            assert got[m] == fails[m] + 1, (m, got[m])
        else:
            assert got[m] == 0
            want = data[m].copy()
            oracle.factor_plain(n, k, k + 1, want)
            assert oracle.max_scaled_diff(n, k, out[m], k + 1, want, k + 1) <= L_TOL, m


def test_pipelined_fused_solve_with_failing_member():
    n, k, B = 2048, 100, 6
    data = np.stack([generate_spd(n, k, s).data for s in range(B)])
    rhs = np.stack([make_rhs(n, s) for s in range(B)])
    data[4, 1000 * (k + 1)] = -2.0
    dev, dvb = torch.from_numpy(data.copy()).cuda(), torch.from_numpy(rhs.copy()).cuda()
    info = bc.dpbsv_batched_device(dev, n, k, k + 1, dvb, B).cpu().numpy()
    assert info[4] == 1001 and all(info[m] == 0 for m in range(B) if m != 4)
    x = dvb.cpu().numpy()
    for m in range(B):
        if m == 4:
            continue
        want = data[m].copy()
        oracle.factor_plain(n, k, k + 1, want)
        xs = oracle.solve(n, k, k + 1, want, rhs[m])
        assert np.linalg.norm(x[m] - xs) <= X_TOL * np.linalg.norm(xs), m


@pytest.mark.parametrize("n,k,ld", [(257, 100, 101), (1001, 40, 41), (999, 63, 64), (1000, 33, 40), (130, 100, 101)])
def test_pipelined_odd_shapes_factor_and_solve(n, k, ld):
    a0 = generate_spd(n, k, n)
    a = bc.BandedMatrix(n, k, ld)
    a.data.reshape(n, ld)[:, :k + 1] = a0.data.reshape(n, k + 1)
    want = a.data.copy()
    oracle.factor_plain(n, k, ld, want)
    data = a.data.copy()[None]
    b = make_rhs(n, 1)[None].copy()
    dev, dvb = torch.from_numpy(data.copy()).cuda(), torch.from_numpy(b.copy()).cuda()
    info = bc.dpbsv_batched_device(dev, n, k, ld, dvb, 1).cpu().numpy()
    assert info[0] == 0
    out = dev.cpu().numpy()[0]
    assert oracle.max_scaled_diff(n, k, out, ld, want, ld) <= L_TOL
    pad = np.ones(ld * n, dtype=bool)
    for j in range(n):
        pad[j * ld: j * ld + min(k, n - 1 - j) + 1] = False
    assert np.array_equal(out[pad], data[0][pad])  # padding untouched
    xs = oracle.solve(n, k, ld, want, b[0])
    assert np.linalg.norm(dvb.cpu().numpy()[0] - xs) <= X_TOL * np.linalg.norm(xs)


@pytest.mark.parametrize("k", [100, 50, 64, 128])
def test_compile_time_geometry_matches_runtime_geometry(k):
    """kd in {50, 64, 100, 128} with ldab = kd + 1 runs a GeomFixed<kd> instantiation, a padded
    ldab the runtime one: the same arithmetic in the same order, so L must agree bit for bit."""
    n, B = 1200, 5
    data = np.stack([generate_spd(n, k, s).data for s in range(B)])
    a = torch.from_numpy(data.copy()).cuda()
    assert int(bc.dpbtrf_batched_device(a, n, k, k + 1, B).abs().sum().item()) == 0
    ld = k + 3
    padded = np.zeros((B, ld * n))
    padded.reshape(B, n, ld)[:, :, :k + 1] = data.reshape(B, n, k + 1)
    p = torch.from_numpy(padded).cuda()
    assert int(bc.dpbtrf_batched_device(p, n, k, ld, B).abs().sum().item()) == 0
    got = a.cpu().numpy().reshape(B, n, k + 1)
    ref = p.cpu().numpy().reshape(B, n, ld)[:, :, :k + 1]
    assert np.array_equal(got, ref)
