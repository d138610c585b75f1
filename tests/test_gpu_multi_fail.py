"""Failure and abort paths of the whole-GPU factorization kernel (kd >= 160: band_multi.cuh).

A non-positive or NaN pivot anywhere must come back as the reference's
NotPositiveDefinite(column) with the FIRST failing global column (reference.py:56-57,
test_blocked.py:396-402) and the kernel must terminate: every worker spin polls the abort
word the pivot CTA sets (band_multi.cuh spin_ge).  The same workspace then factors a
healthy matrix to exactly the bytes of a fresh run (the launch clears the flags).
Both geometries run: 8-warp workers (kd < 1000) and the 4-group wide-band workers.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2305_04635_b200 as bc  # noqa: E402
from paper_2305_04635_b200 import _lib  # noqa: E402
from paper_2305_04635_b200.inputs import generate_spd  # noqa: E402

# (n, kd): 32-column tiles; columns at a tile edge, mid-tile, first and last
GEOMS = [(3000, 200), (4000, 1000)]


def _cols(n):
    return [0, 1, 31, 32, 33, 63, 64, n // 2, n // 2 + 17, n - 33, n - 32, n - 2, n - 1]


def _factor_on(ws, a, n, k):
    dev = torch.from_numpy(a.copy()).cuda()
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    rc = _lib.load().bcg_dpbtrf(n, k, dev.data_ptr(), k + 1, info.data_ptr(), ws.data_ptr(), ws.numel(),
                                torch.cuda.current_stream().cuda_stream)
    _lib.check(rc, "bcg_dpbtrf")
    torch.cuda.synchronize()
    return int(info.item()), dev.cpu().numpy()


@pytest.mark.parametrize("n,k", GEOMS)
def test_negative_pivot_columns_and_workspace_reuse(n, k):
    assert _lib.load().bcg_dpbtrf_workspace_size(n, k, k + 1) > 0  # the whole-GPU kernel
    base = generate_spd(n, k, 1).data
    ws = torch.zeros(int(_lib.load().bcg_dpbtrf_workspace_size(n, k, k + 1)), dtype=torch.uint8, device="cuda")
    good_info, good = _factor_on(ws, base, n, k)
    assert good_info == 0
    for col in _cols(n):
        bad = base.copy()
        bad[col * (k + 1)] = -1.0
        info, _ = _factor_on(ws, bad, n, k)
        assert info == col + 1, (n, k, col, info)
    # the same workspace after the aborted runs: exactly the healthy result
    info, again = _factor_on(ws, base, n, k)
    assert info == 0 and again.tobytes() == good.tobytes()


@pytest.mark.parametrize("n,k", GEOMS)
def test_nan_pivot_and_first_failure_wins(n, k):
    base = generate_spd(n, k, 2).data
    bad = base.copy()
    bad[777 * (k + 1)] = float("nan")
    with pytest.raises(bc.NotPositiveDefinite) as err:
        bc.factor_blocked_serial(bc.BandedMatrix(n, k, data=bad))
    assert err.value.column == 777
    two = base.copy()
    two[900 * (k + 1)] = -1.0
    two[(n - 5) * (k + 1)] = -1.0
    with pytest.raises(bc.NotPositiveDefinite) as err:
        bc.factor_blocked_serial(bc.BandedMatrix(n, k, data=two))
    assert err.value.column == 900


def test_batched_whole_gpu_path_reports_member():
    """Batched matrices too wide for one CTA run the whole-GPU kernel one after another on
    the caller's workspace; a failing member is reported by index and column."""
    n, k = 2000, 200
    data = np.stack([generate_spd(n, k, s).data for s in range(3)])
    data[1, 1234 * (k + 1)] = -2.0
    with pytest.raises(bc.NotPositiveDefinite) as err:
        bc.factor_batched(data, n, k)
    assert err.value.matrix == 1 and err.value.column == 1234


@pytest.mark.parametrize("n,k", GEOMS)
def test_row_owner_and_per_link_scheduling_agree(n, k, monkeypatch):
    """Row-owner scheduling (one worker group runs a row's whole TRSM/update chain) and the
    one-ticket-per-link fallback (grids without spare groups; forced with BCG_MULTI_NO_OWNER)
    apply the same updates in the same order: identical bytes, and failures come back alike."""
    base = generate_spd(n, k, 4).data
    ws = torch.zeros(int(_lib.load().bcg_dpbtrf_workspace_size(n, k, k + 1)), dtype=torch.uint8, device="cuda")
    info_o, with_owner = _factor_on(ws, base, n, k)
    monkeypatch.setenv("BCG_MULTI_NO_OWNER", "1")
    info_l, per_link = _factor_on(ws, base, n, k)
    assert info_o == 0 and info_l == 0
    assert with_owner.tobytes() == per_link.tobytes()
    bad = base.copy()
    col = n // 2 + 5
    bad[col * (k + 1)] = float("nan")
    info, _ = _factor_on(ws, bad, n, k)
    assert info == col + 1
