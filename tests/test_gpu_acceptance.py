"""Config-scale parity gates on the GPU (BASELINE.json north_star), through the C ABI.

Mirrors the reference's shipping gates (pkg/tests/test_acceptance.py:34-61 sweep +
residual, :64-74 byte determinism) at the five BASELINE configs:
  * L elementwise: max over EVERY in-band entry of |L_gpu - L_ref| / max(|L_ref|, 1) <= 1e-10
    (test_acceptance.py:49's scale); L_ref from the oracle (C2/C5: oracle.factor_plain,
    pinned to the reference in tests/test_oracle.py; C3/C4: oracle.factor_blocked_dense,
    the blocked tile algebra in numpy, pinned in tests/test_oracle.py).
  * backward error ||A - L L^T||_F / ||A||_F <= 10 * n * eps, computed on the device
    (bcg_band_residual; C5: bcg_band_residual_batched, every member).
  * determinism: bitwise run to run for the one-CTA kernel (C5 shape) and the whole-GPU
    ticketed kernel (C2 shape).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import EPS, L_TOL, X_TOL, band_matvec_batched

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2305_04635_b200 as bc  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2305_04635_b200.inputs import CONFIGS, generate_spd, make_rhs  # noqa: E402


def _device_factor(a):
    n, k = a.dim, a.bandwidth
    dev = torch.from_numpy(a.data).cuda()
    orig = dev.clone()
    info = bc.dpbtrf_device(dev, n, k, k + 1)
    assert int(info.item()) == 0
    res = float(bc.band_residual_device(orig, dev, n, k, k + 1, k + 1).item())
    return dev.cpu().numpy(), res


@pytest.mark.parametrize("tag", ["C1", "C2", "C3", "C4"])
def test_single_config_full_l_and_backward_error(tag):
    cfg = CONFIGS[tag]
    a = cfg.matrix(0)
    n, k = cfg.dim, cfg.bandwidth
    got, res = _device_factor(a)
    assert res <= 10 * n * EPS, (tag, res)
    want = a.data.copy()
    if tag in ("C3", "C4"):
        oracle.factor_blocked_dense(n, k, k + 1, want)
    elif tag == "C1":
        oracle.factor_reference(n, k, k + 1, want)  # the bit-exact restatement
    else:
        oracle.factor_plain(n, k, k + 1, want)
    err = oracle.max_scaled_diff(n, k, got, k + 1, want, k + 1)
    assert err <= L_TOL, (tag, err)


def test_c5_every_member_l_and_backward_error():
    cfg = CONFIGS["C5"]
    n, k, B = cfg.dim, cfg.bandwidth, cfg.batch
    data = np.empty((B, (k + 1) * n))
    rhs = np.empty((B, n))
    for s in range(B):
        data[s] = generate_spd(n, k, s).data
        rhs[s] = make_rhs(n, s)
    dab = torch.from_numpy(data).cuda()
    orig = dab.clone()
    db = torch.from_numpy(rhs).cuda()
    info = bc.dpbsv_batched_device(dab, n, k, k + 1, db, B)
    assert not info.cpu().numpy().any()
    res = bc.band_residual_batched_device(orig, dab, n, k, k + 1, k + 1, B).cpu().numpy()
    assert res.shape == (B,) and float(res.max()) <= 10 * n * EPS, float(res.max())
    got = dab.cpu().numpy()
    want = data.copy()
    fail = oracle.factor_plain_batched(n, k, k + 1, want)
    assert (fail < 0).all()
    worst = max(oracle.max_scaled_diff(n, k, got[s], k + 1, want[s], k + 1) for s in range(B))
    assert worst <= L_TOL, worst
    x = db.cpu().numpy()
    r = band_matvec_batched(n, k, k + 1, data, x) - rhs
    assert (np.linalg.norm(r, axis=1) / np.linalg.norm(rhs, axis=1)).max() <= 1e-10
    for s in (0, 511, 1023):
        xs = oracle.solve(n, k, k + 1, want[s], rhs[s])
        assert np.linalg.norm(x[s] - xs) <= X_TOL * np.linalg.norm(xs)


def test_batched_residual_matches_single():
    n, k, B = 1000, 60, 5
    data = np.stack([generate_spd(n, k, s).data for s in range(B)])
    fac = data.copy()
    oracle.factor_plain_batched(n, k, k + 1, fac)
    fac[3] *= 1.0 + 1e-6  # a perturbed member: a residual well above rounding
    a_d, l_d = torch.from_numpy(data).cuda(), torch.from_numpy(fac).cuda()
    batched = bc.band_residual_batched_device(a_d, l_d, n, k, k + 1, k + 1, B).cpu().numpy()
    for s in range(B):
        one = float(bc.band_residual_device(a_d[s], l_d[s], n, k, k + 1, k + 1).item())
        want = oracle.residual_norm(n, k, data[s], k + 1, fac[s], k + 1)
        assert abs(batched[s] - one) <= 1e-12 * max(one, 1e-300) or abs(batched[s] - one) <= 1e-20
        assert abs(batched[s] - want) <= 1e-9 * max(want, 1e-16) + 1e-15


def test_multi_cta_determinism_bitwise_c2():
    """The whole-GPU kernel (ticketed workers) gives byte-identical L run to run."""
    cfg = CONFIGS["C2"]
    a = cfg.matrix(0)
    n, k = cfg.dim, cfg.bandwidth
    outs = []
    for _ in range(3):
        dev = torch.from_numpy(a.data).cuda()
        assert int(bc.dpbtrf_device(dev, n, k, k + 1).item()) == 0
        outs.append(dev.cpu().numpy().tobytes())
    assert outs[0] == outs[1] == outs[2]


def test_cta_kernel_determinism_bitwise_c5_shape():
    n, k, B = 4096, 100, 8
    data = np.stack([generate_spd(n, k, s).data for s in range(B)])
    outs = []
    for _ in range(3):
        dev = torch.from_numpy(data).cuda()
        assert not bc.dpbtrf_batched_device(dev, n, k, k + 1, B).cpu().numpy().any()
        outs.append(dev.cpu().numpy().tobytes())
    assert outs[0] == outs[1] == outs[2]
