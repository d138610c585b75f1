"""GPU side of SURVEY §8(f): device residual (item 4), BNDM straight to device (item 3),
the CSV harness end to end (item 2)."""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import L_TOL

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2305_04635_b200 as bc  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2305_04635_b200 import harness  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("n,k,ld", [(1, 0, 1), (2, 1, 2), (37, 5, 8), (300, 16, 17), (1000, 50, 51),
                                    (513, 130, 140)])
def test_device_residual_matches_oracle(n, k, ld):
    a = bc.generate_spd(n, k, seed=n)
    if ld != k + 1:
        b = bc.BandedMatrix(n, k, ld)
        b.data.reshape(n, ld)[:, : k + 1] = a.data.reshape(n, k + 1)
        a = b
    lf = a.copy()
    oracle.factor_plain(n, k, ld, lf.data)
    # at the exact factor both values are rounding noise of recon itself (~eps): bound them
    bound = 10 * n * np.finfo(float).eps
    assert bc.residual_norm(a, lf) <= bound
    assert oracle.residual_norm(n, k, a.data, ld, lf.data, ld) <= bound
    # a perturbed factor gives a well-conditioned residual: device == restated reference
    rng = np.random.default_rng(n)
    lf.data[:] *= 1.0 + 1e-6 * rng.standard_normal(lf.data.size)
    want = oracle.residual_norm(n, k, a.data, ld, lf.data, ld)
    got = bc.residual_norm(a, lf)
    assert want > 1e-8
    assert abs(got - want) <= 1e-9 * want


def test_device_residual_zero_and_deterministic():
    a = bc.BandedMatrix(8, 2)
    assert bc.residual_norm(a, a.copy()) == 0.0
    b = bc.generate_spd(3000, 64, seed=1)
    f = bc.factor_blocked_serial(b.copy())
    r1, r2 = bc.residual_norm(b, f), bc.residual_norm(b, f)
    assert r1 == r2


def test_fixture_to_device_factor():
    dev, n, k, ld = bc.load_matrix_device(os.path.join(GOLDEN, "fixture_ref.bndm"))
    assert (n, k, ld) == (37, 5, 8) and dev.is_cuda
    want = bc.load_matrix(os.path.join(GOLDEN, "fixture_ref.bndm"))
    assert np.array_equal(dev.cpu().numpy(), want.data)
    info = bc.dpbtrf_device(dev, n, k, ld)
    assert int(info.item()) == 0
    ref = want.data.copy()
    oracle.factor_reference(n, k, ld, ref)
    assert oracle.max_scaled_diff(n, k, dev.cpu().numpy(), ld, ref, ld) <= L_TOL


def test_harness_end_to_end(tmp_path):
    cfg = harness.BenchConfig(dim=2000, bandwidths=(7, 50, 200), repetitions=3, check=True)
    recs = harness.run_benchmark(cfg)
    assert [(r.bandwidth, r.impl) for r in recs] == [(k, i) for k in (7, 50, 200) for i in harness.IMPL_CHOICES]
    for r in recs:
        assert not r.failed and r.median_seconds > 0 and r.gflops > 0
        assert r.residual <= harness.RESIDUAL_LIMIT
    out = tmp_path / "gpu.csv"
    harness.emit_csv(recs, out)
    assert harness.parse_csv(out) == recs
    assert harness.main(["--dim", "500", "--bandwidths", "9", "--reps", "2", "--check",
                         "--out", str(tmp_path / "cli.csv")]) == 0


def test_device_primitives_reject_bad_buffers():
    n, k = 64, 4
    ab = torch.zeros((k + 1) * n, dtype=torch.float64, device="cuda")
    with pytest.raises(bc.ShapeMismatch):
        bc.dpbtrf_device(ab[: -1], n, k, k + 1)  # too small
    with pytest.raises(bc.ShapeMismatch):
        bc.dpbtrf_device(ab.float(), n, k, k + 1)  # wrong dtype
    with pytest.raises(bc.ShapeMismatch):
        bc.dpbtrf_device(ab.cpu(), n, k, k + 1)  # host memory
    with pytest.raises(bc.ShapeMismatch):
        bc.dpbtrf_batched_device(ab, n, k, k + 1, 2)  # batch larger than the buffer
    b = torch.zeros(n, dtype=torch.float64, device="cuda")
    with pytest.raises(bc.ShapeMismatch):
        bc.dpbtrs_device(ab, n, k, k + 1, b, nrhs=2)
    with pytest.raises(bc.ShapeMismatch):
        bc.dpbsv_batched_device(ab, n, k, k + 1, b, 1, info=torch.zeros(1, dtype=torch.int64, device="cuda"))
