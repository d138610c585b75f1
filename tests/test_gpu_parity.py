"""GPU parity: the CUDA path (through the C ABI) against the oracle and the reference's outputs.

Tolerances (BASELINE.json north_star), written here where they are checked:
  * L:  max |L_gpu - L_ref| / max(|L_ref|, 1) <= 1e-10   (pkg/tests/test_acceptance.py:49)
  * backward error ||A - L L^T||_F / ||A||_F <= 10 * n * eps
  * solve: ||x_gpu - x_ref|| / ||x_ref|| <= 1e-10        (pkg/tests/test_core.py:214-220)
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import EPS, L_TOL, X_TOL, band_matvec, band_matvec_batched, scaled_diff, sha

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2305_04635_b200 as bc  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2305_04635_b200.inputs import generate_spd, generate_spd_wide, make_rhs  # noqa: E402


def _cases(golden_meta):
    return sorted(golden_meta["cases"].items())


def test_library_is_the_engine():
    import ctypes
    assert bc.library_version() >= 100
    # the loaded object is our in-tree library
    from paper_2305_04635_b200 import _lib
    assert isinstance(_lib.load(), ctypes.CDLL)


def test_small_cases_vs_reference(golden_meta, small):
    for name, meta in _cases(golden_meta):
        n, k, ld = meta["n"], meta["k"], meta["lead_dim"]
        m = bc.BandedMatrix(n, k, ld, small[f"{name}/A"].copy())
        out = bc.factor_blocked_serial(m)
        assert out is m  # in place, same object (blocked.py:385)
        want = small[f"{name}/L_ref"]
        err = oracle.max_scaled_diff(n, k, m.data, ld, want, ld)
        assert err <= L_TOL, (name, err)
        # padding slots untouched (test_blocked.py:412-418)
        pad = np.ones(ld * n, dtype=bool)
        for j in range(n):
            pad[j * ld: j * ld + min(k, n - 1 - j) + 1] = False
        assert np.array_equal(m.data[pad], small[f"{name}/A"][pad]), name
        res = oracle.residual_norm(n, k, small[f"{name}/A"], ld, m.data, ld)
        assert res <= 10 * n * EPS, (name, res)


def test_hand_cases_exact(small):
    m = bc.BandedMatrix(2, 1, data=small["hand_2x2/A"].copy())
    bc.factor_blocked_serial(m)
    assert (m.get(0, 0), m.get(1, 0), m.get(1, 1)) == (2.0, 1.0, 2.0)
    ident = bc.BandedMatrix(30, 4, data=small["identity_30_4/A"].copy())
    bc.factor_blocked_parallel(ident, 3)
    assert np.array_equal(ident.data, small["identity_30_4/A"])


def test_failure_columns(golden_meta, small):
    for name, want in golden_meta["failures"].items():
        n, k = want["n"], want["k"]
        m = bc.BandedMatrix(n, k, data=small[f"{name}/A"].copy())
        with pytest.raises(bc.NotPositiveDefinite) as err:
            bc.factor_blocked_serial(m)
        assert err.value.column == want["column"], name


def test_nan_pivot_fails():
    a = generate_spd(50, 4, 1)
    a.set(20, 20, float("nan"))
    with pytest.raises(bc.NotPositiveDefinite) as err:
        bc.factor_blocked_serial(a)
    assert err.value.column == 20


def test_solve_vs_reference(golden_meta, small):
    for name, meta in _cases(golden_meta):
        n, k, ld = meta["n"], meta["k"], meta["lead_dim"]
        fac = bc.BandedMatrix(n, k, ld, small[f"{name}/L_ref"].copy())
        x = bc.solve_with_factor(fac, small[f"{name}/rhs"])
        want = small[f"{name}/x"]
        assert np.linalg.norm(x - want) <= X_TOL * max(np.linalg.norm(want), 1e-300), name


def test_solve_singular_and_zero_rhs():
    ident = bc.BandedMatrix(4, 1)
    for i in range(4):
        ident.set(i, i, 1.0)
    ident.set(2, 2, 0.0)
    with pytest.raises(bc.SingularFactor):
        bc.solve_with_factor(ident, np.ones(4))
    fac = bc.factor_blocked_serial(generate_spd(20, 3, 4))
    assert np.array_equal(bc.solve_with_factor(fac, np.zeros(20)), np.zeros(20))


@pytest.mark.parametrize("n,k,seed", [(2000, 50, 0), (2000, 100, 0), (4096, 100, 7), (1000, 150, 1),
                                      (777, 31, 2), (1500, 255, 3), (300, 299, 4)])
def test_mid_sizes_vs_oracle(n, k, seed):
    a = generate_spd(n, k, seed)
    want = a.data.copy()
    oracle.factor_reference(n, k, k + 1, want)
    got = a.copy()
    bc.factor_blocked_serial(got)
    assert oracle.max_scaled_diff(n, k, got.data, k + 1, want, k + 1) <= L_TOL
    assert oracle.residual_fast(n, k, a.data, k + 1, got.data, k + 1) <= 10 * n * EPS


def test_c1_full_fingerprint(golden_meta):
    fp = golden_meta["fingerprints"]["C1"]
    a = generate_spd(fp["n"], fp["k"], fp["seed"])
    assert sha(a.data) == fp["sha_A"]
    want = a.data.copy()
    oracle.factor_reference(fp["n"], fp["k"], fp["k"] + 1, want)
    assert sha(want) == fp["sha_L_ref"]
    got = bc.factor_blocked_serial(a.copy())
    assert oracle.max_scaled_diff(fp["n"], fp["k"], got.data, fp["k"] + 1, want, fp["k"] + 1) <= L_TOL


def test_c2_full(golden_meta, large):
    meta = golden_meta["large"]["C2"]
    n, k = meta["n"], meta["k"]
    a = generate_spd(n, k, 0)
    want = a.data.copy()
    oracle.factor_plain(n, k, k + 1, want)
    got = bc.factor_blocked_serial(a.copy())
    assert oracle.max_scaled_diff(n, k, got.data, k + 1, want, k + 1) <= L_TOL
    cols = large["C2/cols"]
    sampled = np.stack([got.data[c * (k + 1):(c + 1) * (k + 1)] for c in cols])
    assert scaled_diff(sampled, large["C2/L_blocked_cols"]) <= L_TOL
    assert oracle.residual_fast(n, k, a.data, k + 1, got.data, k + 1) <= 10 * n * EPS
    x = bc.solve_with_factor(got, make_rhs(n, 0))
    assert np.linalg.norm(x - large["C2/x"]) / np.linalg.norm(large["C2/x"]) <= X_TOL


@pytest.mark.parametrize("tag", ["C3", "C4"])
def test_large_configs_sampled(golden_meta, large, tag):
    meta = golden_meta["large"][tag]
    n, k = meta["n"], meta["k"]
    a = (generate_spd_wide if meta["wide_diagonal"] else generate_spd)(n, k, meta["seed"])
    got = bc.factor_blocked_serial(a.copy())
    cols = large[f"{tag}/cols"]
    sampled = np.stack([got.data[c * (k + 1):(c + 1) * (k + 1)] for c in cols])
    assert scaled_diff(sampled, large[f"{tag}/L_blocked_cols"]) <= L_TOL
    # backward error through a size-independent property: A x = b for x from L
    b = make_rhs(n, 5)
    x = bc.solve_with_factor(got, b)
    r = band_matvec(n, k, k + 1, a.data, x) - b
    assert np.linalg.norm(r) / np.linalg.norm(b) <= 1e-10


def test_determinism_bitwise():
    a = generate_spd(5000, 100, 3)
    one = bc.factor_blocked_serial(a.copy()).data
    two = bc.factor_blocked_serial(a.copy()).data
    assert one.tobytes() == two.tobytes()


def test_batched_factor_vs_single(golden_meta):
    n, k, B = 4096, 100, 16
    data = np.stack([generate_spd(n, k, s).data for s in range(B)])
    orig = data.copy()
    info = bc.factor_batched(data, n, k)
    assert not info.any()
    for s in (0, 1, 2):
        want = orig[s].copy()
        oracle.factor_reference(n, k, k + 1, want)
        assert sha(want) == golden_meta["fingerprints"][f"C5_s{s}"]["sha_L_ref"]
        assert oracle.max_scaled_diff(n, k, data[s], k + 1, want, k + 1) <= L_TOL


def test_batched_failure_reports_matrix_and_column():
    n, k = 200, 10
    data = np.stack([generate_spd(n, k, s).data for s in range(6)])
    data[3, 57 * (k + 1)] = -1.0
    with pytest.raises(bc.NotPositiveDefinite) as err:
        bc.factor_batched(data, n, k)
    assert err.value.matrix == 3 and err.value.column == 57


def test_c5_fused_full_batch(golden_meta, large):
    """C5: 1024 x (4096, 100) factor + solve; parity on sampled members, A x = b on all."""
    cfg = bc.CONFIGS["C5"]
    n, k, B = cfg.dim, cfg.bandwidth, cfg.batch
    data = np.empty((B, (k + 1) * n))
    rhs = np.empty((B, n))
    for s in range(B):
        data[s] = generate_spd(n, k, s).data
        rhs[s] = make_rhs(n, s)
    a0 = data.copy()
    b0 = rhs.copy()
    info = bc.factor_solve_batched(data, rhs, n, k)
    assert not info.any()
    for s in (0, 1, 2, 1023):
        x_ref = large[f"C5_s{s}/x"]
        assert np.linalg.norm(rhs[s] - x_ref) / np.linalg.norm(x_ref) <= X_TOL
    for s in (0, 511, 1023):
        want = a0[s].copy()
        oracle.factor_plain(n, k, k + 1, want)
        assert oracle.max_scaled_diff(n, k, data[s], k + 1, want, k + 1) <= L_TOL
    r = band_matvec_batched(n, k, k + 1, a0, rhs) - b0
    rel = np.linalg.norm(r, axis=1) / np.linalg.norm(b0, axis=1)
    assert rel.max() <= 1e-10


def test_batched_solve_matches_single():
    n, k, B = 1000, 40, 8
    data = np.stack([generate_spd(n, k, s).data for s in range(B)])
    bc.factor_batched(data, n, k)
    rhs = np.stack([make_rhs(n, s) for s in range(B)])
    x = bc.solve_batched(data, rhs, n, k)
    for s in range(B):
        xs = oracle.solve(n, k, k + 1, data[s], rhs[s])
        assert np.linalg.norm(x[s] - xs) <= X_TOL * np.linalg.norm(xs)


def test_multi_rhs_device_solve():
    n, k, R = 3000, 64, 5
    a = bc.factor_blocked_serial(generate_spd(n, k, 9))
    B = np.stack([make_rhs(n, s) for s in range(R)])
    dab = torch.from_numpy(a.data).cuda()
    db = torch.from_numpy(B.copy()).cuda()
    info = bc.dpbtrs_device(dab, n, k, k + 1, db, nrhs=R)
    assert int(info.item()) == 0
    got = db.cpu().numpy()
    for s in range(R):
        xs = oracle.solve(n, k, k + 1, a.data, B[s])
        assert np.linalg.norm(got[s] - xs) <= X_TOL * np.linalg.norm(xs)


@pytest.mark.parametrize("n,k", [(1, 0), (7, 0), (33, 1), (100, 3), (257, 15), (300, 16), (301, 17),
                                 (500, 40), (640, 63), (1000, 64), (777, 100), (1500, 130)])
def test_fused_factor_solve_shapes(n, k):
    """The fused batched factor + solve (one CTA per matrix) across block-edge shapes."""
    B = 3
    data = np.stack([generate_spd(n, k, 100 + s).data for s in range(B)])
    rhs = np.stack([make_rhs(n, s) for s in range(B)])
    a0, b0 = data.copy(), rhs.copy()
    info = bc.factor_solve_batched(data, rhs, n, k)
    assert not info.any()
    for s in range(B):
        want = a0[s].copy()
        oracle.factor_plain(n, k, k + 1, want)
        assert oracle.max_scaled_diff(n, k, data[s], k + 1, want, k + 1) <= L_TOL
        xs = oracle.solve(n, k, k + 1, want, b0[s])
        assert np.linalg.norm(rhs[s] - xs) <= X_TOL * np.linalg.norm(xs)


def test_fused_failure_keeps_matrix_and_column():
    n, k = 600, 30
    data = np.stack([generate_spd(n, k, s).data for s in range(4)])
    rhs = np.stack([make_rhs(n, s) for s in range(4)])
    data[2, 333 * (k + 1)] = -5.0
    with pytest.raises(bc.NotPositiveDefinite) as err:
        bc.factor_solve_batched(data, rhs, n, k)
    assert err.value.matrix == 2 and err.value.column == 333
