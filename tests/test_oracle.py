"""Pin the CPU oracle (oracle/) and the input generator against the reference's own outputs.

Golden data: tests/golden/ (made by tests/golden/make_golden.py from the reference).
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import band_matvec, scaled_diff, sha
from oracle import oracle
from paper_2305_04635_b200.inputs import generate_spd, generate_spd_wide, make_rhs


def _cases(golden_meta):
    return sorted(golden_meta["cases"].items())


def test_fsum_matches_math_fsum():
    rng = np.random.default_rng(0)
    for trial in range(200):
        v = rng.standard_normal(rng.integers(0, 300)) * 10.0 ** rng.integers(-30, 30, size=1)
        if trial % 3 == 0 and v.size:
            v = np.concatenate([v, -v[::-1] * (1 + 1e-16), [1e100, -1e100]])
        assert oracle.fsum(v) == math.fsum(v.tolist())
    assert oracle.fsum([1e100, 1.0, -1e100, 1e-100, 1e50, -1.0, -1e50]) == 1e-100
    assert oracle.fsum([]) == 0.0


def test_oracle_bit_exact_on_small_cases(golden_meta, small):
    """bco_factor_reference reproduces factor_reference (reference.py:32-63) byte for byte."""
    for name, meta in _cases(golden_meta):
        n, k, ld = meta["n"], meta["k"], meta["lead_dim"]
        got = small[f"{name}/A"].copy()
        oracle.factor_reference(n, k, ld, got)
        assert got.tobytes() == small[f"{name}/L_ref"].tobytes(), name


@pytest.mark.parametrize("tag", ["C1", "n2000_k100", "C5_s0", "C5_s1", "C5_s2", "C5_s1023"])
def test_oracle_bit_exact_fingerprints(golden_meta, tag):
    fp = golden_meta["fingerprints"][tag]
    a = generate_spd(fp["n"], fp["k"], fp["seed"])
    assert sha(a.data) == fp["sha_A"]  # generator == core.py:155-181, byte for byte
    oracle.factor_reference(fp["n"], fp["k"], fp["k"] + 1, a.data)
    assert sha(a.data) == fp["sha_L_ref"]


def test_oracle_bit_exact_c2(golden_meta):
    fp = golden_meta["fingerprints"]["C2"]
    a = generate_spd(fp["n"], fp["k"], fp["seed"])
    assert sha(a.data) == fp["sha_A"]
    oracle.factor_reference(fp["n"], fp["k"], fp["k"] + 1, a.data)
    assert sha(a.data) == fp["sha_L_ref"]


def test_generator_large_configs(golden_meta):
    for tag, meta in golden_meta["large"].items():
        gen = generate_spd_wide if meta["wide_diagonal"] else generate_spd
        a = gen(meta["n"], meta["k"], meta["seed"])
        assert sha(a.data) == meta["sha_A"], tag


def test_c3_wide_diagonal_is_dominant():
    a = generate_spd_wide(3000, 40, 0)
    p = a.panel
    off = np.zeros(3000)
    for d in range(1, 41):
        off[d:] += np.abs(p[d, : 3000 - d])
        off[: 3000 - d] += np.abs(p[d, : 3000 - d])
    assert np.all(p[0] > off)
    ratio = (p[0] - 1.0) / off
    assert ratio.min() >= 1.05 - 1e-12 and ratio.max() > 100.0  # log-uniform [1, 1e4] spread


def test_oracle_failure_columns(golden_meta, small):
    for name, want in golden_meta["failures"].items():
        a = small[f"{name}/A"].copy()
        with pytest.raises(oracle.OracleFailure) as err:
            oracle.factor_reference(want["n"], want["k"], want["k"] + 1, a)
        assert err.value.column == want["column"], name


def test_oracle_solve_matches_reference(golden_meta, small):
    for name, meta in _cases(golden_meta):
        n, k, ld = meta["n"], meta["k"], meta["lead_dim"]
        x = oracle.solve(n, k, ld, small[f"{name}/L_ref"], small[f"{name}/rhs"])
        want = small[f"{name}/x"]
        assert np.linalg.norm(x - want) <= 1e-13 * max(np.linalg.norm(want), 1e-300), name


def test_oracle_solve_singular():
    ld = np.zeros(8)
    ld[0::2] = 1.0
    ld[4] = 0.0  # diag of column 2
    with pytest.raises(oracle.OracleFailure) as err:
        oracle.solve(4, 1, 2, ld, np.ones(4))
    assert err.value.column == 2


def test_oracle_residual_matches_reference(golden_meta, small):
    for name, meta in _cases(golden_meta):
        n, k, ld = meta["n"], meta["k"], meta["lead_dim"]
        a, l = small[f"{name}/A"], small[f"{name}/L_ref"]
        r1 = oracle.residual_norm(n, k, a, ld, l, ld)
        r2 = oracle.residual_fast(n, k, a, ld, l, ld)
        assert r1 == pytest.approx(meta["residual"], rel=1e-6, abs=1e-18), name
        assert r2 == pytest.approx(meta["residual"], rel=1e-2, abs=1e-17), name


def test_plain_oracle_close_to_reference(golden_meta, small):
    for name, meta in _cases(golden_meta):
        n, k, ld = meta["n"], meta["k"], meta["lead_dim"]
        a = small[f"{name}/A"].copy()
        oracle.factor_plain(n, k, ld, a)
        assert oracle.max_scaled_diff(n, k, a, ld, small[f"{name}/L_ref"], ld) <= 1e-13, name


def test_reference_blocked_engine_close_to_fsum(golden_meta, small):
    """The reference's own two engines agree to ~1e-16 scaled (context for L_TOL)."""
    for name, meta in _cases(golden_meta):
        if "blocked_grid" not in meta:
            continue
        n, k, ld = meta["n"], meta["k"], meta["lead_dim"]
        assert oracle.max_scaled_diff(n, k, small[f"{name}/L_blocked"], ld,
                                      small[f"{name}/L_ref"], ld) <= 1e-13, name


@pytest.mark.parametrize("tag", ["C2", "C3"])
def test_plain_oracle_on_large_samples(golden_meta, large, tag):
    meta = golden_meta["large"][tag]
    n, k = meta["n"], meta["k"]
    a = (generate_spd_wide if meta["wide_diagonal"] else generate_spd)(n, k, meta["seed"])
    oracle.factor_plain(n, k, k + 1, a.data)
    cols = large[f"{tag}/cols"]
    got = np.stack([a.data[c * (k + 1):(c + 1) * (k + 1)] for c in cols])
    assert scaled_diff(got, large[f"{tag}/L_blocked_cols"]) <= 1e-12
    if tag == "C2":
        x = oracle.solve(n, k, k + 1, a.data, make_rhs(n, 0))
        want = large["C2/x"]
        assert np.linalg.norm(x - want) / np.linalg.norm(want) <= 1e-12


def test_solve_golden_is_a_solution(golden_meta, small):
    name = "spd_150_9_5"
    meta = golden_meta["cases"][name]
    a, x, b = small[f"{name}/A"], small[f"{name}/x"], small[f"{name}/rhs"]
    r = band_matvec(meta["n"], meta["k"], meta["lead_dim"], a, x) - b
    assert np.linalg.norm(r) / np.linalg.norm(b) <= 1e-12


def test_blocked_dense_oracle_close_to_reference(golden_meta, small):
    """oracle.factor_blocked_dense (the C3/C4 full-L checker) against the reference's
    factor_reference on every small golden case, at several tile sizes."""
    for name, meta in _cases(golden_meta):
        n, k, ld = meta["n"], meta["k"], meta["lead_dim"]
        for nb in (3, 16, 64):
            a = small[f"{name}/A"].copy()
            oracle.factor_blocked_dense(n, k, ld, a, nb)
            assert oracle.max_scaled_diff(n, k, a, ld, small[f"{name}/L_ref"], ld) <= 1e-13, (name, nb)
            pad = np.ones(ld * n, dtype=bool)  # padding never written
            for j in range(n):
                pad[j * ld: j * ld + min(k, n - 1 - j) + 1] = False
            assert np.array_equal(a[pad], small[f"{name}/A"][pad]), name


@pytest.mark.parametrize("tag", ["C2", "C3"])
def test_blocked_dense_oracle_on_large_samples(golden_meta, large, tag):
    meta = golden_meta["large"][tag]
    n, k = meta["n"], meta["k"]
    a = (generate_spd_wide if meta["wide_diagonal"] else generate_spd)(n, k, meta["seed"])
    oracle.factor_blocked_dense(n, k, k + 1, a.data)
    cols = large[f"{tag}/cols"]
    got = np.stack([a.data[c * (k + 1):(c + 1) * (k + 1)] for c in cols])
    assert scaled_diff(got, large[f"{tag}/L_blocked_cols"]) <= 1e-12


def test_blocked_dense_oracle_failure_column(golden_meta, small):
    for name, want in golden_meta["failures"].items():
        a = small[f"{name}/A"].copy()
        with pytest.raises(oracle.OracleFailure) as err:
            oracle.factor_blocked_dense(want["n"], want["k"], want["k"] + 1, a, 16)
        assert err.value.column == want["column"], name


def test_plain_batched_is_plain():
    n, k = 700, 30
    data = np.stack([generate_spd(n, k, s).data for s in range(6)])
    data[4, 123 * (k + 1)] = -1.0
    want = data.copy()
    info = oracle.factor_plain_batched(n, k, k + 1, data)
    assert list(info) == [-1, -1, -1, -1, 123, -1]
    for s in (0, 1, 2, 3, 5):
        oracle.factor_plain(n, k, k + 1, want[s])
        assert data[s].tobytes() == want[s].tobytes()
