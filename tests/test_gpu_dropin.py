"""The drop-in on genuine reference objects: the unmodified `bandchol` package (installed
offline into baseline/_ref, it travels with the repo) with its engines rebound to the GPU by
paper_2305_04635_b200.dropin.install.  The assertions restate the reference's own engine and
acceptance gates on `bandchol.BandedMatrix` instances created by the reference itself:
  * correctness sweep: pkg/tests/test_acceptance.py:34-61 (residual_norm <= 1e-10 with the
    reference's residual, elementwise <= 1e-11 against factor_reference (its bit-exact C
    restatement), scale
    max(|ref|, 1); k < 2 padded to 2 like the reference test),
  * byte determinism serial vs parallel: test_acceptance.py:64-74,
  * engine tests: pkg/tests/test_blocked.py:342-418 (identity, embedded hand case, residual
    contract, equivalence across grids, grid argument errors, failure column, padding rows),
  * solve: pkg/tests/test_core.py:191-227 (hand 2x2, identity, SingularFactor).
Skipped when baseline/_ref is absent.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
if not os.path.isdir(os.path.join(REF, "bandchol")):  # pragma: no cover
    pytest.skip("baseline/_ref (the reference package) is not installed", allow_module_level=True)
if REF not in sys.path:
    sys.path.insert(0, REF)

import bandchol  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_2305_04635_b200 import dropin  # noqa: E402


def factor_reference_rows(a):
    """band_panel() of the reference's factor_reference(a) (reference.py:32-63), from the
    oracle's bit-exact C restatement (pinned in tests/test_oracle.py; the Python original
    takes minutes at n = 5000)."""
    f = a.copy()
    oracle.factor_reference(f.dim, f.bandwidth, f.lead_dim, f.data)
    return f.band_panel()


@pytest.fixture
def gpu_bandchol():
    handle = dropin.install(bandchol)
    yield bandchol
    handle.uninstall()


def test_install_rebinds_every_entry_point(gpu_bandchol):
    mods = sys.modules
    for mod, name in ((bandchol, "factor_blocked_serial"), (mods["bandchol.blocked"], "factor_blocked_serial"),
                      (bandchol, "factor_blocked_parallel"), (mods["bandchol.parallel"], "factor_blocked_parallel"),
                      (bandchol, "solve_with_factor"), (mods["bandchol.core"], "solve_with_factor")):
        assert getattr(getattr(mod, name), "__wrapped_gpu__", False), (mod.__name__, name)


def test_correctness_sweep(gpu_bandchol):
    bc = gpu_bandchol
    for n_dim in (64, 257, 1000, 5000):
        for k in (0, 1, 2, 8, 50, 100):
            if k >= n_dim:
                continue
            for seed in range(3):
                a = bc.generate_spd(n_dim, k, seed)
                ref_rows = factor_reference_rows(a)
                scale = np.maximum(np.abs(ref_rows), 1.0)
                blocked_in = bc.pad_bandwidth(a, 2) if k < 2 else a
                ser = bc.factor_blocked_serial(blocked_in.copy(), 3)
                par = bc.factor_blocked_parallel(blocked_in.copy(), 3, bc.ExecPolicy(worker_count=4))
                for fac in (ser, par):
                    assert isinstance(fac, bc.BandedMatrix)
                    got = fac.band_panel()[:k + 1]
                    assert np.max(np.abs(got - ref_rows) / scale) <= 1e-11, (n_dim, k, seed)
                assert bc.residual_norm(blocked_in, ser) <= 1e-10, (n_dim, k, seed)


def test_determinism_byte_identical(gpu_bandchol):
    bc = gpu_bandchol
    a = bc.generate_spd(2000, 100, seed=0)
    for n in (3, 5):
        want = bc.factor_blocked_serial(a.copy(), n).data.tobytes()
        for workers in (1, 2, 4, 8):
            for _ in range(5):
                got = bc.factor_blocked_parallel(a.copy(), n, bc.ExecPolicy(worker_count=workers))
                assert got.data.tobytes() == want, (n, workers)


def test_engine_cases(gpu_bandchol):
    bc = gpu_bandchol
    # identity is a fixed point
    a = bc.BandedMatrix(20, 2)
    for i in range(20):
        a.set(i, i, 1.0)
    before = a.band_panel().copy()
    assert np.array_equal(bc.factor_blocked_serial(a, 3).band_panel(), before)
    # embedded hand case [[4,2],[2,5]] -> [[2,0],[1,2]]
    a = bc.BandedMatrix(20, 2)
    for i in range(20):
        a.set(i, i, 1.0)
    a.set(0, 0, 4.0)
    a.set(1, 0, 2.0)
    a.set(1, 1, 5.0)
    fac = bc.factor_blocked_serial(a, 3)
    assert fac is a  # in place, same object
    assert (fac.get(0, 0), fac.get(1, 0), fac.get(1, 1)) == (2.0, 1.0, 2.0)
    # residual contract and grid independence
    a = bc.generate_spd(300, 12, seed=6)
    assert bc.residual_norm(a, bc.factor_blocked_serial(a.copy(), 4)) <= 1e-10
    a = bc.generate_spd(120, 8, seed=7)
    outs = [bc.factor_blocked_serial(a.copy(), n).band_panel() for n in (3, 5, 9)]
    for other in outs[1:]:
        assert np.max(np.abs(other - outs[0]) / np.maximum(np.abs(outs[0]), 1.0)) <= 1e-11
    # the grid argument errors, as the reference's own classes
    with pytest.raises(bc.BandwidthNotDivisible):
        bc.factor_blocked_serial(bc.generate_spd(30, 5, seed=0), 3)
    with pytest.raises(bc.GridTooSmall):
        bc.factor_blocked_serial(bc.generate_spd(30, 4, seed=0), 2)
    # the global failure column, as the reference's NotPositiveDefinite
    a = bc.generate_spd(40, 4, seed=8)
    a.set(17, 17, -1.0)
    with pytest.raises(bc.NotPositiveDefinite) as err:
        bc.factor_blocked_serial(a, 3)
    assert err.value.column == 17
    a = bc.generate_spd(40, 4, seed=8)
    a.set(23, 23, float("nan"))
    with pytest.raises(bc.NotPositiveDefinite) as err:
        bc.factor_blocked_parallel(a, 3, bc.ExecPolicy(worker_count=2))
    assert err.value.column == 23
    # padding rows stay zero
    panel = bc.factor_blocked_serial(bc.generate_spd(45, 6, seed=10), 3).panel
    for j in range(45):
        top = min(44, j + 6) - j
        assert np.all(panel[top + 1:, j] == 0.0)


def test_solve_cases(gpu_bandchol):
    bc = gpu_bandchol
    f = bc.BandedMatrix(2, 1)
    f.set(0, 0, 2.0)
    f.set(1, 0, 1.0)
    f.set(1, 1, 2.0)
    x = bc.solve_with_factor(f, np.array([2.0, 5.0]))  # L L^T = [[4,2],[2,5]]
    assert np.allclose(x, [0.0, 1.0], atol=1e-15)
    ident = bc.BandedMatrix(7, 2)
    for i in range(7):
        ident.set(i, i, 1.0)
    b = np.arange(7, dtype=np.float64)
    assert np.array_equal(bc.solve_with_factor(ident, b), b)
    a = bc.generate_spd(150, 9, seed=5)
    fac = bc.factor_blocked_serial(a.copy(), 4)
    rhs = np.random.default_rng(6).standard_normal(150)
    x = bc.solve_with_factor(fac, rhs)
    dense = a.to_dense()
    assert np.linalg.norm(dense @ x - rhs) <= 1e-10 * np.linalg.norm(rhs)
    ident.set(3, 3, 0.0)
    with pytest.raises(bc.SingularFactor):
        bc.solve_with_factor(ident, b)
    with pytest.raises(bc.ShapeMismatch):
        bc.solve_with_factor(fac, np.zeros(149))


def test_uninstall_restores_reference():
    handle = dropin.install(bandchol)
    handle.uninstall()
    assert not getattr(bandchol.factor_blocked_serial, "__wrapped_gpu__", False)
    assert bandchol.factor_blocked_serial is sys.modules["bandchol.blocked"].factor_blocked_serial
