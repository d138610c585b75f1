"""Host-side logic of the drop-in: layout, errors, flop counts, validation order, no CPU fallback."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2305_04635_b200 as bc
from paper_2305_04635_b200 import (BandedMatrix, BandwidthNotDivisible, DeviceError, GridTooSmall,
                                   InvalidBandwidth, OutOfBand, ShapeMismatch, index_map)
from paper_2305_04635_b200.flops import flops_approx, flops_exact, flops_model


def test_index_map_kats():  # pkg/tests/test_core.py:17-50
    assert index_map(0, 0, 5) == 0
    assert index_map(5, 3, 5) == 17
    with pytest.raises(OutOfBand):
        index_map(3, 5, 5)
    with pytest.raises(OutOfBand):
        index_map(9, 3, 5)


def test_banded_matrix_round_trips():
    a = bc.generate_spd(40, 6, seed=2)
    again = BandedMatrix.from_dense(a.to_dense(), 6)
    assert np.array_equal(a.band_panel(), again.band_panel())
    m = BandedMatrix(6, 2)
    m.set(3, 1, 2.5)
    assert m.get(1, 3) == 2.5 and m.get(5, 0) == 0.0
    with pytest.raises(InvalidBandwidth):
        BandedMatrix(4, 4)
    with pytest.raises(ShapeMismatch):
        BandedMatrix(4, 2, lead_dim=2)


def test_flop_counts():  # pkg/tests/test_acceptance.py:77-89
    assert flops_exact(4, 1) == 34
    assert flops_exact(1000, 0) == 4000
    e, ap = flops_exact(100000, 1000), flops_approx(100000, 1000)
    assert 100 * abs(ap - e) <= e
    assert flops_model(20000, 2000) == 20000 * 2000 * 2003
    assert bc.CONFIGS["C5"].model_flops() == 1024 * 4096 * 100 * 103


def test_configs_match_baseline():
    c = bc.CONFIGS
    assert (c["C1"].dim, c["C1"].bandwidth) == (2000, 50)
    assert (c["C2"].dim, c["C2"].bandwidth, c["C2"].solve) == (20000, 200, True)
    assert (c["C3"].dim, c["C3"].bandwidth, c["C3"].wide_diagonal) == (50000, 500, True)
    assert (c["C4"].dim, c["C4"].bandwidth) == (20000, 2000)
    assert (c["C5"].dim, c["C5"].bandwidth, c["C5"].batch) == (4096, 100, 1024)


def test_grid_validation_mirrors_plan_windows():  # blocked.py:91-98, test_blocked.py:386-391
    with pytest.raises(BandwidthNotDivisible):
        bc.factor_blocked_serial(bc.generate_spd(30, 5, seed=0), 3)
    with pytest.raises(GridTooSmall):
        bc.factor_blocked_serial(bc.generate_spd(30, 4, seed=0), 2)
    with pytest.raises(InvalidBandwidth):
        bc.factor_blocked_parallel(bc.generate_spd(30, 1, seed=0), 3)


def test_solve_shape_checked_before_device():
    with pytest.raises(ShapeMismatch):
        bc.solve_with_factor(BandedMatrix(4, 1), np.ones(5))


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    """Without a GPU the product path raises; it never computes on the CPU."""
    with pytest.raises(DeviceError):
        bc.factor_blocked_serial(bc.generate_spd(20, 3, seed=0))
    with pytest.raises(DeviceError):
        bc.factor_batched(np.zeros((2, 4 * 20)), 20, 3)


def test_reference_matrix_accepted_by_validation():
    """Duck typing: anything with dim/bandwidth/lead_dim/data passes check_matrix."""
    from paper_2305_04635_b200.core import check_matrix

    class Foreign:  # shaped like bandchol.BandedMatrix
        def __init__(self):
            self.dim, self.bandwidth, self.lead_dim = 10, 2, 3
            self.data = np.zeros(30)
    assert check_matrix(Foreign())[:3] == (10, 2, 3)
    bad = Foreign()
    bad.data = np.zeros(29)
    with pytest.raises(ShapeMismatch):
        check_matrix(bad)
