"""B200-native fp64 banded Cholesky: a drop-in for the bandchol factorization path.

Public names follow the reference package (pkg/src/bandchol/__init__.py:5-37) for
everything on the factorization path: BandedMatrix and the packed layout, the
exception tree, factor_blocked_serial / factor_blocked_parallel /
solve_with_factor (running on the GPU through libbandchol_b200.so), the seeded
generator and the flop counts.  Batched / device-resident entry points are
added for the interior-point use case.
"""

from .core import BandedMatrix, index_map
from .engine import (BatchedBandSolver, TraceEvent, pinned_empty, dpbsv_batched_device, dpbtrf_fwd_batched_device,
                     dpbtrs_bwd_batched_device, dpbtrf_batched_device, dpbtrf_device,
                     dpbtrs_batched_device, dpbtrs_device, factor_batched,
                     factor_blocked_parallel, factor_blocked_serial, factor_solve_batched,
                     library_version, solve_batched, solve_many, solve_with_factor)
from .engine import band_residual_batched_device, band_residual_device, residual_norm
from .fixtures import load_matrix, load_matrix_device, save_matrix
from .errors import (BandCholError, BandwidthNotDivisible, CountOverflow, DeviceError,
                     GridTooSmall, InvalidBandwidth, NotPositiveDefinite, OutOfBand,
                     ShapeMismatch, SingularFactor)
from .flops import flops_approx, flops_exact, flops_model
from .inputs import CONFIGS, BandConfig, generate_spd, generate_spd_wide, make_rhs

__version__ = "0.1.0"

__all__ = [
    "BandedMatrix", "index_map", "TraceEvent", "BatchedBandSolver", "pinned_empty", "dpbsv_batched_device", "dpbtrf_fwd_batched_device", "dpbtrs_bwd_batched_device", "dpbtrf_batched_device",
    "dpbtrf_device", "dpbtrs_batched_device", "dpbtrs_device", "factor_batched",
    "factor_blocked_parallel", "factor_blocked_serial", "factor_solve_batched", "library_version",
    "solve_batched", "solve_many", "solve_with_factor", "BandCholError", "BandwidthNotDivisible", "CountOverflow",
    "DeviceError", "GridTooSmall", "InvalidBandwidth", "NotPositiveDefinite", "OutOfBand",
    "ShapeMismatch", "SingularFactor", "flops_approx", "flops_exact", "flops_model", "CONFIGS",
    "BandConfig", "generate_spd", "generate_spd_wide", "make_rhs",
    "band_residual_device", "band_residual_batched_device", "residual_norm", "load_matrix", "load_matrix_device", "save_matrix",
]
