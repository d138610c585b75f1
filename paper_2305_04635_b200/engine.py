"""Host-side mirror of the reference's factorization / solve interface, on the GPU.

Same names, argument meaning and error behaviour as the reference entry points:

* `factor_blocked_serial(matrix, grid_dim, *, backend, trace, check_invariants)`
  -- pkg/src/bandchol/blocked.py:363-385
* `factor_blocked_parallel(matrix, grid_dim, policy, *, backend, trace, check_invariants)`
  -- pkg/src/bandchol/parallel.py:130-166
* `solve_with_factor(factor, rhs)` -- pkg/src/bandchol/core.py:216-240

`matrix` is any object with the BandedMatrix fields (ours or the reference's):
its `.data` is overwritten with L in place and the same object is returned
(blocked.py:385).  The arithmetic runs in libbandchol_b200.so; this module only
moves buffers (torch is used for device memory and streams) and maps the
device `info` word onto the reference's exceptions:
NotPositiveDefinite(column) for the first failing pivot, SingularFactor for a
non-positive diagonal in the solve.  There is no CPU path: without the library
or a GPU every call raises DeviceError.

`grid_dim` is accepted for signature compatibility.  The GPU engine chooses its
own tiles and needs no divisibility, but when a grid is passed the reference's
plan_windows validation (blocked.py:91-98) is applied first so the same inputs
raise the same errors.  `backend` is ignored (the CUDA kernels are the only
engine); `trace` receives one TraceEvent per kernel launch.

Batched and device-resident entry points (`factor_batched`, `solve_batched`,
`factor_solve_batched`, `DeviceBatch`) serve the interior-point use case
(BASELINE.json config C5).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import check_matrix
from .errors import (BandCholError, BandwidthNotDivisible, DeviceError, GridTooSmall,
                     InvalidBandwidth, NotPositiveDefinite, ShapeMismatch, SingularFactor)


@dataclass(frozen=True)
class TraceEvent:
    """One kernel launch (the reference records one event per tile op, blocked.py:289-294)."""
    kind: str
    window: int
    row: int
    col: int


def _torch():
    try:
        import torch
    except ImportError as exc:  # pragma: no cover
        raise DeviceError(f"torch is required for device memory: {exc}") from None
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device is visible; the band Cholesky runs only on the GPU")
    return torch


def _stream_for(torch, device, stream):
    """The launch stream: `stream`, else the current stream of `device` (never of whatever
    device happens to be current)."""
    if stream is None:
        return torch.cuda.current_stream(device)
    if stream.device != device:
        raise ShapeMismatch(f"stream is on {stream.device}, tensors on {device}")
    return stream


def _stream_handle(torch, stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


class _on_device:
    """Make `device` current for the C-ABI call (the library launches on the current
    device; every pointer passed must live there)."""

    def __init__(self, torch, device):
        self.guard = torch.cuda.device(device)

    def __enter__(self):
        self.guard.__enter__()
        return self

    def __exit__(self, *exc):
        return self.guard.__exit__(*exc)


def _same_device(device, **tensors) -> None:
    for name, t in tensors.items():
        if t is not None and t.device != device:
            raise ShapeMismatch(f"{name} is on {t.device}, ab on {device}")


def _workspace(torch, n: int, kd: int, ldab: int, device, stream):
    """Workspace of the multi-CTA kernel, allocated per call in stream order on `stream`
    (torch's caching allocator makes this cheap); the kernel launch clears it, so calls on
    different streams never share flags."""
    need = int(_lib.load().bcg_dpbtrf_workspace_size(n, kd, ldab))
    if need == 0:
        return None, 0
    with torch.cuda.stream(stream):
        ws = torch.empty(need, dtype=torch.uint8, device=device)
    return ws, need


def _validate_grid(n: int, k: int, grid_dim) -> None:
    """plan_windows' argument checks (blocked.py:91-98), only when a grid is given."""
    if grid_dim is None:
        return
    if grid_dim < 3:
        raise GridTooSmall(f"grid dimension {grid_dim} < 3")
    if k < 2 or k >= n:
        raise InvalidBandwidth(
            f"blocked factorization needs 2 <= bandwidth < dim, got k={k}, N={n}")
    if k % (grid_dim - 1):
        raise BandwidthNotDivisible(
            f"bandwidth {k} not divisible by grid_dim-1 = {grid_dim - 1}")


# -- device-resident primitives ---------------------------------------------------

def _dev(t, torch, dtype, numel: int, name: str):
    """Argument check for a device buffer handed to the C ABI as a raw pointer: the
    kernels index it up to `numel`, so dtype, device, layout and size must hold."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ShapeMismatch(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise ShapeMismatch(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ShapeMismatch(f"{name} must be contiguous")
    if t.numel() < numel:
        raise ShapeMismatch(f"{name} holds {t.numel()} elements, needs {numel}")
    return t


def _info(torch, info, count: int, device):
    if info is None:
        return torch.zeros(count, dtype=torch.int32, device=device)
    return _dev(info, torch, torch.int32, count, "info")


def dpbtrf_device(ab, n: int, kd: int, ldab: int, info=None, stream=None):
    """Factor one band matrix held in a CUDA float64 tensor, in place.  Returns info."""
    torch = _torch()
    _dev(ab, torch, torch.float64, ldab * n, "ab")
    info = _info(torch, info, 1, ab.device)
    _same_device(ab.device, info=info)
    with _on_device(torch, ab.device):
        st = _stream_for(torch, ab.device, stream)
        ws, need = _workspace(torch, n, kd, ldab, ab.device, st)
        rc = _lib.load().bcg_dpbtrf(n, kd, ab.data_ptr(), ldab, info.data_ptr(),
                                    ws.data_ptr() if ws is not None else None, need, st.cuda_stream)
        if ws is not None:
            ws.record_stream(st)
    _lib.check(rc, "bcg_dpbtrf")
    return info


def dpbtrf_batched_device(ab, n: int, kd: int, ldab: int, batch: int, info=None, stream=None):
    """Factor `batch` matrices stored back to back (stride ldab*n) in a CUDA tensor."""
    torch = _torch()
    _dev(ab, torch, torch.float64, ldab * n * batch, "ab")
    info = _info(torch, info, batch, ab.device)
    _same_device(ab.device, info=info)
    with _on_device(torch, ab.device):
        st = _stream_for(torch, ab.device, stream)
        lib = _lib.load()
        need = int(lib.bcg_dpbtrf_batched_workspace_size(n, kd, ldab, batch))
        ws = None
        if need:
            with torch.cuda.stream(st):
                ws = torch.empty(need, dtype=torch.uint8, device=ab.device)
        rc = lib.bcg_dpbtrf_batched(n, kd, ab.data_ptr(), ldab, ldab * n, batch, info.data_ptr(),
                                    ws.data_ptr() if ws is not None else None, need, st.cuda_stream)
        if ws is not None:
            ws.record_stream(st)
    _lib.check(rc, "bcg_dpbtrf_batched")
    return info


def dpbtrs_device(ab, n: int, kd: int, ldab: int, b, nrhs: int = 1, info=None, stream=None):
    """Solve L L^T x = b in place for nrhs right-hand sides (columns of length n)."""
    torch = _torch()
    _dev(ab, torch, torch.float64, ldab * n, "ab")
    _dev(b, torch, torch.float64, n * nrhs, "b")
    info = _info(torch, info, 1, ab.device)
    _same_device(ab.device, b=b, info=info)
    with _on_device(torch, ab.device):
        st = _stream_for(torch, ab.device, stream)
        rc = _lib.load().bcg_dpbtrs(n, kd, ab.data_ptr(), ldab, b.data_ptr(), n, nrhs,
                                    info.data_ptr(), st.cuda_stream)
    _lib.check(rc, "bcg_dpbtrs")
    return info


def dpbtrs_batched_device(ab, n: int, kd: int, ldab: int, b, batch: int, nrhs: int = 1, info=None,
                          stream=None):
    """Solve every system of a factored batch (L from dpbtrf_batched_device) in place in b:
    matrix i has nrhs right-hand sides, b[i] of shape (nrhs, n)."""
    torch = _torch()
    _dev(ab, torch, torch.float64, ldab * n * batch, "ab")
    _dev(b, torch, torch.float64, n * nrhs * batch, "b")
    info = _info(torch, info, batch, ab.device)
    _same_device(ab.device, b=b, info=info)
    with _on_device(torch, ab.device):
        st = _stream_for(torch, ab.device, stream)
        lib = _lib.load()
        if nrhs == 1:
            rc = lib.bcg_dpbtrs_batched(n, kd, ab.data_ptr(), ldab, ldab * n, b.data_ptr(), n,
                                        batch, info.data_ptr(), st.cuda_stream)
        else:
            rc = lib.bcg_dpbtrs_batched_nrhs(n, kd, ab.data_ptr(), ldab, ldab * n, b.data_ptr(), n,
                                             n * nrhs, nrhs, batch, info.data_ptr(), st.cuda_stream)
    _lib.check(rc, "bcg_dpbtrs_batched")
    return info


def dpbsv_batched_device(ab, n: int, kd: int, ldab: int, b, batch: int, info=None, stream=None):
    """Factor + solve of `batch` systems: ab -> L, b -> x (bcg_dpbsv_batched: the batched
    factorization with the forward sweep fused in -- y goes to the workspace -- then the
    backward sweep, which skips failed matrices and leaves their b untouched)."""
    torch = _torch()
    _dev(ab, torch, torch.float64, ldab * n * batch, "ab")
    _dev(b, torch, torch.float64, n * batch, "b")
    info = _info(torch, info, batch, ab.device)
    _same_device(ab.device, b=b, info=info)
    with _on_device(torch, ab.device):
        st = _stream_for(torch, ab.device, stream)
        lib = _lib.load()
        need = int(lib.bcg_dpbsv_batched_workspace_size(n, kd, ldab, batch))
        ws = None
        if need:
            with torch.cuda.stream(st):
                ws = torch.empty(need, dtype=torch.uint8, device=ab.device)
        rc = lib.bcg_dpbsv_batched(n, kd, ab.data_ptr(), ldab, ldab * n, b.data_ptr(), n,
                                   batch, info.data_ptr(), ws.data_ptr() if ws is not None else None,
                                   need, st.cuda_stream)
        if ws is not None:
            ws.record_stream(st)
    _lib.check(rc, "bcg_dpbsv_batched")
    return info


def dpbtrf_fwd_batched_device(ab, n: int, kd: int, ldab: int, b, y, batch: int, info=None, stream=None):
    """First half of dpbsv_batched_device's fused path (bcg_dpbtrf_fwd_batched): ab -> L with
    the forward sweep L y = b fused into the factorization kernel; b is only read, y
    (batch * n doubles) receives the intermediate vectors."""
    torch = _torch()
    _dev(ab, torch, torch.float64, ldab * n * batch, "ab")
    _dev(b, torch, torch.float64, n * batch, "b")
    _dev(y, torch, torch.float64, n * batch, "y")
    info = _info(torch, info, batch, ab.device)
    _same_device(ab.device, b=b, y=y, info=info)
    with _on_device(torch, ab.device):
        st = _stream_for(torch, ab.device, stream)
        rc = _lib.load().bcg_dpbtrf_fwd_batched(n, kd, ab.data_ptr(), ldab, ldab * n, b.data_ptr(), n, batch,
                                                info.data_ptr(), y.data_ptr(), st.cuda_stream)
    _lib.check(rc, "bcg_dpbtrf_fwd_batched")
    return info


def dpbtrs_bwd_batched_device(ab, n: int, kd: int, ldab: int, y, x, batch: int, info, stream=None):
    """Second half (bcg_dpbtrs_bwd_batched): L^T x = y for the matrices with info == 0."""
    torch = _torch()
    _dev(ab, torch, torch.float64, ldab * n * batch, "ab")
    _dev(y, torch, torch.float64, n * batch, "y")
    _dev(x, torch, torch.float64, n * batch, "x")
    _same_device(ab.device, y=y, x=x, info=info)
    with _on_device(torch, ab.device):
        st = _stream_for(torch, ab.device, stream)
        rc = _lib.load().bcg_dpbtrs_bwd_batched(n, kd, ab.data_ptr(), ldab, ldab * n, y.data_ptr(), x.data_ptr(), n,
                                                batch, info.data_ptr(), st.cuda_stream)
    _lib.check(rc, "bcg_dpbtrs_bwd_batched")
    return info


def band_residual_device(a, l, n: int, kd: int, lda: int, ldl: int, out=None, stream=None):
    """Device ||A - L L^T||_F / ||A||_F (core.py:186-213) of CUDA float64 tensors; returns
    a 1-element CUDA tensor (no host synchronisation)."""
    torch = _torch()
    lib = _lib.load()
    _dev(a, torch, torch.float64, lda * n, "a")
    _dev(l, torch, torch.float64, ldl * n, "l")
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device=a.device)
    _dev(out, torch, torch.float64, 1, "out")
    _same_device(a.device, l=l, out=out)
    with _on_device(torch, a.device):
        st = _stream_for(torch, a.device, stream)
        need = int(lib.bcg_band_residual_workspace_size())
        with torch.cuda.stream(st):
            ws = torch.empty(need // 8 + 1, dtype=torch.float64, device=a.device)
        rc = lib.bcg_band_residual(n, kd, a.data_ptr(), lda, l.data_ptr(), ldl, out.data_ptr(), ws.data_ptr(),
                                   need, st.cuda_stream)
        ws.record_stream(st)
    _lib.check(rc, "bcg_band_residual")
    return out


def band_residual_batched_device(a, l, n: int, kd: int, lda: int, ldl: int, batch: int, out=None,
                                 stream=None):
    """Per-matrix backward error of a batch (a: original matrices, l: their factors, rows
    of lda*n / ldl*n doubles); returns a CUDA float64 tensor of `batch` residuals."""
    torch = _torch()
    lib = _lib.load()
    _dev(a, torch, torch.float64, lda * n * batch, "a")
    _dev(l, torch, torch.float64, ldl * n * batch, "l")
    if out is None:
        out = torch.empty(max(batch, 1), dtype=torch.float64, device=a.device)
    _dev(out, torch, torch.float64, batch, "out")
    _same_device(a.device, l=l, out=out)
    with _on_device(torch, a.device):
        st = _stream_for(torch, a.device, stream)
        need = int(lib.bcg_band_residual_batched_workspace_size(batch))
        with torch.cuda.stream(st):
            ws = torch.empty(need // 8 + 1, dtype=torch.float64, device=a.device)
        rc = lib.bcg_band_residual_batched(n, kd, a.data_ptr(), lda, lda * n, l.data_ptr(), ldl, ldl * n, batch,
                                           out.data_ptr(), ws.data_ptr(), need, st.cuda_stream)
        ws.record_stream(st)
    _lib.check(rc, "bcg_band_residual_batched")
    return out[:batch]


def residual_norm(original, factor) -> float:
    """residual_norm(original, factor) of the reference (core.py:186-213), computed on the GPU."""
    check_matrix(original)
    check_matrix(factor)
    if original.dim != factor.dim or original.bandwidth != factor.bandwidth:
        raise ShapeMismatch(
            f"matrix ({original.dim}, k={original.bandwidth}) vs "
            f"factor ({factor.dim}, k={factor.bandwidth})")
    torch = _torch()
    a = torch.from_numpy(np.ascontiguousarray(original.data)).to("cuda")
    f = torch.from_numpy(np.ascontiguousarray(factor.data)).to("cuda")
    r = band_residual_device(a, f, original.dim, original.bandwidth, original.lead_dim, factor.lead_dim)
    return float(r.item())


def _raise_factor_info(info_value: int) -> None:
    if info_value > 0:
        raise NotPositiveDefinite(info_value - 1)


# -- reference-shaped host API ----------------------------------------------------

def _factor(matrix, grid_dim, trace) -> object:
    n, k, ld, data = check_matrix(matrix)
    _validate_grid(n, k, grid_dim)
    torch = _torch()
    dev = torch.from_numpy(data).to("cuda", non_blocking=False)
    info = dpbtrf_device(dev, n, k, ld)
    info_h = int(info.item())
    if trace is not None:
        trace.append(TraceEvent("gpu_dpbtrf", 0, 0, 0))
    if info_h > 0:
        raise NotPositiveDefinite(info_h - 1)
    data[...] = dev.cpu().numpy()
    return matrix


def factor_blocked_serial(matrix, grid_dim=None, *, backend=None, trace=None,
                          check_invariants: bool = False):
    """GPU drop-in for blocked.py:363-385: overwrites matrix.data with L, returns matrix."""
    return _factor(matrix, grid_dim, trace)


def factor_blocked_parallel(matrix, grid_dim=None, policy=None, *, backend=None, trace=None,
                            check_invariants: bool = False):
    """GPU drop-in for parallel.py:130-166 (same engine; the policy has nothing to steer)."""
    if policy is not None:
        workers = getattr(policy, "worker_count", None)
        if workers is not None and workers < 1:
            raise BandCholError(f"worker count must be positive, got {workers}")
    return _factor(matrix, grid_dim, trace)


def solve_with_factor(factor, rhs) -> np.ndarray:
    """GPU drop-in for core.py:216-240: returns x with L L^T x = rhs."""
    n, k, ld, data = check_matrix(factor)
    b = np.asarray(rhs, dtype=np.float64)
    if b.shape != (n,):
        raise ShapeMismatch(f"rhs shape {b.shape} does not match dimension {n}")
    torch = _torch()
    dab = torch.from_numpy(data).to("cuda")
    db = torch.from_numpy(np.ascontiguousarray(b)).to("cuda")
    info = dpbtrs_device(dab, n, k, ld, db)
    info_h = int(info.item())
    if info_h > 0:
        raise SingularFactor(f"factor diagonal not positive at column {info_h - 1}")
    return db.cpu().numpy()


# -- batched host API -------------------------------------------------------------

def _batch_array(data: np.ndarray, n: int, ld: int) -> np.ndarray:
    a = np.asarray(data)
    if a.dtype != np.float64 or a.ndim != 2 or a.shape[1] != ld * n or not a.flags.c_contiguous:
        raise ShapeMismatch(f"batched band data must be C-contiguous float64 (batch, {ld * n})")
    return a


def factor_batched(data: np.ndarray, dim: int, bandwidth: int, lead_dim: int | None = None) -> np.ndarray:
    """Factor every row of `data` (batch, lead_dim*dim) in place; returns per-matrix info.

    Raises NotPositiveDefinite for the first failing matrix (its `.matrix` index is set).
    """
    ld = bandwidth + 1 if lead_dim is None else lead_dim
    a = _batch_array(data, dim, ld)
    torch = _torch()
    dev = torch.from_numpy(a).to("cuda")
    info = dpbtrf_batched_device(dev, dim, bandwidth, ld, a.shape[0]).cpu().numpy()
    a[...] = dev.cpu().numpy()
    _raise_batch(info)
    return info


def factor_solve_batched(data: np.ndarray, rhs: np.ndarray, dim: int, bandwidth: int,
                         lead_dim: int | None = None) -> np.ndarray:
    """Factor every matrix in place and solve its system; rhs (batch, dim) -> x in place."""
    ld = bandwidth + 1 if lead_dim is None else lead_dim
    a = _batch_array(data, dim, ld)
    r = np.asarray(rhs)
    if r.dtype != np.float64 or r.shape != (a.shape[0], dim) or not r.flags.c_contiguous:
        raise ShapeMismatch(f"rhs must be C-contiguous float64 ({a.shape[0]}, {dim})")
    torch = _torch()
    dab = torch.from_numpy(a).to("cuda")
    db = torch.from_numpy(r).to("cuda")
    info = dpbsv_batched_device(dab, dim, bandwidth, ld, db, a.shape[0]).cpu().numpy()
    a[...] = dab.cpu().numpy()
    r[...] = db.cpu().numpy()
    _raise_batch(info)
    return info


def solve_batched(factors: np.ndarray, rhs: np.ndarray, dim: int, bandwidth: int,
                  lead_dim: int | None = None) -> np.ndarray:
    """x_i = solve_with_factor(L_i, rhs_i) for every matrix.  rhs (batch, dim) -> x (batch, dim),
    or (batch, nrhs, dim) -> X (batch, nrhs, dim): every right-hand side of a matrix is served
    by the same pass over its factor (bcg_dpbtrs_batched_nrhs)."""
    ld = bandwidth + 1 if lead_dim is None else lead_dim
    a = _batch_array(factors, dim, ld)
    r = np.ascontiguousarray(rhs, dtype=np.float64)
    if r.ndim == 2 and r.shape == (a.shape[0], dim):
        nrhs = 1
    elif r.ndim == 3 and r.shape[0] == a.shape[0] and r.shape[2] == dim:
        nrhs = r.shape[1]
    else:
        raise ShapeMismatch(f"rhs must be ({a.shape[0]}, {dim}) or ({a.shape[0]}, nrhs, {dim})")
    torch = _torch()
    dab = torch.from_numpy(a).to("cuda")
    db = torch.from_numpy(r.copy()).to("cuda")
    info = dpbtrs_batched_device(dab, dim, bandwidth, ld, db, a.shape[0], nrhs=nrhs).cpu().numpy()
    bad = np.nonzero(info)[0]
    if bad.size:
        err = SingularFactor(f"matrix {bad[0]}: factor diagonal not positive at column {info[bad[0]] - 1}")
        err.matrix = int(bad[0])
        raise err
    return db.cpu().numpy()


def solve_many(factor, rhs) -> np.ndarray:
    """Several right-hand sides against one factor: rhs (nrhs, N) -> X (nrhs, N), one pass
    over L per 16 right-hand sides (the repeated solves of an interior-point iteration,
    PAPER.md:20).  Same checks and errors as solve_with_factor (core.py:216-240)."""
    n, k, ld, data = check_matrix(factor)
    b = np.asarray(rhs, dtype=np.float64)
    if b.ndim != 2 or b.shape[1] != n:
        raise ShapeMismatch(f"rhs shape {b.shape} is not (nrhs, {n})")
    torch = _torch()
    dab = torch.from_numpy(data).to("cuda")
    db = torch.from_numpy(np.ascontiguousarray(b).copy()).to("cuda")
    info = dpbtrs_device(dab, n, k, ld, db, nrhs=b.shape[0])
    info_h = int(info.item())
    if info_h > 0:
        raise SingularFactor(f"factor diagonal not positive at column {info_h - 1}")
    return db.cpu().numpy()


def _raise_batch(info: np.ndarray) -> None:
    bad = np.nonzero(info)[0]
    if bad.size:
        err = NotPositiveDefinite(int(info[bad[0]]) - 1,
                                  f"matrix {bad[0]} is not positive definite at column {info[bad[0]] - 1}")
        err.matrix = int(bad[0])
        raise err


def library_version() -> int:
    return int(_lib.load().bcg_version())


__all__ = [
    "band_residual_device", "band_residual_batched_device", "residual_norm",
    "TraceEvent", "dpbtrf_device", "dpbtrf_batched_device", "dpbtrs_device", "dpbtrs_batched_device",
    "dpbsv_batched_device", "factor_blocked_serial", "factor_blocked_parallel", "solve_with_factor",
    "factor_batched", "factor_solve_batched", "solve_batched", "solve_many", "library_version",
    "BatchedBandSolver", "pinned_empty",
]


# -- repeated batched solves with host buffers (interior-point loop) -----------------

def pinned_empty(shape, dtype=np.float64) -> np.ndarray:
    """Page-locked host array (so host<->device copies run at full PCIe rate, async)."""
    torch = _torch()
    t = torch.empty(shape, dtype=torch.float64 if dtype == np.float64 else torch.int32, pin_memory=True)
    return t.numpy()  # the ndarray's base is the tensor: it keeps the pinned pages alive


class BatchedBandSolver:
    """Device-resident workspace for repeated factor + solve of a fixed-shape batch.

    `factor_solve(ab_host, b_host)` copies the batch in, factors every matrix and
    solves its system (bcg_dpbsv_batched), and copies L and x back into the same
    host arrays.  Three streams form a pipeline over `chunks` slices of the batch:
    host->device copies run back to back on one copy stream, each chunk's kernel starts
    when its slice has landed, and device->host copies drain on a third stream, so both
    PCIe directions stay busy and only the last chunk's kernel and read-back are
    exposed.  Host arrays from `pinned_empty` give asynchronous copies.  Raises
    NotPositiveDefinite (with `.matrix`) after the whole batch completes if any
    matrix failed.
    """

    def __init__(self, batch: int, dim: int, bandwidth: int, lead_dim: int | None = None,
                 chunks: int = 16):
        torch = _torch()
        self.torch = torch
        self.batch, self.n, self.kd = int(batch), int(dim), int(bandwidth)
        self.ld = self.kd + 1 if lead_dim is None else int(lead_dim)
        self.chunks = max(1, min(int(chunks), self.batch))
        self.ab = torch.empty((self.batch, self.ld * self.n), dtype=torch.float64, device="cuda")
        self.b = torch.empty((self.batch, self.n), dtype=torch.float64, device="cuda")
        self.info = torch.zeros(self.batch, dtype=torch.int32, device="cuda")
        self.h2d, self.comp, self.d2h = (torch.cuda.Stream() for _ in range(3))
        bounds = np.linspace(0, self.batch, self.chunks + 1).astype(int)
        self.ranges = [(int(bounds[i]), int(bounds[i + 1])) for i in range(self.chunks)
                       if bounds[i + 1] > bounds[i]]
        self.launches = 0

    def factor_solve(self, ab_host: np.ndarray, b_host: np.ndarray, check: bool = True) -> np.ndarray:
        torch = self.torch
        a = _batch_array(ab_host, self.n, self.ld)
        if a.shape[0] != self.batch or b_host.shape != (self.batch, self.n):
            raise ShapeMismatch("host arrays do not match the solver's batch shape")
        ta = torch.from_numpy(a)
        tb = torch.from_numpy(b_host)
        cur = torch.cuda.current_stream()
        for s in (self.h2d, self.comp, self.d2h):
            s.wait_stream(cur)
        landed, done = [], []
        with torch.cuda.stream(self.h2d):
            for lo, hi in self.ranges:
                self.ab[lo:hi].copy_(ta[lo:hi], non_blocking=True)
                self.b[lo:hi].copy_(tb[lo:hi], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.h2d)
                landed.append(ev)
        with torch.cuda.stream(self.comp):
            for (lo, hi), ev in zip(self.ranges, landed):
                self.comp.wait_event(ev)
                dpbsv_batched_device(self.ab[lo:hi], self.n, self.kd, self.ld, self.b[lo:hi], hi - lo,
                                     info=self.info[lo:hi], stream=self.comp)
                self.launches += 1
                e2 = torch.cuda.Event()
                e2.record(self.comp)
                done.append(e2)
        with torch.cuda.stream(self.d2h):
            for (lo, hi), ev in zip(self.ranges, done):
                self.d2h.wait_event(ev)
                ta[lo:hi].copy_(self.ab[lo:hi], non_blocking=True)
                tb[lo:hi].copy_(self.b[lo:hi], non_blocking=True)
        for s in (self.h2d, self.comp, self.d2h):
            cur.wait_stream(s)
        info = self.info.cpu().numpy()  # synchronises
        if check:
            _raise_batch(info)
        return info
