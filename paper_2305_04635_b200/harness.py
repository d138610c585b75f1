"""GPU benchmark harness with the reference's CSV schema.

Mirrors ``bandchol.bench`` (pkg/src/bandchol/bench.py): one record per (bandwidth, impl),
median time over repetitions after one untimed warm-up, throughput from the exact
analytic operation count ``flops_exact`` (bench.py:150-151, flops.py:29-39), optional
residual check, and the CSV header ``N,k,n,workers,impl,backend,reps,median_seconds,
gflops,residual`` written with 17 significant digits (bench.py:33, :205-220), so the
paper-style sweeps and the reference's plotting read GPU rows unchanged.

Implementations (the reference harness rejects a backend named ``cuda``,
pkg/tests/test_bench.py:108-109, so the tags are new):

* ``b200``       -- the device-resident factorization (``dpbtrf_device``): a fresh
  device-to-device copy of the input before every repetition, outside the CUDA events
  that time the call.
* ``b200-host``  -- the reference-shaped host call ``factor_blocked_serial(copy)``
  timed with the host clock, host<->device copies included (the reference also copies
  the matrix inside its timed region, bench.py:149-151).

``n`` and ``workers`` are empty (the GPU engine has no window grid or worker pool);
``backend`` is ``sm_100a``.  The bandwidth is used as given: the GPU engine needs none of
the reference's padding (bench.py:70-78).  Residuals use the device ``residual_norm``.
"""

from __future__ import annotations

import argparse
import statistics
import sys
import time
from dataclasses import dataclass

from .errors import BandCholError, InvalidBandwidth, ShapeMismatch
from .flops import flops_exact
from .inputs import generate_spd

IMPL_CHOICES = ("b200", "b200-host")
BACKEND = "sm_100a"
CSV_HEADER = "N,k,n,workers,impl,backend,reps,median_seconds,gflops,residual"
RESIDUAL_LIMIT = 1e-10


@dataclass
class BenchConfig:
    dim: int
    bandwidths: tuple
    impls: tuple = IMPL_CHOICES
    repetitions: int = 10
    seed: int = 0
    check: bool = False
    out: str | None = None


@dataclass
class BenchRecord:
    dim: int
    bandwidth: int
    grid_dim: int | None
    workers: int | None
    impl: str
    backend: str | None
    repetitions: int
    median_seconds: float | None
    gflops: float | None
    residual: float | None

    @property
    def failed(self) -> bool:
        return self.median_seconds is None


def validate(config: BenchConfig) -> list[int]:
    """The reference harness's argument checks (bench.py:80-113), minus the grid rules."""
    if config.dim < 1:
        raise ShapeMismatch(f"dimension must be positive, got {config.dim}")
    if config.repetitions < 1:
        raise BandCholError(f"repetitions must be positive, got {config.repetitions}")
    if not config.bandwidths:
        raise BandCholError("at least one bandwidth is required")
    if not config.impls:
        raise BandCholError("at least one implementation is required")
    for impl in config.impls:
        if impl not in IMPL_CHOICES:
            raise BandCholError(f"unknown implementation {impl!r}")
    out = []
    for k in config.bandwidths:
        if k < 0:
            raise InvalidBandwidth(f"bandwidth must be non-negative, got {k}")
        if k >= config.dim:
            raise InvalidBandwidth(f"bandwidth {k} must stay below dimension {config.dim}")
        out.append(int(k))
    return out


def _time_device(matrix, reps: int) -> tuple[list[float], object]:
    from .engine import _torch, dpbtrf_device

    torch = _torch()
    n, k, ld = matrix.dim, matrix.bandwidth, matrix.lead_dim
    src = torch.from_numpy(matrix.data.copy()).to("cuda")
    work = torch.empty_like(src)
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for rep in range(reps + 1):  # rep 0: warm-up, never timed
        work.copy_(src)
        torch.cuda.synchronize()
        e0.record()
        dpbtrf_device(work, n, k, ld, info)
        e1.record()
        e1.synchronize()
        if int(info.item()):
            from .errors import NotPositiveDefinite
            raise NotPositiveDefinite(int(info.item()) - 1)
        if rep:
            times.append(e0.elapsed_time(e1) * 1e-3)
    return times, work


def _time_host(matrix, reps: int, timer) -> tuple[list[float], object]:
    from .engine import factor_blocked_serial

    factor_blocked_serial(matrix.copy())  # warm-up
    times, last = [], None
    for _ in range(reps):
        t0 = timer()
        last = factor_blocked_serial(matrix.copy())
        times.append(timer() - t0)
    return times, last


def run_benchmark(config: BenchConfig, *, timer=time.perf_counter) -> list[BenchRecord]:
    """One record per (k, impl); a failed factorization yields a record with empty timings."""
    from .engine import _torch, band_residual_device, residual_norm

    bandwidths = validate(config)
    records: list[BenchRecord] = []
    for k in bandwidths:
        matrix = generate_spd(config.dim, k, config.seed)
        ops = flops_exact(config.dim, k)
        for impl in config.impls:
            try:
                if impl == "b200":
                    times, work = _time_device(matrix, config.repetitions)
                else:
                    times, last = _time_host(matrix, config.repetitions, timer)
            except BandCholError as exc:
                print(f"{impl} failed at N={config.dim} k={k}: {exc}", file=sys.stderr)
                records.append(BenchRecord(config.dim, k, None, None, impl, BACKEND, config.repetitions,
                                           None, None, None))
                continue
            median = statistics.median(times)
            gflops = ops / median / 1e9 if median > 0 else float("inf")
            residual = None
            if config.check:
                if impl == "b200":
                    torch = _torch()
                    a = torch.from_numpy(matrix.data.copy()).to("cuda")
                    residual = float(band_residual_device(a, work, matrix.dim, k, matrix.lead_dim,
                                                          matrix.lead_dim).item())
                else:
                    residual = residual_norm(matrix, last)
            records.append(BenchRecord(config.dim, k, None, None, impl, BACKEND, config.repetitions,
                                       median, gflops, residual))
    return records


def _fmt(value) -> str:
    if value is None:
        return ""
    if isinstance(value, float):
        return f"{value:.17g}"
    return str(value)


def emit_csv(records: list[BenchRecord], path) -> None:
    """Write records in the reference CSV schema (refuses an empty record list)."""
    if not records:
        raise BandCholError("no benchmark records to emit")
    lines = [CSV_HEADER]
    for r in records:
        lines.append(",".join([
            _fmt(r.dim), _fmt(r.bandwidth), _fmt(r.grid_dim), _fmt(r.workers), r.impl, r.backend or "",
            _fmt(r.repetitions), _fmt(r.median_seconds), _fmt(r.gflops), _fmt(r.residual),
        ]))
    with open(path, "w", encoding="utf-8", newline="") as fh:
        fh.write("\n".join(lines) + "\n")


def parse_csv(path) -> list[BenchRecord]:
    """Read back an emit_csv file (reference or GPU rows); empty fields become None."""
    with open(path, "r", encoding="utf-8") as fh:
        lines = fh.read().splitlines()
    if not lines or lines[0] != CSV_HEADER:
        raise BandCholError(f"unrecognized CSV header in {path}")
    out = []
    for line in lines[1:]:
        p = line.split(",")
        if len(p) != 10:
            raise BandCholError(f"malformed CSV row: {line!r}")
        oi = (lambda s: int(s) if s else None)
        of = (lambda s: float(s) if s else None)
        out.append(BenchRecord(int(p[0]), int(p[1]), oi(p[2]), oi(p[3]), p[4], p[5] or None, int(p[6]),
                               of(p[7]), of(p[8]), of(p[9])))
    return out


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description="GPU band Cholesky sweep in the reference CSV schema")
    ap.add_argument("--dim", "-N", type=int, required=True)
    ap.add_argument("--bandwidths", "-k", type=int, nargs="+", required=True)
    ap.add_argument("--impls", nargs="+", default=list(IMPL_CHOICES), choices=IMPL_CHOICES)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--out", default=None)
    a = ap.parse_args(argv)
    cfg = BenchConfig(a.dim, tuple(a.bandwidths), tuple(a.impls), a.reps, a.seed, a.check, a.out)
    recs = run_benchmark(cfg)
    if a.out:
        emit_csv(recs, a.out)
    else:
        print(CSV_HEADER)
        for r in recs:
            print(",".join([_fmt(r.dim), _fmt(r.bandwidth), "", "", r.impl, r.backend or "", _fmt(r.repetitions),
                            _fmt(r.median_seconds), _fmt(r.gflops), _fmt(r.residual)]))
    bad = any(r.failed for r in recs) or (a.check and any(
        r.residual is not None and r.residual > RESIDUAL_LIMIT for r in recs))
    return 1 if bad else 0


if __name__ == "__main__":  # pragma: no cover
    sys.exit(main())
