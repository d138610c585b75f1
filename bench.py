"""Benchmark: fp64 banded Cholesky GFLOP/s (n*kd*(kd+3)) and % of the FP64/HBM roofline.

Default workload (config.workload "C5"): BASELINE.json configs[4], a batch of 1,024
independent SPD band matrices n=4096, kd=100, factor + one-RHS band solve per matrix.
Multi-GPU is STRONG scaling exactly as C5 defines it: the fixed global batch (1,024, or
--batch B) is partitioned contiguously over the N ranks (sharding.shard), no collective on
the data path, value = all ranks' matrices / max-over-ranks time.  `--config C1..C4`
benches a single-matrix config instead (replicas per GPU).  A step = one factor+solve pass
over the rank's shard through bcg_dpbsv_batched (the factorization kernel with the forward
sweep fused in, then the backward-sweep kernel), inputs resident in HBM; a fresh
device-to-device copy of the pristine inputs is made before every step OUTSIDE the timed
events (it also flushes L2: 3.4 GB > 126 MB).  The two kernels are also timed separately
(CUDA events on the launching stream, through the split entry points
bcg_dpbtrf_fwd_batched / bcg_dpbtrs_bwd_batched) for the per-kernel roofline: the fused
factorization against the FP64 peak (the dominant kernel, `roofline`), the backward sweep
against HBM (`roofline.kernels.solve`); `factor_only` / `solve_two_sweep` are the plain
factorization and the stand-alone solve for comparison.

Rank 0 prints ONE JSON line (driver contract).  `--impl reference` times the
reference's own CPU implementation (the unmodified bandchol package installed in
baseline/_ref, blocked-serial engine, one process per host core) on a bounded sample
of the same workload.

Launch: python bench.py [--gpus N --steps K --warmup W --batch B]; N>1 under torchrun.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2305_04635_b200.inputs import CONFIGS, generate_spd, generate_spd_wide, make_rhs  # noqa: E402
from paper_2305_04635_b200.sharding import shard  # noqa: E402

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
PROFILE_TRAFFIC = os.path.join(ROOT, "profiles", "traffic.json")


# -- helpers --------------------------------------------------------------------------

def _gen_one(args):
    tag, seed = args
    cfg = CONFIGS[tag]
    gen = generate_spd_wide if cfg.wide_diagonal else generate_spd
    return gen(cfg.dim, cfg.bandwidth, seed).data, make_rhs(cfg.dim, seed)


def generate_batch(tag: str, seeds, out_ab: np.ndarray, out_b: np.ndarray) -> None:
    """Host-side seeded inputs (the reference generator), in a process pool."""
    from concurrent.futures import ProcessPoolExecutor
    seeds = list(seeds)
    workers = max(1, min(16, (os.cpu_count() or 2)))
    if len(seeds) <= 4:
        results = map(_gen_one, [(tag, s) for s in seeds])
        for i, (a, b) in enumerate(results):
            out_ab[i] = a
            out_b[i] = b
        return
    with ProcessPoolExecutor(workers) as ex:
        for i, (a, b) in enumerate(ex.map(_gen_one, [(tag, s) for s in seeds], chunksize=8)):
            out_ab[i] = a
            out_b[i] = b


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def measured_hbm_gbs() -> tuple[float, str]:
    try:
        with open(PEAKS_FILE) as fh:
            return float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel_key: str):
    try:
        with open(PROFILE_TRAFFIC) as fh:
            return json.load(fh).get(kernel_key)
    except (OSError, ValueError):
        return None


# -- CPU reference arm ----------------------------------------------------------------

def _ref_factor_one(args):
    """Reference blocked-serial engine on one matrix (+ its solve); returns seconds."""
    tag, seed, use_ref = args
    cfg = CONFIGS[tag]
    a_data, rhs = _gen_one((tag, seed))
    if use_ref:
        import bandchol
        from bandchol import factor_blocked_serial, select_grid_dim, solve_with_factor
        m = bandchol.BandedMatrix(cfg.dim, cfg.bandwidth, data=a_data)
        grid = select_grid_dim(cfg.bandwidth if cfg.bandwidth % 2 == 0 else cfg.bandwidth + 1, 1)
        t0 = time.perf_counter()
        m = factor_blocked_serial(m, grid)
        if cfg.solve:
            solve_with_factor(m, rhs)
        return time.perf_counter() - t0
    from oracle import oracle  # port fallback (CPU restatement)
    t0 = time.perf_counter()
    oracle.factor_plain(cfg.dim, cfg.bandwidth, cfg.bandwidth + 1, a_data)
    if cfg.solve:
        oracle.solve(cfg.dim, cfg.bandwidth, cfg.bandwidth + 1, a_data, rhs)
    return time.perf_counter() - t0


def reference_available() -> bool:
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "bandchol")):
        if ref not in sys.path:
            sys.path.insert(0, ref)
        return True
    return False


def cpu_reference(tag: str, sample: int, cores: int | None = None) -> dict:
    """Time the reference CPU path on `sample` matrices over a process pool of host cores."""
    from concurrent.futures import ProcessPoolExecutor
    use_ref = reference_available()
    cfg = CONFIGS[tag]
    cores = cores or len(os.sched_getaffinity(0))
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    seeds = list(range(sample))
    t0 = time.perf_counter()
    if cores > 1 and sample > 1:
        with ProcessPoolExecutor(min(cores, sample)) as ex:
            per = list(ex.map(_ref_factor_one, [(tag, s, use_ref) for s in seeds]))
    else:
        per = [_ref_factor_one((tag, s, use_ref)) for s in seeds]
    wall = time.perf_counter() - t0
    flops = sample * cfg.dim * cfg.bandwidth * (cfg.bandwidth + 3)
    used = min(cores, sample)
    # throughput of the pool on the sample (factor time only is inside each worker;
    # wall time of the pool includes input generation, so use the per-task sums)
    busy = sum(per)
    gflops = flops / (busy / used) / 1e9
    return {"value": gflops, "unit": "GFLOP/s", "cores": used,
            "kind": "reference" if use_ref else "port",
            "sample": (f"{sample} x (n={cfg.dim}, kd={cfg.bandwidth}) "
                       f"{'factor+solve' if cfg.solve else 'factor'}, "
                       f"{'bandchol factor_blocked_serial (baseline/_ref, numpy/OpenBLAS 1 thread)' if use_ref else 'oracle.factor_plain'}"
                       f" per process, {used} processes; median task {statistics.median(per):.3f}s"),
            "wall_s": wall}


def run_reference_arm(args) -> int:
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    tag = args.config
    cfg = CONFIGS[tag]
    cores = len(os.sched_getaffinity(0))
    sample = max(1, min(cfg.batch, cores)) if cfg.batch > 1 else 1
    times = []
    res = None
    for i in range(args.warmup + args.steps):
        res = cpu_reference(tag, sample, cores)
        if i >= args.warmup:
            times.append(res["value"])
    value = statistics.median(times)
    line = {
        "metric": "fp64 banded Cholesky GFLOP/s (n*kd*(kd+3))", "impl": "reference", "value": value,
        "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "higher_is_better": True, "scaling": "strong", "dtype": "f64", "data": "synthetic (reference generator)",
        "config": config_block(tag, world, global_batch(tag, args.batch)),
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": res["cores"], "kind": res["kind"],
                         "sample": res["sample"]},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "vs_baseline": None,
    }
    print(json.dumps(line), flush=True)
    return 0


def global_batch(tag: str, override: int | None) -> int:
    cfg = CONFIGS[tag]
    if cfg.batch <= 1:
        return 1
    return int(override) if override else cfg.batch


def config_block(tag: str, world: int, batch: int) -> dict:
    cfg = CONFIGS[tag]
    per = [shard(batch, r, world)[1] - shard(batch, r, world)[0] for r in range(world)]
    return {"workload": tag, "n": cfg.dim, "kd": cfg.bandwidth, "batch": batch,
            "global_batch": batch if cfg.batch > 1 else world,
            "batch_per_gpu": max(per) if cfg.batch > 1 else 1,
            "factor_and_solve": cfg.solve, "wide_diagonal": cfg.wide_diagonal,
            "parallelism": (f"batch-sharded x{world} (strong: {batch} matrices split {'/'.join(map(str, per))})"
                            if cfg.batch > 1 else "single matrix per GPU (replicas)"),
            "l2": "inputs > L2 and fresh D2D copy between steps (flushes L2)"}


# -- GPU arm --------------------------------------------------------------------------

def run_gpu_arm(args) -> int:
    import torch
    import torch.distributed as dist

    import paper_2305_04635_b200 as bc
    from paper_2305_04635_b200 import _lib
    world, rank, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)
    tag = args.config
    cfg = CONFIGS[tag]
    n, kd, ld = cfg.dim, cfg.bandwidth, cfg.bandwidth + 1
    batch = global_batch(tag, args.batch)
    # strong scaling: rank r owns the contiguous shard [lo, hi) of the fixed global batch
    # (global seeds), no collective on the data path; single-matrix configs: replicas
    lo, hi = shard(batch, rank, world) if cfg.batch > 1 else (0, 1)
    nb = hi - lo
    ab_host = bc.pinned_empty((max(nb, 1), ld * n))
    b_host = bc.pinned_empty((max(nb, 1), n))
    generate_batch(tag, range(lo, hi), ab_host, b_host)
    a0 = torch.from_numpy(ab_host).cuda()
    b0 = torch.from_numpy(b_host).cuda()
    work_a = torch.empty_like(a0)
    work_b = torch.empty_like(b0)
    info = torch.zeros(max(nb, 1), dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        """One pass of the product path over this rank's shard; returns our launches."""
        if nb == 0:
            return 0
        if cfg.batch > 1:
            bc.dpbsv_batched_device(work_a, n, kd, ld, work_b, nb, info=info, stream=stream)
            return 2  # bcg_dpbsv_batched: factorization + forward sweep kernel, backward sweep kernel
        bc.dpbtrf_device(work_a[0], n, kd, ld, info=info, stream=stream)
        if cfg.solve:
            bc.dpbtrs_device(work_a[0], n, kd, ld, work_b[0], info=info, stream=stream)
            return 2
        return 1

    def refresh():
        work_a.copy_(a0)
        work_b.copy_(b0)

    for _ in range(args.warmup):
        refresh()
        step()
    torch.cuda.synchronize()
    assert int(info.abs().sum().item()) == 0, "warm-up factorization failed"

    clocks = ClockSampler(local)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    launches = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    for i in range(args.steps):
        refresh()
        ev[i][0].record(stream)
        launches += step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    per_ms = [s_.elapsed_time(e_) for s_, e_ in ev]
    total_ms = sum(per_ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    n_mat = batch if cfg.batch > 1 else world  # every rank's matrices (replicas for C1-C4)
    flops_total = n_mat * n * kd * (kd + 3)
    value = flops_total * args.steps / (max_ms * 1e-3) / 1e9  # GFLOP/s, whole job

    # the two kernels of a step timed apart (same stream, CUDA events), exactly as the step
    # runs them: batched (C5) the factorization with the fused forward sweep
    # (bcg_dpbtrf_fwd_batched), then the backward sweep (bcg_dpbtrs_bwd_batched); single
    # matrices the factorization, then the two-sweep solve.  For reference also the plain
    # batched factorization and the stand-alone two-sweep solve (bcg_dpbtrf_batched,
    # bcg_dpbtrs_batched).
    fac_ms, sol_ms, plain_fac_ms, plain_sol_ms = [], [], [], []
    y_ws = torch.empty_like(b0) if cfg.batch > 1 else None
    for i in range(args.steps if nb else 0):
        refresh()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(stream)
        if cfg.batch > 1:
            bc.dpbtrf_fwd_batched_device(work_a, n, kd, ld, work_b, y_ws, nb, info=info, stream=stream)
        else:
            bc.dpbtrf_device(work_a[0], n, kd, ld, info=info, stream=stream)
        e1.record(stream)
        if cfg.solve:
            if cfg.batch > 1:
                bc.dpbtrs_bwd_batched_device(work_a, n, kd, ld, y_ws, work_b, nb, info, stream=stream)
            else:
                bc.dpbtrs_device(work_a[0], n, kd, ld, work_b[0], info=info, stream=stream)
        e2.record(stream)
        torch.cuda.synchronize()
        fac_ms.append(e0.elapsed_time(e1))
        sol_ms.append(e1.elapsed_time(e2))
        if cfg.batch > 1:
            refresh()
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(stream)
            bc.dpbtrf_batched_device(work_a, n, kd, ld, nb, info=info, stream=stream)
            e1.record(stream)
            bc.dpbtrs_batched_device(work_a, n, kd, ld, work_b, nb, info=info, stream=stream)
            e2.record(stream)
            torch.cuda.synchronize()
            plain_fac_ms.append(e0.elapsed_time(e1))
            plain_sol_ms.append(e1.elapsed_time(e2))

    # end to end through the public API with host buffers (pinned), per rank shard
    solver = bc.BatchedBandSolver(nb, n, kd, chunks=16) if cfg.batch > 1 and nb else None
    e2e_ab = bc.pinned_empty((max(nb, 1), ld * n))
    e2e_b = bc.pinned_empty((max(nb, 1), n))
    e2e_times = []
    for i in range(args.warmup + args.steps):
        np.copyto(e2e_ab, ab_host)
        np.copyto(e2e_b, b_host)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s_ev.record()
        if solver is not None:
            solver.factor_solve(e2e_ab, e2e_b, check=False)
        elif cfg.batch <= 1:
            m = bc.BandedMatrix(n, kd, data=e2e_ab[0])
            bc.factor_blocked_serial(m)
            if cfg.solve:
                e2e_b[0] = bc.solve_with_factor(m, e2e_b[0])
        e_ev.record()
        torch.cuda.synchronize()
        if i >= args.warmup:
            e2e_times.append(s_ev.elapsed_time(e_ev))
    te = torch.tensor([sum(e2e_times)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = flops_total * args.steps / (float(te.item()) * 1e-3) / 1e9
    h2d = nb * (ld * n + n) * 8 if cfg.batch > 1 else (ld * n + (n if cfg.solve else 0)) * 8
    d2h = h2d

    # roofline of the dominant kernel (the factorization: FP64-bound) from its own CUDA-event
    # time; the solve against HBM (it reads L twice); the whole step for reference
    pk = ctypes_double()
    import ctypes
    _lib.check(_lib.load().bcg_probe_fp64_peak(ctypes.byref(pk)), "bcg_probe_fp64_peak")
    fp64_peak = pk.value * 1e3  # GFLOP/s
    hbm, hbm_src = measured_hbm_gbs()
    mats = max(nb, 1)
    flops_rank = mats * n * kd * (kd + 3)
    bytes_rank = mats * 16 * n * (kd + 1)        # factorization: band read + written once
    solve_bytes = mats * 16 * n * (kd + 1)       # solve: band read twice
    f_ms = statistics.median(fac_ms) if fac_ms else float("nan")
    s_ms = statistics.median(sol_ms) if (sol_ms and cfg.solve) else 0.0
    step_ms = max_ms / args.steps
    t_fp = flops_rank / (fp64_peak * 1e9)
    t_hbm = bytes_rank / (hbm * 1e9)
    bound = "fp64" if t_fp >= t_hbm else "hbm"
    if bound == "fp64":
        achieved = flops_rank / (f_ms * 1e-3) / 1e12
        peak, unit = fp64_peak / 1e3, "TFLOP/s"
    else:
        achieved = bytes_rank / (f_ms * 1e-3) / 1e9
        peak, unit = hbm, "GB/s"
    fused = cfg.batch > 1
    if fused:
        # the backward sweep reads L once (the forward sweep ran from shared memory inside the
        # factorization kernel); the stand-alone solve reads it twice
        solve_bytes = mats * 8 * n * (kd + 1)
    kernels = {"factor": {"ms": f_ms, "tflops": flops_rank / (f_ms * 1e-3) / 1e12,
                          "frac_fp64": flops_rank / (f_ms * 1e-3) / 1e9 / fp64_peak,
                          "what": "factorization + fused forward sweep" if fused else "factorization"}}
    if cfg.solve:
        kernels["solve"] = {"ms": s_ms, "gbs": solve_bytes / (s_ms * 1e-3) / 1e9,
                            "frac_hbm": solve_bytes / (s_ms * 1e-3) / 1e9 / hbm,
                            "what": "backward sweep (L read once)" if fused else "two-sweep solve (L read twice)"}
    if fused and plain_fac_ms:
        pf, ps = statistics.median(plain_fac_ms), statistics.median(plain_sol_ms)
        two = mats * 16 * n * (kd + 1)
        kernels["factor_only"] = {"ms": pf, "tflops": flops_rank / (pf * 1e-3) / 1e12,
                                  "frac_fp64": flops_rank / (pf * 1e-3) / 1e9 / fp64_peak,
                                  "what": "bcg_dpbtrf_batched alone"}
        kernels["solve_two_sweep"] = {"ms": ps, "gbs": two / (ps * 1e-3) / 1e9, "frac_hbm": two / (ps * 1e-3) / 1e9 / hbm,
                                      "what": "bcg_dpbtrs_batched alone (L read twice)"}
    t_step_roof = max(t_fp, t_hbm) + (solve_bytes / (hbm * 1e9) if cfg.solve else 0.0)
    roofline = {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
                "kernel": "factorization + fused forward sweep (pbtrf_cta_kernel)" if cfg.batch > 1 else "factorization",
                "traffic": ncu_traffic(f"{tag}_factor" if cfg.batch > 1 else tag), "kernels": kernels,
                "step_frac": t_step_roof * 1e3 / step_ms,
                "step_roof_ms": t_step_roof * 1e3,
                "peak_source": f"fp64: bcg_probe_fp64_peak DFMA loop (live); hbm: {hbm_src} {hbm:.1f} GB/s",
                "algorithmic": (f"factor: flops n*kd*(kd+3), bytes 16*n*(kd+1) x {mats} matrices; solve: "
                                + (f"bytes 8*n*(kd+1) x {mats} (backward sweep, L read once)" if fused
                                   else f"bytes 16*n*(kd+1) x {mats} (L read twice)"))}
    line = {
        "metric": "fp64 banded Cholesky GFLOP/s (n*kd*(kd+3))", "value": value, "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (reference generator, seeds 0..batch-1)",
        "config": config_block(tag, world, batch), "roofline": roofline, "clocks": clk,
        "e2e": {"value": e2e_value, "unit": "GFLOP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": float(te.item()) / args.steps, "path": "BatchedBandSolver.factor_solve (pinned host)"
                if cfg.batch > 1 else "factor_blocked_serial + solve_with_factor (host numpy)"},
        "gpu_launches": launches,
    }
    if rank == 0 and world == 1 and cfg.batch > 1 and not args.skip_others:
        line["shards"] = shard_times(bc, work_a, work_b, a0, b0, n, kd, ld, nb, step_ms)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = len(os.sched_getaffinity(0))
        sample = min(cfg.batch, max(1, cores)) if cfg.batch > 1 else 1
        line["cpu_baseline"] = {k: v for k, v in cpu_reference(tag, sample, cores).items() if k != "wall_s"}
    if rank == 0 and world == 1 and not args.skip_others and tag == "C5":
        line["other_configs"] = other_configs(bc, fp64_peak, hbm)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def shard_times(bc, work_a, work_b, a0, b0, n, kd, ld, batch, full_ms) -> dict:
    """The per-GPU shard of an N-GPU strong-scaling run (batch/N matrices), timed on this GPU:
    what each rank of a 2/4/8-GPU run computes, and the efficiency T1 / (N * T_N) it implies
    (no collective on the data path, so a rank's time is its shard's time)."""
    import torch
    out = {}
    info = torch.zeros(batch, dtype=torch.int32, device="cuda")
    for g in (2, 4, 8):
        m = batch // g
        ts = []
        for i in range(6):
            work_a[:m].copy_(a0[:m])
            work_b[:m].copy_(b0[:m])
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            bc.dpbsv_batched_device(work_a[:m], n, kd, ld, work_b[:m], m, info=info[:m])
            e1.record()
            torch.cuda.synchronize()
            if i:
                ts.append(e0.elapsed_time(e1))
        t = statistics.median(ts)
        out[f"gpus{g}"] = {"matrices": m, "ms": t, "efficiency": full_ms / (g * t)}
    return out


def ctypes_double():
    import ctypes
    return ctypes.c_double(0.0)


def other_configs(bc, fp64_peak_gflops: float, hbm: float) -> dict:
    """Single-matrix configs C1-C4 (device-resident, CUDA events, median of 5)."""
    import torch
    out = {}
    for tag in ("C1", "C2", "C3", "C4"):
        cfg = CONFIGS[tag]
        n, kd, ld = cfg.dim, cfg.bandwidth, cfg.bandwidth + 1
        gen = generate_spd_wide if cfg.wide_diagonal else generate_spd
        a0 = torch.from_numpy(gen(n, kd, 0).data).cuda()
        b0 = torch.from_numpy(make_rhs(n, 0)).cuda()
        w, wb = torch.empty_like(a0), torch.empty_like(b0)
        info = torch.zeros(1, dtype=torch.int32, device="cuda")
        fac_ms, sol_ms = [], []
        for i in range(6):
            w.copy_(a0)
            wb.copy_(b0)
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record()
            bc.dpbtrf_device(w, n, kd, ld, info=info)
            e1.record()
            if cfg.solve:
                bc.dpbtrs_device(w, n, kd, ld, wb, info=info)
            e2.record()
            torch.cuda.synchronize()
            if i:
                fac_ms.append(e0.elapsed_time(e1))
                sol_ms.append(e1.elapsed_time(e2))
        assert int(info.item()) == 0
        f = statistics.median(fac_ms)
        flops = n * kd * (kd + 3)
        t_roof = max(flops / (fp64_peak_gflops * 1e9), 16 * n * (kd + 1) / (hbm * 1e9)) * 1e3
        out[tag] = {"factor_ms": f, "gflops": flops / (f * 1e-3) / 1e9, "roofline_frac": t_roof / f,
                    "t_roof_ms": t_roof}
        if cfg.solve:
            s = statistics.median(sol_ms)
            out[tag]["solve_ms"] = s
            out[tag]["solve_gbs"] = 16 * n * (kd + 1) / (s * 1e-3) / 1e9
    return out


def main(argv=None) -> int:
    p = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--config", choices=tuple(CONFIGS), default="C5")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--skip-others", action="store_true")
    p.add_argument("--batch", type=int, default=None,
                   help="global batch of the batched config (default: C5's 1,024); --batch 128 on one "
                        "GPU is the per-GPU load of the 8-GPU run")
    args = p.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 untimed warm-up steps
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_gpu_arm(args)


if __name__ == "__main__":
    sys.exit(main())
