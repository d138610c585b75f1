"""Quick device timings of the library entry points (CUDA events), for development.

usage: python tools/timing.py [c5|single|rhs|all] [--batch B]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_04635_b200 as bc  # noqa: E402
from paper_2305_04635_b200.inputs import CONFIGS, generate_spd, generate_spd_wide, make_rhs  # noqa: E402


def timed(fn, reps=3):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts), ts


def c5(batch):
    n, k = 4096, 100
    ld = k + 1
    a = np.stack([generate_spd(n, k, s).data for s in range(min(batch, 64))])
    reps = (batch + a.shape[0] - 1) // a.shape[0]
    a = np.concatenate([a] * reps)[:batch]
    b = np.stack([make_rhs(n, s) for s in range(batch)])
    a0 = torch.from_numpy(a).cuda()
    b0 = torch.from_numpy(b).cuda()
    w, wb = a0.clone(), b0.clone()
    info = torch.zeros(batch, dtype=torch.int32, device="cuda")
    flops = batch * n * k * (k + 3)

    def fac():
        w.copy_(a0)
        torch.cuda.synchronize()
        return bc.dpbtrf_batched_device(w, n, k, ld, batch, info=info)

    def sv():
        return bc.dpbsv_batched_device(w, n, k, ld, wb, batch, info=info)

    def refresh():
        w.copy_(a0); wb.copy_(b0)
    out = {}
    for name, f in (("dpbtrf_batched", lambda: bc.dpbtrf_batched_device(w, n, k, ld, batch, info=info)),
                    ("dpbsv_batched", sv),
                    ("dpbtrs_batched", lambda: bc.dpbtrs_batched_device(w, n, k, ld, wb, batch, info=info))):
        ts = []
        for _ in range(3):
            refresh()
            if name == "dpbtrs_batched":
                bc.dpbtrf_batched_device(w, n, k, ld, batch, info=info)
            torch.cuda.synchronize()
            ms, _ = timed(f, 1)
            ts.append(ms)
        out[name] = {"ms": min(ts), "gflops": flops / (min(ts) * 1e-3) / 1e9}
    assert int(info.abs().sum().item()) == 0
    print(json.dumps({"c5_batch": batch, **out}), flush=True)


def rhs_sweep():
    """Multi-right-hand-side solve: one factor, nrhs = 1..16 (one pass over L per 16), and
    the batched C5 shape with 1 and 16 right-hand sides per matrix."""
    n, k = 4096, 100
    a = generate_spd(n, k, 0)
    bc.factor_blocked_serial(a)
    dab = torch.from_numpy(a.data).cuda()
    out = {}
    for R in (1, 2, 4, 8, 16, 32):
        db = torch.from_numpy(np.stack([make_rhs(n, s) for s in range(R)])).cuda()
        ms, _ = timed(lambda: bc.dpbtrs_device(dab, n, k, k + 1, db, nrhs=R), 5)
        out[f"single_nrhs{R}_ms"] = ms
    batch = 1024
    w = dab.repeat(batch)
    info = torch.zeros(batch, dtype=torch.int32, device="cuda")
    for R in (1, 4, 16):
        db = torch.from_numpy(np.stack([make_rhs(n, s) for s in range(R)])).cuda().repeat(batch, 1)
        ms, _ = timed(lambda: bc.dpbtrs_batched_device(w, n, k, k + 1, db, batch, nrhs=R, info=info), 3)
        out[f"batch1024_nrhs{R}_ms"] = ms
        out[f"batch1024_nrhs{R}_GBs"] = 2 * batch * n * (k + 1) * 8 / (ms * 1e-3) / 1e9
    print(json.dumps(out), flush=True)


def single(tags):
    for tag in tags:
        cfg = CONFIGS[tag]
        n, k = cfg.dim, cfg.bandwidth
        gen = generate_spd_wide if cfg.wide_diagonal else generate_spd
        a0 = torch.from_numpy(gen(n, k, 0).data).cuda()
        w = a0.clone()
        info = torch.zeros(1, dtype=torch.int32, device="cuda")
        ts = []
        for _ in range(3):
            w.copy_(a0)
            torch.cuda.synchronize()
            ms, _ = timed(lambda: bc.dpbtrf_device(w, n, k, k + 1, info=info), 1)
            ts.append(ms)
        assert int(info.item()) == 0, int(info.item())
        flops = n * k * (k + 3)
        print(json.dumps({"config": tag, "factor_ms": min(ts), "gflops": flops / (min(ts) * 1e-3) / 1e9,
                          "all_ms": ts}), flush=True)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    batch = int(sys.argv[sys.argv.index("--batch") + 1]) if "--batch" in sys.argv else 296
    if what in ("c5", "all"):
        c5(batch)
    if what in ("single", "all"):
        single(["C1", "C2", "C3", "C4"])
    if what in ("rhs", "all"):
        rhs_sweep()


def trace(tag):
    """Pivot phase breakdown of the multi-CTA kernel (bcg_set_trace)."""
    from paper_2305_04635_b200 import _lib
    cfg = CONFIGS[tag]
    n, k = cfg.dim, cfg.bandwidth
    gen = generate_spd_wide if cfg.wide_diagonal else generate_spd
    a0 = torch.from_numpy(gen(n, k, 0).data).cuda()
    buf = torch.zeros(1 + 8 * (n // 16 + 2), dtype=torch.int64, device="cuda")
    lib = _lib.load()
    w = a0.clone()
    bc.dpbtrf_device(w, n, k, k + 1)
    torch.cuda.synchronize()
    lib.bcg_set_trace(buf.data_ptr(), buf.numel() * 8)
    w = a0.clone()
    bc.dpbtrf_device(w, n, k, k + 1)
    torch.cuda.synchronize()
    lib.bcg_set_trace(None, 0)
    t = buf.cpu().numpy()
    steps = int(t[0])
    st = t[1:1 + 8 * steps].reshape(steps, 8).astype(np.float64)
    # pivot stamps: 0 step start, 1 POTRF done, 2 stage-A barrier passed (lookback done too),
    # 3 TRSM product done, 4 SYRK done, 5 closing barrier; 6 (service thread) L(j+1,j-1) flag
    # seen, 7 (warp 2) lookback product done
    # pivot stamps (SM cycles): 0 step start, 1 POTRF done, 2 stage barrier passed, 4 TRSM + SYRK
    # done; service: 7 / 6 flags of A(j+1,j) / A(j+1,j+1) seen, 5 warps 6-7 done with the
    # previous step's TRSM of row j+1, 3 lookback products start
    rel = lambda k: float(np.median(st[2:-2, k] - st[2:-2, 0]))  # noqa: E731
    out = {"config": tag, "steps": steps, "unit": "cycles", "total_cycles": float(st[-1, 1] - st[0, 0]),
           "step": float(np.median(np.diff(st[:, 0]))), "potrf_done": rel(1), "stage_barrier": rel(2),
           "tiles_loaded": rel(7), "flags_seen": rel(6), "diag_warp_free": rel(5), "diag_flag_seen": rel(4),
           "diag_loaded": rel(3)}
    if t[-2] > 0:
        out["row_task_cycles"] = float(t[-3]) / float(t[-2])
    nb = (n + 31) // 32
    xs = t[1 + 8 * nb:1 + 16 * nb].reshape(nb, 8).astype(np.float64)[4:-4]
    ok = (xs[:, 7] > 0) & (xs[:, 0] > 0) & (xs[:, 3] > 0) & (xs[:, 6] > 0)
    if ok.any():
        rel = lambda k: float(np.median(xs[ok, k] - xs[ok, 7]))  # noqa: E731  ns after the pivot's step start
        out["x_ns_after_step_start"] = {"owner_last_linv_seen": rel(0), "owner_last_trsm_published": rel(1),
                                        "owner_last_deps2_seen": rel(2), "owner_last_tc_published": rel(3),
                                        "pivot_prev_linv_released": rel(6)}
        out["step_ns"] = float(np.median(np.diff(xs[:, 7])))
    wk = t[-8:-3].astype(np.float64)
    if wk.sum() > 0:
        out["worker_share"] = {k: round(float(v / wk.sum()), 3)
                               for k, v in zip(["ticket", "deps", "loads", "compute_store", "publish"], wk)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "trace":
    for tg in sys.argv[2:] or ["C2", "C3", "C4"]:
        trace(tg)


def trace_cta(tag, batch=1):
    """Phase breakdown of the one-CTA kernel (block 0, matrix 0)."""
    from paper_2305_04635_b200 import _lib
    cfg = CONFIGS[tag]
    n, k = cfg.dim, cfg.bandwidth
    a = np.stack([generate_spd(n, k, s).data for s in range(min(batch, 8))])
    a = np.concatenate([a] * ((batch + 7) // 8))[:batch]
    a0 = torch.from_numpy(a).cuda()
    buf = torch.zeros(1 + 8 * (n // 16 + 2), dtype=torch.int64, device="cuda")
    lib = _lib.load()
    w = a0.clone()
    bc.dpbtrf_batched_device(w, n, k, k + 1, batch)
    torch.cuda.synchronize()
    lib.bcg_set_trace(buf.data_ptr(), buf.numel() * 8)
    w = a0.clone()
    bc.dpbtrf_batched_device(w, n, k, k + 1, batch)
    torch.cuda.synchronize()
    lib.bcg_set_trace(None, 0)
    t = buf.cpu().numpy()
    steps = int(t[0])
    st = t[1:1 + 8 * steps].reshape(steps, 8).astype(np.float64)[:-2]
    med = lambda a, b: float(np.median(st[:, b] - st[:, a]))  # noqa: E731  (SM cycles)
    out = {"config": tag, "batch": batch, "steps": steps, "unit": "cycles",
           "trsm": med(0, 7), "wait": med(7, 1), "store_part1": med(1, 2),
           "potrf": med(3, 4), "rest_update": med(2, 5), "lookahead_total": med(2, 6),
           "step": float(np.median(np.diff(st[:, 0])))}
    print(json.dumps(out), flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "trace_cta":
    trace_cta("C1", 1)
    trace_cta("C5", 1)
    trace_cta("C5", 296)


def trace_solve(batch=1, nrhs=1):
    """Per-step phase breakdown of the streamed solve (band_sweep.cuh, CTA 0), SM cycles."""
    from paper_2305_04635_b200 import _lib
    n, k = 4096, 100
    a = np.stack([generate_spd(n, k, s).data for s in range(min(batch, 8))])
    a = np.concatenate([a] * ((batch + 7) // 8))[:batch]
    a0 = torch.from_numpy(a).cuda()
    bc.dpbtrf_batched_device(a0, n, k, k + 1, batch)
    b0 = torch.from_numpy(np.stack([make_rhs(n, s) for s in range(batch * nrhs)])).cuda()
    nblk = n // 16
    buf = torch.zeros(1 + 8 * (2 * nblk + 4), dtype=torch.int64, device="cuda")
    lib = _lib.load()
    bc.dpbtrs_batched_device(a0, n, k, k + 1, b0.clone(), batch, nrhs=nrhs)
    torch.cuda.synchronize()
    lib.bcg_set_trace(buf.data_ptr(), buf.numel() * 8)
    bc.dpbtrs_batched_device(a0, n, k, k + 1, b0.clone(), batch, nrhs=nrhs)
    torch.cuda.synchronize()
    lib.bcg_set_trace(None, 0)
    t = buf.cpu().numpy()[1:1 + 8 * 2 * nblk].reshape(2 * nblk, 8).astype(np.float64)
    med = lambda x: float(np.median(x))  # noqa: E731
    out = {"batch": batch, "nrhs": nrhs}
    for name, sl in (("fwd", slice(4, nblk - 4)), ("bwd", slice(nblk + 4, 2 * nblk - 4))):
        u = t[sl]
        out[name] = {"step": med(np.diff(u[:, 0])), "chain_wait": med(u[:, 1] - u[:, 0]),
                     "chain_work": med(u[:, 2] - u[:, 1]), "far_work": med(u[:, 4] - u[:, 3]),
                     "t_waits_after_subst": med(u[:, 6] - u[:, 5]), "t_work": med(u[:, 7] - u[:, 6]),
                     "chain_wake_after_t": med(u[:, 1] - u[:, 7]),
                     "t_inputs_after_prev2_chain_end": (med(u[2:, 6] - u[:-2, 2]) if name == "fwd"
                                                        else med(u[2:, 6] - u[:-2, 2]))}
    out["fwd"]["far_start_after_ydone"] = med(t[4:nblk - 4, 3] - t[4:nblk - 4, 2])
    out["total_cycles"] = float(t[-1, 2] - t[0, 0])
    print(json.dumps(out), flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "trace_solve":
    trace_solve(1)
    trace_solve(296)
    trace_solve(1, 16)


def trace_la(tag, batch=1, solve=False):
    """Phase breakdown of the pipelined one-CTA factorization (block 0, matrix 0).

    Pivot stamps per step: 0 start, 1 after waiting update(k-2), 2 after SYRK(0,0),
    3 after POTRF, 4 after waiting column 0 of update(k-1), 5 after TRSM + signal;
    worker 0: 6 after the panel signal, 7 after its share of update(k)."""
    from paper_2305_04635_b200 import _lib
    cfg = CONFIGS[tag]
    n, k = cfg.dim, cfg.bandwidth
    a = np.stack([generate_spd(n, k, s).data for s in range(min(batch, 8))])
    a = np.concatenate([a] * ((batch + 7) // 8))[:batch]
    a0 = torch.from_numpy(a).cuda()
    nblk = (n + 15) // 16
    buf = torch.zeros(1 + 8 * (3 * nblk + 6), dtype=torch.int64, device="cuda")
    lib = _lib.load()
    b0 = torch.from_numpy(np.stack([make_rhs(n, s) for s in range(batch)])).cuda()

    def run():
        w = a0.clone()
        if solve:
            bc.dpbsv_batched_device(w, n, k, k + 1, b0.clone(), batch)
        else:
            bc.dpbtrf_batched_device(w, n, k, k + 1, batch)
        torch.cuda.synchronize()
    run()
    lib.bcg_set_trace(buf.data_ptr(), buf.numel() * 8)
    run()
    lib.bcg_set_trace(None, 0)
    t = buf.cpu().numpy()
    steps = nblk
    allst = t[1:].reshape(-1, 8).astype(np.float64)
    st = allst[:nblk][2:-2]
    wt = allst[2 * nblk + 2: 3 * nblk + 2][2:-2]
    wmed = lambda a, b: float(np.median(wt[:, b] - wt[:, a]))  # noqa: E731
    med = lambda a, b: float(np.median(st[:, b] - st[:, a]))  # noqa: E731  (SM cycles)
    out = {"config": tag, "batch": batch, "solve": solve, "steps": steps, "unit": "cycles",
           "wait_W": med(0, 1), "syrk": med(1, 2), "potrf": med(2, 3), "wait_W1": med(3, 4),
           "trsm_signal": med(4, 5), "worker_wake": med(5, 6), "worker_step": med(6, 7),
           "step": float(np.median(np.diff(st[:, 0]))),
           "w_load": wmed(0, 1), "w_barA": wmed(1, 2), "w_trsm": wmed(2, 3), "w_col0": wmed(3, 4),
           "w_barB": wmed(4, 5), "w_rest": wmed(5, 6), "fwd_step": float(np.median(wt[:, 7]))}
    print(json.dumps(out), flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "trace_la":
    trace_la("C5", 1)
    trace_la("C5", 296)
    trace_la("C5", 1, True)
    trace_la("C5", 296, True)
