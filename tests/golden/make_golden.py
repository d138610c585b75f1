"""Generate the golden fixtures by running the REFERENCE itself (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs (committed, small):
  small_cases.npz      full arrays for small (n, k) cases: input band A, the
                       reference's factor_reference L (exactly rounded, reference.py:32-63),
                       factor_blocked_serial L where the grid allows, rhs, and
                       solve_with_factor x (core.py:216-240), residual_norm.
  fingerprints.json    SHA-256 of the input bytes (generate_spd, core.py:155-181) and of
                       the factor_reference output bytes for config-sized matrices
                       (C1, C2, C5 members), plus residuals and failure columns.
  sampled_large.npz    C2/C3/C4: sampled band columns of the reference blocked engine's L
                       (factor_blocked_serial, blocked.py:363-385), and solve x for C2/C5.

Nothing at test time imports the reference: the tests only read these files.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import bandchol  # noqa: E402  (the reference package)
from bandchol import (BandedMatrix, NotPositiveDefinite, factor_blocked_serial,  # noqa: E402
                      generate_spd, residual_norm, select_grid_dim, solve_with_factor)
from bandchol.reference import factor_reference  # noqa: E402

from paper_2305_04635_b200.inputs import generate_spd_wide, make_rhs  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def blocked_grid(k: int):
    for n in (3, 5, 6, 4, 9, 11):
        if k >= 2 and k % (n - 1) == 0:
            return n
    return None


def sample_columns(n: int, count: int = 16) -> np.ndarray:
    cols = set(np.linspace(0, n - 1, count).astype(int).tolist())
    cols.update([1, 2, n - 2, n // 2 + 1])
    return np.array(sorted(c for c in cols if 0 <= c < n), dtype=np.int64)


def small_cases():
    cases = []
    hand = BandedMatrix(2, 1)
    hand.set(0, 0, 4.0); hand.set(1, 0, 2.0); hand.set(1, 1, 5.0)
    cases.append(("hand_2x2", hand, 0))
    ident = BandedMatrix(30, 4)
    for i in range(30):
        ident.set(i, i, 1.0)
    cases.append(("identity_30_4", ident, 0))
    for (n, k, seed) in [(1, 0, 0), (2, 1, 0), (3, 2, 1), (17, 5, 2), (80, 13, 3), (300, 32, 4),
                         (50, 3, 11), (120, 8, 5), (64, 8, 0), (257, 50, 1), (257, 100, 2),
                         (1000, 2, 0), (150, 9, 5), (200, 7, 3), (333, 33, 4), (64, 0, 1),
                         (500, 1, 2), (129, 64, 6), (97, 96, 7), (400, 16, 2)]:
        cases.append((f"spd_{n}_{k}_{seed}", generate_spd(n, k, seed), seed))
    # padded lead dimension (lead_dim > k+1): padding must stay untouched
    base = generate_spd(100, 7, 9)
    wide = BandedMatrix(100, 7, lead_dim=12)
    wide.panel[:8, :] = base.band_panel()
    cases.append(("spd_100_7_9_ld12", wide, 9))
    return cases


def main():
    t0 = time.time()
    arrays = {}
    meta = {"reference_version": bandchol.__version__, "cases": {}}
    for name, a, seed in small_cases():
        n, k, ld = a.dim, a.bandwidth, a.lead_dim
        L = factor_reference(a.copy()).factor
        rhs = make_rhs(n, seed)
        x = solve_with_factor(L, rhs)
        arrays[f"{name}/A"] = a.data.copy()
        arrays[f"{name}/L_ref"] = L.data.copy()
        arrays[f"{name}/rhs"] = rhs
        arrays[f"{name}/x"] = x
        entry = {"n": n, "k": k, "lead_dim": ld, "seed": seed,
                 "residual": residual_norm(a, L)}
        g = blocked_grid(k)
        if g is not None and ld == k + 1:
            Lb = factor_blocked_serial(a.copy(), g)
            arrays[f"{name}/L_blocked"] = Lb.data.copy()
            entry["blocked_grid"] = g
        meta["cases"][name] = entry
    # failure columns (test_reference.py:76-82, test_parallel.py:60-74)
    fails = {}
    for col in (0, 4, 11):
        a = generate_spd(20, 3, seed=1)
        a.set(col, col, -1.0)
        arrays[f"fail_20_3_{col}/A"] = a.data.copy()
        try:
            factor_reference(a.copy())
            fails[f"fail_20_3_{col}"] = None
        except NotPositiveDefinite as e:
            fails[f"fail_20_3_{col}"] = {"n": 20, "k": 3, "column": e.column}
    a = generate_spd(60, 6, seed=5)
    a.set(41, 41, -5.0)
    a.set(53, 53, -5.0)
    arrays["fail_60_6_41_53/A"] = a.data.copy()
    try:
        factor_reference(a.copy())
    except NotPositiveDefinite as e:
        fails["fail_60_6_41_53"] = {"n": 60, "k": 6, "column": e.column}
    a = generate_spd(40, 4, seed=8)
    a.set(17, 17, -1.0)
    arrays["fail_40_4_17/A"] = a.data.copy()
    try:
        factor_blocked_serial(a.copy(), 3)
    except NotPositiveDefinite as e:
        fails["fail_40_4_17"] = {"n": 40, "k": 4, "column": e.column}
    meta["failures"] = fails
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **arrays)
    print(f"small cases done {time.time() - t0:.1f}s", flush=True)

    # config-sized fingerprints of the exactly-rounded reference factor
    fp = {}
    for tag, (n, k, seed) in {"C1": (2000, 50, 0), "n2000_k100": (2000, 100, 0),
                              "C5_s0": (4096, 100, 0), "C5_s1": (4096, 100, 1),
                              "C5_s2": (4096, 100, 2), "C5_s1023": (4096, 100, 1023),
                              "C2": (20000, 200, 0)}.items():
        a = generate_spd(n, k, seed)
        L = factor_reference(a.copy()).factor
        fp[tag] = {"n": n, "k": k, "seed": seed, "sha_A": sha(a.data), "sha_L_ref": sha(L.data),
                   "residual": residual_norm(a, L)}
        print(tag, f"{time.time() - t0:.1f}s", flush=True)
    meta["fingerprints"] = fp

    # reference blocked engine on the large configs: sampled columns + solves
    large = {}
    for tag, (n, k, seed, wide) in {"C2": (20000, 200, 0, False), "C3": (50000, 500, 0, True),
                                    "C4": (20000, 2000, 0, False)}.items():
        a = (generate_spd_wide if wide else generate_spd)(n, k, seed)
        if wide:
            a = BandedMatrix(n, k, data=a.data)  # reference type for the reference engine
        grid = select_grid_dim(k, 8)
        L = factor_blocked_serial(a.copy(), grid)
        cols = sample_columns(n)
        ld = k + 1
        large[f"{tag}/cols"] = cols
        large[f"{tag}/L_blocked_cols"] = np.stack([L.data[c * ld:(c + 1) * ld] for c in cols])
        large[f"{tag}/A_cols"] = np.stack([a.data[c * ld:(c + 1) * ld] for c in cols])
        meta.setdefault("large", {})[tag] = {"n": n, "k": k, "seed": seed, "grid": grid,
                                             "wide_diagonal": wide, "sha_A": sha(a.data)}
        if tag == "C2":
            rhs = make_rhs(n, seed)
            large["C2/x"] = solve_with_factor(L, rhs)
        print(tag, "blocked", f"{time.time() - t0:.1f}s", flush=True)
    for seed in (0, 1, 2, 1023):
        a = generate_spd(4096, 100, seed)
        L = factor_blocked_serial(a.copy(), 3)
        large[f"C5_s{seed}/x"] = solve_with_factor(L, make_rhs(4096, seed))
    np.savez_compressed(os.path.join(HERE, "sampled_large.npz"), **large)
    with open(os.path.join(HERE, "fingerprints.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print(f"done {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
