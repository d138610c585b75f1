"""e2e pipeline depth sweep: BatchedBandSolver.factor_solve on the C5 batch (pinned host)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2305_04635_b200 as bc  # noqa: E402
from paper_2305_04635_b200.inputs import generate_spd, make_rhs  # noqa: E402

n, k, B = 4096, 100, 1024
base = np.stack([generate_spd(n, k, s).data for s in range(16)])
ab = bc.pinned_empty((B, (k + 1) * n))
b = bc.pinned_empty((B, n))
for ch in [int(c) for c in sys.argv[1:]] or [4, 8, 16, 32]:
    solver = bc.BatchedBandSolver(B, n, k, chunks=ch)
    ts = []
    for it in range(4):
        ab[:] = np.tile(base, (B // 16, 1))
        b[:] = 1.0
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        solver.factor_solve(ab, b, check=False)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print({"chunks": ch, "ms": [round(t * 1e3, 1) for t in ts]}, flush=True)
