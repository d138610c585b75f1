"""Run the streamed batched solve `reps` times (for ncu captures).

usage: python tools/prof_solve.py [batch] [nrhs] [reps]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_04635_b200 as bc  # noqa: E402
from paper_2305_04635_b200.inputs import generate_spd, make_rhs  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 296
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
n, k = 4096, 100
a = generate_spd(n, k, 0)
bc.factor_blocked_serial(a)
ab = torch.from_numpy(a.data).cuda().repeat(batch)
b0 = torch.from_numpy(np.stack([make_rhs(n, s) for s in range(nrhs)])).cuda().repeat(batch, 1)
for _ in range(reps):
    b = b0.clone()
    info = bc.dpbtrs_batched_device(ab, n, k, k + 1, b, batch, nrhs=nrhs)
    torch.cuda.synchronize()
    assert int(info.abs().sum().item()) == 0
print("ok", batch, nrhs)
