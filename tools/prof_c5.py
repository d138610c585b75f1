"""One dpbtrf_batched launch on `batch` C5-shaped matrices (for ncu)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_04635_b200 as bc  # noqa: E402
from paper_2305_04635_b200.inputs import generate_spd  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 148
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
n, k = 4096, 100
a = np.stack([generate_spd(n, k, s).data for s in range(8)])
a = np.concatenate([a] * ((batch + 7) // 8))[:batch]
a0 = torch.from_numpy(a).cuda()
solve = len(sys.argv) > 3 and sys.argv[3] == "solve"
b0 = torch.from_numpy(np.stack([np.linspace(-1, 1, n)] * batch)).cuda()
for _ in range(reps):
    w = a0.clone()
    wb = b0.clone()
    info = (bc.dpbsv_batched_device(w, n, k, k + 1, wb, batch) if solve
            else bc.dpbtrf_batched_device(w, n, k, k + 1, batch))
    torch.cuda.synchronize()
    assert int(info.abs().sum().item()) == 0
print("ok")
