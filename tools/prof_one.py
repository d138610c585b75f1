"""Run one config's factorization `reps` times (for ncu / compute-sanitizer captures).

usage: python tools/prof_one.py C1|C2|C3|C4|C5 [reps] [batch]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_04635_b200 as bc  # noqa: E402
from paper_2305_04635_b200.inputs import CONFIGS, generate_spd, generate_spd_wide, make_rhs  # noqa: E402

tag = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = CONFIGS[tag]
n, k = cfg.dim, cfg.bandwidth
if tag == "C5":
    batch = int(sys.argv[3]) if len(sys.argv) > 3 else 296
    a = np.stack([generate_spd(n, k, s).data for s in range(min(batch, 32))])
    a = np.concatenate([a] * ((batch + 31) // 32))[:batch]
    b = np.stack([make_rhs(n, s) for s in range(batch)])
    a0, b0 = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    for _ in range(reps):
        w, wb = a0.clone(), b0.clone()
        info = bc.dpbsv_batched_device(w, n, k, k + 1, wb, batch)
        torch.cuda.synchronize()
        assert int(info.abs().sum().item()) == 0
else:
    gen = generate_spd_wide if cfg.wide_diagonal else generate_spd
    a0 = torch.from_numpy(gen(n, k, 0).data).cuda()
    for _ in range(reps):
        w = a0.clone()
        info = bc.dpbtrf_device(w, n, k, k + 1)
        torch.cuda.synchronize()
        assert int(info.item()) == 0
print("ok", tag)
