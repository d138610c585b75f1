"""Pinned host <-> device copy bandwidth, one direction and both at once (the ceiling of the
e2e path: 3.42 GB in and 3.42 GB out per C5 step)."""
import json
import time

import torch

n = 3422552064 // 8
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t


def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


for _ in range(2):
    th = timed(lambda: d_a.copy_(h_in, non_blocking=True))
    td = timed(lambda: h_out.copy_(d_b, non_blocking=True))
    tb = timed(both)
gb = n * 8 / 1e9
print(json.dumps({"bytes_each_way": n * 8, "h2d_gbs": gb / th, "d2h_gbs": gb / td, "both_ms": tb * 1e3,
                  "both_gbs_each": gb / tb}))
